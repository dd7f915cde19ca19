/*
 * vd.h -- C ABI of libvd, the B200 (sm_100a) implementation of the data-parallel hot path
 * of arXiv 2209.00117, "GPU Voronoi Diagrams for Random Moving Seeds" (dJFA).
 *
 * Citations: "P:n" = line n of the paper's LaTeX source; "R-n" = a reading of
 * an ambiguous passage, listed in DESIGN.md §3.
 *
 * The calls follow the paper's problem statement: a Voronoi diagram VD over an N x N
 * pixel grid X with seed set S = {P_1 .. P_s}, built once by the Jump Flooding
 * Algorithm and then advanced one simulation step at a time by dJFA
 * (Algorithm 1: Data VD, S, A -> Result VD), compared with Eq. 5.
 *
 * Data layout (all device-resident, owned by the handle):
 *   label   uint32, (y << 16) | x of the claimed seed's CURRENT position (R-1);
 *           EMPTY = 0xFFFFFFFF (R-4).  At N = 65536 the pixel (65535,65535) is reserved.
 *   diagram row-major N x N labels, rows padded to a pitch that is a multiple of 32
 *           labels (128 B); two ping-pong buffers (gather passes, R-12).
 *   seeds   uint32 labels [s]; plus a direct-mapped forward map used by dJFA (N x 65536, indexed
 *           by the label itself, where a frame fuses its remap into the first pass; else N x N).
 * Host arrays crossing the ABI are dense (no pitch): seeds_xy / disp_xy are interleaved
 * x0,y0,x1,y1,...; label maps are N*N row-major (or the rank's band of rows).
 *
 * Ownership: input pointers are borrowed for the duration of the call and copied
 * (a pointer may be host memory -- pageable or pinned -- or device memory; the library
 * asks the driver which).  Output pointers are caller-allocated host memory.
 *
 * Synchrony: vd_jfa, vd_move_seeds and vd_djfa_step only enqueue work on the handle's
 * stream and return.  Calls that return data (vd_similarity*, vd_label_hash, vd_get_*,
 * vd_pass_timing) synchronise the stream.  A handle is not thread-safe; distinct handles
 * are independent.
 *
 * Errors: no exception crosses the ABI.  Every entry point returns a vd_status; a CUDA or
 * NCCL failure is sticky (every later call on that handle returns it).  vd_last_error
 * gives a human-readable message.
 *
 * Multi-GPU (row bands): world > 1 splits the rows into `world`
 * contiguous bands of N/world rows, one per rank (one process per GPU); every jump pass
 * first exchanges width-k halos with the ranks that own rows y +- k through NCCL
 * point-to-point calls on the handle's stream.  Results are bit-identical for any world
 * size (the per-pixel minimum does not depend on where the pixel is computed).
 * virtual_shards > 1 runs the same banded code path inside ONE handle on one GPU,
 * exchanging halos with device-to-device copies -- used to test the band path where only
 * one GPU is available.
 */
#ifndef VD_H
#define VD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vd_ctx* vd_handle;
typedef int32_t vd_status;

enum {
    VD_OK = 0,
    VD_ERR_ARG = -1,   /* invalid argument (sizes, NULL, mismatched handles)            */
    VD_ERR_RANGE = -2, /* seed outside [0,N)^2, or the reserved pixel at N = 65536     */
    VD_ERR_STATE = -3, /* call out of order (e.g. vd_djfa_step before any diagram)     */
    VD_ERR_CUDA = -4,  /* CUDA runtime error (sticky)                                  */
    VD_ERR_NCCL = -5,  /* NCCL error or NCCL unavailable (sticky)                      */
    VD_ERR_OOM = -6    /* device or host allocation failed                             */
};

#define VD_EMPTY 0xFFFFFFFFu
#define VD_METRIC_EUCLIDEAN 0u
#define VD_METRIC_MANHATTAN 1u
#define VD_PASS_VON_NEUMANN 1u

typedef struct {
    int32_t device;         /* CUDA ordinal; -1 = the calling thread's current device      */
    void* stream;           /* cudaStream_t to run on; NULL = the handle creates its own    */
    int32_t rank, world;    /* row-band sharding across processes; world = 1: single GPU    */
    const void* nccl_id;    /* 128-byte ncclUniqueId (from vd_nccl_unique_id on rank 0),
                               required when world > 1                                     */
    uint32_t extra_passes;  /* trailing k = 1 passes after JFA / dJFA schedules (P:114,
                               P:150 "An extra step may be included"); default 0 (R-6)     */
    uint32_t virtual_shards;/* > 1: emulate that many row bands in this handle (world = 1) */
    uint32_t metric;        /* VD_METRIC_EUCLIDEAN (default, dJFAe) or VD_METRIC_MANHATTAN
                               (dJFAm); used by every pass of the handle         */
    uint32_t vn_waves;      /* the first vn_waves passes of each vd_djfa_step use the Von
                               Neumann neighbourhood (the 4 axis offsets of Table 1), the
                               rest Moore ("Von Neumann for the first two
                               waves"); default 0 = Moore only                              */
    uint32_t jfa_vn_waves;  /* same for vd_jfa (Fig. 5 / P:163-168: Von Neumann-only JFA)   */
    uint32_t peer_halos;    /* 1: halo rows for the next pass are pushed by the pass kernels
                               straight into the neighbouring bands' halo buffers (NEXT-3).
                               virtual_shards: immediate; world > 1: after vd_peer_attach, and
                               then nccl_id may be NULL (only steps with 2k < band rows run) */
    uint32_t reserved[2];   /* must be zero                                                */
} vd_config;

/* Fill *cfg with defaults: device -1, stream NULL, rank 0, world 1, no extras,
 * Euclidean metric, Moore neighbourhood. */
void vd_config_init(vd_config* cfg);

/* Write a fresh 128-byte ncclUniqueId to out128 (rank 0 calls it, then broadcasts the
 * bytes to the other ranks, e.g. with torch.distributed).  VD_ERR_NCCL if NCCL cannot be
 * loaded. */
vd_status vd_nccl_unique_id(void* out128);

/* Create a diagram context for an N x N grid and s seeds at seeds_xy (x0,y0,x1,y1,...;
 * host or device).  2 <= N <= 65536; 1 <= s <= N*N; seeds inside
 * [0,N)^2 and not the reserved pixel (65535,65535) at N = 65536 (R-4), else VD_ERR_RANGE.
 * Co-located seeds are allowed.  world > 1 requires N a power of two divisible by
 * world.  No diagram exists until vd_jfa. */
vd_status vd_create(vd_handle* out, uint32_t N, uint64_t s, const uint16_t* seeds_xy,
                    const vd_config* cfg);

/* Full JFA on the current seeds: all pixels EMPTY, each seed pixel <- its own
 * label, then passes k = 2^(ceil(log2 N)-1), ..., 1 (Eq. 2; R-5) plus
 * extra_passes k = 1 passes, each out[p] = argmin over {in[p]} U {in[p + o*k] : o in
 * Table 1, inside the grid} of the key (d2(p, c), c) (R-2, R-3, R-11). */
vd_status vd_jfa(vd_handle h);

/* Standard Flooding (Fig. 2a): the JFA initialisation, then k = 1 Moore passes
 * (with the handle's metric) until no pixel is EMPTY -- the grid is "fully flooded"
 * (reading R-22).  *passes (optional) gets the number of passes.  Synchronises once per
 * pass (the stopping test reads an EMPTY count back). */
vd_status vd_stf(vd_handle h, uint32_t* passes);

/* SimulateParticles (Alg. 1) only: new = clamp(old + disp) per axis (R-10; at
 * N = 65536 a seed landing on (65535,65535) goes to (65534,65535), R-4).  disp_xy: s
 * int16 pairs, host or device.  Leaves the diagram stale (use before vd_jfa for the JFA
 * baseline of the same frame). */
vd_status vd_move_seeds(vd_handle h, const int16_t* disp_xy);

/* One dJFA time step (Alg. 1 body): move the seeds as vd_move_seeds, then
 * reuse VD_{t-1} (R-9): every label follows its seed to the new position
 * (co-located seeds: the smallest new label wins), each new seed pixel is re-stamped,
 * then passes delta_1, ..., 1 with delta_1 = 2^ceil(log2(max(2 L_avg, d_max))),
 * L_avg = sqrt(N^2/s) (Eq. 3-4; exact integer form R-7, capped at JFA's k_1),
 * plus extra_passes.  Requires a diagram (vd_jfa first): else VD_ERR_STATE.  d_max is
 * the motion bound of the model; it must bound |disp| for the diagram to be
 * complete, but the library does not check the displacements against it. */
vd_status vd_djfa_step(vd_handle h, const int16_t* disp_xy, uint32_t d_max);

/* vd_djfa_step followed by vd_label_hash_async, with the checksum accumulated by the step's last
 * jump pass where it can (Euclidean Moore step 1 on grids with N % 512 == 0; else a separate
 * label_hash kernel): *pinned_out (pinned host memory) receives the new diagram's vd_label_hash
 * when the handle's stream reaches that point; the call itself only enqueues.  Summed over
 * ranks when world > 1.  Errors as vd_djfa_step; VD_ERR_ARG if pinned_out is NULL. */
vd_status vd_djfa_step_hash(vd_handle h, const int16_t* disp_xy, uint32_t d_max, uint64_t* pinned_out);

/* Replace the current diagram with a host label map (N*N dense; this rank's band when
 * world > 1).  Every label must be EMPTY or an in-grid position (else VD_ERR_RANGE; the
 * reserved pixel is EMPTY itself at N = 65536).  Afterwards the handle holds "a diagram"
 * (vd_djfa_step is allowed) iff no label is EMPTY; the caller then guarantees every label
 * is a current seed position, as after vd_jfa.  Synchronises. */
vd_status vd_set_labels(vd_handle h, const uint32_t* labels);

/* Peer halos across processes (NEXT-3; SURVEY section 8(e) "device-initiated halo exchange").
 * Each rank exports CUDA IPC handles of its halo buffers and flag words (vd_peer_export: writes
 * *len = blob size bytes to out when cap suffices; out = NULL only queries *len), the caller
 * all-gathers the blobs in rank order (e.g. torch.distributed.all_gather_object) and every rank
 * calls vd_peer_attach(h, blobs, len) once before its next pass.  From then on a pass with
 * 2k < B rows stores the rows its neighbours' next pass needs straight into their halo buffers
 * from inside the pass kernel, and publishes a per-pass sequence number into their flag words
 * (st.release.sys); the next pass's edge strips start after a device-side acquire wait.  The
 * first pass of each call copies its edge rows the same way (push_rows).  A wait that does not
 * complete within ~20 s sets a sticky flag readable with vd_peer_status (no hang). */
vd_status vd_peer_export(vd_handle h, void* out, size_t cap, size_t* len);
vd_status vd_peer_attach(vd_handle h, const void* blobs, size_t len_each);
vd_status vd_peer_status(vd_handle h, uint32_t* timed_out);

/* One jump pass with step k >= 1 on the current diagram (the body of every JFA / dJFA
 * wave, in gather form R-12), including the halo exchange when sharded, with
 * the handle's metric.  flags: VD_PASS_VON_NEUMANN = only the 4 axis neighbours
 * (P:154-160), else the Moore 8 of Table 1.  Powers of two use the fast kernel; any
 * other k the generic one (same results).  On a handle holding a diagram (no EMPTY, as
 * after vd_jfa / vd_djfa_step / a complete vd_set_labels, world == 1) the EMPTY-free
 * kernels run, including the windowed one for 32768 < N <= 65536, k <= 4096. */
vd_status vd_pass(vd_handle h, uint32_t k, uint32_t flags);

/* Eq. 5: 100 * matching pixels / total pixels between the diagrams of h and
 * ref (same N and sharding; ref may be h).  *matches (optional) gets the integer count.
 * With world > 1 the count is summed over ranks (every rank gets the total). */
vd_status vd_similarity(vd_handle h, vd_handle ref, double* pct, uint64_t* matches);

/* Eq. 5 against a host label map (N*N dense, or this rank's band when world > 1:
 * rows [band_row0, band_row0 + band_rows) of vd_band). */
vd_status vd_similarity_host(vd_handle h, const uint32_t* ref_labels, double* pct,
                             uint64_t* matches);

/* Order-independent checksum of the current diagram: sum over pixels p = y*N + x of
 * fmix32((uint32)(p * 0x9E3779B9) ^ label[p]) in uint64 (fmix32 = MurmurHash3's 32-bit
 * finaliser; summed over ranks when world > 1).  Reads the whole diagram once and returns
 * 8 bytes; used as the per-step result read-back. */
vd_status vd_label_hash(vd_handle h, uint64_t* out);
/* Same checksum, enqueued on the handle's stream without waiting: the value lands in
 * *pinned_out (page-locked host memory: cudaHostAlloc / cudaHostRegister / torch pin_memory)
 * once the stream reaches it, i.e. after vd_synchronize or any later synchronising call. Lets
 * a time-stepping loop read each step's result without a host round trip per step. */
vd_status vd_label_hash_async(vd_handle h, uint64_t* pinned_out);

/* Copy the diagram to host: N*N labels (world = 1, any virtual_shards), or this rank's
 * band_rows*N labels (world > 1). */
vd_status vd_get_labels(vd_handle h, uint32_t* out);

/* Copy the current seed positions (x0,y0,...) to host. */
vd_status vd_get_seeds(vd_handle h, uint16_t* out_xy);

/* This handle's rows: [*row0, *row0 + *rows). */
vd_status vd_band(vd_handle h, uint32_t* row0, uint32_t* rows);

/* Number of jump passes in the last vd_jfa / vd_djfa_step. */
vd_status vd_last_passes(vd_handle h, uint32_t* passes);

/* How many passes of the last vd_jfa / vd_djfa_step ran the packed-key evaluation (a pass
 * whose input labels all lie within Euclidean distance 63 of their pixels, with k <= 64:
 * one 31-bit key (d2, dy, dx) per candidate, same result as the lexicographic key of Table 1 /
 * P:112 with the (d2, label) tie-break).  The locality of each pass's input is decided on the
 * device by the kernel that wrote it (remap, or the previous pass); this call synchronises
 * the handle's stream to read those flags.  Tracked for Moore passes with either metric (not
 * Von Neumann waves; 0 with env VD_NO_PACK=1).  Sharded: a band's flag covers its own rows only, so there the
 * count is of passes whose interior launch (rows that read no halo) ran packed; the edge
 * strips keep the exact evaluation. */
vd_status vd_last_packed_passes(vd_handle h, uint32_t* passes);

/* Wait for all work enqueued on the handle's stream. */
vd_status vd_synchronize(vd_handle h);

/* Instrumentation: when enabled, CUDA events are recorded around every jump-pass launch
 * on the handle's stream; vd_pass_timing returns the summed device time (ms) of the jump
 * passes, their number and the pixels they covered, then resets the accumulators. */
vd_status vd_set_pass_timing(vd_handle h, int enable);
vd_status vd_pass_timing(vd_handle h, double* ms, uint64_t* launches, uint64_t* pixels);
/* The timed intervals accumulated since the last vd_pass_timing, one per jump pass (all of
 * its launches): device time ms[i] and step ks[i], for i < min(*n, cap); *n = how many
 * there are.  A vd_djfa_step's remap is also an interval, with ks[i] = 0 (it covers no
 * pass pixels).  Does not reset (vd_pass_timing does).  ms / ks may be NULL. */
vd_status vd_pass_times(vd_handle h, float* ms, uint32_t* ks, uint32_t cap, uint32_t* n);

/* Number of kernels this handle has launched since creation. */
vd_status vd_launch_count(vd_handle h, uint64_t* n);

/* Host-only helpers (no GPU needed). */
/* Eq. 2 k-list (+ extras) into ks[0..*n); VD_ERR_ARG if cap is too small or N < 2. */
vd_status vd_schedule_jfa(uint32_t N, uint32_t extras, uint32_t* ks, uint32_t cap, uint32_t* n);
/* Eq. 4 delta-list (+ extras), exact integer form R-7. */
vd_status vd_schedule_djfa(uint32_t N, uint64_t s, uint32_t d_max, uint32_t extras,
                           uint32_t* ks, uint32_t cap, uint32_t* n);

/* Halo plan of one pass with step k for rank `rank` of `world` row bands of N/world rows
 * (SURVEY.md §8(e)).  With B = N/world, d = ceil(k/B), h = min(k, B):
 *   recv_top_rank = rank - d (or -1): its rows [B-h, B) land in the top halo, which holds
 *                   global rows [top_row0, top_row0 + h), top_row0 = rank*B - k;
 *   recv_bot_rank = rank + d (or -1): its rows [0, h) land in the bottom halo, which holds
 *                   global rows [bot_row0, bot_row0 + h), bot_row0 = rank*B + d*B;
 *   this rank sends its rows [0, h) to recv_top_rank and rows [B-h, B) to recv_bot_rank.
 * Every pixel of the band needs exactly these rows and no others. */
typedef struct {
    int32_t recv_top_rank, recv_bot_rank; /* -1: none (grid edge)                     */
    uint32_t halo_rows;                   /* h                                        */
    int64_t top_row0, bot_row0;           /* global row of halo row 0                 */
    uint32_t send_top_row0;               /* first local row sent to recv_top_rank (0) */
    uint32_t send_bot_row0;               /* first local row sent to recv_bot_rank    */
} vd_halo_plan_t;
vd_status vd_halo_plan(uint32_t N, uint32_t world, uint32_t rank, uint32_t k, vd_halo_plan_t* out);

/* Destroy (NULL-safe).  Frees every device buffer the handle owns. */
void vd_destroy(vd_handle h);

const char* vd_status_str(vd_status s);
const char* vd_last_error(vd_handle h);

#ifdef __cplusplus
}
#endif
#endif /* VD_H */
