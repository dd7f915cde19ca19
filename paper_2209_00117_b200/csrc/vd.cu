// vd.cu -- libvd: host runtime + C ABI (include/vd.h) of the B200 dJFA hot path.
//
// One handle = one diagram on one GPU (or one rank's row band).  The handle owns every
// device buffer; work is enqueued on one CUDA stream (the caller's, e.g. torch's current
// stream, or its own).  Multi-GPU halo exchange uses NCCL point-to-point calls, loaded
// at run time with dlopen (the library itself does not link NCCL).
//
// "P:n" = line n of the paper's LaTeX source; "R-n" = reading n in DESIGN.md §3.
#include <cuda.h>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled (fetched with cudaGetDriverEntryPoint)
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX: ranges per frame and per pass (no-ops unless a tool attaches)

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/vd.h"
#include "vd_kernels.cuh"
#include "vd_launch.h"

namespace {

// ------------------------------------------------------------------ NCCL (dlopen)
struct Nccl {
  bool tried = false, ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};
Nccl g_nccl;

bool nccl_load() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { g_nccl.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror(); return false; }
#define VD_SYM(field, name)                                                   \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));    \
  if (!g_nccl.field) { g_nccl.err = std::string("missing symbol ") + name; return false; }
  VD_SYM(GetUniqueId, "ncclGetUniqueId");
  VD_SYM(CommInitRank, "ncclCommInitRank");
  VD_SYM(CommDestroy, "ncclCommDestroy");
  VD_SYM(GroupStart, "ncclGroupStart");
  VD_SYM(GroupEnd, "ncclGroupEnd");
  VD_SYM(Send, "ncclSend");
  VD_SYM(Recv, "ncclRecv");
  VD_SYM(AllReduce, "ncclAllReduce");
  VD_SYM(GetErrorString, "ncclGetErrorString");
  VD_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
  VD_SYM(CommAbort, "ncclCommAbort");
#undef VD_SYM
  g_nccl.ok = true;
  return true;
}

// NVTX range for the lifetime of a scope: "vd_jfa", "vd_djfa_step", "pass k=..." (profilers
// such as nsys / ncu --nvtx show the host-side enqueue structure of a frame).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------------ schedules (host)
uint32_t ceil_log2_u64(uint64_t n) {
  uint32_t e = 0;
  while ((1ull << e) < n) ++e;
  return e;
}

// Eq. 2, R-5: k_1 = 2^(ceil(log2 N) - 1), halving to 1, + extras (R-6).
int schedule_jfa(uint32_t N, uint32_t extras, std::vector<uint32_t>& ks) {
  ks.clear();
  if (N < 2) return -1;
  for (uint32_t k = 1u << (ceil_log2_u64(N) - 1); k >= 1; k >>= 1) ks.push_back(k);
  for (uint32_t i = 0; i < extras; ++i) ks.push_back(1);
  return 0;
}

// Eq. 3-4 in exact integers (R-7): delta_1 = 2^e with
// e = min(max(e_L, e_d), log2 k_1), e_L = min{e : s 4^e >= 4 N^2}, e_d = ceil(log2 d_max).
int schedule_djfa(uint32_t N, uint64_t s, uint32_t d_max, uint32_t extras, std::vector<uint32_t>& ks) {
  ks.clear();
  if (N < 2 || s == 0) return -1;
  const unsigned __int128 target = (unsigned __int128)4 * N * N;
  uint32_t eL = 0;
  while (((unsigned __int128)s << (2 * eL)) < target) ++eL;
  const uint32_t ed = d_max <= 1 ? 0 : ceil_log2_u64(d_max);
  uint32_t e = std::max(eL, ed);
  e = std::min(e, ceil_log2_u64(N) - 1);
  for (int i = (int)e; i >= 0; --i) ks.push_back(1u << i);
  for (uint32_t i = 0; i < extras; ++i) ks.push_back(1);
  return 0;
}

void halo_plan(uint32_t N, uint32_t world, uint32_t rank, uint32_t k, vd_halo_plan_t& p) {
  const uint32_t B = N / world;
  const uint32_t d = (k + B - 1) / B;
  const uint32_t h = std::min(k, B);
  p.halo_rows = h;
  p.recv_top_rank = (int64_t)rank - (int64_t)d >= 0 ? (int32_t)(rank - d) : -1;
  p.recv_bot_rank = (uint64_t)rank + d < world ? (int32_t)(rank + d) : -1;
  p.top_row0 = (int64_t)rank * B - (int64_t)k;
  p.bot_row0 = (int64_t)rank * B + (int64_t)d * B;
  p.send_top_row0 = 0;
  p.send_bot_row0 = B - h;
}

constexpr uint32_t kLocSlots = 64;  // locality flags per frame (>= passes + 2)
constexpr uint32_t kLocPrev = kLocSlots - 1;  // persistent: the current diagram's flag (0 = every label local)

struct Shard {
  uint32_t row0 = 0, rows = 0;
  uint32_t* buf[2] = {nullptr, nullptr};  // ping-pong diagrams, rows x pitch
  uint32_t* top[2] = {nullptr, nullptr};  // halo from the band above, hcap x pitch, by pass parity
  uint32_t* bot[2] = {nullptr, nullptr};  // halo from the band below
};

}  // namespace

struct vd_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint32_t N = 0;
  uint64_t s = 0;
  int64_t pitch = 0;
  int rank = 0, world = 1;
  uint32_t vshards = 1;
  uint32_t extras = 0;
  int metric = 0;           // 0 Euclidean (dJFAe), 1 Manhattan (dJFAm)
  uint32_t vn_waves = 0;    // Von Neumann waves at the start of each dJFA step
  bool force_rel = false;   // test hook (env VD_FORCE_WINDOWED=1): windowed kernel at any N
  bool force_wsk = false;   // test hook (env VD_FORCE_WSK=1): the wide exact pass at any N (its arithmetic holds for N <= 65536)
  bool track_empty = false; // jump_pass_wide reports EMPTY outputs into `counter` (vd_jfa)
  uint32_t jfa_vn_waves = 0;// ... and of each full JFA (Fig. 5)
  uint32_t hcap = 0;  // halo rows allocated per side
  std::vector<Shard> shards;
  int cur = 0;        // which ping-pong buffer holds the diagram
  bool has_diagram = false;
  uint32_t* seeds = nullptr;      // [s] current positions (labels)
  uint32_t* seeds_new = nullptr;  // [s] scratch for the move
  short2* disp_buf[2] = {nullptr, nullptr};  // [s] displacements on device, two slots
  int disp_slot = 0;
  cudaEvent_t disp_used[2] = {nullptr, nullptr};  // last kernel reading each slot done
  cudaStream_t copy_stream = nullptr;             // host -> device uploads
  cudaStream_t halo_stream = nullptr;             // halo exchange overlapped with interior rows
  cudaEvent_t halo_ready = nullptr, halo_done = nullptr;
  cudaEvent_t copy_done = nullptr;
  uint32_t* fwd = nullptr;        // forward map (dJFA), allocated on first use: [N x 65536] or [N x N]
  int fwd_pitch = 0;              // this frame's layout: 0 = indexed by the label itself; N = y N + x (vdk::fwd_index)
  bool fwd_fusable = false;       // fwd sized N x 65536 (a frame may fuse), else N x N
  uint32_t* bits = nullptr;       // 2 x [N * ceil(N/32)] occupancy bitmaps (JFA's sparse passes), allocated on first use
  unsigned long long* counter = nullptr;     // device u64 for reductions
  // Locality flags of one frame (packed-key pass, vd_kernels.cuh): loc[i] = 0 iff every label
  // of the input of the frame's i-th tracked pass lies within kLocR of its pixel.
  uint32_t* loc = nullptr;     // device u32[kLocSlots]
  bool loc_on = false;         // a JFA / dJFA frame is tracking locality
  bool loc_valid = false;      // loc[loc_idx] describes the current diagram
  uint32_t loc_idx = 0;
  std::vector<std::pair<int32_t, uint32_t>> loc_passes;  // per tracked pass: (loc slot of its input or -1, k)
  std::vector<std::pair<int32_t, uint32_t>> loc_last;    // ... of the last frame
  const uint32_t* pass_loc_in = nullptr;  // the running pass's input flag (null: unknown)
  uint32_t* pass_loc_out = nullptr;       // ... and output flag (null: not tracked)
  bool pass_loc_ok = false;               // every launch of the pass reported into pass_loc_out
  bool pass_loc_used = false;             // some launch of the pass could take the packed walk
  bool fuse_remap = false;                // the next pass remaps its staged rows (NEXT-1, jump_pass_sk_remap)
  bool fuse_pack = false;                 // ... and may take the packed walk (previous flag + move bound)
  bool in_djfa = false;                   // passes of a vd_djfa_step are running
  bool hash_pass = false;                 // the running pass also accumulates the label checksum
  bool lat_pass = false;                  // the running pass belongs to vd_jfa's schedule (lattice invariant holds)
  bool rst_pending = false;               // fwd[rst_seeds[i]] <- EMPTY still to do (folded into the next jump_pass_sk)
  const uint32_t* rst_seeds = nullptr;    // ... the old seed positions
  unsigned long long* counter_h = nullptr;   // pinned host copy
  uint32_t last_passes = 0;
  uint64_t launches = 0;
  vd_status sticky = VD_OK;
  std::string err;
  // instrumentation
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  std::vector<uint32_t> ev_k;  // step k of each timed interval
  size_t ev_used = 0;
  uint64_t timed_px = 0, timed_launches = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  // Peer halos (NEXT-3): the pass kernels push the rows the neighbours' next pass needs
  // straight into their halo buffers (peer memory via CUDA IPC across processes).
  bool peer = false;           // enabled (vshards: by config; world > 1: after vd_peer_attach)
  uint32_t hpar = 0;           // halo buffers read by the next pass: top[hpar] / bot[hpar]
  uint32_t pushed_k = 0;       // the previous pass pushed this step's halos (0: none)
  uint32_t pass_seq = 0;       // passes run (same on every rank): signal sequence numbers
  uint32_t* flags = nullptr;   // device u32[2]: seq published by the band above / below
  uint32_t* peer_err = nullptr;// device view of peer_err_h
  uint32_t* peer_err_h = nullptr;  // mapped pinned host u32: a peer wait timed out (checked by every call)
  uint32_t* nbr_bot[2] = {nullptr, nullptr};  // band above's bottom halos (peer pointers)
  uint32_t* nbr_top[2] = {nullptr, nullptr};  // band below's top halos
  uint32_t* nbr_flag_above = nullptr;         // band above's flags[1]
  uint32_t* nbr_flag_below = nullptr;         // band below's flags[0]
  std::vector<void*> ipc_opened;
};

namespace {

// Locality tracking for one JFA / dJFA frame on one band (packed-key passes, vd_kernels.cuh).
// Env VD_NO_PACK=1 turns it off (A/B timing and tests of the exact kernel).
bool loc_begin(vd_ctx* h) {
  static const bool off = [] { const char* e = getenv("VD_NO_PACK"); return e && e[0] == '1'; }();
  h->loc_on = !off;
  h->loc_idx = 0;
  h->loc_valid = false;
  h->loc_passes.clear();
  if (h->loc_on && cudaMemsetAsync(h->loc, 0, kLocPrev * sizeof(uint32_t), h->stream) != cudaSuccess)
    h->loc_on = false;
  return h->loc_on;
}
// The diagram changed outside a tracked frame (set_labels, a single pass, StF): its locality is
// unknown, which reads as "not local".
void loc_forget(vd_ctx* h) { cudaMemsetAsync(h->loc + kLocPrev, 0x01, sizeof(uint32_t), h->stream); }
// One pass: its input flag is the previous pass's output flag; all of its launches (one per
// shard, or interior + edge strips) OR into one output slot.
void loc_pass_begin(vd_ctx* h, uint32_t k) {
  h->pass_loc_in = nullptr;
  h->pass_loc_out = nullptr;
  h->pass_loc_ok = false;
  h->pass_loc_used = false;
  if (!h->loc_on || h->loc_idx + 2 >= kLocSlots) return;
  int32_t in_slot = h->loc_valid ? (int32_t)h->loc_idx : -1;
  if (h->fuse_remap) in_slot = h->fuse_pack ? (int32_t)kLocPrev : -1;  // the previous frame's flag
  h->pass_loc_in = in_slot >= 0 ? h->loc + in_slot : nullptr;
  h->pass_loc_out = h->loc + h->loc_idx + 1;
  h->pass_loc_ok = true;
  h->loc_passes.emplace_back(in_slot, k);
}
void loc_pass_end(vd_ctx* h) {
  if (h->pass_loc_out && !h->pass_loc_used) h->loc_passes.back().first = -1;  // no launch could pack
  if (h->pass_loc_out) ++h->loc_idx;
  h->loc_valid = h->pass_loc_out && h->pass_loc_ok;
  h->pass_loc_in = nullptr;
  h->pass_loc_out = nullptr;
}
void loc_end(vd_ctx* h) {
  // keep the frame's final flag for the next frame's fused first pass
  if (h->loc_on && h->loc_valid)
    cudaMemcpyAsync(h->loc + kLocPrev, h->loc + h->loc_idx, sizeof(uint32_t), cudaMemcpyDeviceToDevice, h->stream);
  else
    loc_forget(h);
  h->loc_on = h->loc_valid = false;
  h->loc_last.swap(h->loc_passes);
  h->loc_passes.clear();
}

vd_status fail(vd_ctx* h, vd_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) {
    if (st == VD_ERR_CUDA || st == VD_ERR_NCCL) h->sticky = st;
    h->err = buf;
  }
  return st;
}

#define CK(expr)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return fail(h, e_ == cudaErrorMemoryAllocation ? VD_ERR_OOM : VD_ERR_CUDA, \
                                       "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define CKN(expr)                                                                             \
  do {                                                                                        \
    ncclResult_t r_ = (expr);                                                                 \
    if (r_ != ncclSuccess) return fail(h, VD_ERR_NCCL, "%s: %s", #expr, g_nccl.GetErrorString(r_)); \
  } while (0)

// A peer-halo wait that timed out on the device (vdk::peer_wait) wrote 1 into mapped host
// memory: the halos of that pass were never received, so the diagram is wrong.  Every
// entry point turns it into a sticky error before doing anything else.
vd_status check_async(vd_ctx* h) {
  if (h->sticky != VD_OK) return h->sticky;
  if (h->peer_err_h && *(volatile uint32_t*)h->peer_err_h)
    return fail(h, VD_ERR_CUDA, "a peer-halo wait timed out on the device (neighbour never signalled)");
  return VD_OK;
}

#define CHECK_HANDLE(h)                                \
  do {                                                 \
    if (!(h)) return VD_ERR_ARG;                       \
    if (vd_status s_ = check_async(h)) return s_;      \
  } while (0)

// Row-sweep kernels (remap, match_count, label_hash, count_value): CTAs stride over rows.
int rows_grid(const vd_ctx* h, int64_t rows) { return (int)std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)h->num_sms * 8)); }

int grid_for(const vd_ctx* h, int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)h->num_sms * 32));
}

vd_status after_launch(vd_ctx* h, const char* what) {
  h->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, VD_ERR_CUDA, "launch %s: %s", what, cudaGetErrorString(e));
  return VD_OK;
}

// Wait for the handle's stream.  With an NCCL communicator, poll instead of blocking, so
// that a failed or stuck collective (a dead peer) becomes VD_ERR_NCCL rather than a hang:
// ncclCommGetAsyncError is checked while the stream is busy, and after VD_NCCL_TIMEOUT_S
// seconds (default 600) the communicator is aborted.
vd_status sync_stream(vd_ctx* h) {
  if (!h->comm) {
    CK(cudaStreamSynchronize(h->stream));
    return check_async(h);
  }
  static const double limit = [] {
    const char* e = getenv("VD_NCCL_TIMEOUT_S");
    return e ? atof(e) : 600.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  while (true) {
    const cudaError_t q = cudaStreamQuery(h->stream);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return fail(h, VD_ERR_CUDA, "stream: %s", cudaGetErrorString(q));
    ncclResult_t ar = ncclSuccess;
    if (g_nccl.CommGetAsyncError(h->comm, &ar) != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
      g_nccl.CommAbort(h->comm);
      h->comm = nullptr;
      return fail(h, VD_ERR_NCCL, "NCCL asynchronous error: %s", g_nccl.GetErrorString(ar));
    }
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
      g_nccl.CommAbort(h->comm);
      h->comm = nullptr;
      return fail(h, VD_ERR_NCCL, "NCCL: stream did not finish within %.0f s (VD_NCCL_TIMEOUT_S); communicator aborted",
                  limit);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  return check_async(h);
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Bring s displacement pairs (host or device) into one of two device slots and return it.
// Host data (pinned or pageable) is copied on a separate copy stream -- overlapping the
// kernels still running on the handle's stream -- after the previous reader of that slot
// (two calls ago) has finished; the call returns once the copy is complete (the caller may
// reuse its array), and the handle's stream waits for it.  Device data is copied on the
// handle's stream.  The caller records h->disp_used[slot] after the kernel reading it.
vd_status upload_disp(vd_ctx* h, const int16_t* disp_xy, const short2** dev, int* slot_out) {
  const size_t bytes = h->s * sizeof(short2);
  const int slot = h->disp_slot;
  h->disp_slot ^= 1;
  short2* dst = h->disp_buf[slot];
  if (is_device_ptr(disp_xy)) {
    CK(cudaMemcpyAsync(dst, disp_xy, bytes, cudaMemcpyDeviceToDevice, h->stream));
  } else {
    CK(cudaStreamWaitEvent(h->copy_stream, h->disp_used[slot], 0));
    CK(cudaMemcpyAsync(dst, disp_xy, bytes, cudaMemcpyHostToDevice, h->copy_stream));
    CK(cudaEventRecord(h->copy_done, h->copy_stream));
    CK(cudaEventSynchronize(h->copy_done));
    CK(cudaStreamWaitEvent(h->stream, h->copy_done, 0));
  }
  *dev = dst;
  *slot_out = slot;
  return VD_OK;
}

vd_status timed_begin(vd_ctx* h) {
  if (!h->timing) return VD_OK;
  while (h->ev.size() < h->ev_used + 2) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    h->ev.push_back(e);
  }
  CK(cudaEventRecord(h->ev[h->ev_used], h->stream));
  return VD_OK;
}
vd_status timed_end(vd_ctx* h, uint64_t px, uint32_t k) {
  if (!h->timing) return VD_OK;
  CK(cudaEventRecord(h->ev[h->ev_used + 1], h->stream));
  h->ev_k.resize(h->ev_used / 2 + 1);
  h->ev_k[h->ev_used / 2] = k;
  h->ev_used += 2;
  h->timed_px += px;
  h->timed_launches++;
  return VD_OK;
}

// Shared-term kernel (jump_pass_sk): one band or banded, Euclidean Moore, N % 512 == 0, and
// k in {1, 2} (adjacent columns) or 32 <= k <= N/4 (stride columns).  VD_NO_SK=1 disables it
// (A/B timing).
// VD_SK_MASK (hex bitmask over log2 k) selects the steps it takes, for A/B timing.
// Beyond N = 32768 it takes complete diagrams with k <= 64 (dJFA's passes): packed walk when the
// input is local, else exact 64-bit keys; the rest stays on the windowed / wide kernels.
bool sk_ok(const vd_ctx* h, uint32_t k, bool vn, bool may_empty) {
  static const bool off = [] { const char* e = getenv("VD_NO_SK"); return e && e[0] == '1'; }();
  static const uint64_t mask = [] { const char* e = getenv("VD_SK_MASK"); return e ? strtoull(e, nullptr, 16) : ~0ull; }();
  uint32_t lk = 0;
  while ((1u << lk) < k) ++lk;
  // beyond 32768 only inside dJFA frames, whose inputs are local (packed walk); JFA's passes there
  // are never local and keep the windowed exact walk, which beats 64-bit keys
  if (h->force_rel || (h->N > 32768 && (may_empty || k > (uint32_t)vdk::kPackMaxK || !h->in_djfa))) return false;
  if (h->force_wsk && k >= 256) return false;  // (test hook: those steps go to the wide pass)
  if (may_empty && h->N > 16384) return false;  // the virtual far seed needs 2N - 1 < 2^15 (as jump_pass_fast)
  return !off && ((mask >> lk) & 1) && !vn && h->metric == 0 && h->N % 512 == 0 && 4 * k <= h->N;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (libvd does not link libcuda).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Tensor map of one band's input viewed as [rows][N/k][k] (uint32), box {128, 6, 1}: one copy
// stages the six 128-column spans x0 + j k (j = -1..4) of a row (jump_pass_sk, k >= 256).
bool encode_span_map(const vd_ctx* h, const uint32_t* in, uint32_t rows, uint32_t k, CUtensorMap* tm) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {k, h->N / k, rows};
  const cuuint64_t strides[2] = {(cuuint64_t)k * 4, (cuuint64_t)h->pitch * 4};
  const cuuint32_t box[3] = {128, 6, 1}, es[3] = {1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(in), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Wide exact pass (jump_pass_wsk): grids beyond N = 32768 (33-bit squared distances), any labels,
// EMPTY allowed, Euclidean Moore, power-of-two 256 <= k <= N / 4, N % 512 == 0 (JFA's large steps
// at C5).  VD_NO_WSK=1 disables it (A/B against the windowed / 64-bit kernels).
bool wsk_ok(const vd_ctx* h, uint32_t k, bool vn) {
  static const bool off = [] { const char* e = getenv("VD_NO_WSK"); return e && e[0] == '1'; }();
  return !off && !h->force_rel && (h->N > 32768 || h->force_wsk) && h->N % 512 == 0 && h->metric == 0 && !vn && k >= 256 &&
         (k & (k - 1)) == 0 && 4 * k <= h->N;
}

bool fast_ok(uint32_t N, bool may_empty) { return may_empty ? N <= 16384 : N <= 32768; }
// Windowed fast pass (REL) for complete diagrams with 32768 < N <= 65536 and steps small
// enough that a walk and its neighbour rows fit the 32768-wide window (dJFA's delta passes,
// JFA's last 13 once no EMPTY is left).  Walks meeting far labels are recomputed exactly.
bool rel_ok(uint32_t N, bool may_empty, uint32_t k) { return !may_empty && !fast_ok(N, false) && k <= 4096; }

// One pass over output rows [y_lo, y_hi) of shard sh (global rows; default: the whole band).
struct Push {  // where a launch also stores the rows the neighbours' next pass needs
  uint32_t* top = nullptr;
  uint32_t* bot = nullptr;
  uint32_t k = 0;
};

uint32_t unclaimed_label(const vd_ctx* h);
vd_status launch_pass(vd_ctx* h, Shard& sh, uint32_t k, bool may_empty, bool vn, int64_t y_lo = -1,
                      int64_t y_hi = -1, const Push* push = nullptr) {
  vdk::PassArgs a;
  a.res_in_y = 0;
  a.nwalk = 0;
  a.tmap = 0;
  a.fwd = nullptr;
  a.prefetch = 0;
  a.hash_out = nullptr;
  a.rst_fwd = nullptr;
  a.rst_seeds = nullptr;
  a.rst_s = 0;
  a.lat = 0;
  a.lat_empty = VD_EMPTY;
  a.lat_min = h->N < 65536 ? h->N << 16 : VD_EMPTY;
  a.lat_vl = 0;
  a.in = sh.buf[h->cur];
  a.out = sh.buf[h->cur ^ 1];
  a.top = sh.top[h->hpar];
  a.bot = sh.bot[h->hpar];
  a.push_top = a.push_bot = nullptr;
  a.push_k = 0;
  if (push && push->k) {
    a.push_top = push->top;
    a.push_bot = push->bot;
    a.push_k = (int)push->k;
  }
  a.pitch = h->pitch;
  a.N = (int)h->N;
  a.row0 = (int)sh.row0;
  a.rows = (int)sh.rows;
  const uint32_t B = sh.rows;
  const uint32_t d = (k + B - 1) / B;
  a.top_row0 = (int)sh.row0 - (int)k;
  a.bot_row0 = (int)(sh.row0 + d * B);
  a.k = (int)k;
  a.xblocks = (int)((h->N + vdk::kW - 1) / vdk::kW);  // 512-column chunks (fast pass)
  const uint32_t C = 2 * h->N - 1;
  a.vempty = (C << 16) | C;
  a.sh16 = 65536u;
  a.one = 1u;
  a.metric = h->metric;
  a.vn = vn ? 1 : 0;
  a.empty_flag = h->track_empty ? h->counter : nullptr;
  a.loc_in = nullptr;
  a.loc_out = nullptr;
  if (y_lo < 0) { y_lo = (int64_t)sh.row0; y_hi = (int64_t)(sh.row0 + sh.rows); }
  a.y_lo = (int)y_lo;
  a.y_hi = (int)y_hi;
  const uint32_t R = (uint32_t)(y_hi - y_lo);  // output rows of this launch
  if (R == 0) return VD_OK;
  // JFA's lattice walk (jump_pass_sk LAT): a pass of vd_jfa's schedule (its input congruent to the
  // pixels mod 2k), Euclidean Moore, stride step k >= 4; lattice coordinates below 64 (N <= 64k), or
  // below 128 once no EMPTY is left (N <= 128k, the packed key's range).  Beyond N = 32768 only, where
  // it replaces the wide pass; below, the 32-bit exact walk is as fast (measured).
  // VD_NO_LAT=1 disables it, VD_LAT_ALL=1 also takes N <= 32768 (A/B).
  static const bool no_lat = [] { const char* e = getenv("VD_NO_LAT"); return e && e[0] == '1'; }();
  static const bool lat_all = [] { const char* e = getenv("VD_LAT_ALL"); return e && e[0] == '1'; }();
  uint32_t lk = 0;
  while ((1u << lk) < k) ++lk;
  const uint32_t lmax = (h->N - 1) >> lk;  // largest lattice coordinate
  const bool lat_geo = !no_lat && h->lat_pass && !vn && h->metric == 0 && (k & (k - 1)) == 0 && k >= 4 &&
                       4 * k <= h->N && h->N % 512 == 0 && !h->force_rel && (h->N > 32768 || lat_all);
  const bool no_unclaimed = !may_empty && h->N > 16384;  // (N <= 16384 runs on the virtual far seed)
  // 3: the exact 32-bit walk in lattice units (lattice coordinates < 2^14 for k >= 4), with the
  // unclaimed labels at (2L+1, 2L+1) like the virtual far seed; VD_NO_LATX=1 disables it (A/B)
  static const bool no_latx = [] { const char* e = getenv("VD_NO_LATX"); return e && e[0] == '1'; }();
  // (lat 3 only for k >= 256, where it replaces the wide pass: 12.3 -> 9.6 ms at C5's k = 256; for
  // k <= 128 the windowed walk stays, 0.3 ms faster, `profiles/r02c_latx_ab_c5.txt`)
  // 4: the same without unclaimed labels (C5's k = 128 ... 4 once EMPTY is gone; VD_NO_LAT4=1: the
  // windowed walk there instead, A/B)
  static const bool no_lat4 = [] { const char* e = getenv("VD_NO_LAT4"); return e && e[0] == '1'; }();
  const int lat_kind = !lat_geo ? 0 : lmax <= 63 ? (no_unclaimed ? 2 : 1) : (lmax <= 127 && no_unclaimed) ? 2
                     : no_latx ? 0 : (no_unclaimed && !no_lat4) ? 4 : k >= 256 ? 3 : 0;
  const bool lat = lat_kind > 0;
  const bool sk = lat || (sk_ok(h, k, vn, may_empty) && (k & (k - 1)) == 0);
  const bool wsk = !sk && wsk_ok(h, k, vn);
  const bool rel = !sk && !wsk && (rel_ok(h->N, may_empty, k) || (h->force_rel && !may_empty && k <= 4096));
  if ((sk || wsk || fast_ok(h->N, may_empty) || rel) && (k & (k - 1)) == 0) {
    const uint32_t nres = std::min(k, R);
    const uint32_t per_res = (R + k - 1) / k;
    // dJFA's stride passes (and its fused first pass) at five CTAs per SM with a 44-KB stage
    static const bool no_five = [] { const char* e = getenv("VD_NO_FIVE"); return e && e[0] == '1'; }();
    const bool five = sk && h->in_djfa && !may_empty && (h->fuse_remap || (!no_five && k >= 4 && k <= 64));
    const int budget = five ? vdk::kSmemBudget5 : vdk::kSmemBudget;
    a.walk = sk || wsk ? vdk::walk_len_sk((int)k, budget) : vdk::walk_len((int)k, rel);
    if (rel) a.walk = std::max(1, std::min(a.walk, (int)(8192 / k) + 1));  // walk span <= 8192 rows
    // Small grids (C2: 1024^2 at k = 1 is 2 x 1 x 43 walks of 24 rows): shorten the walks until
    // there are about two waves of resident CTAs, else a few long walks leave SMs idle.
    const int64_t base = (int64_t)a.xblocks * nres;
    const int64_t want = (int64_t)h->num_sms * 8;
    if (base * (int64_t)((per_res + a.walk - 1) / a.walk) < want) {
      const int64_t segs_want = (want + base - 1) / base;
      a.walk = (int)std::max<int64_t>(2, std::min<int64_t>(a.walk, ((int64_t)per_res + segs_want - 1) / segs_want));
    }
    a.segs = (int)((per_res + a.walk - 1) / a.walk);
    a.lk = 0;
    while ((1u << a.lk) < k) ++a.lk;
    // Grid order (VD_ORDER, experiment): 0 = residue slowest, 1 = segment slowest
    static const int order = [] { const char* e = getenv("VD_ORDER"); return e ? atoi(e) : 0; }();
    // the fused remap pass defaults to segment-slowest order: concurrent CTAs then cover a band
    // of rows, whose seeds' fwd entries stay in L2 (VD_FUSE_ORDER=0: residue slowest)
    static const int fuse_order = [] { const char* e = getenv("VD_FUSE_ORDER"); return e ? atoi(e) : 1; }();
    a.res_in_y = h->fuse_remap ? (fuse_order == 1 || fuse_order == 2 ? fuse_order : 0) : (order == 1 ? 1 : 0);
    // Whole residue classes per CTA (jump_pass_sk FULL walks) when one class fits the stage: a
    // one-band pass over the whole grid with k >= N / (walk + 2) (JFA's large steps).
    // VD_NO_FULL=1 disables it (A/B).
    static const bool no_full = [] { const char* e = getenv("VD_NO_FULL"); return e && e[0] == '1'; }();
    const bool banded = sh.top[0] != nullptr;
    a.nwalk = 0;
    unsigned gz = a.res_in_y ? (unsigned)a.segs : nres, gy = a.res_in_y ? nres : (unsigned)a.segs;
    if ((sk || wsk) && !h->fuse_remap && !no_full && !banded && y_lo == 0 && y_hi == (int64_t)h->N && h->N % k == 0) {
      const uint32_t per = h->N / k, fit = (uint32_t)vdk::walk_len_sk((int)k, budget) + 2;  // (the launch's stage budget)
      // (at least two classes per CTA: C4's k = 2048 0.555 -> 0.522 ms against segment walks, once the
      // FULL walks stopped copying rows; one class per CTA is slower.  VD_FULL_MIN=m: at least m, A/B)
      static const uint32_t full_min = [] { const char* e = getenv("VD_FULL_MIN"); return e ? (uint32_t)atoi(e) : 2u; }();
      if (full_min * per <= fit) {
        // as many classes per CTA as fit, but keep >= 4 CTAs per SM in the grid
        const int64_t cap = std::max<int64_t>(1, (int64_t)a.xblocks * k / ((int64_t)h->num_sms * 4));
        a.nwalk = (int)std::min<int64_t>(fit / per, cap);
        a.walk = vdk::walk_len_sk((int)k, budget);
        a.segs = 1;
        a.res_in_y = 0;
        gy = 1;
        gz = (k + (uint32_t)a.nwalk - 1) / (uint32_t)a.nwalk;
      }
    }
    // spans (k >= 256): groups of 4k columns, k / 128 CTAs each; the last group is partial when
    // 4k does not divide N
    const unsigned gx = (sk || wsk) && k >= 256 ? (unsigned)(((h->N + 4 * k - 1) / (4 * k)) * (k / 128))
                                                : (unsigned)a.xblocks;
    const dim3 grid(gx, gy, gz), blk(vdk::kThreads);
    // locality (the kernels' LOC variants: Euclidean Moore).  A launch whose rows read halo
    // rows (written by other bands, whose locality this band's flag does not cover) keeps
    // the exact walk; the interior launch of an overlapped sharded pass reads none.
    if (h->pass_loc_out && !vn) {
      const bool reads_halo = banded && (a.y_lo < a.row0 + (int)k || a.y_hi > a.row0 + a.rows - (int)k);
      a.loc_in = reads_halo || k > (uint32_t)vdk::kPackMaxK ? nullptr : h->pass_loc_in;
      a.loc_out = h->pass_loc_out;
      h->pass_loc_used |= a.loc_in != nullptr;
    } else {
      h->pass_loc_ok = false;
    }
    const size_t sm = sk || wsk ? vdk::pass_smem_sk((int)k, budget) : vdk::pass_smem((int)k, rel);
    cudaError_t e;
    if (sk || wsk) {
      // k >= 256 on one band: one tensor copy per staged row (VD_NO_TMAP=1: six bulk copies)
      static const bool no_tmap = [] { const char* e = getenv("VD_NO_TMAP"); return e && e[0] == '1'; }();
      CUtensorMap tm;
      memset(&tm, 0, sizeof tm);
      a.tmap = 0;
      // (the row viewed as [N/k][k]: needs k | N)
      if (k >= 256 && h->N % k == 0 && !banded && !no_tmap && encode_span_map(h, a.in, sh.rows, k, &tm)) a.tmap = 1;
      if (wsk) {
        e = vdl::launch_wsk(h->device, may_empty, banded, a, tm, grid, blk, sm, h->stream);
      } else if (h->fuse_remap) {  // first dJFA pass with the remap fused in (vd_djfa_step checked the conditions)
        a.fwd = h->fwd;
        static const int pf = [] { const char* e = getenv("VD_FUSE_PF"); return e ? atoi(e) : 1; }();
        a.prefetch = pf;
        a.loc_in = h->pass_loc_in;  // the previous frame's locality, when the moves keep the packed key valid
        a.nwalk = 0;
        const dim3 g2 = a.res_in_y == 2 ? dim3(nres, (unsigned)a.xblocks, (unsigned)a.segs)
                                        : dim3((unsigned)a.xblocks, a.res_in_y ? nres : (unsigned)a.segs,
                                               a.res_in_y ? (unsigned)a.segs : nres);
        e = vdl::launch_sk_remap(h->device, k, a, tm, g2, blk, sm, h->stream);
      } else {
        if (h->rst_pending && !banded) {  // the fused frame's fwd reset, folded into this pass
          a.rst_fwd = h->fwd;
          a.rst_seeds = h->rst_seeds;
          a.rst_s = (int64_t)h->s;
          h->rst_pending = false;
        }
        if (k == 1 && h->hash_pass && !may_empty) a.hash_out = h->counter;  // the frame's last pass also sums the checksum
        if (lat) {
          a.lat = lat_kind;
          a.lat_empty = unclaimed_label(h);
          a.lat_vl = ((2 * lmax + 1) << 16) | (2 * lmax + 1);
        }
        e = vdl::launch_sk(h->device, k, may_empty && !lat, banded, five, a.hash_out != nullptr, a, tm, grid, blk, sm,
                           h->stream);
      }
    } else {
      e = vdl::launch_fast(h->device, k, may_empty, banded, rel, h->metric, vn, a, grid, blk, sm, h->stream);
    }
    CK(e);
  } else {
    h->pass_loc_ok = false;  // the wide kernel does not report locality
    const uint32_t nres = std::min(k, R);
    a.segs = (int)((R + k - 1) / k);  // rows per residue class
    a.walk = 1;
    const int64_t blocks = (int64_t)a.xblocks * nres * a.segs;
    const dim3 g((unsigned)blocks), b(vdk::kThreads);
    CK(vdl::launch_wide(k, h->metric, vn, a, g, b, h->stream));
  }
  return after_launch(h, "jump_pass");
}

// Halo exchange for step k (vd_halo_plan), then one pass on every local shard.
// Halo exchange of one pass (vd_halo_plan) on stream `st`.
vd_status exchange_halos(vd_ctx* h, uint32_t k, cudaStream_t st) {
  const size_t row_bytes = (size_t)h->pitch * sizeof(uint32_t);
  if (h->world > 1) {
    vd_halo_plan_t p;
    halo_plan(h->N, (uint32_t)h->world, (uint32_t)h->rank, k, p);
    Shard& sh = h->shards[0];
    const size_t cnt = (size_t)p.halo_rows * h->pitch;
    CKN(g_nccl.GroupStart());
    if (p.recv_top_rank >= 0) {
      CKN(g_nccl.Recv(sh.top[h->hpar], cnt, ncclUint32, p.recv_top_rank, h->comm, st));
      CKN(g_nccl.Send(sh.buf[h->cur] + (size_t)p.send_top_row0 * h->pitch, cnt, ncclUint32, p.recv_top_rank, h->comm, st));
    }
    if (p.recv_bot_rank >= 0) {
      CKN(g_nccl.Recv(sh.bot[h->hpar], cnt, ncclUint32, p.recv_bot_rank, h->comm, st));
      CKN(g_nccl.Send(sh.buf[h->cur] + (size_t)p.send_bot_row0 * h->pitch, cnt, ncclUint32, p.recv_bot_rank, h->comm, st));
    }
    CKN(g_nccl.GroupEnd());
  } else if (h->vshards > 1) {
    for (uint32_t g = 0; g < h->vshards; ++g) {
      vd_halo_plan_t p;
      halo_plan(h->N, h->vshards, g, k, p);
      Shard& sh = h->shards[g];
      if (p.recv_top_rank >= 0)
        CK(cudaMemcpyAsync(sh.top[h->hpar], h->shards[p.recv_top_rank].buf[h->cur] + (size_t)(sh.rows - p.halo_rows) * h->pitch,
                           p.halo_rows * row_bytes, cudaMemcpyDeviceToDevice, st));
      if (p.recv_bot_rank >= 0)
        CK(cudaMemcpyAsync(sh.bot[h->hpar], h->shards[p.recv_bot_rank].buf[h->cur], p.halo_rows * row_bytes,
                           cudaMemcpyDeviceToDevice, st));
    }
  }
  return VD_OK;
}

// One pass on every shard.  Sharded with 2k < B: the halos travel on halo_stream while the
// interior rows [k, B-k) of each band, which read no halo, are computed; then the two edge
// strips ("compute interior rows while the halos are in flight").
// Peer halos (h->peer, NEXT-3): the edge strips also store the rows the neighbours' next pass
// (step k_next) reads straight into their halo buffers, so that pass needs no exchange; across
// processes a flag in the neighbour's memory announces them (peer_signal / peer_wait).
vd_status run_pass_body(vd_ctx* h, uint32_t k, bool may_empty, bool vn, uint32_t k_next);
vd_status run_pass(vd_ctx* h, uint32_t k, bool may_empty, bool vn = false, uint32_t k_next = 0) {
  char name[32];
  snprintf(name, sizeof name, "pass k=%u", k);
  NvtxRange range(name);
  loc_pass_begin(h, k);
  const vd_status st = run_pass_body(h, k, may_empty, vn, k_next);
  loc_pass_end(h);
  return st;
}
vd_status run_pass_body(vd_ctx* h, uint32_t k, bool may_empty, bool vn, uint32_t k_next) {
  vd_status st;
  const bool sharded = h->world > 1 || h->vshards > 1;
  const uint32_t B = h->shards[0].rows;
  const bool overlap = sharded && 2 * k < B;
  const uint32_t seq = ++h->pass_seq;
  const bool multi_peer = h->peer && h->world > 1;
  if (!overlap) {
    if (sharded) {
      if (h->world > 1 && !h->comm) return fail(h, VD_ERR_STATE, "step %u needs the NCCL exchange (no communicator)", k);
      if ((st = exchange_halos(h, k, h->stream))) return st;
    }
    for (auto& sh : h->shards) {
      if ((st = timed_begin(h))) return st;
      if ((st = launch_pass(h, sh, k, may_empty, vn))) return st;
      if ((st = timed_end(h, (uint64_t)sh.rows * h->N, k))) return st;
    }
    h->pushed_k = 0;
    h->hpar ^= 1;
    h->cur ^= 1;
    return VD_OK;
  }
  const bool have = h->peer && h->pushed_k == k;  // the previous pass pushed this pass's halos
  const bool push_next = h->peer && k_next > 0 && 2 * k_next < B && k_next <= h->hcap;
  const bool has_above = h->rank > 0, has_below = h->rank + 1 < h->world;
  if (!have) {
    CK(cudaEventRecord(h->halo_ready, h->stream));  // this pass's input is complete
    CK(cudaStreamWaitEvent(h->halo_stream, h->halo_ready, 0));
    if (multi_peer) {  // copy the edge rows into the neighbours' halos, then announce them
      const Shard& sh = h->shards[0];
      const int64_t n4 = (int64_t)k * (h->pitch / 4);
      vdk::push_rows<<<(unsigned)std::min<int64_t>((n4 + 255) / 256, (int64_t)h->num_sms * 8), 256, 0, h->halo_stream>>>(
          sh.buf[h->cur], h->pitch, (int)sh.rows, (int)h->N, (int)k, has_above ? h->nbr_bot[h->hpar] : nullptr,
          has_below ? h->nbr_top[h->hpar] : nullptr);
      if ((st = after_launch(h, "push_rows"))) return st;
      vdk::peer_signal<<<1, 1, 0, h->halo_stream>>>(h->nbr_flag_above, h->nbr_flag_below, seq);
      if ((st = after_launch(h, "peer_signal"))) return st;
    } else if ((st = exchange_halos(h, k, h->halo_stream))) {
      return st;
    }
    CK(cudaEventRecord(h->halo_done, h->halo_stream));
  }
  // one timed interval per pass: first interior launch .. last edge strip
  if ((st = timed_begin(h))) return st;
  uint64_t px = 0;
  for (auto& sh : h->shards) {  // interior rows read no halo
    const int64_t r0 = (int64_t)sh.row0, r1 = r0 + (int64_t)sh.rows;
    if ((st = launch_pass(h, sh, k, may_empty, vn, r0 + k, r1 - k))) return st;
    px += (uint64_t)sh.rows * h->N;
  }
  if (!have) CK(cudaStreamWaitEvent(h->stream, h->halo_done, 0));
  if (multi_peer) {
    vdk::peer_wait<<<1, 1, 0, h->stream>>>(h->flags, has_above, has_below, seq, h->peer_err);
    if ((st = after_launch(h, "peer_wait"))) return st;
  }
  const uint32_t nxt = h->hpar ^ 1;
  for (size_t g = 0; g < h->shards.size(); ++g) {
    Shard& sh = h->shards[g];
    Push push;
    if (push_next) {
      push.k = k_next;
      if (h->world > 1) {
        push.top = has_above ? h->nbr_bot[nxt] : nullptr;
        push.bot = has_below ? h->nbr_top[nxt] : nullptr;
      } else {
        push.top = g > 0 ? h->shards[g - 1].bot[nxt] : nullptr;
        push.bot = g + 1 < h->shards.size() ? h->shards[g + 1].top[nxt] : nullptr;
      }
    }
    const int64_t r0 = (int64_t)sh.row0, r1 = r0 + (int64_t)sh.rows;
    if ((st = launch_pass(h, sh, k, may_empty, vn, r0, r0 + k, &push))) return st;  // top strip
    if ((st = launch_pass(h, sh, k, may_empty, vn, r1 - k, r1, &push))) return st;  // bottom strip
  }
  if (multi_peer && push_next) {
    vdk::peer_signal<<<1, 1, 0, h->stream>>>(h->nbr_flag_above, h->nbr_flag_below, seq + 1);
    if ((st = after_launch(h, "peer_signal"))) return st;
  }
  if ((st = timed_end(h, px, k))) return st;
  h->pushed_k = push_next ? k_next : 0;
  h->hpar ^= 1;
  h->cur ^= 1;
  return VD_OK;
}

vd_status stamp_all(vd_ctx* h, const uint32_t* seeds) {
  for (auto& sh : h->shards) {
    vdk::stamp<<<grid_for(h, (int64_t)h->s, 256), 256, 0, h->stream>>>(sh.buf[h->cur], h->pitch, (int)sh.row0,
                                                                   (int)sh.rows, seeds, (int64_t)h->s);
    vd_status st = after_launch(h, "stamp");
    if (st) return st;
  }
  return VD_OK;
}

vd_status move_seeds(vd_ctx* h, const int16_t* disp_xy) {
  const short2* d;
  int slot;
  vd_status st = upload_disp(h, disp_xy, &d, &slot);
  if (st) return st;
  vdk::move_clamp<<<grid_for(h, (int64_t)h->s, 256), 256, 0, h->stream>>>(h->seeds, d, h->seeds_new, (int64_t)h->s,
                                                                       (int)h->N);
  if ((st = after_launch(h, "move_clamp"))) return st;
  CK(cudaEventRecord(h->disp_used[slot], h->stream));
  return VD_OK;
}

vd_status reduce_to_host(vd_ctx* h, uint64_t* out) {
  if (h->world > 1) {
    if (!h->comm) return fail(h, VD_ERR_STATE, "no NCCL communicator for the cross-rank sum");
    CKN(g_nccl.AllReduce(h->counter, h->counter, 1, ncclUint64, ncclSum, h->comm, h->stream));
  }
  CK(cudaMemcpyAsync(h->counter_h, h->counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream));
  if (vd_status st = sync_stream(h)) return st;
  *out = *h->counter_h;
  return VD_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int now;
    if (prev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != prev) cudaSetDevice(prev);
  }
};

void free_all(vd_ctx* h) {
  for (auto& sh : h->shards) {
    cudaFree(sh.buf[0]);
    cudaFree(sh.buf[1]);
    for (int i = 0; i < 2; ++i) {
      cudaFree(sh.top[i]);
      cudaFree(sh.bot[i]);
    }
  }
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  h->ipc_opened.clear();
  cudaFree(h->flags);
  if (h->peer_err_h) cudaFreeHost(h->peer_err_h);
  h->shards.clear();
  cudaFree(h->seeds);
  cudaFree(h->seeds_new);
  cudaFree(h->disp_buf[0]);
  cudaFree(h->disp_buf[1]);
  cudaFree(h->fwd);
  cudaFree(h->bits);
  cudaFree(h->counter);
  cudaFree(h->loc);

  if (h->counter_h) cudaFreeHost(h->counter_h);
  for (auto e : h->disp_used)
    if (e) cudaEventDestroy(e);
  if (h->copy_done) cudaEventDestroy(h->copy_done);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->halo_stream) cudaStreamDestroy(h->halo_stream);
  if (h->halo_ready) cudaEventDestroy(h->halo_ready);
  if (h->halo_done) cudaEventDestroy(h->halo_done);
  for (auto e : h->ev) cudaEventDestroy(e);
  h->ev.clear();
  if (h->comm && g_nccl.ok) g_nccl.CommDestroy(h->comm);
  h->comm = nullptr;
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  h->stream = nullptr;
}

// JFA / StF initialisation: every pixel unclaimed, each seed pixel holds itself.
// For N <= 16384 "unclaimed" is the virtual far seed V = (2N-1, 2N-1) instead of EMPTY:
// V is farther from every pixel than any real seed and larger than every real label, so
// in every pass it loses exactly as EMPTY (key +infinity) would, and the passes can run
// the kernel variant without EMPTY handling.  Returns the value used.
uint32_t unclaimed_label(const vd_ctx* h) {
  const uint32_t C = 2 * h->N - 1;
  return h->N <= 16384 ? ((C << 16) | C) : VD_EMPTY;
}

vd_status jfa_init(vd_ctx* h) {
  const uint32_t u = unclaimed_label(h);
  for (auto& sh : h->shards) {
    const int64_t n4 = (int64_t)sh.rows * h->pitch / 4;
    vdk::fill_value<<<grid_for(h, n4, 256), 256, 0, h->stream>>>(reinterpret_cast<uint4*>(sh.buf[h->cur]), n4, u);
    vd_status st = after_launch(h, "fill_value");
    if (st) return st;
  }
  return stamp_all(h, h->seeds);
}

// V -> EMPTY for pixels no pass reached (Von Neumann-only waves can leave some, Fig. 5).
vd_status jfa_finish(vd_ctx* h) {
  const uint32_t u = unclaimed_label(h);
  if (u == VD_EMPTY) return VD_OK;
  for (auto& sh : h->shards) {
    const int64_t n4 = (int64_t)sh.rows * h->pitch / 4;
    vdk::replace_value<<<grid_for(h, n4, 256), 256, 0, h->stream>>>(reinterpret_cast<uint4*>(sh.buf[h->cur]), n4, u,
                                                                 VD_EMPTY);
    vd_status st = after_launch(h, "replace_value");
    if (st) return st;
  }
  return VD_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

void vd_config_init(vd_config* cfg) {
  if (!cfg) return;
  memset(cfg, 0, sizeof *cfg);
  cfg->device = -1;
  cfg->world = 1;
}

const char* vd_status_str(vd_status s) {
  switch (s) {
    case VD_OK: return "VD_OK";
    case VD_ERR_ARG: return "VD_ERR_ARG";
    case VD_ERR_RANGE: return "VD_ERR_RANGE";
    case VD_ERR_STATE: return "VD_ERR_STATE";
    case VD_ERR_CUDA: return "VD_ERR_CUDA";
    case VD_ERR_NCCL: return "VD_ERR_NCCL";
    case VD_ERR_OOM: return "VD_ERR_OOM";
    default: return "VD_ERR_UNKNOWN";
  }
}

const char* vd_last_error(vd_handle h) { return h ? h->err.c_str() : "null handle"; }

vd_status vd_nccl_unique_id(void* out128) {
  if (!out128) return VD_ERR_ARG;
  if (!nccl_load()) return VD_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return VD_ERR_NCCL;
  memcpy(out128, &id, sizeof id);
  return VD_OK;
}

vd_status vd_schedule_jfa(uint32_t N, uint32_t extras, uint32_t* ks, uint32_t cap, uint32_t* n) {
  std::vector<uint32_t> v;
  if (!ks || !n || schedule_jfa(N, extras, v) != 0 || v.size() > cap) return VD_ERR_ARG;
  std::copy(v.begin(), v.end(), ks);
  *n = (uint32_t)v.size();
  return VD_OK;
}

vd_status vd_schedule_djfa(uint32_t N, uint64_t s, uint32_t d_max, uint32_t extras, uint32_t* ks, uint32_t cap,
                           uint32_t* n) {
  std::vector<uint32_t> v;
  if (!ks || !n || schedule_djfa(N, s, d_max, extras, v) != 0 || v.size() > cap) return VD_ERR_ARG;
  std::copy(v.begin(), v.end(), ks);
  *n = (uint32_t)v.size();
  return VD_OK;
}

vd_status vd_halo_plan(uint32_t N, uint32_t world, uint32_t rank, uint32_t k, vd_halo_plan_t* out) {
  if (!out || world == 0 || rank >= world || k == 0 || N % world != 0) return VD_ERR_ARG;
  halo_plan(N, world, rank, k, *out);
  return VD_OK;
}

vd_status vd_create(vd_handle* out, uint32_t N, uint64_t s, const uint16_t* seeds_xy, const vd_config* cfg_in) {
  if (!out) return VD_ERR_ARG;
  *out = nullptr;
  vd_config cfg;
  vd_config_init(&cfg);
  if (cfg_in) cfg = *cfg_in;
  if (N < 2 || N > 65536 || s == 0 || s > (uint64_t)N * N || !seeds_xy) return VD_ERR_ARG;
  if (cfg.world < 1 || cfg.rank < 0 || cfg.rank >= cfg.world) return VD_ERR_ARG;
  const bool pow2 = (N & (N - 1)) == 0;
  const uint32_t vsh = cfg.virtual_shards ? cfg.virtual_shards : 1;
  const uint32_t G = cfg.world > 1 ? (uint32_t)cfg.world : vsh;
  if (cfg.world > 1 && vsh > 1) return VD_ERR_ARG;
  if (G > 1 && (!pow2 || N % G != 0 || (G & (G - 1)) != 0)) return VD_ERR_ARG;
  for (int i = 0; i < 2; ++i)
    if (cfg.reserved[i]) return VD_ERR_ARG;
  if (cfg.peer_halos > 1) return VD_ERR_ARG;
  if (cfg.world > 1 && !cfg.nccl_id && !cfg.peer_halos) return VD_ERR_ARG;
  if (cfg.metric > 1) return VD_ERR_ARG;

  // Validate and pack the seeds on the host (R-1, R-4).
  std::vector<uint16_t> hxy;
  const uint16_t* xy = seeds_xy;
  if (is_device_ptr(seeds_xy)) {
    hxy.resize(2 * s);
    if (cudaMemcpy(hxy.data(), seeds_xy, 4 * s, cudaMemcpyDeviceToHost) != cudaSuccess) return VD_ERR_CUDA;
    xy = hxy.data();
  }
  std::vector<uint32_t> packed(s);
  for (uint64_t i = 0; i < s; ++i) {
    const uint32_t x = xy[2 * i], y = xy[2 * i + 1];
    if (x >= N || y >= N) return VD_ERR_RANGE;
    if (N == 65536 && x == 65535 && y == 65535) return VD_ERR_RANGE;
    packed[i] = (y << 16) | x;
  }

  vd_ctx* h = new vd_ctx();
  h->N = N;
  h->s = s;
  h->pitch = ((int64_t)N + 31) / 32 * 32;
  h->rank = cfg.rank;
  h->world = cfg.world;
  h->vshards = cfg.world > 1 ? 1 : vsh;
  h->extras = cfg.extra_passes;
  h->metric = (int)cfg.metric;
  {
    const char* f = std::getenv("VD_FORCE_WINDOWED");
    h->force_rel = f && f[0] == '1';
    const char* w = std::getenv("VD_FORCE_WSK");
    h->force_wsk = w && w[0] == '1';
  }
  h->vn_waves = cfg.vn_waves;
  h->jfa_vn_waves = cfg.jfa_vn_waves;
  if (cfg.device >= 0) h->device = cfg.device;
  else if (cudaGetDevice(&h->device) != cudaSuccess) { delete h; return VD_ERR_CUDA; }
  DeviceGuard guard(h->device);
  if (cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess) {
    delete h;
    return VD_ERR_CUDA;
  }

  auto bail = [&](vd_status st) {
    free_all(h);
    delete h;
    return st;
  };
#define CKC(expr)                                                                        \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess) return bail(e_ == cudaErrorMemoryAllocation ? VD_ERR_OOM : VD_ERR_CUDA); \
  } while (0)

  if (cfg.stream) h->stream = (cudaStream_t)cfg.stream;
  else {
    CKC(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  // Bands: one per rank (world > 1) or `vshards` inside this handle.
  const uint32_t B = N / G;
  const uint32_t k1 = 1u << (ceil_log2_u64(N) - 1);
  h->hcap = G > 1 ? std::min(k1, B) : 0;
  const uint32_t nloc = cfg.world > 1 ? 1 : h->vshards;
  for (uint32_t g = 0; g < nloc; ++g) {
    Shard sh;
    const uint32_t band = cfg.world > 1 ? (uint32_t)cfg.rank : g;
    sh.row0 = G > 1 ? band * B : 0;
    sh.rows = G > 1 ? B : N;
    h->shards.push_back(sh);
    Shard& r = h->shards.back();
    const size_t bytes = (size_t)r.rows * h->pitch * sizeof(uint32_t);
    CKC(cudaMalloc(&r.buf[0], bytes));
    CKC(cudaMalloc(&r.buf[1], bytes));
    CKC(cudaMemsetAsync(r.buf[0], 0xFF, bytes, h->stream));
    CKC(cudaMemsetAsync(r.buf[1], 0xFF, bytes, h->stream));
    if (h->hcap) {
      const size_t hb = (size_t)h->hcap * h->pitch * sizeof(uint32_t);
      for (int i = 0; i < 2; ++i) {
        CKC(cudaMalloc(&r.top[i], hb));
        CKC(cudaMalloc(&r.bot[i], hb));
        CKC(cudaMemsetAsync(r.top[i], 0xFF, hb, h->stream));
        CKC(cudaMemsetAsync(r.bot[i], 0xFF, hb, h->stream));
      }
    }
  }
  CKC(cudaMalloc(&h->seeds, s * sizeof(uint32_t)));
  CKC(cudaMalloc(&h->seeds_new, s * sizeof(uint32_t)));
  CKC(cudaMalloc(&h->disp_buf[0], s * sizeof(short2)));
  CKC(cudaMalloc(&h->disp_buf[1], s * sizeof(short2)));
  CKC(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  CKC(cudaStreamCreateWithFlags(&h->halo_stream, cudaStreamNonBlocking));
  CKC(cudaEventCreateWithFlags(&h->halo_ready, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&h->halo_done, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&h->copy_done, cudaEventDisableTiming));
  for (auto& e : h->disp_used) {
    CKC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CKC(cudaEventRecord(e, h->stream));
  }
  CKC(cudaMalloc(&h->counter, sizeof(unsigned long long)));
  CKC(cudaMalloc(&h->loc, kLocSlots * sizeof(uint32_t)));
  CKC(cudaMemsetAsync(h->loc, 0x01, kLocSlots * sizeof(uint32_t), h->stream));  // nothing known to be local
  CKC(cudaMalloc(&h->flags, 2 * sizeof(uint32_t)));
  CKC(cudaMemset(h->flags, 0, 2 * sizeof(uint32_t)));
  CKC(cudaHostAlloc(&h->peer_err_h, sizeof(uint32_t), cudaHostAllocMapped));
  *h->peer_err_h = 0;
  CKC(cudaHostGetDevicePointer(&h->peer_err, h->peer_err_h, 0));
  h->peer = cfg.peer_halos && cfg.world == 1 && h->vshards > 1;  // across processes: vd_peer_attach
  CKC(cudaMallocHost(&h->counter_h, sizeof(unsigned long long)));
  CKC(cudaMemcpyAsync(h->seeds, packed.data(), s * sizeof(uint32_t), cudaMemcpyHostToDevice, h->stream));
  CKC(cudaStreamSynchronize(h->stream));
  if (cfg.world > 1 && cfg.nccl_id) {
    if (!nccl_load()) return bail(VD_ERR_NCCL);
    ncclUniqueId id;
    memcpy(&id, cfg.nccl_id, sizeof id);
    if (g_nccl.CommInitRank(&h->comm, cfg.world, id, cfg.rank) != ncclSuccess) return bail(VD_ERR_NCCL);
  }
#undef CKC
  *out = h;
  return VD_OK;
}

void vd_destroy(vd_handle h) {
  if (!h) return;
  DeviceGuard guard(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  free_all(h);
  delete h;
}

namespace {
// Pass k_1 of a JFA straight from the seeds (jfa_first_pass): fill the band with the
// unclaimed label, then scatter every seed's offers.  Same result as init + stamp + gather
// pass; needs no halo exchange (every rank holds every seed).
vd_status jfa_init_first_pass(vd_ctx* h, uint32_t k1, bool vn) {
  const uint32_t u = unclaimed_label(h);
  // VD_FIRST_GATHER=1: a gather from a seed bitmap instead of the scatter (k_1 >= 32; measured slower:
  // C4 JFA 7.19 vs 6.62 ms, C5 135.5 vs 134.2 ms, `profiles/r02c_first_gather_ab_*.txt`)
  static const bool gather = [] { const char* e = getenv("VD_FIRST_GATHER"); return e && e[0] == '1'; }();
  if (gather && k1 >= 32) {
    const int64_t wpr = (h->N + 31) / 32;
    const size_t bytes = (size_t)h->N * wpr * sizeof(uint32_t);
    if (!h->bits) CK(cudaMalloc(&h->bits, 2 * bytes));  // (two bitmaps: the sparse passes ping-pong them)
    CK(cudaMemsetAsync(h->bits, 0, bytes, h->stream));
    vdk::seed_bits<<<grid_for(h, (int64_t)h->s, 256), 256, 0, h->stream>>>(h->bits, wpr, h->seeds, (int64_t)h->s);
    vd_status st = after_launch(h, "seed_bits");
    if (st) return st;
    for (auto& sh : h->shards) {
      const dim3 gg((unsigned)((wpr + 255) / 256), (unsigned)std::min<int64_t>(sh.rows, (int64_t)h->num_sms * 32));
      vdk::jfa_first_gather<<<gg, 256, 0, h->stream>>>(
          sh.buf[h->cur], h->pitch, (int)sh.row0, (int)sh.rows, (int)h->N, (int)k1, h->bits, wpr, u, vn ? 1 : 0);
      if ((st = after_launch(h, "jfa_first_gather"))) return st;
    }
    ++h->pass_seq;
    h->hpar ^= 1;
    h->pushed_k = 0;
    return VD_OK;
  }
  for (auto& sh : h->shards) {
    const int64_t n4 = (int64_t)sh.rows * h->pitch / 4;
    vdk::fill_value<<<grid_for(h, n4, 256), 256, 0, h->stream>>>(reinterpret_cast<uint4*>(sh.buf[h->cur]), n4, u);
    vd_status st = after_launch(h, "fill_value");
    if (st) return st;
    vdk::jfa_first_pass<<<grid_for(h, (int64_t)h->s, 256), 256, 0, h->stream>>>(
        sh.buf[h->cur], h->pitch, (int)sh.row0, (int)sh.rows, (int)h->N, (int)k1, h->seeds, (int64_t)h->s, u,
        h->metric, vn ? 1 : 0);
    if ((st = after_launch(h, "jfa_first_pass"))) return st;
  }
  ++h->pass_seq;  // keeps the peer-halo sequence numbers counting passes
  h->hpar ^= 1;
  h->pushed_k = 0;
  return VD_OK;
}
}  // namespace

vd_status vd_jfa(vd_handle h) {
  CHECK_HANDLE(h);
  DeviceGuard guard(h->device);
  NvtxRange range("vd_jfa");
  std::vector<uint32_t> ks;
  schedule_jfa(h->N, h->extras, ks);
  // P:68 + pass k_1, fused (VD_NO_FIRST_SCATTER=1: init + stamp + gather pass, for A/B)
  static const bool no_scatter = [] { const char* e = getenv("VD_NO_FIRST_SCATTER"); return e && e[0] == '1'; }();
  vd_status st = no_scatter ? jfa_init(h) : jfa_init_first_pass(h, ks[0], h->jfa_vn_waves > 0);
  if (st) return st;
  const size_t first = no_scatter ? 0 : 1;
  const bool virt = unclaimed_label(h) != VD_EMPTY;
  // Beyond N = 16384 EMPTY is real and the passes run the 64-bit kernel, which reports
  // whether it left any EMPTY (summed over ranks); from the first pass that leaves none on,
  // the remaining passes take the EMPTY-free kernels (a complete map stays complete).
  bool may_empty = !virt;
  const bool track = may_empty;
  loc_begin(h);  // the passes report locality; once it holds, the rest take the packed-key kernel
  // Sparse passes (r02c, opt-in VD_SPARSE=1, measured slower): the passes right after the first one,
  // while their input is mostly EMPTY, read an occupancy bitmap and load labels only where it is set
  // (one band, Euclidean Moore, N > 32768, N % 128 == 0, lattice keys: k >= N/64).  VD_SPARSE_PASSES=n
  // sets how many (2: k = N/4 and N/8 at C5, inputs 98% and 94% EMPTY).  C5: 19.2 and 29.3 ms against
  // 10 ms for the dense lattice passes (`profiles/r02c_sparse_ab_c5.txt`).
  static const bool no_sparse = [] { const char* e = getenv("VD_SPARSE"); return !(e && e[0] == '1'); }();
  static const int sparse_n = [] { const char* e = getenv("VD_SPARSE_PASSES"); return e ? atoi(e) : 2; }();
  const bool sparse_ok = !no_sparse && first == 1 && h->N > 32768 && h->N % 128 == 0 && h->metric == 0 &&
                         h->world == 1 && h->vshards == 1 && h->jfa_vn_waves == 0 && !h->force_rel && may_empty;
  const int64_t wpr = (h->N + 31) / 32;
  int sparse_done = 0;
  uint32_t* occ_in = nullptr;
  uint32_t* occ_out = nullptr;
  for (size_t i = first; i < ks.size(); ++i) {
    const bool vn = i < h->jfa_vn_waves;
    const uint32_t kk = ks[i];
    if (sparse_ok && sparse_done < sparse_n && (uint64_t)kk * 64 >= h->N && i + 1 < ks.size()) {
      const size_t bytes = (size_t)h->N * wpr * sizeof(uint32_t);
      if (!h->bits) CK(cudaMalloc(&h->bits, 2 * bytes));
      if (sparse_done == 0) {  // the first pass's occupancy, from the seeds it placed
        occ_in = h->bits;
        occ_out = h->bits + (size_t)h->N * wpr;
        CK(cudaMemsetAsync(occ_in, 0, bytes, h->stream));
        vdk::occ_from_seeds<<<grid_for(h, (int64_t)h->s, 256), 256, 0, h->stream>>>(occ_in, wpr, h->seeds,
                                                                                  (int64_t)h->s, (int)h->N, (int)ks[0]);
        if ((st = after_launch(h, "occ_from_seeds"))) return loc_end(h), st;
      }
      CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned long long), h->stream));
      uint32_t lk = 0;
      while ((1u << lk) < kk) ++lk;
      Shard& sh = h->shards[0];
      loc_pass_begin(h, kk);
      h->pass_loc_ok = false;  // (locality is not reported by this kernel)
      if ((st = timed_begin(h))) return loc_end(h), st;
      const bool last_sparse = sparse_done + 1 >= sparse_n;
      const dim3 gs2((unsigned)((h->N / 4 + 255) / 256), (unsigned)std::min<int64_t>(h->N, (int64_t)h->num_sms * 16));
      vdk::jfa_sparse_pass<<<gs2, 256, 0, h->stream>>>(
          sh.buf[h->cur], sh.buf[h->cur ^ 1], h->pitch, (int)h->N, (int)kk, (int)lk, occ_in,
          last_sparse ? nullptr : occ_out, wpr, h->counter);
      if ((st = after_launch(h, "jfa_sparse_pass"))) return loc_end(h), st;
      if ((st = timed_end(h, (uint64_t)h->N * h->N, kk))) return loc_end(h), st;
      loc_pass_end(h);
      ++h->pass_seq;
      h->hpar ^= 1;
      h->cur ^= 1;
      h->pushed_k = 0;
      std::swap(occ_in, occ_out);
      ++sparse_done;
      uint64_t any = 1;
      if ((st = reduce_to_host(h, &any))) return loc_end(h), st;
      may_empty = any != 0;
      continue;
    }
    if (track && may_empty) {
      CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned long long), h->stream));
      h->track_empty = true;
    }
    // JFA's labels are still far from their pixels at large steps: there the windowed kernel
    // would recompute most walks, and the 64-bit one is cheaper (C5: 31 vs 68 ms at k = 512).
    const bool far = h->N > 32768 && ks[i] > 256 && !wsk_ok(h, ks[i], vn);
    // the passes of the schedule proper (not the extra k = 1 passes) keep every label congruent to
    // its pixel mod the step: the lattice walk may take them
    h->lat_pass = i < ks.size() - h->extras;
    st = run_pass(h, ks[i], may_empty || far, vn, i + 1 < ks.size() ? ks[i + 1] : 0);
    h->lat_pass = false;
    h->track_empty = false;
    if (st) return loc_end(h), st;
    if (track && may_empty) {
      uint64_t any = 1;
      if ((st = reduce_to_host(h, &any))) return loc_end(h), st;
      may_empty = any != 0;
    }
  }
  loc_end(h);
  // A Moore JFA reaches every pixel (k_1 = 2^(ceil(log2 N)-1) covers every offset), so no V
  // survives; Von Neumann waves may leave some.
  h->last_passes = (uint32_t)ks.size();
  if (h->jfa_vn_waves > 0) {
    if ((st = jfa_finish(h))) return st;
    // dJFA needs a complete diagram: count what is still EMPTY (synchronises)
    CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned long long), h->stream));
    for (auto& sh : h->shards) {
      vdk::count_value<<<rows_grid(h, sh.rows), 256, 0, h->stream>>>(sh.buf[h->cur], h->pitch, (int)sh.rows, (int)h->N,
                                                                  VD_EMPTY, h->counter);
      if ((st = after_launch(h, "count_value"))) return st;
    }
    uint64_t empty = 0;
    if ((st = reduce_to_host(h, &empty))) return st;
    h->has_diagram = empty == 0;
    return VD_OK;
  }
  h->last_passes = (uint32_t)ks.size();
  h->has_diagram = true;
  return VD_OK;
}

vd_status vd_stf(vd_handle h, uint32_t* passes) {
  CHECK_HANDLE(h);
  DeviceGuard guard(h->device);
  vd_status st = jfa_init(h);  // as JFA
  if (st) return st;
  const uint32_t u = unclaimed_label(h);
  uint32_t n = 0;
  while (true) {  // "until the grid is fully flooded": stop once no EMPTY is left
    CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned long long), h->stream));
    for (auto& sh : h->shards) {
      vdk::count_value<<<rows_grid(h, sh.rows), 256, 0, h->stream>>>(sh.buf[h->cur], h->pitch, (int)sh.rows, (int)h->N,
                                                                  u, h->counter);
      if ((st = after_launch(h, "count_value"))) return st;
    }
    uint64_t empty = 0;
    if ((st = reduce_to_host(h, &empty))) return st;
    if (empty == 0) break;
    if ((st = run_pass(h, 1, u == VD_EMPTY))) return st;
    ++n;
  }
  h->last_passes = n;
  h->has_diagram = true;
  loc_forget(h);
  if (passes) *passes = n;
  return VD_OK;
}

vd_status vd_move_seeds(vd_handle h, const int16_t* disp_xy) {
  CHECK_HANDLE(h);
  if (!disp_xy) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  vd_status st = move_seeds(h, disp_xy);
  if (st) return st;
  std::swap(h->seeds, h->seeds_new);
  h->has_diagram = false;  // the diagram no longer matches the seeds
  return VD_OK;
}

namespace {
vd_status enqueue_label_hash(vd_ctx* h);
// One dJFA step (vd_djfa_step).  hash: also leave the new diagram's label checksum in h->counter,
// accumulated by the last pass when it can (jump_pass_sk HASH, k = 1), else by label_hash.
vd_status djfa_step(vd_ctx* h, const int16_t* disp_xy, uint32_t d_max, bool hash) {
  NvtxRange range("vd_djfa_step");
  if (!h->fwd) {  // forward map, kept all-EMPTY between steps
    // indexed by the label itself ((y << 16) | x) where the fused frame can run (one band, Euclidean,
    // Moore), else by y N + x
    // (the layout is chosen per frame, below; the table is all-EMPTY between frames in both, and is
    // sized for the label-indexed one only where a frame can fuse)
    h->fwd_fusable = h->metric == 0 && h->world == 1 && h->vshards == 1 && h->vn_waves == 0;
    const size_t bytes = (size_t)h->N * (h->fwd_fusable ? 65536 : h->N) * sizeof(uint32_t);
    CK(cudaMalloc(&h->fwd, bytes));
    CK(cudaMemsetAsync(h->fwd, 0xFF, bytes, h->stream));
  }
  std::vector<uint32_t> ks;
  schedule_djfa(h->N, h->s, d_max, h->extras, ks);
  struct InDjfa {
    vd_ctx* h;
    ~InDjfa() { h->in_djfa = h->hash_pass = false; }
  } in_djfa{h};
  h->in_djfa = true;
  // the fused checksum needs the last pass to be a Moore step 1 on jump_pass_sk
  const bool hash_fused = hash && ks.back() == 1 && ks.size() > h->vn_waves && sk_ok(h, 1, false, false);
  if (hash) CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned long long), h->stream));
  const short2* dd;
  int slot;
  vd_status st = upload_disp(h, disp_xy, &dd, &slot);
  if (st) return st;
  const int gs = grid_for(h, (int64_t)h->s, 256);
  // 1. SimulateParticles + forward map old -> new (R-9); fwd is all EMPTY on entry
  const bool loc = loc_begin(h);
  // NEXT-1: on one band the first pass remaps its own staged rows (jump_pass_sk_remap): the
  // new seed pixels are marked first (EMPTY, by move_fwd), the remapped diagram never goes to HBM,
  // and fwd is reset after that pass.  VD_NO_FUSE=1: the separate remap kernel.
  static const bool no_fuse = [] { const char* e = getenv("VD_NO_FUSE"); return e && e[0] == '1'; }();
  const uint32_t k1 = ks[0];
  const bool fuse = !no_fuse && loc && h->world == 1 && h->vshards == 1 && h->vn_waves == 0 && h->fwd_fusable &&
                    sk_ok(h, k1, false, false) && k1 >= 4 && k1 <= 128;
  // fwd indexed by the label itself for the fused pass (one address computation per gather), by
  // y N + x for the separate remap, whose row-order sweep then gathers over a quarter of the address
  // range at C4 (0.47 vs 0.72 ms; `profiles/r02c_remap_layout_ab_c4.txt`)
  h->fwd_pitch = fuse ? 0 : (int)h->N;
  vdk::move_fwd<<<gs, 256, 0, h->stream>>>(h->seeds, dd, h->seeds_new, h->fwd, h->fwd_pitch, (int64_t)h->s, (int)h->N,
                                           fuse ? h->shards[0].buf[h->cur] : nullptr, h->pitch);
  if ((st = after_launch(h, "move_fwd"))) return st;
  CK(cudaEventRecord(h->disp_used[slot], h->stream));
  if (fuse) {
    // Packed walk for the fused pass: every label of the previous diagram within kLocR of its
    // pixel (its flag, kLocPrev) and seeds that moved at most d_max per axis leave every remapped
    // label within kLocR + d_max*sqrt(2) of its pixel, so a candidate is within that + k1 per
    // axis; the packed key needs <= 127.  Otherwise the exact walk.
    const bool pack_ok = k1 <= (uint32_t)vdk::kPackMaxK && (uint64_t)vdk::kLocR + (3ull * d_max + 1) / 2 + k1 <= 127;
    h->fuse_pack = pack_ok;
    h->fuse_remap = true;
    st = run_pass(h, k1, false, false, ks.size() > 1 ? ks[1] : 0);
    h->fuse_remap = false;
    if (st) return loc_end(h), st;
    // fwd back to all-EMPTY: folded into the second pass when it runs on jump_pass_sk (VD_NO_RST_FOLD=1:
    // the separate fwd_reset kernel), else a kernel of its own
    static const bool no_fold = [] { const char* e = getenv("VD_NO_RST_FOLD"); return e && e[0] == '1'; }();
    h->rst_seeds = h->seeds;
    h->rst_pending = !no_fold && ks.size() > 1;
    std::swap(h->seeds, h->seeds_new);
    for (size_t i = 1; i < ks.size(); ++i) {
      h->hash_pass = hash_fused && i + 1 == ks.size();
      if ((st = run_pass(h, ks[i], false, false, i + 1 < ks.size() ? ks[i + 1] : 0))) {
        h->rst_pending = false;
        return loc_end(h), st;
      }
      if (h->rst_pending) {  // that pass could not carry it
        h->rst_pending = false;
        vdk::fwd_reset<<<gs, 256, 0, h->stream>>>(h->fwd, h->fwd_pitch, (int)h->N, h->rst_seeds, (int64_t)h->s);
        if ((st = after_launch(h, "fwd_reset"))) return st;
      }
    }
    if (h->rst_pending || ks.size() == 1 || no_fold) {  // no second pass (or the fold is off)
      h->rst_pending = false;
      vdk::fwd_reset<<<gs, 256, 0, h->stream>>>(h->fwd, h->fwd_pitch, (int)h->N, h->rst_seeds, (int64_t)h->s);
      if ((st = after_launch(h, "fwd_reset"))) return st;
    }
    loc_end(h);
    h->last_passes = (uint32_t)ks.size();
    if (hash && !(hash_fused && ks.size() > 1)) return enqueue_label_hash(h);
    return VD_OK;
  }
  // 2. labels follow their seeds (reuse of VD_{t-1})
  //    (one band: the remap also reports whether every label is within kLocR of its pixel,
  //    which lets the passes take the packed-key kernel)
  static const int remap_kind = [] { const char* e = getenv("VD_REMAP"); return e ? atoi(e) : 0; }();
  if ((st = timed_begin(h))) return st;  // timed as an interval with k = 0 (vd_pass_times)
  for (auto& sh : h->shards) {
    if (remap_kind == 1)
      vdk::remap_lanes<<<rows_grid(h, sh.rows), 256, 0, h->stream>>>(sh.buf[h->cur], h->pitch, (int)sh.rows, (int)h->N,
                                                                     h->fwd, h->fwd_pitch, (int)sh.row0, loc ? h->loc : nullptr);
    else
      vdk::remap<<<rows_grid(h, sh.rows), 256, 0, h->stream>>>(sh.buf[h->cur], h->pitch, (int)sh.rows, (int)h->N,
                                                               h->fwd, h->fwd_pitch, (int)sh.row0, loc ? h->loc : nullptr);
    if ((st = after_launch(h, "remap"))) return st;
  }
  if ((st = timed_end(h, 0, 0))) return st;
  h->loc_valid = loc;
  // 3. re-stamp the new seed pixels; fwd back to all-EMPTY
  for (size_t g = 0; g < h->shards.size(); ++g) {
    Shard& sh = h->shards[g];
    vdk::reset_stamp<<<gs, 256, 0, h->stream>>>(h->fwd, h->fwd_pitch, (int)h->N, h->seeds, h->seeds_new, sh.buf[h->cur], h->pitch,
                                                (int)sh.row0, (int)sh.rows, (int64_t)h->s, g == 0 ? 1 : 0);
    if ((st = after_launch(h, "reset_stamp"))) return st;
  }
  std::swap(h->seeds, h->seeds_new);
  // 4. passes delta_1 .. 1 (Eq. 4).  The remapped diagram is complete (every label is a
  //    seed), so no EMPTY exists.
  for (size_t i = 0; i < ks.size(); ++i) {
    h->hash_pass = hash_fused && i + 1 == ks.size();
    if ((st = run_pass(h, ks[i], false, i < h->vn_waves, i + 1 < ks.size() ? ks[i + 1] : 0))) return loc_end(h), st;
  }
  loc_end(h);
  h->last_passes = (uint32_t)ks.size();
  if (hash && !hash_fused) return enqueue_label_hash(h);
  return VD_OK;
}
}  // namespace

vd_status vd_djfa_step(vd_handle h, const int16_t* disp_xy, uint32_t d_max) {
  CHECK_HANDLE(h);
  if (!disp_xy) return VD_ERR_ARG;
  if (!h->has_diagram) return fail(h, VD_ERR_STATE, "vd_djfa_step needs a diagram: call vd_jfa first");
  DeviceGuard guard(h->device);
  return djfa_step(h, disp_xy, d_max, false);
}

vd_status vd_djfa_step_hash(vd_handle h, const int16_t* disp_xy, uint32_t d_max, uint64_t* pinned_out) {
  CHECK_HANDLE(h);
  if (!disp_xy || !pinned_out) return VD_ERR_ARG;
  if (!h->has_diagram) return fail(h, VD_ERR_STATE, "vd_djfa_step needs a diagram: call vd_jfa first");
  DeviceGuard guard(h->device);
  vd_status st = djfa_step(h, disp_xy, d_max, true);
  if (st) return st;
  if (h->world > 1) {
    if (!h->comm) return fail(h, VD_ERR_STATE, "no NCCL communicator for the cross-rank sum");
    CKN(g_nccl.AllReduce(h->counter, h->counter, 1, ncclUint64, ncclSum, h->comm, h->stream));
  }
  CK(cudaMemcpyAsync(pinned_out, h->counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream));
  return VD_OK;
}

vd_status vd_set_labels(vd_handle h, const uint32_t* labels) {
  CHECK_HANDLE(h);
  if (!labels) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  loc_forget(h);
  uint64_t rows_total = 0;
  for (auto& sh : h->shards) rows_total += sh.rows;
  const uint64_t n = rows_total * h->N;
  bool any_empty = false;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t c = labels[i];
    if (c == VD_EMPTY) { any_empty = true; continue; }
    if ((c & 0xFFFFu) >= h->N || (c >> 16) >= h->N) return fail(h, VD_ERR_RANGE, "label %u outside the grid", c);
  }
  size_t off_rows = 0;
  for (auto& sh : h->shards) {
    CK(cudaMemcpy2DAsync(sh.buf[h->cur], h->pitch * sizeof(uint32_t), labels + off_rows * h->N,
                         h->N * sizeof(uint32_t), h->N * sizeof(uint32_t), sh.rows, cudaMemcpyHostToDevice, h->stream));
    off_rows += sh.rows;
  }
  if (vd_status st_ = sync_stream(h)) return st_;
  h->has_diagram = !any_empty;
  return VD_OK;
}

vd_status vd_pass(vd_handle h, uint32_t k, uint32_t flags) {
  CHECK_HANDLE(h);
  if (k == 0 || k >= 65536) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  if (h->world > 1 || h->vshards > 1) {
    const uint32_t G = h->world > 1 ? (uint32_t)h->world : h->vshards;
    const uint32_t B = h->N / G;
    if (k > B && k % B != 0) return fail(h, VD_ERR_ARG, "sharded pass needs k < band rows or a multiple of them");
    if (k > h->hcap && k < B) return fail(h, VD_ERR_ARG, "halo capacity exceeded");
  }
  // A complete map (no EMPTY, known on every shard of this handle) stays complete under a
  // pass, so the EMPTY-free kernels apply; across ranks completeness is not known globally.
  const bool may_empty = !h->has_diagram || h->world > 1;
  loc_forget(h);
  return run_pass(h, k, may_empty, (flags & VD_PASS_VON_NEUMANN) != 0);
}

// ---- peer halos across processes (NEXT-3) ----
namespace {
struct PeerBlob {
  int32_t rank, world;
  uint32_t N, hcap;
  cudaIpcMemHandle_t top[2], bot[2], flags;
};
}  // namespace

vd_status vd_peer_export(vd_handle h, void* out, size_t cap, size_t* len) {
  CHECK_HANDLE(h);
  if (len) *len = sizeof(PeerBlob);
  if (!out) return len ? VD_OK : VD_ERR_ARG;
  if (cap < sizeof(PeerBlob)) return VD_ERR_ARG;
  if (h->world < 2) return fail(h, VD_ERR_STATE, "vd_peer_export needs world > 1");
  DeviceGuard guard(h->device);
  PeerBlob b{};
  b.rank = h->rank;
  b.world = h->world;
  b.N = h->N;
  b.hcap = h->hcap;
  const Shard& sh = h->shards[0];
  for (int i = 0; i < 2; ++i) {
    CK(cudaIpcGetMemHandle(&b.top[i], sh.top[i]));
    CK(cudaIpcGetMemHandle(&b.bot[i], sh.bot[i]));
  }
  CK(cudaIpcGetMemHandle(&b.flags, h->flags));
  memcpy(out, &b, sizeof b);
  return VD_OK;
}

vd_status vd_peer_attach(vd_handle h, const void* blobs, size_t len_each) {
  CHECK_HANDLE(h);
  if (!blobs || len_each != sizeof(PeerBlob)) return VD_ERR_ARG;
  if (h->world < 2 || h->peer) return fail(h, VD_ERR_STATE, "vd_peer_attach: needs world > 1, once");
  DeviceGuard guard(h->device);
  const auto* all = static_cast<const PeerBlob*>(blobs);
  for (int r = 0; r < h->world; ++r)
    if (all[r].rank != r || all[r].world != h->world || all[r].N != h->N || all[r].hcap != h->hcap)
      return fail(h, VD_ERR_ARG, "vd_peer_attach: blob %d does not match this grid", r);
  auto open = [&](const cudaIpcMemHandle_t& hd, uint32_t** out) -> vd_status {
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
    h->ipc_opened.push_back(p);
    *out = static_cast<uint32_t*>(p);
    return VD_OK;
  };
  vd_status st;
  uint32_t* f = nullptr;
  if (h->rank > 0) {  // the band above: its bottom halos and its "from below" flag
    const PeerBlob& b = all[h->rank - 1];
    for (int i = 0; i < 2; ++i)
      if ((st = open(b.bot[i], &h->nbr_bot[i]))) return st;
    if ((st = open(b.flags, &f))) return st;
    h->nbr_flag_above = f + 1;
  }
  if (h->rank + 1 < h->world) {  // the band below: its top halos and its "from above" flag
    const PeerBlob& b = all[h->rank + 1];
    for (int i = 0; i < 2; ++i)
      if ((st = open(b.top[i], &h->nbr_top[i]))) return st;
    if ((st = open(b.flags, &f))) return st;
    h->nbr_flag_below = f;
  }
  h->peer = true;
  return VD_OK;
}

vd_status vd_peer_status(vd_handle h, uint32_t* timed_out) {
  if (!h || !timed_out) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  CK(cudaStreamSynchronize(h->stream));
  *timed_out = *(volatile uint32_t*)h->peer_err_h;
  return VD_OK;
}

vd_status vd_similarity(vd_handle h, vd_handle ref, double* pct, uint64_t* matches) {
  CHECK_HANDLE(h);
  CHECK_HANDLE(ref);
  if (!pct && !matches) return VD_ERR_ARG;
  if (ref->N != h->N || ref->world != h->world || ref->rank != h->rank || ref->vshards != h->vshards ||
      ref->device != h->device)
    return fail(h, VD_ERR_ARG, "vd_similarity: handles differ in N, sharding or device");
  DeviceGuard guard(h->device);
  if (ref->stream != h->stream) CK(cudaStreamSynchronize(ref->stream));
  CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned long long), h->stream));
  for (size_t g = 0; g < h->shards.size(); ++g) {
    const Shard& a = h->shards[g];
    const Shard& b = ref->shards[g];
    vdk::match_count<<<rows_grid(h, a.rows), 256, 0, h->stream>>>(a.buf[h->cur], b.buf[ref->cur], h->pitch,
                                                                (int)a.rows, (int)h->N, h->counter);
    vd_status st = after_launch(h, "match_count");
    if (st) return st;
  }
  uint64_t m = 0;
  vd_status st = reduce_to_host(h, &m);
  if (st) return st;
  if (matches) *matches = m;
  if (pct) *pct = 100.0 * (double)m / ((double)h->N * (double)h->N);
  return VD_OK;
}

vd_status vd_similarity_host(vd_handle h, const uint32_t* ref_labels, double* pct, uint64_t* matches) {
  CHECK_HANDLE(h);
  if (!ref_labels || (!pct && !matches)) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned long long), h->stream));
  size_t off_rows = 0;
  for (auto& sh : h->shards) {
    // the idle ping-pong buffer is scratch between calls
    uint32_t* scratch = sh.buf[h->cur ^ 1];
    CK(cudaMemcpy2DAsync(scratch, h->pitch * sizeof(uint32_t), ref_labels + off_rows * h->N, h->N * sizeof(uint32_t),
                         h->N * sizeof(uint32_t), sh.rows, cudaMemcpyDefault, h->stream));
    vdk::match_count<<<rows_grid(h, sh.rows), 256, 0, h->stream>>>(sh.buf[h->cur], scratch, h->pitch, (int)sh.rows,
                                                                (int)h->N, h->counter);
    vd_status st = after_launch(h, "match_count");
    if (st) return st;
    off_rows += sh.rows;
  }
  uint64_t m = 0;
  vd_status st = reduce_to_host(h, &m);
  if (st) return st;
  if (matches) *matches = m;
  if (pct) *pct = 100.0 * (double)m / ((double)h->N * (double)h->N);
  return VD_OK;
}

namespace {
vd_status enqueue_label_hash(vd_ctx* h) {
  CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned long long), h->stream));
  for (auto& sh : h->shards) {
    vdk::label_hash<<<rows_grid(h, sh.rows), 256, 0, h->stream>>>(sh.buf[h->cur], h->pitch, (int)sh.row0,
                                                               (int)sh.rows, (int)h->N, h->counter);
    vd_status st = after_launch(h, "label_hash");
    if (st) return st;
  }
  return VD_OK;
}
}  // namespace

vd_status vd_label_hash(vd_handle h, uint64_t* out) {
  CHECK_HANDLE(h);
  if (!out) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  vd_status st = enqueue_label_hash(h);
  if (st) return st;
  return reduce_to_host(h, out);
}

vd_status vd_label_hash_async(vd_handle h, uint64_t* pinned_out) {
  CHECK_HANDLE(h);
  if (!pinned_out) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  vd_status st = enqueue_label_hash(h);
  if (st) return st;
  if (h->world > 1) {
    if (!h->comm) return fail(h, VD_ERR_STATE, "no NCCL communicator for the cross-rank sum");
    CKN(g_nccl.AllReduce(h->counter, h->counter, 1, ncclUint64, ncclSum, h->comm, h->stream));
  }
  CK(cudaMemcpyAsync(pinned_out, h->counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream));
  return VD_OK;
}

vd_status vd_get_labels(vd_handle h, uint32_t* out) {
  CHECK_HANDLE(h);
  if (!out) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  size_t off_rows = 0;
  for (auto& sh : h->shards) {
    CK(cudaMemcpy2DAsync(out + off_rows * h->N, h->N * sizeof(uint32_t), sh.buf[h->cur], h->pitch * sizeof(uint32_t),
                         h->N * sizeof(uint32_t), sh.rows, cudaMemcpyDeviceToHost, h->stream));
    off_rows += sh.rows;
  }
  if (vd_status st_ = sync_stream(h)) return st_;
  return VD_OK;
}

vd_status vd_get_seeds(vd_handle h, uint16_t* out_xy) {
  CHECK_HANDLE(h);
  if (!out_xy) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  std::vector<uint32_t> p(h->s);
  CK(cudaMemcpyAsync(p.data(), h->seeds, h->s * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
  if (vd_status st_ = sync_stream(h)) return st_;
  for (uint64_t i = 0; i < h->s; ++i) {
    out_xy[2 * i] = (uint16_t)(p[i] & 0xFFFFu);
    out_xy[2 * i + 1] = (uint16_t)(p[i] >> 16);
  }
  return VD_OK;
}

vd_status vd_band(vd_handle h, uint32_t* row0, uint32_t* rows) {
  if (!h || !row0 || !rows) return VD_ERR_ARG;
  if (h->world > 1) {
    *row0 = h->shards[0].row0;
    *rows = h->shards[0].rows;
  } else {
    *row0 = 0;
    *rows = h->N;
  }
  return VD_OK;
}

vd_status vd_last_passes(vd_handle h, uint32_t* passes) {
  if (!h || !passes) return VD_ERR_ARG;
  *passes = h->last_passes;
  return VD_OK;
}

vd_status vd_last_packed_passes(vd_handle h, uint32_t* passes) {
  CHECK_HANDLE(h);
  if (!passes) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  uint32_t flags[kLocSlots];
  if (vd_status st_ = sync_stream(h)) return st_;
  CK(cudaMemcpy(flags, h->loc, sizeof flags, cudaMemcpyDeviceToHost));
  uint32_t n = 0;
  for (const auto& p : h->loc_last)
    if (p.first >= 0 && p.second <= (uint32_t)vdk::kPackMaxK && flags[p.first] == 0u) ++n;
  *passes = n;
  return VD_OK;
}

vd_status vd_synchronize(vd_handle h) {
  CHECK_HANDLE(h);
  DeviceGuard guard(h->device);
  if (vd_status st_ = sync_stream(h)) return st_;
  return VD_OK;
}

vd_status vd_set_pass_timing(vd_handle h, int enable) {
  CHECK_HANDLE(h);
  h->timing = enable != 0;
  return VD_OK;
}

vd_status vd_pass_timing(vd_handle h, double* ms, uint64_t* launches, uint64_t* pixels) {
  CHECK_HANDLE(h);
  DeviceGuard guard(h->device);
  if (vd_status st_ = sync_stream(h)) return st_;
  double total = 0.0;
  uint64_t passes = 0;
  for (size_t i = 0; i + 1 < h->ev_used; i += 2) {
    if (h->ev_k[i / 2] == 0) continue;  // a remap interval, not a pass
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, h->ev[i], h->ev[i + 1]));
    total += t;
    ++passes;
  }
  if (ms) *ms = total;
  if (launches) *launches = passes;
  if (pixels) *pixels = h->timed_px;
  h->ev_used = 0;
  h->timed_launches = 0;
  h->timed_px = 0;
  return VD_OK;
}

vd_status vd_pass_times(vd_handle h, float* ms, uint32_t* ks, uint32_t cap, uint32_t* n) {
  CHECK_HANDLE(h);
  if (!n) return VD_ERR_ARG;
  DeviceGuard guard(h->device);
  if (vd_status st_ = sync_stream(h)) return st_;
  const uint32_t cnt = (uint32_t)(h->ev_used / 2);
  *n = cnt;
  for (uint32_t i = 0; i < cnt && i < cap; ++i) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, h->ev[2 * i], h->ev[2 * i + 1]));
    if (ms) ms[i] = t;
    if (ks) ks[i] = h->ev_k[i];
  }
  return VD_OK;
}

vd_status vd_launch_count(vd_handle h, uint64_t* n) {
  if (!h || !n) return VD_ERR_ARG;
  *n = h->launches;
  return VD_OK;
}

}  // extern "C"
