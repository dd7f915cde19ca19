// vd_kernels.cuh -- sm_100a kernels of the dJFA hot path (arXiv 2209.00117).
//
// "P:n" = line n of the paper's LaTeX source; "R-n" = reading n in DESIGN.md §3.
// Independent of oracle/: nothing here is shared with, or derived from, the CPU oracle.
//
// Label: uint32 (y << 16) | x of the claimed seed (R-1); EMPTY = 0xFFFFFFFF (R-4).
// Diagram rows are padded to `pitch` labels (a multiple of 32 -> 128-B aligned rows), so
// every thread moves 4 labels with one 128-bit load / store.
#pragma once
#include <cstdint>
#include <cuda.h>  // CUtensorMap (type only; the map is encoded on the host through the runtime's driver entry point)
#include <cuda_runtime.h>

namespace vdk {

constexpr uint32_t EMPTY = 0xFFFFFFFFu;
#ifndef VD_VEC
#define VD_VEC 4               // labels per thread in the fast pass (2 or 4): one 64/128-bit access
#endif
constexpr int kVec = VD_VEC;
constexpr int kThreads = 512 / kVec;  // threads per CTA of the fast pass: a CTA covers 512 columns
#ifndef VD_MIN_BLOCKS
#define VD_MIN_BLOCKS 4        // CTAs per SM the register allocation must allow (VEC=4: 128 regs, a few spills)
#endif

// ------------------------------------------------------------------ arguments

// One jump pass over a band of rows [row0, row0 + rows) of the N x N grid.
// Global row r of the INPUT diagram lives in
//   in  + (r - row0)     * pitch   if row0 <= r < row0 + rows      (own band)
//   top + (r - top_row0) * pitch   if r < row0                     (halo from rank above)
//   bot + (r - bot_row0) * pitch   if r >= row0 + rows             (halo from rank below)
// (vd.h vd_halo_plan).  With one band (row0 = 0, rows = N) the halos are never touched.
struct PassArgs {
  const uint32_t* __restrict__ in;
  const uint32_t* __restrict__ top;
  const uint32_t* __restrict__ bot;
  uint32_t* __restrict__ out;
  int64_t pitch;
  int32_t N, row0, rows, top_row0, bot_row0, k;
  int32_t y_lo, y_hi;  // output rows [y_lo, y_hi) (global), inside the band: the whole band, or the
                       // interior / an edge strip when the halo exchange is overlapped
  int32_t lk;       // log2(k) (fast pass: k is a power of two)
  int32_t segs;     // walk segments per residue class: ceil(ceil(rows / k) / walk)
  int32_t walk;     // output rows per walk (walk_len(k))
  int32_t xblocks;  // CTAs across one row: ceil(N / (4 * kThreads))
  int32_t res_in_y; // grid order: 0 = (x-block, segment, residue), 1 = (x-block, residue, segment),
                    // 2 = (residue, x-block, segment) (jump_pass_sk_remap only)
  int32_t nwalk;    // jump_pass_sk: > 0 = whole residue classes, nwalk of them per CTA (FULL walks)
  int32_t tmap;     // jump_pass_sk, k >= 256, one band: stage each row's six spans with ONE tensor copy
  const uint32_t* fwd;  // jump_pass_sk_remap: the forward map (old seed position -> new label), indexed by the label
  int32_t prefetch;     // jump_pass_sk_remap: also pull the fwd lines of the row after next into L1
  unsigned long long* hash_out;  // jump_pass_sk<1> HASH: add the outputs' label checksum here
  // jump_pass_sk: also restore fwd[rst_seeds[i]] = EMPTY for i < rst_s (the fused dJFA frame's
  // fwd reset, folded into its second pass: a few scattered stores per CTA, hidden behind staging)
  uint32_t* rst_fwd;
  const uint32_t* rst_seeds;
  int64_t rst_s;
  // jump_pass_sk LAT (JFA's steps with N <= 64k): every input label is congruent to its pixel mod 2k,
  // so candidates are evaluated in lattice units (coordinate >> log2 k) by the packed walk; EMPTY and
  // the virtual far seed map to the lattice point (127, 127); lat_empty = the unclaimed label to output
  int32_t lat;         // 0 off, 1 lattice walk with unclaimed labels possible, 2 none possible
  uint32_t lat_empty;  // the unclaimed label (EMPTY, or the virtual far seed)
  uint32_t lat_min;    // labels >= lat_min are unclaimed (N << 16, or EMPTY at N = 65536)
  uint32_t lat_vl;     // lat 3: the lattice stand-in for unclaimed labels, (2L+1, 2L+1) for lattice size L
  uint32_t vempty;  // in-kernel stand-in for EMPTY (MAY_EMPTY variant), see jump_pass_fast
  uint32_t sh16;    // 65536 (a run-time value on purpose)
  uint32_t one;     // 1 (a run-time value on purpose: keeps x*1+y an IMAD on the FMA pipe)
  int32_t metric;   // 0 Euclidean, 1 Manhattan (jump_pass_wide; the fast kernel templates it)
  int32_t vn;       // Von Neumann neighbourhood (jump_pass_wide)
  unsigned long long* empty_flag;  // jump_pass_wide: set non-zero if any output is EMPTY (or null)
  // Fused halo push (peer halos, NEXT-3): output rows [row0, row0 + push_k) are also stored
  // into the band above's bottom halo (push_top, row y at y - row0) and rows
  // [row0 + rows - push_k, row0 + rows) into the band below's top halo (push_bot, row y at
  // y - (row0 + rows - push_k)); peer memory when the bands live on other GPUs.
  uint32_t* push_top;
  uint32_t* push_bot;
  int32_t push_k;
  // Locality flags (packed-key pass, see walk): loc_in -> 0 iff every label of the INPUT lies
  // within Euclidean distance kLocR of its own pixel (written by the previous kernel of the
  // frame); null = unknown.  loc_out (or null): set to 1 if some OUTPUT label may lie farther.
  const uint32_t* loc_in;
  uint32_t* loc_out;
};

// Locality radius of the packed-key pass: with every input label within kLocR of its pixel
// and k <= kPackMaxK, every candidate of every pixel has |dx|, |dy| <= kLocR + k <= 127.
constexpr int kLocR = 63;
constexpr int kPackMaxK = 64;
constexpr uint32_t kLocD2 = (uint32_t)kLocR * kLocR;  // d2 bound of a "local" label

// Store one output vector of row y (band-local pointer po) and, for the rows a neighbour's
// next pass reads as halo, the same vector into its halo buffer.
template <typename V>
__device__ __forceinline__ void store_out(const PassArgs& a, bool banded, int y, int x, uint32_t* po, const V& v) {
  *reinterpret_cast<V*>(po) = v;
  if (banded && a.push_k) {
    if (a.push_top && y < a.row0 + a.push_k)
      *reinterpret_cast<V*>(a.push_top + (int64_t)(y - a.row0) * a.pitch + x) = v;
    const int b0 = a.row0 + a.rows - a.push_k;
    if (a.push_bot && y >= b0) *reinterpret_cast<V*>(a.push_bot + (int64_t)(y - b0) * a.pitch + x) = v;
  }
}

__device__ __forceinline__ const uint32_t* row_ptr(const PassArgs& a, int r) {
  if (r >= a.row0 && r < a.row0 + a.rows) return a.in + (int64_t)(r - a.row0) * a.pitch;
  if (r < a.row0) return a.top + (int64_t)(r - a.top_row0) * a.pitch;
  return a.bot + (int64_t)(r - a.bot_row0) * a.pitch;
}

__device__ __forceinline__ uint4 ld4(const uint32_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

__device__ __forceinline__ uint32_t get(const uint4& v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

// ------------------------------------------------------------------ fast jump pass
//
// out[p] = argmin over c in {in[p]} U {in[p + o*k] : o in Table 1, p + o*k in
// the grid} of key(p, c) = (d2(p, c), c) lexicographically ("the distance function
// is used as a criterion to check which flood carries the closest seed"; R-2, R-3, R-11).
//
// Shape (B200-first, not the paper's one-thread-per-pixel launch of P:204):
//  * a thread owns 4 adjacent columns x..x+3 (one 128-bit load/store per row) and walks
//    down its residue class y, y+k, y+2k, ... for up to kMaxWalk output rows, keeping the three
//    input rows y-k, y, y+k in registers: each step loads ONE new row (3 x LDG.128: the
//    columns x-k, x, x+k), so every input label is fetched once per thread and serves
//    the three outputs above/at/below it;
//  * per label, dx^2 to its output column is computed once when the row is loaded and
//    reused by the three outputs (dy differs);
//  * CTAs are ordered x-fastest, then consecutive walk segments of one residue class, so
//    the x +- k neighbours of a row are fetched by CTAs running at the same time (L2 hits)
//    and DRAM sees each input label about once (8 B per pixel per pass).
//  * Out-of-grid neighbours are replaced by a label that is already a candidate (the
//    pixel's own column in the same row, or the centre row): a duplicate candidate cannot
//    change a minimum, so no per-candidate validity test is needed.
//  * Integer pipes: the per-pixel work is ~9 x (dy, d2, tie) + 2 nine-way minima, all
//    exact 32-bit integer ops.  Distances run on the FMA pipe (IMAD, IMAD.HI), the
//    tie-break and minima on the ALU pipe (VIADDMNMX, VIMNMX3), so both pipes share the
//    load:  dx<<16 = IMAD(c, 2^16, -x<<16) (exact while |dx| < 2^15), dx^2 = mulhi(D, D);
//    dy = mad.hi(c, 2^16, -y) = (c >> 16) - y; d2 = IMAD(dy, dy, dx^2).
//  * Tie-break without 64-bit compares ("resolve later"): m = min_i d2_i, then
//    out = min_i max(c_i, m - d2_i) in uint32.  For d2_i = m the term is c_i; for
//    d2_i > m, m - d2_i wraps to >= 2^31, above every label in use (< 2^31).
//    Requires N <= 32768 (so d2 < 2^31 and y < 2^15).
//  * MAY_EMPTY (JFA passes): EMPTY is first mapped to the virtual label vempty =
//    (C << 16) | C, C = 2N - 1 <= 32767: a point farther from every pixel than any real
//    seed (min d2 = 2 N^2 > 2 (N-1)^2), still a label < 2^31 above every real label, and
//    mapped back to EMPTY on store.  Requires N <= 16384.
// One input row as seen by one thread, for its kVec output columns x..x+kVec-1: for each
// output column e, the labels of input columns x+e-k (L), x+e (C), x+e+k (R), and per
// label cy and Q = cy^2 + (cx - (x+e))^2.  For an output pixel (x+e, y) every candidate
// then has d2 - y^2 = Q - 2 y cy: ONE integer multiply-add per candidate, and since y^2
// is common to the nine candidates of a pixel the minimum and every difference m - d2
// (hence the tie-break) are unchanged.
struct Row {
  uint32_t c[3 * kVec];  // labels: [0, kVec) L, [kVec, 2 kVec) C, [2 kVec, 3 kVec) R
  int32_t cy[3 * kVec];  // c >> 16
  int32_t q[3 * kVec];   // cy^2 + (cx - (x+e))^2
};

__device__ __forceinline__ uint32_t mad_hi_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// ---- shared-memory row staging with cp.async.bulk (TMA bulk copies) -----------------
constexpr int kW = kVec * kThreads;      // columns per CTA (512)
#ifndef VD_MAX_WALK
#define VD_MAX_WALK 24
#endif
#ifndef VD_SMEM_KB
#define VD_SMEM_KB 56
#endif
#ifndef VD_REL_MAX_WALK
#define VD_REL_MAX_WALK 32
#endif
#ifndef VD_REL_SMEM_KB
#define VD_REL_SMEM_KB 72
#endif
constexpr int kMaxWalk = VD_MAX_WALK;    // output rows per walk (upper bound)
constexpr int kSmemBudget = VD_SMEM_KB * 1024;  // staged rows per CTA
// The windowed variant (REL) runs 3 CTAs per SM (its extra live values spill at 4), so each
// CTA can stage more rows: longer walks amortise the two extra staged rows per walk.
constexpr int kMaxWalkRel = VD_REL_MAX_WALK;
constexpr int kSmemBudgetRel = VD_REL_SMEM_KB * 1024;

// Elements of one staged input row: columns [x0 - K4, x0 + W + K4) when k < W (K4 = k
// rounded up to 4), else three W-wide spans at x0 - k, x0, x0 + k.
__host__ __device__ inline int stage_elems(int k) {
  return k >= kW ? 3 * kW : kW + 2 * ((k + 3) & ~3);
}
// Output rows per walk so that walk + 2 staged rows fit the budget.
__host__ __device__ inline int walk_len(int k, bool rel = false) {
  const int rows = (rel ? kSmemBudgetRel : kSmemBudget) / (stage_elems(k) * 4 + 8);
  const int mx = rel ? kMaxWalkRel : kMaxWalk;
  return rows - 2 < 1 ? 1 : (rows - 2 > mx ? mx : rows - 2);
}
__host__ __device__ inline size_t pass_smem(int k, bool rel = false) {
  return (size_t)(walk_len(k, rel) + 2) * (stage_elems(k) * 4 + 8);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// One lane of the (converged) warp: elect.sync.
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile(
      "{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(e));
  return e != 0u;
}

template <int V>
struct VecT;
template <>
struct VecT<2> { using T = uint2; };
template <>
struct VecT<4> { using T = uint4; };

__device__ __forceinline__ void unpack(const uint2& v, uint32_t* w) { w[0] = v.x; w[1] = v.y; }
__device__ __forceinline__ void unpack(const uint4& v, uint32_t* w) { w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w; }

// Build one Row from a staged input row.  li / ci / ri: element offsets of the left /
// centre / right vectors in the stage.  KM = min(k, kVec): KM == kVec means the neighbour
// vectors at x -+ k are aligned; KM < kVec takes the neighbours from the adjacent vectors.
// METRIC 0: Euclidean (q = cy^2 + dx^2); METRIC 1: Manhattan, dJFAm (q = |dx|).
// REL (grids wider than 32768): labels are first moved into the CTA's 32768-wide window,
// c' = (cy - oy, cx - ox) as two 16-bit lanes (nbase2 = -(oy, ox)); a label outside the
// window sets bit 15 of a lane, which `bad` accumulates (the walk is then recomputed
// exactly).  xr = x - ox is the thread's column in the window.
template <int KM, bool MAY_EMPTY, bool FIX, int METRIC, bool REL = false>
__device__ __forceinline__ void row_from_smem(const uint32_t* __restrict__ st, int li, int ci, int ri, int x, int k,
                                              int N, uint32_t vempty, uint32_t sh16, const int (&xs16)[kVec], Row& R,
                                              uint32_t nbase2 = 0, uint32_t* bad = nullptr, int xr = 0) {
  using V = typename VecT<kVec>::T;
  uint32_t w[3 * kVec];
  unpack(*reinterpret_cast<const V*>(st + li), w);
  unpack(*reinterpret_cast<const V*>(st + ci), w + kVec);
  unpack(*reinterpret_cast<const V*>(st + ri), w + 2 * kVec);
#pragma unroll
  for (int e = 0; e < kVec; ++e) {
    if constexpr (KM >= kVec) { R.c[e] = w[e]; R.c[2 * kVec + e] = w[2 * kVec + e]; }
    else { R.c[e] = w[kVec + e - KM]; R.c[2 * kVec + e] = w[kVec + e + KM]; }
    R.c[kVec + e] = w[kVec + e];
  }
  if constexpr (FIX) {  // an out-of-grid column -> the pixel's own column (a duplicate)
#pragma unroll
    for (int e = 0; e < kVec; ++e) {
      if (x + e - k < 0) R.c[e] = w[kVec + e];
      if (x + e + k >= N) R.c[2 * kVec + e] = w[kVec + e];
    }
  }
#pragma unroll
  for (int i = 0; i < 3 * kVec; ++i) {
    uint32_t c = R.c[i];
    if (MAY_EMPTY && !REL) { c = __vminu2(c, vempty); R.c[i] = c; }  // EMPTY -> virtual far seed
    if constexpr (REL) {  // window coordinates (no EMPTY on this path)
      c = __vadd2(c, nbase2);
      R.c[i] = c;
      *bad |= c;
    }
    // uint32 arithmetic throughout (wrapping is defined; labels outside a window give
    // don't-care values there, never undefined behaviour)
    const uint32_t cy = c >> 16;
    R.cy[i] = (int)cy;
    if constexpr (METRIC == 0) {
      const uint32_t D = c * sh16 + (uint32_t)xs16[i % kVec];  // (cx - (x+e)) << 16  (exact, |dx| < 2^15)
      const int dx = (int)D >> 16;                                // cx - (x+e)
      R.q[i] = (int)(cy * cy + (uint32_t)(dx * dx));              // cy^2 + dx^2
    } else {
      R.q[i] = (int)__sad((int)(c & 0xFFFFu), (REL ? xr : x) + (i % kVec), 0u);  // |cx - (x+e)|
    }
  }
}

// Output label of pixel (x+e, y): candidates = column e of the three rows (Moore), or
// only the centre column of the rows above / below plus the centre row (Von Neumann,
// P:154-160).  Euclidean: d'_i = d2_i - y^2 = Q_i - 2 y cy_i (int32, may be negative; y^2
// is common to all candidates of the pixel).  Manhattan: d_i = |cy_i - y| + |dx_i|.
// m = min d_i (signed), then out = min_i max(c_i, m - d_i) in uint32 -- for d_i = m the
// term is c_i, for d_i > m the difference wraps to >= 2^31, above every label in use
// (< 2^31).
template <int METRIC, bool VN>
__device__ __forceinline__ uint32_t best_of(const Row& A, const Row& B, const Row& Cn, int e, int y, int& mo) {
  constexpr int n = VN ? 5 : 9;
  uint32_t c[9];
  int d[9];
  auto dist = [&](const Row& R, int i) -> int {
    if constexpr (METRIC == 0) return (int)((uint32_t)R.q[i] + (uint32_t)R.cy[i] * (uint32_t)(-2 * y));
    else return (int)__sad(R.cy[i], y, (unsigned)R.q[i]);
  };
  if constexpr (!VN) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      c[j] = A.c[kVec * j + e];     d[j] = dist(A, kVec * j + e);
      c[3 + j] = B.c[kVec * j + e]; d[3 + j] = dist(B, kVec * j + e);
      c[6 + j] = Cn.c[kVec * j + e]; d[6 + j] = dist(Cn, kVec * j + e);
    }
  } else {
    c[0] = A.c[kVec + e];  d[0] = dist(A, kVec + e);
    c[1] = Cn.c[kVec + e]; d[1] = dist(Cn, kVec + e);
#pragma unroll
    for (int j = 0; j < 3; ++j) { c[2 + j] = B.c[kVec * j + e]; d[2 + j] = dist(B, kVec * j + e); }
  }
  int m;
  if constexpr (VN) m = __vimin3_s32(__vimin3_s32(d[0], d[1], d[2]), d[3], d[4]);
  else m = __vimin3_s32(__vimin3_s32(d[0], d[1], d[2]), __vimin3_s32(d[3], d[4], d[5]), __vimin3_s32(d[6], d[7], d[8]));
  mo = m;
  uint32_t w[9];
#pragma unroll
  for (int i = 0; i < n; ++i) w[i] = __viaddmax_u32((uint32_t)m, 0u - (uint32_t)d[i], c[i]);  // max(m - d_i, c_i)
  if constexpr (VN) return __vimin3_u32(__vimin3_u32(w[0], w[1], w[2]), w[3], w[4]);
  else return __vimin3_u32(__vimin3_u32(w[0], w[1], w[2]), __vimin3_u32(w[3], w[4], w[5]),
                           __vimin3_u32(w[6], w[7], w[8]));
}

// ---- packed-key pass (labels local to their pixels: dJFA after the remap) -----------
// When every candidate of a pixel (X, y) has |dx|, |dy| <= 127 (dx = cx - X, dy = cy - y),
// the lexicographic key (d2, c) of R-3 -- for a fixed pixel the same order as (d2, dy, dx) --
// fits ONE 31-bit integer:
//   key = d2 * 2^16 + (dy + 128) * 2^8 + (dx + 128),   d2 <= 2 * 127^2 < 2^15,
// so a single nine-way minimum (no tie-break pass) picks the winner, and its label is
// recovered from the key's low bytes: ((y + dy) << 16) | (X + dx).  Per label (once per
// staged row) Qk = (cy^2 + dx^2) * 2^16 + dx; per candidate ONE IMAD, Qk + cy * M_y with
// M_y = 256 - 2y * 2^16, gives key - C_y (mod 2^32), C_y = y^2 2^16 - 256 y + 32896 common to
// the pixel's candidates.  Those values lie in [-C_y, -C_y + 2^31) mod 2^32, an interval that
// does not wrap as unsigned when -C_y <= 2^31 and as signed otherwise; the comparison kind is
// chosen per output row (y is uniform over the CTA).
// Manhattan (dJFAm), METRIC 1: key = d * 2^16 + (dy + 128) * 2^8 + (dx + 128) with
// d = |dx| + |dy| <= 254.  Per label Qm = |dx| * 2^16 + dx + 256 cy, kept with chi = cy << 16;
// per candidate ONE VABSDIFF, |chi - (y << 16)| + Qm = key - C'_y, C'_y = 32896 - 256 y.
template <int KM, bool FIX, int METRIC = 0>
__device__ __forceinline__ void row_packed(const uint32_t* __restrict__ st, int li, int ci, int ri, int x, int k, int N,
                                           uint32_t sh16, const int (&xs16p)[kVec], Row& R) {
  using V = typename VecT<kVec>::T;
  uint32_t w[3 * kVec];
  uint32_t c[3 * kVec];
  unpack(*reinterpret_cast<const V*>(st + li), w);
  unpack(*reinterpret_cast<const V*>(st + ci), w + kVec);
  unpack(*reinterpret_cast<const V*>(st + ri), w + 2 * kVec);
#pragma unroll
  for (int e = 0; e < kVec; ++e) {
    if constexpr (KM >= kVec) { c[e] = w[e]; c[2 * kVec + e] = w[2 * kVec + e]; }
    else { c[e] = w[kVec + e - KM]; c[2 * kVec + e] = w[kVec + e + KM]; }
    c[kVec + e] = w[kVec + e];
  }
  if constexpr (FIX) {
#pragma unroll
    for (int e = 0; e < kVec; ++e) {
      if (x + e - k < 0) c[e] = w[kVec + e];
      if (x + e + k >= N) c[2 * kVec + e] = w[kVec + e];
    }
  }
  if constexpr (METRIC == 1) {
#pragma unroll
    for (int i = 0; i < 3 * kVec; ++i) {
      const uint32_t chi = c[i] & 0xFFFF0000u;                          // cy << 16
      const uint32_t D = c[i] * sh16 + (uint32_t)(xs16p[i % kVec] - 1);  // (cx - X) << 16
      const int dx = (int)D >> 16;
      R.cy[i] = (int)chi;
      R.q[i] = (int)(__sad((int)D, 0, (uint32_t)dx) + (chi >> 8));     // |dx| << 16 + dx + 256 cy
    }
  } else {
#pragma unroll
  for (int i = 0; i < 3 * kVec; ++i) {
    const uint32_t cy = c[i] >> 16;
    const uint32_t D1 = c[i] * sh16 + (uint32_t)xs16p[i % kVec];  // (cx - X) << 16 | 1
    const uint32_t dx = (uint32_t)((int)D1 >> 16);
    R.cy[i] = (int)cy;
#ifdef VD_CHI_IMAD
    const uint32_t chi = cy * sh16;  // cy << 16 on the FMA pipe (experiment knob)
#else
    const uint32_t chi = c[i] & 0xFFFF0000u;  // cy << 16
#endif
    R.q[i] = (int)(dx * D1 + cy * chi);  // (dx^2 + cy^2) << 16 + dx  (mod 2^32)
  }
  }
}

template <bool SIGNED, int METRIC = 0>
__device__ __forceinline__ uint32_t min9_packed(const Row& A, const Row& B, const Row& Cn, int e, uint32_t My) {
  uint32_t kk[9];
  auto key = [&](const Row& R, int i) -> uint32_t {
    if constexpr (METRIC == 1) return __usad((uint32_t)R.cy[i], My, (uint32_t)R.q[i]);  // My = y << 16
    else return (uint32_t)R.q[i] + (uint32_t)R.cy[i] * My;
  };
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    kk[j] = key(A, kVec * j + e);
    kk[3 + j] = key(B, kVec * j + e);
    kk[6 + j] = key(Cn, kVec * j + e);
  }
  if constexpr (SIGNED)
    return (uint32_t)__vimin3_s32(__vimin3_s32((int)kk[0], (int)kk[1], (int)kk[2]),
                                  __vimin3_s32((int)kk[3], (int)kk[4], (int)kk[5]),
                                  __vimin3_s32((int)kk[6], (int)kk[7], (int)kk[8]));
  else
    return __vimin3_u32(__vimin3_u32(kk[0], kk[1], kk[2]), __vimin3_u32(kk[3], kk[4], kk[5]),
                        __vimin3_u32(kk[6], kk[7], kk[8]));
}

// Exact candidate test, key (distance, label) with EMPTY = +infinity, metric fixed at compile
// time: |dx|, |dy| <= 65535, so each square fits 32 bits and only the sum needs 33 (uint64).
template <int METRIC>
__device__ __forceinline__ void consider64(uint32_t c, int x, int y, uint64_t& bd, uint32_t& bc) {
  if (c == EMPTY) return;
  const uint32_t dx = (uint32_t)abs((int)(c & 0xFFFFu) - x), dy = (uint32_t)abs((int)(c >> 16) - y);
  const uint64_t d = METRIC == 0 ? (uint64_t)(dx * dx) + (uint64_t)(dy * dy) : (uint64_t)(dx + dy);
  if (d < bd || (d == bd && c < bc)) { bd = d; bc = c; }
}

// One CTA = 512 columns x one walk (up to kMaxWalk output rows of one residue class
// y0, y0+k, ...).  At entry, thread 0 stages ALL of the walk's input rows
// y0-k, y0, ..., y_last+k into shared memory with cp.async.bulk, one mbarrier per row;
// the threads then consume the rows in order as they land -- no ring, no refills, no block
// barriers in the loop.  Every thread turns a staged row into registers (Row) once and the
// three row registers rotate as in a column walk.  Rows outside the grid are replaced by
// the centre row (the producer stages that row again), columns outside the grid by the
// pixel's own column: duplicates never change a minimum.
// BANDED: rows beyond the band come from the halo buffers (row_ptr).
// PACK: the packed-key evaluation (row_packed / min9_packed), taken when the input's locality
// flag is clear and k <= kPackMaxK.  LOC variants (Euclidean Moore, one band) also report the
// output's locality into a.loc_out.
template <int KM, bool MAY_EMPTY, bool BANDED, bool FIX, int METRIC, bool VN, bool REL, bool PACK>
__device__ __forceinline__ void walk(const PassArgs& a, int x0, int y0, uint32_t* smem) {
  const int k = a.k, N = a.N;
  const int tid = (int)threadIdx.x;
  const int x = x0 + kVec * tid;
  const int yend = a.y_hi;
  const int nout = min(a.walk, (yend - y0 + k - 1) >> a.lk);  // output rows of this walk (k = 2^lk)
  const int nlist = nout + 2;                              // staged input rows
  const bool spans3 = k >= kW;
  const int K4 = (k + 3) & ~3;
  const int SE = stage_elems(k);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)(a.walk + 2) * SE);

  if (tid < nlist) mbar_init(&bars[tid], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();  // barrier initialisation visible to every thread (and to the async proxy)
  {  // warp w stages every kThreads/32-th row, in row order; one elected lane issues the copies
    // (the loop is warp-uniform, so the copy operands stay in uniform registers)
    const int warp = __shfl_sync(0xFFFFFFFFu, tid >> 5, 0);
    const int P = (int)a.pitch;
    const int base = x0 - K4;
    const int lo = max(base, 0), hi = min(x0 + kW + K4, P);
    const int lL = max(x0 - k, 0), hL = min(x0 - k + kW, P);
    const int hC = min(x0 + kW, P);
    const int lR = max(x0 + k, 0), hR = min(x0 + k + kW, P);
    const uint32_t tx = spans3 ? 4u * (uint32_t)(max(hL - lL, 0) + (hC - x0) + max(hR - lR, 0)) : (uint32_t)(hi - lo) * 4u;
    if (!BANDED && !spans3) {
      // one band, whole rows: the warp's rows i = warp, warp + W, ... advance by constant
      // strides (W = kThreads/32 rows of k grid rows each); a row outside the grid is the centre
      // row again (k rows back or forward)
      constexpr int W = kThreads / 32;
      const int64_t kp = (int64_t)k * a.pitch;
      int r = y0 + (warp - 1) * k;
      const uint32_t* src = a.in + (int64_t)(r - a.row0) * a.pitch + lo;
      uint32_t dst = smem_u32(smem + (size_t)warp * SE + (lo - base));
      uint32_t bar = smem_u32(&bars[warp]);
      const uint32_t bytes = (uint32_t)(hi - lo) * 4u;
      for (int i = warp; i < nlist; i += W, r += W * k, src += W * kp, dst += W * SE * 4, bar += W * 8) {
        const uint32_t* s = r < 0 ? src + kp : (r >= N ? src - kp : src);
        if (elect_one()) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
              "l"(s), "r"(bytes), "r"(bar)
              : "memory");
        }
        __syncwarp();
      }
    } else for (int i = warp; i < nlist; i += kThreads / 32) {
      int r = y0 + (i - 1) * k;       // outside the grid: stage the centre row again
      if (r < 0) r += k;
      else if (r >= N) r -= k;
      const uint32_t* src = BANDED ? row_ptr(a, r) : a.in + (int64_t)(r - a.row0) * a.pitch;
      uint32_t* dst = smem + (size_t)i * SE;
      if (elect_one()) {
        mbar_expect_tx(&bars[i], tx);
        if (!spans3) {
          bulk_g2s(dst + (lo - base), src + lo, (uint32_t)(hi - lo) * 4u, &bars[i]);
        } else {
          if (lL < hL) bulk_g2s(dst + (lL - (x0 - k)), src + lL, (uint32_t)(hL - lL) * 4u, &bars[i]);
          bulk_g2s(dst + kW, src + x0, (uint32_t)(hC - x0) * 4u, &bars[i]);
          if (lR < hR) bulk_g2s(dst + 2 * kW + (lR - (x0 + k)), src + lR, (uint32_t)(hR - lR) * 4u, &bars[i]);
        }
      }
      __syncwarp();
    }
  }

  // vector offsets in a stage (out-of-grid neighbour vectors -> the centre vector)
  const int nstep = KM >= kVec ? k : kVec;  // distance to the neighbour vectors
  const int ci = spans3 ? kW + kVec * tid : K4 + kVec * tid;
  const int li = (x - nstep >= 0) ? (spans3 ? kVec * tid : ci - nstep) : ci;
  const int ri = (x + nstep < N) ? (spans3 ? 2 * kW + kVec * tid : ci + nstep) : ci;
  const uint32_t sh16 = a.sh16;  // 65536, from memory so ptxas keeps the multiply on the FMA pipe
  // REL: the window origin (ox, oy) in [0, max(N-32768, 0)]^2, centred on the walk where the
  // grid allows, so that a label outside the window always sets bit 15 of a 16-bit lane
  // after the subtraction.
  int ox = 0, oy = 0;
  if constexpr (REL && !PACK) {
    const int omax = max(N - 32768, 0);  // window kept inside the grid
    ox = min(max(x0 + kW / 2 - 16384, 0), omax);
    oy = min(max(y0 + ((nout - 1) * k) / 2 - 16384, 0), omax);
  }
  const uint32_t base2 = ((uint32_t)oy << 16) | (uint32_t)ox;
  const uint32_t nbase2 = __vsub2(0u, base2);
  uint32_t bad = 0;
  int xs16[kVec];
#pragma unroll
  for (int e = 0; e < kVec; ++e) xs16[e] = -((x - ox + e) << 16);
  int xs16p[kVec], xb[kVec];
#pragma unroll
  for (int e = 0; e < kVec; ++e) { xs16p[e] = 1 - ((x + e) << 16); xb[e] = x + e - 128; }
  const bool active = x < N;
  constexpr bool LOC = !VN;
  uint32_t loc_acc = 0;    // PACK: max true key of this thread's outputs
  bool loc_bad = false;    // exact path: some output label farther than kLocR

  auto consume = [&](int i, Row& R) {
    mbar_wait(&bars[i], 0u);
    if constexpr (PACK) row_packed<KM, FIX, METRIC>(smem + (size_t)i * SE, li, ci, ri, x, k, N, sh16, xs16p, R);
    else
      row_from_smem<KM, MAY_EMPTY, FIX, METRIC, REL>(smem + (size_t)i * SE, li, ci, ri, x, k, N, a.vempty, sh16, xs16,
                                                     R, nbase2, &bad, x - ox);
  };

  Row r0, r1, r2;
  consume(0, r0);
  consume(1, r1);
  int y = y0;
  uint32_t* po = a.out + (int64_t)(y0 - a.row0) * a.pitch + x;
  const int64_t kp = (int64_t)k * a.pitch;
  int j = 0;
  // Output row j: P = row j (y-k), C = row j+1 (y), Nx <- row j+2 (y+k).
  using V = typename VecT<kVec>::T;
  auto step = [&](const Row& P, const Row& C, Row& Nx) -> bool {
    consume(j + 2, Nx);
    uint32_t o[kVec];
    if constexpr (PACK) {
      const uint32_t uy = (uint32_t)y;
      // Euclidean: M_y, C_y of row_packed's note; Manhattan: y << 16 and C'_y
      const uint32_t My = METRIC == 1 ? uy << 16 : 256u - (uy << 17);
      const uint32_t Cy = METRIC == 1 ? 32896u - 256u * uy : uy * uy * 65536u - 256u * uy + 32896u;
      const uint32_t Yb = (uy - 128u) << 16;
      uint32_t sk[kVec];
      if (0u - Cy <= 0x80000000u) {
#pragma unroll
        for (int e = 0; e < kVec; ++e) sk[e] = min9_packed<false, METRIC>(P, C, Nx, e, My) + Cy;
      } else {
#pragma unroll
        for (int e = 0; e < kVec; ++e) sk[e] = min9_packed<true, METRIC>(P, C, Nx, e, My) + Cy;
      }
#pragma unroll
      for (int e = 0; e < kVec; ++e) o[e] = __byte_perm(sk[e], 0u, 0x4140) + Yb + (uint32_t)xb[e];
      if constexpr (kVec == 4) loc_acc = __vimax3_u32(__vimax3_u32(loc_acc, sk[0], sk[1]), sk[2], sk[3]);
      else loc_acc = __vimax3_u32(loc_acc, sk[0], sk[1]);
    } else {
      int mm = -0x7FFFFFFF - 1;
#pragma unroll
      for (int e = 0; e < kVec; ++e) {
        int me;
        uint32_t v = best_of<METRIC, VN>(P, C, Nx, e, y - oy, me);
        if constexpr (LOC) mm = max(mm, me);
        if (MAY_EMPTY && !REL) v = (v == a.vempty) ? EMPTY : v;
        if (REL) v = __vadd2(v, base2);  // back to absolute coordinates
        o[e] = v;
      }
      // max d2 of the row's outputs = mm + (y - oy)^2 (m = d2 - y^2, see best_of)
      if constexpr (LOC) {
        if constexpr (METRIC == 1) loc_bad |= mm > kLocR;  // m = |dy| + |dx| (>= Chebyshev)
        else loc_bad |= mm > (int)kLocD2 - (y - oy) * (y - oy);
      }
    }
    if (active) {
      if constexpr (kVec == 4) store_out(a, BANDED, y, x, po, make_uint4(o[0], o[1], o[2], o[3]));
      else store_out(a, BANDED, y, x, po, make_uint2(o[0], o[1]));
    }
    po += kp;
    y += k;
    return ++j < nout;
  };
#pragma unroll 1
  while (true) {
    if (!step(r0, r1, r2)) break;
    if (!step(r1, r2, r0)) break;
    if (!step(r2, r0, r1)) break;
  }
  if constexpr (LOC) {
    if (a.loc_out) {
      bool far;
      if constexpr (PACK) far = active && loc_acc >= (((METRIC == 1 ? (uint32_t)kLocR : kLocD2) + 1u) << 16);
      else far = active && loc_bad;
      if constexpr (REL && !PACK) far = far || (bad & 0x80008000u) != 0u;  // recomputed below: unknown
      if (__syncthreads_or(far) && tid == 0) atomicOr(a.loc_out, 1u);
    }
  }
  if constexpr (REL && !PACK) {
    // Some label of this walk lay outside the window: redo the walk exactly (64-bit keys)
    // from the staged rows, which are still in shared memory.  Never happens for a
    // converged dJFA diagram with dense seeds; keeps every grid exact.
    if (__syncthreads_or((bad & 0x80008000u) != 0u)) {
      for (int jj = 0; jj < nout; ++jj) {
        const int yy = y0 + jj * k;
        uint32_t o[kVec];
#pragma unroll
        for (int e = 0; e < kVec; ++e) {
          const int xe = x + e;
          uint64_t bd = ~0ull;
          uint32_t bc = EMPTY;
          for (int rr = -1; rr <= 1; ++rr) {
            const int r = yy + rr * k;
            if (r < 0 || r >= N) continue;
            const uint32_t* st = smem + (size_t)(jj + 1 + rr) * SE;
            for (int cc = -1; cc <= 1; ++cc) {
              if (VN && rr != 0 && cc != 0) continue;
              const int q = xe + cc * k;
              if (q < 0 || q >= N || xe >= N) continue;
              const int off = spans3 ? (cc + 1) * kW + (q - (x0 + cc * k)) : q - (x0 - K4);
              consider64<METRIC>(st[off], xe, yy, bd, bc);
            }
          }
          o[e] = bc;
        }
        if (active) {
          uint32_t* pw = a.out + (int64_t)(yy - a.row0) * a.pitch + x;
          if constexpr (kVec == 4) store_out(a, BANDED, yy, x, pw, make_uint4(o[0], o[1], o[2], o[3]));
          else store_out(a, BANDED, yy, x, pw, make_uint2(o[0], o[1]));
        }
      }
    }
  }
}

#ifndef VD_REL_MIN_BLOCKS
#define VD_REL_MIN_BLOCKS 3
#endif
template <int KM, bool MAY_EMPTY, bool BANDED, int METRIC = 0, bool VN = false, bool REL = false>
__global__ void __launch_bounds__(kThreads, REL ? VD_REL_MIN_BLOCKS : VD_MIN_BLOCKS) jump_pass_fast(PassArgs a) {
  static_assert(!(MAY_EMPTY && REL), "the windowed path takes complete diagrams only");
  extern __shared__ __align__(128) uint32_t dyn_smem[];
  // grid (xblocks, segs, residues): launched x-fastest, then the walk segments of one residue
  const int xb = (int)blockIdx.x;
  const int seg = (int)(a.res_in_y ? blockIdx.z : blockIdx.y), res = (int)(a.res_in_y ? blockIdx.y : blockIdx.z);
  const int x0 = xb * kW;
  const int y0 = a.y_lo + res + seg * a.walk * a.k;
  if (res >= a.k || y0 >= a.y_hi) return;  // uniform over the CTA
  // CTAs whose vectors can be partly outside the grid (a vector that straddles N, or
  // k < kVec at the left edge) take the per-element path; for k >= kVec and N % kVec == 0
  // a neighbour vector is either wholly inside or wholly outside the grid, and the latter
  // is exact as a centre-vector substitution.
  const int nstep = KM >= kVec ? a.k : kVec;
  const bool fix = (KM < kVec || (a.N & (kVec - 1))) && (x0 < nstep + kVec || x0 + kW + nstep + kVec > a.N);
  constexpr bool CAN_PACK = !VN && !MAY_EMPTY;
  if constexpr (CAN_PACK) {
    if (a.loc_in && a.k <= kPackMaxK && *(volatile const uint32_t*)a.loc_in == 0u) {
      if (fix) walk<KM, MAY_EMPTY, BANDED, true, METRIC, VN, REL, true>(a, x0, y0, dyn_smem);
      else walk<KM, MAY_EMPTY, BANDED, false, METRIC, VN, REL, true>(a, x0, y0, dyn_smem);
      return;
    }
  }
  if (fix) walk<KM, MAY_EMPTY, BANDED, true, METRIC, VN, REL, false>(a, x0, y0, dyn_smem);
  else walk<KM, MAY_EMPTY, BANDED, false, METRIC, VN, REL, false>(a, x0, y0, dyn_smem);
}

// MurmurHash3's 32-bit finaliser: the per-pixel term of the label checksum (label_hash).
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v) {
  __shared__ uint64_t part[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) part[wid] = v;
  __syncthreads();
  uint64_t t = 0;
  if (wid == 0) {
    t = (lane < (int)(blockDim.x >> 5)) ? part[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xFFFFFFFFu, t, o);
  }
  return t;  // valid in thread 0
}

// ------------------------------------------------------------------ shared-term jump pass (r02)
//
// The pass of jump_pass_fast (Euclidean, Moore, N % 512 == 0), with the per-row terms of each
// staged label computed ONCE for all the outputs of the thread that use it.  A label at column
// cx serves output column X as its left neighbour (X = cx + k), centre (X = cx) or right
// neighbour (X = cx - k); the three terms differ only through dx = cx - X:
//   exact:  q(dx) = cy^2 + dx^2;             q(dx -+ k) = q(dx) + k^2 -+ 2k dx
//   packed: Qk(dx) = (cy^2 + dx^2) 2^16 + dx; Qk(dx -+ k) = Qk(dx) + k^2 2^16 -+ k -+ 2k 2^16 dx
// so each further use costs one add + one IMAD instead of a six-instruction row build.
// Threads own columns so that the uses of a label fall in ONE thread:
//  * KS = k in {1, 2} ("adjacent"): columns X..X+3 (X = x0 + 4t) as in jump_pass_fast; label
//    slots s = 0 .. 3+2k hold columns X - k + s, read as three 128-bit vectors.
//  * k >= 32 ("stride", KS = 1): columns X, X+k, X+2k, X+3k, consecutive threads on
//    consecutive X (coalesced 32-bit stores); slots s = 0..5 hold columns X + (s-1) k.
//    k <= 128: a CTA covers the 512 contiguous columns [x0, x0+512) in groups of 4k;
//    k >= 256: it covers four 128-column spans x0 + j k + [0, 128), j = 0..3, and stages six
//    spans (j = -1..4) per row instead of jump_pass_fast's three 512-wide ones.
// Output e of the thread takes L = slot e, C = slot e + KS, R = slot e + 2 KS.  Results are
// identical to jump_pass_fast (same keys, same minimum); only the instruction count changes.
template <int NS>
struct RowS {
  uint32_t c[NS];  // labels (exact walk only)
  int32_t cy[NS];  // c >> 16
  int32_t qL[kVec], qC[kVec], qR[kVec];  // per output: the term of its L / C / R candidate
};

__host__ __device__ inline int stage_elems_sk(int k) { return k >= 256 ? 6 * 128 : stage_elems(k); }
// Five CTAs per SM (dJFA's stride passes, 4 <= k <= 64, and the fused first pass): <= 102
// registers and a 44-KB stage, measured 2.5-5% faster than four CTAs with 56 KB for those passes
// (and slower for the exact walk of JFA and for k <= 2, which keep four).
#ifndef VD_SMEM_KB5
#define VD_SMEM_KB5 44
#endif
constexpr int kSmemBudget5 = VD_SMEM_KB5 * 1024;
__host__ __device__ inline int walk_len_sk(int k, int budget = kSmemBudget) {
  const int rows = budget / (stage_elems_sk(k) * 4 + 8);
  return rows - 2 < 1 ? 1 : (rows - 2 > kMaxWalk ? kMaxWalk : rows - 2);
}
__host__ __device__ inline size_t pass_smem_sk(int k, int budget = kSmemBudget) {
  return (size_t)(walk_len_sk(k, budget) + 2) * (stage_elems_sk(k) * 4 + 8);
}

// Row build from the NS slot labels.  xs_home[s]: -(column of slot s) << 16 (+1 for PACK);
// xs_out[e]: the same for output column e (single-use edge slots are computed against it).
// kk = (k^2, 2k) for the exact walk, (k^2 2^16 - k, k^2 2^16 + k, 2k 2^16) for the packed one.
template <int KS, bool MAY_EMPTY, bool PACK>
__device__ __forceinline__ void build_sk(uint32_t (&lab)[4 + 2 * KS], const int (&xs_home)[4 + 2 * KS],
                                         const int (&xs_out)[kVec], uint32_t vempty, uint32_t sh16, uint32_t k2,
                                         uint32_t m1, uint32_t m2, uint32_t m3, RowS<4 + 2 * KS>& R) {
  constexpr int NS = 4 + 2 * KS;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    uint32_t c = lab[s];
    if constexpr (MAY_EMPTY && !PACK) c = __vminu2(c, vempty);  // EMPTY -> virtual far seed
    const bool hasL = s <= 3, hasC = s - KS >= 0 && s - KS <= 3, hasR = s - 2 * KS >= 0;
    const uint32_t cy = c >> 16;
    if constexpr (!PACK) R.c[s] = c;
    R.cy[s] = (int)cy;
    if constexpr (!PACK) {
      if (hasC) {
        const uint32_t D = c * sh16 + (uint32_t)xs_home[s];
        const uint32_t dx = (uint32_t)((int)D >> 16);
        const uint32_t q = dx * dx + cy * cy;
        R.qC[s - KS] = (int)q;
        const uint32_t t = q + k2;  // q(dx -+ k) = q + k^2 -+ 2k dx
        if (hasL) R.qL[s] = (int)(t - m1 * dx);
        if (hasR) R.qR[s - 2 * KS] = (int)(t + m1 * dx);
      } else {
        const int e = hasL ? s : s - 2 * KS;
        const uint32_t D = c * sh16 + (uint32_t)xs_out[e];
        const uint32_t dx = (uint32_t)((int)D >> 16);
        const uint32_t q = dx * dx + cy * cy;
        if (hasL) R.qL[e] = (int)q;
        else R.qR[e] = (int)q;
      }
    } else {
      const uint32_t chi = c & 0xFFFF0000u;  // cy << 16
      if (hasC) {
        const uint32_t D1 = c * sh16 + (uint32_t)xs_home[s];  // (cx - X) << 16 | 1
        const uint32_t dx = (uint32_t)((int)D1 >> 16);
        const uint32_t Qk = dx * D1 + cy * chi;                 // (dx^2 + cy^2) << 16 + dx
        R.qC[s - KS] = (int)Qk;
        if (hasL) R.qL[s] = (int)((Qk + k2) - m3 * dx);        // k2 = k^2 2^16 - k
        if (hasR) R.qR[s - 2 * KS] = (int)((Qk + m1) + m3 * dx);  // m1 = k^2 2^16 + k
      } else {
        const int e = hasL ? s : s - 2 * KS;
        const uint32_t D1 = c * sh16 + (uint32_t)xs_out[e];
        const uint32_t dx = (uint32_t)((int)D1 >> 16);
        const uint32_t Qk = dx * D1 + cy * chi;
        if (hasL) R.qL[e] = (int)Qk;
        else R.qR[e] = (int)Qk;
      }
    }
    (void)m2;
  }
}

template <int KS>
__device__ __forceinline__ uint32_t best_sk(const RowS<4 + 2 * KS>& A, const RowS<4 + 2 * KS>& B,
                                            const RowS<4 + 2 * KS>& Cn, int e, int y, int& mo) {
  uint32_t c[9];
  int d[9];
  const uint32_t m2y = (uint32_t)(-2 * y);
  auto put = [&](const RowS<4 + 2 * KS>& R, int j) {
    c[3 * j + 0] = R.c[e];          d[3 * j + 0] = (int)((uint32_t)R.qL[e] + (uint32_t)R.cy[e] * m2y);
    c[3 * j + 1] = R.c[e + KS];     d[3 * j + 1] = (int)((uint32_t)R.qC[e] + (uint32_t)R.cy[e + KS] * m2y);
    c[3 * j + 2] = R.c[e + 2 * KS]; d[3 * j + 2] = (int)((uint32_t)R.qR[e] + (uint32_t)R.cy[e + 2 * KS] * m2y);
  };
  put(A, 0);
  put(B, 1);
  put(Cn, 2);
  const int m = __vimin3_s32(__vimin3_s32(d[0], d[1], d[2]), __vimin3_s32(d[3], d[4], d[5]),
                             __vimin3_s32(d[6], d[7], d[8]));
  mo = m;
  uint32_t w[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) w[i] = __viaddmax_u32((uint32_t)m, 0u - (uint32_t)d[i], c[i]);
  return __vimin3_u32(__vimin3_u32(w[0], w[1], w[2]), __vimin3_u32(w[3], w[4], w[5]), __vimin3_u32(w[6], w[7], w[8]));
}

template <bool SIGNED, int KS>
__device__ __forceinline__ uint32_t min9_sk(const RowS<4 + 2 * KS>& A, const RowS<4 + 2 * KS>& B,
                                            const RowS<4 + 2 * KS>& Cn, int e, uint32_t My) {
  uint32_t kk[9];
  auto put = [&](const RowS<4 + 2 * KS>& R, int j) {
    kk[3 * j + 0] = (uint32_t)R.qL[e] + (uint32_t)R.cy[e] * My;
    kk[3 * j + 1] = (uint32_t)R.qC[e] + (uint32_t)R.cy[e + KS] * My;
    kk[3 * j + 2] = (uint32_t)R.qR[e] + (uint32_t)R.cy[e + 2 * KS] * My;
  };
  put(A, 0);
  put(B, 1);
  put(Cn, 2);
  if constexpr (SIGNED)
    return (uint32_t)__vimin3_s32(__vimin3_s32((int)kk[0], (int)kk[1], (int)kk[2]),
                                  __vimin3_s32((int)kk[3], (int)kk[4], (int)kk[5]),
                                  __vimin3_s32((int)kk[6], (int)kk[7], (int)kk[8]));
  else
    return __vimin3_u32(__vimin3_u32(kk[0], kk[1], kk[2]), __vimin3_u32(kk[3], kk[4], kk[5]),
                        __vimin3_u32(kk[6], kk[7], kk[8]));
}

// One CTA of the shared-term pass (see walk() for the staging and the walk structure).
// KM: 1 or 2 (adjacent, KS = k), 4 .. 4096 (stride with k == KM known at compile time), 8192
// (stride, any larger k).  FULL: the CTA runs a.nwalk whole residue classes (a one-band pass whose classes
// have at most a.walk rows: JFA's large steps); their neighbour rows outside the grid are not
// staged at all (the centre row is reused from registers), and the classes' rows are all staged
// at entry, so one CTA hides the staging latency of several short walks.  Otherwise the CTA
// runs one walk segment of a.walk rows starting at y0, as jump_pass_fast.
//
// REMAP (NEXT-1, the first pass of a dJFA step, one band, stride steps 4 <= k <= 128): the
// input holds the previous frame's labels, except the new seed pixels, which hold the marker EMPTY
// (written by move_fwd; a dJFA diagram is complete, so EMPTY is free at every N, 65536 included).
// Every slot label is remapped as the thread reads it from the stage -- labels[p] <- fwd[labels[p]]
// (Alg. 1's reuse of VD_{t-1}; R-9), a marker becomes the pixel's own position (the
// re-stamp) -- so the remapped diagram is never written to HBM.  The gathers of
// row j + 3 are issued while output row j is computed (one row of look-ahead), and neighbouring
// lanes mostly ask for the same fwd entry, which the L1 serves once per warp instruction.
// X64 (grids beyond N = 32768, whose labels are not all local): the same walk with the exact key
// evaluated in 64 bits per candidate (consider64); the packed walk needs no such fallback, since
// its arithmetic is mod 2^32 (jump_pass_fast's windowed kernel relies on the same property).
template <int KS>
__device__ __forceinline__ uint32_t best64_sk(const RowS<4 + 2 * KS>& A, const RowS<4 + 2 * KS>& B,
                                              const RowS<4 + 2 * KS>& Cn, int e, int xe, int y) {
  uint64_t bd = ~0ull;
  uint32_t bc = EMPTY;
  const RowS<4 + 2 * KS>* rows[3] = {&A, &B, &Cn};
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    consider64<0>(rows[j]->c[e], xe, y, bd, bc);
    consider64<0>(rows[j]->c[e + KS], xe, y, bd, bc);
    consider64<0>(rows[j]->c[e + 2 * KS], xe, y, bd, bc);
  }
  return bc;
}

// Stage every input row of a walk (walk_sk, walk_wsk) into shared memory: one mbarrier per row,
// warp w issues the copies of rows w, w + 4, ... (one elected lane).  FULL: a.nwalk whole residue
// classes (y0 + w), stage slot w * nout + j = row y0 + w + j k; else one walk segment, slot i = row
// y0 + (i - 1) k, rows outside the grid replaced by the centre row.  spans (k >= 256): six
// 128-column spans x0 + j k (j = -1..4) per row, with one tensor copy when a.tmap.
template <bool FULL, bool BANDED>
__device__ __forceinline__ void stage_walk(const PassArgs& a, const CUtensorMap* tm, int x0, int y0, int k, int nout,
                                           int nlist, bool spans, int K4, int SE, uint32_t* smem, uint64_t* bars) {
  const int tid = (int)threadIdx.x, N = a.N;
  for (int i = tid; i < nlist; i += kThreads) mbar_init(&bars[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  {  // staging: warp w issues the copies of rows w, w + 4, ... (one elected lane)
    const int warp = __shfl_sync(0xFFFFFFFFu, tid >> 5, 0);
    const int P = (int)a.pitch;
    const int base = x0 - K4;
    const int lo = max(base, 0), hi = min(x0 + kW + K4, P);
    int nsp = 0;
    if (spans)
      for (int j = -1; j <= 4; ++j) nsp += (x0 + j * k >= 0 && x0 + j * k < N);
    const uint32_t tx = spans ? (!BANDED && a.tmap ? 3072u : 512u * (uint32_t)nsp) : (uint32_t)(hi - lo) * 4u;
    for (int i = warp; i < nlist; i += kThreads / 32) {
      int r;
      if constexpr (FULL) {
        const int w = i / nout;
        r = y0 + w + (i - w * nout) * k;
      } else {
        r = y0 + (i - 1) * k;  // outside the grid: stage the centre row again
        if (r < 0) r += k;
        else if (r >= N) r -= k;
      }
      const uint32_t* src = BANDED ? row_ptr(a, r) : a.in + (int64_t)(r - a.row0) * a.pitch;
      uint32_t* dst = smem + (size_t)i * SE;
      if (elect_one()) {
        mbar_expect_tx(&bars[i], tx);
        if (!spans) {
          bulk_g2s(dst + (lo - base), src + lo, (uint32_t)(hi - lo) * 4u, &bars[i]);
        } else if (!BANDED && a.tmap) {
          // the row as a [N/k][k] array: box {128 columns, 6 blocks} at (x0 mod k, j = g*4 - 1);
          // blocks outside the grid arrive zero-filled (replaced by the FIX substitution)
          const int c0 = x0 & (k - 1), c1 = (x0 >> a.lk) - 1;
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
              "[%5];" ::"r"(smem_u32(dst)),
              "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(r - a.row0), "r"(smem_u32(&bars[i]))
              : "memory");
        } else {
#pragma unroll 1
          for (int j = -1; j <= 4; ++j) {
            const int cs = x0 + j * k;
            if (cs >= 0 && cs < N) bulk_g2s(dst + (j + 1) * 128, src + cs, 512u, &bars[i]);
          }
        }
      }
      __syncwarp();
    }
  }
}

// HASH (the last pass of an e2e dJFA step, KM = 1): every output label is also added to the
// frame's checksum, sum over p of fmix32((y N + x) * 0x9E3779B9 ^ label) mod 2^64 (label_hash),
// so the step needs no separate 4-B/px read for its result.
__device__ __forceinline__ uint32_t fwd_index(uint32_t c, int fp) {
  return fp ? c + (c >> 16) * (uint32_t)(fp - 65536) : c;  // y 2^16 + x + y (fp - 2^16) = y fp + x
}
#ifndef VD_FWD_HINT
#define VD_FWD_HINT 0  // 1: the fused pass's fwd gathers carry an L2 evict_last policy (A/B)
#endif
__device__ __forceinline__ uint32_t ld_fwd(const uint32_t* p, uint64_t pol) {
#if VD_FWD_HINT
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
#else
  (void)pol;
  return __ldg(p);
#endif
}
#ifndef VD_FUSE_LA
#define VD_FUSE_LA 1  // rows of fwd-gather look-ahead in the fused remap pass (1 or 2)
#endif
constexpr int kFuseLA = VD_FUSE_LA;
// LAT (with PACK, stride steps): the JFA lattice walk.  After passes N/2 .. 2k of a JFA every label
// is congruent to its pixel mod 2k (the first pass takes seeds at p + o k1; a pass k takes a label of
// p + o k), so every candidate of pass k lies at (dx, dy) = k (a, b) with integers a, b, and
// (d2, c) orders as (a^2 + b^2, b, a).  In lattice coordinates (>> log2 k) that is the packed key
// with (a, b) for (dx, dy): exact when N <= 64 k (|a|, |b| <= 63).  EMPTY and the virtual far seed go
// to the lattice point (127, 127): at least 64 units from every pixel, so they lose to every real
// label, and an output decoded as (127, 127) had only such candidates.  The output is the lattice
// label scaled back, (o << log2 k) | (y mod k, X mod k).
constexpr uint32_t kLatEmpty = (127u << 16) | 127u;
template <int KM, bool MAY_EMPTY, bool BANDED, bool FIX, bool PACK, bool FULL, bool REMAP = false, bool PRE = false,
          bool X64 = false, bool HASH = false, int LAT = 0>
__device__ __forceinline__ void walk_sk(const PassArgs& a, const CUtensorMap* tm, int x0, int X, int y0,
                                        uint32_t* smem) {
  constexpr int KS = KM < kVec ? KM : 1;
  constexpr int NS = 4 + 2 * KS;
  constexpr bool STRIDE = KM >= kVec;
  constexpr int KC = (STRIDE && KM <= 4096) ? KM : 0;  // compile-time step: immediate offsets
  const int k = KC ? KC : a.k, N = a.N;
  const int tid = (int)threadIdx.x;
  // FULL: walks y0 + w (w < nw), each of nout rows; stage slot of (walk w, row j) = w * nout + j.
  // Else: one walk; stage slot i = logical row i (0 = the row above the first output row).
  const int nw = FULL ? min(a.nwalk, k - (y0 - a.y_lo)) : 1;
  const int nout = FULL ? (a.y_hi - y0 + k - 1) >> a.lk : min(a.walk, (a.y_hi - y0 + k - 1) >> a.lk);
  const int nlist = FULL ? nw * nout : nout + 2;
  const bool spans = STRIDE && k >= 256;
  const int K4 = (k + 3) & ~3;
  const int SE = stage_elems_sk(k);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)(a.walk + 2) * SE);

  if constexpr (!PRE) stage_walk<FULL, BANDED>(a, tm, x0, y0, k, nout, nlist, spans, K4, SE, smem, bars);

  // per-thread slot offsets in a stage, columns, and edge flags.  The key arithmetic runs on
  // (Xa, ka): the columns and step themselves, or (LAT) their lattice units X >> log2 k and 1
  static_assert(LAT == 0 || (STRIDE && PACK == (LAT < 3)), "lattice walks: packed (1, 2) or exact (3, 4), stride steps");
  const int ka = LAT ? 1 : k;
  const int Xa = LAT ? (X >> a.lk) : X;
  const uint32_t sh16 = a.sh16;
  int xs_home[NS], xs_out[kVec];
  constexpr uint32_t P1 = PACK ? 1u : 0u;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int col = STRIDE ? Xa + (s - 1) * ka : X + s - KS;
    xs_home[s] = (int)(P1 - ((uint32_t)col << 16));
  }
#pragma unroll
  for (int e = 0; e < kVec; ++e) xs_out[e] = (int)(P1 - ((uint32_t)(STRIDE ? Xa + e * ka : X + e) << 16));
  const bool left_out = FIX && (STRIDE ? X - k < 0 : X - KS < 0);
  const bool right_out = FIX && (STRIDE ? X + 4 * k >= N : X + 3 + KS >= N);
  // stride: slot s (column X + (s-1) k) lies in the grid iff s - 1 < nc, output e iff e < nc.  With
  // spans (k >= 256) on a grid that is not a multiple of 4k the last group of 4k columns is partial:
  // there nc < 4 (outputs beyond the grid are not stored, slots beyond it duplicate their left slot)
  const int nc = (STRIDE && FIX) ? (X >= N ? 0 : ((N - 1 - X) >> a.lk) + 1) : 8;
  int xb[kVec];
#pragma unroll
  for (int e = 0; e < kVec; ++e) xb[e] = (STRIDE ? Xa + e * ka : X + e) - 128;
  // constants (uniform): exact (k^2, 2k); packed (k^2 2^16 - k, k^2 2^16 + k, 2k 2^16)
  const uint32_t uk = (uint32_t)ka;
  bool any_e = false;  // LAT: some output stayed unclaimed
  const uint32_t k2 = PACK ? uk * uk * 65536u - uk : uk * uk;
  const uint32_t m1 = PACK ? uk * uk * 65536u + uk : 2u * uk;
  const uint32_t m3 = 2u * uk * 65536u;
  const int sbase = STRIDE ? (spans ? tid : (X - x0) + K4 - k) : 4 * tid;  // stage index of slot 0's vector / label

  uint32_t loc_acc = 0;
  bool loc_bad = false;
  uint64_t hacc = 0;  // HASH
  using R_t = RowS<NS>;
  // REMAP: slot labels of a staged row, remapped through fwd (loads in flight until build)
  uint64_t fwd_pol = 0;
#if VD_FWD_HINT
  if constexpr (REMAP) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(fwd_pol));
#endif
  auto fetch = [&](int i, uint32_t (&lab)[NS]) {
    if constexpr (!PRE) mbar_wait(&bars[i], 0u);
    const uint32_t* st = smem + (size_t)i * SE;
#pragma unroll
    for (int s = 0; s < NS; ++s) lab[s] = st[sbase + s * (spans ? 128 : k)];
    if constexpr (FIX) {
#pragma unroll
      for (int s = 0; s < KS; ++s) lab[s] = left_out ? lab[s + KS] : lab[s];
#pragma unroll
      for (int s = 4 + KS; s < NS; ++s) lab[s] = right_out ? lab[s - KS] : lab[s];
    }
    // a new seed pixel holds the marker EMPTY (move_fwd; a dJFA diagram has no EMPTY): its label is
    // its own position -- the row of stage slot i (rows outside the grid were staged as the centre
    // row) and the slot's column (an out-of-grid slot holds its in-grid duplicate's label)
    int r = y0 + (i - 1) * k;
    if (r < 0) r += k;
    else if (r >= N) r -= k;
    const uint32_t own0 = ((uint32_t)r << 16) + (uint32_t)(X - k);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const uint32_t c = lab[s];
      uint32_t own = own0 + (uint32_t)(s * k);
      if (FIX && s == 0 && left_out) own += (uint32_t)k;
      if (FIX && s == NS - 1 && right_out) own -= (uint32_t)k;
      lab[s] = c == EMPTY ? own : ld_fwd(a.fwd + c, fwd_pol);  // (the fused frame's fwd: indexed by the label itself)
    }
  };
  auto consume = [&](int i, R_t& R) {
    if constexpr (!PRE) mbar_wait(&bars[i], 0u);
    const uint32_t* st = smem + (size_t)i * SE;
    uint32_t lab[NS];
    if constexpr (!STRIDE) {
      uint32_t w[12];
      unpack(*reinterpret_cast<const uint4*>(st + sbase), w);
      unpack(*reinterpret_cast<const uint4*>(st + sbase + 4), w + 4);
      unpack(*reinterpret_cast<const uint4*>(st + sbase + 8), w + 8);
#pragma unroll
      for (int s = 0; s < NS; ++s) lab[s] = w[s - KS + 4];
    } else {
#pragma unroll
      for (int s = 0; s < NS; ++s) lab[s] = st[sbase + s * (spans ? 128 : k)];
    }
    if constexpr (FIX) {  // out-of-grid neighbour -> the same output's centre label (a duplicate)
#pragma unroll
      for (int s = 0; s < KS; ++s) lab[s] = left_out ? lab[s + KS] : lab[s];
      if constexpr (STRIDE) {
        if (nc < 4) {  // the partial last group of 4k columns (spans on a grid that 4k does not divide)
#pragma unroll
          for (int s = 1; s < NS - 1; ++s) lab[s] = s >= nc + 1 ? lab[s - 1] : lab[s];
        }
        lab[NS - 1] = right_out ? lab[NS - 2] : lab[NS - 1];
      } else {
#pragma unroll
        for (int s = 4 + KS; s < NS; ++s) lab[s] = right_out ? lab[s - KS] : lab[s];
      }
    }
    if constexpr (LAT > 0) {  // labels to lattice coordinates (both 16-bit halves >> log2 k)
      const uint32_t msk = (0xFFFFu >> a.lk) * 0x10001u;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const uint32_t c = lab[s];
        // LAT 1: EMPTY / the virtual far seed (labels at or beyond row N: c >= a.lat_min) -> (127, 127)
        const bool E = LAT == 1 && c >= a.lat_min;
#ifdef VD_CHECK  // the lattice invariant (debug builds): label = pixel (mod k) in both coordinates
        if (!(c == EMPTY || c == a.lat_empty) &&
            ((((c & 0xFFFFu) - (uint32_t)X) | ((c >> 16) - (uint32_t)y0)) & (uint32_t)(k - 1)) != 0u)
          __trap();
        if ((LAT == 2 || LAT == 4) && (c == EMPTY || c == a.lat_empty)) __trap();
#endif
        const bool E3 = LAT == 3 && c >= a.lat_min;
        lab[s] = E ? kLatEmpty : E3 ? a.lat_vl : ((c >> a.lk) & msk);
      }
    }
    build_sk<KS, MAY_EMPTY, PACK>(lab, xs_home, xs_out, a.vempty, sh16, k2, m1, 0u, m3, R);
  };

  const int64_t kp = (int64_t)k * a.pitch;
  // One walk: output rows yw, yw + k, ... (n rows).  Logical input row i (0 = the row above the
  // first output, n + 1 = the row below the last) is stage slot ibase + i; FULL walks have no
  // rows 0 and n + 1 in the stage (outside the grid: the centre row is a duplicate candidate).
  auto run = [&](int yw, int n, int ibase) {
    R_t r0, r1, r2;
    uint32_t pend[NS];   // REMAP: the next row's remapped slot labels
    uint32_t pend2[NS];  // ... and, with two rows of look-ahead (VD_FUSE_LA = 2), the row after
    if constexpr (REMAP) {
      uint32_t l0[NS];
      fetch(ibase, l0);
      fetch(ibase + 1, pend);
      build_sk<KS, MAY_EMPTY, PACK>(l0, xs_home, xs_out, a.vempty, sh16, k2, m1, 0u, m3, r0);
      build_sk<KS, MAY_EMPTY, PACK>(pend, xs_home, xs_out, a.vempty, sh16, k2, m1, 0u, m3, r1);
      fetch(ibase + 2, pend);
      if (kFuseLA == 2 && 3 < n + 2) fetch(ibase + 3, pend2);
    } else if constexpr (FULL) {
      consume(ibase + 1, r1);  // (the row above the first output is outside the grid: r1 serves as both)
    } else {
      consume(ibase, r0);
      consume(ibase + 1, r1);
    }
    int y = yw;
    uint32_t* po = a.out + (int64_t)(yw - a.row0) * a.pitch + X;
    int j = 0;
    auto eval = [&](const R_t& Pv, const R_t& Cv, const R_t& Nx) {
      uint32_t o[kVec];
      if constexpr (X64) {
#pragma unroll
        for (int e = 0; e < kVec; ++e) o[e] = best64_sk<KS>(Pv, Cv, Nx, e, STRIDE ? X + e * k : X + e, y);
        loc_bad = true;  // not tracked on this path
      } else if constexpr (PACK) {
        const uint32_t uy = LAT > 0 ? (uint32_t)(y >> a.lk) : (uint32_t)y;
        const uint32_t My = 256u - (uy << 17);
        const uint32_t Cy = uy * uy * 65536u - 256u * uy + 32896u;
        const uint32_t Yb = (uy - 128u) << 16;
        uint32_t sk[kVec];
        if (0u - Cy <= 0x80000000u) {
#pragma unroll
          for (int e = 0; e < kVec; ++e) sk[e] = min9_sk<false, KS>(Pv, Cv, Nx, e, My) + Cy;
        } else {
#pragma unroll
          for (int e = 0; e < kVec; ++e) sk[e] = min9_sk<true, KS>(Pv, Cv, Nx, e, My) + Cy;
        }
#pragma unroll
        for (int e = 0; e < kVec; ++e) o[e] = __byte_perm(sk[e], 0u, 0x4140) + Yb + (uint32_t)xb[e];
        if constexpr (LAT > 0) {  // lattice label -> label: (o << log2 k) | (y mod k, X mod k)
          const uint32_t low = ((uint32_t)(y & (k - 1)) << 16) | (uint32_t)(X & (k - 1));
#pragma unroll
          for (int e = 0; e < kVec; ++e) {
            if constexpr (LAT == 1) {
              const bool E = o[e] == kLatEmpty;
              any_e |= E;
              o[e] = E ? a.lat_empty : ((o[e] << a.lk) | low);
            } else {
              o[e] = (o[e] << a.lk) | low;
            }
          }
        } else {
          loc_acc = __vimax3_u32(__vimax3_u32(loc_acc, sk[0], sk[1]), sk[2], sk[3]);
        }
      } else if constexpr (LAT >= 3) {  // exact walk in lattice units (any N <= 65536 with k >= 4)
        const int ye = y >> a.lk;
        const uint32_t low = ((uint32_t)(y & (k - 1)) << 16) | (uint32_t)(X & (k - 1));
#pragma unroll
        for (int e = 0; e < kVec; ++e) {
          int me;
          const uint32_t v = best_sk<KS>(Pv, Cv, Nx, e, ye, me);
          if constexpr (LAT == 3) {
            const bool E = v == a.lat_vl;
            any_e |= E;
            o[e] = E ? a.lat_empty : ((v << a.lk) | low);
          } else {  // 4: no unclaimed label can be present
            o[e] = (v << a.lk) | low;
          }
        }
      } else {
        int mm = -0x7FFFFFFF - 1;
#pragma unroll
        for (int e = 0; e < kVec; ++e) {
          int me;
          uint32_t v = best_sk<KS>(Pv, Cv, Nx, e, y, me);
          mm = max(mm, me);
          if (MAY_EMPTY) v = (v == a.vempty) ? EMPTY : v;
          o[e] = v;
        }
        loc_bad |= mm > (int)kLocD2 - y * y;
      }
      if constexpr (HASH) {
        const uint32_t b = ((uint32_t)y * (uint32_t)N + (uint32_t)X) * 0x9E3779B9u;
#pragma unroll
        for (int e = 0; e < kVec; ++e) hacc += fmix32((b + (uint32_t)e * 0x9E3779B9u) ^ o[e]);
      }
      if constexpr (!STRIDE) {
        store_out(a, BANDED, y, X, po, make_uint4(o[0], o[1], o[2], o[3]));
      } else {
#pragma unroll
        for (int e = 0; e < kVec; ++e)
          if (e < nc) store_out(a, BANDED, y, X + e * k, po + e * k, o[e]);
      }
      po += kp;
      y += k;
    };
    auto step = [&](const R_t& Pv, const R_t& Cv, R_t& Nx) -> bool {
      if constexpr (REMAP) {
        build_sk<KS, MAY_EMPTY, PACK>(pend, xs_home, xs_out, a.vempty, sh16, k2, m1, 0u, m3, Nx);
        if constexpr (kFuseLA == 2) {
#pragma unroll
          for (int s = 0; s < NS; ++s) pend[s] = pend2[s];
          if (j + 4 < n + 2) fetch(ibase + j + 4, pend2);  // gathers in flight during two rows
        } else {
          if (j + 3 < n + 2) fetch(ibase + j + 3, pend);  // gathers in flight during this row
        }
        if (a.prefetch && j + 3 + kFuseLA < n + 2) {  // and the row after that: its fwd lines into L1
          mbar_wait(&bars[ibase + j + 3 + kFuseLA], 0u);
          const uint32_t* st = smem + (size_t)(ibase + j + 3 + kFuseLA) * SE;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const uint32_t c = st[sbase + s * (spans ? 128 : k)];
            if (c != EMPTY)
              asm volatile("prefetch.global.L1 [%0];" ::"l"(a.fwd + c));
          }
        }
        eval(Pv, Cv, Nx);
      } else if (!FULL || j + 1 < n) {
        consume(ibase + j + 2, Nx);
        eval(Pv, Cv, Nx);
      } else {
        eval(Pv, Cv, Cv);  // FULL: the row below the last output is outside the grid
      }
      return ++j < n;
    };
    if (FULL) {
      if (step(r1, r1, r2)) {
#pragma unroll 1
        while (true) {
          if (!step(r1, r2, r0)) break;
          if (!step(r2, r0, r1)) break;
          if (!step(r0, r1, r2)) break;
        }
      }
    } else {
#pragma unroll 1
      while (true) {
        if (!step(r0, r1, r2)) break;
        if (!step(r1, r2, r0)) break;
        if (!step(r2, r0, r1)) break;
      }
    }
  };
  if constexpr (FULL) {
#pragma unroll 1
    for (int w = 0; w < nw; ++w) run(y0 + w, nout, w * nout - 1);
  } else {
    run(y0, nout, 0);
  }
  if (a.loc_out) {
    bool far;
    if constexpr (LAT > 0) far = true;  // (locality is not tracked in lattice units)
    else if constexpr (PACK) far = loc_acc >= ((kLocD2 + 1u) << 16);
    else far = loc_bad;
    if (__syncthreads_or(far) && tid == 0) atomicOr(a.loc_out, 1u);
  }
  if constexpr (LAT == 1 || LAT == 3) {
    if (a.empty_flag != nullptr && __syncthreads_or(any_e) && tid == 0) atomicOr(a.empty_flag, 1ull);
  }
  if constexpr (HASH) {
    const uint64_t t = block_sum_u64(hacc);
    if (tid == 0) atomicAdd(a.hash_out, (unsigned long long)t);
  }
}

__host__ __device__ constexpr int ilog2_c(int v) { return v <= 1 ? 0 : 1 + ilog2_c(v / 2); }

// grid (xblocks, segs, residues) as jump_pass_fast; with a.nwalk > 0 (FULL) the z index counts
// groups of a.nwalk residue classes.  Host: N % 512 == 0, k a power of two, k <= N / 4;
// Euclidean Moore passes, no window (N <= 32768).  KM: k itself for k <= 4096 (compile-time
// step), 8192 for any larger k.
__device__ __forceinline__ void folded_fwd_reset(const PassArgs& a) {
  if (a.rst_fwd == nullptr) return;
  const int64_t nb = (int64_t)gridDim.x * gridDim.y * gridDim.z;
  const int64_t b = blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z);
  for (int64_t i = b * blockDim.x + threadIdx.x; i < a.rst_s; i += nb * blockDim.x) a.rst_fwd[a.rst_seeds[i]] = EMPTY;
}

template <int KM, bool MAY_EMPTY, bool BANDED, bool HASH = false, int MINB = VD_MIN_BLOCKS>
__global__ void __launch_bounds__(kThreads, MINB) jump_pass_sk(PassArgs a, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(128) uint32_t dyn_smem[];
  folded_fwd_reset(a);
  const int xb = (int)blockIdx.x;
  const bool full = a.nwalk > 0;
  const int seg = full ? 0 : (int)(a.res_in_y ? blockIdx.z : blockIdx.y);
  const int res = full ? (int)blockIdx.z * a.nwalk : (int)(a.res_in_y ? blockIdx.y : blockIdx.z);
  const int y0 = a.y_lo + res + seg * a.walk * a.k;
  if (res >= a.k || y0 >= a.y_hi) return;
  const int k = a.k, tid = (int)threadIdx.x;
  int x0, X;
  bool fix;
  if constexpr (KM < kVec) {
    x0 = xb * kW;
    X = x0 + kVec * tid;
    fix = x0 == 0 || x0 + kW >= a.N;
  } else if constexpr (KM <= 128) {  // k == KM
    x0 = xb * kW;
    X = x0 + 4 * KM * (tid / KM) + (tid % KM);
    fix = x0 == 0 || x0 + kW >= a.N;
  } else {
    const int lr = (KM <= 4096 ? ilog2_c(KM) : a.lk) - 7;  // k / 128 residue blocks per group of 4k columns
    const int g = xb >> lr, rb = xb & ((1 << lr) - 1);
    x0 = 4 * k * g + 128 * rb;
    X = x0 + tid;
    fix = g == 0 || x0 + 4 * k + 128 > a.N;  // some right neighbour column (X + 4k) beyond the grid
    if (x0 >= a.N) return;  // (the partial last group of a grid that is not a multiple of 4k)
  }
  if constexpr (KM >= kVec && !MAY_EMPTY && MINB == VD_MIN_BLOCKS && !HASH) {
    // JFA's lattice walk: 1 = unclaimed labels possible (N <= 64k), 2 = none left (N <= 128k)
    if (a.lat == 1) {
      if (full) {
        if (fix) walk_sk<KM, false, BANDED, true, true, true, false, false, false, false, 1>(a, &tm, x0, X, y0, dyn_smem);
        else walk_sk<KM, false, BANDED, false, true, true, false, false, false, false, 1>(a, &tm, x0, X, y0, dyn_smem);
      } else {
        if (fix) walk_sk<KM, false, BANDED, true, true, false, false, false, false, false, 1>(a, &tm, x0, X, y0, dyn_smem);
        else walk_sk<KM, false, BANDED, false, true, false, false, false, false, false, 1>(a, &tm, x0, X, y0, dyn_smem);
      }
      return;
    }
    if (a.lat == 3) {
      if (full) {
        if (fix) walk_sk<KM, false, BANDED, true, false, true, false, false, false, false, 3>(a, &tm, x0, X, y0, dyn_smem);
        else walk_sk<KM, false, BANDED, false, false, true, false, false, false, false, 3>(a, &tm, x0, X, y0, dyn_smem);
      } else {
        if (fix) walk_sk<KM, false, BANDED, true, false, false, false, false, false, false, 3>(a, &tm, x0, X, y0, dyn_smem);
        else walk_sk<KM, false, BANDED, false, false, false, false, false, false, false, 3>(a, &tm, x0, X, y0, dyn_smem);
      }
      return;
    }
    if (a.lat == 4) {
      if (full) {
        if (fix) walk_sk<KM, false, BANDED, true, false, true, false, false, false, false, 4>(a, &tm, x0, X, y0, dyn_smem);
        else walk_sk<KM, false, BANDED, false, false, true, false, false, false, false, 4>(a, &tm, x0, X, y0, dyn_smem);
      } else {
        if (fix) walk_sk<KM, false, BANDED, true, false, false, false, false, false, false, 4>(a, &tm, x0, X, y0, dyn_smem);
        else walk_sk<KM, false, BANDED, false, false, false, false, false, false, false, 4>(a, &tm, x0, X, y0, dyn_smem);
      }
      return;
    }
    if (a.lat == 2) {
      if (full) {
        if (fix) walk_sk<KM, false, BANDED, true, true, true, false, false, false, false, 2>(a, &tm, x0, X, y0, dyn_smem);
        else walk_sk<KM, false, BANDED, false, true, true, false, false, false, false, 2>(a, &tm, x0, X, y0, dyn_smem);
      } else {
        if (fix) walk_sk<KM, false, BANDED, true, true, false, false, false, false, false, 2>(a, &tm, x0, X, y0, dyn_smem);
        else walk_sk<KM, false, BANDED, false, true, false, false, false, false, false, 2>(a, &tm, x0, X, y0, dyn_smem);
      }
      return;
    }
  }
  if (full) {  // JFA's large steps: exact walk (their diagrams are never local)
    if (fix) walk_sk<KM, MAY_EMPTY, BANDED, true, false, true, false, false, false, HASH>(a, &tm, x0, X, y0, dyn_smem);
    else walk_sk<KM, MAY_EMPTY, BANDED, false, false, true, false, false, false, HASH>(a, &tm, x0, X, y0, dyn_smem);
    return;
  }
  if constexpr (!MAY_EMPTY) {
    if (a.loc_in && k <= kPackMaxK && *(volatile const uint32_t*)a.loc_in == 0u) {
      if (fix) walk_sk<KM, MAY_EMPTY, BANDED, true, true, false, false, false, false, HASH>(a, &tm, x0, X, y0, dyn_smem);
      else walk_sk<KM, MAY_EMPTY, BANDED, false, true, false, false, false, false, HASH>(a, &tm, x0, X, y0, dyn_smem);
      return;
    }
    if constexpr (KM <= 64) {
      if (a.N > 32768) {  // 32-bit squared distances would overflow: exact 64-bit keys
        if (fix) walk_sk<KM, false, BANDED, true, false, false, false, false, true, HASH>(a, &tm, x0, X, y0, dyn_smem);
        else walk_sk<KM, false, BANDED, false, false, false, false, false, true, HASH>(a, &tm, x0, X, y0, dyn_smem);
        return;
      }
    }
  }
  if (fix) walk_sk<KM, MAY_EMPTY, BANDED, true, false, false, false, false, false, HASH>(a, &tm, x0, X, y0, dyn_smem);
  else walk_sk<KM, MAY_EMPTY, BANDED, false, false, false, false, false, false, HASH>(a, &tm, x0, X, y0, dyn_smem);
}

// The first pass of a dJFA step with the remap fused in (walk_sk REMAP): one band, stride steps
// 4 <= k <= 128.
template <int KM>
__global__ void __launch_bounds__(kThreads, 5) jump_pass_sk_remap(PassArgs a, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(128) uint32_t dyn_smem[];
  // grid order 2 = (residue, x-block, segment): the CTAs resident at once cover every residue class
  // of a few 512-column blocks of one row band, so each fwd entry is gathered by all of them while
  // it is in L2 (the other orders: see PassArgs::res_in_y)
  const int xb = (int)(a.res_in_y == 2 ? blockIdx.y : blockIdx.x);
  const int seg = (int)(a.res_in_y ? blockIdx.z : blockIdx.y);
  const int res = (int)(a.res_in_y == 2 ? blockIdx.x : a.res_in_y ? blockIdx.y : blockIdx.z);
  const int y0 = a.y_lo + res + seg * a.walk * a.k;
  if (res >= a.k || y0 >= a.y_hi) return;
  const int tid = (int)threadIdx.x;
  const int x0 = xb * kW;
  const int X = x0 + 4 * KM * (tid / KM) + (tid % KM);
  const bool fix = x0 == 0 || x0 + kW >= a.N;
  // packed walk when the previous frame's diagram was local and the moves keep every
  // candidate within the packed key's range (the host passes loc_in only then)
  if (a.loc_in && *(volatile const uint32_t*)a.loc_in == 0u) {
    if (fix) walk_sk<KM, false, false, true, true, false, true>(a, &tm, x0, X, y0, dyn_smem);
    else walk_sk<KM, false, false, false, true, false, true>(a, &tm, x0, X, y0, dyn_smem);
    return;
  }
  if (a.N > 32768) {  // 32-bit squared distances would overflow: exact 64-bit keys (X64)
    if (fix) walk_sk<KM, false, false, true, false, false, true, false, true>(a, &tm, x0, X, y0, dyn_smem);
    else walk_sk<KM, false, false, false, false, false, true, false, true>(a, &tm, x0, X, y0, dyn_smem);
    return;
  }
  if (fix) walk_sk<KM, false, false, true, false, false, true>(a, &tm, x0, X, y0, dyn_smem);
  else walk_sk<KM, false, false, false, false, false, true>(a, &tm, x0, X, y0, dyn_smem);
}

// ------------------------------------------------------------------ wide exact pass (r02: N <= 65536)
//
// The exact pass (key (d2, c) lexicographically, R-3) for grids beyond N = 32768, whose
// squared distances need 33 bits, with EMPTY allowed: JFA's large steps at C5, where labels are far
// from their pixels (jump_pass_wide did these with per-candidate 64-bit compares, ~200 instructions
// per pixel).  Stride layout with spans (k >= 256, power of two, 4k <= N, N % 512 == 0) and the
// staging of walk_sk; one thread = output columns Xo_e = X + e k (e = 0..3) of each output row.
//
// Per output row y let h = y >> 1 and p = y & 1 (p is the same for every row of a walk, k even).
// For a label c = (cy, cx) and output column Xo, with c~ = cy - p and n = Xo - cx:
//   d2 = n^2 + (cy - y)^2 = n^2 + c~^2 - 4 h c~ + 4 h^2,  so  D = d2 - 4 h^2 = Q - 4 h c~, Q = n^2 + c~^2.
// 4 h^2 is common to the nine candidates of the pixel.  Squares are 0 or 1 mod 4, so with
//   Qh = (n^2 >> 2) + (c~^2 >> 2)  (< 2^31)  and  Ql = (n & 1) + (c~ & 1)  (in {0, 1, 2}):
//   D >> 2 = Qh - h c~  (ONE integer multiply-add per candidate, in [-2^30, 2^31)),  D & 3 = Ql.
// The key (d2, c) is then, for one pixel, the same order as (hi, lo) with hi = Qh - h c~ and
//   lo = Ql 2^18 + cy 2 + [n < 0]
// (equal d2 and equal cy leave |dx| equal: the two labels are mirror images about the pixel's
// column, and the one with dx < 0, the smaller cx, wins).  The nine-way minimum is the walk_sk
// "resolve later" pair: m = min hi (signed), then min over max(m - hi, lo) (unsigned): for hi > m
// the difference wraps to >= 2^31 (hi - m <= 2 65535^2 / 4 + 1 < 2^31), above every lo (< 2^20).
// The label is decoded from the winner: cy and the sign from lo, |dx| = sqrt(d2 - dy^2) with
// d2 = 4 m + Ql + 4 h^2 (exact in uint32 arithmetic: dx^2 < 2^32; the float square root of a perfect
// square below 2^32 rounds to the exact root).
// Per staged label (once per row, shared by its up to three column uses, k a multiple of 4):
//   Qh(n +- k) = Qh(n) + k^2/4 +- (k/2) n,  lo(n +- k) = lo(n) - [n < 0] + [n +- k < 0].
// EMPTY (MAY_EMPTY): hi = INT_MAX (c~ = 0, Qh = INT_MAX), above every real hi (<= 2147418112); an
// output whose minimum is INT_MAX stays EMPTY.
struct RowW {
  int32_t cyt[6];                 // c~ = cy - p of slot s (0 for EMPTY)
  uint32_t qL[4], qC[4], qR[4];   // Qh of output e's left / centre / right candidate (slots e, e+1, e+2)
  uint32_t lL[4], lC[4], lR[4];   // lo of the same
};

__device__ __forceinline__ uint32_t isqrt_square(uint32_t v) {  // v = a^2 < 2^32 -> a
  const float f = __uint2float_rn(v);
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f));
  return __float2uint_rn(r);
}

// Terms of one staged row.  lab[s]: label of slot s (column X + (s-1) k); Xo: the thread's output
// columns.  Slots 1..4 sit on output columns (their n is exact); slots 0 and 5 serve one output each
// (output 0's left, output 3's right) and are computed against that output's column directly.
#ifndef VD_WSK_SGN
#define VD_WSK_SGN 1  // sign bits of lo: 1 = high word of 2n on the FMA pipe (IMAD.HI), 0 = shift + or (ALU)
#endif
__device__ __forceinline__ uint32_t add_sign(uint32_t lob, int n) {  // lob + [n < 0]
#if VD_WSK_SGN
  return mad_hi_u32((uint32_t)n, 2u, lob);
#else
  return lob + ((uint32_t)n >> 31);
#endif
}
// (one = 1 and sh16 = 2^16 are run-time values, so that the additions below stay IMADs on the FMA
// pipe: the pass is ALU-bound)
template <bool MAY_EMPTY>
__device__ __forceinline__ void build_w(const uint32_t (&lab)[6], const int (&Xo)[4], uint32_t p, uint32_t k,
                                        uint32_t k2q, uint32_t kh, uint32_t one, uint32_t sh16, RowW& R) {
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const uint32_t c = lab[s];
    const uint32_t cy = c >> 16;
    const int cyt = (int)(cy * one - p);
    const uint32_t cy2 = (uint32_t)(cyt * cyt);
    const int col = s == 0 ? Xo[0] : s == 5 ? Xo[3] : Xo[s - 1];
    const int n = (int)(cy * sh16 + ((uint32_t)col - c));  // col - cx, with cx = c - cy 2^16
    const uint32_t n2 = (uint32_t)(n * n);
    const uint32_t qh = (n2 >> 2) + (cy2 >> 2);
    // Ql = (n^2 + c~^2) mod 4 (the square sum mod 2^32 keeps its low bits); lo base (Ql, cy, 0)
    const uint32_t lob = (((n2 + cy2) << 18) & (3u << 18)) + 2u * cy;
    const bool E = MAY_EMPTY && c == EMPTY;
    constexpr uint32_t BIG = 0x7FFFFFFFu;
    if (s == 0) {
      R.qL[0] = E ? BIG : qh;
      R.lL[0] = add_sign(lob, n);
    } else if (s == 5) {
      R.qR[3] = E ? BIG : qh;
      R.lR[3] = add_sign(lob, n);
    } else {
      R.qC[s - 1] = E ? BIG : qh;
      R.lC[s - 1] = add_sign(lob, n);
      const uint32_t t = qh + k2q;
      if (s <= 3) {  // left candidate of output s: column Xo + k
        R.qL[s] = E ? BIG : t + kh * (uint32_t)n;
        R.lL[s] = add_sign(lob, (int)((uint32_t)n * one + k));
      }
      if (s >= 2) {  // right candidate of output s - 2: column Xo - k
        R.qR[s - 2] = E ? BIG : t - kh * (uint32_t)n;
        R.lR[s - 2] = add_sign(lob, (int)((uint32_t)n * one - k));
      }
    }
    R.cyt[s] = E ? 0 : cyt;
  }
}

// Output label of column Xo[e] in row y (h = y >> 1, hh = 4 h^2) from the rows above (A), at (B),
// below (Cn).  Returns EMPTY when every candidate is EMPTY.
template <bool MAY_EMPTY>
__device__ __forceinline__ uint32_t best_w(const RowW& A, const RowW& B, const RowW& Cn, int e, int Xo, int y,
                                           uint32_t mh, uint32_t hh) {
  int hi[9];
  uint32_t lo[9];
  auto put = [&](const RowW& R, int j) {
    hi[3 * j + 0] = (int)(R.qL[e] + (uint32_t)R.cyt[e] * mh);
    hi[3 * j + 1] = (int)(R.qC[e] + (uint32_t)R.cyt[e + 1] * mh);
    hi[3 * j + 2] = (int)(R.qR[e] + (uint32_t)R.cyt[e + 2] * mh);
    lo[3 * j + 0] = R.lL[e];
    lo[3 * j + 1] = R.lC[e];
    lo[3 * j + 2] = R.lR[e];
  };
  put(A, 0);
  put(B, 1);
  put(Cn, 2);
  const int m = __vimin3_s32(__vimin3_s32(hi[0], hi[1], hi[2]), __vimin3_s32(hi[3], hi[4], hi[5]),
                             __vimin3_s32(hi[6], hi[7], hi[8]));
  uint32_t w[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) w[i] = __viaddmax_u32((uint32_t)m, 0u - (uint32_t)hi[i], lo[i]);
  const uint32_t ww = __vimin3_u32(__vimin3_u32(w[0], w[1], w[2]), __vimin3_u32(w[3], w[4], w[5]),
                                   __vimin3_u32(w[6], w[7], w[8]));
  const uint32_t cy = (ww >> 1) & 0xFFFFu;
  const int dy = (int)cy - y;
  const uint32_t dx2 = (uint32_t)m * 4u + (ww >> 18) + hh - (uint32_t)(dy * dy);
  const uint32_t ad = isqrt_square(dx2);
  const uint32_t cx = (ww & 1u) ? (uint32_t)Xo + ad : (uint32_t)Xo - ad;
  const uint32_t lab = (cy << 16) | cx;
  if (MAY_EMPTY && m == 0x7FFFFFFF) return EMPTY;
#ifdef VD_CHECK  // debug builds (compute-sanitizer is not available on the pool): the decoded label
                 // must lie in the grid and reproduce the winning key exactly
  {
    const int64_t ddx = (int64_t)cx - Xo, ddy = (int64_t)cy - y;
    const int64_t d2 = ddx * ddx + ddy * ddy;
    if (cx > 65535u || d2 != 4 * (int64_t)m + (ww >> 18) + 4 * (int64_t)(y >> 1) * (y >> 1) ||
        ((ww & 1u) != (cx > (uint32_t)Xo ? 1u : 0u) && ad != 0u))
      __trap();
  }
#endif
  return lab;
}

template <bool MAY_EMPTY, bool BANDED, bool FIX, bool FULL>
__device__ __forceinline__ void walk_wsk(const PassArgs& a, const CUtensorMap* tm, int x0, int X, int y0,
                                         uint32_t* smem) {
  const int k = a.k;
  const int tid = (int)threadIdx.x;
  const int nw = FULL ? min(a.nwalk, k - (y0 - a.y_lo)) : 1;
  const int nout = FULL ? (a.y_hi - y0 + k - 1) >> a.lk : min(a.walk, (a.y_hi - y0 + k - 1) >> a.lk);
  const int nlist = FULL ? nw * nout : nout + 2;
  const int SE = stage_elems_sk(k);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)(a.walk + 2) * SE);
  stage_walk<FULL, BANDED>(a, tm, x0, y0, k, nout, nlist, true, (k + 3) & ~3, SE, smem, bars);

  int Xo[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) Xo[e] = X + e * k;
  const bool left_out = FIX && X - k < 0;
  const int nc = FIX ? (X >= a.N ? 0 : ((a.N - 1 - X) >> a.lk) + 1) : 8;  // in-grid slot columns (walk_sk)
  const uint32_t uk = (uint32_t)k, k2q = uk * uk / 4u, kh = uk / 2u;
  bool any_empty = false;

  auto consume = [&](int i, uint32_t p, RowW& R) {
    mbar_wait(&bars[i], 0u);
    const uint32_t* st = smem + (size_t)i * SE + tid;
    uint32_t lab[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) lab[s] = st[s * 128];
    if constexpr (FIX) {  // an out-of-grid neighbour column -> the same output's centre label (a duplicate)
      lab[0] = left_out ? lab[1] : lab[0];
      if (nc < 4) {  // the partial last group of 4k columns
#pragma unroll
        for (int s = 1; s < 5; ++s) lab[s] = s >= nc + 1 ? lab[s - 1] : lab[s];
      }
      lab[5] = nc <= 4 ? lab[4] : lab[5];
    }
    build_w<MAY_EMPTY>(lab, Xo, p, uk, k2q, kh, a.one, a.sh16, R);
  };

  const int64_t kp = (int64_t)k * a.pitch;
  auto run = [&](int yw, int n, int ibase) {
    const uint32_t p = (uint32_t)yw & 1u;
    RowW r0, r1, r2;
    if constexpr (FULL) {
      consume(ibase + 1, p, r1);  // (the row above the first output is outside the grid: r1 serves as both)
    } else {
      consume(ibase, p, r0);
      consume(ibase + 1, p, r1);
    }
    int y = yw;
    uint32_t* po = a.out + (int64_t)(yw - a.row0) * a.pitch + X;
    int j = 0;
    auto eval = [&](const RowW& Pv, const RowW& Cv, const RowW& Nx) {
      const uint32_t h = (uint32_t)y >> 1;
      const uint32_t mh = 0u - h, hh = 4u * h * h;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t o = best_w<MAY_EMPTY>(Pv, Cv, Nx, e, Xo[e], y, mh, hh);
        if (e < nc) {
          if (MAY_EMPTY) any_empty |= o == EMPTY;
          store_out(a, BANDED, y, Xo[e], po + e * k, o);
        }
      }
      po += kp;
      y += k;
    };
    auto step = [&](const RowW& Pv, const RowW& Cv, RowW& Nx) -> bool {
      if (!FULL || j + 1 < n) {
        consume(ibase + j + 2, p, Nx);
        eval(Pv, Cv, Nx);
      } else {
        eval(Pv, Cv, Cv);  // FULL: the row below the last output is outside the grid
      }
      return ++j < n;
    };
    if (FULL) {
      if (step(r1, r1, r2)) {
#pragma unroll 1
        while (true) {
          if (!step(r1, r2, r0)) break;
          if (!step(r2, r0, r1)) break;
          if (!step(r0, r1, r2)) break;
        }
      }
    } else {
#pragma unroll 1
      while (true) {
        if (!step(r0, r1, r2)) break;
        if (!step(r1, r2, r0)) break;
        if (!step(r2, r0, r1)) break;
      }
    }
  };
  if constexpr (FULL) {
#pragma unroll 1
    for (int w = 0; w < nw; ++w) run(y0 + w, nout, w * nout - 1);
  } else {
    run(y0, nout, 0);
  }
  if (a.loc_out && tid == 0) atomicOr(a.loc_out, 1u);  // locality is not tracked on this path
  if (MAY_EMPTY && a.empty_flag != nullptr && __syncthreads_or(any_empty) && tid == 0) atomicOr(a.empty_flag, 1ull);
}

// grid as jump_pass_sk with k >= 256 (groups of 4k columns, k / 128 residue blocks each); runtime k.
template <bool MAY_EMPTY, bool BANDED>
__global__ void __launch_bounds__(kThreads, VD_MIN_BLOCKS) jump_pass_wsk(PassArgs a, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(128) uint32_t dyn_smem[];
  const int xb = (int)blockIdx.x;
  const bool full = a.nwalk > 0;
  const int seg = full ? 0 : (int)(a.res_in_y ? blockIdx.z : blockIdx.y);
  const int res = full ? (int)blockIdx.z * a.nwalk : (int)(a.res_in_y ? blockIdx.y : blockIdx.z);
  const int y0 = a.y_lo + res + seg * a.walk * a.k;
  if (res >= a.k || y0 >= a.y_hi) return;  // (uniform: the whole CTA leaves)
  const int k = a.k;
  const int lr = a.lk - 7;  // k / 128 residue blocks per group of 4k columns
  const int g = xb >> lr, rb = xb & ((1 << lr) - 1);
  const int x0 = 4 * k * g + 128 * rb;
  if (x0 >= a.N) return;  // (the partial last group of a grid that is not a multiple of 4k)
  const int X = x0 + (int)threadIdx.x;
  const bool fix = g == 0 || x0 + 4 * k + 128 > a.N;  // some right neighbour column (X + 4k) beyond the grid
  if (full) {
    if (fix) walk_wsk<MAY_EMPTY, BANDED, true, true>(a, &tm, x0, X, y0, dyn_smem);
    else walk_wsk<MAY_EMPTY, BANDED, false, true>(a, &tm, x0, X, y0, dyn_smem);
  } else {
    if (fix) walk_wsk<MAY_EMPTY, BANDED, true, false>(a, &tm, x0, X, y0, dyn_smem);
    else walk_wsk<MAY_EMPTY, BANDED, false, false>(a, &tm, x0, X, y0, dyn_smem);
  }
}

// ------------------------------------------------------------------ wide jump pass
//
// Same pass for what the fast kernels do not take: steps that are not powers of two, steps
// > 4096 beyond N = 32768 (> 256 with EMPTY beyond N = 16384).

// Generic pass (any k, any N <= 65536, EMPTY allowed): one thread = 4 pixels of one row,
// 64-bit keys, candidates read straight from global memory (L2-friendly for the large steps
// it serves).  V4: k % 4 == 0, so the neighbour columns are 16-byte aligned vectors.
// Rows are launched residue class by residue class (y_lo + r, y_lo + r + k, ... = a.segs rows
// per class), so that consecutive CTA rows share two of their three input rows in L2.
template <int METRIC, bool VN, bool V4>
__global__ void __launch_bounds__(kThreads) jump_pass_wide(PassArgs a) {
  const int xb = (int)(blockIdx.x % (unsigned)a.xblocks);
  const int j = (int)(blockIdx.x / (unsigned)a.xblocks);
  const int res = j / a.segs, seg = j - res * a.segs;
  const int x = (xb * kThreads + (int)threadIdx.x) * 4;
  const int y = a.y_lo + res + seg * a.k, k = a.k, N = a.N;
  const bool live = x < N && y < a.y_hi && res < a.k;
  bool any_empty = false;
  if (live) {
    uint32_t best[4];
    uint64_t bd[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) { best[e] = EMPTY; bd[e] = ~0ull; }
#pragma unroll
    for (int oy = -1; oy <= 1; ++oy) {
      const int r = y + oy * k;
      if (r < 0 || r >= N) continue;
      const uint32_t* p = row_ptr(a, r);
#pragma unroll
      for (int ox = -1; ox <= 1; ++ox) {
        if (VN && ox != 0 && oy != 0) continue;  // Von Neumann: no diagonals
        const int q0 = x + ox * k;
        if constexpr (V4) {
          if (q0 < 0 || q0 >= N) continue;  // the whole aligned vector is out of the grid
          const uint4 v = *reinterpret_cast<const uint4*>(p + q0);
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (q0 + e < N) consider64<METRIC>(w[e], x + e, y, bd[e], best[e]);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int q = q0 + e;
            if (x + e >= N || q < 0 || q >= N) continue;
            consider64<METRIC>(p[q], x + e, y, bd[e], best[e]);
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) any_empty |= (x + e < N) && best[e] == EMPTY;
    // columns >= N of the ragged tail hold don't-care values (never read as pixels)
    store_out(a, true, y, x, a.out + (int64_t)(y - a.row0) * a.pitch + x, make_uint4(best[0], best[1], best[2], best[3]));
  }
  if (a.empty_flag != nullptr && __syncthreads_or(any_empty) && threadIdx.x == 0) atomicOr(a.empty_flag, 1ull);
}

#ifndef VD_TEMPLATE_KERNELS_ONLY  // the non-template kernels live in vd.cu's translation unit only
// ------------------------------------------------------------------ peer halos (NEXT-3)
// Copy this band's first / last k rows into the neighbours' halo buffers (the first pass of
// a sequence; later passes push from inside the pass kernel, store_out).
__global__ void push_rows(const uint32_t* __restrict__ band, int64_t pitch, int rows, int N, int k,
                          uint32_t* __restrict__ to_top, uint32_t* __restrict__ to_bot) {
  const int64_t n4 = (int64_t)k * (pitch / 4);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (pitch / 4), c = (i % (pitch / 4)) * 4;
    if (c >= N) continue;
    if (to_top) *reinterpret_cast<uint4*>(to_top + r * pitch + c) = *reinterpret_cast<const uint4*>(band + r * pitch + c);
    if (to_bot)
      *reinterpret_cast<uint4*>(to_bot + r * pitch + c) =
          *reinterpret_cast<const uint4*>(band + (int64_t)(rows - k + r) * pitch + c);
  }
}

// After this rank's pushes for the neighbours' next pass: make them visible system-wide,
// then publish `seq` into each neighbour's flag word (its flags[1] = "from the band above",
// flags[0] = "from the band below").
__global__ void peer_signal(uint32_t* flag_top_nbr, uint32_t* flag_bot_nbr, uint32_t seq) {
  __threadfence_system();
  if (flag_top_nbr) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag_top_nbr), "r"(seq) : "memory");
  if (flag_bot_nbr) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag_bot_nbr), "r"(seq) : "memory");
}

// Wait until the neighbours published `seq` (their pushes into this rank's halos landed).
// Bounded: after ~20 s it records an error instead of hanging the GPU.
__global__ void peer_wait(const uint32_t* flags, int need_top, int need_bot, uint32_t seq, uint32_t* err) {
  for (int side = 0; side < 2; ++side) {
    if (!(side == 0 ? need_top : need_bot)) continue;
    const uint32_t* f = flags + side;
    for (long long it = 0;; ++it) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if ((int32_t)(v - seq) >= 0) break;
      if (it > (1ll << 24)) {  // err: mapped host memory, read by the host at every libvd call
        *(volatile uint32_t*)err = 1u;
        __threadfence_system();
        return;
      }
      __nanosleep(1000);
    }
  }
}

// ------------------------------------------------------------------ JFA init
// P:68 "defining the positions as the starting points for each flood": every pixel
// EMPTY, then each seed pixel holds its own label.
__global__ void fill_value(uint4* __restrict__ p, int64_t n4, uint32_t value) {
  const uint4 v = make_uint4(value, value, value, value);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// After a JFA / StF that started from the virtual far seed V (vd.cu: jfa_init), turn the
// V labels that survived (only possible with Von Neumann-only waves) back into EMPTY.
__global__ void replace_value(uint4* __restrict__ p, int64_t n4, uint32_t from, uint32_t to) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = p[i];
    v.x = v.x == from ? to : v.x;
    v.y = v.y == from ? to : v.y;
    v.z = v.z == from ? to : v.z;
    v.w = v.w == from ? to : v.w;
    p[i] = v;
  }
}

// labels[seed pixel] <- seed label, for seeds whose row lies in [row0, row0 + rows).
// Co-located seeds write the same value, so the unordered writes are benign.
__global__ void stamp(uint32_t* __restrict__ g, int64_t pitch, int row0, int rows,
                      const uint32_t* __restrict__ seeds, int64_t s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = seeds[i];
    int y = (int)(c >> 16) - row0, x = (int)(c & 0xFFFFu);
    if (y >= 0 && y < rows) g[(int64_t)y * pitch + x] = c;
  }
}

// First JFA pass fused with the initialisation.  The input of pass k_1 is "unclaimed
// everywhere, each seed pixel holds its seed", so its output at pixel p is the best of
// the seeds at p and at p + o k_1, o in Table 1: Alg. 1's scatter form of the
// pass (R-12), where every seed offers itself to the pixels q - o k_1.  The grid
// (this band) must already hold `unclaimed` everywhere (fill_value).  An offer is a CAS loop
// on the pixel's label with the exact key (distance in uint64, then label; R-3), so the
// result is the minimum over all offers in any order -- the gather pass's result.
// metric 0/1 (Euclidean / Manhattan), vn: Von Neumann offsets only (Table 1's axis ones).
__device__ __forceinline__ uint64_t dist_c(uint32_t c, int x, int y, int metric) {
  const uint32_t dx = (uint32_t)abs((int)(c & 0xFFFFu) - x), dy = (uint32_t)abs((int)(c >> 16) - y);
  return metric == 0 ? (uint64_t)(dx * dx) + (uint64_t)(dy * dy) : (uint64_t)(dx + dy);
}
__global__ void jfa_first_pass(uint32_t* __restrict__ g, int64_t pitch, int row0, int rows, int N, int k,
                               const uint32_t* __restrict__ seeds, int64_t s, uint32_t unclaimed, int metric, int vn) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = seeds[i];
    const int cx = (int)(c & 0xFFFFu), cy = (int)(c >> 16);
#pragma unroll
    for (int oy = -1; oy <= 1; ++oy) {
#pragma unroll
      for (int ox = -1; ox <= 1; ++ox) {
        if (vn && ox != 0 && oy != 0) continue;
        const int px = cx - ox * k, py = cy - oy * k;  // the pixel whose neighbour o*k is this seed
        if (px < 0 || px >= N || py < row0 || py >= row0 + rows || py >= N) continue;
        uint32_t* a = g + (int64_t)(py - row0) * pitch + px;
        const uint64_t dc = dist_c(c, px, py, metric);
        uint32_t cur = *(volatile uint32_t*)a;
        while (cur == unclaimed || dc < dist_c(cur, px, py, metric) || (dc == dist_c(cur, px, py, metric) && c < cur)) {
          const uint32_t prev = atomicCAS(a, cur, c);
          if (prev == cur) break;
          cur = prev;
        }
      }
    }
  }
}

// JFA's first pass as a gather from a seed bitmap (r02c): bits[y * wpr + x / 32] bit x % 32 = a seed
// at (x, y).  Pass k_1 gives pixel p the best seed among p + o k_1 (Table 1); since a seed's label is
// its position, the key (d2, c) of an offset o depends on o alone, and the nine offsets have a fixed
// order for both metrics: the centre, then the axis offsets by label (row above, left, right, row
// below), then the diagonals by label.  One thread per 32-pixel word of a row: the word is written
// unclaimed, then every set bit of each in-grid neighbour word, lowest priority first, overwrites its
// pixel (program order keeps the best).  The scatter's result, without the fill or the CAS loops.
__global__ void seed_bits(uint32_t* __restrict__ bits, int64_t wpr, const uint32_t* __restrict__ seeds, int64_t s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = seeds[i];
    const uint32_t x = c & 0xFFFFu, y = c >> 16;
    atomicOr(&bits[(int64_t)y * wpr + (x >> 5)], 1u << (x & 31));
  }
}
__global__ void jfa_first_gather(uint32_t* __restrict__ g, int64_t pitch, int row0, int rows, int N, int k,
                                 const uint32_t* __restrict__ bits, int64_t wpr, uint32_t unclaimed, int vn) {
  const int kw = k >> 5;  // k in words (k >= 32)
  // 2-D grid: blockIdx.x over the words of a row, blockIdx.y strided over rows (no 64-bit division)
  for (int r = blockIdx.y; r < rows; r += gridDim.y)
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < (int)wpr; w += gridDim.x * blockDim.x) {
    const int y = row0 + r, x0 = w << 5;
    uint32_t* out = g + (int64_t)r * pitch + x0;
    const uint4 u = make_uint4(unclaimed, unclaimed, unclaimed, unclaimed);
#pragma unroll
    for (int q = 0; q < 8; ++q) reinterpret_cast<uint4*>(out)[q] = u;
    // offsets in increasing priority (the last store to a pixel wins): diagonals, axis, centre
    constexpr int OX[9] = {1, -1, 1, -1, 0, 1, -1, 0, 0};
    constexpr int OY[9] = {1, 1, -1, -1, 1, 0, 0, -1, 0};
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      if (vn && OX[i] != 0 && OY[i] != 0) continue;
      const int qy = y + OY[i] * k, qw = w + OX[i] * kw;
      if (qy < 0 || qy >= N || qw < 0 || (int64_t)qw >= wpr) continue;
      uint32_t b = __ldg(bits + (int64_t)qy * wpr + qw);
      const uint32_t base = ((uint32_t)qy << 16) | (uint32_t)(qw << 5);
      while (b) {
        const int j = __ffs(b) - 1;
        b &= b - 1;
        out[j] = base | (uint32_t)j;
      }
    }
  }
}

// Sparse JFA passes (r02c): JFA's second and third passes at C5 read inputs that are 94-98% EMPTY.
// An occupancy bitmap (bit = the pixel holds a label) lets a thread skip the EMPTY candidates: one
// thread per four pixels of a row (a warp = 128 pixels = four bitmap words) reads the nine candidate
// nibbles and loads labels only where a nibble is set.  Keys in lattice units (§5.6: every label is
// congruent to its pixel mod 2k, N <= 64k): (a^2 + b^2, b + 128, a + 128) packed in 32 bits.  The pass
// also writes its output's bitmap for the next sparse pass.
__global__ void occ_from_seeds(uint32_t* __restrict__ bits, int64_t wpr, const uint32_t* __restrict__ seeds,
                               int64_t s, int N, int k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = seeds[i];
    const int sx = (int)(c & 0xFFFFu), sy = (int)(c >> 16);
#pragma unroll
    for (int oy = -1; oy <= 1; ++oy)
#pragma unroll
      for (int ox = -1; ox <= 1; ++ox) {  // the pixels of JFA's first pass that this seed claims
        const int px = sx - ox * k, py = sy - oy * k;
        if (px >= 0 && px < N && py >= 0 && py < N) atomicOr(&bits[(int64_t)py * wpr + (px >> 5)], 1u << (px & 31));
      }
  }
}
__global__ void __launch_bounds__(256) jfa_sparse_pass(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                       int64_t pitch, int N, int k, int lk,
                                                       const uint32_t* __restrict__ bits_in, uint32_t* __restrict__ bits_out,
                                                       int64_t wpr, unsigned long long* empty_flag) {
  // 2-D grid: blockIdx.x over quads of a row, blockIdx.y strided over rows (no 64-bit division);
  // N / 4 is a multiple of 32, so every lane of a warp runs the same iterations
  const int per_row = N >> 2;
  const int lane = (int)threadIdx.x & 31;
  bool any_e = false;
  for (int y = blockIdx.y; y < N; y += gridDim.y)
  for (int xq = blockIdx.x * blockDim.x + threadIdx.x; xq < per_row; xq += gridDim.x * blockDim.x) {
    const int x = xq << 2;
    uint32_t best[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
#pragma unroll
    for (int oy = -1; oy <= 1; ++oy) {
      const int qy = y + oy * k;
      if (qy < 0 || qy >= N) continue;
#pragma unroll
      for (int ox = -1; ox <= 1; ++ox) {
        const int qx = x + ox * k;
        if (qx < 0 || qx >= N) continue;
        const uint32_t nib = (__ldg(bits_in + (int64_t)qy * wpr + (qx >> 5)) >> (qx & 31)) & 0xFu;
        if (nib == 0u) continue;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(in + (int64_t)qy * pitch + qx));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (!((nib >> e) & 1u)) continue;
          const uint32_t c = w[e];
          const int a = ((int)(c & 0xFFFFu) - (x + e)) >> lk, b = ((int)(c >> 16) - y) >> lk;  // exact (lattice)
          const uint32_t key = ((uint32_t)(a * a + b * b) << 16) | ((uint32_t)(b + 128) << 8) | (uint32_t)(a + 128);
          best[e] = min(best[e], key);
        }
      }
    }
    uint32_t o[4], onib = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (best[e] == 0xFFFFFFFFu) {
        o[e] = EMPTY;
        any_e = true;
      } else {
        const int a = (int)(best[e] & 0xFFu) - 128, b = (int)((best[e] >> 8) & 0xFFu) - 128;
        o[e] = ((uint32_t)(y + (b << lk)) << 16) | (uint32_t)(x + e + (a << lk));
        onib |= 1u << e;
      }
    }
    *reinterpret_cast<uint4*>(out + (int64_t)y * pitch + x) = make_uint4(o[0], o[1], o[2], o[3]);
    if (bits_out != nullptr) {  // eight lanes = one 32-pixel word of the output's bitmap
      uint32_t wv = onib << ((lane & 7) * 4);
      wv |= __shfl_xor_sync(0xFFFFFFFFu, wv, 1);
      wv |= __shfl_xor_sync(0xFFFFFFFFu, wv, 2);
      wv |= __shfl_xor_sync(0xFFFFFFFFu, wv, 4);
      if ((lane & 7) == 0) bits_out[(int64_t)y * wpr + (x >> 5)] = wv;
    }
  }
  if (empty_flag != nullptr && __any_sync(0xFFFFFFFFu, any_e) && lane == 0) atomicOr(empty_flag, 1ull);
}

// ------------------------------------------------------------------ dJFA
// SimulateParticles (Alg. 1): new = clamp(old + disp) per axis (R-10); at
// N = 65536 the EMPTY pixel (65535, 65535) is reserved -> (65534, 65535) (R-4).
__global__ void move_clamp(const uint32_t* __restrict__ old_s, const short2* __restrict__ disp,
                           uint32_t* __restrict__ new_s, int64_t s, int N) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = old_s[i];
    short2 d = disp[i];
    int x = (int)(c & 0xFFFFu) + d.x, y = (int)(c >> 16) + d.y;
    x = min(max(x, 0), N - 1);
    y = min(max(y, 0), N - 1);
    if (N == 65536 && x == 65535 && y == 65535) x = 65534;
    new_s[i] = ((uint32_t)y << 16) | (uint32_t)x;
  }
}

// fwd's index of label c: the label itself (fp = 0: rows of 2^16 entries, the fused dJFA frame's
// layout) or (y, x) -> y fp + x (fp = N: the N x N layout of the separate remap's runs, whose gathers
// then spread over a quarter of the address range at C4; r02c).
// SimulateParticles (Alg. 1) fused with the forward map (R-9):
// new = clamp(old + disp) per axis (R-10; the reserved pixel at N = 65536, R-4), then
// fwd[old] <- min(fwd[old], new): co-located seeds leave the smallest new label.  fwd is indexed
// by the label value itself (rows of 2^16 entries, N rows: one address computation per lookup).  fwd is
// all EMPTY between dJFA steps (reset_stamp restores it).
// flag_g (or null): the fused frame (NEXT-1) also marks the new seed pixel here, BEFORE the first
// pass, with EMPTY, which the pass's in-stage remap turns into the pixel's own position (R-9:
// remap, then re-stamp).  A dJFA diagram holds no EMPTY, so the marker is free.  One band.
__global__ void move_fwd(const uint32_t* __restrict__ old_s, const short2* __restrict__ disp,
                         uint32_t* __restrict__ new_s, uint32_t* __restrict__ fwd, int fp, int64_t s, int N,
                         uint32_t* __restrict__ flag_g = nullptr, int64_t pitch = 0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = old_s[i];
    const short2 d = disp[i];
    int x = (int)(c & 0xFFFFu) + d.x, y = (int)(c >> 16) + d.y;
    x = min(max(x, 0), N - 1);
    y = min(max(y, 0), N - 1);
    if (N == 65536 && x == 65535 && y == 65535) x = 65534;
    const uint32_t nw = ((uint32_t)y << 16) | (uint32_t)x;
    new_s[i] = nw;
    atomicMin(&fwd[fwd_index(c, fp)], nw);
    if (flag_g) flag_g[(int64_t)y * pitch + x] = EMPTY;  // marker: "new seed here" (jump_pass_sk_remap)
  }
}

// After the remap: restore fwd to all-EMPTY (its entries at the old seed pixels) and
// re-stamp the new seed pixels of this band (R-9: remap, then re-stamp).  Co-located seeds
// write the same values, so the unordered writes are benign.
__global__ void reset_stamp(uint32_t* __restrict__ fwd, int fp, int N, const uint32_t* __restrict__ old_s,
                            const uint32_t* __restrict__ new_s, uint32_t* __restrict__ g, int64_t pitch, int row0,
                            int rows, int64_t s, int do_reset) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    if (do_reset) {
      const uint32_t o = old_s[i];
      fwd[fwd_index(o, fp)] = EMPTY;
    }
    const uint32_t c = new_s[i];
    const int y = (int)(c >> 16) - row0, x = (int)(c & 0xFFFFu);
    if (y >= 0 && y < rows) g[(int64_t)y * pitch + x] = c;
  }
}

// Fused dJFA frame (NEXT-1), after the first pass: fwd back to all-EMPTY (its entries at the old
// seed pixels).
__global__ void fwd_reset(uint32_t* __restrict__ fwd, int fp, int N, const uint32_t* __restrict__ old_s, int64_t s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = old_s[i];
    fwd[fwd_index(o, fp)] = EMPTY;
  }
}

// Reuse VD_{t-1}: every label moves with its seed, labels[p] <- fwd[labels[p]].
// Neighbouring pixels mostly share a label, so the gathers hit L1.
// Row-major sweeps below (launch bounds: 8 CTAs of 256 threads resident per SM, the grid being
// num_sms x 8: at 36 registers only 7 fit, and the eighth CTA per SM ran as a second, nearly empty
// wave -- the separate remap took 0.72 instead of 0.47 ms at C4, r02c): CTAs stride over rows, threads over 4-label quads of a row, with
// the quad loop unrolled so that several 128-bit loads are in flight per thread.
#ifndef VD_REMAP_UNROLL
#define VD_REMAP_UNROLL 4
#endif
constexpr int kRemapUnroll = VD_REMAP_UNROLL;  // row quads in flight per remap thread
// loc (or null): set to 1 unless every remapped label lies within Chebyshev distance 44 of
// its pixel (hence within Euclidean 63 = kLocR, 44 * sqrt(2) < 63): the packed-key passes'
// precondition (walk).  Tracked as max over pixels of (cy - y + 44, cx - x + 44) in two
// 16-bit lanes (a lane outside [0, 88] wraps high).
__global__ void __launch_bounds__(256, 8) remap(uint32_t* __restrict__ g, int64_t pitch, int rows, int N, const uint32_t* __restrict__ fwd, int fp,
                      int row0, uint32_t* __restrict__ loc) {
  uint32_t mx = 0;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    uint32_t* row = g + (int64_t)r * pitch;
    const uint32_t nb = __vsub2(0x002C002Cu, ((uint32_t)(row0 + r) << 16));  // (44 - y, 44) per lane
#pragma unroll kRemapUnroll
    for (int x = 4 * (int)threadIdx.x; x < N; x += 4 * (int)blockDim.x) {
      uint4* p = reinterpret_cast<uint4*>(row + x);
      uint4 v = *p;
      uint32_t w[4] = {v.x, v.y, v.z, v.w};
      const uint32_t nbx = __vsub2(nb, (uint32_t)x);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t c = w[e];
        if (x + e < N) {
          const uint32_t nc = c != EMPTY ? __ldg(fwd + fwd_index(c, fp)) : EMPTY;
          w[e] = nc;
          // (cy - y + 44, cx - x - e + 44); EMPTY is far
          mx = __vmaxu2(mx, nc == EMPTY ? 0xFFFFFFFFu : __vadd2(nc, __vsub2(nbx, (uint32_t)e)));
        }
      }
      *p = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  const bool far = (mx >> 16) > 88u || (mx & 0xFFFFu) > 88u;
  if (loc && __syncthreads_or(far) && threadIdx.x == 0) atomicOr(loc, 1u);
}

// The same remap with lanes on consecutive pixels, software-pipelined.  A warp covers 128
// consecutive pixels of a row per round (lane t: pixels x0 + t + 32 e, e < 4), so one gather
// instruction touches the fwd entries of the 2-3 seeds whose regions cross 32 pixels.  The
// remap is latency-bound (a DRAM load of the labels, then a dependent L2 gather of fwd), so
// each thread loads the labels of its NEXT round before it gathers and stores the current one:
// the two latencies overlap instead of adding up.  Same result and locality flag as remap().
__global__ void __launch_bounds__(256, 8) remap_lanes(uint32_t* __restrict__ g, int64_t pitch, int rows, int N, const uint32_t* __restrict__ fwd, int fp,
                            int row0, uint32_t* __restrict__ loc) {
  uint32_t mx = 0;
  const int lane = (int)threadIdx.x & 31, warp = (int)threadIdx.x >> 5, nwarps = (int)blockDim.x >> 5;
  // the warp's rounds: (row r, chunk x0) in row-major order over this CTA's rows
  const uint32_t per_row = (uint32_t)(N + 127) / 128u;
  const int nround = ((rows - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * (int)per_row;
  auto round_at = [&](int i, int& r, int& x0) {
    const uint32_t q = (uint32_t)i / per_row;
    r = (int)blockIdx.x + (int)q * (int)gridDim.x;
    x0 = (int)((uint32_t)i - q * per_row) * 128;
  };
  auto load = [&](int i, uint32_t (&c)[4]) {
    int r, x0;
    round_at(i, r, x0);
    const uint32_t* row = g + (int64_t)r * pitch;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int x = x0 + 32 * e + lane;
      c[e] = x < N ? row[x] : EMPTY;
    }
  };
  uint32_t cur[4], nxt[4] = {EMPTY, EMPTY, EMPTY, EMPTY};
  int i = warp;
  if (i < nround) load(i, cur);
  for (; i < nround; i += nwarps) {
    if (i + nwarps < nround) load(i + nwarps, nxt);  // next round's labels: in flight during the gathers
    uint32_t nc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      nc[e] = cur[e] != EMPTY ? __ldg(fwd + fwd_index(cur[e], fp)) : EMPTY;
    int r, x0;
    round_at(i, r, x0);
    uint32_t* row = g + (int64_t)r * pitch;
    const uint32_t nb = __vsub2(0x002C002Cu, ((uint32_t)(row0 + r) << 16));  // (44 - y, 44) per lane
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int x = x0 + 32 * e + lane;
      if (x < N) {
        row[x] = nc[e];
        mx = __vmaxu2(mx, nc[e] == EMPTY ? 0xFFFFFFFFu : __vadd2(nc[e], __vsub2(nb, (uint32_t)x)));
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) cur[e] = nxt[e];
  }
  const bool far = (mx >> 16) > 88u || (mx & 0xFFFFu) > 88u;
  if (loc && __syncthreads_or(far) && threadIdx.x == 0) atomicOr(loc, 1u);
}

// ------------------------------------------------------------------ reductions (block_sum_u64 above)

// Eq. 5 numerator: count of pixels with equal labels in a band.
__global__ void __launch_bounds__(256, 8) match_count(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t pitch,
                            int rows, int N, unsigned long long* __restrict__ out) {
  uint32_t cnt = 0;  // per thread: at most rows/gridDim * N/blockDim*... < 2^32 for any grid we allow
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint32_t* ra = a + (int64_t)r * pitch;
    const uint32_t* rb = b + (int64_t)r * pitch;
#pragma unroll 4
    for (int x = 4 * (int)threadIdx.x; x < N; x += 4 * (int)blockDim.x) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(ra + x));
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(rb + x));
      const int nv = min(4, N - x);
      cnt += (u.x == v.x) + (nv > 1 && u.y == v.y) + (nv > 2 && u.z == v.z) + (nv > 3 && u.w == v.w);
    }
  }
  uint64_t t = block_sum_u64(cnt);
  if (threadIdx.x == 0 && t) atomicAdd(out, (unsigned long long)t);
}

// Number of pixels of a band holding `value` (StF's "fully flooded" test).
__global__ void __launch_bounds__(256, 8) count_value(const uint32_t* __restrict__ g, int64_t pitch, int rows, int N, uint32_t value,
                            unsigned long long* __restrict__ out) {
  uint32_t cnt = 0;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint32_t* row = g + (int64_t)r * pitch;
#pragma unroll 4
    for (int x = 4 * (int)threadIdx.x; x < N; x += 4 * (int)blockDim.x) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(row + x));
      const int nv = min(4, N - x);
      cnt += (u.x == value) + (nv > 1 && u.y == value) + (nv > 2 && u.z == value) + (nv > 3 && u.w == value);
    }
  }
  uint64_t t = block_sum_u64(cnt);
  if (threadIdx.x == 0 && t) atomicAdd(out, (unsigned long long)t);
}

// Checksum sum_p fmix32((uint32)(p * 0x9E3779B9) ^ label[p]) in uint64 over a band
// (p = global y*N + x < 2^32).
__global__ void __launch_bounds__(256, 8) label_hash(const uint32_t* __restrict__ g, int64_t pitch, int row0, int rows, int N,
                           unsigned long long* __restrict__ out) {
  // sum over p of fmix32(p * 0x9E3779B9 ^ label[p]) mod 2^64 (p = y * N + x).  The position
  // term advances by a constant per column, so it costs one add per pixel.
  constexpr uint32_t C = 0x9E3779B9u;
  uint64_t h = 0;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint32_t* row = g + (int64_t)r * pitch;
    const uint32_t pc0 = (uint32_t)(row0 + r) * (uint32_t)N * C;
#pragma unroll 4
    for (int x = 4 * (int)threadIdx.x; x < N; x += 4 * (int)blockDim.x) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(row + x));
      const uint32_t b = pc0 + (uint32_t)x * C;
      if (x + 3 < N) {
        h += (uint64_t)fmix32(b ^ u.x) + fmix32((b + C) ^ u.y);
        h += (uint64_t)fmix32((b + 2 * C) ^ u.z) + fmix32((b + 3 * C) ^ u.w);
      } else {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (x + e < N) h += fmix32((b + (uint32_t)e * C) ^ w[e]);
      }
    }
  }
  uint64_t t = block_sum_u64(h);
  if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)t);
}

#endif  // VD_TEMPLATE_KERNELS_ONLY

}  // namespace vdk
