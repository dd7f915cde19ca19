// jump_pass_fast instantiations (see vd_launch.h).
#include "vd_launch.h"

namespace vdl {

template <int KM, bool ME, bool BD, int MT, bool VN, bool REL>
static cudaError_t fast_one(int dev, const vdk::PassArgs& a, dim3 grid, dim3 blk, size_t sm, cudaStream_t st) {
  static std::atomic<uint64_t> opted{0};
  const cudaError_t e = opt_in_smem(opted, dev, vdk::jump_pass_fast<KM, ME, BD, MT, VN, REL>,
                                    REL ? vdk::kSmemBudgetRel : vdk::kSmemBudget);
  if (e != cudaSuccess) return e;
  vdk::jump_pass_fast<KM, ME, BD, MT, VN, REL><<<grid, blk, sm, st>>>(a);
  return cudaSuccess;
}
template <int KM, bool ME, bool BD, bool REL>
static cudaError_t fast_mv(int dev, int metric, bool vn, const vdk::PassArgs& a, dim3 g, dim3 b, size_t sm,
                           cudaStream_t st) {
  if (metric == 0)
    return vn ? fast_one<KM, ME, BD, 0, true, REL>(dev, a, g, b, sm, st) : fast_one<KM, ME, BD, 0, false, REL>(dev, a, g, b, sm, st);
  return vn ? fast_one<KM, ME, BD, 1, true, REL>(dev, a, g, b, sm, st) : fast_one<KM, ME, BD, 1, false, REL>(dev, a, g, b, sm, st);
}
template <int KM>
static cudaError_t fast_k(int dev, bool me, bool bd, bool rel, int metric, bool vn, const vdk::PassArgs& a, dim3 g,
                          dim3 b, size_t sm, cudaStream_t st) {
  if (rel)  // windowed coordinates (complete diagrams beyond the plain fast kernel's range)
    return bd ? fast_mv<KM, false, true, true>(dev, metric, vn, a, g, b, sm, st)
              : fast_mv<KM, false, false, true>(dev, metric, vn, a, g, b, sm, st);
  if (me) return bd ? fast_mv<KM, true, true, false>(dev, metric, vn, a, g, b, sm, st)
                    : fast_mv<KM, true, false, false>(dev, metric, vn, a, g, b, sm, st);
  return bd ? fast_mv<KM, false, true, false>(dev, metric, vn, a, g, b, sm, st)
            : fast_mv<KM, false, false, false>(dev, metric, vn, a, g, b, sm, st);
}

cudaError_t launch_fast(int dev, uint32_t k, bool me, bool bd, bool rel, int metric, bool vn, const vdk::PassArgs& a,
                        dim3 g, dim3 b, size_t sm, cudaStream_t st) {
  if (k == 1) return fast_k<1>(dev, me, bd, rel, metric, vn, a, g, b, sm, st);
  if (k == 2) return fast_k<2>(dev, me, bd, rel, metric, vn, a, g, b, sm, st);
  return fast_k<4>(dev, me, bd, rel, metric, vn, a, g, b, sm, st);
}

}  // namespace vdl
