// jump_pass_wsk instantiations (wide exact pass, N <= 65536; see vd_launch.h).
#include "vd_launch.h"

namespace vdl {

template <bool ME, bool BD>
static cudaError_t wsk_one(int dev, const vdk::PassArgs& a, const CUtensorMap& tm, dim3 g, dim3 b, size_t sm,
                           cudaStream_t st) {
  static std::atomic<uint64_t> opted{0};
  const cudaError_t e = opt_in_smem(opted, dev, vdk::jump_pass_wsk<ME, BD>, vdk::kSmemBudget);
  if (e != cudaSuccess) return e;
  vdk::jump_pass_wsk<ME, BD><<<g, b, sm, st>>>(a, tm);
  return cudaSuccess;
}

cudaError_t launch_wsk(int dev, bool me, bool bd, const vdk::PassArgs& a, const CUtensorMap& tm, dim3 g, dim3 b,
                       size_t sm, cudaStream_t st) {
  if (me) return bd ? wsk_one<true, true>(dev, a, tm, g, b, sm, st) : wsk_one<true, false>(dev, a, tm, g, b, sm, st);
  return bd ? wsk_one<false, true>(dev, a, tm, g, b, sm, st) : wsk_one<false, false>(dev, a, tm, g, b, sm, st);
}

}  // namespace vdl
