// jump_pass_sk instantiations for k >= 512 (see vd_launch.h): compile-time steps up to 4096,
// KM = 8192 for any larger step.
#include "vd_launch.h"

namespace vdl {

cudaError_t launch_sk_large_a(int dev, uint32_t k, bool me, bool bd, const vdk::PassArgs& a, const CUtensorMap& tm,
                            dim3 g, dim3 b, size_t sm, cudaStream_t st) {
  switch (k) {
    case 512: return sk_k<512>(dev, me, bd, a, tm, g, b, sm, st);
    case 1024: return sk_k<1024>(dev, me, bd, a, tm, g, b, sm, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vdl
