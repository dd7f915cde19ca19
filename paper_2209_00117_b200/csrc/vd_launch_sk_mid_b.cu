// jump_pass_sk instantiations for 32 <= k <= 256 (see vd_launch.h).
#include "vd_launch.h"

namespace vdl {

cudaError_t launch_sk_mid_b(int dev, uint32_t k, bool me, bool bd, bool five, const vdk::PassArgs& a,
                          const CUtensorMap& tm, dim3 g, dim3 b, size_t sm, cudaStream_t st) {
  switch (k) {
    case 128: return sk_k<128>(dev, me, bd, a, tm, g, b, sm, st);
    case 256: return sk_k<256>(dev, me, bd, a, tm, g, b, sm, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vdl
