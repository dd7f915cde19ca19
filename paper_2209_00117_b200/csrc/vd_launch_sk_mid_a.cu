// jump_pass_sk instantiations for 32 <= k <= 256 (see vd_launch.h).
#include "vd_launch.h"

namespace vdl {

cudaError_t launch_sk_mid_a(int dev, uint32_t k, bool me, bool bd, bool five, const vdk::PassArgs& a,
                          const CUtensorMap& tm, dim3 g, dim3 b, size_t sm, cudaStream_t st) {
  switch (k) {
    case 32: return sk_k5<32>(dev, me, bd, five, a, tm, g, b, sm, st);
    case 64: return sk_k5<64>(dev, me, bd, five, a, tm, g, b, sm, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vdl
