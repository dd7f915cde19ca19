// jump_pass_sk instantiations for k <= 16 (see vd_launch.h).
#include "vd_launch.h"

namespace vdl {

cudaError_t launch_sk_small_b(int dev, uint32_t k, bool me, bool bd, bool five, bool hash, const vdk::PassArgs& a,
                            const CUtensorMap& tm, dim3 g, dim3 b, size_t sm, cudaStream_t st) {
  switch (k) {
    case 4: return sk_k5<4>(dev, me, bd, five, a, tm, g, b, sm, st);
    case 8: return sk_k5<8>(dev, me, bd, five, a, tm, g, b, sm, st);
    case 16: return sk_k5<16>(dev, me, bd, five, a, tm, g, b, sm, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vdl
