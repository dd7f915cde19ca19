// jump_pass_sk instantiations for k <= 16 (see vd_launch.h).
#include "vd_launch.h"

namespace vdl {

cudaError_t launch_sk_small_a(int dev, uint32_t k, bool me, bool bd, bool five, bool hash, const vdk::PassArgs& a,
                            const CUtensorMap& tm, dim3 g, dim3 b, size_t sm, cudaStream_t st) {
  switch (k) {
    case 1:
      if (hash && !me)  // the frame's last pass also sums the label checksum
        return bd ? sk_one<1, false, true, true>(dev, a, tm, g, b, sm, st) : sk_one<1, false, false, true>(dev, a, tm, g, b, sm, st);
      return sk_k<1>(dev, me, bd, a, tm, g, b, sm, st);
    case 2: return sk_k<2>(dev, me, bd, a, tm, g, b, sm, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vdl
