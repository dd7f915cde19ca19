// jump_pass_wide instantiations (see vd_launch.h).
#include "vd_launch.h"

namespace vdl {

cudaError_t launch_wide(uint32_t k, int metric, bool vn, const vdk::PassArgs& a, dim3 g, dim3 b, cudaStream_t st) {
  const bool v4 = (k % 4) == 0;
  if (metric == 0) {
    if (vn) v4 ? vdk::jump_pass_wide<0, true, true><<<g, b, 0, st>>>(a) : vdk::jump_pass_wide<0, true, false><<<g, b, 0, st>>>(a);
    else v4 ? vdk::jump_pass_wide<0, false, true><<<g, b, 0, st>>>(a) : vdk::jump_pass_wide<0, false, false><<<g, b, 0, st>>>(a);
  } else {
    if (vn) v4 ? vdk::jump_pass_wide<1, true, true><<<g, b, 0, st>>>(a) : vdk::jump_pass_wide<1, true, false><<<g, b, 0, st>>>(a);
    else v4 ? vdk::jump_pass_wide<1, false, true><<<g, b, 0, st>>>(a) : vdk::jump_pass_wide<1, false, false><<<g, b, 0, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace vdl
