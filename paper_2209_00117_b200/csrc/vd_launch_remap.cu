// jump_pass_sk_remap instantiations (see vd_launch.h).
#include "vd_launch.h"

namespace vdl {

template <int KM>
static cudaError_t remap_one(int dev, const vdk::PassArgs& a, const CUtensorMap& tm, dim3 g, dim3 b, size_t sm,
                             cudaStream_t st) {
  static std::atomic<uint64_t> opted{0};
  const cudaError_t e = opt_in_smem(opted, dev, vdk::jump_pass_sk_remap<KM>, vdk::kSmemBudget5);
  if (e != cudaSuccess) return e;
  vdk::jump_pass_sk_remap<KM><<<g, b, sm, st>>>(a, tm);
  return cudaSuccess;
}

cudaError_t launch_sk_remap(int dev, uint32_t k, const vdk::PassArgs& a, const CUtensorMap& tm, dim3 g, dim3 b,
                            size_t sm, cudaStream_t st) {
  switch (k) {
    case 4: return remap_one<4>(dev, a, tm, g, b, sm, st);
    case 8: return remap_one<8>(dev, a, tm, g, b, sm, st);
    case 16: return remap_one<16>(dev, a, tm, g, b, sm, st);
    case 32: return remap_one<32>(dev, a, tm, g, b, sm, st);
    case 64: return remap_one<64>(dev, a, tm, g, b, sm, st);
    default: return remap_one<128>(dev, a, tm, g, b, sm, st);
  }
}

}  // namespace vdl
