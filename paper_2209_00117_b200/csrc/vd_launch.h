// vd_launch.h -- internal: the jump-pass launchers, one translation unit per kernel family
// (vd_launch_*.cu), so that nvcc compiles the ~170 kernel instantiations in parallel.
// Each returns the launch's cudaError_t (attribute setting or launch configuration); the
// caller (vd.cu launch_pass) turns errors into vd_status.  Not part of the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>

#ifndef VD_TEMPLATE_KERNELS_ONLY
#define VD_TEMPLATE_KERNELS_ONLY  // launcher TUs instantiate only the pass templates
#endif
#include "vd_kernels.cuh"

namespace vdl {

// jump_pass_fast: k in {1, 2} (KM = k) or any power of two >= 4 (KM = 4); windowed (rel),
// EMPTY-carrying (me), banded (bd), metric / Von Neumann variants.
cudaError_t launch_fast(int dev, uint32_t k, bool me, bool bd, bool rel, int metric, bool vn,
                        const vdk::PassArgs& a, dim3 grid, dim3 blk, size_t smem, cudaStream_t st);

// jump_pass_sk (Euclidean Moore, shared terms): power-of-two k.  five = dJFA's 5-CTA/SM
// instantiation (4 <= k <= 64, no EMPTY); hash = the checksum-summing k = 1 pass.
// Split by k range over six TUs (vd_launch_sk_{small,mid,large}_{a,b}.cu).
cudaError_t launch_sk_small_a(int dev, uint32_t k, bool me, bool bd, bool five, bool hash, const vdk::PassArgs& a,
                              const CUtensorMap& tm, dim3 grid, dim3 blk, size_t smem, cudaStream_t st);
cudaError_t launch_sk_small_b(int dev, uint32_t k, bool me, bool bd, bool five, bool hash, const vdk::PassArgs& a,
                              const CUtensorMap& tm, dim3 grid, dim3 blk, size_t smem, cudaStream_t st);
cudaError_t launch_sk_mid_a(int dev, uint32_t k, bool me, bool bd, bool five, const vdk::PassArgs& a,
                            const CUtensorMap& tm, dim3 grid, dim3 blk, size_t smem, cudaStream_t st);
cudaError_t launch_sk_mid_b(int dev, uint32_t k, bool me, bool bd, bool five, const vdk::PassArgs& a,
                            const CUtensorMap& tm, dim3 grid, dim3 blk, size_t smem, cudaStream_t st);
cudaError_t launch_sk_large_a(int dev, uint32_t k, bool me, bool bd, const vdk::PassArgs& a, const CUtensorMap& tm,
                              dim3 grid, dim3 blk, size_t smem, cudaStream_t st);
cudaError_t launch_sk_large_b(int dev, uint32_t k, bool me, bool bd, const vdk::PassArgs& a, const CUtensorMap& tm,
                              dim3 grid, dim3 blk, size_t smem, cudaStream_t st);
inline cudaError_t launch_sk(int dev, uint32_t k, bool me, bool bd, bool five, bool hash, const vdk::PassArgs& a,
                             const CUtensorMap& tm, dim3 grid, dim3 blk, size_t smem, cudaStream_t st) {
  if (k <= 2) return launch_sk_small_a(dev, k, me, bd, five, hash, a, tm, grid, blk, smem, st);
  if (k <= 16) return launch_sk_small_b(dev, k, me, bd, five, hash, a, tm, grid, blk, smem, st);
  if (k <= 64) return launch_sk_mid_a(dev, k, me, bd, five, a, tm, grid, blk, smem, st);
  if (k <= 256) return launch_sk_mid_b(dev, k, me, bd, five, a, tm, grid, blk, smem, st);
  if (k <= 1024) return launch_sk_large_a(dev, k, me, bd, a, tm, grid, blk, smem, st);
  return launch_sk_large_b(dev, k, me, bd, a, tm, grid, blk, smem, st);
}

// jump_pass_sk_remap (first dJFA pass with the remap fused in): 4 <= k <= 128.
cudaError_t launch_sk_remap(int dev, uint32_t k, const vdk::PassArgs& a, const CUtensorMap& tm, dim3 grid, dim3 blk,
                            size_t smem, cudaStream_t st);

// jump_pass_wsk (wide exact pass for N <= 65536, EMPTY allowed): power-of-two 256 <= k <= N / 4.
cudaError_t launch_wsk(int dev, bool me, bool bd, const vdk::PassArgs& a, const CUtensorMap& tm, dim3 grid, dim3 blk,
                       size_t smem, cudaStream_t st);

// jump_pass_wide (generic 64-bit pass: any k, any N <= 65536, EMPTY allowed).
cudaError_t launch_wide(uint32_t k, int metric, bool vn, const vdk::PassArgs& a, dim3 grid, dim3 blk,
                        cudaStream_t st);

// Set a kernel's dynamic shared-memory opt-in once per (instantiation, device): a per-
// instantiation device bitmask (a concurrent first use on two threads sets the same value twice,
// which is harmless).
template <typename F>
inline cudaError_t opt_in_smem(std::atomic<uint64_t>& opted, int dev, F* fn, int bytes) {
  const uint64_t bit = 1ull << (dev & 63);
  if (opted.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  opted.fetch_or(bit, std::memory_order_release);
  return cudaSuccess;
}

}  // namespace vdl

namespace vdl {

// One jump_pass_sk instantiation, with its shared-memory opt-in.
template <int KM, bool ME, bool BD, bool HASH = false, int MINB = VD_MIN_BLOCKS>
cudaError_t sk_one(int dev, const vdk::PassArgs& a, const CUtensorMap& tm, dim3 grid, dim3 blk, size_t sm,
                   cudaStream_t st) {
  static std::atomic<uint64_t> opted{0};
  const cudaError_t e = opt_in_smem(opted, dev, vdk::jump_pass_sk<KM, ME, BD, HASH, MINB>,
                                    MINB == 5 ? vdk::kSmemBudget5 : vdk::kSmemBudget);
  if (e != cudaSuccess) return e;
  vdk::jump_pass_sk<KM, ME, BD, HASH, MINB><<<grid, blk, sm, st>>>(a, tm);
  return cudaSuccess;
}
template <int KM>
cudaError_t sk_k(int dev, bool me, bool bd, const vdk::PassArgs& a, const CUtensorMap& tm, dim3 g, dim3 b, size_t sm,
                 cudaStream_t st) {
  if (me) return bd ? sk_one<KM, true, true>(dev, a, tm, g, b, sm, st) : sk_one<KM, true, false>(dev, a, tm, g, b, sm, st);
  return bd ? sk_one<KM, false, true>(dev, a, tm, g, b, sm, st) : sk_one<KM, false, false>(dev, a, tm, g, b, sm, st);
}
// dJFA's stride passes at five CTAs per SM (no EMPTY)
template <int KM>
cudaError_t sk_k5(int dev, bool me, bool bd, bool five, const vdk::PassArgs& a, const CUtensorMap& tm, dim3 g, dim3 b,
                  size_t sm, cudaStream_t st) {
  if (five) return bd ? sk_one<KM, false, true, false, 5>(dev, a, tm, g, b, sm, st)
                      : sk_one<KM, false, false, false, 5>(dev, a, tm, g, b, sm, st);
  return sk_k<KM>(dev, me, bd, a, tm, g, b, sm, st);
}

}  // namespace vdl
