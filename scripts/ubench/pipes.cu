// Throughput microbenchmark of the integer ops the jump pass uses (sm_100a).
// Each thread runs 8 independent dependency chains of one op; we report issued warp
// instructions per SM per cycle (4.0 = one per SMSP per cycle).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void kern(uint32_t* out, int iters, uint32_t s1, uint32_t s2) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7 + i;
  uint32_t b = s1, c = s2;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) a[i] = min(a[i], b + i);                                   // IMNMX (2-input)
        if (OP == 1) a[i] = __vimin3_u32(a[i], b, c + i);                      // VIMNMX3
        if (OP == 2) a[i] = __viaddmax_u32(a[i], b, c + i);                    // VIADDMNMX
        if (OP == 3) a[i] = a[i] * b + c;                                       // IMAD
        if (OP == 4) a[i] = __umulhi(a[i], b) + c;                              // IMAD.HI (+add)
        if (OP == 5) a[i] = (a[i] >> 16) + b;                                   // LEA.HI
        if (OP == 6) a[i] = __sad((int)a[i], (int)b, c);                        // VABSDIFF
        if (OP == 7) a[i] = a[i] ^ (b + i);                                     // LOP3
        if (OP == 8) a[i] = __vimin3_s32((int)a[i], (int)b, (int)(c + i));     // VIMNMX3 signed
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <int OP>
void run(const char* name, uint32_t* d, int sms) {
  const int iters = 2000, threads = 1024, blocks = sms * 2;
  kern<OP><<<blocks, threads>>>(d, 10, 3, 5);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<OP><<<blocks, threads>>>(d, iters, 3, 5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz (max)
  double warp_instr = (double)blocks * (threads / 32) * iters * 16 * 8;  // op instructions only
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-12s %.3f ms  %.2f warp-instr/SM/cycle (at max clock)\n", name, ms, warp_instr / sms / cycles);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* d; cudaMalloc(&d, sms * 2 * 1024 * 4);
  run<0>("IMNMX", d, sms); run<1>("VIMNMX3.U32", d, sms); run<8>("VIMNMX3.S32", d, sms);
  run<2>("VIADDMNMX", d, sms); run<3>("IMAD", d, sms); run<4>("IMAD.HI+add", d, sms);
  run<5>("LEA.HI", d, sms); run<6>("VABSDIFF", d, sms); run<7>("LOP3", d, sms);
  return 0;
}
