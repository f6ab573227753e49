// Microbenchmark: ex2 throughput with ONE warp per SM sub-partition (the FMHA softmax situation):
// f32 MUFU.EX2 vs packed bf16x2 / f16x2, independent chains of 16 registers per thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void k(unsigned* out, int iters, long long* cyc) {
  unsigned a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x + i);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (V == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(a[i]));
      if (V == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
      if (V == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
    }
  }
  const long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 0x1234567u) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned* d;
  long long* cyc;
  cudaMalloc(&d, 64);
  cudaMalloc(&cyc, 8 * 1024);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"ex2 f32", "ex2 bf16x2", "ex2 f16x2"};
  const int per[] = {1, 2, 2};
  for (int v = 0; v < 3; ++v)
    for (int threads : {128, 256, 512}) {
      const int iters = 4096;
      auto launch = [&]() {
        if (v == 0) k<0><<<sms, threads>>>(d, iters, cyc);
        if (v == 1) k<1><<<sms, threads>>>(d, iters, cyc);
        if (v == 2) k<2><<<sms, threads>>>(d, iters, cyc);
      };
      launch();
      launch();
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double instr = double(iters) * 16 * threads;  // thread-instructions per SM
      printf("%-11s warps/SMSP %d: %.2f results/clk/SM (%.2f instr-lanes/clk/SM)\n", names[v], threads / 128,
             instr * per[v] / h, instr / h);
    }
  return 0;
}
