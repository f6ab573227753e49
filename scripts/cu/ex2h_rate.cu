// Microbenchmark: ex2.approx.f16x2 / ex2.approx.ftz.bf16x2 throughput vs ex2.approx.f32 on B200.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

template <int V>
__global__ void k(unsigned* out, const unsigned* src, int iters) {
  unsigned a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = src[i * 1024 + threadIdx.x];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (V == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(a[i]));
        if (V == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
        if (V == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
        if (V == 3) {  // f32 pair -> f16x2 pack
          unsigned t;
          asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(t) : "f"(__uint_as_float(a[i])), "f"(__uint_as_float(a[(i + 1) & 7])));
          a[i] ^= t;
        }
        if (V == 4) {  // f16x2 -> two f32 (unpack)
          float lo, hi;
          asm volatile("{.reg .f16 l, h;\n mov.b32 {l, h}, %2;\n cvt.f32.f16 %0, l;\n cvt.f32.f16 %1, h;}" : "=f"(lo), "=f"(hi) : "r"(a[i]));
          a[i] ^= __float_as_uint(lo) + __float_as_uint(hi);
        }
      }
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 0x1234567u) out[0] = s;
}

int main() {
  unsigned *d, *src;
  cudaMalloc(&d, 64);
  cudaMalloc(&src, 8 * 1024 * 4);
  cudaMemset(src, 0x3c, 8 * 1024 * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"ex2 f32", "ex2 f16x2", "ex2 bf16x2", "cvt f16x2.f32", "f16x2->2xf32"};
  const double per[] = {1, 2, 2, 1, 1};  // elements (or instr-lanes) per op
  for (int v = 0; v < 5; ++v) {
    const int iters = 2048, threads = 1024;
    auto launch = [&]() {
      switch (v) {
        case 0: k<0><<<sms, threads>>>(d, src, iters); break;
        case 1: k<1><<<sms, threads>>>(d, src, iters); break;
        case 2: k<2><<<sms, threads>>>(d, src, iters); break;
        case 3: k<3><<<sms, threads>>>(d, src, iters); break;
        case 4: k<4><<<sms, threads>>>(d, src, iters); break;
      }
    };
    launch();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(sms) * threads * iters * 32;
    printf("%-16s %.1f instr-lanes/SM/ns  -> %.1f results per SM per clk at 1.9 GHz (%s)\n", names[v],
           ops / sms / (ms * 1e6), ops * per[v] / sms / (ms * 1e6) / 1.9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
