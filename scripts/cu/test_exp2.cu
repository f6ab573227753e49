// dev check of exp2_poly2 (df_ptx.cuh) on special inputs
#include <cstdio>
#include "../../paper_2601_20499_b200/csrc/df_ptx.cuh"
using namespace dfb;
__global__ void k(const float* x, float* y, int n) {
  int i = threadIdx.x * 2;
  if (i + 1 < n + 1) {
    float2 r = exp2_poly2(make_float2(x[i], x[i + 1]));
    y[i] = r.x; y[i + 1] = r.y;
  }
}
int main() {
  const int n = 16;
  float hx[n] = {-INFINITY, -1000.f, -200.f, -127.f, -126.5f, -126.f, -100.f, -10.25f, -1.f, -0.5f, 0.f, 0.5f, 1.f, 7.9f, 8.f, -3.3f};
  float *dx, *dy, hy[n];
  cudaMalloc(&dx, sizeof(hx)); cudaMalloc(&dy, sizeof(hx));
  cudaMemcpy(dx, hx, sizeof(hx), cudaMemcpyHostToDevice);
  k<<<1, n / 2>>>(dx, dy, n);
  cudaMemcpy(hy, dy, sizeof(hy), cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i) printf("x=%g poly=%g exact=%g\n", hx[i], hy[i], exp2f(hx[i]));
  return 0;
}
