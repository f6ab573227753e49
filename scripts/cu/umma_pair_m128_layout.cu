// Dev probe: where does tcgen05.mma.cta_group::2 with M = 128 put its accumulator rows and columns in
// the two CTAs' TMEM?  A[r][0] = row id (per CTA, 128 rows staged), B[n][0] = column id (per CTA, N/2
// rows staged), K = 16; each CTA dumps TMEM lanes 0-127 x N columns.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2601_20499_b200/csrc -I../../include umma_pair_m128_layout.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include "df_ptx.cuh"
using namespace dfb;

constexpr int N = 64;

template <int M>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* out, int mode) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[(N / 2) * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t crank = cluster_ctarank();
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // K-major SWIZZLE_128B tiles: element (r, c) at r*128 + (((c*2)/16) ^ (r%8))*16 + (c*2)%16
  for (int i = t; i < 128 * 64; i += 128) {
    const int r = i / 64, c = i % 64;
    float v = 0.f;
    if (c == 0) v = mode == 0 ? float(crank * 128 + r + 1) : 1.f;
    *reinterpret_cast<__nv_bfloat16*>(sa + r * 128 + ((((c * 2) / 16) ^ (r % 8)) * 16) + (c * 2) % 16) = __float2bfloat16(v);
  }
  for (int i = t; i < (N / 2) * 64; i += 128) {
    const int r = i / 64, c = i % 64;
    float v = 0.f;
    if (c == 0) v = mode == 0 ? 1.f : float(crank * (N / 2) + r + 1);
    *reinterpret_cast<__nv_bfloat16*>(sb + r * 128 + ((((c * 2) / 16) ^ (r % 8)) * 16) + (c * 2) % 16) = __float2bfloat16(v);
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc_pair(&tslot, 128);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0 && crank == 0) {
    const uint64_t da = sdesc_sw128(smem_u32(sa), 16, 1024), db = sdesc_sw128(smem_u32(sb), 16, 1024);
    umma_ss_pair_elect(tmem, da, db, idesc_bf16(M, N, false), 0u);
    umma_commit_pair_elect(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) out[(crank * 128 + warp * 32 + lane) * N + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 128);
  }
}

template <int M>
void run(int mode) {
  float* d;
  cudaMalloc(&d, 2 * 128 * N * 4);
  cudaMemset(d, 0, 2 * 128 * N * 4);
  probe<M><<<2, 128>>>(d, mode);
  cudaError_t e = cudaDeviceSynchronize();
  static float h[2 * 128 * N];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("M=%d mode=%s err=%s\n", M, mode == 0 ? "rows (value = row id)" : "cols (value = column id)", cudaGetErrorString(e));
  for (int cr = 0; cr < 2; ++cr)
    for (int lane = 0; lane < 128; ++lane) {
      const float* row = h + (cr * 128 + lane) * N;
      bool any = false;
      for (int c = 0; c < N; ++c) any |= row[c] != 0.f;
      if (!any) continue;
      if (mode == 0) {
        printf("  cta %d lane %3d: col0 %.0f col%d %.0f\n", cr, lane, row[0], N - 1, row[N - 1]);
      } else if (lane % 32 == 0) {
        printf("  cta %d lane %3d: cols:", cr, lane);
        for (int c = 0; c < N; c += 8) printf(" [%d]=%.0f", c, row[c]);
        printf("\n");
      }
    }
  cudaFree(d);
}

int main() {
  run<256>(0);
  run<128>(0);
  run<128>(1);
  return 0;
}
