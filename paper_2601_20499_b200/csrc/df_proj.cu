// df_proj.cu -- the two projection GEMMs around the attention launch of a
// Dummy Forcing layer, on the 5th-gen tensor cores (sm_100a), with the data
// movement the reference does afterwards fused into the epilogue.
//
//   df_qkv_project  [q|k|v] = x @ [W_q|W_k|W_v]   (scenario.py:102-114)
//                   epilogue: Q -> (head, row) layout read by df_attn_fwd,
//                   K/V -> each head's pending ring slot (engine.py:423-426
//                   FrameBlock + the append copy of kv_cache.py:177-185).
//   df_out_project  x += merge(o) @ W_o            (scenario.py:116-120 and
//                   the residual of engine.py:443); A is read per head
//                   straight from the FMHA output, so the head merge
//                   (transpose) costs nothing.
//
// Persistent kernel, one CTA per SM, 320 threads:
//   warp 0      TMA producer: [128 x 64] A box + [BN x 64] B box per stage
//               (SWIZZLE_128B), kStages-deep ring
//   warp 1      TMEM allocator + tcgen05.mma issuer (elected lane),
//               accumulators double-buffered in TMEM (2 x BN fp32 columns)
//   warps 2-9   epilogue (two per TMEM lane quadrant, half the columns
//               each): tcgen05.ld 32 columns, staged through shared memory,
//               row-contiguous fused loads/stores, overlapping the next
//               tile's main loop
// Tiles are walked m-fastest so consecutive CTAs share the same W tile in L2.
// df_proj_pair_kernel is the CTA-pair (cta_group::2, M = 256) form of the same
// GEMM; pick_tiling chooses the variant and N per shape by whole-wave cost.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "df_b200.h"
#include "df_internal.h"
#include "df_ptx.cuh"

namespace dfb {
namespace {

constexpr int kPBM = 128;
constexpr int kPBK = 64;  // one 128-byte swizzle atom of bf16 per stage
constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant, each half of the tile's columns
constexpr int kPThreads = 64 + 32 * kEpiWarps;

enum { kEpiQKV = 0, kEpiOut = 1 };

// Per epilogue warp, one 32-column chunk of its 32 rows is staged in shared
// memory (rows padded by 16 B: conflict-free row-per-lane writes), then
// written out row-contiguously (4-8 rows x 64-128 B per warp instruction).
template <int kEpi>
struct StageRow {
  static constexpr int kBytes = kEpi == kEpiQKV ? 64 + 16 : 128 + 16;  // bf16 / fp32 chunk row
};

template <int BN, int kEpi>
struct ProjCfg {
  static constexpr int kABytes = kPBM * kPBK * 2;
  static constexpr int kBBytes = BN * kPBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStgWarp = 32 * StageRow<kEpi>::kBytes;
  static constexpr int kBudget = 232448 - 1024 - 256;
  static constexpr int kFit = (kBudget - kEpiWarps * kStgWarp) / kStageBytes;
  static constexpr int kStages = kFit > 6 ? 6 : kFit;
  static constexpr int kStgOff = kStages * kStageBytes;
  static constexpr int kBarOff = kStgOff + kEpiWarps * kStgWarp;
  static constexpr int kSmem = kBarOff + (2 * kStages + 4) * 8 + 16 + 1024;
  static constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;  // power of two
  static_assert(kStages >= 3, "pipeline too shallow");
  static_assert(kSmem <= 232448, "shared memory");
};

struct ProjParams {
  CUtensorMap amap;
  CUtensorMap bmap;
  int32_t m, n, kblocks;
  int32_t m_tiles, tiles;
  int32_t a_cols;        // A column extent before the next head chunk starts
  int32_t a_chunk_rows;  // row offset between consecutive A column chunks
  int32_t hw, head_dim;
  int32_t qkv_cols;  // num_heads * head_dim (QKV epilogue)
  int32_t out_ld;    // x row stride (out-projection epilogue)
  __nv_bfloat16* q_out;
  __nv_bfloat16* k_dst[DF_MAX_HEADS];
  __nv_bfloat16* v_dst[DF_MAX_HEADS];
  int64_t kv_ld;
  float* x;
  __nv_bfloat16* x_bf16;
};

// One 32-column chunk (accumulator registers r, thread = row `lane` of the
// warp's 32 rows starting at tile row `row0`).
// The residual rows of one out-projection chunk (x[row0 .. row0+31][n0 .. n0+31], fp32), four rows
// x 128 B per warp instruction.  Issued one chunk ahead of its use -- the first chunk of a tile
// before the accumulator is ready -- so the epilogue does not stall on HBM latency per chunk.
__device__ __forceinline__ void load_residual(const ProjParams& p, int lane, int row0, int n0, float4 (&xv)[8]) {
#if defined(DF_DIAG_OPROJ_NOLOAD) || defined(DF_DIAG_OPROJ_NOEPI)
  return;  // dev: epilogue cost diagnostics (wrong results)
#endif
  if (n0 >= p.n) return;
  const int piece = lane & 7;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int row = row0 + 4 * k + (lane >> 3);
    if (row < p.m) xv[k] = *reinterpret_cast<const float4*>(p.x + static_cast<int64_t>(row) * p.out_ld + n0 + 4 * piece);
  }
}

template <int kEpi>
__device__ __forceinline__ void epilogue_chunk(const ProjParams& p, uint8_t* stg, int lane, int row0, int n0,
                                               const uint32_t (&r)[32], const float4 (&xv)[8]) {
  constexpr int kRow = StageRow<kEpi>::kBytes;
  if constexpr (kEpi == kEpiQKV) {
    uint4* srow = reinterpret_cast<uint4*>(stg + lane * kRow);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 v;
      v.x = pack_bf16x2(__uint_as_float(r[8 * i + 0]), __uint_as_float(r[8 * i + 1]));
      v.y = pack_bf16x2(__uint_as_float(r[8 * i + 2]), __uint_as_float(r[8 * i + 3]));
      v.z = pack_bf16x2(__uint_as_float(r[8 * i + 4]), __uint_as_float(r[8 * i + 5]));
      v.w = pack_bf16x2(__uint_as_float(r[8 * i + 6]), __uint_as_float(r[8 * i + 7]));
      srow[i] = v;
    }
    __syncwarp();
    if (n0 < p.n) {
      const int which = n0 / p.qkv_cols;  // 0 q, 1 k, 2 v (warp-uniform)
      const int rem = n0 - which * p.qkv_cols;
      const int h = rem / p.head_dim;
      const int col = rem - h * p.head_dim;
      __nv_bfloat16* base;
      int64_t ld;
      if (which == 0) {
        base = p.q_out + static_cast<int64_t>(h) * p.hw * p.head_dim + col;
        ld = p.head_dim;
      } else {
        base = (which == 1 ? p.k_dst[h] : p.v_dst[h]) + col;
        ld = p.kv_ld;
      }
      const int piece = lane & 3;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int rl = 8 * k + (lane >> 2);
        const int row = row0 + rl;
        if (row < p.m)
          *reinterpret_cast<uint4*>(base + row * ld + piece * 8) =
              *reinterpret_cast<const uint4*>(stg + rl * kRow + piece * 16);
      }
    }
    __syncwarp();
  } else {
    float4* srow = reinterpret_cast<float4*>(stg + lane * kRow);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      srow[i] = make_float4(__uint_as_float(r[4 * i + 0]), __uint_as_float(r[4 * i + 1]),
                            __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
    __syncwarp();
#ifdef DF_DIAG_OPROJ_NOEPI
    if (false) {
#else
    if (n0 < p.n) {
#endif
      const int piece = lane & 7;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int rl = 4 * k + (lane >> 3);
        const int row = row0 + rl;
        if (row < p.m) {
          const float4 a = *reinterpret_cast<const float4*>(stg + rl * kRow + piece * 16);
          float4 v = xv[k];
          v.x += a.x;
          v.y += a.y;
          v.z += a.z;
          v.w += a.w;
          const int64_t off = static_cast<int64_t>(row) * p.out_ld + n0 + 4 * piece;
          *reinterpret_cast<float4*>(p.x + off) = v;
          if (p.x_bf16) {
            uint2 b;
            b.x = pack_bf16x2(v.x, v.y);
            b.y = pack_bf16x2(v.z, v.w);
            *reinterpret_cast<uint2*>(p.x_bf16 + off) = b;
          }
        }
      }
    }
    __syncwarp();
  }
}

// Drain one accumulator tile (this warp's kPer 32-column chunks of its 32 rows).  xv[c] holds the
// residual of chunk c on entry; as each chunk is consumed, its slot is refilled with chunk c of the
// next tile (next_row0 / next_n0, when has_next), which then has a whole mainloop to arrive.
template <int BN, int kEpi>
__device__ __forceinline__ void drain_tile(const ProjParams& p, uint8_t* stg, int lane, uint32_t taddr, int row0,
                                           int n0, float4 (&xv)[BN / 64][8], bool has_next, int next_row0,
                                           int next_n0) {
  constexpr int kPer = BN / 64;
#pragma unroll
  for (int c = 0; c < kPer; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    tmem_wait_ld();
    epilogue_chunk<kEpi>(p, stg, lane, row0, n0 + c * 32, r, xv[c]);
    if constexpr (kEpi == kEpiOut)
      if (has_next) load_residual(p, lane, next_row0, next_n0 + c * 32, xv[c]);
  }
}

template <int BN, int kEpi>
__global__ void __launch_bounds__(kPThreads, 1) df_proj_kernel(const __grid_constant__ ProjParams p) {
  using C = ProjCfg<BN, kEpi>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* empty = full + C::kStages;
  uint64_t* acc_full = empty + C::kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, kEpiWarps);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&p.amap);
      prefetch_tmap(&p.bmap);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const int mb = tile % p.m_tiles;
        const int nb = tile / p.m_tiles;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          mbar_expect_tx(full + stage, C::kStageBytes);
          const int kk = kb * kPBK;
          const int chunk = kk / p.a_cols;
          uint8_t* sa = smem + stage * C::kStageBytes;
          tma_load_2d(sa, &p.amap, full + stage, kk - chunk * p.a_cols, mb * kPBM + chunk * p.a_chunk_rows);
          tma_load_2d(sa + C::kABytes, &p.bmap, full + stage, kk, nb * BN);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Warp-wide loop, elected lane issues; descriptors are a precomputed base
    // plus compile-time offsets (as the FMHA issuer).
    {
      constexpr uint32_t idesc = idesc_bf16(kPBM, BN, false);
      const uint64_t d0 = sdesc_sw128(smem_u32(smem), 16, 1024);
      constexpr uint64_t kStageDesc = C::kStageBytes >> 4, kBDesc = C::kABytes >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        mbar_wait(acc_empty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint64_t da = d0 + stage * kStageDesc;
#pragma unroll
          for (int k = 0; k < kPBK / 16; ++k)
            umma_ss_elect(d, da + ((k * 32) >> 4), da + kBDesc + ((k * 32) >> 4), idesc, (kb | k) != 0);
          umma_commit_elect(empty + stage);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_elect(acc_full + acc);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;  // TMEM lanes 32*quad .. 32*quad+31
    constexpr int kPer = BN / 64;  // 32-column chunks per epilogue warp
    const int c0 = ((warp - 2) >> 2) * kPer;
    uint8_t* stg = smem + C::kStgOff + (warp - 2) * C::kStgWarp;
    int acc = 0;
    uint32_t acc_phase = 0;
    float4 xv[kPer][8];
    auto tile_row0 = [&](int t) { return (t % p.m_tiles) * kPBM + quad * 32; };
    auto tile_n0 = [&](int t) { return (t / p.m_tiles) * BN + c0 * 32; };
    if constexpr (kEpi == kEpiOut)
      if (static_cast<int>(blockIdx.x) < p.tiles)
#pragma unroll
        for (int c = 0; c < kPer; ++c) load_residual(p, lane, tile_row0(blockIdx.x), tile_n0(blockIdx.x) + c * 32, xv[c]);
    for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
      const int next = tile + static_cast<int>(gridDim.x);
      mbar_wait(acc_full + acc, acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem + acc * BN + (static_cast<uint32_t>(quad * 32) << 16) + c0 * 32;
      drain_tile<BN, kEpi>(p, stg, lane, taddr, tile_row0(tile), tile_n0(tile), xv, next < p.tiles, tile_row0(next),
                           tile_n0(next));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + acc);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2, M = 256 per MMA).  A cluster of two CTAs on
// one TPC computes a 256 x BN tile: each CTA stages its 128 rows of A and half
// of the BN rows of B, so per SM the B reads and B TMA writes halve -- the
// 1-CTA kernel moves ~192 B/clk through shared memory per 128-cycle UMMA
// against a 128 B/clk port, this one ~128.  The leader's elected lane issues
// for both SMs; each CTA's epilogue warps drain its own 128 accumulator rows
// and release the accumulator on the leader's barrier.
template <int BN, int kEpi>
struct PairCfg {
  static constexpr int kABytes = kPBM * kPBK * 2;
  static constexpr int kBBytes = (BN / 2) * kPBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStgWarp = 32 * StageRow<kEpi>::kBytes;
  static constexpr int kBudget = 232448 - 1024 - 256;
  static constexpr int kFit = (kBudget - kEpiWarps * kStgWarp) / kStageBytes;
  static constexpr int kStages = kFit > 8 ? 8 : kFit;
  static constexpr int kStgOff = kStages * kStageBytes;
  static constexpr int kBarOff = kStgOff + kEpiWarps * kStgWarp;
  static constexpr int kSmem = kBarOff + (2 * kStages + 4) * 8 + 16 + 1024;
  static constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;
  static_assert(kStages >= 3, "pipeline too shallow");
  static_assert(kSmem <= 232448, "shared memory");
};

template <int BN, int kEpi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPThreads, 1)
    df_proj_pair_kernel(const __grid_constant__ ProjParams p) {
  using C = PairCfg<BN, kEpi>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kBarOff);  // leader: A + B of both CTAs landed
  uint64_t* empty = full + C::kStages;                               // both: the stage's MMAs are done
  uint64_t* acc_full = empty + C::kStages;                           // [2] both
  uint64_t* acc_empty = acc_full + 2;                                // [2] leader: both epilogues drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const int cid = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, 2 * kEpiWarps);  // one arrive per epilogue warp of either CTA
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, C::kTmemCols);
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      prefetch_tmap(&p.amap);
      prefetch_tmap(&p.bmap);
      const uint64_t pol = policy_evict_last();  // W and x tiles are re-read by other clusters
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < p.tiles; tile += nclusters) {
        const int mb = tile % p.m_tiles;
        const int nb = tile / p.m_tiles;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          if (crank == 0) mbar_expect_tx(full + stage, 2 * C::kStageBytes);
          const uint32_t lbar = mapa_shared(smem_u32(full + stage), 0);
          const int kk = kb * kPBK;
          const int chunk = kk / p.a_cols;
          uint8_t* sa = smem + stage * C::kStageBytes;
          tma_load_2d_pair(sa, &p.amap, lbar, kk - chunk * p.a_cols,
                           mb * 2 * kPBM + static_cast<int>(crank) * kPBM + chunk * p.a_chunk_rows, pol);
          tma_load_2d_pair(sa + C::kABytes, &p.bmap, lbar, kk, nb * BN + static_cast<int>(crank) * (BN / 2), pol);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader, warp-wide, elected lane)
    if (crank == 0) {
      constexpr uint32_t idesc = idesc_bf16(2 * kPBM, BN, false);
      const uint64_t d0 = sdesc_sw128(smem_u32(smem), 16, 1024);
      constexpr uint64_t kStageDesc = C::kStageBytes >> 4, kBDesc = C::kABytes >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = cid; tile < p.tiles; tile += nclusters) {
        mbar_wait_cluster(acc_empty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait_cluster(full + stage, phase);
          tc_fence_after();
          const uint64_t da = d0 + stage * kStageDesc;
#pragma unroll
          for (int k = 0; k < kPBK / 16; ++k)
            umma_ss_pair_elect(d, da + ((k * 32) >> 4), da + kBDesc + ((k * 32) >> 4), idesc, (kb | k) != 0);
          umma_commit_pair_elect(empty + stage);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair_elect(acc_full + acc);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs, own 128 rows)
    const int quad = warp & 3;
    constexpr int kPer = BN / 64;
    const int c0 = ((warp - 2) >> 2) * kPer;
    uint8_t* stg = smem + C::kStgOff + (warp - 2) * C::kStgWarp;
    const uint32_t leader_acc_empty = mapa_shared(smem_u32(acc_empty), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    float4 xv[kPer][8];
    auto tile_row0 = [&](int t) { return (t % p.m_tiles) * 2 * kPBM + static_cast<int>(crank) * kPBM + quad * 32; };
    auto tile_n0 = [&](int t) { return (t / p.m_tiles) * BN + c0 * 32; };
    if constexpr (kEpi == kEpiOut)
      if (cid < p.tiles)
#pragma unroll
        for (int c = 0; c < kPer; ++c) load_residual(p, lane, tile_row0(cid), tile_n0(cid) + c * 32, xv[c]);
    for (int tile = cid; tile < p.tiles; tile += nclusters) {
      const int next = tile + nclusters;
      mbar_wait_cluster(acc_full + acc, acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem + acc * BN + (static_cast<uint32_t>(quad * 32) << 16) + c0 * 32;
      drain_tile<BN, kEpi>(p, stg, lane, taddr, tile_row0(tile), tile_n0(tile), xv, next < p.tiles, tile_row0(next),
                           tile_n0(next));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_acc_empty + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's smem and TMEM stay live until the leader's MMAs are done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, C::kTmemCols);
  }
}

template <int BN, int kEpi>
int launch_proj_pair(const ProjParams& p, int grid, cudaStream_t stream) {
  auto kern = df_proj_pair_kernel<BN, kEpi>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<BN, kEpi>::kSmem);
    if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(df_proj_pair_kernel)", e);
    configured = true;
  }
  kern<<<grid, kPThreads, PairCfg<BN, kEpi>::kSmem, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("df_proj_pair_kernel launch", e);
  return DF_OK;
}

template <int BN, int kEpi>
int launch_proj(const ProjParams& p, int grid, cudaStream_t stream) {
  auto kern = df_proj_kernel<BN, kEpi>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ProjCfg<BN, kEpi>::kSmem);
    if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(df_proj_kernel)", e);
    configured = true;
  }
  kern<<<grid, kPThreads, ProjCfg<BN, kEpi>::kSmem, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("df_proj_kernel launch", e);
  return DF_OK;
}

template <int kEpi>
int launch_bn(int bn, bool pair, const ProjParams& p, int grid, cudaStream_t s) {
  if (pair) {
    if (bn == 256) return launch_proj_pair<256, kEpi>(p, grid, s);
    if (bn == 192) return launch_proj_pair<192, kEpi>(p, grid, s);
    return launch_proj_pair<128, kEpi>(p, grid, s);
  }
  if (bn == 256) return launch_proj<256, kEpi>(p, grid, s);
  if (bn == 192) return launch_proj<192, kEpi>(p, grid, s);
  return launch_proj<128, kEpi>(p, grid, s);
}

// CTA-pair GEMM unless DF_PROJ_PAIR=0 (dev A/B).
bool use_pair_gemm() {
  static const bool on = [] {
    const char* env = std::getenv("DF_PROJ_PAIR");
    return !(env && env[0] == '0');
  }();
  return on;
}

// Tiling of an (m x n) projection: tile width, 1-CTA or pair, tiles and grid.
struct Tiling {
  int bn;
  bool pair;
  int32_t m_tiles, tiles;
  int grid;
};

Tiling pick_tiling(int64_t m, int64_t n) {
  // Smallest modelled time over whole waves of the persistent grid: cost = waves x N / eff, with eff the
  // measured per-SM rate of a 128 x N slice (1-CTA: shared-memory bound below N = 256, 0.66 at 128,
  // 0.86 at 192; the pair halves B traffic: 1.07 at N = 256 against the 1-CTA N = 256 rate).  Wan:
  // QKV takes the pair at N = 256 (342 pair tiles), the out-projection the 1-CTA kernel at N = 192
  // (296 tiles = 2 waves; the pair's 114 tiles waste half a wave).
  int forced = 0;
  if (const char* env = std::getenv("DF_PROJ_BN")) {
    const int v = std::atoi(env);
    forced = (v == 128 || v == 192 || v == 256) ? v : 0;
  }
  const int64_t sms = sm_count_cached();
  Tiling best{256, false, 0, 0, 0};
  double best_cost = 1e300;
  for (int pair = use_pair_gemm() ? 1 : 0; pair >= 0; --pair) {
    const int64_t rows = pair ? 2 * kPBM : kPBM;
    const int64_t units = pair ? sms / 2 : sms;
    for (int cand : {256, 192, 128}) {
      if (forced && cand != forced) continue;
      const double eff = pair ? (cand == 256 ? 1.07 : (cand == 192 ? 1.0 : 0.9))
                              : (cand == 256 ? 1.0 : (cand == 192 ? 0.86 : 0.66));
      const int64_t tiles = ((m + rows - 1) / rows) * ((n + cand - 1) / cand);
      const int64_t waves = (tiles + units - 1) / units;
      const double cost = double(waves) * cand / eff;
      if (cost < best_cost * 0.999) {
        best_cost = cost;
        best.bn = cand;
        best.pair = pair != 0;
        best.m_tiles = static_cast<int32_t>((m + rows - 1) / rows);
        best.tiles = static_cast<int32_t>(tiles);
        const int64_t u = tiles < units ? tiles : units;
        best.grid = static_cast<int>(pair ? 2 * u : u);
      }
    }
  }
  return best;
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

int check_dims(const char* fn, int32_t hw, int32_t heads, int32_t d) {
  if (hw < 1) return set_error(DF_E_SHAPE, "%s: hw %d < 1", fn, hw);
  if (heads < 1 || heads > DF_MAX_HEADS)
    return set_error(DF_E_SHAPE, "%s: num_heads %d outside [1, %d]", fn, heads, DF_MAX_HEADS);
  if (d != 64 && d != 128) return set_error(DF_E_SHAPE, "%s: head_dim %d not 64 or 128", fn, d);
  return DF_OK;
}

}  // namespace
}  // namespace dfb

using namespace dfb;

extern "C" int df_qkv_project(const df_qkv_args* a, void* stream) {
  if (!a || !a->x || !a->w_qkv || !a->q_out) return set_error(DF_E_ARG, "df_qkv_project: null argument");
  int rc = check_dims("df_qkv_project", a->hw, a->num_heads, a->head_dim);
  if (rc != DF_OK) return rc;
  if (a->in_dim < 8 || a->in_dim % 8) return set_error(DF_E_SHAPE, "df_qkv_project: in_dim %d not a multiple of 8", a->in_dim);
  if (a->kv_ld < a->head_dim || a->kv_ld % 8)
    return set_error(DF_E_SHAPE, "df_qkv_project: kv_ld %lld (head_dim %d)", (long long)a->kv_ld, a->head_dim);
  if (!aligned16(a->q_out)) return set_error(DF_E_ARG, "df_qkv_project: q_out not 16-byte aligned");
  ProjParams p;
  std::memset(&p, 0, sizeof(p));
  for (int h = 0; h < a->num_heads; ++h) {
    if (!a->k_dst[h] || !a->v_dst[h] || !aligned16(a->k_dst[h]) || !aligned16(a->v_dst[h]))
      return set_error(DF_E_ARG, "df_qkv_project: head %d K/V destination null or not 16-byte aligned", h);
    p.k_dst[h] = static_cast<__nv_bfloat16*>(a->k_dst[h]);
    p.v_dst[h] = static_cast<__nv_bfloat16*>(a->v_dst[h]);
  }
  const int32_t cols = a->num_heads * a->head_dim;
  p.m = a->hw;
  p.n = 3 * cols;
  p.kblocks = (a->in_dim + kPBK - 1) / kPBK;
  p.a_cols = p.kblocks * kPBK;  // one chunk: A is x itself
  p.a_chunk_rows = 0;
  p.hw = a->hw;
  p.head_dim = a->head_dim;
  p.qkv_cols = cols;
  p.q_out = static_cast<__nv_bfloat16*>(a->q_out);
  p.kv_ld = a->kv_ld;
  const Tiling t = pick_tiling(p.m, p.n);
  rc = encode_bf16_2d(&p.amap, a->x, a->hw, a->in_dim, a->in_dim, kPBM);
  if (rc != DF_OK) return rc;
  rc = encode_bf16_2d(&p.bmap, a->w_qkv, int64_t(p.n), a->in_dim, a->in_dim, t.pair ? t.bn / 2 : t.bn);
  if (rc != DF_OK) return rc;
  p.m_tiles = t.m_tiles;
  p.tiles = t.tiles;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return launch_bn<kEpiQKV>(t.bn, t.pair, p, t.grid, s);
}

extern "C" int df_out_project(const df_oproj_args* a, void* stream) {
  if (!a || !a->o || !a->w_o || !a->x) return set_error(DF_E_ARG, "df_out_project: null argument");
  int rc = check_dims("df_out_project", a->hw, a->num_heads, a->head_dim);
  if (rc != DF_OK) return rc;
  if (a->out_dim < 32 || a->out_dim % 32)
    return set_error(DF_E_SHAPE, "df_out_project: out_dim %d not a multiple of 32", a->out_dim);
  if (!aligned16(a->x) || (a->x_bf16 && !aligned16(a->x_bf16)))
    return set_error(DF_E_ARG, "df_out_project: x / x_bf16 not 16-byte aligned");
  ProjParams p;
  std::memset(&p, 0, sizeof(p));
  const int32_t kdim = a->num_heads * a->head_dim;
  p.m = a->hw;
  p.n = a->out_dim;
  p.kblocks = kdim / kPBK;
  p.a_cols = a->head_dim;  // K index h*d + c lives in row h*hw + m, column c of the FMHA output
  p.a_chunk_rows = a->hw;
  p.hw = a->hw;
  p.head_dim = a->head_dim;
  p.out_ld = a->out_dim;
  p.x = a->x;
  p.x_bf16 = static_cast<__nv_bfloat16*>(a->x_bf16);
  const Tiling t = pick_tiling(p.m, p.n);
  rc = encode_bf16_2d(&p.amap, a->o, int64_t(a->num_heads) * a->hw, a->head_dim, a->head_dim, kPBM);
  if (rc != DF_OK) return rc;
  rc = encode_bf16_2d(&p.bmap, a->w_o, a->out_dim, kdim, kdim, t.pair ? t.bn / 2 : t.bn);
  if (rc != DF_OK) return rc;
  p.m_tiles = t.m_tiles;
  p.tiles = t.tiles;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return launch_bn<kEpiOut>(t.bn, t.pair, p, t.grid, s);
}
