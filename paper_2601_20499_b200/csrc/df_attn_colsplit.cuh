// df_attn_colsplit.cuh -- included by df_attn.cu (shares AttnParams / AttnCfg).
//
// Column-split softmax variant of df_attn_kernel (d = 128, no probe epilogue):
// the same work item, TMA producer, MMA issuer, TMEM map and issue order, but
// every query tile's softmax runs on 8 warps instead of 4 -- two warps per TMEM
// lane quadrant, one per half of the 128 keys of a kv tile.
//
// Why: the two query tiles' softmax phases alternate (tile 1's S lands while
// tile 0's P is being consumed), so with one warp per row only one softmax warp
// per SM sub-partition is busy at a time, and a lone warp reaches ~11 of the
// 16 ex2/clk/SM (scripts/cu/softmax_warps.cu: 1450 cycles per 128-key row
// against the 1024-cycle budget a 2 x 128-row tile pair leaves at the MMA
// bound).  Two warps per sub-partition on the same tile reach ~15/clk and halve
// each warp's exp count.
//
// Row statistics: each warp takes the max of its 64 columns, the pair swaps the
// halves through shared memory (named barrier per pair, double-buffered by kv
// tile parity), and both derive the identical row max, rescale decision and
// reference.  Each warp keeps its own half of the row sum; O rescales are split
// by columns and fenced by a pair barrier before either half of P is released
// (the first PV half writes all D columns of O).
//
// Warp map (18 warps, 576 threads, 112 registers): warp 0 TMA producer, warp 1
// TMEM allocator + MMA issuer, warps 2..17 softmax: sw = warp - 2, tile
// t = sw >> 3, key half h = (sw >> 2) & 1, TMEM lane quadrant q = warp & 3.
// P half h of tile t is TMEM columns [t*128 + 32h, +32): warp h=1's P overwrites
// S columns 32-63, which are warp h=0's scores -- h=0 has loaded them before it
// reaches the pair barrier that precedes any P store.

namespace dfb {

constexpr int kCsWarps = 18;
constexpr int kCsThreads = kCsWarps * 32;

template <int D>
struct CsCfg {
  using C = AttnCfg<D>;
  static constexpr int kXchOff = C::kBarOff + C::kNumBars * 8 + 32;  // [2 parity][2 tiles][128 rows][2 halves] f32
  static constexpr int kXchBytes = 2 * 2 * 128 * 2 * 4;
  static constexpr int kSmem = kXchOff + kXchBytes + 1024;
};

__device__ __forceinline__ void pair_bar_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

template <int D>
__global__ void __maxnreg__(96) df_attn_cs_kernel(const __grid_constant__ AttnParams p) {
  static_assert(D == 128, "column-split softmax is built for d = 128");
  using C = AttnCfg<D>;
  using X = CsCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + C::kStagesK;
  uint64_t* v_full = k_empty + C::kStagesK;
  uint64_t* v_empty = v_full + C::kStagesV;
  uint64_t* s_full = v_empty + C::kStagesV;  // [2]
  uint64_t* p_full = s_full + 2;             // [2 tiles][2 halves of P]
  uint64_t* o_full = p_full + 4;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);
  int32_t* last_flag = reinterpret_cast<int32_t*>(tmem_slot + 1);
  float* xch = reinterpret_cast<float*>(smem + X::kXchOff);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  int rank = 0;
  while (rank + 1 < p.n_heads && p.item_prefix[rank + 1] <= static_cast<int>(blockIdx.x)) ++rank;
  const int h = p.head_order[rank];
  const HeadParam hd = p.heads[h];
  const int local = blockIdx.x - p.item_prefix[rank];
  const int ns = hd.n_split;
  const int qp = local / ns;
  const int piece = local - qp * ns;
  const int n_kv_total = (hd.n_tok + kBN - 1) / kBN;
  const int kv_begin = (piece * n_kv_total) / ns;
  const int n_kv = ((piece + 1) * n_kv_total) / ns - kv_begin;
  const bool two = qp * 2 * kBM + kBM < p.hw;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::kStagesK; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < C::kStagesV; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(s_full + t, 1);
      mbar_init(p_full + 2 * t, 128);
      mbar_init(p_full + 2 * t + 1, 128);
      mbar_init(o_full + t, 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const void* kmap = &p.kvmap[DF_MAPS_PER_ARENA * hd.arena];
      const void* vmap = &p.kvmap[DF_MAPS_PER_ARENA * hd.arena + 1];
      prefetch_tmap(&p.qmap);
      prefetch_tmap(kmap);
      prefetch_tmap(vmap);
      const uint64_t keep = policy_evict_last();
      const int qrow0 = hd.q_head * p.hw + qp * 2 * kBM;
      const int nq = two ? 2 : 1;
      mbar_expect_tx(q_full, nq * C::kTileBytes);
      for (int t = 0; t < nq; ++t)
        for (int b = 0; b < C::kBoxes; ++b)
          tma_load_2d(smem + C::kQOff + t * C::kTileBytes + b * C::kBoxBytes, &p.qmap, q_full, b * 64,
                      qrow0 + t * kBM);
      for (int jj = 0; jj < n_kv; ++jj) {
        const int row = hd.base_row + (kv_begin + jj) * kBN;
        {
          const int s = jj % C::kStagesK;
          mbar_wait(k_empty + s, ((jj / C::kStagesK) & 1) ^ 1);
          mbar_expect_tx(k_full + s, C::kTileBytes);
          for (int b = 0; b < C::kBoxes; ++b)
            tma_load_2d_hint(smem + C::kKOff + s * C::kTileBytes + b * C::kBoxBytes, kmap, k_full + s, b * 64,
                             row, keep);
        }
        {
          const int s = jj % C::kStagesV;
          mbar_wait(v_empty + s, ((jj / C::kStagesV) & 1) ^ 1);
          mbar_expect_tx(v_full + s, C::kTileBytes);
          for (int b = 0; b < C::kBoxes; ++b)
            tma_load_2d_hint(smem + C::kVOff + s * C::kTileBytes + b * C::kBoxBytes, vmap, v_full + s, b * 64,
                             row, keep);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (as df_attn_kernel)
    constexpr uint32_t idesc_qk = idesc_bf16(kBM, kBN, false);
    constexpr uint32_t idesc_pv = idesc_bf16(kBM, D, true);
    const uint64_t dQ = sdesc_sw128(smem_u32(smem + C::kQOff), 16, 1024);
    const uint64_t dK = sdesc_sw128(smem_u32(smem + C::kKOff), 16, 1024);
    const uint64_t dV = sdesc_sw128(smem_u32(smem + C::kVOff), C::kBoxBytes, 1024);
    constexpr uint64_t kTileDesc = C::kTileBytes >> 4;
    const uint32_t tS0 = tmem, tS1 = tmem + 128;
    const uint32_t tO0 = tmem + C::kTmemO, tO1 = tmem + C::kTmemO + D;

    auto qk = [&](uint32_t d_tmem, int t, int ks) {
      const uint64_t qa = dQ + t * kTileDesc;
      const uint64_t kb = dK + ks * kTileDesc;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint64_t off = ((kk >> 2) * C::kBoxBytes + (kk & 3) * 32) >> 4;
        umma_ss_elect(d_tmem, qa + off, kb + off, idesc_qk, kk > 0);
      }
    };
    auto pv = [&](int t, int jj) {
      const int vs = jj % C::kStagesV;
      mbar_wait(p_full + 2 * t, jj & 1);
      tc_fence_after();
      if (t == 0) {
        mbar_wait(v_full + vs, (jj / C::kStagesV) & 1);
        tc_fence_after();
      }
      const uint64_t vb = dV + vs * kTileDesc;
      const uint32_t tP = t ? tS1 : tS0;
      const uint32_t tO = t ? tO1 : tO0;
#pragma unroll
      for (int kk = 0; kk < kBN / 16; ++kk) {
        if (kk == kBN / 32) {
          mbar_wait(p_full + 2 * t + 1, jj & 1);
          tc_fence_after();
        }
        umma_ts_elect(tO, tP + kk * 8, vb + ((kk * 2048) >> 4), idesc_pv, (jj > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit_elect(o_full + t);
      if (t == 1 || !two) umma_commit_elect(v_empty + vs);
    };

    mbar_wait(q_full, 0);
    tc_fence_after();
    for (int jj = 0; jj < n_kv; ++jj) {
      const int ks = jj % C::kStagesK;
      if (lane == 0) DF_STAMP(2, jj, 0);
      mbar_wait(k_full + ks, (jj / C::kStagesK) & 1);
      tc_fence_after();
      if (lane == 0) DF_STAMP(2, jj, 1);
      qk(tS0, 0, ks);
      umma_commit_elect(s_full + 0);
      if (two) {
        if (lane == 0) DF_STAMP(2, jj, 2);
        if (jj > 0) pv(1, jj - 1);
        if (lane == 0) DF_STAMP(2, jj, 3);
        qk(tS1, 1, ks);
        umma_commit_elect(s_full + 1);
      }
      umma_commit_elect(k_empty + ks);
      if (lane == 0) DF_STAMP(2, jj, 4);
      pv(0, jj);
      if (lane == 0) DF_STAMP(2, jj, 5);
    }
    if (two) pv(1, n_kv - 1);
  } else if (warp >= 2 && (two || warp < 10)) {
    // ------------------------------------------------------------ softmax (half a row per thread)
    const int sw = warp - 2;
    const int t = sw >> 3;
    const int hf = (sw >> 2) & 1;  // key half of every kv tile: columns [64 hf, 64 hf + 64)
    const int quad = warp & 3;
    const int row_local = quad * 32 + lane;
    const int bar_id = 2 + t * 4 + quad;  // the two warps sharing these 32 rows
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + lane_off + t * 128;
    const uint32_t tO = tmem + lane_off + C::kTmemO + t * D;
    constexpr int kHalfD = D / 2;  // O columns this warp rescales / stores
    const float sl2 = p.scale_log2;
    const float2 scale2 = make_float2(sl2, sl2);
    float m = -INFINITY;
    float l = 0.f;  // this half's share of the row sum
    auto xslot = [&](int par, int half) { return xch + ((par * 2 + t) * 128 + row_local) * 2 + half; };

    const bool stamp = lane == 0 && quad == 0 && hf == 0;
    for (int jj = 0; jj < n_kv; ++jj) {
      const int j = kv_begin + jj;
      if (stamp) DF_STAMP(t, jj, 0);
      mbar_wait(s_full + t, jj & 1);
      tc_fence_after();
      if (stamp) DF_STAMP(t, jj, 1);
      uint32_t r[64];
      tmem_ld32(tS + 64 * hf, r);
      tmem_ld32(tS + 64 * hf + 32, r + 32);
      tmem_wait_ld();
      if (stamp) DF_STAMP(t, jj, 2);
      const int valid = hd.n_tok - j * kBN - 64 * hf;
      if (valid < 64) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c >= valid) r[c] = __float_as_uint(-INFINITY);
      }
      float mx[4] = {__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]), __uint_as_float(r[3])};
#pragma unroll
      for (int c = 4; c < 60; c += 8)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mx[k] = fmax3(mx[k], __uint_as_float(r[c + 2 * k]), __uint_as_float(r[c + 2 * k + 1]));
      const float my_max = fmax3(fmax3(mx[0], mx[1], __uint_as_float(r[60])), fmax3(mx[2], mx[3], __uint_as_float(r[61])),
                                 fmaxf(__uint_as_float(r[62]), __uint_as_float(r[63])));
      *xslot(jj & 1, hf) = my_max;
      pair_bar_sync(bar_id);
      const float m_tile = fmaxf(my_max, *xslot(jj & 1, hf ^ 1)) * sl2;
      if (stamp) DF_STAMP(t, jj, 3);
      if (jj == 0) {
        m = m_tile;
      } else {
        const bool need = m_tile > m + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {  // same decision in both warps of the pair
          const float alpha = need ? ex2(m - m_tile) : 1.f;
          if (need) m = m_tile;
          l *= alpha;
          mbar_wait(o_full + t, (jj - 1) & 1);  // O += P_{jj-1} V_{jj-1} has landed
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < kHalfD / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(tO + kHalfD * hf + c * 16, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(tO + kHalfD * hf + c * 16, o);
          }
          tmem_wait_st();
          tc_fence_before();
          pair_bar_sync(bar_id);  // both column halves of O rescaled before either P half goes out
          tc_fence_after();
        }
      }
      const float2 negm2 = make_float2(-m, -m);
      float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int quarter = 0; quarter < 2; ++quarter) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = quarter * 32 + 2 * i;
          const float2 x = fma2(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), scale2, negm2);
          float2 e;
          if (emulated_pair(c / 2)) {
            e = exp2_poly2(x, p.exp_unit);
          } else {
            e = make_float2(ex2(x.x), ex2(x.y));
          }
          sum2 = add2(sum2, e);
          pk[i] = pack_bf16x2(e.x, e.y);
        }
        tmem_st16(tS + 32 * hf + 16 * quarter, pk);
      }
      l += sum2.x + sum2.y;
      tmem_wait_st();
      if (stamp) DF_STAMP(t, jj, 4);
      tc_fence_before();
      mbar_arrive(p_full + 2 * t + hf);
      if (stamp) DF_STAMP(t, jj, 5);
    }

    // ------------------------------------------------------------ epilogue
    *xslot(n_kv & 1, hf) = l;
    pair_bar_sync(bar_id);
    const float l_row = l + *xslot(n_kv & 1, hf ^ 1);
    mbar_wait(o_full + t, (n_kv - 1) & 1);
    tc_fence_after();
    const int prow = t * kBM + row_local;
    const int row = qp * 2 * kBM + prow;
    const bool row_ok = row < p.hw;
    __nv_bfloat16* orow = p.out + (static_cast<int64_t>(hd.o_head) * p.hw + row) * p.out_ld;
    auto store_row = [&](const float* o, int c0, float scale) {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int col = c0 + v * 8;
        if (col < p.d_out) {
          uint4 w;
          w.x = pack_bf16x2(o[v * 8 + 0] * scale, o[v * 8 + 1] * scale);
          w.y = pack_bf16x2(o[v * 8 + 2] * scale, o[v * 8 + 3] * scale);
          w.z = pack_bf16x2(o[v * 8 + 4] * scale, o[v * 8 + 5] * scale);
          w.w = pack_bf16x2(o[v * 8 + 6] * scale, o[v * 8 + 7] * scale);
          *reinterpret_cast<uint4*>(orow + col) = w;
        }
      }
    };
    if (ns == 1) {
      const float inv_l = 1.f / l_row;
#pragma unroll
      for (int c = 0; c < kHalfD / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + kHalfD * hf + c * 32, o);
        tmem_wait_ld();
        if (row_ok) store_row(reinterpret_cast<const float*>(o), kHalfD * hf + c * 32, inv_l);
      }
    } else {
      // split-KV: publish this piece's (O, m, l); the last piece of the pair combines
      const int group = hd.group_base + qp;
      const int64_t slot0 = static_cast<int64_t>(hd.part_base) + static_cast<int64_t>(qp) * ns;
      constexpr int kRowsWs = 2 * kBM;
      float4* my_o = reinterpret_cast<float4*>(p.ws_o) + (slot0 + piece) * (D / 4) * kRowsWs + prow;
#pragma unroll
      for (int c = 0; c < kHalfD / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + kHalfD * hf + c * 32, o);
        tmem_wait_ld();
        const int c4 = (kHalfD * hf + c * 32) / 4;
#pragma unroll
        for (int v = 0; v < 8; ++v)
          __stcg(my_o + (c4 + v) * kRowsWs,
                 make_float4(__uint_as_float(o[4 * v]), __uint_as_float(o[4 * v + 1]), __uint_as_float(o[4 * v + 2]),
                             __uint_as_float(o[4 * v + 3])));
      }
      if (hf == 0) {
        float4* ml = reinterpret_cast<float4*>(p.ws_ml + ((slot0 + piece) * 2 * kBM + prow) * 8);
        __stcg(ml, make_float4(m, l_row, 0.f, 0.f));
      }
      __threadfence();
      const int nthreads = two ? 512 : 256;
      softmax_bar_sync(nthreads);
      if (threadIdx.x == 64) {
        const int prev = atomicAdd(p.ws_cnt + group, 1);
        *last_flag = (prev == ns - 1);
        if (prev == ns - 1) p.ws_cnt[group] = 0;
        __threadfence();
      }
      softmax_bar_sync(nthreads);
      if (*last_flag && row_ok) {
        float mi[16], li[16];
        float M = -INFINITY;
        for (int i = 0; i < ns; ++i) {
          const float4 ml = __ldcg(reinterpret_cast<const float4*>(p.ws_ml + ((slot0 + i) * 2 * kBM + prow) * 8));
          mi[i] = ml.x;
          li[i] = ml.y;
          M = fmaxf(M, ml.x);
        }
        float den = 0.f;
        for (int i = 0; i < ns; ++i) {
          mi[i] = ex2(mi[i] - M);
          den += mi[i] * li[i];
        }
        const float inv = 1.f / den;
#pragma unroll
        for (int c = 0; c < kHalfD / 32; ++c) {
          const int c0 = kHalfD * hf + c * 32;
          float acc[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) acc[e] = 0.f;
          for (int i = 0; i < ns; ++i) {
            const float4* src = reinterpret_cast<const float4*>(p.ws_o) + (slot0 + i) * (D / 4) * kRowsWs + prow;
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const float4 x = __ldcg(src + (c0 / 4 + v) * kRowsWs);
              acc[4 * v + 0] += mi[i] * x.x;
              acc[4 * v + 1] += mi[i] * x.y;
              acc[4 * v + 2] += mi[i] * x.z;
              acc[4 * v + 3] += mi[i] * x.w;
            }
          }
          store_row(acc, c0, inv);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
static int launch_attn_cs(const AttnParams& p, int grid, cudaStream_t stream) {
  using X = CsCfg<D>;
  auto kern = df_attn_cs_kernel<D>;
  static bool configured = false;  // benign race: idempotent attribute set
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, X::kSmem);
    if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(df_attn_cs_kernel)", e);
    configured = true;
  }
  kern<<<grid, kCsThreads, X::kSmem, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("df_attn_cs_kernel launch", e);
  return DF_OK;
}

}  // namespace dfb
