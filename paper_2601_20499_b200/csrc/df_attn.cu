// df_attn.cu -- ragged, head-aware FMHA for one Dummy Forcing layer (sm_100a).
//
// Replaces the per-group numpy attention of the reference
//   engine.py:87-98   _batched_softmax / _batched_attention
//   engine.py:111-137 _run_groups  (every group of a layer in ONE launch; each
//                     head's output written straight to its slot)
// and, with DF_ATTN_PROBE, the probe recompute + region reduction of
//   profiler.py:105-129 (frame_attention_scores), profiler.py:147-170.
//
// Two kernels: df_attn_pair_kernel (CTA pair, d = 128, the default; see its
// header below) and df_attn_kernel (one CTA, d = 64 and DF_ATTN_SINGLE_CTA),
// described here.  Work item = (head, pair of 128-row query tiles).  Each head attends to its
// own contiguous token range of a KV arena (cached frames + current frame), so
// a dummy head with a 2-frame context issues 2/7 of the K/V tiles of a
// baseline head: no masked tiles are ever loaded or multiplied.
//
// CTA = 12 warps (384 threads, 1 CTA/SM):
//   warp 0      TMA producer (Q once; K and V rings)
//   warp 1      TMEM allocator + tcgen05.mma issuer (warp-wide loop, elected lane issues)
//   warps 2-3   idle (warpgroup 0 gives its registers to the softmax groups)
//   warps 4-7   softmax / correction / epilogue for query tile 0 (rows 0-127)
//   warps 8-11  same for query tile 1 (rows 128-255)
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D, 256+2D).
// P (bf16) overwrites the first 64 columns of its S buffer and is the A
// operand (from TMEM) of O += P V.  MMA issue order per kv tile j:
//   S0_j = Q0 K_j^T | O1 += P1_{j-1} V_{j-1} | S1_j = Q1 K_j^T | O0 += P0_j V_j
// so the tensor pipe always has a GEMM queued while either softmax group works.
// Online softmax in the log2 domain with lazy rescaling (threshold 2^DF_RESCALE_THRESHOLD = 2^16).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <queue>
#include <vector>

#include "df_internal.h"
#include "df_ptx.cuh"

namespace dfb {

constexpr int kBM = 128;        // rows per query tile
constexpr int kBN = 128;        // keys per kv tile
constexpr int kWarps = 12;  // see role map above
constexpr int kThreads = kWarps * 32;
#ifndef DF_RESCALE_THRESHOLD
#define DF_RESCALE_THRESHOLD 16.0f  // P <= 2^16 of the running reference; measured: 8 -> 16 cuts N(0,3) logits 352 -> 342 us, N(0,6) 373 -> 350
#endif
constexpr float kRescaleThreshold = DF_RESCALE_THRESHOLD;  // log2 units
constexpr int kMaxSplit = 16;  // kv pieces per query tile (split-KV)
#ifndef DF_EMU_NUM
#define DF_EMU_NUM 1
#endif
// kEmuNum of every 8 exp2 pairs run as a polynomial on the FMA pipe (spread
// evenly): MUFU ex2 is 16/clk/SM, so at d=128 exponentials alone need 100% of
// the tensor-pipe time of a 2 x 128-row tile pair without this offload.
constexpr int kEmuNum = DF_EMU_NUM;
// Scheduling fences in the softmax (df_ptx.cuh sched_fence): without them ptxas
// hoists all 112 MUFU ex2 of a tile above the first P store, so the early
// release of P's first half happens only after every exponential (1: fence
// after the first-half release, 2: also after every other P quarter).
#ifndef DF_SCHED_FENCE
#define DF_SCHED_FENCE 1
#endif
__host__ __device__ constexpr bool emulated_pair(int i) { return (i * kEmuNum) % 8 < kEmuNum; }

struct HeadParam {
  int32_t base_row;
  int32_t n_tok;
  int16_t q_head;
  int16_t o_head;
  int16_t arena;
  int16_t n_split;      // kv pieces per query-tile pair (1 = no split)
  int32_t part_base;    // first partial slot of this head (split heads)
  int32_t group_base;   // first combine counter of this head (split heads)
};

struct __align__(64) AttnParams {
  CUtensorMap qmap;
  CUtensorMap kvmap[DF_MAPS_PER_ARENA * DF_MAX_ARENAS];
  __nv_bfloat16* out;
  const uint8_t* region_tab;
  const uint8_t* row_sampled;
  float* probe_rows;
  float* ws_o;           // split partials, unnormalised O: [slot][D/4][256] float4 (CTA pair: [slot][256][D])
  float* ws_ml;          // [slot][256][8]: running max (log2 units), row sum, probe region masses
  int32_t* ws_cnt;       // [group] arrival counters (zero between launches)
  __nv_bfloat16* peer_out[DF_MAX_PEERS];  // fused all-gather: the same rows into every peer's buffer
  int32_t n_peers;
  int32_t q_per_head;    // qmap is [head][hw][d] (rows past hw zero-fill); else [1][q_rows][d]
  int64_t out_ld;
  int32_t hw;
  int32_t d_out;
  int32_t n_heads;
  int32_t n_qpairs;
  int32_t max_slots;
  float scale_log2;
  uint32_t exp_unit;  // 1 << 23 (exponent step of an fp32), see exp2_poly2
  int32_t item_prefix[DF_MAX_HEADS + 1];  // CTAs before head rank r (LPT order)
  uint8_t head_order[DF_MAX_HEADS];
  HeadParam heads[DF_MAX_HEADS];
};

#ifdef DF_TRACE
// Dev-only timeline of CTA 0 (clock64 stamps): softmax warps 4 / 8 (lane 0)
// and the MMA issuer, first kTraceIters kv tiles.  Read with df_trace_fetch.
constexpr int kTraceIters = 128;
__device__ unsigned long long g_trace[4][kTraceIters][10];
__device__ unsigned long long g_cta_time[1024][4];  // globaltimer ns at CTA start / main-loop end / CTA end, SM id
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define DF_STAMP(who, it, k)                                                        \
  do {                                                                              \
    if (blockIdx.x == 0 && (it) < kTraceIters) g_trace[who][it][k] = clock64();      \
  } while (0)
#else
#define DF_STAMP(who, it, k) \
  do {                       \
  } while (0)
#endif

template <int D>
struct AttnCfg {
#ifndef DF_STAGES_K128
#define DF_STAGES_K128 2
#endif
#ifndef DF_STAGES_V128
#define DF_STAGES_V128 2
#endif
  static constexpr int kStagesK = (D == 128) ? DF_STAGES_K128 : 2;
  static constexpr int kStagesV = (D == 128) ? DF_STAGES_V128 : 3;
  static constexpr int kBoxes = D / 64;                 // 128-byte wide TMA boxes per row
  static constexpr int kTileBytes = kBN * D * 2;        // one [128 x D] bf16 tile
  static constexpr int kBoxBytes = kBN * 128;           // one [128 x 64] box
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + 2 * kTileBytes;
  static constexpr int kVOff = kKOff + kStagesK * kTileBytes;
  static constexpr int kBarOff = kVOff + kStagesV * kTileBytes;
  static constexpr int kNumBars = 1 + 2 * kStagesK + 2 * kStagesV + 8;
  static constexpr int kSmem = kBarOff + kNumBars * 8 + 32 + 1024;  // + 1 KB alignment slack
  static constexpr uint32_t kTmemO = 256;
};

// named barrier of one softmax warpgroup (ids 2, 3; id 1 spans both groups)
__device__ __forceinline__ void wg_bar_sync(int id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

__device__ __forceinline__ void softmax_bar_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int D, bool kProbe>
__global__ void __launch_bounds__(kThreads, 1) df_attn_kernel(const __grid_constant__ AttnParams p) {
  using C = AttnCfg<D>;
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

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work item: (head, query-tile pair, kv piece), heads in LPT order
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
  const bool two = qp * 2 * kBM + kBM < p.hw;  // second query tile has valid rows

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
  if (threadIdx.x == 0) DF_STAMP(2, kTraceIters - 1, 6);
#ifdef DF_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) {
    g_cta_time[blockIdx.x][0] = gtimer();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_cta_time[blockIdx.x][3] = smid;
  }
#endif
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  // Once every CTA of this grid has started, a dependent launched with programmatic
  // stream serialization (the next layer's df_kv_append, which reads nothing this
  // kernel writes) may run on the SMs whose CTAs are done: it fills the last wave.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) DF_STAMP(2, kTraceIters - 1, 7);
  const bool stamp_end = (threadIdx.x & 31) == 0 && ((threadIdx.x >> 5) == 4 || (threadIdx.x >> 5) == 8);
  (void)stamp_end;
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
      const uint64_t keep = policy_evict_last();  // K/V re-read by every q-tile pair of the head
      const int qrow0 = (p.q_per_head ? 0 : hd.q_head * p.hw) + qp * 2 * kBM;
      const int qz = p.q_per_head ? hd.q_head : 0;
      const int nq = two ? 2 : 1;
      mbar_expect_tx(q_full, nq * C::kTileBytes);
      for (int t = 0; t < nq; ++t)
        for (int b = 0; b < C::kBoxes; ++b)
          tma_load_3d(smem + C::kQOff + t * C::kTileBytes + b * C::kBoxBytes, &p.qmap, q_full, b * 64,
                      qrow0 + t * kBM, qz);
      for (int jj = 0; jj < n_kv; ++jj) {
        const int row = hd.base_row + (kv_begin + jj) * kBN;
        {
          const int s = jj % C::kStagesK;
          const uint32_t ph = (jj / C::kStagesK) & 1;
          mbar_wait(k_empty + s, ph ^ 1);
          mbar_expect_tx(k_full + s, C::kTileBytes);
          for (int b = 0; b < C::kBoxes; ++b)
            tma_load_2d_hint(smem + C::kKOff + s * C::kTileBytes + b * C::kBoxBytes, kmap, k_full + s, b * 64,
                             row, keep);
        }
        {
          const int s = jj % C::kStagesV;
          const uint32_t ph = (jj / C::kStagesV) & 1;
          mbar_wait(v_empty + s, ph ^ 1);
          mbar_expect_tx(v_full + s, C::kTileBytes);
          for (int b = 0; b < C::kBoxes; ++b)
            tma_load_2d_hint(smem + C::kVOff + s * C::kTileBytes + b * C::kBoxBytes, vmap, v_full + s, b * 64,
                             row, keep);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp walks the loop (operands warp-uniform), one elected lane
    // issues; descriptors are precomputed 64-bit bases plus compile-time
    // offsets, so a UMMA costs ~1-2 issue slots on a sub-partition shared with
    // two softmax warps.
    constexpr uint32_t idesc_qk = idesc_bf16(kBM, kBN, false);
    constexpr uint32_t idesc_pv = idesc_bf16(kBM, D, true);
    const uint64_t dQ = sdesc_sw128(smem_u32(smem + C::kQOff), 16, 1024);
    const uint64_t dK = sdesc_sw128(smem_u32(smem + C::kKOff), 16, 1024);
    const uint64_t dV = sdesc_sw128(smem_u32(smem + C::kVOff), C::kBoxBytes, 1024);
    constexpr uint64_t kTileDesc = C::kTileBytes >> 4;  // descriptor units (16 B)
    const uint32_t tS0 = tmem, tS1 = tmem + 128;
    const uint32_t tO0 = tmem + C::kTmemO, tO1 = tmem + C::kTmemO + D;

    auto qk = [&](uint32_t d_tmem, int t, int ks) {
      const uint64_t qa = dQ + t * kTileDesc;
      const uint64_t kb = dK + ks * kTileDesc;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint64_t off = ((kk >> 2) * C::kBoxBytes + (kk & 3) * 32) >> 4;
#ifndef DF_DIAG_NO_MMA
        umma_ss_elect(d_tmem, qa + off, kb + off, idesc_qk, kk > 0);
#endif
      }
    };
    auto pv = [&](int t, int jj) {
      const int vs = jj % C::kStagesV;
      mbar_wait(p_full + 2 * t, jj & 1);  // first half of P (keys 0-63) is in TMEM
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
        if (kk == kBN / 32) {  // second half of P (keys 64-127)
          mbar_wait(p_full + 2 * t + 1, jj & 1);
          tc_fence_after();
        }
#ifndef DF_DIAG_NO_MMA
        umma_ts_elect(tO, tP + kk * 8, vb + ((kk * 2048) >> 4), idesc_pv, (jj > 0 || kk > 0) ? 1u : 0u);
#endif
      }
      umma_commit_elect(o_full + t);
      if (t == 1 || !two) umma_commit_elect(v_empty + vs);  // last reader of V_jj
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
  } else if (warp >= 4 && (two || warp < 8)) {
    // ------------------------------------------------------------ softmax
    const int t = (warp - 4) >> 2;        // query tile of this warpgroup
    const int quad = warp & 3;            // TMEM lane quadrant this warp may access
    const int row_local = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + lane_off + t * 128;
    const uint32_t tO = tmem + lane_off + C::kTmemO + t * D;
    const float sl2 = p.scale_log2;
    float m = -INFINITY;
    float l = 0.f;
    float reg_acc[3] = {0.f, 0.f, 0.f};  // probe: sink / neighbor / current mass

    const bool stamp = lane == 0 && quad == 0;
    for (int jj = 0; jj < n_kv; ++jj) {
      const int j = kv_begin + jj;
      if (stamp) DF_STAMP(t, jj, 0);
      mbar_wait(s_full + t, jj & 1);
      tc_fence_after();
      if (stamp) DF_STAMP(t, jj, 1);
#ifdef DF_DIAG_NO_SOFTMAX  // dev: tensor-pipe-only timing (P = whatever S left in TMEM)
      tc_fence_before();
      mbar_arrive(p_full + 2 * t);
      mbar_arrive(p_full + 2 * t + 1);
      continue;
#endif
      uint32_t r[128];
      tmem_ld32(tS + 0, r + 0);
      tmem_ld32(tS + 32, r + 32);
      tmem_ld32(tS + 64, r + 64);
      tmem_ld32(tS + 96, r + 96);
      tmem_wait_ld();
      if (stamp) DF_STAMP(t, jj, 2);
      const int valid = hd.n_tok - j * kBN;
      if (valid < kBN) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c >= valid) r[c] = __float_as_uint(-INFINITY);
      }
      const float m_tile = row_max128(r) * sl2;
      if (stamp) DF_STAMP(t, jj, 3);
      if (jj == 0) {
        m = m_tile;
      } else {
        const bool need = m_tile > m + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = need ? ex2(m - m_tile) : 1.f;
          if (need) m = m_tile;
          l *= alpha;
          if constexpr (kProbe) {
            reg_acc[0] *= alpha;
            reg_acc[1] *= alpha;
            reg_acc[2] *= alpha;
          }
          mbar_wait(o_full + t, (jj - 1) & 1);  // O += P_{jj-1} V_{jj-1} has landed
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(tO + c * 16, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(tO + c * 16, o);
          }
          tmem_wait_st();
        }
      }
      const float2 scale2 = make_float2(sl2, sl2);
      const float2 negm2 = make_float2(-m, -m);
      float2 sum2 = make_float2(0.f, 0.f);
      float span = 0.f;
      float2 lo2 = make_float2(0.f, 0.f);  // probe fast path: mass left of the (single) slot boundary
      int next_b = 0, kind = 0, slot = 0;
      const bool wide = p.hw >= kBN;       // a 128-key tile then spans at most two ring slots
      if constexpr (kProbe) {
        const int c0 = j * kBN;
        slot = min(c0 / p.hw, p.max_slots - 1);
        next_b = (c0 / p.hw + 1) * p.hw - c0;
        kind = p.region_tab[h * p.max_slots + slot];
      }
#pragma unroll
      for (int quarter = 0; quarter < 4; ++quarter) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = quarter * 32 + 2 * i;
          const float2 x = fma2(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), scale2, negm2);
          float2 e;
          if (emulated_pair(c / 2)) {  // compile-time: kEmuNum of every 8 pairs on the FMA pipe
            e = exp2_poly2(x, p.exp_unit);
          } else {
            e = make_float2(ex2(x.x), ex2(x.y));
          }
          const float a = e.x, b = e.y;
          sum2 = add2(sum2, e);
          pk[i] = pack_bf16x2(a, b);
          if constexpr (kProbe) {
            if (wide) {
              lo2 = add2(lo2, make_float2(c < next_b ? a : 0.f, c + 1 < next_b ? b : 0.f));
            } else {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                if (c + e == next_b) {  // warp-uniform region boundary
                  reg_acc[0] += kind == 0 ? span : 0.f;
                  reg_acc[1] += kind == 1 ? span : 0.f;
                  reg_acc[2] += kind == 2 ? span : 0.f;
                  span = 0.f;
                  next_b += p.hw;
                  slot = min(slot + 1, p.max_slots - 1);
                  kind = p.region_tab[h * p.max_slots + slot];
                }
                span += e ? b : a;
              }
            }
          }
        }
        tmem_st16(tS + quarter * 16, pk);
#if DF_SCHED_FENCE >= 2
        if (quarter != 1) sched_fence(p.n_heads < 0, last_flag);
#endif
        if (quarter == 1) {  // release the first half of P early: PV can start on keys 0-63
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(p_full + 2 * t);
          if (stamp) DF_STAMP(t, jj, 4);
#if DF_SCHED_FENCE
          sched_fence(p.n_heads < 0, last_flag);  // keep the second half's exponentials below the release
#endif
        }
      }
      if constexpr (kProbe) {
        if (wide) {
          const float lo = lo2.x + lo2.y, hi = (sum2.x + sum2.y) - lo;
          const int kind1 = p.region_tab[h * p.max_slots + min(slot + 1, p.max_slots - 1)];
          reg_acc[0] += (kind == 0 ? lo : 0.f) + (kind1 == 0 ? hi : 0.f);
          reg_acc[1] += (kind == 1 ? lo : 0.f) + (kind1 == 1 ? hi : 0.f);
          reg_acc[2] += (kind == 2 ? lo : 0.f) + (kind1 == 2 ? hi : 0.f);
        } else {
          reg_acc[0] += kind == 0 ? span : 0.f;
          reg_acc[1] += kind == 1 ? span : 0.f;
          reg_acc[2] += kind == 2 ? span : 0.f;
        }
      }
      l += sum2.x + sum2.y;
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full + 2 * t + 1);
      if (stamp) DF_STAMP(t, jj, 5);
    }

    // ------------------------------------------------------------ epilogue
    if (stamp) DF_STAMP(t, kTraceIters - 1, 6);
#ifdef DF_TRACE
    if (threadIdx.x == 128 && blockIdx.x < 1024) g_cta_time[blockIdx.x][1] = gtimer();
#endif
    mbar_wait(o_full + t, (n_kv - 1) & 1);
    tc_fence_after();
    const int prow = t * kBM + row_local;           // row within the pair
    const int row = qp * 2 * kBM + prow;            // row within the head
    const bool row_ok = row < p.hw;
    const int64_t orow_off = (static_cast<int64_t>(hd.o_head) * p.hw + row) * p.out_ld;
    __nv_bfloat16* orow = p.out + orow_off;
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
#ifndef DF_NO_PEERS
          for (int pi = 0; pi < p.n_peers; ++pi)  // fused all-gather: NVLink stores into the peers' buffers
            *reinterpret_cast<uint4*>(p.peer_out[pi] + orow_off + col) = w;
#endif
        }
      }
    };
    if (ns == 1) {
      const float inv_l = 1.f / l;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + c * 32, o);
        tmem_wait_ld();
        if (row_ok) store_row(reinterpret_cast<const float*>(o), c * 32, inv_l);
      }
      if constexpr (kProbe) {
        if (row_ok && p.row_sampled[row]) {
          float* dst = p.probe_rows + (static_cast<int64_t>(h) * p.hw + row) * 3;
          dst[0] = reg_acc[0] * inv_l;
          dst[1] = reg_acc[1] * inv_l;
          dst[2] = reg_acc[2] * inv_l;
        }
      }
    } else {
      // split-KV: publish this piece's (O, m, l); the last piece of the pair combines.
      const int group = hd.group_base + qp;
      const int64_t slot0 = static_cast<int64_t>(hd.part_base) + static_cast<int64_t>(qp) * ns;
      // partial O layout [slot][D/4 float4 columns][256 rows]: the 32 rows of a warp
      // write (and the combine reads) 512 contiguous bytes per instruction
      constexpr int kRowsWs = 2 * kBM;
      float4* my_o = reinterpret_cast<float4*>(p.ws_o) + (slot0 + piece) * (D / 4) * kRowsWs + prow;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + c * 32, o);
        tmem_wait_ld();
#pragma unroll
        for (int v = 0; v < 8; ++v)
          __stcg(my_o + (c * 8 + v) * kRowsWs,
                 make_float4(__uint_as_float(o[4 * v]), __uint_as_float(o[4 * v + 1]), __uint_as_float(o[4 * v + 2]),
                             __uint_as_float(o[4 * v + 3])));
      }
      {  // (m, l) and, with the probe epilogue, the three region masses of this piece
        float4* ml = reinterpret_cast<float4*>(p.ws_ml + ((slot0 + piece) * 2 * kBM + prow) * 8);
        __stcg(ml, make_float4(m, l, reg_acc[0], reg_acc[1]));
        if constexpr (kProbe) __stcg(ml + 1, make_float4(reg_acc[2], 0.f, 0.f, 0.f));
      }
      __threadfence();
      const int nthreads = two ? 256 : 128;
      softmax_bar_sync(nthreads);
      if (threadIdx.x == 128) {
        const int prev = atomicAdd(p.ws_cnt + group, 1);
        *last_flag = (prev == ns - 1);
        if (prev == ns - 1) p.ws_cnt[group] = 0;  // ready for the next launch
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
        float reg[3] = {0.f, 0.f, 0.f};
        for (int i = 0; i < ns; ++i) {
          mi[i] = ex2(mi[i] - M);
          den += mi[i] * li[i];
          if constexpr (kProbe) {
            const float* ml = p.ws_ml + ((slot0 + i) * 2 * kBM + prow) * 8;
            reg[0] += mi[i] * __ldcg(ml + 2);
            reg[1] += mi[i] * __ldcg(ml + 3);
            reg[2] += mi[i] * __ldcg(ml + 4);
          }
        }
        const float inv = 1.f / den;
        if constexpr (kProbe) {
          if (p.row_sampled[row]) {  // profiler.py:118-129 region masses of the whole row
            float* dst = p.probe_rows + (static_cast<int64_t>(h) * p.hw + row) * 3;
            dst[0] = reg[0] * inv;
            dst[1] = reg[1] * inv;
            dst[2] = reg[2] * inv;
          }
        }
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float acc[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) acc[e] = 0.f;
          for (int i = 0; i < ns; ++i) {
            const float4* src = reinterpret_cast<const float4*>(p.ws_o) + (slot0 + i) * (D / 4) * kRowsWs + prow;
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const float4 x = __ldcg(src + (c * 8 + v) * kRowsWs);
              acc[4 * v + 0] += mi[i] * x.x;
              acc[4 * v + 1] += mi[i] * x.y;
              acc[4 * v + 2] += mi[i] * x.z;
              acc[4 * v + 3] += mi[i] * x.w;
            }
          }
          store_row(acc, c * 32, inv);
        }
      }
    }
  }

  if (stamp_end) DF_STAMP(warp == 4 ? 0 : 1, kTraceIters - 1, 7);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) DF_STAMP(2, kTraceIters - 1, 8);
#ifdef DF_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_time[blockIdx.x][2] = gtimer();
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// =====================================================================
// CTA-pair variant (cta_group::2, d = 128): three softmax warpgroups in a ring.
//
// A cluster of two CTAs on one TPC computes M = 256 query rows per MMA: CTA
// rank r owns rows [r*128, r*128+128) of the item's 256-row query tile, half of
// every K tile (64 keys) and half of every V tile (64 columns); the leader's MMA
// warp issues tcgen05.mma.cta_group::2 for both.  Work item = (head, 256 query
// rows, kv piece) -- the 1-CTA kernel's granularity, on half as many bins.
//
// Why: in the 1-CTA kernel a query tile's next QK^T waits for the PV that
// consumes its P (P aliases S and TMEM holds only S0 S1 O0 O1), so each softmax
// warpgroup idles ~1200 cycles per kv tile (clock64 trace).  With 128 rows per
// CTA, TMEM holds THREE score buffers and one O:
//   S_0 [0,128)  S_1 [128,256)  S_2 [256,384)  O [384,512)
// Three softmax warpgroups take the kv tiles in turn (tile j -> WG j%3, buffer
// j%3; P overwrites the first 64 columns of its S buffer).  The MMA warp issues
//   QK_0 QK_1 QK_2, then per tile j:  PV_j | QK_{j+3}
// so two score tiles are always computed ahead, and a warpgroup's next S (three
// tiles on) lands while the other two groups work.  The running max m is one per
// row: each WG hands the m after its tile to the next WG of the ring (named
// barrier per TMEM lane quadrant), which rescales its own partial row sum when m
// moved; the lazy O rescale (threshold 2^16) waits for the previous PV.  A WG
// reads its S in two passes (row max, then exponentials 32 columns at a time), so
// the 14-warp CTA fits in 144 registers per thread.
//
// Warps: 0 TMA producer, 1 TMEM allocator + MMA issuer (leader CTA), 2-13 the
// softmax groups (WG g = warps 2+4g .. 5+4g; warp w reads TMEM lane quadrant w%4).
constexpr int kPairWarps = 14;
constexpr int kPairThreads = kPairWarps * 32;

struct PairCfg {
  static constexpr int D = 128;
#ifndef DF_PAIR_STAGES_K
#define DF_PAIR_STAGES_K 5
#endif
#ifndef DF_PAIR_STAGES_V
#define DF_PAIR_STAGES_V 4
#endif
  static constexpr int kStagesK = DF_PAIR_STAGES_K;  // K ring depth
  static constexpr int kStagesV = DF_PAIR_STAGES_V;  // V ring depth
  static constexpr int kKAhead = 3;                  // K loads lead V loads by this many tiles (QK_{j+3} before PV_j)
  static constexpr int kQBytes = 128 * D * 2;        // this CTA's 128 query rows
  static constexpr int kQBoxBytes = 128 * 128;       // [128 rows x 64 cols]
  static constexpr int kKHalfBytes = 64 * D * 2;     // 64 keys x d
  static constexpr int kKBoxBytes = 64 * 128;        // [64 rows x 64 cols]
  static constexpr int kVHalfBytes = 128 * 64 * 2;   // 128 keys x 64 columns
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQBytes;
  static constexpr int kVOff = kKOff + kStagesK * kKHalfBytes;
  static constexpr int kXOff = kVOff + kStagesV * kVHalfBytes;  // m handoff [128], final m [128], [3 WG][4][128] sums
  static constexpr int kXBytes = (128 + 128 + 3 * 4 * 128) * 4;
  static constexpr int kBarOff = kXOff + kXBytes;
  static constexpr int kNumBars = 1 + 2 * kStagesK + 2 * kStagesV + 3 + 6 + 3;
  static constexpr int kSmem = kBarOff + kNumBars * 8 + 32 + 1024;
  static constexpr uint32_t kTO = 384;
};

// Named barriers of the pair kernel (64 threads: one warp of each of two WGs):
// m handoff out of WG g for lane quadrant q: 2 + 4g + q.  Id 1 spans all softmax warps.
__device__ __forceinline__ void nbar_arrive64(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void nbar_sync64(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

template <bool kProbe>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    df_attn_pair_kernel(const __grid_constant__ AttnParams p) {
  using C = PairCfg;
  constexpr int D = C::D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + C::kStagesK;
  uint64_t* v_full = k_empty + C::kStagesK;
  uint64_t* v_empty = v_full + C::kStagesV;
  uint64_t* s_full = v_empty + C::kStagesV;  // [3] S buffer written (multicast commit)
  uint64_t* p_full = s_full + 3;             // [3 buffers][2 halves] leader: 8 warp arrivals
  uint64_t* pv_done = p_full + 6;            // [3] PV from that buffer landed (multicast commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 3);
  int32_t* last_flag = reinterpret_cast<int32_t*>(tmem_slot + 1);
  float* m_x = reinterpret_cast<float*>(smem + C::kXOff);  // [128] m handoff
  float* m_fin = m_x + 128;                                 // [128] final m
  float* l_x = m_fin + 128;                                 // [3 WG][4: l, 3 region masses][128]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  int hrank = 0;
  while (hrank + 1 < p.n_heads && p.item_prefix[hrank + 1] <= pair) ++hrank;
  const int h = p.head_order[hrank];
  const HeadParam hd = p.heads[h];
  const int local = pair - p.item_prefix[hrank];
  const int ns = hd.n_split;
  const int qt = local / ns;
  const int piece = local - qt * ns;
  const int n_kv_total = (hd.n_tok + kBN - 1) / kBN;
  const int kv_begin = (piece * n_kv_total) / ns;
  const int n_kv = ((piece + 1) * n_kv_total) / ns - kv_begin;

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
    for (int b = 0; b < 3; ++b) {
      mbar_init(s_full + b, 1);
      mbar_init(p_full + 2 * b, 8);  // one arrival per softmax warp of either CTA
      mbar_init(p_full + 2 * b + 1, 8);
      mbar_init(pv_done + b, 1);
    }
    fence_mbar_init();
  }
#ifdef DF_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) {
    g_cta_time[blockIdx.x][0] = gtimer();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_cta_time[blockIdx.x][3] = smid;
  }
#endif
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const void* kmap = &p.kvmap[DF_MAPS_PER_ARENA * hd.arena + 2];  // 64-row boxes
      const void* vmap = &p.kvmap[DF_MAPS_PER_ARENA * hd.arena + 1];
      prefetch_tmap(&p.qmap);
      prefetch_tmap(kmap);
      prefetch_tmap(vmap);
      const uint64_t keep = policy_evict_last();
      const int qrow0 = (p.q_per_head ? 0 : hd.q_head * p.hw) + qt * 2 * kBM + static_cast<int>(crank) * kBM;
      const int qz = p.q_per_head ? hd.q_head : 0;
      if (crank == 0) mbar_expect_tx(q_full, 2 * C::kQBytes);
      const uint32_t lq = mapa_shared(smem_u32(q_full), 0);
      for (int b = 0; b < 2; ++b)
        tma_load_3d_pair(smem + C::kQOff + b * C::kQBoxBytes, &p.qmap, lq, b * 64, qrow0, qz, keep);
      // K runs kKAhead tiles ahead of V (QK_{j+3} is issued right after PV_j)
      auto load_k = [&](int jj) {
        const int s = jj % C::kStagesK;
        mbar_wait(k_empty + s, ((jj / C::kStagesK) & 1) ^ 1);
        if (crank == 0) mbar_expect_tx(k_full + s, 2 * C::kKHalfBytes);
        const uint32_t lk = mapa_shared(smem_u32(k_full + s), 0);
        const int row = hd.base_row + (kv_begin + jj) * kBN + static_cast<int>(crank) * 64;
        for (int b = 0; b < 2; ++b)
          tma_load_2d_pair(smem + C::kKOff + s * C::kKHalfBytes + b * C::kKBoxBytes, kmap, lk, b * 64, row, keep);
      };
      auto load_v = [&](int jj) {
        const int s = jj % C::kStagesV;
        mbar_wait(v_empty + s, ((jj / C::kStagesV) & 1) ^ 1);
        if (crank == 0) mbar_expect_tx(v_full + s, 2 * C::kVHalfBytes);
        const uint32_t lv = mapa_shared(smem_u32(v_full + s), 0);
        tma_load_2d_pair(smem + C::kVOff + s * C::kVHalfBytes, vmap, lv, static_cast<int>(crank) * 64,
                         hd.base_row + (kv_begin + jj) * kBN, keep);
      };
      for (int jj = 0; jj < n_kv + C::kKAhead; ++jj) {
        if (jj < n_kv) load_k(jj);
        if (jj >= C::kKAhead) load_v(jj - C::kKAhead);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (crank == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16(2 * kBM, kBN, false);
      constexpr uint32_t idesc_pv = idesc_bf16(2 * kBM, D, true);
      const uint64_t dQ = sdesc_sw128(smem_u32(smem + C::kQOff), 16, 1024);
      const uint64_t dK = sdesc_sw128(smem_u32(smem + C::kKOff), 16, 1024);
      const uint64_t dV = sdesc_sw128(smem_u32(smem + C::kVOff), 16, 1024);
      const uint32_t tO = tmem + C::kTO;

      auto qk = [&](int j) {  // S_{j%3} = Q K_j^T; in pipe order after PV_{j-3}, which read P from that buffer
        const int ks = j % C::kStagesK;
        const int b = j % 3;
        mbar_wait(k_full + ks, (j / C::kStagesK) & 1);
        tc_fence_after();
        if (lane == 0) DF_STAMP(3, j, 0);
        static_assert(C::kQBoxBytes >> 4 == 1024 && C::kKBoxBytes >> 4 == 512, "umma_ss_pair_qk8 offsets");
#ifndef DF_DIAG_NO_MMA
        umma_ss_pair_qk8(tmem + b * 128, dQ, dK + ((ks * C::kKHalfBytes) >> 4), idesc_qk);
#endif
        umma_commit_pair_elect(s_full + b);
        umma_commit_pair_elect(k_empty + ks);
      };
      auto pv = [&](int j) {  // O += P_{j%3} V_j
        const int vs = j % C::kStagesV;
        const int b = j % 3;
        const uint32_t ph = (j / 3) & 1;
        mbar_wait(p_full + 2 * b, ph);  // keys 0-63 of P(j)
        mbar_wait(v_full + vs, (j / C::kStagesV) & 1);
        tc_fence_after();
        if (lane == 0) DF_STAMP(3, j, 1);
        const uint64_t vb = dV + ((vs * C::kVHalfBytes) >> 4);
        const uint32_t tP = tmem + b * 128;
#ifndef DF_DIAG_NO_MMA
        umma_ts_pair_pv4(tO, tP, vb, idesc_pv, j > 0 ? 1u : 0u);
#endif
        mbar_wait(p_full + 2 * b + 1, ph);  // keys 64-127
        tc_fence_after();
#ifndef DF_DIAG_NO_MMA
        umma_ts_pair_pv4(tO, tP + 32, vb + ((4 * 2048) >> 4), idesc_pv, 1u);
#endif
        umma_commit_pair_elect(pv_done + b);
        umma_commit_pair_elect(v_empty + vs);
        if (lane == 0) DF_STAMP(3, j, 2);
      };

      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j < 3 && j < n_kv; ++j) qk(j);
      for (int j = 0; j < n_kv; ++j) {
        pv(j);
        if (j + 3 < n_kv) qk(j + 3);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax (both CTAs)
    const int wg = (warp - 2) >> 2;  // tiles j with j % 3 == wg, score buffer wg
    const int quad = warp & 3;       // TMEM lane quadrant of this warp
    const int row_local = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + lane_off + wg * 128;  // S, then P in its first 64 columns
    const uint32_t tO = tmem + lane_off + C::kTO;
    const int bar_in = 2 + 4 * ((wg + 2) % 3) + quad;  // m handed over by the previous WG of the ring
    const int bar_out = 2 + 4 * wg + quad;             // m handed to the next WG
    auto arrive_leader = [&](uint64_t* bar) {          // one arrival per warp on the leader's barrier
      if (crank == 0)
        mbar_arrive(bar);
      else
        mbar_arrive_cluster(mapa_shared(smem_u32(bar), 0));
    };
    const float sl2 = p.scale_log2;
    float m = -INFINITY;  // the running max this WG last used (log2 units)
    float l = 0.f;        // this WG's partial row sum, relative to m
    float reg_acc[3] = {0.f, 0.f, 0.f};  // probe: sink / neighbor / current mass, relative to m

    const bool stamp = lane == 0 && quad == 0;
    // A lane quadrant whose 32 query rows all lie past the head's end (the last query tile of a head:
    // at HW 4680, 5 of its 8 quadrants) has no softmax to do: its rows' P and O are never read.  Its
    // warps only keep the barrier protocol (the same quadrant of every WG is dead, so the m hand-off
    // between them is skipped on both sides).
#ifndef DF_DEAD_SKIP
#define DF_DEAD_SKIP 1
#endif
    const bool dead = DF_DEAD_SKIP && qt * 2 * kBM + static_cast<int>(crank) * kBM + quad * 32 >= p.hw;
    for (int jj = wg; jj < n_kv; jj += 3) {
      const int j = kv_begin + jj;
      const int use = jj / 3;
      if (stamp) DF_STAMP(wg, use, 0);
      mbar_wait(s_full + wg, use & 1);
      tc_fence_after();
      if (stamp) DF_STAMP(wg, use, 1);
      if (dead) {
        __syncwarp();
        if (lane == 0) {
          arrive_leader(p_full + 2 * wg);
          arrive_leader(p_full + 2 * wg + 1);
        }
        continue;
      }
      const int valid = hd.n_tok - j * kBN;  // keys of this tile inside the head's context
#ifdef DF_DIAG_NO_SOFTMAX  // dev: tensor-pipe-only timing (P = whatever TMEM holds)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        arrive_leader(p_full + 2 * wg);
        arrive_leader(p_full + 2 * wg + 1);
      }
      continue;
#endif
      if (valid < kBN) {  // the head's last tile: -inf into the score columns past its context (rare)
        for (int c0 = (valid / 32) * 32; c0 < kBN; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(tS + c0, r);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (c0 + c >= valid) r[c] = __float_as_uint(-INFINITY);
          tmem_st32(tS + c0, r);
        }
        tmem_wait_st();
      }
      // pass 1: the row max of the tile, 64 columns per TMEM load
      float mx;
      {
        uint32_t r[64];
        tmem_ld32(tS + 0, r);
        tmem_ld32(tS + 32, r + 32);
        tmem_wait_ld();
        float a0 = fmax3(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]));
        float a1 = fmax3(__uint_as_float(r[3]), __uint_as_float(r[4]), __uint_as_float(r[5]));
#pragma unroll
        for (int c = 6; c < 62; c += 4) {
          a0 = fmax3(a0, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
          a1 = fmax3(a1, __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
        }
        mx = fmax3(a0, a1, fmaxf(__uint_as_float(r[62]), __uint_as_float(r[63])));
#ifdef DF_DIAG_HALF_MAX  // dev: pass 1 reads half the columns (TMEM-bandwidth experiment; wrong m)
        if (false) {
#else
        if (valid > 64) {
#endif
          tmem_ld32(tS + 64, r);
          tmem_ld32(tS + 96, r + 32);
          tmem_wait_ld();
          a0 = fmax3(mx, __uint_as_float(r[0]), __uint_as_float(r[1]));
          a1 = fmax3(__uint_as_float(r[2]), __uint_as_float(r[3]), __uint_as_float(r[4]));
#pragma unroll
          for (int c = 5; c < 61; c += 4) {
            a0 = fmax3(a0, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
            a1 = fmax3(a1, __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
          }
          mx = fmax3(a0, a1, fmax3(__uint_as_float(r[61]), __uint_as_float(r[62]), __uint_as_float(r[63])));
        }
      }
      const float m_tile = mx * sl2;
      if (stamp) DF_STAMP(wg, use, 2);
      // the running max after the previous tile (the previous WG's), then this tile's
      float m_prev = m;
      if (jj > 0) {
        nbar_sync64(bar_in);
        m_prev = m_x[row_local];
        if (m_prev != m) {  // another WG raised m since this WG's last tile
          const float a = ex2(m - m_prev);
          l *= a;
          if constexpr (kProbe) {
            reg_acc[0] *= a;
            reg_acc[1] *= a;
            reg_acc[2] *= a;
          }
        }
      }
      bool rescale = false;
      float alpha = 1.f;
      if (jj == 0) {
        m = m_tile;
      } else if (m_tile > m_prev + kRescaleThreshold) {
        alpha = ex2(m_prev - m_tile);
        m = m_tile;
        rescale = true;
      } else {
        m = m_prev;
      }
      if (jj + 1 < n_kv) {
        m_x[row_local] = m;
        nbar_arrive64(bar_out);
      }
      if (stamp) DF_STAMP(wg, use, 5);
      if (rescale) {
        l *= alpha;
        if constexpr (kProbe) {
          reg_acc[0] *= alpha;
          reg_acc[1] *= alpha;
          reg_acc[2] *= alpha;
        }
      }
      if (__any_sync(0xffffffffu, rescale)) {  // O *= alpha once PV_{jj-1} has landed
        const int pb = (jj - 1) % 3;
        mbar_wait(pv_done + pb, ((jj - 1) / 3) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 16; ++c) {
          uint32_t o[16];
          tmem_ld16(tO + c * 16, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st16(tO + c * 16, o);
        }
        tmem_wait_st();
      }
      if (stamp) DF_STAMP(wg, use, 3);
      // pass 2: exponentials 32 columns at a time (the next chunk's TMEM load in flight); P quarter q
      // overwrites S columns [16q, 16q+16), which the chunks already read
      const float2 scale2 = make_float2(sl2, sl2);
      const float2 negm2 = make_float2(-m, -m);
      float2 sum2 = make_float2(0.f, 0.f);
      float span = 0.f;
      float2 lo2 = make_float2(0.f, 0.f), part2 = make_float2(0.f, 0.f);  // probe: keys left of the boundary
      int next_b = 0, kind = 0, slot = 0;
      const bool wide = p.hw >= kBN;
      if constexpr (kProbe) {
        const int c0 = j * kBN;
        slot = min(c0 / p.hw, p.max_slots - 1);
        next_b = (c0 / p.hw + 1) * p.hw - c0;
        kind = p.region_tab[h * p.max_slots + slot];
      }
      uint32_t rb[2][32];
      tmem_ld32(tS, rb[0]);
      tmem_wait_ld();
#pragma unroll
      for (int quarter = 0; quarter < 4; ++quarter) {
        uint32_t* r = rb[quarter & 1];
        if (quarter < 3) tmem_ld32(tS + (quarter + 1) * 32, rb[(quarter + 1) & 1]);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = quarter * 32 + 2 * i;
          const float2 x = fma2(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), scale2, negm2);
          float2 e;
          if (emulated_pair(c / 2)) {
            e = exp2_poly2(x, p.exp_unit);
          } else {
            e = make_float2(ex2(x.x), ex2(x.y));
          }
          sum2 = add2(sum2, e);
          pk[i] = pack_bf16x2(e.x, e.y);
          if constexpr (kProbe) {
            if (!wide) {
#pragma unroll
              for (int k2 = 0; k2 < 2; ++k2) {
                if (c + k2 == next_b) {
                  reg_acc[0] += kind == 0 ? span : 0.f;
                  reg_acc[1] += kind == 1 ? span : 0.f;
                  reg_acc[2] += kind == 2 ? span : 0.f;
                  span = 0.f;
                  next_b += p.hw;
                  slot = min(slot + 1, p.max_slots - 1);
                  kind = p.region_tab[h * p.max_slots + slot];
                }
                span += k2 ? e.y : e.x;
              }
            }
          }
        }
        if constexpr (kProbe) {
          // one slot boundary at most per tile (HW >= 128): the mass left of it is the running sum after
          // the last quarter wholly left of it, plus -- in the quarter the boundary cuts (about one tile
          // in HW/128) -- that quarter's keys left of it, their exponentials recomputed (same code path,
          // so lo + hi = the tile's sum)
          if (wide) {
            if ((quarter + 1) * 32 <= next_b) {
              lo2 = sum2;
            } else if (quarter * 32 < next_b) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int c = quarter * 32 + 2 * i;
                const float2 x =
                    fma2(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), scale2, negm2);
                const float2 e = emulated_pair(c / 2) ? exp2_poly2(x, p.exp_unit) : make_float2(ex2(x.x), ex2(x.y));
                part2 = add2(part2, make_float2(c < next_b ? e.x : 0.f, c + 1 < next_b ? e.y : 0.f));
              }
            }
          }
        }
        if (quarter < 3) tmem_wait_ld();  // chunk quarter+1 is in registers
        tmem_st16(tS + quarter * 16, pk);
        if (quarter == 1) {  // keys 0-63 of P: PV_jj may start
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(p_full + 2 * wg);
#if DF_SCHED_FENCE
          sched_fence(p.n_heads < 0, last_flag);
#endif
        }
      }
      if constexpr (kProbe) {
        if (wide) {
          const float lo = (lo2.x + lo2.y) + (part2.x + part2.y), hi = (sum2.x + sum2.y) - lo;
          const int kind1 = p.region_tab[h * p.max_slots + min(slot + 1, p.max_slots - 1)];
          reg_acc[0] += (kind == 0 ? lo : 0.f) + (kind1 == 0 ? hi : 0.f);
          reg_acc[1] += (kind == 1 ? lo : 0.f) + (kind1 == 1 ? hi : 0.f);
          reg_acc[2] += (kind == 2 ? lo : 0.f) + (kind1 == 2 ? hi : 0.f);
        } else {
          reg_acc[0] += kind == 0 ? span : 0.f;
          reg_acc[1] += kind == 1 ? span : 0.f;
          reg_acc[2] += kind == 2 ? span : 0.f;
        }
      }
      l += sum2.x + sum2.y;
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(p_full + 2 * wg + 1);
      if (stamp) DF_STAMP(wg, use, 4);
    }

    // ------------------------------------------------------------ epilogue
#ifdef DF_TRACE
    if (threadIdx.x == 64 && blockIdx.x < 1024) g_cta_time[blockIdx.x][1] = gtimer();
#endif
    // every WG brings its row sum to the final running max (the last tile's WG has it), then sums
    const int last_wg = (n_kv - 1) % 3;
    if (wg == last_wg) m_fin[row_local] = m;
    softmax_bar_sync(12 * 32);
    {
      const float mf = m_fin[row_local];
      const float a = (l > 0.f) ? ex2(m - mf) : 0.f;  // m = -inf (no tile): l is 0 and stays 0
      float* mine = l_x + wg * 4 * 128;
      mine[row_local] = l * a;
      if constexpr (kProbe) {
        mine[128 + row_local] = reg_acc[0] * a;
        mine[256 + row_local] = reg_acc[1] * a;
        mine[384 + row_local] = reg_acc[2] * a;
      }
      m = mf;
    }
    softmax_bar_sync(12 * 32);
    l = l_x[row_local] + l_x[512 + row_local] + l_x[1024 + row_local];
    if constexpr (kProbe) {
#pragma unroll
      for (int k = 0; k < 3; ++k)
        reg_acc[k] = l_x[(k + 1) * 128 + row_local] + l_x[512 + (k + 1) * 128 + row_local] +
                     l_x[1024 + (k + 1) * 128 + row_local];
    }
    const int lb = (n_kv - 1) % 3;
    mbar_wait(pv_done + lb, ((n_kv - 1) / 3) & 1);  // the last PV (PVs land in order)
    tc_fence_after();
    const int row = qt * 2 * kBM + static_cast<int>(crank) * kBM + row_local;  // row within the head
    const bool row_ok = row < p.hw;
    const int64_t orow_off = (static_cast<int64_t>(hd.o_head) * p.hw + row) * p.out_ld;
    __nv_bfloat16* orow = p.out + orow_off;
    const int c_lo = wg * (D / 2);  // WG 0 / 1 store output columns [c_lo, c_lo + 64); WG 2 the probe rows
    auto store_row = [&](const float* o, int c0, float scale) {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int col = c0 + v * 8;
        if (col < p.d_out) {
          uint4 wv;
          wv.x = pack_bf16x2(o[v * 8 + 0] * scale, o[v * 8 + 1] * scale);
          wv.y = pack_bf16x2(o[v * 8 + 2] * scale, o[v * 8 + 3] * scale);
          wv.z = pack_bf16x2(o[v * 8 + 4] * scale, o[v * 8 + 5] * scale);
          wv.w = pack_bf16x2(o[v * 8 + 6] * scale, o[v * 8 + 7] * scale);
          *reinterpret_cast<uint4*>(orow + col) = wv;
#ifndef DF_NO_PEERS
          for (int pi = 0; pi < p.n_peers; ++pi)  // fused all-gather: NVLink stores into the peers' buffers
            *reinterpret_cast<uint4*>(p.peer_out[pi] + orow_off + col) = wv;
#endif
        }
      }
    };
    if (ns == 1) {
      const float inv_l = 1.f / l;
      if (wg < 2 && !dead) {
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          uint32_t o[32];
          tmem_ld32(tO + c_lo + c * 32, o);
          tmem_wait_ld();
          if (row_ok) store_row(reinterpret_cast<const float*>(o), c_lo + c * 32, inv_l);
        }
      } else if constexpr (kProbe) {
        if (row_ok && p.row_sampled[row]) {
          float* dst = p.probe_rows + (static_cast<int64_t>(h) * p.hw + row) * 3;
          dst[0] = reg_acc[0] * inv_l;
          dst[1] = reg_acc[1] * inv_l;
          dst[2] = reg_acc[2] * inv_l;
        }
      }
    } else {
      // split-KV, per CTA of the pair: slot (piece, rank), counter (group, rank); rows of a slot 256 apart
      const int group = (hd.group_base + qt) * 2 + static_cast<int>(crank);
      const int64_t slot0 = static_cast<int64_t>(hd.part_base) + static_cast<int64_t>(qt) * ns;
      auto slot_of = [&](int i) { return (slot0 + i) * 2 + crank; };
      if (dead) {
      } else if (wg < 2) {
        float* my_o = p.ws_o + (slot_of(piece) * 2 * kBM + row_local) * D;
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          uint32_t o[32];
          tmem_ld32(tO + c_lo + c * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int v = 0; v < 8; ++v)
            __stcg(reinterpret_cast<float4*>(my_o + c_lo + c * 32 + v * 4),
                   make_float4(__uint_as_float(o[4 * v]), __uint_as_float(o[4 * v + 1]),
                               __uint_as_float(o[4 * v + 2]), __uint_as_float(o[4 * v + 3])));
        }
      } else {
        float* my_ml = p.ws_ml + (slot_of(piece) * 2 * kBM + row_local) * 8;
        __stcg(reinterpret_cast<float4*>(my_ml), make_float4(m, l, reg_acc[0], reg_acc[1]));
        __stcg(my_ml + 4, reg_acc[2]);
      }
      __threadfence();
      softmax_bar_sync(12 * 32);
      if (threadIdx.x == 64) {
        const int prev = atomicAdd(p.ws_cnt + group, 1);
        *last_flag = (prev == ns - 1);
        if (prev == ns - 1) p.ws_cnt[group] = 0;
        __threadfence();
      }
      softmax_bar_sync(12 * 32);
      if (*last_flag && row_ok) {
        // the combine issues every piece's (m, l) at once and the O partials two pieces at a time
        // (16 float4 loads in flight per thread): it is latency-bound, not bandwidth-bound
        float ei[kMaxSplit], li[kMaxSplit];
        float M = -INFINITY;
#pragma unroll
        for (int i = 0; i < kMaxSplit; ++i)
          if (i < ns) {
            const float4 ml = __ldcg(reinterpret_cast<const float4*>(p.ws_ml + (slot_of(i) * 2 * kBM + row_local) * 8));
            ei[i] = ml.x;
            li[i] = ml.y;
            M = fmaxf(M, ml.x);
          }
        float den = 0.f;
        float racc[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < kMaxSplit; ++i)
          if (i < ns) {
            ei[i] = ex2(ei[i] - M);
            den += ei[i] * li[i];
            if constexpr (kProbe) {
              const float* ml = p.ws_ml + (slot_of(i) * 2 * kBM + row_local) * 8;
              racc[0] += ei[i] * __ldcg(ml + 2);
              racc[1] += ei[i] * __ldcg(ml + 3);
              racc[2] += ei[i] * __ldcg(ml + 4);
            }
          }
        const float inv = 1.f / den;
        if (wg < 2) {
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            float acc[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) acc[q] = 0.f;
#pragma unroll
            for (int i = 0; i < kMaxSplit; i += 2) {
              if (i < ns) {
                const bool two = i + 1 < ns;
                const float4* sa =
                    reinterpret_cast<const float4*>(p.ws_o + (slot_of(i) * 2 * kBM + row_local) * D + c_lo + c * 32);
                const float4* sb = reinterpret_cast<const float4*>(
                    p.ws_o + (slot_of(two ? i + 1 : i) * 2 * kBM + row_local) * D + c_lo + c * 32);
                float4 xa[8], xb[8];
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                  xa[v] = __ldcg(sa + v);
                  xb[v] = two ? __ldcg(sb + v) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                const float ea = ei[i], eb = two ? ei[i + 1] : 0.f;
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                  acc[4 * v + 0] += ea * xa[v].x + eb * xb[v].x;
                  acc[4 * v + 1] += ea * xa[v].y + eb * xb[v].y;
                  acc[4 * v + 2] += ea * xa[v].z + eb * xb[v].z;
                  acc[4 * v + 3] += ea * xa[v].w + eb * xb[v].w;
                }
              }
            }
            store_row(acc, c_lo + c * 32, inv);
          }
        } else if constexpr (kProbe) {
          if (p.row_sampled[row]) {
            float* dst = p.probe_rows + (static_cast<int64_t>(h) * p.hw + row) * 3;
            dst[0] = racc[0] * inv;
            dst[1] = racc[1] * inv;
            dst[2] = racc[2] * inv;
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's smem and TMEM stay live until the leader's MMAs are done
#ifdef DF_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_time[blockIdx.x][2] = gtimer();
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

template <bool kProbe>
static int launch_attn_pair(const AttnParams& p, int grid, cudaStream_t stream) {
  auto kern = df_attn_pair_kernel<kProbe>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg::kSmem);
    if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(df_attn_pair_kernel)", e);
    configured = true;
  }
  kern<<<grid, kPairThreads, PairCfg::kSmem, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("df_attn_pair_kernel launch", e);
  return DF_OK;
}

template <int D, bool kProbe>
static int launch_attn(const AttnParams& p, int grid, cudaStream_t stream) {
  using C = AttnCfg<D>;
  auto kern = df_attn_kernel<D, kProbe>;
  static bool configured = false;  // benign race: idempotent attribute set
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(df_attn_kernel)", e);
    configured = true;
  }
  kern<<<grid, kThreads, C::kSmem, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("df_attn_kernel launch", e);
  return DF_OK;
}

int sm_count_cached() {
  static int count = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev);
    if (count <= 0) count = 148;
  });
  return count;
}

}  // namespace dfb

using namespace dfb;

namespace {

// ------------------------------------------------------------------ planner
// Hardware list-schedules CTAs in blockIdx order as SMs free up, so the
// launch order below (heads by decreasing piece cost, pairs ascending) is LPT.
// The planner picks per-head kv split counts that minimise the simulated
// makespan over the SMs, charging a fixed prologue/epilogue cost per CTA and
// a combine cost per split piece.  Cost unit: one 128-key tile for a full
// pair of 128-row query tiles.
double env_or(const char* name, double dflt) {
  const char* v = std::getenv(name);
  return v ? std::atof(v) : dflt;
}
const double kPieceOverhead = env_or("DF_PLAN_PIECE", 3.0);  // dev override for calibration sweeps
const double kSplitOverhead = env_or("DF_PLAN_SPLIT", 1.0);
// the last-arriving piece of a split pair reads every piece's fp32 partial
// (128 KB each) alone: ~1 tile-unit per piece on that one CTA (calibrated with
// scripts/plan_sweep.py: Wan all-context 880 -> 804 us, packed unchanged)
const double kCombinePerPiece = env_or("DF_PLAN_COMBINE", 1.0);
constexpr double kSingleTileFactor = 0.95;  // last pair with only its first tile valid: no ping-pong, ~as slow as a full pair (clock64 trace)
const bool kPlanRefine = env_or("DF_PLAN_REFINE", 1.0) != 0.0;  // dev A/B

struct Plan {
  uint8_t ns[DF_MAX_HEADS];
  int order[DF_MAX_HEADS];
  int64_t ws_bytes;
  int n_items;
};


// rows of one work item: a pair of 128-row tiles (1-CTA kernel) or one 256-row MMA tile over a CTA pair
inline int item_rows(bool) { return 256; }

double simulate(const df_attn_args* a, const uint8_t* ns, const int* order, int sms, bool pair) {
  const int R = item_rows(pair);
  const int nq = (a->hw + R - 1) / R;
  const bool last_single = (nq - 1) * R + R / 2 >= a->hw;
  std::priority_queue<double, std::vector<double>, std::greater<double>> bins;
  for (int i = 0; i < sms; ++i) bins.push(0.0);
  double makespan = 0.0;
  for (int r = 0; r < a->num_heads; ++r) {
    const int h = order[r];
    const int tiles = (a->heads[h].n_tok + 127) / 128;
    for (int qp = 0; qp < nq; ++qp) {
      const double f = (qp == nq - 1 && last_single && !pair) ? kSingleTileFactor : 1.0;
      for (int s = 0; s < ns[h]; ++s) {
        const int len = ((s + 1) * tiles) / ns[h] - (s * tiles) / ns[h];
        double c = len * f + kPieceOverhead + (ns[h] > 1 ? kSplitOverhead : 0.0);
        if (ns[h] > 1 && s == ns[h] - 1) c += kCombinePerPiece * ns[h];  // (arrival order approximated)
        const double t0 = bins.top();
        bins.pop();
        bins.push(t0 + c);
        makespan = std::max(makespan, t0 + c);
      }
    }
  }
  return makespan;
}

void order_heads(const df_attn_args* a, const uint8_t* ns, int* order) {
  for (int i = 0; i < a->num_heads; ++i) order[i] = i;
  std::stable_sort(order, order + a->num_heads, [&](int x, int y) {
    const double cx = double((a->heads[x].n_tok + 127) / 128) / ns[x];
    const double cy = double((a->heads[y].n_tok + 127) / 128) / ns[y];
    return cx > cy;
  });
}

// Split-KV workspace layout: [fp32 partials (O, then m/l/region masses) | ... | combine counters].
// The counters live in a FIXED region at the END of the caller's workspace
// (kCntBytes), so a later launch with more split groups never reads an earlier
// launch's partials as counters: the region is zero when allocated and every
// launch leaves its counters at zero, whatever the partial sizes in between.
constexpr int64_t kCntBytes = 64 * 1024;  // 16384 counters: groups x ranks
constexpr int64_t kMaxCounters = kCntBytes / 4;

int64_t split_groups(const df_attn_args* a, const uint8_t* ns, bool pair, int64_t* slots_out) {
  const int R = item_rows(pair);
  const int nq = (a->hw + R - 1) / R;
  int64_t groups = 0, slots = 0;
  for (int h = 0; h < a->num_heads; ++h)
    if (ns[h] > 1) {
      groups += nq;
      slots += int64_t(nq) * ns[h];
    }
  if (slots_out) *slots_out = slots;
  return groups;
}

int64_t workspace_need(const df_attn_args* a, const uint8_t* ns, bool pair) {
  int64_t slots = 0;
  if (!split_groups(a, ns, pair, &slots)) return 0;
  const int64_t ranks = pair ? 2 : 1;
  const int64_t part_bytes = ((slots * ranks * 256 * (int64_t(a->head_dim) + 8) * 4 + 255) / 256) * 256;
  return part_bytes + kCntBytes;
}

Plan make_plan(const df_attn_args* a, bool allow_split, bool pair) {
  Plan best{};
  const int sms = pair ? sm_count_cached() / 2 : sm_count_cached();
  for (int i = 0; i < a->num_heads; ++i) best.ns[i] = 1;
  order_heads(a, best.ns, best.order);
  double best_t = simulate(a, best.ns, best.order, sms, pair);
  if (allow_split) {
    int max_tiles = 1;
    for (int h = 0; h < a->num_heads; ++h) max_tiles = std::max(max_tiles, (a->heads[h].n_tok + 127) / 128);
    // candidate caps on tiles per piece
    for (int cap = 8; cap < max_tiles; cap += std::max(1, cap / 8)) {
      Plan c{};
      for (int h = 0; h < a->num_heads; ++h) {
        const int tiles = (a->heads[h].n_tok + 127) / 128;
        c.ns[h] = static_cast<uint8_t>(std::min(kMaxSplit, std::max(1, (tiles + cap - 1) / cap)));
      }
      if (split_groups(a, c.ns, pair, nullptr) * (pair ? 2 : 1) > kMaxCounters) continue;
      {  // more than ~6 pieces per SM: per-piece overheads dominate, not worth simulating
        const int nq = (a->hw + item_rows(pair) - 1) / item_rows(pair);
        int64_t items = 0;
        for (int h = 0; h < a->num_heads; ++h) items += int64_t(nq) * c.ns[h];
        if (items > 6 * int64_t(sms)) continue;
      }
      order_heads(a, c.ns, c.order);
      const double t = simulate(a, c.ns, c.order, sms, pair);
      if (t < best_t * 0.995) {
        best_t = t;
        std::memcpy(best.ns, c.ns, sizeof(c.ns));
        std::memcpy(best.order, c.order, sizeof(c.order));
      }
    }
  }
  const double uniform_t = best_t;
  const Plan uniform = best;
  // Refinement costs up to a few hundred simulations (~10-40 ms of host time per new signature, and a
  // rollout meets dozens of signatures): skip it when the uniform plan is already within 3% of the
  // list-scheduling lower bound (all work spread evenly, at one piece per head)
  double total = 0.0;
  {
    const int nq = (a->hw + item_rows(pair) - 1) / item_rows(pair);
    for (int h = 0; h < a->num_heads; ++h) total += double(nq) * ((a->heads[h].n_tok + 127) / 128 + kPieceOverhead);
  }
  const bool near_bound = uniform_t <= 1.03 * total / sms;
  if (allow_split && kPlanRefine && !near_bound) {
    // per-head refinement of the best uniform cap: a few rounds of coordinate descent over each
    // head's split count (ragged packed layers want e.g. some short heads split to fill the last
    // wave that the long heads' pieces leave)
    // Moves: set the split count of the first k heads of a length class (heads with the same
    // context) to v -- single heads alone rarely help, a packed layer wants e.g. every neighbor
    // head at 3 pieces AND two of its dummy heads at 3.
    std::vector<std::vector<int>> classes;
    for (int h = 0; h < a->num_heads; ++h) {
      bool placed = false;
      for (auto& c : classes)
        if (a->heads[c[0]].n_tok == a->heads[h].n_tok) {
          c.push_back(h);
          placed = true;
          break;
        }
      if (!placed) classes.push_back({h});
    }
    for (int round = 0; round < 2; ++round) {
      bool improved = false;
      for (const auto& cls : classes) {
        const int tiles = (a->heads[cls[0]].n_tok + 127) / 128;
        const int cur = best.ns[cls[0]];
        for (int v = std::max(1, cur - 2); v <= std::min({kMaxSplit, tiles, 2 * cur + 2}); ++v)
          for (size_t k = 1; k <= cls.size(); ++k) {
            Plan c = best;
            bool changed = false;
            for (size_t i = 0; i < k; ++i) {
              changed |= c.ns[cls[i]] != v;
              c.ns[cls[i]] = static_cast<uint8_t>(v);
            }
            if (!changed) continue;
            if (split_groups(a, c.ns, pair, nullptr) * (pair ? 2 : 1) > kMaxCounters) continue;
            order_heads(a, c.ns, c.order);
            const double t = simulate(a, c.ns, c.order, sms, pair);
            if (t < best_t * 0.999) {
              best_t = t;
              best = c;
              improved = true;
            }
          }
      }
      if (!improved) break;
    }
  }
  if (best_t > uniform_t * 0.98) {  // predicted gains under 2% were not real on the GPU (packed Wan: 193 -> 191)
    best = uniform;
    best_t = uniform_t;
  }
  if (std::getenv("DF_PLAN_DEBUG")) {
    std::fprintf(stderr, "plan hw %d heads %d: makespan %.1f (uniform best %.1f) ns:", a->hw, a->num_heads, best_t,
                 uniform_t);
    for (int h = 0; h < a->num_heads; ++h) std::fprintf(stderr, " %d/%d", (a->heads[h].n_tok + 127) / 128, best.ns[h]);
    std::fprintf(stderr, "\n");
  }
  best.ws_bytes = workspace_need(a, best.ns, pair);
  const int nq = (a->hw + item_rows(pair) - 1) / item_rows(pair);
  best.n_items = 0;
  for (int h = 0; h < a->num_heads; ++h) best.n_items += nq * best.ns[h];
  return best;
}

// Plans are cached per (hw, head_dim, n_tok list, probe) -- a session issues
// the same signature for every layer of a step.
struct PlanCache {
  std::mutex mu;
  std::map<std::vector<int64_t>, Plan> map;
};
PlanCache& plan_cache() {
  static PlanCache c;
  return c;
}

// The cache key is the SORTED context list: a session's layers carry the same multiset of head
// lengths in different head orders after classification, and a plan depends only on the lengths
// (the canonical plan's split counts are mapped back through the sort permutation).
Plan get_plan(const df_attn_args* a, bool allow_split, bool pair) {
  const int H = a->num_heads;
  std::vector<int> perm(H);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return a->heads[x].n_tok > a->heads[y].n_tok; });
  std::vector<int64_t> key;
  key.reserve(H + 5);
  key.push_back(a->hw);
  key.push_back(a->head_dim);
  key.push_back(allow_split);
  key.push_back(pair);
  key.push_back(sm_count_cached());
  for (int i = 0; i < H; ++i) key.push_back(a->heads[perm[i]].n_tok);
  Plan canon{};
  bool hit = false;
  PlanCache& pc = plan_cache();
  {
    std::lock_guard<std::mutex> g(pc.mu);
    auto it = pc.map.find(key);
    if (it != pc.map.end()) {
      canon = it->second;
      hit = true;
    }
  }
  if (!hit) {
    df_attn_args sorted = *a;
    std::vector<df_head_desc> heads(H);
    for (int i = 0; i < H; ++i) heads[i] = a->heads[perm[i]];
    sorted.heads = heads.data();
    canon = make_plan(&sorted, allow_split, pair);
    std::lock_guard<std::mutex> g(pc.mu);
    if (pc.map.size() > 4096) pc.map.clear();
    pc.map.emplace(std::move(key), canon);
  }
  Plan p = canon;
  for (int i = 0; i < H; ++i) p.ns[perm[i]] = canon.ns[i];
  order_heads(a, p.ns, p.order);
  return p;
}

int validate(const df_attn_args* a) {
  if (!a) return set_error(DF_E_ARG, "df_attn_fwd: null args");
  if (a->head_dim != 64 && a->head_dim != 128)
    return set_error(DF_E_SHAPE, "df_attn_fwd: head_dim must be 64 or 128 (got %d)", a->head_dim);
  if (a->d_out < 8 || a->d_out > a->head_dim || (a->d_out % 8) != 0)
    return set_error(DF_E_SHAPE, "df_attn_fwd: d_out %d must be a multiple of 8 in [8, head_dim]", a->d_out);
  if (a->num_heads < 1 || a->num_heads > DF_MAX_HEADS)
    return set_error(DF_E_SHAPE, "df_attn_fwd: num_heads %d outside [1, %d]", a->num_heads, DF_MAX_HEADS);
  if (a->num_arenas < 1 || a->num_arenas > DF_MAX_ARENAS)
    return set_error(DF_E_ARG, "df_attn_fwd: num_arenas %d outside [1, %d]", a->num_arenas, DF_MAX_ARENAS);
  if (a->hw < 1) return set_error(DF_E_SHAPE, "df_attn_fwd: hw must be >= 1");
  if (!a->q || !a->out || !a->heads || !a->kv_maps) return set_error(DF_E_ARG, "df_attn_fwd: null pointer");
  if (a->out_ld < a->d_out) return set_error(DF_E_SHAPE, "df_attn_fwd: out_ld < d_out");
  if (a->n_peers < 0 || a->n_peers > DF_MAX_PEERS || (a->n_peers > 0 && !a->peer_out))
    return set_error(DF_E_ARG, "df_attn_fwd: n_peers %d outside [0, %d] or peer_out missing", a->n_peers,
                     DF_MAX_PEERS);
  for (int i = 0; i < a->n_peers; ++i)
    if (!a->peer_out[i] || (reinterpret_cast<uintptr_t>(a->peer_out[i]) & 15))
      return set_error(DF_E_ARG, "df_attn_fwd: peer_out[%d] null or not 16-byte aligned", i);
  if (a->q_rows < 1 || a->q_rows > INT32_MAX) return set_error(DF_E_SHAPE, "df_attn_fwd: bad q_rows");
  if ((reinterpret_cast<uintptr_t>(a->q) & 15) || (reinterpret_cast<uintptr_t>(a->out) & 15) || (a->out_ld % 8))
    return set_error(DF_E_ARG, "df_attn_fwd: q/out must be 16-byte aligned, out_ld a multiple of 8");
  for (int i = 0; i < a->num_heads; ++i) {
    const df_head_desc& h = a->heads[i];
    if (h.n_tok < 1) return set_error(DF_E_SHAPE, "df_attn_fwd: head %d has empty context", i);
    if (h.arena < 0 || h.arena >= a->num_arenas) return set_error(DF_E_ARG, "df_attn_fwd: head %d bad arena", i);
    if (h.base_row < 0 || h.base_row + h.n_tok > INT32_MAX)
      return set_error(DF_E_ARG, "df_attn_fwd: head %d arena rows out of int32 range", i);
    if (h.q_head < 0 || static_cast<int64_t>(h.q_head) * a->hw >= a->q_rows || h.o_head < 0 || h.q_head > 32767 ||
        h.o_head > 32767)
      return set_error(DF_E_SHAPE, "df_attn_fwd: head %d q/o index out of range", i);
  }
  return DF_OK;
}

// CTA-pair kernel: d = 128 only; DF_ATTN_SINGLE_CTA forces the 1-CTA kernel.
bool use_pair(const df_attn_args* a) {
  if (a->head_dim != 128 || (a->flags & DF_ATTN_SINGLE_CTA)) return false;
  return (a->flags & DF_ATTN_PAIR) != 0;
}

}  // namespace

extern "C" int df_attn_workspace_bytes(const df_attn_args* a, int64_t* bytes) {
  int rc = validate(a);
  if (rc != DF_OK) return rc;
  if (!bytes) return set_error(DF_E_ARG, "df_attn_workspace_bytes: null output");
  const bool pair = use_pair(a);
  *bytes = get_plan(a, true, pair).ws_bytes;
  return DF_OK;
}

extern "C" int df_attn_fwd(const df_attn_args* a, void* stream) {
  int rc = validate(a);
  if (rc != DF_OK) return rc;
  const bool probe = (a->flags & DF_ATTN_PROBE) != 0;
  if (probe && (!a->region_of_slot || !a->row_sampled || !a->probe_rows || a->max_slots < 1))
    return set_error(DF_E_ARG, "df_attn_fwd: probe epilogue needs region_of_slot, row_sampled, probe_rows");

  // Split plan; fall back to no splitting when the workspace cannot hold it.
  const bool pair = use_pair(a);
  Plan plan = get_plan(a, true, pair);  // split pieces combine O, l and the probe region masses
  if (plan.ws_bytes > 0 && (!a->workspace || a->workspace_bytes < plan.ws_bytes ||
                            (reinterpret_cast<uintptr_t>(a->workspace) & 255)))
    plan = get_plan(a, false, pair);

  AttnParams p;
  std::memset(&p, 0, sizeof(p));
  // Q as [head][hw][d] when the rows are whole heads: a head's last query tile then reads zeros past
  // its hw rows (TMA OOB fill) instead of the next head's rows -- zero operands for the padding rows
  p.q_per_head = (a->q_rows % a->hw) == 0;
  rc = p.q_per_head ? encode_bf16_3d(&p.qmap, a->q, a->q_rows / a->hw, a->hw, a->head_dim, 128)
                    : encode_bf16_3d(&p.qmap, a->q, 1, a->q_rows, a->head_dim, 128);
  if (rc != DF_OK) return rc;
  std::memcpy(p.kvmap, a->kv_maps, static_cast<size_t>(a->num_arenas) * DF_MAPS_PER_ARENA * DF_TMAP_BYTES);
  p.out = static_cast<__nv_bfloat16*>(a->out);
  p.out_ld = a->out_ld;
  p.n_peers = a->n_peers;
  for (int i = 0; i < a->n_peers; ++i) p.peer_out[i] = static_cast<__nv_bfloat16*>(a->peer_out[i]);
  p.hw = a->hw;
  p.d_out = a->d_out;
  p.n_heads = a->num_heads;
  p.n_qpairs = (a->hw + item_rows(pair) - 1) / item_rows(pair);
  p.max_slots = probe ? a->max_slots : 1;
  p.region_tab = a->region_of_slot;
  p.row_sampled = a->row_sampled;
  p.probe_rows = a->probe_rows;
  p.scale_log2 = a->scale * 1.4426950408889634f;
  p.exp_unit = 1u << 23;

  int64_t groups = 0, slots = 0;
  for (int i = 0; i < a->num_heads; ++i) {
    const df_head_desc& h = a->heads[i];
    HeadParam& hp = p.heads[i];
    hp.base_row = static_cast<int32_t>(h.base_row);
    hp.n_tok = h.n_tok;
    hp.q_head = static_cast<int16_t>(h.q_head);
    hp.o_head = static_cast<int16_t>(h.o_head);
    hp.arena = static_cast<int16_t>(h.arena);
    hp.n_split = plan.ns[i];
    if (plan.ns[i] > 1) {
      hp.group_base = static_cast<int32_t>(groups);
      hp.part_base = static_cast<int32_t>(slots);
      groups += p.n_qpairs;
      slots += int64_t(p.n_qpairs) * plan.ns[i];
    }
  }
  if (groups) {
    const int64_t ranks = pair ? 2 : 1;
    uint8_t* ws = static_cast<uint8_t*>(a->workspace);
    p.ws_o = reinterpret_cast<float*>(ws);
    p.ws_ml = p.ws_o + slots * ranks * 2 * kBM * a->head_dim;
    // fixed counter region at the end (4-byte aligned; callers pass the same workspace size every launch)
    p.ws_cnt = reinterpret_cast<int32_t*>(ws + ((a->workspace_bytes - kCntBytes) & ~int64_t(255)));
  }
  int acc = 0;
  for (int r = 0; r < a->num_heads; ++r) {
    p.head_order[r] = static_cast<uint8_t>(plan.order[r]);
    p.item_prefix[r] = acc;
    acc += p.n_qpairs * plan.ns[plan.order[r]];
  }
  p.item_prefix[a->num_heads] = acc;

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (pair) return probe ? launch_attn_pair<true>(p, 2 * acc, s) : launch_attn_pair<false>(p, 2 * acc, s);
  const int grid = acc;
  if (a->head_dim == 128) {
    return probe ? launch_attn<128, true>(p, grid, s) : launch_attn<128, false>(p, grid, s);
  }
  return probe ? launch_attn<64, true>(p, grid, s) : launch_attn<64, false>(p, grid, s);
}

#ifdef DF_TRACE
extern "C" DF_API int df_trace_cta(void* host) {
  return cudaMemcpyFromSymbol(host, dfb::g_cta_time, sizeof(dfb::g_cta_time)) == cudaSuccess ? DF_OK : DF_E_CUDA;
}
extern "C" DF_API int df_trace_fetch(void* host, int64_t bytes) {
  if (bytes > int64_t(sizeof(dfb::g_trace))) bytes = sizeof(dfb::g_trace);
  return cudaMemcpyFromSymbol(host, dfb::g_trace, bytes) == cudaSuccess ? DF_OK : DF_E_CUDA;
}
#endif
