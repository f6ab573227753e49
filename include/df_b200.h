/*
 * df_b200.h -- C ABI of the B200 (sm_100a) Dummy Forcing attention hot path.
 *
 * Plain pointers, sizes and a CUDA stream; no torch types.  Every entry point
 * returns an int status (DF_OK == 0).  On error df_last_error() returns a
 * thread-local message and the host mirror maps the code onto the reference's
 * exception type (see paper_2601_20499_b200/_lib.py and
 * /root/reference/pkg/src/dummy_forcing/errors.py:4-33).
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/dummy_forcing/):
 *
 *   df_attn_fwd        engine.py:87-98   _batched_softmax / _batched_attention
 *                      engine.py:111-137 _run_groups (all groups of one layer
 *                                        in ONE ragged launch; outputs written
 *                                        straight into their head slot, K7)
 *                      engine.py:140-195 baseline_step / hma_step / packed_step
 *     + DF_ATTN_PROBE  profiler.py:105-129 frame_attention_scores and the
 *                      probe recompute in profiler.py:147-170 (global_scores),
 *                      fused into the attention epilogue
 *   df_scores_finalize profiler.py:118-129 (mean of region masses over the
 *                      sampled rows, profiler.py:132-144)
 *   df_kv_append       kv_cache.py:177-185 append_and_evict (data movement of
 *                      the appended frame into its ring slot) and the current
 *                      frame of kv_cache.py:211-213 gather_context
 *   df_kv_pack         kv_cache.py:199-201 rebuild (+ _evict 187-197): the
 *                      classification-time compaction of retained frames into
 *                      the packed per-class layout
 *   df_greedy_classify head_programming.py:141-164 greedy_classify
 *                      (lexsort tie rules, F0 >= F1 sink rule, numpy pairwise
 *                      objective sum)
 *   df_kv_arena_maps   (no reference counterpart: builds the TMA descriptors of
 *                      a device KV arena once per allocation)
 *   df_qkv_project     scenario.py:102-114 ToyModel.qkv (x @ W_q|k|v, split
 *                      into heads) + engine.py:423-426 FrameBlock wrap: the
 *                      epilogue writes Q in the FMHA layout and the current
 *                      K/V straight into each head's pending ring slot, so no
 *                      append/staging copy remains
 *   df_out_project     scenario.py:116-120 ToyModel.mix (merge heads, @ W_o)
 *                      + engine.py:443 residual x = x + mix(...), fused into
 *                      one GEMM epilogue
 */
#ifndef DF_B200_H
#define DF_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DF_API __attribute__((visibility("default")))
#else
#define DF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> errors.py exception types */
#define DF_OK 0
#define DF_E_SHAPE 1    /* ShapeError       errors.py:8   */
#define DF_E_PACKING 2  /* PackingError     errors.py:24  */
#define DF_E_ORDER 3    /* OrderingError    errors.py:16  */
#define DF_E_CONFIG 4   /* ConfigError      errors.py:20  */
#define DF_E_ASSIGN 5   /* AssignmentError  errors.py:28  */
#define DF_E_CUDA 6     /* CUDA runtime / launch failure   */
#define DF_E_ARG 7      /* invalid argument (ValueError)   */

#define DF_MAX_HEADS 64     /* heads per df_attn_fwd launch */
#define DF_MAX_ARENAS 4     /* distinct KV arenas per launch */
#define DF_TMAP_BYTES 128   /* one CUtensorMap */
#define DF_MAPS_PER_ARENA 3 /* K (128-row box), V (128-row box), K (64-row box) */
#define DF_MAX_APPEND_SEGS 128
#define DF_MAX_PEERS 7      /* peer output buffers of the fused head-output all-gather */

/* df_attn_args.flags */
#define DF_ATTN_PROBE 1u       /* fused DHP region-mass epilogue */
#define DF_ATTN_PAIR 2u        /* d = 128: CTA-pair (cta_group::2, M = 256) kernel */
#define DF_ATTN_SINGLE_CTA 4u  /* force the 1-CTA kernel */

/* One head of one layer.  Its context is the contiguous token range
 * [base_row, base_row + n_tok) of arena `arena` (K and V share row indices);
 * rows are head_dim bf16 wide.  The ring manager keeps the cached frames plus
 * the current frame in that range (softmax is invariant to key order). */
typedef struct df_head_desc {
  int64_t base_row;
  int32_t n_tok;     /* (cached frames + 1) * hw, >= 1 */
  int32_t q_head;    /* Q rows [q_head*hw, q_head*hw + hw) */
  int32_t o_head;    /* output rows [o_head*hw, ...) */
  int32_t arena;     /* index into kv_maps, < num_arenas */
} df_head_desc;

typedef struct df_attn_args {
  const void* q;          /* device bf16 [q_rows][head_dim]; when q_rows is a multiple of hw it is
                             read as [q_rows/hw][hw][head_dim], so a head's last query tile never
                             touches the next head's rows (padding rows read as zeros) */
  int64_t q_rows;
  void* out;              /* device bf16; element (o_head*hw + r, c) at out[(o_head*hw+r)*out_ld + c] */
  int64_t out_ld;         /* elements */
  int32_t hw;             /* tokens per frame (query rows per head) */
  int32_t head_dim;       /* 64 or 128: width of Q and arena rows */
  int32_t d_out;          /* output columns (<= head_dim, multiple of 8) */
  float scale;            /* logit scale, reference 1/sqrt(head_dim) (engine.py:120) */
  int32_t num_heads;      /* <= DF_MAX_HEADS */
  int32_t num_arenas;     /* <= DF_MAX_ARENAS */
  const df_head_desc* heads;  /* host [num_heads] */
  const uint8_t* kv_maps;     /* host [num_arenas][DF_MAPS_PER_ARENA][DF_TMAP_BYTES] from df_kv_arena_maps */
  uint32_t flags;
  int32_t max_slots;              /* probe: row stride of region_of_slot */
  const uint8_t* region_of_slot;  /* probe, device [num_heads][max_slots]; 0 sink 1 neighbor 2 current */
  const uint8_t* row_sampled;     /* probe, device [hw] (profiler.py:132-144) */
  float* probe_rows;              /* probe, device [num_heads][hw][3] region masses per sampled row */
  /* Split-KV workspace (device, caller-owned, zero-filled once).  Layout:
   * fp32 partials from the start, combine counters in the LAST 64 KB; every
   * launch leaves its counters at zero, so pass the same buffer with the same
   * workspace_bytes every time (the counters' position follows the size).
   * NULL or smaller than df_attn_workspace_bytes => no kv splitting. */
  void* workspace;
  int64_t workspace_bytes;
  /* Fused head-output all-gather (head-parallel sessions, SURVEY 8(e) / 8(f)
   * row 2; replaces the NCCL all-gather after engine.py:111-137 scatters the
   * outputs): the epilogue also stores every output row, at the same offset
   * as in `out`, into each of these buffers -- the other ranks' gathered-
   * output buffers mapped into this process (CUDA IPC / symmetric memory),
   * so the stores travel over NVLink as tiles finish.  The caller orders the
   * peers' reads after the launch (a cross-rank barrier on the stream).
   * NULL / 0 = none.  Not supported with DF_ATTN_PAIR. */
  void* const* peer_out;  /* host array [n_peers] of device pointers */
  int32_t n_peers;        /* <= DF_MAX_PEERS */
} df_attn_args;

/* A row-strided device copy: `rows` rows of `row_bytes` bytes. row_bytes and
 * both strides must be multiples of 16 (16-byte vectorised). */
typedef struct df_copy_seg {
  const void* src;
  void* dst;
  int64_t rows;
  int64_t src_ld;    /* bytes */
  int64_t dst_ld;    /* bytes */
  int64_t row_bytes;
} df_copy_seg;

/* ---- attention (tcgen05 / TMEM / TMA, sm_100a) ---- */
DF_API int df_attn_fwd(const df_attn_args* args, void* stream);
/* Workspace df_attn_fwd would use for these heads (LPT split plan over the
 * device's SMs); 0 when no head is split. */
DF_API int df_attn_workspace_bytes(const df_attn_args* args, int64_t* bytes);

/* TMA descriptors (DF_MAPS_PER_ARENA*DF_TMAP_BYTES bytes: K, V, K-half maps)
 * of an arena whose K and V planes are device bf16 [rows][head_dim]. */
DF_API int df_kv_arena_maps(const void* k_base, const void* v_base, int64_t rows,
                     int32_t head_dim, uint8_t* out_maps);

/* ---- ring manager data movement ---- */
/* Up to DF_MAX_APPEND_SEGS segments passed by value (one launch). */
DF_API int df_kv_append(const df_copy_seg* segs, int32_t n_segs, void* stream);
/* Same copy, launched with programmatic stream serialization: if the kernel
 * before it on the stream is df_attn_fwd, it may start while that launch's last
 * wave is still running.  Only when the copy writes no byte the preceding
 * df_attn_fwd reads or writes (Q, the K/V rows up to each head's last 128-row
 * tile, out, probe buffers, workspace) and reads none it writes, e.g. the next
 * layer's ring slots; the caller checks this (the Python layer compares merged
 * byte ranges at launch time, kernels.PreparedLaunch). */
DF_API int df_kv_append_overlapped(const df_copy_seg* segs, int32_t n_segs, void* stream);
/* Bulk compaction: segment list already in device memory; chunk_prefix is a
 * device int64 [n_segs+1] exclusive prefix of per-segment 16-byte-chunk
 * counts divided by chunk granularity (see df_kv_pack_plan). */
DF_API int df_kv_pack(const df_copy_seg* segs_dev, const int64_t* block_prefix_dev,
               int32_t n_segs, int64_t total_blocks, void* stream);
/* Host helper: fills block_prefix_host[n_segs+1] for df_kv_pack; returns the
 * number of CTAs through *total_blocks. */
DF_API int df_kv_pack_plan(const df_copy_seg* segs_host, int32_t n_segs,
                    int64_t* block_prefix_host, int64_t* total_blocks);

/* ---- DHP ---- */
/* F[h][k] = mean over sampled rows r of probe_rows[h][r][k] (fp64, fixed
 * order).  F is device double [num_heads][3]. */
DF_API int df_scores_finalize(const float* probe_rows, const uint8_t* row_sampled,
                       int32_t num_heads, int32_t hw, double* F, void* stream);
/* Host.  classes_out: 0 sink, 1 neighbor, 2 dummy (head_programming.py:38, _CLASS_CODES). */
DF_API int df_greedy_classify(const double* F, int64_t total_heads, int64_t n_dummy,
                       int8_t* classes_out, double* objective_out);

/* ---- misc ---- */
/* ---- fused projections (tcgen05 GEMM, persistent, bf16 in / fp32 accumulate) */
typedef struct df_qkv_args {
  const void* x;        /* bf16 [hw, in_dim] row-major: the layer input             */
  const void* w_qkv;    /* bf16 [3*num_heads*head_dim, in_dim]: rows = the columns of
                           W_q, then W_k, then W_v of these heads ([W_q|W_k|W_v]^T)  */
  int32_t hw, num_heads, head_dim;  /* head_dim 64 or 128                          */
  int32_t in_dim;       /* multiple of 8 (16-byte rows)                             */
  void* q_out;          /* bf16 [num_heads*hw, head_dim] (df_attn_fwd's q)           */
  void* k_dst[DF_MAX_HEADS]; /* bf16 row 0 of each head's destination K block       */
  void* v_dst[DF_MAX_HEADS]; /* (the pending ring slot), rows strided by kv_ld      */
  int64_t kv_ld;        /* elements between consecutive K/V rows (arena width)      */
} df_qkv_args;
DF_API int df_qkv_project(const df_qkv_args* args, void* stream);

typedef struct df_oproj_args {
  const void* o;        /* bf16 [num_heads*hw, head_dim]: df_attn_fwd's output     */
  const void* w_o;      /* bf16 [out_dim, num_heads*head_dim]: rows = columns of W_o */
  int32_t hw, num_heads, head_dim;
  int32_t out_dim;      /* multiple of 32                                           */
  float* x;             /* fp32 [hw, out_dim], updated in place: x += merge(o)@W_o  */
  void* x_bf16;         /* bf16 [hw, out_dim] copy of the updated x, or NULL        */
} df_oproj_args;
DF_API int df_out_project(const df_oproj_args* args, void* stream);

DF_API const char* df_last_error(void);
DF_API int df_version(void);
/* DF_OK when a compute-capability-10.x device is visible. */
DF_API int df_device_check(int32_t* sm_count);

#ifdef __cplusplus
}
#endif
#endif /* DF_B200_H */
