// df_kv.cu -- KV ring data movement and the DHP score finalisation.
//
//   df_kv_append  kv_cache.py:177-185 (append of the current frame into its
//                 ring slot; one launch for all heads of a layer)
//   df_kv_pack    kv_cache.py:199-201 rebuild / 187-197 _evict: compaction
//                 of retained frames into the packed per-class layout
//   df_scores_finalize  profiler.py:118-129 mean region mass over rows
//
// Both copy kernels move 16-byte vectors with 8 independent loads in flight
// per thread (HBM-bound; roofline = bytes read + written over measured copy
// bandwidth).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "df_internal.h"

namespace dfb {

constexpr int kCopyThreads = 256;
constexpr int kCopyUnroll = 8;
constexpr int64_t kChunkVecs = kCopyThreads * kCopyUnroll;  // 16-byte vectors per CTA chunk (32 KB)

struct Seg {
  const uint8_t* src;
  uint8_t* dst;
  int64_t rows;
  int64_t src_ld;
  int64_t dst_ld;
  int64_t row_bytes;
};

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Copy chunk `chunk` (kChunkVecs vectors) of one segment.
__device__ __forceinline__ void copy_chunk(const Seg& s, int64_t chunk) {
  const int64_t vec_per_row = s.row_bytes >> 4;
  const int64_t total = vec_per_row * s.rows;
  const int64_t v0 = chunk * kChunkVecs + threadIdx.x;
  const bool contiguous = (s.src_ld == s.row_bytes) && (s.dst_ld == s.row_bytes);
  int4 buf[kCopyUnroll];
  int64_t so[kCopyUnroll], dof[kCopyUnroll];
#pragma unroll
  for (int u = 0; u < kCopyUnroll; ++u) {
    const int64_t v = v0 + u * kCopyThreads;
    if (contiguous) {
      so[u] = v << 4;
      dof[u] = v << 4;
    } else {
      const int64_t r = v / vec_per_row, c = (v - r * vec_per_row) << 4;
      so[u] = r * s.src_ld + c;
      dof[u] = r * s.dst_ld + c;
    }
    if (v < total) buf[u] = ld_stream(reinterpret_cast<const int4*>(s.src + so[u]));
  }
#pragma unroll
  for (int u = 0; u < kCopyUnroll; ++u) {
    const int64_t v = v0 + u * kCopyThreads;
    if (v < total) *reinterpret_cast<int4*>(s.dst + dof[u]) = buf[u];
  }
}

struct AppendParams {
  int32_t n;
  int32_t chunks_per_seg;
  Seg segs[DF_MAX_APPEND_SEGS];
};

__global__ void __launch_bounds__(kCopyThreads) df_append_kernel(const __grid_constant__ AppendParams p) {
  const int seg = blockIdx.y;
  const Seg& s = p.segs[seg];
  const int64_t total = (s.row_bytes >> 4) * s.rows;
  for (int64_t c = blockIdx.x; c * kChunkVecs < total; c += gridDim.x) copy_chunk(s, c);
}

__global__ void __launch_bounds__(kCopyThreads)
    df_pack_kernel(const Seg* __restrict__ segs, const int64_t* __restrict__ prefix, int32_t n_segs) {
  // prefix[i] = first CTA of segment i; find the segment of this CTA.
  const int64_t b = blockIdx.x;
  int lo = 0, hi = n_segs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(prefix + mid) <= b) lo = mid; else hi = mid - 1;
  }
  const Seg s = segs[lo];
  copy_chunk(s, b - __ldg(prefix + lo));
}

__global__ void df_scores_kernel(const float* __restrict__ rows, const uint8_t* __restrict__ sampled, int hw,
                                 double* __restrict__ F) {
  // Deterministic: fixed per-thread row partition, fixed-shape tree reduce.
  __shared__ double red[4][256];
  const int h = blockIdx.x;
  double a0 = 0, a1 = 0, a2 = 0, cnt = 0;
  for (int r = threadIdx.x; r < hw; r += blockDim.x) {
    if (sampled[r]) {
      // renormalise each row in fp64 so every score row sums to 1 exactly
      // (the kernel's per-region and total sums round independently in fp32)
      const float* x = rows + (static_cast<int64_t>(h) * hw + r) * 3;
      const double x0 = x[0], x1 = x[1], x2 = x[2];
      const double inv = 1.0 / (x0 + x1 + x2);
      a0 += x0 * inv;
      a1 += x1 * inv;
      a2 += x2 * inv;
      cnt += 1;
    }
  }
  red[0][threadIdx.x] = a0;
  red[1][threadIdx.x] = a1;
  red[2][threadIdx.x] = a2;
  red[3][threadIdx.x] = cnt;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int k = 0; k < 4; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 3) {
    const double n = red[3][0];
    F[h * 3 + threadIdx.x] = n > 0 ? red[threadIdx.x][0] / n : 0.0;
  }
}

static int check_seg(const df_copy_seg& s, int i) {
  if (!s.src || !s.dst) return set_error(DF_E_ARG, "copy segment %d: null pointer", i);
  if (s.rows < 0 || s.row_bytes < 0) return set_error(DF_E_ARG, "copy segment %d: negative size", i);
  if ((s.row_bytes | s.src_ld | s.dst_ld) & 15)
    return set_error(DF_E_ARG, "copy segment %d: row bytes / strides must be multiples of 16", i);
  if ((reinterpret_cast<uintptr_t>(s.src) | reinterpret_cast<uintptr_t>(s.dst)) & 15)
    return set_error(DF_E_ARG, "copy segment %d: pointers must be 16-byte aligned", i);
  if (s.rows > 1 && (s.src_ld < s.row_bytes || s.dst_ld < s.row_bytes))
    return set_error(DF_E_ARG, "copy segment %d: stride smaller than row", i);
  return DF_OK;
}

static Seg to_seg(const df_copy_seg& s) {
  Seg d;
  d.src = static_cast<const uint8_t*>(s.src);
  d.dst = static_cast<uint8_t*>(s.dst);
  d.rows = s.rows;
  d.row_bytes = s.row_bytes;
  d.src_ld = s.src_ld;
  d.dst_ld = s.dst_ld;
  if (s.src_ld == s.row_bytes && s.dst_ld == s.row_bytes) {  // collapse to one long row
    d.row_bytes = s.row_bytes * s.rows;
    d.rows = s.rows > 0 ? 1 : 0;
    d.src_ld = d.dst_ld = d.row_bytes;
  }
  return d;
}

bool append_overlap() {  // DF_APPEND_PDL=0 turns the programmatic dependent launch off (dev A/B)
  static const bool on = [] {
    const char* env = std::getenv("DF_APPEND_PDL");
    return !(env && env[0] == '0');
  }();
  return on;
}

}  // namespace dfb

using namespace dfb;

static int kv_append(const df_copy_seg* segs, int32_t n, void* stream, bool overlapped);

extern "C" int df_kv_append(const df_copy_seg* segs, int32_t n, void* stream) {
  return kv_append(segs, n, stream, false);
}

extern "C" int df_kv_append_overlapped(const df_copy_seg* segs, int32_t n, void* stream) {
  return kv_append(segs, n, stream, append_overlap());
}

static int kv_append(const df_copy_seg* segs, int32_t n, void* stream, bool overlapped) {
  if (n < 0 || n > DF_MAX_APPEND_SEGS || (n > 0 && !segs))
    return set_error(DF_E_ARG, "df_kv_append: n_segs %d outside [0, %d]", n, DF_MAX_APPEND_SEGS);
  if (n == 0) return DF_OK;
  AppendParams p;
  std::memset(&p, 0, sizeof(p));
  p.n = n;
  int64_t max_vecs = 0;
  for (int i = 0; i < n; ++i) {
    int rc = check_seg(segs[i], i);
    if (rc != DF_OK) return rc;
    p.segs[i] = to_seg(segs[i]);
    const int64_t v = (p.segs[i].row_bytes >> 4) * p.segs[i].rows;
    if (v > max_vecs) max_vecs = v;
  }
  if (max_vecs == 0) return DF_OK;
  int64_t chunks = (max_vecs + kChunkVecs - 1) / kChunkVecs;
  if (chunks > 65535) chunks = 65535;
  dim3 grid(static_cast<unsigned>(chunks), static_cast<unsigned>(n));
  // df_kv_append_overlapped: programmatic dependent launch.  When the previous
  // kernel on the stream is a df_attn_fwd launch (every CTA of which signals
  // griddepcontrol.launch_dependents as it starts), this copy -- the next layer's
  // current frame into its ring, which that launch does not read -- runs on the
  // SMs the FMHA's last wave leaves idle instead of after it drains.  After any
  // other kernel it starts at that kernel's completion, as a plain launch would.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kCopyThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = overlapped ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, df_append_kernel, p);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("df_append_kernel launch", e);
  return DF_OK;
}

extern "C" int df_kv_pack_plan(const df_copy_seg* segs, int32_t n, int64_t* prefix, int64_t* total_blocks) {
  if (n < 0 || (n > 0 && (!segs || !prefix)) || !total_blocks) return set_error(DF_E_ARG, "df_kv_pack_plan: bad args");
  int64_t acc = 0;
  for (int i = 0; i < n; ++i) {
    int rc = check_seg(segs[i], i);
    if (rc != DF_OK) return rc;
    const Seg s = to_seg(segs[i]);
    prefix[i] = acc;
    acc += ((s.row_bytes >> 4) * s.rows + kChunkVecs - 1) / kChunkVecs;
  }
  if (n >= 0 && prefix) prefix[n] = acc;
  *total_blocks = acc;
  return DF_OK;
}

extern "C" int df_kv_pack(const df_copy_seg* segs_dev, const int64_t* prefix_dev, int32_t n, int64_t total_blocks,
                          void* stream) {
  static_assert(sizeof(df_copy_seg) == sizeof(Seg), "segment layouts differ");
  if (n < 0 || total_blocks < 0 || (n > 0 && (!segs_dev || !prefix_dev)))
    return set_error(DF_E_ARG, "df_kv_pack: bad arguments");
  if (n == 0 || total_blocks == 0) return DF_OK;
  if (total_blocks > INT32_MAX) return set_error(DF_E_ARG, "df_kv_pack: too many blocks");
  // Device segments are df_copy_seg already normalised by the caller through
  // df_kv_pack_plan's rules (contiguous runs collapse in-kernel as well).
  df_pack_kernel<<<static_cast<unsigned>(total_blocks), kCopyThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const Seg*>(segs_dev), prefix_dev, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("df_pack_kernel launch", e);
  return DF_OK;
}

extern "C" int df_scores_finalize(const float* rows, const uint8_t* sampled, int32_t num_heads, int32_t hw,
                                  double* F, void* stream) {
  if (!rows || !sampled || !F || num_heads < 1 || hw < 1) return set_error(DF_E_ARG, "df_scores_finalize: bad args");
  df_scores_kernel<<<num_heads, 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, sampled, hw, F);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("df_scores_kernel launch", e);
  return DF_OK;
}
