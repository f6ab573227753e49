// df_host.cpp -- host side of libdfb200: error state, TMA descriptor encoding,
// the greedy head classifier, device checks.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "df_internal.h"

namespace dfb {

static thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int set_cuda_error(const char* what, cudaError_t e) {
  return set_error(DF_E_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

// cuTensorMapEncodeTiled is a driver API entry point; fetch it through the
// runtime so the library links only the static CUDA runtime and loads on a
// machine without libcuda (CPU-only test hosts).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int encode_bf16_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int32_t box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(DF_E_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if (cols < 64 || cols % 8 || ld < cols || ld % 8)
    return set_error(DF_E_SHAPE, "tensor map cols %lld / ld %lld (need >= 64, multiples of 8)", (long long)cols,
                     (long long)ld);
  if (rows < 1 || rows > (int64_t(1) << 31)) return set_error(DF_E_SHAPE, "tensor map rows %lld", (long long)rows);
  if (box_rows < 1 || box_rows > 256) return set_error(DF_E_SHAPE, "tensor map box rows %d", box_rows);
  if (reinterpret_cast<uintptr_t>(base) & 15) return set_error(DF_E_ARG, "tensor map base not 16-byte aligned");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(DF_E_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", int(r));
  return DF_OK;
}

int encode_bf16_3d(CUtensorMap* map, const void* base, int64_t depth, int64_t rows, int64_t cols, int32_t box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(DF_E_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if (cols < 64 || cols % 8) return set_error(DF_E_SHAPE, "tensor map cols %lld", (long long)cols);
  if (rows < 1 || depth < 1 || rows * depth > (int64_t(1) << 31))
    return set_error(DF_E_SHAPE, "tensor map rows %lld x depth %lld", (long long)rows, (long long)depth);
  if (box_rows < 1 || box_rows > 256) return set_error(DF_E_SHAPE, "tensor map box rows %d", box_rows);
  if (reinterpret_cast<uintptr_t>(base) & 15) return set_error(DF_E_ARG, "tensor map base not 16-byte aligned");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(depth)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 2, static_cast<cuuint64_t>(rows * cols) * 2};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(DF_E_CUDA, "cuTensorMapEncodeTiled (3d) failed (CUresult %d)", int(r));
  return DF_OK;
}

int encode_rowmajor_bf16(CUtensorMap* map, const void* base, int64_t rows, int32_t width, int32_t box_rows) {
  if (width != 64 && width != 128) return set_error(DF_E_SHAPE, "tensor map width %d not 64/128", width);
  return encode_bf16_2d(map, base, rows, width, width, box_rows);
}

// numpy's float64 add.reduce of a contiguous 1-D array is one pairwise_sum
// over all n elements (numpy/_core/src/umath/loops_utils.h.src, PW_BLOCKSIZE
// 128, 8-way unroll); verified bitwise against np.sum in tests/test_host_cpu.py.
static double np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] += a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

static double np_sum(const std::vector<double>& v) {
  if (v.empty()) return 0.0;
  return np_pairwise_sum(v.data(), static_cast<int64_t>(v.size()));
}

}  // namespace dfb

using namespace dfb;

extern "C" const char* df_last_error(void) { return g_last_error.c_str(); }

extern "C" int df_version(void) { return 1; }

extern "C" int df_device_check(int32_t* sm_count) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error("cudaGetDevice", e);
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) return set_cuda_error("cudaGetDeviceProperties", e);
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (prop.major != 10)
    return set_error(DF_E_CUDA, "device %d is sm_%d%d; libdfb200 is built for sm_100a only", dev, prop.major,
                     prop.minor);
  return DF_OK;
}

extern "C" int df_kv_arena_maps(const void* k_base, const void* v_base, int64_t rows, int32_t head_dim,
                                uint8_t* out_maps) {
  if (!k_base || !v_base || !out_maps) return set_error(DF_E_ARG, "df_kv_arena_maps: null pointer");
  CUtensorMap maps[DF_MAPS_PER_ARENA];
  int rc = encode_rowmajor_bf16(&maps[0], k_base, rows, head_dim, 128);
  if (rc != DF_OK) return rc;
  rc = encode_rowmajor_bf16(&maps[1], v_base, rows, head_dim, 128);
  if (rc != DF_OK) return rc;
  rc = encode_rowmajor_bf16(&maps[2], k_base, rows, head_dim, 64);  // K halves of the CTA-pair kernel
  if (rc != DF_OK) return rc;
  std::memcpy(out_maps, maps, sizeof(maps));
  return DF_OK;
}

// head_programming.py:141-164.  cost = max(F_sink, F_neighbor); the n_dummy
// smallest costs (ties -> lower index, np.lexsort) become dummy; the rest are
// sink iff F_sink >= F_neighbor.  Objective = np.sum of retained values.
extern "C" int df_greedy_classify(const double* F, int64_t total, int64_t n_dummy, int8_t* classes_out,
                                  double* objective_out) {
  if (total < 0 || (total > 0 && (!F || !classes_out)))
    return set_error(DF_E_ARG, "df_greedy_classify: bad arguments");
  if (n_dummy < 0 || n_dummy > total)
    return set_error(DF_E_CONFIG, "n_dummy=%lld outside [0, %lld]", (long long)n_dummy, (long long)total);
  std::vector<double> cost(static_cast<size_t>(total));
  for (int64_t i = 0; i < total; ++i) {
    const double s = F[3 * i + 0], nb = F[3 * i + 1];
    cost[i] = (std::isnan(s) || std::isnan(nb)) ? NAN : (s > nb ? s : nb);  // np.maximum
  }
  std::vector<int64_t> order(static_cast<size_t>(total));
  std::iota(order.begin(), order.end(), 0);
  // np.lexsort((arange, cost)): ascending cost, NaN last, index breaks ties.
  std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
    const double a = cost[x], b = cost[y];
    if (std::isnan(a)) return false;
    if (std::isnan(b)) return true;
    return a < b;
  });
  std::vector<int8_t> codes(static_cast<size_t>(total));
  for (int64_t i = 0; i < total; ++i) codes[i] = (F[3 * i + 0] >= F[3 * i + 1]) ? 0 : 1;
  for (int64_t k = 0; k < n_dummy; ++k) codes[order[k]] = 2;
  std::vector<double> vals(static_cast<size_t>(total));
  for (int64_t i = 0; i < total; ++i) {
    const double cur = F[3 * i + 2];
    vals[i] = codes[i] == 0 ? F[3 * i + 0] + cur : codes[i] == 1 ? F[3 * i + 1] + cur : cur;
    classes_out[i] = codes[i];
  }
  if (objective_out) *objective_out = np_sum(vals);
  return DF_OK;
}
