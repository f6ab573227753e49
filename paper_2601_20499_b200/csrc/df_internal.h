// df_internal.h -- shared host-side helpers of libdfb200 (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "df_b200.h"

namespace dfb {

// Record a thread-local error message (printf-style) and return `code`.
int set_error(int code, const char* fmt, ...);
int set_cuda_error(const char* what, cudaError_t e);

// TMA descriptor for a row-major bf16 matrix [rows][width] (width 64 or 128),
// box = box_rows rows x 64 columns (128 bytes), SWIZZLE_128B, OOB -> zero.
int encode_rowmajor_bf16(CUtensorMap* map, const void* base, int64_t rows, int32_t width, int32_t box_rows = 128);

// General bf16 [rows][cols] matrix with leading dimension `ld` elements
// (cols, ld multiples of 8, i.e. 16-byte rows); box = box_rows x 64 columns,
// SWIZZLE_128B, OOB -> zero.
int encode_bf16_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int32_t box_rows);

// bf16 [depth][rows][cols] (contiguous), box = box_rows x 64 columns x 1, SWIZZLE_128B, OOB -> zero.
int encode_bf16_3d(CUtensorMap* map, const void* base, int64_t depth, int64_t rows, int64_t cols, int32_t box_rows);

// Multiprocessor count of the current device (148 on B200), cached.
int sm_count_cached();

}  // namespace dfb
