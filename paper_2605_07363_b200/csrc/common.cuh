// Host-side helpers shared by the C-ABI translation units: error state,
// TMA tensor-map encoding through the driver entry point, checks.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/misa_b200.h"

namespace misa {

void set_error(const char* fmt, ...);

#define MISA_REQUIRE(cond, ...)        \
  do {                                 \
    if (!(cond)) {                     \
      ::misa::set_error(__VA_ARGS__);  \
      return MISA_EINVAL;              \
    }                                  \
  } while (0)

#define MISA_CUDA_TRY(expr)                                                                     \
  do {                                                                                          \
    cudaError_t e__ = (expr);                                                                   \
    if (e__ != cudaSuccess) {                                                                   \
      ::misa::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e__), __FILE__, __LINE__); \
      return MISA_ECUDA;                                                                        \
    }                                                                                           \
  } while (0)

#define MISA_LAUNCH_CHECK() MISA_CUDA_TRY(cudaGetLastError())

// 2-D bf16 tensor map: rows of `row_elems` (inner, contiguous) elements, `n_rows`
// rows `row_stride_elems` apart, box {64, box_rows}, 128-B swizzle.
int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t row_elems, uint64_t n_rows,
                      uint64_t row_stride_elems, uint32_t box_rows);

int make_tmap_bf16_gather(CUtensorMap* map, const void* base, uint64_t row_elems, uint64_t n_rows);
int sm_count();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kTileKeys = 128;   // keys per MMA tile (UMMA M)
constexpr int kTileCols = 256;   // (query, head) columns per MMA tile (UMMA N)
constexpr int kQuadrants = 4;    // TMEM lane quadrants / epilogue warps

}  // namespace misa
