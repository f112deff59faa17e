// Row-wise FP8 (e4m3) quantization for the upstream indexer projections (SURVEY §8f row 4:
// "upstream indexer projections (FP8, signed weights)"; PAPER.md:98 — DeepSeek-V3.2 runs its
// indexer in FP8).  Outside the reference: it feeds the projections that
// produce the indexer's q / k / w, which then enter the bf16 parity path unchanged.
//
//   scale[r] = amax_r / 448,   out[r][c] = e4m3(x[r][c] / scale[r])   (round to nearest,
//   saturating; an all-zero row gets scale 1 and zeros)
//
// One CTA per row (grid-strided): a 16-byte-vector amax pass, a block max, then a second pass
// that re-reads the row from L1/L2 and writes 8 e4m3 bytes per vector.  HBM-bound: 2 B read
// + 1 B written per element.  Rows are activations (per token) or weights (per output
// channel); the GEMMs themselves are cuBLASLt row-wise-scaled FP8 (projections.py).
#include <cuda_bf16.h>

#include "common.cuh"

namespace misa {

constexpr int kQuantThreads = 128;

__device__ __forceinline__ uint16_t e4m3x2(float hi, float lo) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

__global__ void __launch_bounds__(kQuantThreads) quant_rows_fp8_kernel(const __nv_bfloat16* __restrict__ x,
                                                                        int64_t n_rows, int cols,
                                                                        uint8_t* __restrict__ out,
                                                                        float* __restrict__ scales) {
  __shared__ float red[kQuantThreads / 32];
  const int nv = cols / 8;  // 16-byte vectors per row
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const uint4* row = reinterpret_cast<const uint4*>(x + r * cols);
    float amax = 0.f;
    for (int v = threadIdx.x; v < nv; v += kQuantThreads) {
      const uint4 u = __ldg(row + v);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
    __syncthreads();
    amax = red[0];
#pragma unroll
    for (int w = 1; w < kQuantThreads / 32; ++w) amax = fmaxf(amax, red[w]);
    const float scale = amax > 0.f ? amax / 448.f : 1.f;
    const float inv = amax > 0.f ? 448.f / amax : 1.f;
    if (threadIdx.x == 0) scales[r] = scale;
    uint2* orow = reinterpret_cast<uint2*>(out + r * cols);
    for (int v = threadIdx.x; v < nv; v += kQuantThreads) {
      const uint4 u = __ldg(row + v);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
      uint16_t p[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        p[j] = e4m3x2(f.y * inv, f.x * inv);  // low byte = the lower-addressed element
      }
      orow[v] = make_uint2((uint32_t)p[0] | ((uint32_t)p[1] << 16), (uint32_t)p[2] | ((uint32_t)p[3] << 16));
    }
    __syncthreads();  // red[] is rewritten by the next row
  }
}

}  // namespace misa

using namespace misa;

extern "C" int misa_quant_rows_fp8(const void* x, int64_t n_rows, int cols, void* out, float* scales, void* stream) {
  MISA_REQUIRE(x && out && scales, "null pointer");
  MISA_REQUIRE(n_rows >= 0 && cols > 0 && cols % 8 == 0, "cols must be a positive multiple of 8, got %d", cols);
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 7) == 0,
               "x must be 16-byte and out 8-byte aligned");
  if (n_rows == 0) return MISA_OK;
  const int64_t cap = (int64_t)sm_count() * 16;
  const unsigned grid = (unsigned)(n_rows < cap ? n_rows : cap);
  quant_rows_fp8_kernel<<<grid, kQuantThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), n_rows, cols, static_cast<uint8_t*>(out), scales);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}
