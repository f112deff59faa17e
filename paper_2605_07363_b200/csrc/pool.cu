// K1: block pooling of indexer keys (pooling.py:57-84) and its decode update
// (pooling.py:87-115).
//
// CTAs per (B-key block, 32 head dims).  Each thread owns 8 head dims (one 16-byte bf16
// vector) of a strided sub-segment of the block, so every warp load is a
// coalesced 512-byte row span.  Three phases: sub-segment sums -> exclusive
// carry across sub-segments (smem) -> re-walk writing the in-block inclusive
// prefix sums P[s] (f32).  P lets a causal row t with a partial last block use
// mean(keys[bB : n_t]) = P[n_t-1] / (n_t - bB) without re-reading keys; the
// full-block means are written in f32 and as an exact 3-way bf16 split
// (hi, mid, lo) that the tcgen05 router consumes at f32-grade precision.
#include "common.cuh"
#include "ptx.cuh"

namespace misa {

__device__ __forceinline__ void split3_store(__nv_bfloat16* planes, int64_t planes_rows, int64_t b, int D, int dim,
                                             float x) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(hi);
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  const float r2 = r1 - __bfloat162float(mid);
  const __nv_bfloat16 lo = __float2bfloat16_rn(r2);
  planes[(0 * planes_rows + b) * D + dim] = hi;
  planes[(1 * planes_rows + b) * D + dim] = mid;
  planes[(2 * planes_rows + b) * D + dim] = lo;
}

// grid (blocks, D / 32): a CTA pools 32 head dims (4 x 16-byte vectors per key row) of one
// block over 64 sub-segments, so a layer launches blocks x D/32 CTAs (every SM busy even at
// 32 blocks) and each thread walks only ceil(B / 64) keys.
template <int D>
__global__ void __launch_bounds__(256) pool_kernel(const __nv_bfloat16* __restrict__ keys, int64_t L, int B,
                                                    float* __restrict__ prefix, float* __restrict__ pooled,
                                                    __nv_bfloat16* __restrict__ planes, int64_t planes_rows) {
  constexpr int CH = 4;            // threads per key row (32 dims of this CTA)
  constexpr int RP = 256 / CH;     // sub-segments
  __shared__ float sums[RP][32 + 1];
  const int b = blockIdx.x;
  const int d0 = blockIdx.y * 32;
  const int64_t start = (int64_t)b * B;
  const int len = (int)((start + B <= L) ? B : (L - start));
  const int sr = threadIdx.x / CH, ch = threadIdx.x % CH;
  // sub-segments sized from B, not from this block's length: a block's prefix sums then do
  // not depend on how many keys follow it (a partial last block gives the same P values as
  // the same keys followed by more keys or by zero padding, e.g. in a packed several-sequence
  // key buffer)
  const int seg = (B + RP - 1) / RP;
  const int s0 = sr * seg, s1 = min(len, s0 + seg);
  const __nv_bfloat16* kb = keys + start * D + d0 + ch * 8;

  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll 4
  for (int s = s0; s < s1; ++s) {
    const uint4 v = *reinterpret_cast<const uint4*>(kb + (int64_t)s * D);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      acc[2 * i] += f.x;
      acc[2 * i + 1] += f.y;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sums[sr][ch * 8 + i] = acc[i];
  __syncthreads();

  if (prefix) {
    float run[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) run[i] = 0.f;
    for (int r = 0; r < sr; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) run[i] += sums[r][ch * 8 + i];
#pragma unroll 4
    for (int s = s0; s < s1; ++s) {
      const uint4 v = *reinterpret_cast<const uint4*>(kb + (int64_t)s * D);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        run[2 * i] += f.x;
        run[2 * i + 1] += f.y;
      }
      float4* dst = reinterpret_cast<float4*>(prefix + (start + s) * D + d0 + ch * 8);
      dst[0] = make_float4(run[0], run[1], run[2], run[3]);
      dst[1] = make_float4(run[4], run[5], run[6], run[7]);
    }
  }

  if (len == B && sr == 0) {
    const float inv = 1.0f / (float)B;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float tot = 0.f;
      for (int r = 0; r < RP; ++r) tot += sums[r][ch * 8 + i];
      const float m = tot * inv;
      const int dim = d0 + ch * 8 + i;
      if (pooled) pooled[(int64_t)b * D + dim] = m;
      if (planes) split3_store(planes, planes_rows, b, D, dim, m);
    }
  }
}

template <int D>
__global__ void pool_append_kernel(const __nv_bfloat16* __restrict__ keys, int64_t s, int B, float* prefix,
                                   float* pooled, __nv_bfloat16* planes, int64_t planes_rows) {
  const int dim = threadIdx.x;
  if (dim >= D) return;
  const int pos = (int)(s % B);
  const int64_t b = s / B;
  float run = __bfloat162float(keys[s * D + dim]);
  if (pos > 0) run += prefix[(s - 1) * D + dim];
  prefix[s * D + dim] = run;
  if (pos == B - 1) {
    const float m = run / (float)B;
    if (pooled) pooled[b * D + dim] = m;
    if (planes && b < planes_rows) split3_store(planes, planes_rows, b, D, dim, m);
  }
}

}  // namespace misa

using namespace misa;

extern "C" int misa_pool_keys(const void* keys, int64_t n_keys, int head_dim, int block_size, float* prefix_sums,
                              float* pooled, void* pooled_planes, int64_t planes_rows, void* stream) {
  MISA_REQUIRE(keys, "null keys");
  MISA_REQUIRE(n_keys >= 1, "prefix must contain at least one key");
  MISA_REQUIRE(block_size >= 1, "block_size must be a positive integer, got %d", block_size);
  MISA_REQUIRE(head_dim == 64 || head_dim == 128, "head_dim must be padded to 64 or 128");
  const int64_t n_full = n_keys / block_size;
  MISA_REQUIRE(!pooled_planes || planes_rows >= n_full, "planes_rows %lld < full blocks %lld",
               (long long)planes_rows, (long long)n_full);
  cudaStream_t st = as_stream(stream);
  if (pooled_planes && planes_rows > n_full) {
    for (int p = 0; p < 3; ++p)
      MISA_CUDA_TRY(cudaMemsetAsync(static_cast<__nv_bfloat16*>(pooled_planes) + (p * planes_rows + n_full) * head_dim,
                                    0, (planes_rows - n_full) * head_dim * 2, st));
  }
  const int64_t nb = (n_keys + block_size - 1) / block_size;
  MISA_REQUIRE(nb < (int64_t(1) << 31), "too many blocks");
  auto* k = static_cast<const __nv_bfloat16*>(keys);
  auto* pl = static_cast<__nv_bfloat16*>(pooled_planes);
  if (head_dim == 128)
    pool_kernel<128><<<dim3((unsigned)nb, 128 / 32), 256, 0, st>>>(k, n_keys, block_size, prefix_sums, pooled, pl, planes_rows);
  else
    pool_kernel<64><<<dim3((unsigned)nb, 64 / 32), 256, 0, st>>>(k, n_keys, block_size, prefix_sums, pooled, pl, planes_rows);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_pool_append(const void* keys, int64_t n_keys_before, int head_dim, int block_size,
                                float* prefix_sums, float* pooled, void* pooled_planes, int64_t planes_rows,
                                void* stream) {
  MISA_REQUIRE(keys && prefix_sums, "null pointer");
  MISA_REQUIRE(n_keys_before >= 0 && block_size >= 1, "bad append arguments");
  MISA_REQUIRE(head_dim == 64 || head_dim == 128, "head_dim must be padded to 64 or 128");
  cudaStream_t st = as_stream(stream);
  auto* k = static_cast<const __nv_bfloat16*>(keys);
  auto* pl = static_cast<__nv_bfloat16*>(pooled_planes);
  if (head_dim == 128)
    pool_append_kernel<128><<<1, 128, 0, st>>>(k, n_keys_before, block_size, prefix_sums, pooled, pl, planes_rows);
  else
    pool_append_kernel<64><<<1, 64, 0, st>>>(k, n_keys_before, block_size, prefix_sums, pooled, pl, planes_rows);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}
