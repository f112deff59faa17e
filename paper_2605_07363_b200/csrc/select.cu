// K4: exact top-k selection (dsa.py:64-92) for the fused streaming selector.
//
// The reference's rule is argsort(-scores, kind="stable")[:k] then sort: the
// k largest scores, ties to the smaller index, returned ascending.  Every
// kernel here implements exactly that order, (score desc, index asc), with a
// block-wide MSD radix select over monotone u32 keys (-0.0 == +0.0):
//   1. skip the common high bits of all keys (one OR-reduction),
//   2. 8-bit digit passes with warp-aggregated smem histograms until the k-th
//      key v is pinned (cnt_gt keys are strictly greater),
//   3. if the keys equal to v over-fill the budget, a second radix select on
//      the complemented index picks the smallest indices among the ties,
//   4. the selected indices are bitonic-sorted ascending in smem.
//
// misa_select_threshold  one CTA per row over the sampled scores (tau)
// misa_select_topk       one CTA per row over the filtered candidates (staged in smem)
// misa_select_dense      one CTA per row over a dense score row (global passes)
// misa_merge_topk        one CTA per row over the gathered per-GPU top-k lists
#include "common.cuh"
#include "ptx.cuh"

namespace misa {

constexpr int kSelThreads = 512;

struct SelShared {
  uint32_t hist[256];
  uint32_t red[32];
  int info[8];
};

__device__ __forceinline__ uint32_t block_or(uint32_t v, SelShared& sh) {
  v = __reduce_or_sync(0xffffffffu, v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh.red[w] = v;
  __syncthreads();
  if (w == 0) {
    uint32_t x = (l < (int)(blockDim.x >> 5)) ? sh.red[l] : 0u;
    x = __reduce_or_sync(0xffffffffu, x);
    if (l == 0) sh.red[0] = x;
  }
  __syncthreads();
  const uint32_t r = sh.red[0];
  __syncthreads();
  return r;
}

// Find the j-th largest (1-indexed, j <= N) among keys key_of(i), i < N.
// Returns v; *j_rem = rank of the target among keys == v (1..cnt_eq); *cnt_eq.
template <typename KeyFn>
__device__ uint32_t radix_select(KeyFn key_of, int N, int j, SelShared& sh, int* j_rem_out, int* cnt_eq_out) {
  const uint32_t first = key_of(0);
  uint32_t diff = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) diff |= key_of(i) ^ first;
  diff = block_or(diff, sh);
  if (diff == 0) {
    *j_rem_out = j;
    *cnt_eq_out = N;
    return first;
  }
  int hi = 31 - __clz(diff);
  uint32_t prefix = (hi == 31) ? 0u : (first & ~((2u << hi) - 1u));
  int j_rem = j;
  int cnt_eq = 0;
  const uint32_t lane_lt = ptx::lanemask_lt();
  (void)lane_lt;
  while (hi >= 0) {
    const int lo = hi >= 7 ? hi - 7 : 0;
    const int width = hi - lo + 1;
    const uint32_t dmask = (width == 32) ? 0xffffffffu : ((1u << width) - 1u);
    const uint32_t mhi = (hi == 31) ? 0u : ~((2u << hi) - 1u);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh.hist[i] = 0;
    __syncthreads();
    // warp-uniform trip count so the aggregation below can use full-mask intrinsics
    const int trips = (N + blockDim.x - 1) / blockDim.x;
    for (int tr = 0; tr < trips; ++tr) {
      const int i = tr * blockDim.x + threadIdx.x;
      bool ok = false;
      uint32_t d = 0;
      if (i < N) {
        const uint32_t k = key_of(i);
        ok = (k & mhi) == (prefix & mhi);
        d = (k >> lo) & dmask;
      }
      const uint32_t act = __ballot_sync(0xffffffffu, ok);
      if (ok) {
        const uint32_t peers = __match_any_sync(act, d);
        if ((__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&sh.hist[d], __popc(peers));
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // lane l owns bins [8l, 8l+8) counted from the top digit down
      const int l = threadIdx.x;
      const int nb = (int)dmask + 1;  // bins in use (<= 256)
      uint32_t c[8];
      uint32_t tot = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int bin = nb - 1 - (8 * l + q);
        c[q] = bin >= 0 ? sh.hist[bin] : 0u;
        tot += c[q];
      }
      uint32_t incl = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (l >= off) incl += y;
      }
      const uint32_t excl = incl - tot;
      const bool here = (excl < (uint32_t)j_rem) && ((uint32_t)j_rem <= incl);
      if (here) {
        uint32_t above = excl;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if ((uint32_t)j_rem <= above + c[q]) {
            sh.info[0] = nb - 1 - (8 * l + q);
            sh.info[1] = (int)above;
            sh.info[2] = (int)c[q];
            break;
          }
          above += c[q];
        }
      }
    }
    __syncthreads();
    const int dsel = sh.info[0];
    j_rem -= sh.info[1];
    cnt_eq = sh.info[2];
    prefix |= (uint32_t)dsel << lo;
    __syncthreads();
    hi = lo - 1;
  }
  *j_rem_out = j_rem;
  *cnt_eq_out = cnt_eq;
  return prefix;
}

// Selected set = keys > v, plus keys == v with index <= idx_thr.  Resolves idx_thr.
template <typename KeyFn, typename IdxFn>
__device__ void select_rule(KeyFn key_of, IdxFn idx_of, int N, int kk, SelShared& sh, uint32_t* v_out,
                            int* idx_thr_out) {
  int j_rem, cnt_eq;
  const uint32_t v = radix_select(key_of, N, kk, sh, &j_rem, &cnt_eq);
  int idx_thr = 0x7fffffff;
  if (j_rem < cnt_eq) {
    int jr2, ce2;
    auto tie_key = [&](int i) -> uint32_t { return key_of(i) == v ? ~(uint32_t)idx_of(i) : 0u; };
    const uint32_t v2 = radix_select(tie_key, N, j_rem, sh, &jr2, &ce2);
    idx_thr = (int)~v2;
  }
  *v_out = v;
  *idx_thr_out = idx_thr;
}

// Bitonic sort of n_pow2 u64 in smem, ascending.
__device__ void bitonic_sort_u64(uint64_t* a, int n_pow2) {
  for (int k = 2; k <= n_pow2; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const uint64_t x = a[i], y = a[ixj];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Collect the selected (idx, score) pairs as u64 = idx << 32 | score_bits, sort, write.
template <typename KeyFn, typename IdxFn>
__device__ void collect_sorted_write(KeyFn key_of, IdxFn idx_of, int N, int kk, uint32_t v, int idx_thr,
                                     uint64_t* buf, int* counter, int32_t* out_idx, float* out_score, int k_out) {
  const int np2 = next_pow2(kk);
  for (int i = threadIdx.x; i < np2; i += blockDim.x) buf[i] = ~0ull;
  if (threadIdx.x == 0) *counter = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const uint32_t k = key_of(i);
    const int ix = idx_of(i);
    if (k > v || (k == v && ix <= idx_thr)) {
      const int pos = atomicAdd(counter, 1);
      if (pos < kk) buf[pos] = (static_cast<uint64_t>(static_cast<uint32_t>(ix)) << 32) | __float_as_uint(key_float(k));
    }
  }
  __syncthreads();
  bitonic_sort_u64(buf, np2);
  for (int i = threadIdx.x; i < k_out; i += blockDim.x) {
    if (i < kk) {
      out_idx[i] = (int32_t)(buf[i] >> 32);
      if (out_score) out_score[i] = __uint_as_float((uint32_t)buf[i]);
    } else {
      out_idx[i] = -1;
      if (out_score) out_score[i] = -INFINITY;
    }
  }
}

// ---------------------------------------------------------------- tau ----
__global__ void __launch_bounds__(kSelThreads) threshold_kernel(const float* __restrict__ s, int64_t ld,
                                                                const int32_t* __restrict__ prefix_len, int T,
                                                                int stride, int k, float beta, int64_t append_all,
                                                                float* __restrict__ tau) {
  __shared__ SelShared sh;
  const int t = blockIdx.x;
  const int n = prefix_len[t];
  if (n <= append_all || n <= k) {
    if (threadIdx.x == 0) tau[t] = -INFINITY;
    return;
  }
  const int m = (n + stride - 1) / stride;
  long long jj = (long long)ceilf(beta * (float)k * (float)m / (float)n);
  if (jj < 1) jj = 1;
  if (jj > m) jj = m;
  const float* row = s + (int64_t)t * ld;
  auto key_of = [&](int i) -> uint32_t { return float_key(row[i]); };
  int jr, ce;
  const uint32_t v = radix_select(key_of, m, (int)jj, sh, &jr, &ce);
  if (threadIdx.x == 0) tau[t] = key_float(v);
}

// -------------------------------------------------- candidates -> top-k ----
__global__ void __launch_bounds__(kSelThreads) topk_kernel(const uint64_t* __restrict__ cand,
                                                           const int32_t* __restrict__ cand_count, int cap,
                                                           const int32_t* __restrict__ prefix_len, int T, int k,
                                                           int32_t* __restrict__ topk, int64_t topk_ld,
                                                           float* __restrict__ topk_scores, int32_t* __restrict__ flags,
                                                           int staged_cap) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ SelShared sh;
  __shared__ int counter;
  const int t = blockIdx.x;
  const int n = prefix_len[t];
  int32_t* out = topk + (int64_t)t * topk_ld;
  float* outs = topk_scores ? topk_scores + (int64_t)t * topk_ld : nullptr;
  if (n <= k) {  // topk_tokens keeps every prefix token when k >= L (dsa.py:73)
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      out[i] = i < n ? i : -1;
      if (outs && i >= n) outs[i] = -INFINITY;
    }
    if (threadIdx.x == 0 && flags) flags[t] = 0;
    return;
  }
  int cnt[kQuadrants];
  int total = 0;
  bool overflow = false;
#pragma unroll
  for (int q = 0; q < kQuadrants; ++q) {
    cnt[q] = cand_count[(int64_t)t * kQuadrants + q];
    overflow |= cnt[q] > cap;
    total += cnt[q] < cap ? cnt[q] : cap;
  }
  const int kk = k;  // n > k here
  if (overflow || total < kk || total > staged_cap) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) out[i] = -1;
    if (threadIdx.x == 0 && flags) flags[t] = overflow || total > staged_cap ? MISA_FLAG_OVERFLOW : MISA_FLAG_UNDERFLOW;
    return;
  }
  uint32_t* skey = reinterpret_cast<uint32_t*>(dsm);
  int32_t* sidx = reinterpret_cast<int32_t*>(dsm + (size_t)staged_cap * 4);
  uint64_t* buf = reinterpret_cast<uint64_t*>(dsm + (size_t)staged_cap * 8);
  int off = 0;
#pragma unroll
  for (int q = 0; q < kQuadrants; ++q) {
    const uint64_t* src = cand + ((int64_t)t * kQuadrants + q) * cap;
    for (int i = threadIdx.x; i < cnt[q]; i += blockDim.x) {
      const uint64_t c = src[i];
      skey[off + i] = float_key(__uint_as_float((uint32_t)c));
      sidx[off + i] = (int32_t)(c >> 32);
    }
    off += cnt[q];
  }
  __syncthreads();
  auto key_of = [&](int i) -> uint32_t { return skey[i]; };
  auto idx_of = [&](int i) -> int { return sidx[i]; };
  uint32_t v;
  int idx_thr;
  select_rule(key_of, idx_of, total, kk, sh, &v, &idx_thr);
  collect_sorted_write(key_of, idx_of, total, kk, v, idx_thr, buf, &counter, out, outs, k);
  if (threadIdx.x == 0 && flags) flags[t] = 0;
}

// ------------------------------------------------------- dense rows ----
__global__ void __launch_bounds__(kSelThreads) dense_kernel(const float* __restrict__ s, int64_t ld,
                                                            const int32_t* __restrict__ idx, int64_t idx_ld,
                                                            const int32_t* __restrict__ row_len,
                                                            const int32_t* __restrict__ rows, int k,
                                                            int32_t* __restrict__ topk, int64_t topk_ld,
                                                            float* __restrict__ topk_scores) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ SelShared sh;
  __shared__ int counter;
  const int r = rows ? rows[blockIdx.x] : blockIdx.x;
  const int n = row_len[r];
  const float* row = s + (int64_t)r * ld;
  const int32_t* irow = idx ? idx + (int64_t)r * idx_ld : nullptr;
  int32_t* out = topk + (int64_t)r * topk_ld;
  float* outs = topk_scores ? topk_scores + (int64_t)r * topk_ld : nullptr;
  uint64_t* buf = reinterpret_cast<uint64_t*>(dsm);
  auto key_of = [&](int i) -> uint32_t { return float_key(row[i]); };
  auto idx_of = [&](int i) -> int { return irow ? irow[i] : i; };
  const int kk = n < k ? n : k;
  if (kk <= 0) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      out[i] = -1;
      if (outs) outs[i] = -INFINITY;
    }
    return;
  }
  uint32_t v = 0;
  int idx_thr = 0x7fffffff;
  if (kk < n) select_rule(key_of, idx_of, n, kk, sh, &v, &idx_thr);
  collect_sorted_write(key_of, idx_of, n, kk, v, idx_thr, buf, &counter, out, outs, k);
}

// -------------------------------------------------- multi-GPU merge ----
__global__ void __launch_bounds__(kSelThreads) merge_kernel(const float* __restrict__ ps, const int32_t* __restrict__ pi,
                                                            int n_parts, int64_t part_stride, int k_in, int k,
                                                            int32_t* __restrict__ topk, int64_t topk_ld) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ SelShared sh;
  __shared__ int counter;
  const int t = blockIdx.x;
  const int N = n_parts * k_in;
  auto at = [&](int i) -> int64_t { return (int64_t)(i / k_in) * part_stride + (int64_t)t * k_in + (i % k_in); };
  // -1 entries (short local lists) rank below every real candidate
  auto key_of = [&](int i) -> uint32_t { return pi[at(i)] < 0 ? 0u : float_key(ps[at(i)]); };
  auto idx_of = [&](int i) -> int { const int x = pi[at(i)]; return x < 0 ? 0x7fffffff : x; };
  int valid = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) valid += pi[at(i)] >= 0;
  valid = __reduce_add_sync(0xffffffffu, valid);
  __shared__ int vsum;
  if (threadIdx.x == 0) vsum = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(&vsum, valid);
  __syncthreads();
  const int kk = vsum < k ? vsum : k;
  int32_t* out = topk + (int64_t)t * topk_ld;
  uint64_t* buf = reinterpret_cast<uint64_t*>(dsm);
  if (kk <= 0) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) out[i] = -1;
    return;
  }
  uint32_t v = 0;
  int idx_thr = 0x7fffffff;
  if (kk < vsum) {
    select_rule(key_of, idx_of, N, kk, sh, &v, &idx_thr);
  } else {
    v = 1u;  // every valid entry (key >= 1 since real keys are never 0) is kept
    idx_thr = 0x7ffffffe;
  }
  collect_sorted_write(key_of, idx_of, N, kk, v, idx_thr, buf, &counter, out, nullptr, k);
}

static size_t sort_bytes(int k) {
  size_t p = 1;
  while ((int)p < k) p <<= 1;
  return p * 8;
}

}  // namespace misa

using namespace misa;

extern "C" int misa_select_threshold(const float* sample_scores, int64_t ld, const int32_t* prefix_len,
                                     int64_t n_rows, int key_stride, int k, float beta, int64_t append_all_len,
                                     float* tau, void* stream) {
  MISA_REQUIRE(sample_scores && prefix_len && tau, "null pointer");
  MISA_REQUIRE(k >= 1 && key_stride >= 1 && beta > 0.f && n_rows >= 1, "bad threshold arguments");
  threshold_kernel<<<(unsigned)n_rows, kSelThreads, 0, as_stream(stream)>>>(sample_scores, ld, prefix_len,
                                                                            (int)n_rows, key_stride, k, beta,
                                                                            append_all_len, tau);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_select_topk(const uint64_t* cand, const int32_t* cand_count, int cap, const int32_t* prefix_len,
                                int64_t n_rows, int k, int32_t* topk, int64_t topk_ld, float* topk_scores,
                                int32_t* flags, void* stream) {
  MISA_REQUIRE(cand && cand_count && prefix_len && topk, "null pointer");
  MISA_REQUIRE(k >= 1 && cap >= 1 && topk_ld >= k && n_rows >= 1, "bad top-k arguments");
  // stage up to 4*cap candidates (keys + indices) plus the sort buffer in smem
  int staged_cap = 4 * cap;
  size_t bytes = (size_t)staged_cap * 8 + sort_bytes(k);
  const size_t limit = 200 * 1024;
  if (bytes > limit) {
    staged_cap = (int)((limit - sort_bytes(k)) / 8);
    bytes = (size_t)staged_cap * 8 + sort_bytes(k);
  }
  MISA_REQUIRE(staged_cap >= k, "k=%d too large for the staged selector", k);
  MISA_CUDA_TRY(cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  topk_kernel<<<(unsigned)n_rows, kSelThreads, bytes, as_stream(stream)>>>(
      cand, cand_count, cap, prefix_len, (int)n_rows, k, topk, topk_ld, topk_scores, flags, staged_cap);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_select_dense(const float* scores, int64_t ld, const int32_t* idx, int64_t idx_ld,
                                 const int32_t* row_len, const int32_t* rows, int64_t n_rows, int k, int32_t* topk,
                                 int64_t topk_ld, float* topk_scores, void* stream) {
  MISA_REQUIRE(scores && row_len && topk, "null pointer");
  MISA_REQUIRE(k >= 1 && topk_ld >= k, "bad k");
  if (n_rows <= 0) return MISA_OK;
  const size_t bytes = sort_bytes(k);
  MISA_REQUIRE(bytes <= 200 * 1024, "k too large");
  MISA_CUDA_TRY(cudaFuncSetAttribute(dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  dense_kernel<<<(unsigned)n_rows, kSelThreads, bytes, as_stream(stream)>>>(scores, ld, idx, idx_ld, row_len, rows, k,
                                                                            topk, topk_ld, topk_scores);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_merge_topk(const float* part_scores, const int32_t* part_idx, int n_parts, int64_t part_stride,
                               int64_t n_rows, int k_in, int k, int32_t* topk, int64_t topk_ld, void* stream) {
  MISA_REQUIRE(part_scores && part_idx && topk, "null pointer");
  MISA_REQUIRE(n_parts >= 1 && k_in >= 1 && k >= 1 && topk_ld >= k, "bad merge arguments");
  if (n_rows <= 0) return MISA_OK;
  const size_t bytes = sort_bytes(k);
  MISA_REQUIRE(bytes <= 200 * 1024, "k too large");
  MISA_CUDA_TRY(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  merge_kernel<<<(unsigned)n_rows, kSelThreads, bytes, as_stream(stream)>>>(part_scores, part_idx, n_parts,
                                                                            part_stride, k_in, k, topk, topk_ld);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}
