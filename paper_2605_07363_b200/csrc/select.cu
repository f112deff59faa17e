// K4: exact top-k selection (dsa.py:64-92) for the fused streaming selector.
//
// The reference's rule is argsort(-scores, kind="stable")[:k] then sort: the
// k largest scores, ties to the smaller index, returned ascending.  Every
// kernel here implements exactly that order, (score desc, index asc), on
// monotone u32 keys (-0.0 == +0.0).
//
// Register selector (one CTA per row, NT threads x EPT elements in registers,
// element e = r*NT + tid):
//   1. the k-th largest key v is built bit by bit from the highest bit that
//      differs across the row: v |= bit while count(key >= v|bit) >= k, each
//      count one compare per element + a warp REDUX + one barrier — no atomics;
//   2. if the keys equal to v over-fill the budget, the same search on the
//      indices of the tied keys keeps the smallest ones;
//   3. output order needs no sort: every input is a few lists already ascending
//      by token index (the scorer appends each TMEM lane quadrant's candidates
//      in key order; candidate / per-GPU lists are ascending by construction).
//      One block scan of per-(round, warp) ballot counts compacts the selected
//      elements per list; position = rank in own list + lower_bound in the others.
//
// misa_select_threshold  tau: j-th largest sampled score per row
// misa_select_topk       4 per-quadrant candidate lists per row
// misa_select_dense      a dense (optionally index-listed) row; rows too long for
//                        registers take a global-memory radix path (exact fallback)
// misa_merge_topk        the gathered per-GPU top-k lists of a row
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace misa {

// Optional phase trace (tools/sel_trace: built with -DMISA_SEL_TRACE, never in the product).
#ifdef MISA_SEL_TRACE
__device__ unsigned long long g_sel_trace[64][16];
__device__ int g_sel_trace_row;
#define SEL_MARK(row_i, ph)                                                   \
  do {                                                                         \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (row_i) < 64) g_sel_trace[row_i][ph] = clock64(); \
  } while (0)
#else
#define SEL_MARK(row_i, ph) \
  do {                      \
  } while (0)
#endif


#ifdef MISA_SEL_TRACE
#define CUT_MARK(ph) SEL_MARK(g_sel_trace_row, ph)
#define CUT_MARK_CB(v)                                                          \
  do {                                                                          \
    if (g_sel_trace_row < 64) g_sel_trace[g_sel_trace_row][15] = (unsigned long long)(v); \
  } while (0)
#else
#define CUT_MARK(ph) \
  do {               \
  } while (0)
#define CUT_MARK_CB(v) \
  do {                 \
  } while (0)
#endif

constexpr int kMaxLists = 8;

template <int NT>
struct SelSh {
  static constexpr int NW = NT / 32;
  int cnt[2][NW];
  int cnt3[2][3][NW];
  uint32_t red[NW];
  int tab[NT];  // per-(round, warp) selected counts, scanned in place
  uint32_t bal[32 * (NT / 32)];  // v3: selection ballot of (round, warp)
  int base[32 * (NT / 32)];      // v3: global rank of the first element of (round, warp)
  int wtot[NW];
  int lst_off[kMaxLists + 1];
  int lst_sel[kMaxLists + 1];
  uint32_t hist[2048];  // histogram cut: bins of (key - lo) >> shift
  uint32_t rmin[NW], rmax[NW];
  int hscan[NW];
  int hb_bin, hb_above, hb_count;
  int lst_g[kMaxLists + 1];  // v5: compacted rank of each list's first selected element
  uint32_t bkey[256];  // boundary bucket (exact cut) staging
  int32_t bidx[256];
  int bcount;
  uint32_t res_v;
  int res_thr;
};

constexpr int kBucketMax = 256;

// Cross-warp combines without serial smem chains: lane i reads warp i's value, then one
// warp reduction / scan (NW <= 32).
template <int NW>
__device__ __forceinline__ int warps_exclusive(const int* vals, int w) {
  const int lane = threadIdx.x & 31;
  int v = lane < NW ? vals[lane] : 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  const int incl_prev = __shfl_sync(0xffffffffu, v, (w + 31) & 31);
  return w == 0 ? 0 : incl_prev;  // inclusive sum of warps [0, w-1]
}
template <int NW>
__device__ __forceinline__ uint32_t warps_min(const uint32_t* vals) {
  const int lane = threadIdx.x & 31;
  return __reduce_min_sync(0xffffffffu, lane < NW ? vals[lane] : 0xffffffffu);
}
template <int NW>
__device__ __forceinline__ uint32_t warps_max(const uint32_t* vals) {
  const int lane = threadIdx.x & 31;
  return __reduce_max_sync(0xffffffffu, lane < NW ? vals[lane] : 0u);
}



// Warp-level: largest v with count(x >= v) >= j among this warp's values (x == 0: empty),
// searching bits [hi, 0] on top of `prefix`.
__device__ __forceinline__ uint32_t warp_kth(const uint32_t (&x)[8], int j, uint32_t prefix, int hi) {
  uint32_t v = prefix;
  for (int b = hi; b >= 0; --b) {
    const uint32_t cand = v | (1u << b);
    int c = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) c += x[i] >= cand;
    if (__reduce_add_sync(0xffffffffu, c) >= j) v = cand;
  }
  return v;
}

template <int NT>
__device__ __forceinline__ uint32_t block_reduce_or(uint32_t v, SelSh<NT>& sh) {
  v = __reduce_or_sync(0xffffffffu, v);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sh.red[w] = v;
  __syncthreads();
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < SelSh<NT>::NW; ++i) r |= sh.red[i];
  __syncthreads();
  return r;
}

// Block-wide count of elements satisfying pred(r) (register slot r of this thread).
template <int NT, int EPT, typename Pred>
__device__ __forceinline__ int block_count(Pred pred, SelSh<NT>& sh, int& parity) {
  int c = 0;
#pragma unroll
  for (int r = 0; r < EPT; ++r) c += pred(r) ? 1 : 0;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) sh.cnt[parity][threadIdx.x >> 5] = c;
  __syncthreads();
  int tot = 0;
#pragma unroll
  for (int i = 0; i < SelSh<NT>::NW; ++i) tot += sh.cnt[parity][i];
  parity ^= 1;
  return tot;
}

// Three block-wide counts (val >= c0, >= c1, >= c2) behind a single barrier.
template <int NT, int EPT, typename Val>
__device__ __forceinline__ void block_count3(Val val, uint32_t c0, uint32_t c1, uint32_t c2, SelSh<NT>& sh,
                                             int& parity, int (&out)[3]) {
  int n0 = 0, n1 = 0, n2 = 0;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const uint32_t x = val(r);
    n0 += x >= c0;
    n1 += x >= c1;
    n2 += x >= c2;
  }
  n0 = __reduce_add_sync(0xffffffffu, n0);
  n1 = __reduce_add_sync(0xffffffffu, n1);
  n2 = __reduce_add_sync(0xffffffffu, n2);
  if ((threadIdx.x & 31) == 0) {
    sh.cnt3[parity][0][threadIdx.x >> 5] = n0;
    sh.cnt3[parity][1][threadIdx.x >> 5] = n1;
    sh.cnt3[parity][2][threadIdx.x >> 5] = n2;
  }
  __syncthreads();
  out[0] = out[1] = out[2] = 0;
#pragma unroll
  for (int i = 0; i < SelSh<NT>::NW; ++i) {
    out[0] += sh.cnt3[parity][0][i];
    out[1] += sh.cnt3[parity][1][i];
    out[2] += sh.cnt3[parity][2][i];
  }
  parity ^= 1;
}

// Largest v such that count(val(r) >= v) >= j, over valid slots; val() >= 1 for valid.
// Returns v and the count of values >= v (*c_ge) (values > v: *c_gt).
template <int NT, int EPT, typename Val>
__device__ uint32_t kth_largest(Val val, int j, SelSh<NT>& sh, int& parity, int* c_ge, int* c_gt,
                                int min_bit = 0) {
  uint32_t lo_or = 0, diff = 0, first = 0;
  // common high bits of the valid values: OR of (val ^ some valid value)
#pragma unroll
  for (int r = 0; r < EPT; ++r) lo_or |= val(r);
  // a value present in the block to xor against: the block OR is not a member, so use
  // per-bit agreement: bits set in every valid value = AND, set in any = OR.
  uint32_t a_and = 0xffffffffu;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const uint32_t x = val(r);
    if (x) a_and &= x;
  }
  const uint32_t any_or = block_reduce_or<NT>(lo_or, sh);
  const uint32_t all_and = ~block_reduce_or<NT>(~a_and, sh);
  diff = any_or ^ all_and;  // bits that differ across the valid values
  first = all_and;          // bits common to all valid values (those above hi are the prefix)
  uint32_t v;
  int cge;
  if (diff == 0) {
    v = first;
    cge = block_count<NT, EPT>([&](int r) { return val(r) >= v; }, sh, parity);
  } else {
    const int hi = 31 - __clz(diff);
    v = (hi == 31) ? 0u : (first & ~((2u << hi) - 1u));
    cge = -1;
    // two bits per barrier: candidates v|11, v|10, v|01 of the next bit pair
    int b = hi;
    for (; b - 1 >= min_bit && min_bit == 0; b -= 2) {
      const uint32_t hb = 1u << b, lb = 1u << (b - 1);
      int c[3];
      block_count3<NT, EPT>(val, v | hb | lb, v | hb, v | lb, sh, parity, c);
      if (c[0] >= j) {
        v |= hb | lb;
        cge = c[0];
      } else if (c[1] >= j) {
        v |= hb;
        cge = c[1];
      } else if (c[2] >= j) {
        v |= lb;
        cge = c[2];
      }
    }
    for (; b >= min_bit; --b) {
      const uint32_t cand = v | (1u << b);
      const int c = block_count<NT, EPT>([&](int r) { return val(r) >= cand; }, sh, parity);
      if (c >= j) {
        v = cand;
        cge = c;
      }
    }
    if (cge < 0) cge = block_count<NT, EPT>([&](int r) { return val(r) >= v; }, sh, parity);
  }
  if (min_bit > 0) {  // approximate mode: v is a lower bound of the j-th value, counts not needed
    *c_ge = cge;
    *c_gt = -1;
    return v;
  }
  const int cgt = (v == 0xffffffffu) ? 0 : block_count<NT, EPT>([&](int r) { return val(r) > v; }, sh, parity);
  *c_ge = cge;
  *c_gt = cgt;
  return v;
}

// Merge path: how many of A's elements are among the first d outputs of merge(A, B)
// (A, B ascending; token indices are unique across lists).
__device__ __forceinline__ int merge_path(const int32_t* A, int na, const int32_t* B, int nb, int d) {
  int lo = d - nb > 0 ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] < B[d - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// All NT threads merge A and B into D (each thread one contiguous output chunk).
template <int NT>
__device__ __forceinline__ void merge_pair(const int32_t* A, const float* As, int na, const int32_t* B,
                                           const float* Bs, int nb, int32_t* D, float* Ds, int t = -1,
                                           int nthr = NT) {
  if (t < 0) t = threadIdx.x;
  const int M = na + nb;
  const int chunk = (M + nthr - 1) / nthr;
  const int d0 = min(M, t * chunk), d1 = min(M, d0 + chunk);
  if (d0 >= d1) return;
  int i = merge_path(A, na, B, nb, d0), j = d0 - i;
  for (int d = d0; d < d1; ++d) {
    const bool take_a = j >= nb || (i < na && A[i] < B[j]);
    if (take_a) {
      D[d] = A[i];
      if (Ds) Ds[d] = As[i];
      ++i;
    } else {
      D[d] = B[j];
      if (Ds) Ds[d] = Bs[j];
      ++j;
    }
  }
}

__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int x) {
  int lo = 0;
  while (n > 0) {
    const int half = n >> 1;
    if (a[lo + half] < x) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo;
}

// ---------------------------------------------------------------- tau ----
// tau_t = a lower bound of the j-th largest sampled score, j = ceil(beta*k*m/n): the
// lower edge of the histogram bin that holds it, with 2048 bins over the sampled key
// range [min, max] (at least 2^-10 relative resolution), so tau never exceeds the j-th
// value and costs one atomic per sample and three barriers per row.  The kernel is
// kept lean (registers, 9 KB smem) so that many rows are in flight per SM.
template <int NT, int EPT>
__device__ __forceinline__ void threshold_row(int t, const float* __restrict__ s, int64_t ld,
                                              const int32_t* __restrict__ prefix_len, int stride, int k,
                                              float beta, int64_t append_all, float* __restrict__ tau,
                                              int elem_step) {
  constexpr int NW = NT / 32, NB = 2048, BPT = NB / NT;
  __shared__ uint32_t hist[NB];
  __shared__ uint32_t rmin[NW], rmax[NW];
  __shared__ int wsum[NW];
  __shared__ int sh_bin, sh_above, sh_above_new;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = prefix_len[t];
  if (n <= append_all || n <= k) {
    if (tid == 0) tau[t] = -INFINITY;
    return;
  }
  const int m = (n + stride - 1) / stride;
  long long jj = (long long)ceilf(beta * (float)k * (float)m / (float)n);
  jj = jj < 1 ? 1 : (jj > m ? m : jj);
  const float* row = s + (int64_t)t * ld;
  uint32_t key[EPT];
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int e = r * NT + tid;
    key[r] = __float_as_uint(row[(int64_t)(e < m ? e : 0) * elem_step]);
  }
  uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const bool ok = r * NT + tid < m;
    key[r] = ok ? float_key(__uint_as_float(key[r])) : 0u;
    if (ok) {
      mn = min(mn, key[r]);
      mx = max(mx, key[r]);
    }
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    rmin[w] = mn;
    rmax[w] = mx;
  }
#pragma unroll
  for (int i = 0; i < BPT; ++i) hist[tid * BPT + i] = 0u;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    mn = min(mn, rmin[i]);
    mx = max(mx, rmax[i]);
  }
  // First try a window of the top 2^24 key ulps below the maximum (two binary orders of
  // magnitude, [max/4, max] for positive scores — where the j-th largest of a 1/32 sample,
  // the top few %, normally lies): 2048 bins of 2^13 ulps = 2^-10 relative, one level.  If
  // the j-th sample is below that window, bin the whole range [min, max] and refine the
  // boundary bin once.
  bool narrow = mx - mn > (1u << 24);
  uint32_t lo = narrow ? mx - (1u << 24) : mn;
  uint32_t span = mx - lo;  // window [lo, lo + span]
  int sft = span == 0u ? 0 : max(0, 32 - __clz(span) - 11);
  for (int level = 0;; ++level) {
    if (tid == 0) sh_bin = -1;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const uint32_t d = key[r] - lo;
      if (key[r] && key[r] >= lo && d <= span) atomicAdd(&hist[d >> sft], 1u);
    }
    __syncthreads();
    // thread tid owns bins [NB - BPT*(tid+1), NB - BPT*tid): descending keys
    uint32_t c[BPT];
    int tot = 0;
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
      c[i] = hist[NB - 1 - (tid * BPT + i)];
      tot += (int)c[i];
    }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    int above = incl - tot + (level ? sh_above : 0) + warps_exclusive<NW>(wsum, w);
    if (above < jj && jj <= above + tot) {
#pragma unroll
      for (int i = 0; i < BPT; ++i) {
        if (above < jj && jj <= above + (int)c[i]) {
          sh_bin = NB - 1 - (tid * BPT + i);
          sh_above_new = above;
        }
        above += (int)c[i];
      }
    }
#pragma unroll
    for (int i = 0; i < BPT; ++i) hist[tid * BPT + i] = 0u;
    __syncthreads();
    const int bin = sh_bin;
    if (bin < 0) {  // the j-th sample lies below the narrow window: whole range, two levels
      narrow = false;
      lo = mn;
      span = mx - mn;
      sft = span == 0u ? 0 : max(0, 32 - __clz(span) - 11);
      level = -1;
      __syncthreads();
      continue;
    }
    lo += (uint32_t)bin << sft;
    if (narrow || level == 1 || sft <= 12) {
      if (tid == 0) tau[t] = key_float(lo);  // lower edge of the bin: <= the j-th sample
      return;
    }
    span = (1u << sft) - 1u;
    sft = sft - 11;
    if (tid == 0) sh_above = sh_above_new;  // samples above the refined window
    __syncthreads();
  }
}

// Persistent over rows (a CTA per row would pay a block launch per ~3K-cycle row).
template <int NT, int EPT>
__global__ void __launch_bounds__(NT, (NT * EPT <= 4096 ? 6 : 1)) threshold_kernel(
    const float* __restrict__ s, int64_t ld, const int32_t* __restrict__ prefix_len, int n_rows, int stride, int k,
    float beta, int64_t append_all, float* __restrict__ tau, int elem_step = 1) {
  for (int t = blockIdx.x; t < n_rows; t += gridDim.x) {
    threshold_row<NT, EPT>(t, s, ld, prefix_len, stride, k, beta, append_all, tau, elem_step);
    __syncthreads();  // histogram / scan scratch reused by the next row
  }
}

// Warp-per-row variant (samples per row <= 16384): no block barriers, a private 2048-bin
// histogram per warp, 24 rows per SM in flight; same windows and rounding as above, so
// tau is identical.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) threshold_warp_kernel(
    const float* __restrict__ s, int64_t ld, const int32_t* __restrict__ prefix_len, int n_rows, int stride, int k,
    float beta, int64_t append_all, float* __restrict__ tau, int elem_step) {
  constexpr int NB = 2048;
  __shared__ uint32_t hist_all[WARPS][NB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t* hist = hist_all[w];
  for (int t = blockIdx.x * WARPS + w; t < n_rows; t += gridDim.x * WARPS) {
    const int n = prefix_len[t];
    if (n <= append_all || n <= k) {
      if (lane == 0) tau[t] = -INFINITY;
      continue;
    }
    const int m = (n + stride - 1) / stride;
    long long jj = (long long)ceilf(beta * (float)k * (float)m / (float)n);
    jj = jj < 1 ? 1 : (jj > m ? m : jj);
    const float* row = s + (int64_t)t * ld;
    // visit(fn): fn(key) for every sample of the row; 16-byte loads, 16 per lane in flight
    const bool vec = elem_step == 1 && ((reinterpret_cast<uintptr_t>(row) & 15) == 0);
    auto visit = [&](auto&& fn) {
      int done = 0;
      if (vec) {
        const int m4 = m >> 2;
        const float4* r4 = reinterpret_cast<const float4*>(row);
        for (int v0 = lane; v0 < m4; v0 += 32 * 4) {
          float4 x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = v0 + 32 * u < m4 ? __ldg(r4 + v0 + 32 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (v0 + 32 * u < m4) {
              fn(float_key(x[u].x));
              fn(float_key(x[u].y));
              fn(float_key(x[u].z));
              fn(float_key(x[u].w));
            }
        }
        done = m4 << 2;
      }
      for (int e0 = done + lane; e0 < m; e0 += 32 * 8) {
        uint32_t kv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) kv[u] = e0 + 32 * u < m ? float_key(row[(int64_t)(e0 + 32 * u) * elem_step]) : 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e0 + 32 * u < m) fn(kv[u]);
      }
    };
    uint32_t mn = 0xffffffffu, mx = 0u;
    visit([&](uint32_t kv) {
      mn = min(mn, kv);
      mx = max(mx, kv);
    });
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    bool narrow = mx - mn > (1u << 24);
    uint32_t lo = narrow ? mx - (1u << 24) : mn;
    uint32_t span = mx - lo;
    int sft = span == 0u ? 0 : max(0, 32 - __clz(span) - 11);
    int above_prev = 0;
    for (int level = 0;; ++level) {
      for (int i = lane * 4; i < NB; i += 128) *reinterpret_cast<uint4*>(hist + i) = make_uint4(0u, 0u, 0u, 0u);
      __syncwarp();
      visit([&](uint32_t kv) {
        const uint32_t d = kv - lo;
        if (kv >= lo && d <= span) atomicAdd(&hist[d >> sft], 1u);
      });
      __syncwarp();
      // lane owns bins [NB - 64(lane+1), NB - 64 lane) (descending keys)
      const int b0 = NB - 64 * (lane + 1);
      int cnt = 0;
#pragma unroll 4
      for (int i = 0; i < 64; i += 4) {
        const uint4 h4 = *reinterpret_cast<const uint4*>(hist + b0 + i);
        cnt += (int)(h4.x + h4.y + h4.z + h4.w);
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int ex = above_prev + incl - cnt;
      const bool mine = ex < jj && jj <= ex + cnt;
      const uint32_t who = __ballot_sync(0xffffffffu, mine);
      if (who == 0u) {  // the j-th sample is below the narrow window: whole range
        narrow = false;
        lo = mn;
        span = mx - mn;
        sft = span == 0u ? 0 : max(0, 32 - __clz(span) - 11);
        above_prev = 0;
        level = -1;
        __syncwarp();
        continue;
      }
      const int src = __ffs(who) - 1;
      int B = 0, A = 0;
      if (lane == src) {
        int a = ex;
        for (int i = 63; i >= 0; --i) {
          const int h = (int)hist[b0 + i];
          if (a < jj && jj <= a + h) {
            B = b0 + i;
            A = a;
            break;
          }
          a += h;
        }
      }
      B = __shfl_sync(0xffffffffu, B, src);
      A = __shfl_sync(0xffffffffu, A, src);
      lo += (uint32_t)B << sft;
      __syncwarp();
      if (narrow || level == 1 || sft <= 12) {
        if (lane == 0) tau[t] = key_float(lo);  // lower edge of the bin: <= the j-th sample
        break;
      }
      span = (1u << sft) - 1u;
      sft = sft - 11;
      above_prev = A;  // samples above the refined window
    }
    __syncwarp();
  }
}

// ---------------------------------------------- v3 row selector core ----
// Warp w owns the contiguous element range [w*WE, (w+1)*WE) of the row's
// concatenated lists (WE = 32*EPT); lane l's slot r is element w*WE + 32r + l.
// Keys live in registers (0 = empty slot), token indices in smem (sidx), so a
// CTA needs few registers and several rows run per SM.
template <int NT, int EPT>
__device__ __forceinline__ int v3_elem(int r) {
  return (threadIdx.x >> 5) * (EPT * 32) + r * 32 + (threadIdx.x & 31);
}

template <int NT, int EPT>
__device__ void v3_cut(const uint32_t (&key)[EPT], const int32_t* sidx, int N, int kk, SelSh<NT>& sh, int& parity,
                       uint32_t& v_out, int& thr_out) {
  uint32_t lo_or = 0, a_and = 0xffffffffu;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    lo_or |= key[r];
    if (key[r]) a_and &= key[r];
  }
  const uint32_t any_or = block_reduce_or<NT>(lo_or, sh);
  const uint32_t all_and = ~block_reduce_or<NT>(~a_and, sh);
  const uint32_t diff = any_or ^ all_and;
  uint32_t v;
  int b, above = 0, cge = N;
  auto val = [&](int r) { return key[r]; };
  if (diff == 0) {
    v = all_and;
    b = -1;
  } else {
    b = 31 - __clz(diff);
    v = (b == 31) ? 0u : (all_and & ~((2u << b) - 1u));
    while (b >= 1 && cge - above > kBucketMax) {
      const uint32_t hb = 1u << b, lb = 1u << (b - 1);
      int c[3];
      block_count3<NT, EPT>(val, v | hb | lb, v | hb, v | lb, sh, parity, c);
      if (c[0] >= kk) {
        v |= hb | lb;
        cge = c[0];
      } else if (c[1] >= kk) {
        above = c[0];
        v |= hb;
        cge = c[1];
      } else if (c[2] >= kk) {
        above = c[1];
        v |= lb;
        cge = c[2];
      } else {
        above = c[2];
      }
      b -= 2;
    }
    if (b == 0 && cge - above > kBucketMax) {
      const int c = block_count<NT, EPT>([&](int r) { return key[r] >= (v | 1u); }, sh, parity);
      if (c >= kk) {
        v |= 1u;
        cge = c;
      } else {
        above = c;
      }
      b = -1;
    }
  }
  const int need = kk - above;
  const int bucket = cge - above;
  const uint32_t bmask = (b + 1 >= 32) ? 0u : ~((b >= 0) ? ((2u << b) - 1u) : 0u);
  if (bucket <= kBucketMax) {
    if (threadIdx.x == 0) sh.bcount = 0;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      if (key[r] != 0u && (key[r] & bmask) == (v & bmask)) {
        const int p = atomicAdd(&sh.bcount, 1);
        sh.bkey[p] = key[r];
        sh.bidx[p] = sidx[v3_elem<NT, EPT>(r)];
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint32_t x[8];
      int32_t xi[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = lane + 32 * i;
        x[i] = e < bucket ? sh.bkey[e] : 0u;
        xi[i] = e < bucket ? sh.bidx[e] : 0x7fffffff;
      }
      const uint32_t vk = warp_kth(x, need, v & bmask, b);
      int gt = 0, eq = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        gt += x[i] > vk;
        eq += x[i] == vk;
      }
      gt = __reduce_add_sync(0xffffffffu, gt);
      eq = __reduce_add_sync(0xffffffffu, eq);
      const int need2 = need - gt;
      int t = 0x7fffffff;
      if (need2 < eq) {
        uint32_t y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = x[i] == vk ? ~static_cast<uint32_t>(xi[i]) : 0u;
        t = static_cast<int>(~warp_kth(y, need2, 0u, 31));
      }
      if (lane == 0) {
        sh.res_v = vk;
        sh.res_thr = t;
      }
    }
    __syncthreads();
    v_out = sh.res_v;
    thr_out = sh.res_thr;
    __syncthreads();
    return;
  }
  // unsplittable bucket (all keys == v): keep the `need` smallest indices
  int c2, c3;
  const uint32_t t2 = kth_largest<NT, EPT>(
      [&](int r) { return (key[r] == v) ? ~static_cast<uint32_t>(sidx[v3_elem<NT, EPT>(r)]) : 0u; }, need, sh,
      parity, &c2, &c3);
  v_out = v;
  thr_out = (need < bucket) ? static_cast<int>(~t2) : 0x7fffffff;
}

// ------------------------------------------- histogram cut (v4) ----
// The (score desc, index asc) cut of the kk-th element: bins of the valid keys' range
// [lo, hi] at 11-bit resolution (2048 bins, one smem atomic per element), one block
// scan from the top bin to the boundary bin, refined by another level only when that
// bin still holds more than kBucketMax elements; the boundary bin's elements are then
// ranked exactly by (key desc, index asc) with one element per thread.
template <int NT, int EPT, typename IdxFn>
__device__ void hist_cut(const uint32_t (&key)[EPT], IdxFn idx_of, int N, int kk, SelSh<NT>& sh, int& parity,
                         uint32_t& v_out, int& thr_out, int rv = EPT, bool staged_minmax = false) {
  // staged_minmax: the caller already zeroed sh.hist and published per-warp sh.rmin /
  // sh.rmax behind a barrier (saves this function's first barrier)
  // rv: warp-uniform number of leading slot rows that can hold valid keys (rows >= rv
  // are skipped without issuing their instructions)
  constexpr int NW = NT / 32;
  constexpr int NB = 2048, BPT = NB / NT;  // bins per thread
  static_assert(NB % NT == 0 && BPT >= 1 && BPT <= 16, "bins per thread");
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t mn = 0xffffffffu, mx = 0u;
  if (!staged_minmax) {
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      if (r < rv && key[r]) {
        mn = min(mn, key[r]);
        mx = max(mx, key[r]);
      }
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) {
      sh.rmin[w] = mn;
      sh.rmax[w] = mx;
    }
#pragma unroll
    for (int i = 0; i < BPT; ++i) sh.hist[tid * BPT + i] = 0u;
    __syncthreads();
  }
  CUT_MARK(9);
  mn = warps_min<NW>(sh.rmin);
  mx = warps_max<NW>(sh.rmax);
  // level window: keys in [lo, lo + span) with span - 1 <= 0xffffffff, bins of 2^sft
  uint32_t lo = mn, span_m1 = mx - mn;
  int sft = span_m1 == 0u ? 0 : max(0, 32 - __clz(span_m1) - 11);
  int need = kk, cB;
  for (;;) {
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      if (r < rv) {
        const uint32_t d = key[r] - lo;
        if (key[r] && d <= span_m1) atomicAdd(&sh.hist[d >> sft], 1u);
      }
    }
    __syncthreads();
    CUT_MARK(10);
    // thread tid owns bins [NB - BPT*(tid+1), NB - BPT*tid): descending key order
    uint32_t c[BPT];
    int tot = 0;
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
      c[i] = sh.hist[NB - 1 - (tid * BPT + i)];
      tot += static_cast<int>(c[i]);
    }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) sh.hscan[w] = incl;
    __syncthreads();
    int above = incl - tot + warps_exclusive<NW>(sh.hscan, w);
    if (above < need && need <= above + tot) {
#pragma unroll
      for (int i = 0; i < BPT; ++i) {
        if (above < need && need <= above + static_cast<int>(c[i])) {
          sh.hb_bin = NB - 1 - (tid * BPT + i);
          sh.hb_above = above;
          sh.hb_count = static_cast<int>(c[i]);
        }
        above += static_cast<int>(c[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < BPT; ++i) sh.hist[tid * BPT + i] = 0u;  // ready for a next level
    if (tid == 0) sh.bcount = 0;
    __syncthreads();
    const int B = sh.hb_bin;
    need -= sh.hb_above;
    cB = sh.hb_count;
    lo += static_cast<uint32_t>(B) << sft;
    span_m1 = sft == 0 ? 0u : ((1u << sft) - 1u);
    CUT_MARK(11);
    if (cB <= kBucketMax || sft == 0) break;
    sft = max(0, sft - 11);
  }
  // the whole boundary bin is selected: the cut is its lower edge (no collect / rank)
  if (need == cB) {
    v_out = lo == 0u ? 0u : lo - 1u;  // selected iff key > lo - 1, i.e. key >= lo
    thr_out = -1;
    return;
  }
  // elements of the boundary bin: keys in [lo, lo + span_m1]
  if (cB <= kBucketMax) {
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      if (r < rv && key[r] && key[r] - lo <= span_m1) {
        const int p = atomicAdd(&sh.bcount, 1);
        sh.bkey[p] = key[r];
        sh.bidx[p] = idx_of(r);
      }
    }
    __syncthreads();
    CUT_MARK(12);
    // exact rank of each boundary element under (key desc, index asc), one warp per
    // element, lanes over the others; the element of rank need-1 is the cut
    for (int e = w; e < cB; e += NW) {
      const uint32_t ke = sh.bkey[e];
      const int ie = sh.bidx[e];
      int rank = 0;
      for (int f = lane; f < cB; f += 32) {
        const uint32_t kf = sh.bkey[f];
        rank += (kf > ke) || (kf == ke && sh.bidx[f] < ie);
      }
      rank = __reduce_add_sync(0xffffffffu, rank);
      if (lane == 0 && rank == need - 1) {
        sh.res_v = ke;
        sh.res_thr = ie;
      }
    }
    __syncthreads();
    CUT_MARK(13);
    if (threadIdx.x == 0 && blockIdx.x == 0) CUT_MARK_CB(cB);
    v_out = sh.res_v;  // res_* are next written by a later row's rank phase, many barriers on
    thr_out = sh.res_thr;
    return;
  }
  // more than kBucketMax copies of one key value: keep the `need` smallest indices
  int c2, c3;
  const uint32_t t2 = kth_largest<NT, EPT>(
      [&](int r) { return (key[r] == lo) ? ~static_cast<uint32_t>(idx_of(r)) : 0u; }, need, sh, parity, &c2, &c3);
  v_out = lo;
  thr_out = (need < cB) ? static_cast<int>(~t2) : 0x7fffffff;
}

// Select the kk best of the N staged elements (NL lists, each ascending by index,
// offsets in sh.lst_off) and write them ascending to out[0..kk) (+ scores), -1 pad.
template <int NT, int EPT>
__device__ void v3_select(const uint32_t (&key)[EPT], const int32_t* sidx, int N, int NL, int kk, SelSh<NT>& sh,
                          int32_t* cidx, float* csc, int32_t* out, float* outs, int k_out) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int parity = 0;
  uint32_t v = 0;
  int thr = 0x7fffffff;
  if (kk < N)
    hist_cut<NT, EPT>(key, [&](int r) { return sidx[v3_elem<NT, EPT>(r)]; }, N, kk, sh, parity, v, thr);
  uint32_t selm = 0;
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    bool sel = key[r] != 0u;
    if (sel && kk < N) sel = key[r] > v || (key[r] == v && sidx[v3_elem<NT, EPT>(r)] <= thr);
    selm |= (sel ? 1u : 0u) << r;
    cnt += __popc(__ballot_sync(0xffffffffu, sel));
  }
  if (lane == 0) sh.wtot[w] = cnt;
  __syncthreads();
  int run = warps_exclusive<NW>(sh.wtot, w);
  const uint32_t lt = ptx::lanemask_lt();
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const bool sel = (selm >> r) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, sel);
    if (lane == 0) {
      sh.bal[r * NW + w] = bal;
      sh.base[r * NW + w] = run;
    }
    if (sel) {
      const int rank = run + __popc(bal & lt);
      cidx[rank] = sidx[v3_elem<NT, EPT>(r)];
      if (csc) csc[rank] = key_float(key[r]);
    }
    run += __popc(bal);
  }
  __syncthreads();
  // compacted-list boundaries: rank of each list's first element (from the stored ballots)
  if (tid <= NL) {
    const int e = sh.lst_off[tid];
    int rk = kk;
    if (e < N) {
      const int ww = e / (EPT * 32), rr = (e % (EPT * 32)) / 32, ll = e % 32;
      rk = sh.base[rr * NW + ww] + __popc(sh.bal[rr * NW + ww] & ((1u << ll) - 1u));
    }
    sh.lst_sel[tid] = rk;
  }
  __syncthreads();
  // pairwise merge-path rounds over the NL sorted runs (pairs of a round run concurrently
  // on disjoint thread groups); the last round writes `out`
  int32_t* src = cidx;
  float* srcs = csc;
  int32_t* tmp = cidx + k_out;
  float* tmps = csc ? csc + k_out : nullptr;
  int runs = NL;
  while (runs > 2) {
    {
      const int npairs = runs / 2;
      const int per = NT / npairs;
      const int p = min(tid / per, npairs - 1) * 2;
      const int a0 = sh.lst_sel[p], a1 = sh.lst_sel[p + 1], b1 = sh.lst_sel[p + 2];
      if (tid / per < npairs)
        merge_pair<NT>(src + a0, srcs ? srcs + a0 : nullptr, a1 - a0, src + a1, srcs ? srcs + a1 : nullptr,
                       b1 - a1, tmp + a0, tmps ? tmps + a0 : nullptr, tid % per, per);
    }
    if (runs & 1) {
      for (int i = sh.lst_sel[runs - 1] + tid; i < sh.lst_sel[runs]; i += NT) {
        tmp[i] = src[i];
        if (tmps) tmps[i] = srcs[i];
      }
    }
    __syncthreads();
    if (tid == 0) {
      int nr = 0;
      for (int p = 0; p < runs; p += 2) sh.lst_sel[nr++] = sh.lst_sel[p];
      sh.lst_sel[nr] = kk;
    }
    runs = (runs + 1) / 2;
    int32_t* t1 = src;
    src = tmp;
    tmp = t1;
    float* t2 = srcs;
    srcs = tmps;
    tmps = t2;
    __syncthreads();
  }
  if (runs == 2) {
    const int a0 = sh.lst_sel[0], a1 = sh.lst_sel[1], b1 = sh.lst_sel[2];
    merge_pair<NT>(src + a0, srcs ? srcs + a0 : nullptr, a1 - a0, src + a1, srcs ? srcs + a1 : nullptr, b1 - a1,
                   out + a0, outs ? outs + a0 : nullptr);
  } else {
    for (int i = tid; i < kk; i += NT) {
      out[i] = src[i];
      if (outs) outs[i] = srcs[i];
    }
  }
  for (int i = kk + tid; i < k_out; i += NT) {
    out[i] = -1;
    if (outs) outs[i] = -INFINITY;
  }
}

// Run the row with the smallest register footprint that holds N elements.
template <int NT, int EPT, typename LoadFn>
__device__ void v3_dispatch(int N, LoadFn load, int NL, int kk, SelSh<NT>& sh, int32_t* sidx, int32_t* cidx,
                            float* csc, int32_t* out, float* outs, int k_out) {
  uint32_t key[EPT];
  load(key, sidx);
  __syncthreads();
  v3_select<NT, EPT>(key, sidx, N, NL, kk, sh, cidx, csc, out, outs, k_out);
}

// -------------------------------------------------- candidates -> top-k ----
// Persistent: CTA b handles rows b, b + grid, ...  The next row's 4 quadrant lists
// are bulk-copied (cp.async.bulk, mbarrier complete_tx) into shared memory while the
// current row is being cut, selected and merged, so no row waits on DRAM latency.
struct TopkPrefetch {
  int row, n, c[kQuadrants];
  bool copy;  // lists in flight (false: row needs no candidates or is past the end)
};

template <int NT, int EPT, bool PF>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1)) topk_kernel(const uint64_t* __restrict__ cand,
                                                  const int32_t* __restrict__ cand_count, int cap,
                                                  const int32_t* __restrict__ prefix_len, int n_rows, int k,
                                                  int32_t* __restrict__ topk, int64_t topk_ld,
                                                  float* __restrict__ topk_scores, int32_t* __restrict__ flags) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ SelSh<NT> sh;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ TopkPrefetch pf;
  uint64_t* raw = reinterpret_cast<uint64_t*>(dsm);  // PF: list q at raw + q*cap
  int32_t* sidx = reinterpret_cast<int32_t*>(raw + (PF ? (size_t)kQuadrants * cap : 0));
  int32_t* cidx = sidx + NT * EPT;
  float* csc = reinterpret_cast<float*>(cidx + 2 * k);
  const bool want_scores = topk_scores != nullptr;

  // thread 0 keeps the (n, counts) of the row after next in registers: their global
  // loads are issued one row ahead of use
  int nx_n = 0, nx_c[kQuadrants] = {0, 0, 0, 0};
  auto load_meta = [&](int row) {
    if (row < n_rows) {
      nx_n = prefix_len[row];
#pragma unroll
      for (int q = 0; q < kQuadrants; ++q) nx_c[q] = cand_count[(int64_t)row * kQuadrants + q];
    }
  };
  auto issue = [&](int row) {  // thread 0: start the copy of `row` (meta in nx_*)
    pf.row = row;
    pf.copy = false;
    if (row >= n_rows) return;
    pf.n = nx_n;
#pragma unroll
    for (int q = 0; q < kQuadrants; ++q) pf.c[q] = nx_c[q];
    if ((nx_n <= k && !want_scores) || nx_n <= 0) return;  // counts unused (may be unset)
    pf.copy = true;
    if (!PF) return;
    uint32_t bytes = 0;
#pragma unroll
    for (int q = 0; q < kQuadrants; ++q) bytes += ((min(max(nx_c[q], 0), cap) * 8u) + 15u) & ~15u;
    ptx::mbar_arrive_expect_tx(&mbar, bytes);
#pragma unroll
    for (int q = 0; q < kQuadrants; ++q) {
      const uint32_t b = ((min(max(nx_c[q], 0), cap) * 8u) + 15u) & ~15u;
      if (b) ptx::bulk_g2s(raw + (size_t)q * cap, cand + ((int64_t)row * kQuadrants + q) * cap, b, &mbar);
    }
    pf.copy = true;
  };
  if (threadIdx.x == 0) {
    ptx::mbar_init(&mbar, 1);
    ptx::fence_mbar_init();
    load_meta(blockIdx.x);
    issue(blockIdx.x);
    load_meta(blockIdx.x + gridDim.x);
  }
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < n_rows; t += gridDim.x) {
    __syncthreads();  // pf (row t) visible; the previous row is done with raw / sidx / cidx
    const int n = pf.n;
    const bool copy = pf.copy;
    int c[kQuadrants];
#pragma unroll
    for (int q = 0; q < kQuadrants; ++q) c[q] = pf.c[q];
    int32_t* out = topk + (int64_t)t * topk_ld;
    float* outs = want_scores ? topk_scores + (int64_t)t * topk_ld : nullptr;
    const int kk = n < k ? n : k;
    if (!copy) {  // topk_tokens keeps every prefix token when k >= L (dsa.py:73)
      __syncthreads();  // everyone has read pf before it is overwritten
      if (threadIdx.x == 0) {
        issue(t + gridDim.x);
        load_meta(t + 2 * gridDim.x);
      }
      for (int i = threadIdx.x; i < k; i += NT) {
        out[i] = i < n ? i : -1;
        if (outs) outs[i] = -INFINITY;
      }
      if (threadIdx.x == 0 && flags) flags[t] = 0;
      continue;
    }
    int off[kQuadrants + 1];
    bool overflow = false;
    off[0] = 0;
#pragma unroll
    for (int q = 0; q < kQuadrants; ++q) {
      overflow |= c[q] > cap;
      off[q + 1] = off[q] + min(max(c[q], 0), cap);
    }
    const int total = off[kQuadrants];
    if (PF) {
      ptx::mbar_wait(&mbar, phase);
      phase ^= 1;
    }
    const bool bad = overflow || total < kk || total > NT * EPT;
    uint32_t key[EPT];
    if (!bad) {
      // PF: from the staged copy; else straight from global with every load issued
      // before its first use (one memory latency per row)
      const uint64_t* src = PF ? raw : cand + (int64_t)t * kQuadrants * cap;
      uint2 rw[EPT];
#pragma unroll
      for (int r = 0; r < EPT; ++r) {
        const int e = v3_elem<NT, EPT>(r);
        const int q = (e >= off[1]) + (e >= off[2]) + (e >= off[3]);
        const uint2* at = reinterpret_cast<const uint2*>(src + (e < total ? (size_t)q * cap + (e - off[q]) : 0));
        rw[r] = PF ? *at : __ldcs(at);
      }
#pragma unroll
      for (int r = 0; r < EPT; ++r) {
        const int e = v3_elem<NT, EPT>(r);
        if (e < total) sidx[e] = static_cast<int32_t>(rw[r].y);
        key[r] = e < total ? float_key(__uint_as_float(rw[r].x)) : 0u;
      }
    }
    if (threadIdx.x <= kQuadrants) sh.lst_off[threadIdx.x] = off[threadIdx.x];
    __syncthreads();  // raw consumed, sidx / lst_off staged
    if (threadIdx.x == 0) {
      issue(t + gridDim.x);
      load_meta(t + 2 * gridDim.x);
    }
    if (bad) {
      for (int i = threadIdx.x; i < k; i += NT) out[i] = -1;
      if (threadIdx.x == 0 && flags)
        flags[t] = (overflow || total > NT * EPT) ? MISA_FLAG_OVERFLOW : MISA_FLAG_UNDERFLOW;
      continue;
    }
    if (kk <= 0) {
      for (int i = threadIdx.x; i < k; i += NT) {
        out[i] = -1;
        if (outs) outs[i] = -INFINITY;
      }
    } else {
      v3_select<NT, EPT>(key, sidx, total, kQuadrants, kk, sh, cidx, outs ? csc : nullptr, out, outs, k);
    }
    if (threadIdx.x == 0 && flags) flags[t] = 0;
  }
}

// ---------------------------------------------- v5 candidates -> top-k ----
// Persistent, prefetching, merge-free.  Warp w owns slots of quadrant list
// q = w / (NW/4) (NT*EPT == 4*cap, cap a multiple of 32*EPT), so extraction is one
// shared load per slot and the compaction order is list-major.  The ascending output
// needs no merge: the scorer's quadrant q holds exactly the 32-key chunks c = idx/32
// with c % 4 == q, so all selected elements of a chunk are contiguous in one list and
//   pos = #selected in chunks < c (block scan of a chunk histogram) + rank within c.
// UO (unordered): the selected set is written in list-major compaction order — four runs,
// each ascending (quadrant q's selected keys), run lengths in runs[t][0..4) — skipping the
// chunk histogram / scan / reposition that the ascending output needs (MISA-dagger's coarse
// candidates: the re-rank's selector merges the runs, misa_select_dense_runs).
template <int NT, int EPT, bool WS, bool UO = false>  // WS: selected scores are returned too (topk_scores)
__global__ void __launch_bounds__(NT, ((NT <= 256 || EPT <= 12) ? 2 : 1)) topk5_kernel(const uint64_t* __restrict__ cand,
                                                      const int32_t* __restrict__ cand_count, int cap,
                                                      const int32_t* __restrict__ prefix_len, int n_rows, int k,
                                                      int n_chunks, int32_t* __restrict__ topk, int64_t topk_ld,
                                                      float* __restrict__ topk_scores, int32_t* __restrict__ flags,
                                                      int32_t* __restrict__ runs = nullptr) {
  constexpr int NW = NT / 32, WPL = NW / kQuadrants, WE = 32 * EPT;
  static_assert(NW % kQuadrants == 0, "warps split evenly over the quadrant lists");
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ SelSh<NT> sh;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ TopkPrefetch pf;
  uint64_t* raw = reinterpret_cast<uint64_t*>(dsm);                    // list q at raw + q*cap
  uint32_t* H = reinterpret_cast<uint32_t*>(raw + (size_t)kQuadrants * cap);  // chunk counts -> prefix
  uint32_t* G0 = H + n_chunks;                                          // first compacted rank of a chunk
  int32_t* cidx = reinterpret_cast<int32_t*>(G0 + n_chunks);            // compacted indices
  float* csc = reinterpret_cast<float*>(cidx + k);                       // compacted scores (optional)
  constexpr bool want_scores = WS;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int q = w / WPL;                       // this warp's quadrant list
  const int i0 = (w % WPL) * WE + lane;        // list position of slot 0 (slot r: i0 + 32r)

  // (n, counts) of the row after next, fetched one row ahead of use straight into shared
  // memory with cp.async (registers are the scarce resource here: 512 threads x 2 CTAs)
  __shared__ int4 meta_c;
  __shared__ int meta_n;
  auto load_meta = [&](int row) {
    if (row < n_rows) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ptx::smem_u32(&meta_n)), "l"(prefix_len + row)
                   : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(&meta_c)),
                   "l"(cand_count + 4 * (int64_t)row)
                   : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  auto publish = [&](int row) {  // pf <- the fetched (n, counts); true if the lists are needed
    pf.row = row;
    pf.copy = false;
    if (row >= n_rows) return false;
    asm volatile("cp.async.wait_all;" ::: "memory");
    const int nn = meta_n;
    const int4 c4 = meta_c;
    pf.n = nn;
    pf.c[0] = c4.x;
    pf.c[1] = c4.y;
    pf.c[2] = c4.z;
    pf.c[3] = c4.w;
    // no candidates needed: every prefix token (n <= k) or an empty prefix (counts unset)
    if ((nn <= k && !want_scores) || nn <= 0) return false;
    pf.copy = true;
    return true;
  };
  // the row's four lists are one contiguous region: a single bulk copy of all of it.  (A
  // cheap issue beats copying only the filled ~2/3: four clamped per-list copies were
  // measured 3.8 -> 4.7 ms at C4 — the issuing thread is on the row's critical path.)
  auto copy_lists = [&](int row) {
    const uint32_t bytes = kQuadrants * cap * 8u;
    ptx::mbar_arrive_expect_tx(&mbar, bytes);
    ptx::bulk_g2s(raw, cand + (int64_t)row * kQuadrants * cap, bytes, &mbar);
  };
  // issue() = stage() + launch().  On the common path they are split: stage() publishes pf
  // right after extraction, launch() starts the copy later, where the issuing thread's
  // chain is short on the critical path (the chunk scan's barrier)
  auto stage = [&](int row) { publish(row); };
  auto launch = [&]() {
    if (pf.copy) copy_lists(pf.row);
  };
  auto issue = [&](int row) {
    if (publish(row)) copy_lists(row);
  };
  if (tid == 0) {
    ptx::mbar_init(&mbar, 1);
    ptx::fence_mbar_init();
    load_meta(blockIdx.x);
    issue(blockIdx.x);
    load_meta(blockIdx.x + gridDim.x);
  }
  __syncthreads();  // mbarrier init and the first row's pf visible to every thread
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < n_rows; t += gridDim.x) {
    // no barrier here: pf was written behind the previous row's barriers (or the prologue's;
    // early-exit paths sync before leaving), and this row's first smem writes follow its
    // extraction barrier
    const int ti_ = (t - blockIdx.x) / gridDim.x;
    (void)ti_;
#ifdef MISA_SEL_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0) g_sel_trace_row = ti_;
#endif
    SEL_MARK(ti_, 0);
    const int n = pf.n;
    const bool copy = pf.copy;
    int c[kQuadrants];
#pragma unroll
    for (int j = 0; j < kQuadrants; ++j) c[j] = pf.c[j];
    int32_t* out = topk + (int64_t)t * topk_ld;
    float* outs = want_scores ? topk_scores + (int64_t)t * topk_ld : nullptr;
    const int kk = n < k ? n : k;
    if (!copy) {  // topk_tokens keeps every prefix token when k >= L (dsa.py:73); empty prefix: none
      __syncthreads();
      if (tid == 0) {
        issue(t + gridDim.x);
        load_meta(t + 2 * gridDim.x);
      }
      for (int i = tid; i < k; i += NT) {
        out[i] = i < n ? i : -1;
        if (outs) outs[i] = -INFINITY;
      }
      if (UO && tid < kQuadrants) runs[(int64_t)t * kQuadrants + tid] = tid == 0 ? max(0, min(n, k)) : 0;
      if (tid == 0 && flags) flags[t] = 0;
      __syncthreads();  // pf (next row) published before anyone reads it
      continue;
    }
    bool overflow = false;
    int total = 0;
#pragma unroll
    for (int j = 0; j < kQuadrants; ++j) {
      overflow |= c[j] > cap;
      total += min(max(c[j], 0), cap);
    }
    const int cq = min(max(q == 0 ? c[0] : q == 1 ? c[1] : q == 2 ? c[2] : c[3], 0), cap);  // no local array
    // slot rows of this warp that can hold list elements (warp-uniform)
    const int rv = EPT;  // unguarded: predicated slots pipeline better than per-row branches
    ptx::mbar_wait(&mbar, phase);
    phase ^= 1;
    SEL_MARK(ti_, 1);
    uint32_t key[EPT];
    int32_t idx[EPT];
    uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      key[r] = 0u;
      idx[r] = 0;
      if (r < rv) {
        const int i = i0 + 32 * r;
        // i < cap always (the warps tile the list capacity): slots past the count read stale
        // words that the key mask below discards
        const uint2 rw = *reinterpret_cast<const uint2*>(raw + (size_t)q * cap + i);
        key[r] = i < cq ? float_key(__uint_as_float(rw.x)) : 0u;
        idx[r] = static_cast<int32_t>(rw.y);
        if (i < cq) {
          mn = min(mn, key[r]);
          mx = max(mx, key[r]);
        }
      }
    }
    // the cut's first phase rides on this barrier: per-warp min / max and a zeroed histogram
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) {
      sh.rmin[w] = mn;
      sh.rmax[w] = mx;
    }
    for (int i = tid; i < 2048; i += NT) sh.hist[i] = 0u;
    __syncthreads();  // raw consumed: the next row's copy may start
    SEL_MARK(ti_, 2);
    const bool go = !(overflow || total < kk);
    if (go && tid == 0) stage(t + gridDim.x);  // pf is free: every thread has read it
    if (overflow || total < kk) {
      if (tid == 0) {
        issue(t + gridDim.x);
        load_meta(t + 2 * gridDim.x);
      }
      for (int i = tid; i < k; i += NT) out[i] = -1;
      if (UO && tid < kQuadrants) runs[(int64_t)t * kQuadrants + tid] = 0;
      if (tid == 0 && flags) flags[t] = overflow ? MISA_FLAG_OVERFLOW : MISA_FLAG_UNDERFLOW;
      __syncthreads();  // pf (next row) published before anyone reads it
      continue;
    }
    // ---- cut: kk-th element under (score desc, index asc)
    uint32_t v = 0;
    int thr = 0x7fffffff;
    int parity = 0;
    if (kk < total)
      hist_cut<NT, EPT>(key, [&](int r) { return idx[r]; }, total, kk, sh, parity, v, thr, rv, /*staged=*/true);
    SEL_MARK(ti_, 3);
    // ---- compaction of the selected elements (list-major order) into cidx / csc
    const int nch = (n + 31) >> 5;
    uint32_t selm = 0;
    int cnt = 0;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      if (r < rv) {
        bool sel = key[r] != 0u;
        if (kk < total) sel = sel && (key[r] > v || (key[r] == v && idx[r] <= thr));
        const uint32_t bal = __ballot_sync(0xffffffffu, sel);
        selm |= (sel ? 1u : 0u) << r;
        cnt += __popc(bal);
      }
    }
    if (lane == 0) sh.wtot[w] = cnt;
    if (!UO) {
      for (int i = tid; i < nch; i += NT) {
        H[i] = 0u;
        G0[i] = 0xffffffffu;
      }
    }
    __syncthreads();
    SEL_MARK(ti_, 4);
    if constexpr (UO) {
      // list-major compaction straight to the output row; run q = the selected keys of list q
      int run = warps_exclusive<NW>(sh.wtot, w);
      const uint32_t lt = ptx::lanemask_lt();
#pragma unroll
      for (int r = 0; r < EPT; ++r) {
        const bool sel = (selm >> r) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, sel);
        if (sel) {
          const int g = run + __popc(bal & lt);
          out[g] = idx[r];
          if (want_scores) outs[g] = key_float(key[r]);
        }
        run += __popc(bal);
      }
      if (tid < kQuadrants) {
        int c = 0;
        for (int i = 0; i < WPL; ++i) c += sh.wtot[tid * WPL + i];
        runs[(int64_t)t * kQuadrants + tid] = c;
      }
      for (int i = kk + tid; i < k; i += NT) {
        out[i] = -1;
        if (outs) outs[i] = -INFINITY;
      }
      __syncthreads();  // wtot / hist reads done before the next row reuses them; pf published
      if (tid == 0) {
        launch();
        load_meta(t + 2 * gridDim.x);
        if (flags) flags[t] = 0;
      }
      continue;
    }
    int run = warps_exclusive<NW>(sh.wtot, w);
    const uint32_t lt = ptx::lanemask_lt();
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      if (r < rv) {
        const bool sel = (selm >> r) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, sel);
        if (sel) {
          const int g = run + __popc(bal & lt);
          cidx[g] = idx[r];
          if (want_scores) csc[g] = key_float(key[r]);
          // a chunk's selected elements are contiguous in this order: count them and keep
          // the smallest rank (the chunk's start)
          const int ch = idx[r] >> 5;
          atomicAdd(&H[ch], 1u);
          atomicMin(&G0[ch], static_cast<uint32_t>(g));
        }
        run += __popc(bal);
      }
    }
    __syncthreads();
    SEL_MARK(ti_, 5);
    // start the next row's copy here rather than right after extraction: the issuing
    // thread's delay then overlaps the chunk scan instead of stalling the cut's barriers
    if (tid == 0) {
      launch();
      SEL_MARK(ti_, 14);
      load_meta(t + 2 * gridDim.x);
    }
    SEL_MARK(ti_, 6);
    // ---- exclusive scan of the chunk histogram (in place)
    {
      const int per = (nch + NT - 1) / NT;
      const int c0 = min(nch, tid * per), c1 = min(nch, c0 + per);
      int s = 0;
      for (int i = c0; i < c1; ++i) s += static_cast<int>(H[i]);
      int incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) sh.hscan[w] = incl;
      __syncthreads();
      int base = incl - s + warps_exclusive<NW>(sh.hscan, w);
      for (int i = c0; i < c1; ++i) {
        const int h = static_cast<int>(H[i]);
        H[i] = static_cast<uint32_t>(base);
        base += h;
      }
    }
    __syncthreads();
    SEL_MARK(ti_, 7);
    for (int g = tid; g < kk; g += NT) {
      const int x = cidx[g];
      const int ch = x >> 5;
      const int pos = static_cast<int>(H[ch]) + g - static_cast<int>(G0[ch]);
      out[pos] = x;
      if (want_scores) outs[pos] = csc[g];
    }
    for (int i = kk + tid; i < k; i += NT) {
      out[i] = -1;
      if (outs) outs[i] = -INFINITY;
    }
    SEL_MARK(ti_, 8);
    if (tid == 0 && flags) flags[t] = 0;
  }
}

#ifdef MISA_SEL_TRACE
extern "C" int misa_debug_sel_trace(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_sel_trace, sizeof(g_sel_trace)) == cudaSuccess ? 0 : -2;
}
#endif

// ------------------------------------------------------- dense rows ----
template <int NT, int EPT, bool HI, bool WS>  // HI: explicit indices (idx), WS: scores returned
__global__ void __launch_bounds__(NT, (NT <= 256 ? 3 : 1)) dense_reg_kernel(const float* __restrict__ s, int64_t ld,
                                                       const int32_t* __restrict__ idx, int64_t idx_ld,
                                                       const int32_t* __restrict__ row_len,
                                                       const int32_t* __restrict__ rows, int k,
                                                       int32_t* __restrict__ topk, int64_t topk_ld,
                                                       float* __restrict__ topk_scores,
                                                       const int32_t* __restrict__ runs = nullptr) {
  // runs (optional): the row is kQuadrants consecutive ascending runs of these lengths
  // (misa_select_topk_runs output) instead of one ascending list
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ SelSh<NT> sh;
  const int rr = rows ? rows[blockIdx.x] : blockIdx.x;
  const int n = min(row_len[rr], (int)ld);  // candidate counts may exceed the staged capacity
  const float* row = s + (int64_t)rr * ld;
  const int32_t* irow = HI ? idx + (int64_t)rr * idx_ld : nullptr;
  int32_t* out = topk + (int64_t)rr * topk_ld;
  float* outs = WS ? topk_scores + (int64_t)rr * topk_ld : nullptr;
  const int kk = n < k ? n : k;
  if (kk <= 0) {
    for (int i = threadIdx.x; i < k; i += NT) {
      out[i] = -1;
      if (outs) outs[i] = -INFINITY;
    }
    return;
  }
  int NL = 1;
  if (runs) {
    NL = kQuadrants;
    if (threadIdx.x == 0) {
      int o = 0;
      for (int q = 0; q < kQuadrants; ++q) {
        sh.lst_off[q] = min(o, n);
        o += runs[(int64_t)rr * kQuadrants + q];
      }
      sh.lst_off[kQuadrants] = n;
    }
  } else if (threadIdx.x == 0) {
    sh.lst_off[0] = 0;
    sh.lst_off[1] = n;
  }
  int32_t* sidx = reinterpret_cast<int32_t*>(dsm);
  int32_t* cidx = sidx + NT * EPT;
  float* csc = reinterpret_cast<float*>(cidx + 2 * k);
  auto load = [&](auto& key, int32_t* si) {
    constexpr int E = sizeof(key) / sizeof(key[0]);
    float x[E];
    int32_t ix[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int e = v3_elem<NT, E>(r);
      const int ec = e < n ? e : 0;
      x[r] = row[ec];
      ix[r] = HI ? irow[ec] : e;
    }
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int e = v3_elem<NT, E>(r);
      key[r] = e < n ? float_key(x[r]) : 0u;
      if (e < n) si[e] = ix[r];
    }
  };
  v3_dispatch<NT, EPT>(n, load, NL, kk, sh, sidx, cidx, outs ? csc : nullptr, out, outs, k);
}

// Global path for rows longer than the register capacity (exact fallback): MSB radix
// passes over global memory with smem histograms, then rank-by-comparison ordering.
constexpr int kGlbThreads = 256;
constexpr int kGlbBins = 2048;
struct GlbShared {
  uint32_t hist[kGlbBins];
  uint32_t red[kGlbThreads / 32], red2[kGlbThreads / 32];
  int info[4];
};

template <typename KeyFn>
__device__ uint32_t glb_radix_select(KeyFn key_of, int N, int j, GlbShared& sh, int* j_rem_out, int* cnt_eq_out) {
  // j-th largest key of a long row streamed from global by one CTA: a min/max pass, then
  // affine windows of 2048 bins over [lo, hi] (scores spread over many bins, so the smem
  // atomics rarely collide), each level narrowing to the boundary bin until it is a
  // single key value.  Returns the value; *j_rem_out = rank of the cut among the keys
  // equal to it, *cnt_eq_out = how many keys equal it.
  constexpr int NW = kGlbThreads / 32, NB = kGlbBins, BPT = NB / kGlbThreads;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t mn = 0xffffffffu, mx = 0u;
  for (int i0 = threadIdx.x; i0 < N; i0 += kGlbThreads * 8) {
    uint32_t kv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * kGlbThreads;
      kv[u] = i < N ? key_of(i) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + u * kGlbThreads < N) {
        mn = min(mn, kv[u]);
        mx = max(mx, kv[u]);
      }
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    sh.red[w] = mn;
    sh.red2[w] = mx;
  }
  __syncthreads();
  mn = sh.red[0];
  mx = sh.red2[0];
  for (int i = 1; i < NW; ++i) {
    mn = min(mn, sh.red[i]);
    mx = max(mx, sh.red2[i]);
  }
  uint32_t lo = mn, span = mx - mn;  // window [lo, lo + span]
  const int need = j;  // absolute rank: keys above the window are counted in every level
  for (;;) {
    if (span == 0u) {  // one key value left: count the keys equal to / above it
      int ceq = 0, cgt = 0;
      for (int i = threadIdx.x; i < N; i += kGlbThreads) {
        const uint32_t kv = key_of(i);
        ceq += kv == lo;
        cgt += kv > lo;
      }
      ceq = __reduce_add_sync(0xffffffffu, ceq);
      cgt = __reduce_add_sync(0xffffffffu, cgt);
      __syncthreads();
      if (lane == 0) {
        sh.red[w] = (uint32_t)ceq;
        sh.red2[w] = (uint32_t)cgt;
      }
      __syncthreads();
      int teq = 0, tgt = 0;
      for (int i = 0; i < NW; ++i) {
        teq += (int)sh.red[i];
        tgt += (int)sh.red2[i];
      }
      __syncthreads();
      *j_rem_out = j - tgt;
      *cnt_eq_out = teq;
      return lo;
    }
    const int sft = max(0, 32 - __clz(span) - 11);
    for (int i = threadIdx.x; i < NB; i += kGlbThreads) sh.hist[i] = 0;
    __syncthreads();
    int above = 0;
    for (int i0 = threadIdx.x; i0 < N; i0 += kGlbThreads * 8) {
      uint32_t kv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * kGlbThreads;
        kv[u] = i < N ? key_of(i) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (i0 + u * kGlbThreads < N && kv[u] >= lo) {
          const uint32_t d = kv[u] - lo;
          if (d <= span) atomicAdd(&sh.hist[d >> sft], 1u);
          else ++above;
        }
      }
    }
    above = __reduce_add_sync(0xffffffffu, above);
    if (lane == 0) sh.red[w] = (uint32_t)above;
    __syncthreads();
    int ab = 0;
    for (int i = 0; i < NW; ++i) ab += (int)sh.red[i];
    // thread owns bins [NB - BPT*(tid+1), NB - BPT*tid) (descending)
    uint32_t c[BPT];
    int tot = 0;
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
      c[i] = sh.hist[NB - 1 - (threadIdx.x * BPT + i)];
      tot += (int)c[i];
    }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) sh.red2[w] = (uint32_t)incl;
    __syncthreads();
    int ex = ab + incl - tot;
    for (int i = 0; i < w; ++i) ex += (int)sh.red2[i];
    if (ex < need && need <= ex + tot) {
#pragma unroll
      for (int i = 0; i < BPT; ++i) {
        if (ex < need && need <= ex + (int)c[i]) {
          sh.info[0] = NB - 1 - (threadIdx.x * BPT + i);
          sh.info[1] = ex;
        }
        ex += (int)c[i];
      }
    }
    __syncthreads();
    const uint32_t b = (uint32_t)sh.info[0];
    // the next window is bin b: [lo + (b << sft), lo + ((b + 1) << sft) - 1] within [lo, lo + span]
    lo += b << sft;
    span = min(span - (b << sft), sft >= 32 ? 0xffffffffu : ((1u << sft) - 1u));
    __syncthreads();
  }
}

__device__ void dense_global_row(const float* __restrict__ s, int64_t ld, const int32_t* __restrict__ idx,
                                 int64_t idx_ld, const int32_t* __restrict__ row_len, int r, int k,
                                 int32_t* __restrict__ topk, int64_t topk_ld, float* __restrict__ topk_scores) {
  __shared__ GlbShared sh;
  const int n = row_len[r];
  const float* row = s + (int64_t)r * ld;
  const int32_t* irow = idx ? idx + (int64_t)r * idx_ld : nullptr;
  int32_t* out = topk + (int64_t)r * topk_ld;
  float* outs = topk_scores ? topk_scores + (int64_t)r * topk_ld : nullptr;
  auto key_of = [&](int i) -> uint32_t { return float_key(row[i]); };
  auto idx_of = [&](int i) -> int { return irow ? irow[i] : i; };
  const int kk = n < k ? n : k;
  uint32_t v = 0;
  int thr = 0x7fffffff;
  if (kk > 0 && kk < n) {
    int j_rem, cnt_eq;
    v = glb_radix_select(key_of, n, kk, sh, &j_rem, &cnt_eq);
    if (j_rem < cnt_eq) {
      int jr2, ce2;
      auto tie_key = [&](int i) -> uint32_t { return key_of(i) == v ? ~(uint32_t)idx_of(i) : 0u; };
      thr = (int)~glb_radix_select(tie_key, n, j_rem, sh, &jr2, &ce2);
    }
  }
  // ordered compaction: 16 consecutive candidates per thread per round (thread-major), one
  // block scan per round, so the output is ascending without a sort
  constexpr int kPer = 16, kRound = kGlbThreads * kPer;
  constexpr int NW = kGlbThreads / 32;
  __shared__ int wtot[NW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int base = 0;
  for (int r0 = 0; r0 < n && base < kk; r0 += kRound) {
    const int i0 = r0 + threadIdx.x * kPer;
    uint32_t selm = 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int i = i0 + e;
      if (i < n) {
        const uint32_t kv = key_of(i);
        const bool sel = kk >= n || kv > v || (kv == v && idx_of(i) <= thr);
        selm |= (sel ? 1u : 0u) << e;
      }
    }
    const int c = __popc(selm);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wtot[w] = incl;
    __syncthreads();
    int pos = base + incl - c;
    int tot = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      pos += i < w ? wtot[i] : 0;
      tot += wtot[i];
    }
    while (selm) {
      const int e = __ffs(selm) - 1;
      selm &= selm - 1;
      if (pos < kk) {
        out[pos] = idx_of(i0 + e);
        if (outs) outs[pos] = row[i0 + e];
      }
      ++pos;
    }
    base += tot;
    __syncthreads();
  }
  for (int i = kk + threadIdx.x; i < k; i += kGlbThreads) {
    out[i] = -1;
    if (outs) outs[i] = -INFINITY;
  }
}

__global__ void __launch_bounds__(kGlbThreads) dense_global_kernel(const float* __restrict__ s, int64_t ld,
                                                                   const int32_t* __restrict__ idx, int64_t idx_ld,
                                                                   const int32_t* __restrict__ row_len,
                                                                   const int32_t* __restrict__ rows, int k,
                                                                   int32_t* __restrict__ topk, int64_t topk_ld,
                                                                   float* __restrict__ topk_scores) {
  dense_global_row(s, ld, idx, idx_ld, row_len, rows ? rows[blockIdx.x] : blockIdx.x, k, topk, topk_ld, topk_scores);
}

// ------------------------------------------- long dense rows, many CTAs ----
// Decode rows (few rows x up to 1M keys): a 1/32-strided sample gives tau_t (as in the
// fused prefill selector), every CTA then counts and compacts its 4096-key segment's
// scores >= tau_t in index order into the row's candidate list (two passes, all SMs),
// and the register selector finishes on <= cap candidates.  Rows whose candidates
// under/overflow are flagged for the single-CTA exact path.
constexpr int kSegThreads = 256, kSegPer = 16, kSeg = kSegThreads * kSegPer;

// The thread's kSegPer consecutive scores of a segment (index order within the thread):
// four 16-byte loads when the row is aligned and the slice is inside the row.
__device__ __forceinline__ void seg_load(const float* __restrict__ row, int i0, int n, bool vec, float (&x)[kSegPer]) {
  if (vec && i0 + kSegPer <= n) {
    const float4* r4 = reinterpret_cast<const float4*>(row + i0);
#pragma unroll
    for (int v = 0; v < kSegPer / 4; ++v) {
      const float4 f = __ldg(r4 + v);
      x[4 * v] = f.x;
      x[4 * v + 1] = f.y;
      x[4 * v + 2] = f.z;
      x[4 * v + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < kSegPer; ++e) x[e] = i0 + e < n ? row[i0 + e] : -INFINITY;
  }
}

__global__ void __launch_bounds__(kSegThreads) seg_count_kernel(const float* __restrict__ s, int64_t ld,
                                                               const int32_t* __restrict__ row_len,
                                                               const float* __restrict__ tau,
                                                               int32_t* __restrict__ seg_cnt, int n_seg) {
  const int t = blockIdx.y, sg = blockIdx.x;
  const int n = row_len[t];
  const float tv = tau[t];
  const float* row = s + (int64_t)t * ld;
  const int i0 = sg * kSeg + threadIdx.x * kSegPer;
  const bool vec = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(s) & 15) == 0);
  float x[kSegPer];
  seg_load(row, i0, n, vec, x);
  int c = 0;
#pragma unroll
  for (int e = 0; e < kSegPer; ++e) c += (i0 + e < n) && x[e] >= tv;
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int ws[kSegThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int i = 0; i < kSegThreads / 32; ++i) tot += ws[i];
    seg_cnt[(int64_t)t * n_seg + sg] = tot;
  }
}

__global__ void __launch_bounds__(kSegThreads) seg_compact_kernel(const float* __restrict__ s, int64_t ld,
                                                                 const int32_t* __restrict__ row_len,
                                                                 const float* __restrict__ tau,
                                                                 const int32_t* __restrict__ seg_cnt, int n_seg,
                                                                 float* __restrict__ cs, int32_t* __restrict__ ci,
                                                                 int cap, int32_t* __restrict__ cnt_out) {
  constexpr int NW = kSegThreads / 32;
  __shared__ int ws[NW];
  __shared__ int sbase;
  const int t = blockIdx.y, sg = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n = row_len[t];
  const float tv = tau[t];
  const float* row = s + (int64_t)t * ld;
  // base = candidates of the row's earlier segments
  int b = 0;
  for (int i = threadIdx.x; i < sg; i += kSegThreads) b += seg_cnt[(int64_t)t * n_seg + i];
  b = __reduce_add_sync(0xffffffffu, b);
  if (lane == 0) ws[w] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int i = 0; i < NW; ++i) tot += ws[i];
    sbase = tot;
  }
  __syncthreads();
  const int base = sbase;
  const int i0 = sg * kSeg + threadIdx.x * kSegPer;
  const bool vec = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(s) & 15) == 0);
  float x[kSegPer];
  seg_load(row, i0, n, vec, x);
  uint32_t selm = 0;
#pragma unroll
  for (int e = 0; e < kSegPer; ++e) selm |= ((i0 + e < n) && x[e] >= tv ? 1u : 0u) << e;
  const int c = __popc(selm);
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  int pos = base + incl - c;
  for (int i = 0; i < w; ++i) pos += ws[i];
#pragma unroll
  for (int e = 0; e < kSegPer; ++e) {
    if ((selm >> e) & 1u) {
      if (pos < cap) {
        cs[(int64_t)t * cap + pos] = x[e];
        ci[(int64_t)t * cap + pos] = i0 + e;
      }
      ++pos;
    }
  }
  if (sg == n_seg - 1 && threadIdx.x == kSegThreads - 1) cnt_out[t] = pos;  // row total (may exceed cap)
}

// Rows whose candidate count is outside [min(k, n), cap] are re-selected exactly by the
// single-CTA path (the others exit at once), so no host round trip is needed.
__global__ void __launch_bounds__(kGlbThreads) seg_fixup_kernel(const float* __restrict__ s, int64_t ld,
                                                               const int32_t* __restrict__ row_len,
                                                               const int32_t* __restrict__ cnt, int cap, int k,
                                                               int32_t* __restrict__ topk, int64_t topk_ld,
                                                               float* __restrict__ topk_scores) {
  const int t = blockIdx.x;
  const int n = row_len[t];
  const int c = cnt[t];
  if (c >= (n < k ? n : k) && c <= cap) return;
  dense_global_row(s, ld, nullptr, 0, row_len, t, k, topk, topk_ld, topk_scores);
}

// -------------------------------------------------- multi-GPU merge ----
template <int NT, int EPT>
__global__ void __launch_bounds__(NT) merge_kernel(const float* __restrict__ ps, const int32_t* __restrict__ pi,
                                                   int n_parts, int64_t part_stride, int k_in, int k,
                                                   int32_t* __restrict__ topk, int64_t topk_ld,
                                                   float* __restrict__ topk_scores) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ SelSh<NT> sh;
  const int t = blockIdx.x;
  // each part's list is ascending with -1 padding at the end; its valid prefix is a list
  if (threadIdx.x < 32) {
    int acc = 0;
    for (int p = 0; p < n_parts; ++p) {
      const int32_t* pidx = pi + p * part_stride + (int64_t)t * k_in;
      int valid = 0;
      for (int i = threadIdx.x; i < k_in; i += 32) valid += pidx[i] >= 0;
      valid = __reduce_add_sync(0xffffffffu, valid);
      if (threadIdx.x == 0) sh.lst_off[p] = acc;
      acc += valid;
    }
    if (threadIdx.x == 0) sh.lst_off[n_parts] = acc;
  }
  __syncthreads();
  const int N = sh.lst_off[n_parts];
  int32_t* out = topk + (int64_t)t * topk_ld;
  float* outs = topk_scores ? topk_scores + (int64_t)t * topk_ld : nullptr;
  const int kk = N < k ? N : k;
  if (kk <= 0) {
    for (int i = threadIdx.x; i < k; i += NT) {
      out[i] = -1;
      if (outs) outs[i] = -INFINITY;
    }
    return;
  }
  int32_t* sidx = reinterpret_cast<int32_t*>(dsm);
  int32_t* cidx = sidx + NT * EPT;
  float* csc = reinterpret_cast<float*>(cidx + 2 * k);
  auto load = [&](auto& key, int32_t* si) {
    constexpr int E = sizeof(key) / sizeof(key[0]);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int e = v3_elem<NT, E>(r);
      key[r] = 0u;
      if (e < N) {
        int p = 0;
        while (p + 1 < n_parts && e >= sh.lst_off[p + 1]) ++p;
        const int64_t at = p * part_stride + (int64_t)t * k_in + (e - sh.lst_off[p]);
        key[r] = float_key(ps[at]);
        si[e] = pi[at];
      }
    }
  };
  v3_dispatch<NT, EPT>(N, load, n_parts, kk, sh, sidx, cidx, outs ? csc : nullptr, out, outs, k);
}

// m-th largest score of each row's list (-inf entries are padding): block-wide bit search.
template <int NT, int EPT>
__global__ void __launch_bounds__(NT) list_kth_kernel(const float* __restrict__ s, int64_t ld, int n_cols, int m,
                                                      float* __restrict__ tau) {
  __shared__ SelSh<NT> sh;
  const float* row = s + (int64_t)blockIdx.x * ld;
  uint32_t key[EPT];
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int i = r * NT + threadIdx.x;
    const float v = i < n_cols ? row[i] : -INFINITY;
    key[r] = v == -INFINITY ? 0u : float_key(v);
  }
  int parity = 0;
  const int nv = block_count<NT, EPT>([&](int r) { return key[r] != 0u; }, sh, parity);
  if (nv < m) {  // block-uniform
    if (threadIdx.x == 0) tau[blockIdx.x] = -INFINITY;
    return;
  }
  int cge, cgt;
  const uint32_t v = kth_largest<NT, EPT>([&](int r) { return key[r]; }, m, sh, parity, &cge, &cgt);
  if (threadIdx.x == 0) tau[blockIdx.x] = key_float(v);
}

// Stable compaction of the entries >= tau (one CTA per row, NT-wide tiles in order).
template <int NT>
__global__ void __launch_bounds__(NT) list_prune_kernel(const float* __restrict__ s, const int32_t* __restrict__ ix,
                                                        int64_t ld, int n_cols, const float* __restrict__ tau, int cap,
                                                        float* __restrict__ os, int32_t* __restrict__ oi,
                                                        int32_t* __restrict__ count) {
  constexpr int NW = NT / 32;
  __shared__ int wsum[NW];
  const int t = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float th = tau[t];
  const float* srow = s + (int64_t)t * ld;
  const int32_t* irow = ix + (int64_t)t * ld;
  float* orow_s = os + (int64_t)t * cap;
  int32_t* orow_i = oi + (int64_t)t * cap;
  int base = 0;
  for (int c0 = 0; c0 < n_cols; c0 += NT) {
    const int i = c0 + threadIdx.x;
    float v = -INFINITY;
    int32_t id = -1;
    if (i < n_cols) {
      v = srow[i];
      id = irow[i];
    }
    const bool keep = id >= 0 && v >= th;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    const int pos = base + warps_exclusive<NW>(wsum, w) + __popc(bal & ptx::lanemask_lt());
    if (keep && pos < cap) {
      orow_s[pos] = v;
      orow_i[pos] = id;
    }
    int tot = 0;
#pragma unroll
    for (int j = 0; j < NW; ++j) tot += wsum[j];
    base += tot;
    __syncthreads();
  }
  for (int p = base + threadIdx.x; p < cap; p += NT) {
    orow_s[p] = -INFINITY;
    orow_i[p] = -1;
  }
  if (threadIdx.x == 0) count[t] = base;
}

// Block-cyclic key shard: local key i of `rank` is global key ((i / bs) * G + rank) * bs + i % bs.
__global__ void shard_map_kernel(int32_t* idx, int64_t n, int bs, int G, int rank) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = idx[i];
  if (x >= 0) idx[i] = ((x / bs) * G + rank) * bs + x % bs;
}

}  // namespace misa

using namespace misa;

extern "C" int misa_shard_map_indices(int32_t* idx, int64_t n, int block, int n_shards, int shard, void* stream) {
  MISA_REQUIRE(idx && n >= 0 && block >= 1 && n_shards >= 1 && shard >= 0 && shard < n_shards,
               "bad shard map arguments");
  if (n == 0) return MISA_OK;
  shard_map_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(idx, n, block, n_shards, shard);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

namespace {
// register-capacity configurations: (threads, elements per thread)
template <template <int, int> class Launch, typename... Args>
int dispatch_capacity(int64_t n, cudaStream_t st, Args... args) {
  if (n <= 256 * 8) return Launch<256, 8>::go(st, args...);
  if (n <= 256 * 16) return Launch<256, 16>::go(st, args...);
  if (n <= 256 * 24) return Launch<256, 24>::go(st, args...);
  if (n <= 256 * 32) return Launch<256, 32>::go(st, args...);
  if (n <= 512 * 32) return Launch<512, 32>::go(st, args...);
  return -100;  // caller falls back
}

template <typename K>
static unsigned persistent_grid(K kern, int nt, int64_t rows, bool persistent = true) {
  if (!persistent) return (unsigned)rows;  // one CTA per row
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  return (unsigned)std::min<int64_t>(rows, (int64_t)sm_count() * per_sm);
}

template <int NT, int EPT>
struct ThresholdStepL {  // samples every `stride`-th element of a dense row
  static int go(cudaStream_t st, const float* s, int64_t ld, const int32_t* pl, int64_t T, int stride, int k,
                float beta, int64_t aa, float* tau) {
    threshold_kernel<NT, EPT><<<persistent_grid(threshold_kernel<NT, EPT>, NT, T, NT * EPT <= 4096), NT, 0, st>>>(
        s, ld, pl, (int)T, stride, k, beta, aa, tau, stride);
    MISA_LAUNCH_CHECK();
    return MISA_OK;
  }
};

template <int NT, int EPT>
struct TopkL {
  static int go(cudaStream_t st, const uint64_t* cand, const int32_t* cc, int cap, const int32_t* pl, int64_t T,
                int k, int32_t* topk, int64_t ld, float* ts, int32_t* flags) {
    const size_t base = (size_t)NT * EPT * 4 + (size_t)k * (ts ? 16 : 8);
    const size_t staged = base + (size_t)kQuadrants * cap * 8;
    if (staged <= 110 * 1024) return run<true>(st, staged, cand, cc, cap, pl, T, k, topk, ld, ts, flags);
    MISA_REQUIRE(base <= 200 * 1024, "selector working set %zu B exceeds shared memory (k %d)", base, k);
    return run<false>(st, base, cand, cc, cap, pl, T, k, topk, ld, ts, flags);
  }
  template <bool PF>
  static int run(cudaStream_t st, size_t bytes, const uint64_t* cand, const int32_t* cc, int cap, const int32_t* pl,
                 int64_t T, int k, int32_t* topk, int64_t ld, float* ts, int32_t* flags) {
    auto kern = topk_kernel<NT, EPT, PF>;
    MISA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    int per_sm = 0;
    MISA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, bytes));
    const int64_t grid = std::min<int64_t>(T, (int64_t)sm_count() * std::max(per_sm, 1));
    kern<<<(unsigned)grid, NT, bytes, st>>>(cand, cc, cap, pl, (int)T, k, topk, ld, ts, flags);
    MISA_LAUNCH_CHECK();
    return MISA_OK;
  }
};

template <int NT, int EPT>
struct DenseL {
  static int go(cudaStream_t st, const float* s, int64_t ld, const int32_t* idx, int64_t idx_ld,
                const int32_t* row_len, const int32_t* rows, int64_t n_rows, int k, int32_t* topk, int64_t tld,
                float* ts, const int32_t* runs = nullptr) {
    const size_t bytes = (size_t)NT * EPT * 4 + (size_t)k * 16;
    auto kern = idx ? (ts ? dense_reg_kernel<NT, EPT, true, true> : dense_reg_kernel<NT, EPT, true, false>)
                    : (ts ? dense_reg_kernel<NT, EPT, false, true> : dense_reg_kernel<NT, EPT, false, false>);
    MISA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    kern<<<(unsigned)n_rows, NT, bytes, st>>>(s, ld, idx, idx_ld, row_len, rows, k, topk, tld, ts, runs);
    MISA_LAUNCH_CHECK();
    return MISA_OK;
  }
};

template <int NT, int EPT>
struct MergeL {
  static int go(cudaStream_t st, const float* ps, const int32_t* pi, int n_parts, int64_t stride, int64_t T, int k_in,
                int k, int32_t* topk, int64_t ld, float* ts) {
    const size_t bytes = (size_t)NT * EPT * 4 + (size_t)k * 16;
    MISA_CUDA_TRY(cudaFuncSetAttribute(merge_kernel<NT, EPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    merge_kernel<NT, EPT><<<(unsigned)T, NT, bytes, st>>>(ps, pi, n_parts, stride, k_in, k, topk, ld, ts);
    MISA_LAUNCH_CHECK();
    return MISA_OK;
  }
};

template <int NT, int EPT>
struct ListKthL {
  static int go(cudaStream_t st, const float* s, int64_t ld, int64_t T, int n_cols, int m, float* tau) {
    list_kth_kernel<NT, EPT><<<(unsigned)T, NT, 0, st>>>(s, ld, n_cols, m, tau);
    MISA_LAUNCH_CHECK();
    return MISA_OK;
  }
};
// v5 selector when the quadrant capacity maps onto whole warps and the staging fits.
template <int NT, int EPT>
static int launch_topk5_t(cudaStream_t st, const uint64_t* cand, const int32_t* cc, int cap, const int32_t* pl,
                          int64_t T, int k, int n_chunks, int32_t* topk, int64_t ld, float* ts, int32_t* flags,
                          int32_t* runs) {
  // unordered (runs): no chunk histogram / compacted staging
  const size_t bytes = (size_t)kQuadrants * cap * 8 + (runs ? 0 : (size_t)n_chunks * 8 + (size_t)k * (ts ? 8 : 4));
  if (bytes > 200 * 1024) return -100;
  auto kern = runs ? (ts ? topk5_kernel<NT, EPT, true, true> : topk5_kernel<NT, EPT, false, true>)
                   : (ts ? topk5_kernel<NT, EPT, true, false> : topk5_kernel<NT, EPT, false, false>);
  MISA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  int per_sm = 0;
  MISA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, bytes));
  const int64_t grid = std::min<int64_t>(T, (int64_t)sm_count() * std::max(per_sm, 1));
  kern<<<(unsigned)grid, NT, bytes, st>>>(cand, cc, cap, pl, (int)T, k, n_chunks, topk, ld, ts, flags, runs);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

static int launch_topk5(cudaStream_t st, const uint64_t* cand, const int32_t* cc, int cap, const int32_t* pl,
                        int64_t T, int k, int64_t max_n, int32_t* topk, int64_t ld, float* ts, int32_t* flags,
                        int32_t* runs = nullptr) {
  const int64_t n_chunks = (max_n + 31) / 32;
  if ((!runs && n_chunks > 8192) || cap > 0xffff) return -100;  // unordered: no chunk histogram
  const int nc = static_cast<int>(n_chunks);
  // NT*EPT == 4*cap with cap a multiple of 32*EPT*(NT/128)
#define MISA_TOPK5_CASE(NT_, EPT_) \
  if (cap == NT_ * EPT_ / 4) return launch_topk5_t<NT_, EPT_>(st, cand, cc, cap, pl, T, k, nc, topk, ld, ts, flags, runs);
  MISA_TOPK5_CASE(256, 8)
  MISA_TOPK5_CASE(256, 16)
  MISA_TOPK5_CASE(512, 12)
  MISA_TOPK5_CASE(512, 16)
  MISA_TOPK5_CASE(256, 32)
  MISA_TOPK5_CASE(512, 24)
  MISA_TOPK5_CASE(512, 32)
#undef MISA_TOPK5_CASE
  return -100;
}

// Ascending sort of each row's first min(k, n_t) entries (bitonic in shared memory, P = the
// next power of two, padded with INT_MAX): turns an unordered selection (misa_select_topk_runs
// over lists whose chunks arrive in any order, e.g. key-split decode) into topk_tokens' output.
template <int NT>
__global__ void __launch_bounds__(NT) sort_rows_kernel(int32_t* __restrict__ rows, int64_t ld,
                                                      const int32_t* __restrict__ prefix_len, int k, int P) {
  extern __shared__ int32_t sv[];
  const int t = blockIdx.x;
  const int n = prefix_len[t];
  const int kk = n < k ? (n > 0 ? n : 0) : k;
  int32_t* row = rows + (int64_t)t * ld;
  for (int i = threadIdx.x; i < P; i += NT) sv[i] = i < kk ? row[i] : 0x7fffffff;
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += NT) {
        const int lo = 2 * i - (i & (stride - 1));  // index with bit `stride` clear
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const int32_t a = sv[lo], b = sv[hi];
        if ((a > b) == up) {
          sv[lo] = b;
          sv[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < kk; i += NT) row[i] = sv[i];
}

// runs[t] = (min(k, n_t), 0, 0, 0): one ascending run (rows selected by an ordered path)
__global__ void single_run_kernel(const int32_t* __restrict__ prefix_len, int64_t n_rows, int k,
                                  int32_t* __restrict__ runs) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n_rows) {
    const int n = prefix_len[t];
    *reinterpret_cast<int4*>(runs + 4 * t) = make_int4(n < k ? (n > 0 ? n : 0) : k, 0, 0, 0);
  }
}
}  // namespace

extern "C" int misa_select_threshold(const float* sample_scores, int64_t ld, const int32_t* prefix_len,
                                     int64_t n_rows, int key_stride, int k, float beta, int64_t append_all_len,
                                     float* tau, void* stream) {
  MISA_REQUIRE(sample_scores && prefix_len && tau, "null pointer");
  MISA_REQUIRE(k >= 1 && key_stride >= 1 && beta > 0.f && n_rows >= 1, "bad threshold arguments");
  // few rows (decode): one CTA per row over the contiguous sample (a warp per row would be
  // latency-bound: ~36 us for one 16384-sample row)
  if (n_rows * 2 <= sm_count() && ld <= 1024 * 16) {
    cudaStream_t st = as_stream(stream);
    if (ld <= 512 * 16)
      threshold_kernel<512, 16><<<(unsigned)n_rows, 512, 0, st>>>(sample_scores, ld, prefix_len, (int)n_rows,
                                                                  key_stride, k, beta, append_all_len, tau, 1);
    else
      threshold_kernel<1024, 16><<<(unsigned)n_rows, 1024, 0, st>>>(sample_scores, ld, prefix_len, (int)n_rows,
                                                                    key_stride, k, beta, append_all_len, tau, 1);
    MISA_LAUNCH_CHECK();
    return MISA_OK;
  }
  // one warp per row: 32 KB of histograms per 4-warp CTA, 6 CTAs (24 rows) per SM
  constexpr int WARPS = 4;
  auto kern = threshold_warp_kernel<WARPS>;
  int per_sm = 0;
  MISA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, 0));
  const int64_t grid = std::min<int64_t>((n_rows + WARPS - 1) / WARPS, (int64_t)sm_count() * std::max(per_sm, 1));
  kern<<<(unsigned)grid, WARPS * 32, 0, as_stream(stream)>>>(sample_scores, ld, prefix_len, (int)n_rows, key_stride,
                                                              k, beta, append_all_len, tau, 1);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_select_topk(const uint64_t* cand, const int32_t* cand_count, int cap, const int32_t* prefix_len,
                                int64_t n_rows, int k, int64_t max_prefix_len, int32_t* topk, int64_t topk_ld,
                                float* topk_scores, int32_t* flags, void* stream) {
  MISA_REQUIRE(cand && cand_count && prefix_len && topk, "null pointer");
  MISA_REQUIRE(k >= 1 && cap >= 1 && topk_ld >= k && n_rows >= 1, "bad top-k arguments");
  MISA_REQUIRE((int64_t)kQuadrants * cap <= 512 * 32, "candidate capacity %d exceeds the register selector", cap);
  MISA_REQUIRE((size_t)k * 16 <= 200 * 1024, "k too large");
  if (max_prefix_len > 0) {
    const int rc = launch_topk5(as_stream(stream), cand, cand_count, cap, prefix_len, n_rows, k, max_prefix_len, topk, topk_ld,
                      topk_scores, flags);
    if (rc != -100) return rc;
  }
  return dispatch_capacity<TopkL>((int64_t)kQuadrants * cap, as_stream(stream), cand, cand_count, cap, prefix_len,
                                  n_rows, k, topk, topk_ld, topk_scores, flags);
}

extern "C" int misa_select_topk_runs(const uint64_t* cand, const int32_t* cand_count, int cap,
                                     const int32_t* prefix_len, int64_t n_rows, int k, int64_t max_prefix_len,
                                     int32_t* topk, int64_t topk_ld, int32_t* runs, int32_t* flags, void* stream) {
  MISA_REQUIRE(cand && cand_count && prefix_len && topk && runs, "null pointer");
  MISA_REQUIRE(k >= 1 && cap >= 1 && topk_ld >= k && n_rows >= 1, "bad top-k arguments");
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(runs) & 15) == 0, "runs must be 16-byte aligned");
  if (max_prefix_len > 0) {
    const int rc = launch_topk5(as_stream(stream), cand, cand_count, cap, prefix_len, n_rows, k, max_prefix_len, topk,
                                topk_ld, nullptr, flags, runs);
    if (rc != -100) return rc;
  }
  // no unordered kernel for this capacity: the ascending selection is one run
  const int rc = misa_select_topk(cand, cand_count, cap, prefix_len, n_rows, k, max_prefix_len, topk, topk_ld,
                                  nullptr, flags, stream);
  if (rc) return rc;
  single_run_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, as_stream(stream)>>>(prefix_len, n_rows, k, runs);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_sort_rows(int32_t* rows, int64_t ld, const int32_t* prefix_len, int64_t n_rows, int k,
                              void* stream) {
  MISA_REQUIRE(rows && prefix_len, "null pointer");
  MISA_REQUIRE(k >= 1 && k <= 16384 && ld >= k && n_rows >= 0, "bad sort arguments (k <= 16384)");
  if (n_rows == 0) return MISA_OK;
  int P = 1;
  while (P < k) P <<= 1;
  const size_t bytes = (size_t)P * 4;
  MISA_CUDA_TRY(cudaFuncSetAttribute(sort_rows_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  sort_rows_kernel<1024><<<(unsigned)n_rows, 1024, bytes, as_stream(stream)>>>(rows, ld, prefix_len, k, P);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_select_dense(const float* scores, int64_t ld, const int32_t* idx, int64_t idx_ld,
                                 const int32_t* row_len, const int32_t* rows, int64_t n_rows, int k, int32_t* topk,
                                 int64_t topk_ld, float* topk_scores, void* stream) {
  MISA_REQUIRE(scores && row_len && topk, "null pointer");
  MISA_REQUIRE(k >= 1 && topk_ld >= k, "bad k");
  MISA_REQUIRE((size_t)k * 16 <= 200 * 1024, "k too large");
  if (n_rows <= 0) return MISA_OK;
  cudaStream_t st = as_stream(stream);
  int rc = dispatch_capacity<DenseL>(ld, st, scores, ld, idx, idx_ld, row_len, rows, n_rows, k, topk, topk_ld,
                                     topk_scores);
  if (rc != -100) return rc;
  dense_global_kernel<<<(unsigned)n_rows, kGlbThreads, 0, st>>>(scores, ld, idx, idx_ld, row_len, rows, k, topk,
                                                                 topk_ld, topk_scores);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_select_dense_runs(const float* scores, int64_t ld, const int32_t* idx, int64_t idx_ld,
                                      const int32_t* row_len, const int32_t* runs, int64_t n_rows, int k,
                                      int32_t* topk, int64_t topk_ld, void* stream) {
  MISA_REQUIRE(scores && idx && row_len && runs && topk, "null pointer");
  MISA_REQUIRE(k >= 1 && topk_ld >= k, "bad k");
  MISA_REQUIRE((size_t)k * 16 <= 200 * 1024, "k too large");
  if (n_rows <= 0) return MISA_OK;
  const int rc = dispatch_capacity<DenseL>(ld, as_stream(stream), scores, ld, idx, idx_ld, row_len, nullptr, n_rows,
                                           k, topk, topk_ld, nullptr, runs);
  MISA_REQUIRE(rc != -100, "row length %lld exceeds the register selector", (long long)ld);
  return rc;
}

extern "C" int misa_merge_topk(const float* part_scores, const int32_t* part_idx, int n_parts, int64_t part_stride,
                               int64_t n_rows, int k_in, int k, int32_t* topk, int64_t topk_ld, float* topk_scores,
                               void* stream) {
  MISA_REQUIRE(part_scores && part_idx && topk, "null pointer");
  MISA_REQUIRE(n_parts >= 1 && n_parts <= kMaxLists && k_in >= 1 && k >= 1 && topk_ld >= k, "bad merge arguments");
  MISA_REQUIRE((size_t)k * 16 <= 200 * 1024, "k too large");
  if (n_rows <= 0) return MISA_OK;
  const int rc = dispatch_capacity<MergeL>((int64_t)n_parts * k_in, as_stream(stream), part_scores, part_idx,
                                           n_parts, part_stride, n_rows, k_in, k, topk, topk_ld, topk_scores);
  MISA_REQUIRE(rc != -100, "n_parts*k_in exceeds the register selector");
  return rc;
}

extern "C" int misa_list_kth(const float* scores, int64_t ld, int64_t n_rows, int n_cols, int m, float* tau,
                             void* stream) {
  MISA_REQUIRE(scores && tau, "null pointer");
  MISA_REQUIRE(n_cols >= 1 && ld >= n_cols && m >= 1, "bad list_kth arguments");
  if (n_rows <= 0) return MISA_OK;
  const int rc = dispatch_capacity<ListKthL>(n_cols, as_stream(stream), scores, ld, n_rows, n_cols, m, tau);
  MISA_REQUIRE(rc != -100, "list length %d exceeds the register selector", n_cols);
  return rc;
}

extern "C" int misa_list_prune(const float* scores, const int32_t* idx, int64_t ld, int64_t n_rows, int n_cols,
                               const float* tau, int cap, float* out_scores, int32_t* out_idx, int32_t* count,
                               void* stream) {
  MISA_REQUIRE(scores && idx && tau && out_scores && out_idx && count, "null pointer");
  MISA_REQUIRE(n_cols >= 1 && ld >= n_cols && cap >= 1, "bad list_prune arguments");
  if (n_rows <= 0) return MISA_OK;
  list_prune_kernel<256><<<(unsigned)n_rows, 256, 0, as_stream(stream)>>>(scores, idx, ld, n_cols, tau, cap,
                                                                          out_scores, out_idx, count);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

static int misa_select_dense_clamped(const float* cs, int64_t ld, const int32_t* ci, int64_t ci_ld,
                                     const int32_t* cnt, int64_t n_rows, int k, int32_t* topk, int64_t topk_ld,
                                     float* topk_scores, cudaStream_t st) {
  // few rows (decode): twice the threads per row halves each row's latency
  if (n_rows * 2 <= sm_count() && ld <= 512 * 16)
    return DenseL<512, 16>::go(st, cs, ld, ci, ci_ld, cnt, nullptr, n_rows, k, topk, topk_ld, topk_scores);
  const int rc = dispatch_capacity<DenseL>(ld, st, cs, ld, ci, ci_ld, cnt, nullptr, n_rows, k, topk, topk_ld,
                                           topk_scores);
  MISA_REQUIRE(rc != -100, "candidate capacity %lld exceeds the register selector", (long long)ld);
  return rc;
}

extern "C" int misa_select_dense_long(const float* scores, int64_t ld, const int32_t* row_len, int64_t n_rows,
                                      int k, int64_t max_len, float beta, float* tau, int32_t* seg_cnt,
                                      float* cand_scores, int32_t* cand_idx, int32_t* cand_count, int cap,
                                      int32_t* topk, int64_t topk_ld, float* topk_scores, void* stream) {
  MISA_REQUIRE(scores && row_len && tau && seg_cnt && cand_scores && cand_idx && cand_count && topk, "null pointer");
  MISA_REQUIRE(k >= 1 && topk_ld >= k && n_rows >= 1 && max_len >= 1 && max_len <= ld, "bad arguments");
  MISA_REQUIRE(cap >= 2 * k && cap <= 16384, "candidate capacity must lie in [2k, 16384]");
  cudaStream_t st = as_stream(stream);
  const int stride = (int)std::max<int64_t>(32, (max_len + 16383) / 16384);  // <= 16384 samples per row
  const int64_t m = (max_len + stride - 1) / stride;
  // tau: ~2k of the row's keys pass; rows with n <= cap keep every key
  MISA_REQUIRE(beta >= 1.0f, "beta must be >= 1");
  const bool few = n_rows * 2 <= sm_count();  // decode: more threads per row, lower latency
  int rc = (few && m <= 512 * 16)
               ? ThresholdStepL<512, 16>::go(st, scores, ld, row_len, n_rows, stride, k, beta, (int64_t)cap, tau)
           : (few && m <= 1024 * 16)
               ? ThresholdStepL<1024, 16>::go(st, scores, ld, row_len, n_rows, stride, k, beta, (int64_t)cap, tau)
               : dispatch_capacity<ThresholdStepL>(m, st, scores, ld, row_len, n_rows, stride, k, beta, (int64_t)cap,
                                                   tau);
  MISA_REQUIRE(rc != -100, "long-row sample exceeds the register selector (max_len %lld)", (long long)max_len);
  if (rc) return rc;
  const int n_seg = (int)((max_len + kSeg - 1) / kSeg);
  dim3 grid(n_seg, (unsigned)n_rows);
  seg_count_kernel<<<grid, kSegThreads, 0, st>>>(scores, ld, row_len, tau, seg_cnt, n_seg);
  MISA_LAUNCH_CHECK();
  seg_compact_kernel<<<grid, kSegThreads, 0, st>>>(scores, ld, row_len, tau, seg_cnt, n_seg, cand_scores, cand_idx,
                                                   cap, cand_count);
  MISA_LAUNCH_CHECK();
  rc = misa_select_dense_clamped(cand_scores, cap, cand_idx, cap, cand_count, n_rows, k, topk, topk_ld, topk_scores,
                                 st);
  if (rc) return rc;
  seg_fixup_kernel<<<(unsigned)n_rows, kGlbThreads, 0, st>>>(scores, ld, row_len, cand_count, cap, k, topk, topk_ld,
                                                             topk_scores);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}
