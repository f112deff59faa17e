// K2: MISA head router (routing.py:38-75).
//
//   E_{t,j} = (1/M_t) * sum_{b < M_t} | w_{t,j} * ReLU(q_{t,j} . kbar_b) |,   M_t = ceil(n_t / B)
//   heads_t = top-h of E_t (ties -> smaller head), ascending
//
// K2a (misa_route_scores) is a tcgen05 GEMM with the flattened (row, head) query
// matrix on the UMMA M axis (128 (t,j) pairs per tile, TMA-loaded once — the Q
// read is the HBM bound of the router) and up to 128 pooled full blocks on N.
// The pooled means are f32; to keep the router at f32-grade precision they are
// split into three bf16 planes (hi + mid + lo == the f32 value exactly) and the
// K loop runs over the three planes into one accumulator, so
// q . kbar = q . hi + q . mid + q . lo with exact bf16 products and f32 sums.
// The epilogue thread owning (t, j) sums ReLU over the row's valid full blocks
// and, in chunk 0, adds the row's partial last block from the in-block prefix
// sums (mean over its real length, pooling.py:75-79).
//
// K2b (misa_route_select) applies |w| / M_t (or the gate_only / query_norm
// importances), then one warp per row picks the top-h heads with warp argmax
// rounds.
#include "common.cuh"
#include "ptx.cuh"

namespace misa {

struct RouteArgs {
  const __nv_bfloat16* __restrict__ q;
  const float* __restrict__ prefix;
  const int32_t* __restrict__ prefix_len;
  const int32_t* __restrict__ it_tile;
  const int32_t* __restrict__ it_chunk;
  const int32_t* __restrict__ it_ncols;
  // several key sequences (null: one): item i serves only the rows of its tile whose pooled
  // blocks start at it_boff[i] (row_boff[t] == it_boff[i]); chunks are relative to that block
  const int32_t* __restrict__ it_boff;
  const int32_t* __restrict__ row_boff;
  int n_items;
  int T, Hp, hp_log2, B;
  int64_t planes_rows;
  float* partial;  // [n_chunks][T][Hp]
};

template <int D>
struct RouteCfg {
  static constexpr int STAGES = 3;
  static constexpr int A_ATOM = 128 * 128;
  static constexpr int A_BYTES = A_ATOM * (D / 64);
  static constexpr int B_ATOM = 128 * 128;      // 128 pooled rows x 64 dims
  static constexpr int B_PLANE = B_ATOM * (D / 64);
  static constexpr int B_BYTES = 3 * B_PLANE;
  static constexpr int P_ROWS = 16;             // query rows per tile (Hp >= 8)
  static constexpr int P_BYTES = P_ROWS * D * 4;  // partial-block prefix rows of a tile
  static constexpr int NUM_THREADS = 192;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = STAGES * A_BYTES;
  static constexpr int OFF_P = OFF_B + B_BYTES;
  static constexpr int OFF_BAR = OFF_P + STAGES * P_BYTES;
  static constexpr int NUM_BARS = 2 * STAGES + 6;
  static constexpr int OFF_TMEM = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;
  static_assert(SMEM_BYTES <= 227 * 1024, "smem budget");
};

__device__ __forceinline__ int route_item(int it, int P, int b) { return (it & 1) ? (it + 1) * P - 1 - b : it * P + b; }

// A work item's metadata, loaded one item ahead by every role: each role walks the same
// item list and would otherwise pay a dependent global-load round trip per tile.
struct RouteItem {
  int idx, chunk, ncols, tile, boff;
};
__device__ __forceinline__ RouteItem load_route_item(const RouteArgs& a, int it, int P, int b) {
  RouteItem m;
  m.idx = route_item(it, P, b);
  m.chunk = m.ncols = m.tile = m.boff = 0;
  if (m.idx < a.n_items) {
    m.chunk = __ldg(a.it_chunk + m.idx);
    m.ncols = __ldg(a.it_ncols + m.idx);
    m.tile = __ldg(a.it_tile + m.idx);
    if (a.it_boff) m.boff = __ldg(a.it_boff + m.idx);
  }
  return m;
}
// Row t belongs to item m (same key sequence)?
__device__ __forceinline__ bool route_row_in(const RouteArgs& a, const RouteItem& m, int t) {
  return !a.row_boff || __ldg(a.row_boff + t) == m.boff;
}

template <int D>
__global__ void __launch_bounds__(192, 1)
    route_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_p,
                 const RouteArgs a) {
  using C = RouteCfg<D>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint8_t* sA = smem + C::OFF_A;
  uint8_t* sB = smem + C::OFF_B;
  float* sP = reinterpret_cast<float*>(smem + C::OFF_P);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full_a = bars;
  uint64_t* empty_a = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint64_t* bempty = bfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = gridDim.x, bid = blockIdx.x;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmap_q);
    ptx::tma_prefetch_desc(&tmap_p);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full_a[i], 1);
      ptx::mbar_init(&empty_a[i], 1 + 128);  // MMA commit + the epilogue's q / prefix reads
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 128);
    }
    ptx::mbar_init(bfull, 1);
    ptx::mbar_init(bempty, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 256);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // the whole warp produces: lane rr owns query row rr of the tile (<= 16 rows) and
    // stages its partial-block prefix row; lane 0 issues the tile loads
    const int rows = 128 >> a.hp_log2;
    auto row_n = [&](const RouteItem& m) {
      const int t = m.tile * rows + lane;
      return (m.idx < a.n_items && lane < rows && t < a.T && route_row_in(a, m, t)) ? __ldg(a.prefix_len + t) : 0;
    };
    int s = 0, cur_chunk = -1, cur_boff = -1, nb = 0;
    uint32_t ph = 0;
    RouteItem nx = load_route_item(a, 0, P, bid);
    int nx_n = row_n(nx);
    for (int it = 0;; ++it) {
      const RouteItem cu = nx;
      const int n = nx_n;
      if (cu.idx >= a.n_items) break;
      nx = load_route_item(a, it + 1, P, bid);
      nx_n = row_n(nx);
      const int chunk = cu.chunk, ncols = cu.ncols, tile = cu.tile;
      if (ncols == 0 && chunk != 0) continue;
      if (ncols > 0 && (chunk != cur_chunk || cu.boff != cur_boff)) {
        if (lane == 0) {
          if (nb > 0) ptx::mbar_wait(bempty, (nb - 1) & 1);
          ptx::mbar_arrive_expect_tx(bfull, C::B_BYTES);
          for (int p = 0; p < 3; ++p)
            for (int at = 0; at < D / 64; ++at)
              ptx::tma_load_2d(sB + p * C::B_PLANE + at * C::B_ATOM, &tmap_p, bfull, at * 64,
                               (int)(p * a.planes_rows + cu.boff + chunk * 128));
        }
        cur_chunk = chunk;
        cur_boff = cu.boff;
        ++nb;
      }
      // chunk 0 also stages each row's partial-block prefix sum P[n-1] for the epilogue
      const bool part = chunk == 0 && n % a.B != 0;  // n == 0 (padding rows) -> false
      const int np = __popc(__ballot_sync(0xffffffffu, part));
      if (lane == 0) {
        ptx::mbar_wait(&empty_a[s], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full_a[s], C::A_BYTES + np * D * 4);
        for (int at = 0; at < D / 64; ++at)
          ptx::tma_load_2d(sA + s * C::A_BYTES + at * C::A_ATOM, &tmap_q, &full_a[s], at * 64, tile * 128);
      }
      __syncwarp();  // stage s is free (lane 0 waited on it) before any lane writes it
      if (part)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                ptx::smem_u32(sP + (s * C::P_ROWS + lane) * D)),
            "l"(a.prefix + ((int64_t)cu.boff * a.B + n - 1) * D), "r"(D * 4), "r"(ptx::smem_u32(&full_a[s]))
            : "memory");
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    if (ptx::elect_one()) {
      int s = 0, acc = 0, cur_chunk = -1, cur_boff = -1, nb = 0;
      uint32_t ph = 0, aph = 0;
      const uint32_t b_base = ptx::smem_u32(sB);
      RouteItem nx = load_route_item(a, 0, P, bid);
      for (int it = 0;; ++it) {
        const RouteItem cu = nx;
        if (cu.idx >= a.n_items) break;
        nx = load_route_item(a, it + 1, P, bid);
        const int chunk = cu.chunk, ncols = cu.ncols;
        if (ncols == 0 && chunk != 0) continue;
        if (ncols == 0) {  // partial-block-only tile: no MMA, just hand the stage back
          ptx::mbar_wait(&full_a[s], ph);
          ptx::mbar_arrive(&empty_a[s]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
          continue;
        }
        if (chunk != cur_chunk || cu.boff != cur_boff) {
          if (nb > 0) ptx::mma_commit(bempty);  // all MMAs on the previous chunk's planes
          ptx::mbar_wait(bfull, nb & 1);
          ptx::tc_fence_after();
          cur_chunk = chunk;
          cur_boff = cu.boff;
          ++nb;
        }
        ptx::mbar_wait(&tempty[acc], aph ^ 1);
        ptx::mbar_wait(&full_a[s], ph);
        ptx::tc_fence_after();
        const uint32_t idesc = ptx::idesc_bf16_f32(128, ncols);
        const uint32_t a_base = ptx::smem_u32(sA + s * C::A_BYTES);
        const uint32_t d_tmem = tmem_base + acc * 128;
        for (int p = 0; p < 3; ++p) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = (kk & 3) * 32;
            const uint64_t ad = ptx::sw128_kmajor_desc(a_base + (kk >> 2) * C::A_ATOM + koff);
            const uint64_t bd = ptx::sw128_kmajor_desc(b_base + p * C::B_PLANE + (kk >> 2) * C::B_ATOM + koff);
            ptx::mma_bf16(d_tmem, ad, bd, idesc, (p | kk) ? 1u : 0u);
          }
        }
        ptx::mma_commit(&empty_a[s]);
        ptx::mma_commit(&tfull[acc]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else {
    const int quad = warp & 3;
    int acc = 0, s = 0;
    uint32_t aph = 0, ph = 0;
    const int lrow = quad * 32 + lane;  // A tile row = (t, j) pair
    auto row_len = [&](const RouteItem& m) {
      const int tt = (int)(((int64_t)m.tile * 128 + lrow) >> a.hp_log2);
      return (m.idx < a.n_items && tt < a.T && route_row_in(a, m, tt)) ? __ldg(a.prefix_len + tt) : -1;
    };
    RouteItem nx = load_route_item(a, 0, P, bid);
    int nx_n = row_len(nx);
    for (int it = 0;; ++it) {
      const RouteItem cu = nx;
      const int n = nx_n;
      if (cu.idx >= a.n_items) break;
      nx = load_route_item(a, it + 1, P, bid);
      nx_n = row_len(nx);
      const int chunk = cu.chunk, ncols = cu.ncols;
      if (ncols == 0 && chunk != 0) continue;
      const int64_t grow = (int64_t)cu.tile * 128 + lrow;
      const int t = (int)(grow >> a.hp_log2);
      const int j = (int)(grow & (a.Hp - 1));
      const bool mine = n >= 0;  // this row belongs to the item (n = -1: another sequence / past T)
      const int nf = mine ? n / a.B : 0;
      // partial last block first (it needs only the A stage, not the MMA): mean over keys
      // [nf*B, n) = P[n-1] / rem, with q from the A stage
      ptx::mbar_wait(&full_a[s], ph);
      float sum = 0.f;
      const int rem = mine ? n - nf * a.B : 0;
      if (mine && chunk == 0 && rem > 0) {
        const uint8_t* qa = sA + s * C::A_BYTES;
        const float4* pv = reinterpret_cast<const float4*>(sP + (s * C::P_ROWS + (lrow >> a.hp_log2)) * D);
        float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;  // four independent FMA chains
#pragma unroll 4
        for (int c = 0; c < D / 8; ++c) {
          const uint4 u = *reinterpret_cast<const uint4*>(qa + ptx::sw128_offset(lrow, c * 8, C::A_ATOM));
          const float4 p0 = pv[2 * c], p1 = pv[2 * c + 1];
          // bf16 -> f32 is exact bit placement: low half << 16, high half masked
          d0 = fmaf(__uint_as_float(u.x << 16), p0.x, d0); d0 = fmaf(__uint_as_float(u.x & 0xffff0000u), p0.y, d0);
          d1 = fmaf(__uint_as_float(u.y << 16), p0.z, d1); d1 = fmaf(__uint_as_float(u.y & 0xffff0000u), p0.w, d1);
          d2 = fmaf(__uint_as_float(u.z << 16), p1.x, d2); d2 = fmaf(__uint_as_float(u.z & 0xffff0000u), p1.y, d2);
          d3 = fmaf(__uint_as_float(u.w << 16), p1.z, d3); d3 = fmaf(__uint_as_float(u.w & 0xffff0000u), p1.w, d3);
        }
        const float dot = (d0 + d1) + (d2 + d3);
        sum = fmaxf(dot / (float)rem, 0.f);
      }
      if (ncols > 0) {
        ptx::mbar_wait(&tfull[acc], aph);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * 128;
        const int lim = nf - chunk * 128;  // valid columns for this row
        // every column slice in flight before one wait; four independent partial sums
        // (column i -> sum i % 4): one warp per SM sub-partition, so nothing may be serial
        uint32_t r[128];
#pragma unroll
        for (int c = 0; c < 128; c += 32)
          if (c < ncols) ptx::tmem_ld_x32p(taddr + c, r + c);  // ncols is uniform per item
#pragma unroll
        for (int c = 0; c < 128; c += 32)
          if (c < ncols) ptx::tmem_wait_ld_dep32p(r + c);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);  // accumulator drained: the next tile's MMA may start
        if (++acc == 2) { acc = 0; aph ^= 1; }
        // column i -> partial sum i % 4, kept as two packed pairs (FADD2); a slice wholly
        // inside the row's valid columns skips the per-column guard
        float2 pa = make_float2(0.f, 0.f), pb = make_float2(0.f, 0.f);
        auto relu = [&](int col) { return fmaxf(__uint_as_float(r[col]), 0.f); };
#pragma unroll
        for (int c = 0; c < 128; c += 32)
          if (c < ncols) {
            if (c + 32 <= lim) {
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                pa = __fadd2_rn(pa, make_float2(relu(c + i), relu(c + i + 1)));
                pb = __fadd2_rn(pb, make_float2(relu(c + i + 2), relu(c + i + 3)));
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                const int e = c + i;
                pa = __fadd2_rn(pa, make_float2(e < lim ? relu(e) : 0.f, e + 1 < lim ? relu(e + 1) : 0.f));
                pb = __fadd2_rn(pb, make_float2(e + 2 < lim ? relu(e + 2) : 0.f, e + 3 < lim ? relu(e + 3) : 0.f));
              }
            }
          }
        // summation order: blocks in column order, then the partial block last
        const float full = (pa.x + pa.y) + (pb.x + pb.y);
        sum = full + sum;
      }
      ptx::mbar_arrive(&empty_a[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
      if (mine) a.partial[((int64_t)chunk * a.T + t) * a.Hp + j] = sum;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, 256);
  }
}

// One warp per row: importance + top-h (value desc, head asc) -> ascending heads.
__global__ void route_select_kernel(const float* __restrict__ partial, int n_chunks, const float* __restrict__ w,
                                    const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ prefix_len,
                                    int T, int H, int Hp, int D, int B, int h, int kind, int32_t* __restrict__ heads,
                                    int heads_ld, float* __restrict__ importance) {
  const int warp_g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_g >= T) return;
  const int t = warp_g;
  const int n = prefix_len[t];
  const int M = (n + B - 1) / B;
  const int nf = n / B;
  const int nch = nf > 0 ? (nf + 127) / 128 : 1;
  float v[4];
  bool taken[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int j = lane + 32 * r;
    taken[r] = false;
    v[r] = -INFINITY;
    if (j < H) {
      const float wj = w[(int64_t)t * Hp + j];
      float e;
      if (kind == MISA_ROUTER_GATE_ONLY) {
        e = wj;
      } else if (kind == MISA_ROUTER_QUERY_NORM) {
        const __nv_bfloat16* qr = q + ((int64_t)t * Hp + j) * D;
        float ss = 0.f;
        for (int c = 0; c < D; ++c) {
          const float x = __bfloat162float(qr[c]);
          ss = fmaf(x, x, ss);
        }
        e = sqrtf(ss);
      } else {
        float s = 0.f;
        const int nc = nch < n_chunks ? nch : n_chunks;
        const float* pp = partial + (int64_t)t * Hp + j;
        const int64_t cs = (int64_t)T * Hp;
        int c = 0;
        for (; c + 4 <= nc; c += 4) {  // four loads in flight, summed in chunk order
          const float a0 = pp[c * cs], a1 = pp[(c + 1) * cs], a2 = pp[(c + 2) * cs], a3 = pp[(c + 3) * cs];
          s += a0;
          s += a1;
          s += a2;
          s += a3;
        }
        for (; c < nc; ++c) s += pp[c * cs];
        e = M > 0 ? fabsf(wj) * s / (float)M : 0.f;
      }
      v[r] = e != e ? -INFINITY : e;  // NaN never wins (and never breaks the argmax)
      if (importance) importance[(int64_t)t * Hp + j] = e;
    }
  }
  const int hh = h < H ? h : H;
  for (int round = 0; round < hh; ++round) {
    float best = -INFINITY;
    int bj = 0x7fffffff;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int j = lane + 32 * r;
      if (j < H && !taken[r] && (v[r] > best || (v[r] == best && j < bj) || bj == 0x7fffffff)) {
        best = v[r];
        bj = j;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
      if (oj != 0x7fffffff && (bj == 0x7fffffff || ob > best || (ob == best && oj < bj))) {
        best = ob;
        bj = oj;
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) taken[r] |= bj == lane + 32 * r;  // static indices: taken stays in registers
  }
  int base = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t bal = __ballot_sync(0xffffffffu, taken[r]);
    if (taken[r]) heads[(int64_t)t * heads_ld + base + __popc(bal & ptx::lanemask_lt())] = lane + 32 * r;
    base += __popc(bal);
  }
  for (int i = base + lane; i < heads_ld; i += 32) heads[(int64_t)t * heads_ld + i] = -1;
}

}  // namespace misa

using namespace misa;

// Work list: items (tile, chunk, ncols[, block offset]) precomputed on the host, chunk-major.
extern "C" int misa_route_scores_varlen(const void* queries, int64_t n_rows, int n_heads_pad, int head_dim,
                                        const void* pooled_planes, int64_t planes_rows, const float* prefix_sums,
                                        const int32_t* prefix_len, int block_size, const int32_t* it_tile,
                                        const int32_t* it_chunk, const int32_t* it_ncols, const int32_t* it_boff,
                                        const int32_t* row_boff, int n_items, float* partial, void* stream) {
  MISA_REQUIRE(queries && pooled_planes && prefix_sums && prefix_len && partial, "null pointer");
  MISA_REQUIRE(head_dim == 64 || head_dim == 128, "head_dim must be padded to 64 or 128");
  MISA_REQUIRE(n_heads_pad >= 8 && n_heads_pad <= 128 && (n_heads_pad & (n_heads_pad - 1)) == 0,
               "n_heads_pad must be a power of two in [8, 128] (<= 16 query rows per 128-row tile)");
  MISA_REQUIRE(block_size >= 1 && n_rows >= 1, "bad sizes");
  MISA_REQUIRE(n_items == 0 || (it_tile && it_chunk && it_ncols), "null work list");
  if (n_items == 0) return MISA_OK;
  CUtensorMap mq, mp;
  int rc = make_tmap_bf16_2d(&mq, queries, head_dim, (uint64_t)n_rows * n_heads_pad, head_dim, 128);
  if (rc) return rc;
  rc = make_tmap_bf16_2d(&mp, pooled_planes, head_dim, 3 * (uint64_t)planes_rows, head_dim, 128);
  if (rc) return rc;
  RouteArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(queries);
  a.prefix = prefix_sums;
  a.prefix_len = prefix_len;
  a.it_tile = it_tile;
  a.it_chunk = it_chunk;
  a.it_ncols = it_ncols;
  a.it_boff = it_boff;
  a.row_boff = row_boff;
  MISA_REQUIRE((it_boff == nullptr) == (row_boff == nullptr), "it_boff and row_boff go together");
  a.n_items = n_items;
  a.T = (int)n_rows;
  a.Hp = n_heads_pad;
  a.hp_log2 = __builtin_ctz(n_heads_pad);
  a.B = block_size;
  a.planes_rows = planes_rows;
  a.partial = partial;
  cudaStream_t st = as_stream(stream);
  const int grid = n_items < sm_count() ? n_items : sm_count();
  if (head_dim == 128) {
    MISA_CUDA_TRY(cudaFuncSetAttribute(route_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       RouteCfg<128>::SMEM_BYTES));
    route_kernel<128><<<grid, 192, RouteCfg<128>::SMEM_BYTES, st>>>(mq, mp, a);
  } else {
    MISA_CUDA_TRY(cudaFuncSetAttribute(route_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       RouteCfg<64>::SMEM_BYTES));
    route_kernel<64><<<grid, 192, RouteCfg<64>::SMEM_BYTES, st>>>(mq, mp, a);
  }
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_route_scores(const void* queries, int64_t n_rows, int n_heads_pad, int head_dim,
                                 const void* pooled_planes, int64_t planes_rows, const float* prefix_sums,
                                 const int32_t* prefix_len, int block_size, const int32_t* it_tile,
                                 const int32_t* it_chunk, const int32_t* it_ncols, int n_items, float* partial,
                                 void* stream) {
  return misa_route_scores_varlen(queries, n_rows, n_heads_pad, head_dim, pooled_planes, planes_rows, prefix_sums,
                                  prefix_len, block_size, it_tile, it_chunk, it_ncols, nullptr, nullptr, n_items,
                                  partial, stream);
}

extern "C" int misa_route_select(const float* partial, int n_chunks, const float* weights, const void* queries,
                                 const int32_t* prefix_len, int64_t n_rows, int n_heads, int n_heads_pad,
                                 int head_dim, int block_size, int h, int kind, int32_t* heads, int heads_ld,
                                 float* importance, void* stream) {
  MISA_REQUIRE(weights && prefix_len && heads, "null pointer");
  MISA_REQUIRE(kind >= 0 && kind <= 2, "unknown router kind %d", kind);
  MISA_REQUIRE(kind != MISA_ROUTER_BLOCK_ATTENTION || (partial && n_chunks >= 1), "null router partial sums");
  MISA_REQUIRE(kind != MISA_ROUTER_QUERY_NORM || queries, "null queries");
  MISA_REQUIRE(h >= 1, "h must be positive, got %d", h);
  MISA_REQUIRE(n_heads >= 1 && n_heads <= n_heads_pad && n_heads_pad <= 128, "bad head counts");
  MISA_REQUIRE(heads_ld >= (h < n_heads ? h : n_heads), "heads_ld too small");
  MISA_REQUIRE(block_size >= 1 && n_rows >= 1, "bad sizes");
  const int threads = 256;
  const int64_t blocks = (n_rows * 32 + threads - 1) / threads;
  route_select_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(
      partial, n_chunks, weights, static_cast<const __nv_bfloat16*>(queries), prefix_len, (int)n_rows, n_heads,
      n_heads_pad, head_dim, block_size, h, kind, heads, heads_ld, importance);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}
