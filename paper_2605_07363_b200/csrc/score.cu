// K3 (MISA gathered-head scoring) and K6 (dense DSA scoring) on tcgen05.
//
//   I_{t,s} = sum_j w_{t,j} * ReLU(q_{t,j} . k_s)          (dsa.py:37-61, routing.py:78-99)
//
// One UMMA tile is D[128 keys x 256 cols] = K_tile[128 x D] * Bq[256 x D]^T where
// the 256 columns are G = 256/HQ query rows x HQ head vectors (HQ = h routed heads
// for MISA, all H heads for DSA).  Keys ride the M axis so that every TMEM lane
// (one epilogue thread) owns one key and all heads of every query: the
// ReLU / gate / head-sum epilogue is in-register with no shuffles.
//
// Warp roles (64 + 32*EPI_WARPS threads, 1 CTA per SM, persistent over work items):
//   warp 0      TMA producer: 128-key tiles (box {64,128}, SWIZZLE_128B) into a
//               STAGES-deep smem ring (mbarrier full/empty)
//   warp 1      MMA issuer: one elected thread issues D/16 tcgen05.mma per tile
//               into a double-buffered TMEM accumulator (2 x 256 columns)
//   warps 2..   epilogue (16 warps, 8 when a query has 128 heads; warp w drains
//               TMEM lane quadrant w%4 and one column split): gather
//               the item's query/head vectors into smem (the B operand, resident
//               for the whole key scan), then per tile a software-pipelined
//               tcgen05.ld of the warp's whole column slice, early release of the
//               accumulator, ReLU * w * sum (packed FFMA2) -> either store
//               the score row (MATERIALIZE) or append (score, key) >= tau to the
//               row's per-quadrant candidate list (FILTER: the fused top-k's
//               candidate pass; each list in ascending key order, no cross-warp sync).
//
// A work item is a group of G consecutive query rows scanning key tiles
// [0, ceil(max_t lim_t / 128)) — causal rows skip every tile past their prefix.
#include "common.cuh"
#include "ptx.cuh"

namespace misa {

// Reduce one 16-column TMEM chunk (warp-local chunk C of its COLS columns) into the
// per-query scores sc[]: HQ columns per query row, gate weights from smem.
template <int HQ, int QW, int C>
__device__ __forceinline__ void reduce16(const uint32_t* r, const float* __restrict__ wcol, float (&sc)[QW],
                                         float2& p0, float2& p1) {
  const float4* w4 = reinterpret_cast<const float4*>(wcol + C * 16);
  if constexpr (HQ <= 16) {
    constexpr int QPC = 16 / HQ;
#pragma unroll
    for (int qq = 0; qq < QPC; ++qq) {
      float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < HQ; jj += 4) {
        const int b = qq * HQ + jj;
        gate_relu4(s0, s1, w4[b / 4], r[b], r[b + 1], r[b + 2], r[b + 3]);
      }
      sc[C * QPC + qq] = gate_relu_finish(s0, s1);
    }
  } else {
#pragma unroll
    for (int jj = 0; jj < 16; jj += 4) gate_relu4(p0, p1, w4[jj / 4], r[jj], r[jj + 1], r[jj + 2], r[jj + 3]);
    if constexpr (((C + 1) * 16) % HQ == 0) {
      sc[(C * 16) / HQ] = gate_relu_finish(p0, p1);
      p0 = make_float2(0.f, 0.f);
      p1 = make_float2(0.f, 0.f);
    }
  }
}

// Drain chunks [C, NCH) of a warp's COLS TMEM columns, x16 loads double-buffered.
template <int HQ, int QW, int NCH, int C>
__device__ __forceinline__ void drain(uint32_t taddr, const float* __restrict__ wcol, float (&sc)[QW], float2& p0,
                                      float2& p1, uint32_t (&ra)[16], uint32_t (&rb)[16]) {
  if constexpr (C < NCH) {
    if constexpr (C + 1 < NCH) ptx::tmem_ld_x16(taddr + (C + 1) * 16, (C & 1) ? ra : rb);
    reduce16<HQ, QW, C>((C & 1) ? rb : ra, wcol, sc, p0, p1);
    if constexpr (C + 1 < NCH) ptx::tmem_wait_ld_dep16((C & 1) ? ra : rb);
    drain<HQ, QW, NCH, C + 1>(taddr, wcol, sc, p0, p1, ra, rb);
  }
}

// Reduce a warp's whole register-resident column slice, chunk by chunk.
template <int HQ, int QW, int NCH, int C>
__device__ __forceinline__ void reduce_all(const uint32_t* r, const float* __restrict__ wcol, float (&sc)[QW],
                                           float2& p0, float2& p1) {
  if constexpr (C < NCH) {
    reduce16<HQ, QW, C>(r + C * 16, wcol, sc, p0, p1);
    reduce_all<HQ, QW, NCH, C + 1>(r, wcol, sc, p0, p1);
  }
}

// FILTER pass masks of one 32-key warp slice (lane = key): one ballot per query.
template <int QW, bool EDGE>
__device__ __forceinline__ void pass_ballots(const float (&sc)[QW], int key, const float* sTau, const int* sLim,
                                             uint32_t (&bal)[QW]) {
#pragma unroll
  for (int q = 0; q < QW; ++q) {
    bool pass = sc[q] >= sTau[q];
    if constexpr (EDGE) pass = pass && key < sLim[q];
    bal[q] = __ballot_sync(0xffffffffu, pass);
  }
}

// Pair layout: ballots of the 4 key slots (key = key0 + 8*s) x 2 queries (a, b).
template <bool EDGE>
__device__ __forceinline__ void pair_ballots(const float2 (&sc)[4], int key0, float tau_a, float tau_b,
                                             const int* sLim, uint32_t (&bal)[4][2]) {
#pragma unroll
  for (int s4 = 0; s4 < 4; ++s4) {
    bool pa = sc[s4].x >= tau_a, pb = sc[s4].y >= tau_b;
    if constexpr (EDGE) {
      pa = pa && key0 + 8 * s4 < sLim[0];
      pb = pb && key0 + 8 * s4 < sLim[1];
    }
    bal[s4][0] = __ballot_sync(0xffffffffu, pa);
    bal[s4][1] = __ballot_sync(0xffffffffu, pb);
  }
}

// Tile column r <-> (query within the item, head slot).  HQ = 8 uses the "pair"
// order (column 8g + q%8 of 64-column slab q/8 is head g of query q), so that a
// 16x256b TMEM load hands every thread all 8 heads of two queries (see gate_relu_pair8);
// other widths are query-major (r = q*HQ + j).
template <int HQ>
__device__ __forceinline__ int col_query(int r) {
  if constexpr (HQ == 8) return (r >> 6) * 8 + (r & 7);
  else return r / HQ;
}
template <int HQ>
__device__ __forceinline__ int col_head(int r) {
  if constexpr (HQ == 8) return (r >> 3) & 7;
  else return r % HQ;
}

struct ScoreArgs {
  const __nv_bfloat16* __restrict__ q;  // [T][Hp][D]
  const float* __restrict__ w;          // [T][Hp]
  const int32_t* __restrict__ heads;    // [T][HQ] or nullptr (dense: head j)
  const int32_t* __restrict__ prefix_len;
  const int32_t* __restrict__ items;
  const int32_t* __restrict__ item_tiles;
  const int32_t* __restrict__ item_tile0;  // MATERIALIZE key split: first tile of item i (null: 0)
  const int32_t* __restrict__ page_table;  // paged key cache: logical page -> physical page (null: flat)
  int page_tiles;                          // 128-key tiles per page
  // several key sequences in one call (null: one sequence, item i = rows [items[i]*G, +G)):
  // item i = rows [items[i], items[i] + item_nrows[i]) of one sequence whose keys start at
  // key row item_key0[i] of the key buffer (key indices stay sequence-relative)
  const int32_t* __restrict__ item_nrows;
  const int32_t* __restrict__ item_key0;
  int n_items;
  int T, H, Hp;
  int key_stride;
  float* out;
  int64_t out_ld;
  const float* __restrict__ tau;
  uint64_t* cand;
  int cap;
  int32_t* cand_count;
  // FILTER over key-split items (several items per row, misa_score_filter_split): each warp
  // reserves its tile's slots of a (row, quadrant) list with one atomicAdd on the zeroed
  // cand_count, so a 32-key chunk's candidates stay contiguous and ascending (the selector's
  // chunk-scan order needs no more) while the chunks of a list come in any order
  int cand_atomic;
};

template <int D, int HQ>
struct ScoreCfg {
  static constexpr int G = kTileCols / HQ;             // query rows per item
  static constexpr int SPLIT = (HQ <= 64) ? 4 : 2;     // column splits per TMEM quadrant
  static constexpr int EPI_WARPS = kQuadrants * SPLIT;  // 16 or 8
  static constexpr int EPI_THREADS = 32 * EPI_WARPS;
  static constexpr int COLS = kTileCols / SPLIT;       // TMEM columns per epilogue warp
  static constexpr int QW = COLS >= HQ ? COLS / HQ : 1;  // query rows per epilogue warp
  static constexpr int NCH = COLS / 16;
  static constexpr int STAGES = (D == 128) ? 4 : 6;
  static constexpr int A_ATOM = kTileKeys * 128;   // bytes of one 64-wide K atom of a key tile
  static constexpr int A_BYTES = A_ATOM * (D / 64);
  static constexpr int B_ATOM = kTileCols * 128;
  static constexpr int B_BYTES = B_ATOM * (D / 64);
  static constexpr int NUM_THREADS = 64 + EPI_THREADS;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
  static constexpr int OFF_W = OFF_B + B_BYTES;
  static constexpr int OFF_LIM = OFF_W + kTileCols * 4;
  static constexpr int OFF_TAU = OFF_LIM + 32 * 4;
  static constexpr int OFF_BAR = OFF_TAU + 32 * 4;
  static constexpr int NUM_BARS = 2 * STAGES + 5;
  static constexpr int OFF_TMEM = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;
  static_assert(G >= 2 && G <= 32, "2..32 query rows per tile");
  static_assert(QW * SPLIT == G, "query rows split evenly over the column splits");
  static_assert(SMEM_BYTES <= 227 * 1024, "smem budget");
};

__device__ __forceinline__ int item_index(int it, int P, int b) {
  // zigzag over CTAs: items are sorted longest first, so consecutive rounds
  // alternate direction to balance the per-CTA total.
  return (it & 1) ? (it + 1) * P - 1 - b : it * P + b;
}

template <int D, int HQ, bool FILTER>
__global__ void __launch_bounds__(ScoreCfg<D, HQ>::NUM_THREADS, 1)
    score_kernel(const __grid_constant__ CUtensorMap tmap_k, const ScoreArgs a) {
  using C = ScoreCfg<D, HQ>;
  constexpr int G = C::G, STAGES = C::STAGES, QW = C::QW, EPI_THREADS = C::EPI_THREADS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint8_t* sA = smem + C::OFF_A;
  uint8_t* sB = smem + C::OFF_B;
  float* sW = reinterpret_cast<float*>(smem + C::OFF_W);
  int* sLim = reinterpret_cast<int*>(smem + C::OFF_LIM);
  float* sTau = reinterpret_cast<float*>(smem + C::OFF_TAU);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full_a = bars;
  uint64_t* empty_a = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int P = gridDim.x, bid = blockIdx.x;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmap_k);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full_a[i], 1);
      ptx::mbar_init(&empty_a[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], EPI_THREADS);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (ptx::elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0;; ++it) {
        const int idx = item_index(it, P, bid);
        if (idx >= a.n_items) break;
        const int nt = a.item_tiles[idx];
        const int j0 = a.item_tile0 ? a.item_tile0[idx] : 0;
        const int key0 = a.item_key0 ? a.item_key0[idx] : 0;
        for (int j = 0; j < nt; ++j) {
          ptx::mbar_wait(&empty_a[s], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&full_a[s], C::A_BYTES);
          const int jj = j0 + j;  // logical tile -> row of the (possibly paged) key pool
          const int row = a.page_table ? a.page_table[jj / a.page_tiles] * (a.page_tiles * kTileKeys) +
                                             (jj % a.page_tiles) * kTileKeys
                                       : key0 + jj * kTileKeys;
#pragma unroll
          for (int at = 0; at < D / 64; ++at)
            ptx::tma_load_2d(sA + s * C::A_BYTES + at * C::A_ATOM, &tmap_k, &full_a[s], at * 64, row);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(kTileKeys, kTileCols);
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      const uint32_t b_base = ptx::smem_u32(sB);
      for (int it = 0;; ++it) {
        const int idx = item_index(it, P, bid);
        if (idx >= a.n_items) break;
        const int nt = a.item_tiles[idx];
        ptx::mbar_wait(bfull, it & 1);
        ptx::tc_fence_after();
        for (int j = 0; j < nt; ++j) {
          ptx::mbar_wait(&tempty[acc], aph ^ 1);
          ptx::mbar_wait(&full_a[s], ph);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(sA + s * C::A_BYTES);
          const uint32_t d_tmem = tmem_base + acc * kTileCols;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = (kk & 3) * 32;
            const uint64_t ad = ptx::sw128_kmajor_desc(a_base + (kk >> 2) * C::A_ATOM + koff);
            const uint64_t bd = ptx::sw128_kmajor_desc(b_base + (kk >> 2) * C::B_ATOM + koff);
            ptx::mma_bf16(d_tmem, ad, bd, idesc, kk > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&empty_a[s]);
          ptx::mma_commit(&tfull[acc]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
          if (++acc == 2) { acc = 0; aph ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------------ epilogue
    // warp w reads TMEM lane quadrant (w % 4) and column split (w - 2) / 4:
    // COLS columns = QW query rows of each 128 x 256 accumulator tile.
    const int e = warp - 2;
    const int et = threadIdx.x - 64;
    const int quad = warp & 3;
    const int split = e >> 2;
    int acc = 0;
    uint32_t aph = 0;
    for (int it = 0;; ++it) {
      const int idx = item_index(it, P, bid);
      if (idx >= a.n_items) break;
      const int nt = a.item_tiles[idx];
      const int j0 = a.item_tile0 ? a.item_tile0[idx] : 0;
      const int row0 = a.item_nrows ? a.items[idx] : a.items[idx] * G;
      // rows of this item: [row0, row_end) (a varlen item stops at its sequence's last row)
      const int row_end = min(a.T, row0 + (a.item_nrows ? a.item_nrows[idx] : G));

      // B operand: row r = q*HQ + j <- Q[row0+q][head(q,j)][:], SW128 K-major layout.
      constexpr int CH = D / 8;  // 16-byte chunks per row
      for (int c = et; c < kTileCols * CH; c += EPI_THREADS) {
        const int r = c / CH, ch = c - r * CH;
        const int qi = col_query<HQ>(r), j = col_head<HQ>(r);
        const int row = row0 + qi;
        int head = -1;
        if (row < row_end) head = a.heads ? a.heads[(int64_t)row * HQ + j] : (j < a.H ? j : -1);
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (head >= 0) v = *reinterpret_cast<const uint4*>(a.q + ((int64_t)row * a.Hp + head) * D + ch * 8);
        *reinterpret_cast<uint4*>(sB + ptx::sw128_offset(r, ch * 8, C::B_ATOM)) = v;
      }
      for (int r = et; r < kTileCols; r += EPI_THREADS) {
        const int qi = col_query<HQ>(r), j = col_head<HQ>(r);
        const int row = row0 + qi;
        float wv = 0.f;
        if (row < row_end) {
          const int head = a.heads ? a.heads[(int64_t)row * HQ + j] : (j < a.H ? j : -1);
          if (head >= 0) wv = a.w[(int64_t)row * a.Hp + head];
        }
        sW[r] = gate_stored(wv, col_head<HQ>(r));  // head slots 2, 3 of each group of four halved
      }
      if (et < G) {
        const int row = row0 + et;
        int lim = 0;
        float tau = 0.f;
        if (row < row_end) {
          const int n = a.prefix_len[row];
          lim = (n + a.key_stride - 1) / a.key_stride;
          if (FILTER) tau = a.tau[row];
        } else if (FILTER) {
          // no row here: nothing can pass (scores are finite), and the row must not pull the
          // item's diagonal-tile bound (lim_min) down to 0
          lim = 0x7fffffff;
          tau = __int_as_float(0x7f800000);  // +inf
        }
        sLim[et] = lim;
        sTau[et] = tau;
      }
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(1, EPI_THREADS);
      if (et == 0) ptx::mbar_arrive(bfull);

      if constexpr (HQ == 8) {
        // ---- pair layout: thread (rr = lane/4, m = lane%4) owns keys quad*32 + rr + 8s
        // (s = 0..3) of queries qa = split*8 + 2m and qa + 1, with all their 8 gate
        // weights in registers for the whole item (no shared-memory reads per tile).
        const int m = lane & 3, rr = lane >> 2;
        const int qa = split * 8 + 2 * m;
        float2 wp[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) wp[g] = *reinterpret_cast<const float2*>(sW + split * 64 + 8 * g + 2 * m);
        const float tau_a = sTau[qa], tau_b = sTau[qa + 1];
        int lim_min = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < 8; ++q) lim_min = min(lim_min, sLim[split * 8 + q]);
        const uint32_t gm = 0x11111111u << m;  // lanes of this query pair
        const uint32_t lm = gm & ptx::lanemask_lt();
        int cnt_a = 0, cnt_b = 0;  // candidates of rows qa / qa+1 appended by this warp
        uint64_t* dst = nullptr;   // list of (row, quad) = cand[(row*4 + quad) * cap]
        if (FILTER) dst = a.cand + (static_cast<int64_t>(row0 + qa) * kQuadrants + quad) * a.cap;
        const uint32_t qs = kQuadrants * a.cap;
        for (int jt = 0; jt < nt; ++jt) {
          ptx::mbar_wait(&tfull[acc], aph);
          ptx::tc_fence_after();
          const uint32_t taddr =
              tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * kTileCols + split * 64;
          uint32_t v0[32], v1[32];
          ptx::tmem_ld_16x256b_x8(taddr, v0);
          ptx::tmem_ld_16x256b_x8(taddr + (16u << 16), v1);
          ptx::tmem_wait_ld_dep32p(v0);
          ptx::tmem_wait_ld_dep32p(v1);
          ptx::tc_fence_before();
          ptx::mbar_arrive(&tempty[acc]);
          if (++acc == 2) { acc = 0; aph ^= 1; }
          float2 sc[4];
          sc[0] = gate_relu_pair8(v0, 0, wp);
          sc[1] = gate_relu_pair8(v0, 2, wp);
          sc[2] = gate_relu_pair8(v1, 0, wp);
          sc[3] = gate_relu_pair8(v1, 2, wp);
          const int kq = (j0 + jt) * kTileKeys + quad * 32;
          if constexpr (FILTER) {
            uint32_t bal[4][2];
            if (kq + 31 >= lim_min)  // warp-uniform: only the diagonal tile tests the prefix bound
              pair_ballots<true>(sc, kq + rr, tau_a, tau_b, sLim + qa, bal);
            else
              pair_ballots<false>(sc, kq + rr, tau_a, tau_b, sLim + qa, bal);
            if (a.cand_atomic) {
              // this tile's slots of rows qa / qa+1 (quadrant quad): lane m reserves for its pair group
#pragma unroll
              for (int b = 0; b < 2; ++b) {
                int tot = 0;
#pragma unroll
                for (int s4 = 0; s4 < 4; ++s4) tot += __popc(bal[s4][b] & gm);
                int base = 0;
                if (lane == m && tot > 0)
                  base = atomicAdd(a.cand_count + (static_cast<int64_t>(row0 + qa + b) * kQuadrants + quad), tot);
                base = __shfl_sync(0xffffffffu, base, m);
                (b ? cnt_b : cnt_a) = base;
              }
            }
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4) {
              const uint32_t key = static_cast<uint32_t>(kq + rr + 8 * s4);
#pragma unroll
              for (int b = 0; b < 2; ++b) {
                const uint32_t bl = bal[s4][b];
                int& cnt = b ? cnt_b : cnt_a;
                const int pos = cnt + __popc(bl & lm);
                ptx::st_global_v2_idx_if(dst, b * qs + pos, __float_as_uint(b ? sc[s4].y : sc[s4].x), key,
                                         ((bl >> lane) & 1u) && pos < a.cap);
                cnt += __popc(bl & gm);
              }
            }
          } else {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const int lim = sLim[qa + b];
              float* o = a.out + static_cast<int64_t>(row0 + qa + b) * a.out_ld;
#pragma unroll
              for (int s4 = 0; s4 < 4; ++s4) {
                const int key = kq + rr + 8 * s4;
                if (key < lim) o[key] = b ? sc[s4].y : sc[s4].x;
              }
            }
          }
        }
        if constexpr (FILTER) {
          if (rr == 0 && !a.cand_atomic) {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const int row = row0 + qa + b;
              if (row < row_end) a.cand_count[(int64_t)row * kQuadrants + quad] = b ? cnt_b : cnt_a;
            }
          }
        }
      } else {
        const int qbase = split * QW;  // first query row (within the item) of this warp
        int lim_min = 0x7fffffff;
  #pragma unroll
        for (int q = 0; q < QW; ++q) lim_min = min(lim_min, sLim[qbase + q]);
        const float* wcol = sW + split * C::COLS;
        // FILTER: cnt[q] = candidates of query qbase+q appended by this warp (warp-uniform)
        int cnt[QW];
  #pragma unroll
        for (int q = 0; q < QW; ++q) cnt[q] = 0;
        const uint32_t lt = ptx::lanemask_lt();
        uint64_t* dst0 = nullptr;  // list of query qbase+q = dst0 + q * qs
        if (FILTER) dst0 = a.cand + (static_cast<int64_t>(row0 + qbase) * kQuadrants + quad) * a.cap;
        const uint32_t qs = kQuadrants * a.cap;
        for (int jt = 0; jt < nt; ++jt) {
          ptx::mbar_wait(&tfull[acc], aph);
          ptx::tc_fence_after();
          const int key0 = (j0 + jt) * kTileKeys + quad * 32;
          const int key = key0 + lane;
          const uint32_t taddr =
              tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * kTileCols + split * C::COLS;
          float sc[QW];
          float2 p0 = make_float2(0.f, 0.f), p1 = make_float2(0.f, 0.f);
          if constexpr (C::COLS <= 64) {
            // whole column slice in registers at once: the accumulator buffer is handed
            // back to the MMA warp before any arithmetic, so the tensor pipe never waits
            // on the epilogue's latency, only on its throughput.
            uint32_t r[C::COLS];
  #pragma unroll
            for (int c = 0; c < C::COLS; c += 32) ptx::tmem_ld_x32p(taddr + c, r + c);
  #pragma unroll
            for (int c = 0; c < C::COLS; c += 32) ptx::tmem_wait_ld_dep32p(r + c);
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
            reduce_all<HQ, QW, C::NCH, 0>(r, wcol, sc, p0, p1);
          } else {
            uint32_t ra[16], rb[16];
            ptx::tmem_ld_x16(taddr, ra);
            ptx::tmem_wait_ld_dep16(ra);
            drain<HQ, QW, C::NCH, 0>(taddr, wcol, sc, p0, p1, ra, rb);
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
          }
          if (++acc == 2) { acc = 0; aph ^= 1; }

          if constexpr (FILTER) {
            uint32_t bal[QW];
            if (key0 + 31 >= lim_min)  // the prefix bound only matters on the diagonal tile
              pass_ballots<QW, true>(sc, key, sTau + qbase, sLim + qbase, bal);
            else
              pass_ballots<QW, false>(sc, key, sTau + qbase, sLim + qbase, bal);
            if (a.cand_atomic) {
#pragma unroll
              for (int q = 0; q < QW; ++q) {
                const int tot = __popc(bal[q]);
                int base = 0;
                if (lane == 0 && tot > 0)
                  base = atomicAdd(a.cand_count + (static_cast<int64_t>(row0 + qbase + q) * kQuadrants + quad), tot);
                cnt[q] = __shfl_sync(0xffffffffu, base, 0);
              }
            }
  #pragma unroll
            for (int q = 0; q < QW; ++q) {
              const int pos = cnt[q] + __popc(bal[q] & lt);
              ptx::st_global_v2_idx_if(dst0, q * qs + pos, __float_as_uint(sc[q]), static_cast<uint32_t>(key),
                                       ((bal[q] >> lane) & 1u) && pos < a.cap);
              cnt[q] += __popc(bal[q]);
            }
          } else {
            float* o = a.out + static_cast<int64_t>(row0 + qbase) * a.out_ld + key;
  #pragma unroll
            for (int q = 0; q < QW; ++q)
              if (key < sLim[qbase + q]) o[q * a.out_ld] = sc[q];
          }
        }
        if constexpr (FILTER) {
          int mine = 0;
  #pragma unroll
          for (int q = 0; q < QW; ++q)
            if (lane == q) mine = cnt[q];
          if (lane < QW && !a.cand_atomic) {
            const int row = row0 + qbase + lane;
            if (row < row_end) a.cand_count[(int64_t)row * kQuadrants + quad] = mine;
          }
        }
      }
      ptx::named_bar_sync(1, EPI_THREADS);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, 512);
  }
}

template <int D, int HQ, bool FILTER>
static int launch_score_t(const CUtensorMap& map, const ScoreArgs& a, cudaStream_t st) {
  using C = ScoreCfg<D, HQ>;
  auto kern = score_kernel<D, HQ, FILTER>;
  MISA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
  const int grid = a.n_items < sm_count() ? a.n_items : sm_count();
  if (grid <= 0) return MISA_OK;
  kern<<<grid, C::NUM_THREADS, C::SMEM_BYTES, st>>>(map, a);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

template <bool FILTER>
static int dispatch_score(int D, int HQ, const CUtensorMap& map, const ScoreArgs& a, cudaStream_t st) {
#define MISA_SCORE_CASE(DD, HH) \
  if (D == DD && HQ == HH) return launch_score_t<DD, HH, FILTER>(map, a, st);
  MISA_SCORE_CASE(128, 8)
  MISA_SCORE_CASE(128, 16)
  MISA_SCORE_CASE(128, 32)
  MISA_SCORE_CASE(128, 64)
  MISA_SCORE_CASE(128, 128)
  MISA_SCORE_CASE(64, 8)
  MISA_SCORE_CASE(64, 16)
  MISA_SCORE_CASE(64, 32)
  MISA_SCORE_CASE(64, 64)
  MISA_SCORE_CASE(64, 128)
#undef MISA_SCORE_CASE
  set_error("unsupported scoring shape: head_dim=%d heads_per_query=%d", D, HQ);
  return MISA_EUNSUPPORTED;
}

static int check_common(int64_t n_keys, int D, int n_heads, int n_heads_pad, int hq, int64_t n_rows,
                        const void* keys, const void* queries, const float* weights, const int32_t* prefix_len,
                        const int32_t* items, const int32_t* item_tiles, int n_items) {
  MISA_REQUIRE(keys && queries && weights && prefix_len, "null input pointer");
  MISA_REQUIRE(n_items == 0 || (items && item_tiles), "null work list");
  MISA_REQUIRE(n_keys >= 1 && n_rows >= 1, "empty keys or rows");
  MISA_REQUIRE(D == 64 || D == 128, "head_dim must be padded to 64 or 128, got %d", D);
  MISA_REQUIRE(n_heads >= 1 && n_heads <= n_heads_pad, "bad head counts %d/%d", n_heads, n_heads_pad);
  MISA_REQUIRE(hq == 8 || hq == 16 || hq == 32 || hq == 64 || hq == 128, "heads_per_query %d", hq);
  MISA_REQUIRE(n_rows < (int64_t(1) << 31) && n_keys < (int64_t(1) << 31), "too many rows/keys");
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(keys) & 15) == 0 && (reinterpret_cast<uintptr_t>(queries) & 15) == 0,
               "keys/queries must be 16-byte aligned");
  return MISA_OK;
}

}  // namespace misa

using namespace misa;

extern "C" int misa_score_materialize_split(const void* keys, int64_t n_keys, int64_t key_stride, int head_dim,
                                            const void* queries, const float* weights, int n_heads, int n_heads_pad,
                                            const int32_t* heads, int heads_per_query, const int32_t* prefix_len,
                                            int64_t n_rows, const int32_t* items, const int32_t* item_tiles,
                                            const int32_t* item_tile0, int n_items, float* out, int64_t out_ld,
                                            void* stream) {
  int rc = check_common(n_keys, head_dim, n_heads, n_heads_pad, heads_per_query, n_rows, keys, queries, weights,
                        prefix_len, items, item_tiles, n_items);
  if (rc) return rc;
  MISA_REQUIRE(out && out_ld >= 1, "null output");
  MISA_REQUIRE(key_stride >= 1, "key_stride must be >= 1");
  MISA_REQUIRE(heads != nullptr || heads_per_query >= n_heads, "dense scoring needs heads_per_query >= n_heads");
  const int64_t n_sample = (n_keys + key_stride - 1) / key_stride;
  CUtensorMap map;
  rc = make_tmap_bf16_2d(&map, keys, head_dim, n_sample, key_stride * head_dim, kTileKeys);
  if (rc) return rc;
  ScoreArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(queries);
  a.w = weights;
  a.heads = heads;
  a.prefix_len = prefix_len;
  a.items = items;
  a.item_tiles = item_tiles;
  a.item_tile0 = item_tile0;
  a.n_items = n_items;
  a.T = static_cast<int>(n_rows);
  a.H = n_heads;
  a.Hp = n_heads_pad;
  a.key_stride = static_cast<int>(key_stride);
  a.out = out;
  a.out_ld = out_ld;
  return dispatch_score<false>(head_dim, heads_per_query, map, a, as_stream(stream));
}

extern "C" int misa_score_materialize_paged(const void* key_pool, int64_t n_pool_keys, int head_dim,
                                            const void* queries, const float* weights, int n_heads, int n_heads_pad,
                                            const int32_t* heads, int heads_per_query, const int32_t* prefix_len,
                                            int64_t n_rows, const int32_t* items, const int32_t* item_tiles,
                                            const int32_t* item_tile0, int n_items, const int32_t* page_table,
                                            int page_size, float* out, int64_t out_ld, void* stream) {
  int rc = check_common(n_pool_keys, head_dim, n_heads, n_heads_pad, heads_per_query, n_rows, key_pool, queries,
                        weights, prefix_len, items, item_tiles, n_items);
  if (rc) return rc;
  MISA_REQUIRE(out && out_ld >= 1 && page_table, "null output / page table");
  MISA_REQUIRE(page_size >= kTileKeys && page_size % kTileKeys == 0, "page_size must be a multiple of %d",
               kTileKeys);
  MISA_REQUIRE(n_pool_keys % page_size == 0, "the key pool must hold whole pages");
  MISA_REQUIRE(heads != nullptr || heads_per_query >= n_heads, "dense scoring needs heads_per_query >= n_heads");
  CUtensorMap map;
  rc = make_tmap_bf16_2d(&map, key_pool, head_dim, n_pool_keys, head_dim, kTileKeys);
  if (rc) return rc;
  ScoreArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(queries);
  a.w = weights;
  a.heads = heads;
  a.prefix_len = prefix_len;
  a.items = items;
  a.item_tiles = item_tiles;
  a.item_tile0 = item_tile0;
  a.page_table = page_table;
  a.page_tiles = page_size / kTileKeys;
  a.n_items = n_items;
  a.T = static_cast<int>(n_rows);
  a.H = n_heads;
  a.Hp = n_heads_pad;
  a.key_stride = 1;
  a.out = out;
  a.out_ld = out_ld;
  return dispatch_score<false>(head_dim, heads_per_query, map, a, as_stream(stream));
}

extern "C" int misa_score_materialize(const void* keys, int64_t n_keys, int64_t key_stride, int head_dim,
                                      const void* queries, const float* weights, int n_heads, int n_heads_pad,
                                      const int32_t* heads, int heads_per_query, const int32_t* prefix_len,
                                      int64_t n_rows, const int32_t* items, const int32_t* item_tiles, int n_items,
                                      float* out, int64_t out_ld, void* stream) {
  return misa_score_materialize_split(keys, n_keys, key_stride, head_dim, queries, weights, n_heads, n_heads_pad,
                                      heads, heads_per_query, prefix_len, n_rows, items, item_tiles, nullptr, n_items,
                                      out, out_ld, stream);
}

extern "C" int misa_score_filter(const void* keys, int64_t n_keys, int head_dim, const void* queries,
                                 const float* weights, int n_heads, int n_heads_pad, const int32_t* heads,
                                 int heads_per_query, const int32_t* prefix_len, int64_t n_rows,
                                 const int32_t* items, const int32_t* item_tiles, int n_items, const float* tau,
                                 uint64_t* cand, int cap, int32_t* cand_count, void* stream) {
  int rc = check_common(n_keys, head_dim, n_heads, n_heads_pad, heads_per_query, n_rows, keys, queries, weights,
                        prefix_len, items, item_tiles, n_items);
  if (rc) return rc;
  MISA_REQUIRE(tau && cand && cand_count && cap >= 1, "null filter buffers");
  MISA_REQUIRE(heads != nullptr || heads_per_query >= n_heads, "dense scoring needs heads_per_query >= n_heads");
  CUtensorMap map;
  rc = make_tmap_bf16_2d(&map, keys, head_dim, n_keys, head_dim, kTileKeys);
  if (rc) return rc;
  ScoreArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(queries);
  a.w = weights;
  a.heads = heads;
  a.prefix_len = prefix_len;
  a.items = items;
  a.item_tiles = item_tiles;
  a.n_items = n_items;
  a.T = static_cast<int>(n_rows);
  a.H = n_heads;
  a.Hp = n_heads_pad;
  a.key_stride = 1;
  a.tau = tau;
  a.cand = cand;
  a.cap = cap;
  a.cand_count = cand_count;
  return dispatch_score<true>(head_dim, heads_per_query, map, a, as_stream(stream));
}

extern "C" int misa_score_filter_split(const void* keys, int64_t n_keys, int head_dim, const void* queries,
                                       const float* weights, int n_heads, int n_heads_pad, const int32_t* heads,
                                       int heads_per_query, const int32_t* prefix_len, int64_t n_rows,
                                       const int32_t* items, const int32_t* item_tiles, const int32_t* item_tile0,
                                       int n_items, const float* tau, uint64_t* cand, int cap, int32_t* cand_count,
                                       void* stream) {
  int rc = check_common(n_keys, head_dim, n_heads, n_heads_pad, heads_per_query, n_rows, keys, queries, weights,
                        prefix_len, items, item_tiles, n_items);
  if (rc) return rc;
  MISA_REQUIRE(tau && cand && cand_count && cap >= 1 && (item_tile0 || n_items == 0), "null filter buffers");
  MISA_REQUIRE(heads != nullptr || heads_per_query >= n_heads, "dense scoring needs heads_per_query >= n_heads");
  CUtensorMap map;
  rc = make_tmap_bf16_2d(&map, keys, head_dim, n_keys, head_dim, kTileKeys);
  if (rc) return rc;
  ScoreArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(queries);
  a.w = weights;
  a.heads = heads;
  a.prefix_len = prefix_len;
  a.items = items;
  a.item_tiles = item_tiles;
  a.item_tile0 = item_tile0;
  a.n_items = n_items;
  a.T = static_cast<int>(n_rows);
  a.H = n_heads;
  a.Hp = n_heads_pad;
  a.key_stride = 1;
  a.tau = tau;
  a.cand = cand;
  a.cap = cap;
  a.cand_count = cand_count;
  a.cand_atomic = 1;
  return dispatch_score<true>(head_dim, heads_per_query, map, a, as_stream(stream));
}

extern "C" int misa_score_materialize_varlen(const void* keys, int64_t n_keys, int64_t key_stride, int head_dim,
                                             const void* queries, const float* weights, int n_heads, int n_heads_pad,
                                             const int32_t* heads, int heads_per_query, const int32_t* prefix_len,
                                             int64_t n_rows, const int32_t* item_row0, const int32_t* item_nrows,
                                             const int32_t* item_key0, const int32_t* item_tiles, int n_items,
                                             float* out, int64_t out_ld, void* stream) {
  int rc = check_common(n_keys, head_dim, n_heads, n_heads_pad, heads_per_query, n_rows, keys, queries, weights,
                        prefix_len, item_row0, item_tiles, n_items);
  if (rc) return rc;
  MISA_REQUIRE(n_items == 0 || (item_nrows && item_key0), "null varlen work list");
  MISA_REQUIRE(out && out_ld >= 1 && key_stride >= 1, "null output / bad key_stride");
  MISA_REQUIRE(heads != nullptr || heads_per_query >= n_heads, "dense scoring needs heads_per_query >= n_heads");
  const int64_t n_sample = (n_keys + key_stride - 1) / key_stride;
  CUtensorMap map;
  rc = make_tmap_bf16_2d(&map, keys, head_dim, n_sample, key_stride * head_dim, kTileKeys);
  if (rc) return rc;
  ScoreArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(queries);
  a.w = weights;
  a.heads = heads;
  a.prefix_len = prefix_len;
  a.items = item_row0;
  a.item_nrows = item_nrows;
  a.item_key0 = item_key0;  // in units of the sampled key rows
  a.item_tiles = item_tiles;
  a.n_items = n_items;
  a.T = static_cast<int>(n_rows);
  a.H = n_heads;
  a.Hp = n_heads_pad;
  a.key_stride = static_cast<int>(key_stride);
  a.out = out;
  a.out_ld = out_ld;
  return dispatch_score<false>(head_dim, heads_per_query, map, a, as_stream(stream));
}

extern "C" int misa_score_filter_varlen(const void* keys, int64_t n_keys, int head_dim, const void* queries,
                                        const float* weights, int n_heads, int n_heads_pad, const int32_t* heads,
                                        int heads_per_query, const int32_t* prefix_len, int64_t n_rows,
                                        const int32_t* item_row0, const int32_t* item_nrows,
                                        const int32_t* item_key0, const int32_t* item_tiles, int n_items,
                                        const float* tau, uint64_t* cand, int cap, int32_t* cand_count,
                                        void* stream) {
  int rc = check_common(n_keys, head_dim, n_heads, n_heads_pad, heads_per_query, n_rows, keys, queries, weights,
                        prefix_len, item_row0, item_tiles, n_items);
  if (rc) return rc;
  MISA_REQUIRE(n_items == 0 || (item_nrows && item_key0), "null varlen work list");
  MISA_REQUIRE(tau && cand && cand_count && cap >= 1, "null filter buffers");
  MISA_REQUIRE(heads != nullptr || heads_per_query >= n_heads, "dense scoring needs heads_per_query >= n_heads");
  CUtensorMap map;
  rc = make_tmap_bf16_2d(&map, keys, head_dim, n_keys, head_dim, kTileKeys);
  if (rc) return rc;
  ScoreArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(queries);
  a.w = weights;
  a.heads = heads;
  a.prefix_len = prefix_len;
  a.items = item_row0;
  a.item_nrows = item_nrows;
  a.item_key0 = item_key0;
  a.item_tiles = item_tiles;
  a.n_items = n_items;
  a.T = static_cast<int>(n_rows);
  a.H = n_heads;
  a.Hp = n_heads_pad;
  a.key_stride = 1;
  a.tau = tau;
  a.cand = cand;
  a.cap = cap;
  a.cand_count = cand_count;
  return dispatch_score<true>(head_dim, heads_per_query, map, a, as_stream(stream));
}
