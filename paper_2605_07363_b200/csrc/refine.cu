// K5: MISA-dagger fine stage (dsa.py:95-115 dsa_rescore, routing.py:144-174).
//
// Row t re-scores its k' coarse candidates with ALL H heads:
//   out[t][i] = sum_j w_{t,j} ReLU(q_{t,j} . k_{cand[t][i]})
// The A operand is a gather of candidate key rows with 16-byte cp.async, half a warp per
// key row so every warp instruction moves two whole rows (coalesced, no partial sectors),
// straight into the 128-B-swizzled K-major layout the UMMA descriptor expects; completion
// is tracked by the stage mbarrier (cp.async.mbarrier.arrive.noinc).  The gather is bound
// by how many cp.async requests are in flight per SM, which grows with the number of
// independent producer warps, not with stages alone (tools/ubench_gather.cu: one group of
// 4 warps 8.5 TB/s, six groups of 2 warps 15.7 TB/s from an L2-resident table), so the
// producers are kRefGroups independent groups: group g fills the tiles g, g + G, ... of the
// CTA's tile sequence, prefetching its next tile's candidate indices while it issues.
// (TMA tile::gather4 and 1-D bulk copies per row were measured slower.)  B = the row's Hp
// query heads and gate weights, TMA-loaded by a dedicated warp into one of two buffers so
// the next row's operands land while this row computes; the epilogue runs kRefSets warp
// sets over a kRefAcc-deep TMEM accumulator ring.
//
// Warps: [0, G*W) producers, G*W MMA issuer, G*W+1 B loader, then 4*kRefSets epilogue
// warps (set = tile % kRefSets, TMEM lane quadrant = warp % 4).
#include "common.cuh"
#include "ptx.cuh"

namespace misa {

struct RefineArgs {
  const __nv_bfloat16* __restrict__ keys;  // [n_keys][D]
  const float* __restrict__ w;
  const int32_t* __restrict__ cand;
  int64_t cand_ld;
  const int32_t* __restrict__ n_cand;
  const int32_t* __restrict__ items;  // rows, longest first
  const int32_t* __restrict__ row_key0;  // several key sequences: row t's keys start at row_key0[t] (null: 0)
  int n_items;
  int n_keys;
  int T, H, Hp;
  float* out;
  int64_t out_ld;
  int dots_tiles;  // DOTS mode: 128-key tiles per work item (item i covers keys from i * 128 * dots_tiles)
  // packed output (misa_refine_candidates): out64[t][i] = cand[t][i] << 32 | score bits — the
  // 4-list candidate layout of misa_select_topk (list q = positions [q*list_cap, (q+1)*list_cap))
  uint64_t* out64;
  int32_t* list_count;  // [T][4]
  int list_cap;
};

#ifndef MISA_REF_GROUPS
#define MISA_REF_GROUPS 6
#endif
constexpr int kRefGroups = MISA_REF_GROUPS;              // independent producer groups
constexpr int kRefGroupWarps = 2;                        // warps per group (64 tile rows each)
constexpr int kRefProd = kRefGroups * kRefGroupWarps;    // cp.async producer warps
#ifndef MISA_REF_ACC
#define MISA_REF_ACC 4
#endif
#ifndef MISA_REF_SETS
#define MISA_REF_SETS 2
#endif
constexpr int kRefAcc = MISA_REF_ACC;                    // TMEM accumulators (ring)
constexpr int kRefSets = MISA_REF_SETS;                  // epilogue warp sets (set = tile % kRefSets)
constexpr int kRefMma = kRefProd;                        // MMA warp index
constexpr int kRefBLoad = kRefProd + 1;                  // B (queries + gates) loader warp
constexpr int kRefEpi0 = kRefProd + 2;                   // first epilogue warp
constexpr int kRefThreads = 32 * (kRefEpi0 + 4 * kRefSets);  // 704
static_assert(kRefAcc % kRefSets == 0, "each set owns whole accumulators");

template <int D, int N>
struct RefineCfg {
  static constexpr int A_ATOM = 128 * 128;
  static constexpr int A_BYTES = A_ATOM * (D / 64);
  static constexpr int B_ATOM = N * 128;
  static constexpr int B_BYTES = B_ATOM * (D / 64);
  static constexpr int B_STRIDE = ((B_BYTES + 1023) / 1024) * 1024;
  // as many gather stages as shared memory holds
  static constexpr int STAGES_FIT = (227 * 1024 - 1024 - 2 * B_STRIDE - 2 * N * 4 - 1024) / A_BYTES;
  static constexpr int STAGES = STAGES_FIT > 12 ? 12 : STAGES_FIT;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = STAGES * A_BYTES;       // 2 buffers
  static constexpr int OFF_W = OFF_B + 2 * B_STRIDE;   // 2 x N f32
  static constexpr int OFF_BAR = OFF_W + 2 * N * 4;
  static constexpr int NUM_BARS = 2 * STAGES + 2 * kRefAcc + 4;
  static constexpr int OFF_TMEM = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;
  static constexpr int TMEM_COLS = (kRefAcc * N <= 32) ? 32 : (kRefAcc * N <= 64) ? 64 : (kRefAcc * N <= 128) ? 128
                                   : (kRefAcc * N <= 256) ? 256 : 512;
  static_assert(kRefAcc * N <= 512, "TMEM accumulator ring");
  static_assert(SMEM_BYTES <= 227 * 1024, "smem budget");
  // a producer group never waits on a stage more than one ring round ahead of the MMA
  // (parity waits cannot tell rounds r and r + 2 apart) when there are no more groups than
  // stages: configurations with fewer stages (large N) leave the extra groups idle
  static constexpr int GROUPS = kRefGroups < STAGES ? kRefGroups : STAGES;
};

// 16-byte async global->shared copy; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ptx::smem_u32(smem_dst)), "l"(gsrc),
               "r"(src_bytes)
               : "memory");
}
// Arrive on an mbarrier when all of this thread's prior cp.async copies have landed.
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(ptx::smem_u32(bar)) : "memory");
}

// DOTS = false: MISA-dagger re-score of gathered candidates (one work item = one query row).
// DOTS = true : relevance_dots (dsa.py:18-34): query row set 0 against contiguous keys, one work
//               item = a run of dots_tiles key tiles, the epilogue stores the raw accumulator.
template <int D, int N, bool DOTS>
__global__ void __launch_bounds__(kRefThreads, 1)
    refine_kernel(const __grid_constant__ CUtensorMap tmap_q, const RefineArgs a) {
  using C = RefineCfg<D, N>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint8_t* sA = smem + C::OFF_A;
  uint8_t* sB = smem + C::OFF_B;
  float* sW = reinterpret_cast<float*>(smem + C::OFF_W);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full_a = bars;
  uint64_t* empty_a = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + kRefAcc;
  uint64_t* bfull = tempty + kRefAcc;   // [2]
  uint64_t* bempty = bfull + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = gridDim.x, bid = blockIdx.x;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmap_q);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full_a[i], 32 * kRefGroupWarps);  // one cp.async completion arrival per group thread
      ptx::mbar_init(&empty_a[i], 1);
    }
    for (int i = 0; i < kRefAcc; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 128);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&bfull[i], 1);
      ptx::mbar_init(&bempty[i], 1 + 4 * kRefSets);  // MMA commit + every epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == kRefMma) ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
  for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) sW[i] = 0.f;  // weights of pad heads (Hp < N)
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto item_at = [&](int it) { return (it & 1) ? (it + 1) * P - 1 - bid : it * P + bid; };
  // (query row, candidate count, first key) of work item idx
  auto item_row = [&](int idx) { return DOTS ? 0 : a.items[idx]; };
  auto item_count = [&](int idx) {
    if constexpr (DOTS) {
      const int64_t k0 = (int64_t)idx * 128 * a.dots_tiles;
      const int64_t rem = a.n_keys - k0;
      return (int)(rem < 128 * a.dots_tiles ? rem : 128 * a.dots_tiles);
    } else {
      return a.n_cand[a.items[idx]];
    }
  };

  if (warp < kRefProd) {
    if (warp / kRefGroupWarps < C::GROUPS) {  // groups past C::GROUPS stay idle
    // ---------------------------------------------------------------- producers
    // group grp fills the CTA-global tiles g == grp (mod G).  Warp wi of the group covers
    // tile rows [64 wi, 64 wi + 64): instruction i moves rows 64 wi + 2i and 2i + 1
    // (lanes 0-15 / 16-31, one 16-byte chunk each).  Lane l holds the key indices of
    // rows 64 wi + l and 64 wi + 32 + l, loaded one of the group's tiles ahead.
    constexpr int RPW = 128 / kRefGroupWarps;
    static_assert(RPW == 64, "two index registers per lane");
    const int grp = warp / kRefGroupWarps, wi = warp % kRefGroupWarps;
    const int half = lane >> 4, ch = lane & 15;
    int g0 = 0;  // CTA-global index of the current item's first tile
    // the group's tiles as (item, tile) pairs, walked in order with a one-tile index prefetch
    int it = 0, idx = item_at(0), j = grp;
    int nt = 0, nc = 0, t = 0;
    const int32_t* cr = nullptr;
    const __nv_bfloat16* keys = a.keys;
    auto enter = [&]() {  // advance (it, j) to the group's next tile; false when done
      for (;;) {
        if (idx >= a.n_items) return false;
        t = item_row(idx);
        nc = item_count(idx);
        nt = (nc + 127) / 128;
        if (j < nt) {
          cr = DOTS ? nullptr : a.cand + (int64_t)t * a.cand_ld;
          keys = a.keys + (DOTS ? (int64_t)idx * 128 * a.dots_tiles * D
                                : (a.row_key0 ? (int64_t)a.row_key0[t] * D : 0));
          return true;
        }
        j -= nt;
        g0 += nt;
        idx = item_at(++it);
      }
    };
    auto load_idx = [&](int jj, int ncc, const int32_t* crr, int (&v)[2]) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = jj * 128 + RPW * wi + 32 * u + lane;
        v[u] = i < ncc ? (DOTS ? i : __ldg(crr + i)) : -1;
      }
    };
    if (enter()) {
      int cur[2];
      load_idx(j, nc, cr, cur);
      for (;;) {
        const int g = g0 + j;
        const int s = g % STAGES;
        const uint32_t ph = (uint32_t)(g / STAGES) & 1u;
        const __nv_bfloat16* kcur = keys;
        // next tile of this group (prefetch its indices before issuing this one)
        j += C::GROUPS;
        const bool more = enter();
        int nxt[2] = {-1, -1};
        if (more) load_idx(j, nc, cr, nxt);
        ptx::mbar_wait(&empty_a[s], ph ^ 1);
        uint8_t* stage = sA + s * C::A_BYTES;
#pragma unroll
        for (int i = 0; i < RPW / 2; ++i) {
          const int r = RPW * wi + 2 * i + half;
          const int ki = __shfl_sync(0xffffffffu, i < 16 ? cur[0] : cur[1], (2 * i + half) & 31);
          const __nv_bfloat16* src = kcur + (int64_t)(ki < 0 ? 0 : ki) * D + ch * 8;
          if (ch * 8 < D)
            cp_async16(stage + ptx::sw128_offset(r, ch * 8, C::A_ATOM), src, ki < 0 ? 0u : 16u);
        }
        cp_async_mbar_arrive(&full_a[s]);
        if (!more) break;
        cur[0] = nxt[0];
        cur[1] = nxt[1];
      }
    }
    }
  } else if (warp == kRefMma) {
    // ---------------------------------------------------------------- MMA issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N);
      int g = 0;  // CTA-global tile counter: stage g % STAGES, accumulator g % kRefAcc
      for (int it = 0;; ++it) {
        const int idx = item_at(it);
        if (idx >= a.n_items) break;
        const int nt = (item_count(idx) + 127) / 128;
        const int b = it & 1;
        ptx::mbar_wait(&bfull[b], (it >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t b_base = ptx::smem_u32(sB + b * C::B_STRIDE);
        for (int j = 0; j < nt; ++j, ++g) {
          const int acc = g % kRefAcc;
          const int s = g % STAGES;
          ptx::mbar_wait(&tempty[acc], ((g / kRefAcc) & 1) ^ 1);
          ptx::mbar_wait(&full_a[s], (g / STAGES) & 1);
          ptx::fence_proxy_async_smem();  // cp.async (generic-proxy) writes -> tensor-core reads
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(sA + s * C::A_BYTES);
          const uint32_t d_tmem = tmem_base + acc * N;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = (kk & 3) * 32;
            const uint64_t ad = ptx::sw128_kmajor_desc(a_base + (kk >> 2) * C::A_ATOM + koff);
            const uint64_t bd = ptx::sw128_kmajor_desc(b_base + (kk >> 2) * C::B_ATOM + koff);
            ptx::mma_bf16(d_tmem, ad, bd, idesc, kk > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&empty_a[s]);
          ptx::mma_commit(&tfull[acc]);
        }
        ptx::mma_commit(&bempty[b]);  // B buffer reusable once this row's MMAs are done
      }
    }
  } else if (warp == kRefBLoad) {
    // ---------------------------------------------------------------- B loader
    // operands of row it into buffer it & 1 once the buffer's previous row is fully consumed.
    // N = max(16, Hp): rows past Hp belong to the next query row (or are zero-filled past the
    // end) and meet zero weights, so they contribute exactly 0
    if (lane == 0) {
      for (int it = 0;; ++it) {
        const int idx = item_at(it);
        if (idx >= a.n_items) break;
        const int t = item_row(idx);
        const int b = it & 1;
        ptx::mbar_wait(&bempty[b], ((it >> 1) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&bfull[b], C::B_BYTES + (DOTS ? 0 : a.Hp * 4));
#pragma unroll
        for (int at = 0; at < D / 64; ++at)
          ptx::tma_load_2d(sB + b * C::B_STRIDE + at * C::B_ATOM, &tmap_q, &bfull[b], at * 64, t * a.Hp);
        if (!DOTS) ptx::bulk_g2s(sW + b * N, a.w + (int64_t)t * a.Hp, a.Hp * 4, &bfull[b]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int quad = warp & 3;
    const int set = (warp - kRefEpi0) >> 2;
    int g = 0;
    for (int it = 0;; ++it) {
      const int idx = item_at(it);
      if (idx >= a.n_items) break;
      const int t = item_row(idx);
      const int nc = item_count(idx);
      const int nt = (nc + 127) / 128;
      const int b = it & 1;
      const int first = (set - g % kRefSets + kRefSets) % kRefSets;  // this set's first tile in the row
      if (first < nt) {
        ptx::mbar_wait(&bfull[b], (it >> 1) & 1);
        __syncwarp();
        const float4* w4 = reinterpret_cast<const float4*>(sW + b * N);
        for (int j = first; j < nt; j += kRefSets) {
          const int gg = g + j;
          const int acc = gg % kRefAcc;
          // packed output: this lane's candidate key, loaded before the wait so its L2 latency
          // overlaps the MMA instead of the epilogue chain
          uint32_t pkey = 0;
          if (!DOTS && a.out64) {
            const int i = j * 128 + quad * 32 + lane;
            if (i < nc) pkey = static_cast<uint32_t>(__ldg(a.cand + (int64_t)t * a.cand_ld + i));
          }
          ptx::mbar_wait(&tfull[acc], (gg / kRefAcc) & 1);
          __syncwarp();  // reconverge before the warp-collective TMEM loads
          ptx::tc_fence_after();
          const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * N;
          if constexpr (DOTS) {
            // raw accumulator row of key i: N query columns, the first H stored
            const int i = j * 128 + quad * 32 + lane;
            float* orow = a.out + ((int64_t)idx * 128 * a.dots_tiles + i) * a.out_ld;
            uint32_t r[32];
#pragma unroll
            for (int c = 0; c < N; c += (N < 32 ? 16 : 32)) {
              if constexpr (N >= 32) {
                ptx::tmem_ld_x32p(taddr + c, r);
                ptx::tmem_wait_ld_dep32p(r);
              } else {
                ptx::tmem_ld_x16(taddr + c, r);
                ptx::tmem_wait_ld_dep16(r);
              }
              if (c + (N < 32 ? 16 : 32) >= N) {
                ptx::tc_fence_before();
                ptx::mbar_arrive(&tempty[acc]);
              }
              if (i < nc) {
#pragma unroll
                for (int jj = 0; jj < (N < 32 ? 16 : 32); ++jj)
                  if (c + jj < a.H) orow[c + jj] = __uint_as_float(r[jj]);
              }
            }
            continue;
          }
          // same head order / accumulators as the dense scorer (score.cu reduce16, HQ > 16;
          // gate_relu4), so an all-head re-score reproduces the dense DSA score bit for bit
          float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < N; c += 32) {
            if constexpr (N >= 32) {
              ptx::tmem_ld_x32p(taddr + c, r);
              ptx::tmem_wait_ld_dep32p(r);
              if (c + 32 >= N) {  // the accumulator can be refilled once the last chunk is in registers
                ptx::tc_fence_before();
                ptx::mbar_arrive(&tempty[acc]);
              }
#pragma unroll
              for (int jj = 0; jj < 32; jj += 4)
                gate_relu4(s0, s1, gate_half_hi(w4[(c + jj) / 4]), r[jj], r[jj + 1], r[jj + 2], r[jj + 3]);
            }
          }
          if constexpr (N < 32) {
            ptx::tmem_ld_x16(taddr, r);
            ptx::tmem_wait_ld_dep16(r);
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
#pragma unroll
            for (int jj = 0; jj < N; jj += 4)
              gate_relu4(s0, s1, gate_half_hi(w4[jj / 4]), r[jj], r[jj + 1], r[jj + 2], r[jj + 3]);
          }
          const float sc = gate_relu_finish(s0, s1);
          const int i = j * 128 + quad * 32 + lane;
          if (a.out64) {
            if (i < nc)
              __stcs(reinterpret_cast<unsigned long long*>(a.out64 + (int64_t)t * a.out_ld + i),
                     (static_cast<unsigned long long>(pkey) << 32) | __float_as_uint(sc));
            if (j == 0 && quad == 0 && lane < 4) {
              const int c = nc - lane * a.list_cap;
              a.list_count[(int64_t)t * 4 + lane] = c < 0 ? 0 : (c > a.list_cap ? a.list_cap : c);
            }
          } else if (i < nc) {
            __stcs(a.out + (int64_t)t * a.out_ld + i, sc);  // streaming: keep L2 for the keys
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bempty[b]);  // this warp no longer reads sW[b]
      g += nt;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kRefMma) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int D, int N, bool DOTS = false>
static int launch_refine_t(const CUtensorMap& mq, const RefineArgs& a, cudaStream_t st) {
  using C = RefineCfg<D, N>;
  auto kern = refine_kernel<D, N, DOTS>;
  MISA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
  const int grid = a.n_items < sm_count() ? a.n_items : sm_count();
  if (grid <= 0) return MISA_OK;
  kern<<<grid, kRefThreads, C::SMEM_BYTES, st>>>(mq, a);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

}  // namespace misa

using namespace misa;

static int refine_launch(const void* keys, int64_t n_keys, int head_dim, const void* queries, const float* weights,
                         int n_heads, int n_heads_pad, const int32_t* cand, int64_t cand_ld, const int32_t* n_cand,
                         const int32_t* rows, int n_items, int64_t n_rows, const int32_t* row_key0, float* out,
                         uint64_t* out64, int32_t* list_count, int64_t out_ld, void* stream) {
  MISA_REQUIRE(keys && queries && weights && cand && n_cand && (out || (out64 && list_count)) && (rows || n_items == 0),
               "null pointer");
  MISA_REQUIRE(head_dim == 64 || head_dim == 128, "head_dim must be padded to 64 or 128");
  MISA_REQUIRE(n_heads >= 1 && n_heads <= n_heads_pad && n_heads_pad <= 128, "bad head counts");
  MISA_REQUIRE(n_rows >= 1 && n_keys >= 1, "empty input");
  if (n_items == 0) return MISA_OK;
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(keys) & 15) == 0, "keys must be 16-byte aligned");
  MISA_REQUIRE(n_heads_pad == 8 || n_heads_pad == 16 || n_heads_pad == 32 || n_heads_pad == 64 ||
                   n_heads_pad == 128, "n_heads_pad must be a power of two in [8, 128]");
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(queries) & 15) == 0 && (reinterpret_cast<uintptr_t>(weights) & 15) == 0,
               "queries / weights must be 16-byte aligned");
  MISA_REQUIRE(n_keys < (int64_t(1) << 31) - 1, "too many keys");
  CUtensorMap mq;
  const int rc = make_tmap_bf16_2d(&mq, queries, head_dim, n_rows * n_heads_pad, head_dim, n_heads_pad < 16 ? 16 : n_heads_pad);
  if (rc) return rc;
  RefineArgs a{};
  a.keys = static_cast<const __nv_bfloat16*>(keys);
  a.w = weights;
  a.cand = cand;
  a.cand_ld = cand_ld;
  a.n_cand = n_cand;
  a.items = rows;
  a.row_key0 = row_key0;
  a.n_items = n_items;
  a.n_keys = (int)n_keys;
  a.T = (int)n_rows;
  a.H = n_heads;
  a.Hp = n_heads_pad;
  a.out = out;
  a.out64 = out64;
  a.list_count = list_count;
  a.list_cap = (int)(out_ld / 4);
  a.out_ld = out_ld;
  cudaStream_t st = as_stream(stream);
  const int N = n_heads_pad < 16 ? 16 : n_heads_pad;
#define MISA_REFINE_CASE(DD, NN) \
  if (head_dim == DD && N == NN) return launch_refine_t<DD, NN>(mq, a, st);
  MISA_REFINE_CASE(128, 16)
  MISA_REFINE_CASE(128, 32)
  MISA_REFINE_CASE(128, 64)
  MISA_REFINE_CASE(128, 128)
  MISA_REFINE_CASE(64, 16)
  MISA_REFINE_CASE(64, 32)
  MISA_REFINE_CASE(64, 64)
  MISA_REFINE_CASE(64, 128)
#undef MISA_REFINE_CASE
  set_error("unsupported refine shape head_dim=%d heads=%d", head_dim, N);
  return MISA_EUNSUPPORTED;
}

extern "C" int misa_refine_scores(const void* keys, int64_t n_keys, int head_dim, const void* queries,
                                  const float* weights, int n_heads, int n_heads_pad, const int32_t* cand,
                                  int64_t cand_ld, const int32_t* n_cand, const int32_t* rows, int n_items,
                                  int64_t n_rows, const int32_t* row_key0, float* out, int64_t out_ld,
                                  void* stream) {
  MISA_REQUIRE(out, "null pointer");
  return refine_launch(keys, n_keys, head_dim, queries, weights, n_heads, n_heads_pad, cand, cand_ld, n_cand, rows,
                       n_items, n_rows, row_key0, out, nullptr, nullptr, out_ld, stream);
}

extern "C" int misa_refine_candidates(const void* keys, int64_t n_keys, int head_dim, const void* queries,
                                      const float* weights, int n_heads, int n_heads_pad, const int32_t* cand,
                                      int64_t cand_ld, const int32_t* n_cand, const int32_t* rows, int n_items,
                                      int64_t n_rows, const int32_t* row_key0, uint64_t* lists, int list_cap,
                                      int32_t* list_count, void* stream) {
  MISA_REQUIRE(lists && list_count, "null pointer");
  MISA_REQUIRE(list_cap >= 1, "bad list capacity");
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(lists) & 15) == 0, "lists must be 16-byte aligned");
  return refine_launch(keys, n_keys, head_dim, queries, weights, n_heads, n_heads_pad, cand, cand_ld, n_cand, rows,
                       n_items, n_rows, row_key0, nullptr, lists, list_count, 4 * (int64_t)list_cap, stream);
}

extern "C" int misa_relevance_dots(const void* keys, int64_t n_keys, int head_dim, const void* queries, int n_queries,
                                   int n_queries_pad, float* out, int64_t out_ld, void* stream) {
  MISA_REQUIRE(keys && queries && out, "null pointer");
  MISA_REQUIRE(head_dim == 64 || head_dim == 128, "head_dim must be padded to 64 or 128");
  MISA_REQUIRE(n_queries >= 1 && n_queries <= n_queries_pad, "bad query counts");
  MISA_REQUIRE(n_queries_pad == 8 || n_queries_pad == 16 || n_queries_pad == 32 || n_queries_pad == 64 ||
                   n_queries_pad == 128, "n_queries_pad must be a power of two in [8, 128]");
  MISA_REQUIRE(out_ld >= n_queries, "out_ld < n_queries");
  MISA_REQUIRE(n_keys >= 1 && n_keys < (int64_t(1) << 31) - 1, "bad key count");
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(keys) & 15) == 0 && (reinterpret_cast<uintptr_t>(queries) & 15) == 0,
               "keys / queries must be 16-byte aligned");
  CUtensorMap mq;
  const int N = n_queries_pad < 16 ? 16 : n_queries_pad;
  // the B box holds N rows: with 8 padded query rows the box reads 8 rows past the set, so
  // the map covers exactly the caller's rows and TMA zero-fills the rest
  const int rc = make_tmap_bf16_2d(&mq, queries, head_dim, n_queries_pad, head_dim, N);
  if (rc) return rc;
  RefineArgs a{};
  a.keys = static_cast<const __nv_bfloat16*>(keys);
  a.n_keys = (int)n_keys;
  a.T = 1;
  a.H = n_queries;
  a.Hp = n_queries_pad;
  a.out = out;
  a.out_ld = out_ld;
  // enough items to fill every SM at least once, >= 4 tiles each
  const int64_t tiles = (n_keys + 127) / 128;
  int per = (int)((tiles + sm_count() - 1) / sm_count());
  a.dots_tiles = per < 4 ? 4 : per;
  a.n_items = (int)((tiles + a.dots_tiles - 1) / a.dots_tiles);
  cudaStream_t st = as_stream(stream);
#define MISA_DOTS_CASE(DD, NN) \
  if (head_dim == DD && N == NN) return launch_refine_t<DD, NN, true>(mq, a, st);
  MISA_DOTS_CASE(128, 16)
  MISA_DOTS_CASE(128, 32)
  MISA_DOTS_CASE(128, 64)
  MISA_DOTS_CASE(128, 128)
  MISA_DOTS_CASE(64, 16)
  MISA_DOTS_CASE(64, 32)
  MISA_DOTS_CASE(64, 64)
  MISA_DOTS_CASE(64, 128)
#undef MISA_DOTS_CASE
  set_error("unsupported relevance_dots shape head_dim=%d queries=%d", head_dim, N);
  return MISA_EUNSUPPORTED;
}
