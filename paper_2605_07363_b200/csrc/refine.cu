// K5: MISA-dagger fine stage (dsa.py:95-115 dsa_rescore, routing.py:144-174).
//
// Row t re-scores its k' coarse candidates with ALL H heads:
//   out[t][i] = sum_j w_{t,j} ReLU(q_{t,j} . k_{cand[t][i]})
// The A operand is a gather of candidate key rows: four producer warps (one
// thread per tile row) copy each row with 16-byte cp.async straight into the
// 128-B-swizzled K-major layout the UMMA descriptor expects, LAG tiles in flight
// per thread (cp.async.wait_group), then fence the generic->async proxy and
// arrive on the stage's mbarrier.  B is the row's Hp query heads (padded to
// N >= 16), resident in smem for the row's tiles.  The contraction is
// L2-bandwidth bound (the whole key set stays L2-resident: 32 MiB at 128K).
//
// Warps: 0-3 producers, 4-7 epilogue (TMEM lane quadrants 0-3), 8 MMA issuer.
#include "common.cuh"
#include "ptx.cuh"

namespace misa {

struct RefineArgs {
  const __nv_bfloat16* __restrict__ keys;  // [n_keys][D]
  const __nv_bfloat16* __restrict__ q;
  const float* __restrict__ w;
  const int32_t* __restrict__ cand;
  int64_t cand_ld;
  const int32_t* __restrict__ n_cand;
  const int32_t* __restrict__ items;  // rows, longest first
  int n_items;
  int T, H, Hp;
  float* out;
  int64_t out_ld;
};

// 16-byte async global->shared copy; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ptx::smem_u32(smem_dst)), "l"(gsrc),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int D, int N>
struct RefineCfg {
  static constexpr int STAGES = (D == 128) ? 5 : 8;
  static constexpr int A_ATOM = 128 * 128;
  static constexpr int A_BYTES = A_ATOM * (D / 64);
  static constexpr int B_ATOM = N * 128;
  static constexpr int B_BYTES = B_ATOM * (D / 64);
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = STAGES * A_BYTES;
  static constexpr int OFF_W = OFF_B + ((B_BYTES + 1023) / 1024) * 1024;
  static constexpr int OFF_BAR = OFF_W + N * 4;
  static constexpr int NUM_BARS = 2 * STAGES + 5;
  static constexpr int OFF_TMEM = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;
  static constexpr int TMEM_COLS = (2 * N <= 32) ? 32 : (2 * N <= 64) ? 64 : (2 * N <= 128) ? 128 : (2 * N <= 256) ? 256 : 512;
  static_assert(SMEM_BYTES <= 227 * 1024, "smem budget");
};

constexpr int kRefineThreads = 288;
constexpr int kLag = 2;  // cp.async tile groups in flight per producer thread

template <int D, int N>
__global__ void __launch_bounds__(kRefineThreads, 1) refine_kernel(const RefineArgs a) {
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
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = gridDim.x, bid = blockIdx.x;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full_a[i], 128);
      ptx::mbar_init(&empty_a[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 128);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 8) ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto item_at = [&](int it) { return (it & 1) ? (it + 1) * P - 1 - bid : it * P + bid; };

  if (warp < 4) {
    // Producers: thread i copies candidate row i of every 128-row tile.
    const int pt = threadIdx.x;  // 0..127
    int s = 0;
    uint32_t ph = 0;
    int pend[kLag + 1];
    int npend = 0;
    for (int it = 0;; ++it) {
      const int idx = item_at(it);
      if (idx >= a.n_items) break;
      const int t = a.items[idx];
      const int nc = a.n_cand[t];
      const int32_t* cr = a.cand + (int64_t)t * a.cand_ld;
      const int nt = (nc + 127) / 128;
      int ki_next = (pt < nc) ? cr[pt] : -1;
      for (int j = 0; j < nt; ++j) {
        const int ki = ki_next;
        if (j + 1 < nt) ki_next = ((j + 1) * 128 + pt < nc) ? cr[(j + 1) * 128 + pt] : -1;
        ptx::mbar_wait(&empty_a[s], ph ^ 1);
        uint8_t* dst = sA + s * C::A_BYTES;
        const __nv_bfloat16* src = a.keys + (int64_t)(ki < 0 ? 0 : ki) * D;
        const uint32_t nb = ki < 0 ? 0u : 16u;
#pragma unroll
        for (int ch = 0; ch < D / 8; ++ch) cp_async16(dst + ptx::sw128_offset(pt, ch * 8, C::A_ATOM), src + ch * 8, nb);
        cp_async_commit();
        pend[npend++] = s;
        if (npend > kLag) {
          cp_async_wait<kLag>();
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(&full_a[pend[0]]);
#pragma unroll
          for (int u = 0; u < kLag; ++u) pend[u] = pend[u + 1];
          --npend;
        }
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
    cp_async_wait<0>();
    ptx::fence_proxy_async_smem();
    for (int u = 0; u < npend; ++u) ptx::mbar_arrive(&full_a[pend[u]]);
  } else if (warp == 8) {
    if (ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N);
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      const uint32_t b_base = ptx::smem_u32(sB);
      for (int it = 0;; ++it) {
        const int idx = item_at(it);
        if (idx >= a.n_items) break;
        const int t = a.items[idx];
        const int nt = (a.n_cand[t] + 127) / 128;
        ptx::mbar_wait(bfull, it & 1);
        ptx::tc_fence_after();
        for (int j = 0; j < nt; ++j) {
          ptx::mbar_wait(&tempty[acc], aph ^ 1);
          ptx::mbar_wait(&full_a[s], ph);
          ptx::fence_proxy_async_smem();
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
          if (++s == STAGES) { s = 0; ph ^= 1; }
          if (++acc == 2) { acc = 0; aph ^= 1; }
        }
      }
    }
  } else {
    const int et = threadIdx.x - 128;
    const int quad = warp & 3;
    int acc = 0;
    uint32_t aph = 0;
    for (int it = 0;; ++it) {
      const int idx = item_at(it);
      if (idx >= a.n_items) break;
      const int t = a.items[idx];
      const int nc = a.n_cand[t];
      const int nt = (nc + 127) / 128;
      constexpr int CH = D / 8;
      for (int c = et; c < N * CH; c += 128) {
        const int r = c / CH, ch = c - r * CH;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (r < a.H) v = *reinterpret_cast<const uint4*>(a.q + ((int64_t)t * a.Hp + r) * D + ch * 8);
        *reinterpret_cast<uint4*>(sB + ptx::sw128_offset(r, ch * 8, C::B_ATOM)) = v;
      }
      for (int r = et; r < N; r += 128) sW[r] = r < a.H ? a.w[(int64_t)t * a.Hp + r] : 0.f;
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(1, 128);
      if (et == 0) ptx::mbar_arrive(bfull);
      for (int j = 0; j < nt; ++j) {
        ptx::mbar_wait(&tfull[acc], aph);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * N;
        // same head order / accumulators as the scorer (ptx.cuh gate_relu4), so an
        // all-head re-score reproduces the dense DSA score bit for bit
        float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
        const float4* w4 = reinterpret_cast<const float4*>(sW);
        uint32_t ra[16], rb[16];
        ptx::tmem_ld_x16(taddr, ra);
        ptx::tmem_wait_ld_dep16(ra);
#pragma unroll
        for (int c = 0; c < N; c += 32) {
          if (c + 16 < N) ptx::tmem_ld_x16(taddr + c + 16, rb);
#pragma unroll
          for (int jj = 0; jj < 16; jj += 4) gate_relu4(s0, s1, w4[(c + jj) / 4], ra[jj], ra[jj + 1], ra[jj + 2], ra[jj + 3]);
          if (c + 16 < N) {
            ptx::tmem_wait_ld_dep16(rb);
            if (c + 32 < N) ptx::tmem_ld_x16(taddr + c + 32, ra);
#pragma unroll
            for (int jj = 0; jj < 16; jj += 4)
              gate_relu4(s0, s1, w4[(c + 16 + jj) / 4], rb[jj], rb[jj + 1], rb[jj + 2], rb[jj + 3]);
            if (c + 32 < N) ptx::tmem_wait_ld_dep16(ra);
          }
        }
        const float sc = gate_relu_finish(s0, s1);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
        if (++acc == 2) { acc = 0; aph ^= 1; }
        const int i = j * 128 + quad * 32 + lane;
        if (i < nc) a.out[(int64_t)t * a.out_ld + i] = sc;
      }
      ptx::named_bar_sync(1, 128);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int D, int N>
static int launch_refine_t(const RefineArgs& a, cudaStream_t st) {
  using C = RefineCfg<D, N>;
  auto kern = refine_kernel<D, N>;
  MISA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
  const int grid = a.n_items < sm_count() ? a.n_items : sm_count();
  if (grid <= 0) return MISA_OK;
  kern<<<grid, kRefineThreads, C::SMEM_BYTES, st>>>(a);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

}  // namespace misa

using namespace misa;

extern "C" int misa_refine_scores(const void* keys, int64_t n_keys, int head_dim, const void* queries,
                                  const float* weights, int n_heads, int n_heads_pad, const int32_t* cand,
                                  int64_t cand_ld, const int32_t* n_cand, const int32_t* rows, int n_items,
                                  int64_t n_rows, float* out, int64_t out_ld, void* stream) {
  MISA_REQUIRE(keys && queries && weights && cand && n_cand && out && (rows || n_items == 0), "null pointer");
  MISA_REQUIRE(head_dim == 64 || head_dim == 128, "head_dim must be padded to 64 or 128");
  MISA_REQUIRE(n_heads >= 1 && n_heads <= n_heads_pad && n_heads_pad <= 128, "bad head counts");
  MISA_REQUIRE(n_rows >= 1 && n_keys >= 1, "empty input");
  if (n_items == 0) return MISA_OK;
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(keys) & 15) == 0, "keys must be 16-byte aligned");
  RefineArgs a{};
  a.keys = static_cast<const __nv_bfloat16*>(keys);
  a.q = static_cast<const __nv_bfloat16*>(queries);
  a.w = weights;
  a.cand = cand;
  a.cand_ld = cand_ld;
  a.n_cand = n_cand;
  a.items = rows;
  a.n_items = n_items;
  a.T = (int)n_rows;
  a.H = n_heads;
  a.Hp = n_heads_pad;
  a.out = out;
  a.out_ld = out_ld;
  cudaStream_t st = as_stream(stream);
  const int N = n_heads_pad < 16 ? 16 : n_heads_pad;
#define MISA_REFINE_CASE(DD, NN) \
  if (head_dim == DD && N == NN) return launch_refine_t<DD, NN>(a, st);
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
