// Sparse attention over the selected set — the indexer's downstream consumer (
// PAPER.md Eq. 3, "Sparse MLA" in its MQA mode): every token stores one latent row c_s shared by
// all query heads, and query row t attends only to its top-k tokens T_t:
//
//   sigma_{t,h,s} = scale * q_{t,h} . c_s          (s in T_t, DQK dims)
//   u_{t,h}       = sum_s softmax_s(sigma_{t,h,:}) * c_s[0:DV]
//
// One work item = one query row: its <= 128 heads ride the UMMA M axis (A = Q_t, TMA-loaded,
// resident for the row), the selected latent rows are gathered 128 at a time with 16-byte
// cp.async into the 128-B-swizzled K-major tile (the refine kernel's gather), and the same
// smem tile serves as K for S = Q K^T (K-major B) and as V for O += P V (the tile read
// MN-major: rows = tokens = K, 64-dim row chunks = N).  Softmax is two-pass per row: pass 1
// streams S tiles for the row max and sum, pass 2 recomputes S, writes P = exp(S - m) / l in
// bf16 to shared memory (the K-major A operand) and accumulates O in TMEM — no O rescaling.
// A row's selected tokens come first, -1 padding after (the indexer's output): every role
// finds the row's count n with a binary search and walks ceil(n / 128) tiles; slots past n
// in the last tile are zero-filled and masked to probability 0; a row with no token gets 0.
//
// Warps: 0-3 gather producers (warp 0 lane 0 also loads Q), 4 MMA issuer, 5-8 softmax /
// epilogue (thread = head, TMEM lane quadrant = warp % 4).
#include "common.cuh"
#include "ptx.cuh"

namespace misa {

struct SattnArgs {
  const __nv_bfloat16* __restrict__ kv;  // [n_keys][DQK]
  const int32_t* __restrict__ topk;      // [T][topk_ld] selected token indices, -1 padded
  int64_t topk_ld;
  int k;           // slots per row
  int n_keys;
  int T;
  float scale_log2;  // scale * log2(e)
  float* out;        // [T][H][DV]
  int H;
};

template <int DQK>
struct SattnCfg {
  static constexpr int ATOM = 128 * 128;              // 128 rows x 64 bf16
  static constexpr int Q_BYTES = ATOM * (DQK / 64);
  static constexpr int KV_BYTES = ATOM * (DQK / 64);  // one 128-token tile
  static constexpr int STAGES = DQK <= 128 ? 4 : 1;
  // independent gather warps (the gather rate scales with producer warps, tools/ubench_gather.cu);
  // never more than stages (parity waits cannot tell ring rounds r and r + 2 apart)
  static constexpr int GROUPS = STAGES;
  static constexpr int P_BYTES = 2 * ATOM;            // 128 heads x 128 tokens, K-major
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = OFF_Q + Q_BYTES;
  static constexpr int OFF_P = OFF_KV + STAGES * KV_BYTES;
  static constexpr int OFF_BAR = OFF_P + P_BYTES;
  static constexpr int NUM_BARS = 2 * STAGES + 4 + 2 + 2 + 2;
  static constexpr int OFF_TMEM = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;
  static_assert(SMEM_BYTES <= 227 * 1024, "smem budget");
};

__device__ __forceinline__ void sattn_cp16(void* smem_dst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ptx::smem_u32(smem_dst)), "l"(gsrc),
               "r"(src_bytes)
               : "memory");
}

// Descriptor of a token tile read MN-major (N = feature dims in 64-wide atoms LBO apart, K =
// tokens in 8-row groups SBO apart): the bytes the K-major gather wrote, viewed transposed.
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(lbo >> 4) << 16;
  d |= static_cast<uint64_t>(sbo >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// MN-major SW128 operand: LBO = stride between 64-wide N atoms, SBO = stride between 8-row K
// groups (probed on a B200: the swapped assignment fails tests/test_gpu_sparse_attention.py)
constexpr uint32_t kLbo = 128u * 128u;
constexpr uint32_t kSbo = 1024u;

constexpr int kSattnProd = 4;                             // producer warp slots
constexpr int kSattnMma = kSattnProd;                     // MMA warp
constexpr int kSattnThreads = 32 * (kSattnProd + 1 + 4);  // + 4 softmax warps

template <int DQK, int DV>
__global__ void __launch_bounds__(kSattnThreads, 1) sattn_kernel(const __grid_constant__ CUtensorMap tmap_q, const SattnArgs a) {
  using C = SattnCfg<DQK>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sKV = smem + C::OFF_KV;
  uint8_t* sP = smem + C::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;                  // [STAGES] gather landed
  uint64_t* empty = bars + STAGES;        // [STAGES] MMAs done with the tile
  uint64_t* tfull = empty + STAGES;       // [2] S buffer computed
  uint64_t* tempty = tfull + 2;           // [2] S buffer read
  uint64_t* pfull = tempty + 2;           // P written
  uint64_t* pempty = pfull + 1;           // P consumed by the PV MMA
  uint64_t* qfull = pempty + 1;           // Q of the row landed
  uint64_t* qempty = qfull + 1;           // the row's MMAs are done with Q
  uint64_t* ofull = qempty + 1;           // O of the row complete
  uint64_t* oempty = ofull + 1;           // O read by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // selected tokens of row t: the length of its non-negative prefix
  auto row_count = [&](int t) {
    const int32_t* sel = a.topk + (int64_t)t * a.topk_ld;
    int lo = 0, hi = a.k;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(sel + mid) >= 0) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmap_q);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 32);  // one producer warp fills a stage
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 128);
    }
    ptx::mbar_init(pfull, 128);
    ptx::mbar_init(pempty, 1);
    ptx::mbar_init(qfull, 1);
    ptx::mbar_init(qempty, 1);
    ptx::mbar_init(ofull, 1);
    ptx::mbar_init(oempty, 128);
    ptx::fence_mbar_init();
  }
  if (warp == kSattnMma) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;  // S buffers at columns 0 / 128, O at 256

  if (warp < kSattnProd) {
    // ------------------------------------------------------------ gather producers
    // warp w gathers the CTA-global tiles g == w (mod GROUPS) of the (row, pass, tile) sequence
    const int grp = warp;
    int g = 0;  // tiles of the sequence so far (both passes): stage g % STAGES
    int rr = 0;
    for (int t = blockIdx.x; t < a.T && grp < C::GROUPS; t += gridDim.x, ++rr) {
      if (grp == 0 && lane == 0) {
        ptx::mbar_wait(qempty, (rr & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(qfull, C::Q_BYTES);
#pragma unroll
        for (int at = 0; at < DQK / 64; ++at) ptx::tma_load_2d(sQ + at * C::ATOM, &tmap_q, qfull, at * 64, t * 128);
      }
      const int32_t* sel = a.topk + (int64_t)t * a.topk_ld;
      const int n = row_count(t);
      const int nt = (n + 127) / 128;
      for (int pass = 0; pass < 2; ++pass) {
        for (int j = 0; j < nt; ++j, ++g) {
          if (g % C::GROUPS != grp) continue;
          const int s = g % STAGES;
          ptx::mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
          uint8_t* stage = sKV + s * C::KV_BYTES;
          // the tile's tokens (clamped into the cache: the indexer only emits valid tokens)
          __shared__ int sTokAll[kSattnProd][128];
          int* sTok = sTokAll[grp];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = j * 128 + 32 * u + lane;
            const int v = i < n ? __ldg(sel + i) : -1;
            sTok[32 * u + lane] = v < 0 ? -1 : (v < a.n_keys ? v : a.n_keys - 1);
          }
          __syncwarp();
          // every instruction moves 32 consecutive 16-byte chunks: whole token rows, coalesced
          constexpr int CH = DQK / 8;  // 16-byte chunks per token row
#pragma unroll 4
          for (int e = lane; e < 128 * CH; e += 32) {
            const int r = e / CH, ch = e % CH;
            const int ti = sTok[r];
            const __nv_bfloat16* src = a.kv + (int64_t)(ti < 0 ? 0 : ti) * DQK + ch * 8;
            sattn_cp16(stage + ptx::sw128_offset(r, ch * 8, C::ATOM), src, ti < 0 ? 0u : 16u);
          }
          __syncwarp();  // sTok is rewritten by the next tile
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(ptx::smem_u32(&full[s]))
                       : "memory");
        }
      }
    }
  } else if (warp == kSattnMma) {
    // ------------------------------------------------------------ MMA issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, 128);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(128, DV) | (1u << 16);  // B (V) read MN-major
      int g = 0, sb = 0, rr = 0, npm = 0;  // gathered tiles, S buffers, rows, P tiles consumed
      const uint32_t q_base = ptx::smem_u32(sQ), p_base = ptx::smem_u32(sP);
      const uint32_t o_tmem = tmem_base + 256;
      for (int t = blockIdx.x; t < a.T; t += gridDim.x, ++rr) {
        const int nt = (row_count(t) + 127) / 128;
        ptx::mbar_wait(qfull, rr & 1);
        ptx::tc_fence_after();
        for (int pass = 0; pass < 2; ++pass) {
          for (int j = 0; j < nt; ++j, ++g, ++sb) {
            const int s = g % STAGES, b = sb & 1;
            const uint32_t kv_base = ptx::smem_u32(sKV + s * C::KV_BYTES);
            ptx::mbar_wait(&tempty[b], ((sb >> 1) & 1) ^ 1);
            ptx::mbar_wait(&full[s], (g / STAGES) & 1);
            ptx::fence_proxy_async_smem();  // cp.async writes -> tensor-core reads
            ptx::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < DQK / 16; ++kk) {
              const uint32_t koff = (kk & 3) * 32;
              ptx::mma_bf16(tmem_base + b * 128, ptx::sw128_kmajor_desc(q_base + (kk >> 2) * C::ATOM + koff),
                            ptx::sw128_kmajor_desc(kv_base + (kk >> 2) * C::ATOM + koff), idesc_s, kk > 0 ? 1u : 0u);
            }
            ptx::mma_commit(&tfull[b]);
            if (pass == 0) {
              ptx::mma_commit(&empty[s]);
              continue;
            }
            if (j == 0) ptx::mbar_wait(oempty, (rr & 1) ^ 1);  // the previous row's O was read
            ptx::mbar_wait(pfull, npm & 1);
            ++npm;
            ptx::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 128 / 16; ++kk) {  // K = this tile's 128 tokens
              const uint32_t koff = (kk & 3) * 32;
              ptx::mma_bf16(o_tmem, ptx::sw128_kmajor_desc(p_base + (kk >> 2) * C::ATOM + koff),
                            sw128_mnmajor_desc(kv_base + kk * 2048, kLbo, kSbo), idesc_o,
                            (j > 0 || kk > 0) ? 1u : 0u);
            }
            ptx::mma_commit(&empty[s]);
            ptx::mma_commit(pempty);
          }
        }
        ptx::mma_commit(ofull);
        ptx::mma_commit(qempty);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int quad = warp & 3;
    const int head = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    int g = 0, sb = 0, np = 0, rr = 0;
    for (int t = blockIdx.x; t < a.T; t += gridDim.x, ++rr) {
      const int n = row_count(t);
      const int nt = (n + 127) / 128;
      float m = -INFINITY, l = 0.f;
      for (int pass = 0; pass < 2; ++pass) {
        for (int j = 0; j < nt; ++j, ++g, ++sb) {
          const int b = sb & 1;
          ptx::mbar_wait(&tfull[b], (sb >> 1) & 1);
          __syncwarp();
          ptx::tc_fence_after();
          const int nv = n - j * 128;  // valid columns of this tile
          const uint32_t s_addr = tmem_base + lane_off + b * 128;
          if (pass == 0) {
            // running max / sum over the tile, 32 columns at a time
            for (int c0 = 0; c0 < 128; c0 += 32) {
              uint32_t x[32];
              ptx::tmem_ld_x32p(s_addr + c0, x);
              ptx::tmem_wait_ld_dep32p(x);
              if (c0 + 32 >= 128) {
                ptx::tc_fence_before();
                ptx::mbar_arrive(&tempty[b]);
              }
              float mx = m;
#pragma unroll
              for (int c = 0; c < 32; ++c)
                if (c0 + c < nv) mx = fmaxf(mx, __uint_as_float(x[c]) * a.scale_log2);
              float acc = 0.f;
#pragma unroll
              for (int c = 0; c < 32; ++c)
                if (c0 + c < nv) acc += exp2f(__uint_as_float(x[c]) * a.scale_log2 - mx);
              l = (m == -INFINITY ? 0.f : l * exp2f(m - mx)) + acc;
              m = mx;
            }
            continue;
          }
          const float inv_l = l > 0.f ? 1.f / l : 0.f;
          // P row (this head, 128 tokens) -> bf16 K-major SW128 (2 atoms of 64 tokens)
          ptx::mbar_wait(pempty, (np & 1) ^ 1);
          __syncwarp();
          for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t x[32];
            ptx::tmem_ld_x32p(s_addr + c0, x);
            ptx::tmem_wait_ld_dep32p(x);
            if (c0 + 32 >= 128) {
              ptx::tc_fence_before();
              ptx::mbar_arrive(&tempty[b]);
            }
#pragma unroll
            for (int c = 0; c < 32; c += 8) {
              uint32_t pk[4];
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                const int cc = c0 + c + e;
                const float p0 = cc < nv ? exp2f(__uint_as_float(x[c + e]) * a.scale_log2 - m) * inv_l : 0.f;
                const float p1 = cc + 1 < nv ? exp2f(__uint_as_float(x[c + e + 1]) * a.scale_log2 - m) * inv_l : 0.f;
                const __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                pk[e / 2] = *reinterpret_cast<const uint32_t*>(&h2);
              }
              *reinterpret_cast<uint4*>(sP + ptx::sw128_offset(head, c0 + c, C::ATOM)) =
                  make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
          }
          ptx::fence_proxy_async_smem();  // generic P writes -> the PV MMA's operand reads
          ptx::mbar_arrive(pfull);
          ++np;
        }
      }
      // epilogue: O row of this head -> out[t][head][0:DV]
      ptx::mbar_wait(ofull, rr & 1);
      __syncwarp();
      ptx::tc_fence_after();
      float* orow = a.out + ((int64_t)t * a.H + head) * DV;
#pragma unroll
      for (int c = 0; c < DV; c += 32) {
        uint32_t o[32];
        ptx::tmem_ld_x32p(tmem_base + lane_off + 256 + c, o);
        ptx::tmem_wait_ld_dep32p(o);
        if (head < a.H) {  // a row without tokens: O was never written, its output is 0
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(orow + c + e) =
                n > 0 ? make_float4(__uint_as_float(o[e]), __uint_as_float(o[e + 1]), __uint_as_float(o[e + 2]),
                                    __uint_as_float(o[e + 3]))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(oempty);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kSattnMma) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace misa

using namespace misa;

template <int DQK, int DV>
static int launch_sattn_t(const CUtensorMap& mq, const SattnArgs& a, cudaStream_t st) {
  using C = SattnCfg<DQK>;
  auto kern = sattn_kernel<DQK, DV>;
  MISA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
  const int grid = a.T < sm_count() ? a.T : sm_count();
  kern<<<grid, kSattnThreads, C::SMEM_BYTES, st>>>(mq, a);
  MISA_LAUNCH_CHECK();
  return MISA_OK;
}

extern "C" int misa_sparse_attention(const void* queries, int64_t n_rows, int n_heads, int head_dim_qk,
                                     const void* kv, int64_t n_keys, const int32_t* topk, int64_t topk_ld, int k,
                                     int head_dim_v, float scale, float* out, void* stream) {
  MISA_REQUIRE(queries && kv && topk && out, "null pointer");
  MISA_REQUIRE(n_rows >= 1 && n_keys >= 1 && k >= 1 && topk_ld >= k, "bad sizes");
  MISA_REQUIRE(n_heads >= 1 && n_heads <= 128, "n_heads must lie in [1, 128] (queries padded to 128 rows)");
  MISA_REQUIRE((head_dim_qk == 128 && (head_dim_v == 64 || head_dim_v == 128)) ||
                   (head_dim_qk == 256 && (head_dim_v == 128 || head_dim_v == 256)),
               "unsupported head dims qk=%d v=%d", head_dim_qk, head_dim_v);
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(queries) & 15) == 0 && (reinterpret_cast<uintptr_t>(kv) & 15) == 0,
               "queries / kv must be 16-byte aligned");
  MISA_REQUIRE(n_keys < (int64_t(1) << 31) && n_rows < (int64_t(1) << 31), "too many rows / keys");
  CUtensorMap mq;
  const int rc = make_tmap_bf16_2d(&mq, queries, head_dim_qk, (uint64_t)n_rows * 128, head_dim_qk, 128);
  if (rc) return rc;
  SattnArgs a{};
  a.kv = static_cast<const __nv_bfloat16*>(kv);
  a.topk = topk;
  a.topk_ld = topk_ld;
  a.k = k;
  a.n_keys = (int)n_keys;
  a.T = (int)n_rows;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.out = out;
  a.H = n_heads;
  cudaStream_t st = as_stream(stream);
  if (head_dim_qk == 128 && head_dim_v == 128) return launch_sattn_t<128, 128>(mq, a, st);
  if (head_dim_qk == 128 && head_dim_v == 64) return launch_sattn_t<128, 64>(mq, a, st);
  if (head_dim_qk == 256 && head_dim_v == 256) return launch_sattn_t<256, 256>(mq, a, st);
  return launch_sattn_t<256, 128>(mq, a, st);
}
