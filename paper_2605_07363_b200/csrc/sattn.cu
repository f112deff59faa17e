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
// MN-major: rows = tokens = K, 64-dim row chunks = N).  Online softmax with a lazily raised
// max: P = exp2(S - m) in bf16 to shared memory (the K-major A operand), O accumulated in
// TMEM and rescaled in place only when a tile's max exceeds m by more than 2^8; O / l at the
// end.  S is double-buffered in TMEM so the next tile's QK overlaps this tile's softmax.
// A row's selected tokens come first, -1 padding after (the indexer's output): the Q loader
// counts them (warp-collective, two dependent load rounds) and publishes n in a ring of smem
// slots (one mbarrier each) for the MMA and softmax warps; the producers count for themselves
// one row ahead; every role walks ceil(n / 128) tiles; slots past n in the last tile are
// zero-filled and masked to probability 0; a row with no token gets 0.  The Q loader also
// prefetches the next row's Q and selection into L2 and loads a row's Q as soon as the
// previous row's last QK is done; the epilogue stages O / l through shared memory so its
// global stores write whole row segments.
//
// Warps: 0-3 gather producers, 4 MMA issuer, 5 .. 5 + 4 * kSattnSplit - 1 softmax / epilogue
// (thread = head and 1/kSattnSplit of its columns, TMEM lane quadrant = warp % 4), then the
// Q loader / L2 prefetcher (warp 13 for the default split of 2).
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
  static constexpr int NUM_BARS = 2 * STAGES + 4 + 2 + 2 + 2 + 8;
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
// Softmax warps per lane quadrant: 4 (16 warps of 32 columns, 80 registers, no spills) was
// measured slower than 2 at the C4 shape (26.5 vs 24.8 ms: the 512-thread max exchange).
#ifndef MISA_SATTN_SPLIT
#define MISA_SATTN_SPLIT 2
#endif
constexpr int kSattnSplit = MISA_SATTN_SPLIT;             // softmax warps per TMEM lane quadrant
static_assert(kSattnSplit == 2 || kSattnSplit == 4, "a head's 128 tile columns split in 2 or 4");
constexpr int kSattnSoft0 = kSattnMma + 1;                // first softmax warp
constexpr int kSattnSoftThreads = 128 * kSattnSplit;      // softmax / epilogue threads
constexpr int kSattnQ = kSattnSoft0 + 4 * kSattnSplit;    // Q loader (and L2 prefetch of the next row)
constexpr int kSattnThreads = 32 * (kSattnQ + 1);

__device__ __forceinline__ void tmem_st_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// 32 lanes x 32 columns of 32 bits from registers into TMEM (the O rescale).
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 2^x with one MUFU.EX2 (P is rounded to bf16 right after: the approximation is far below that)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for two values on the FMA pipe (x <= 126): Cody-Waite split x = i + f, |f| <= 1/2, by the
// 1.5 * 2^23 rounding constant, 2^f by a cubic (least-squares fit on [-1/2, 1/2], relative
// error 7.7e-5, far below P's bf16 rounding), 2^i added into the exponent bits — an option to
// move a share of P's exponentials off MUFU.EX2.  Measured at the C4 shape it does not pay:
// the softmax is latency- not MUFU-bound (tools/sattn_trace.py: ~1.4k of a tile's ~2.5k cycles
// in the P phase, XU pipe ~27% busy): 1 pair in 4 -> +0.6 ms, 2 in 4 -> +1.6 ms; MUFU.EX2 on
// f16x2 pairs (half the MUFU ops) +1.2 ms; loading both S chunks before one wait +0.3 ms.
#ifndef MISA_SATTN_EMU
#define MISA_SATTN_EMU 0  // pairs of every four formed on the FMA pipe (0: none, the fastest)
#endif
__device__ __forceinline__ float2 exp2_fma2(float2 x) {
  x = make_float2(fmaxf(x.x, -127.f), fmaxf(x.y, -127.f));
  const float2 j = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 r = __fadd2_rn(j, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(r, make_float2(-1.f, -1.f), x);
  float2 q = __ffma2_rn(f, make_float2(0.05508868f, 0.05508868f), make_float2(0.24260405f, 0.24260405f));
  q = __ffma2_rn(q, f, make_float2(0.6932762f, 0.6932762f));
  q = __ffma2_rn(q, f, make_float2(0.99992895f, 0.99992895f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(j.y) << 23)));
}

// Online softmax: P is formed against a running max m that is only raised (and O rescaled
// in TMEM) when a tile's max exceeds it by more than kLazy (log2 units) — exp2(x - m) then
// stays <= 2^kLazy, exact enough in the bf16 P and the f32 accumulators, and the rescale is
// rare after the first tiles.
constexpr float kLazy = 8.f;

#ifndef MISA_SATTN_QBAR
#define MISA_SATTN_QBAR 1  // per-quadrant named barriers for the softmax exchanges
#endif
#ifndef MISA_SATTN_PTMEM
#define MISA_SATTN_PTMEM 1  // P through TMEM (A operand of P V read from TMEM) when the columns fit
#endif

#ifdef MISA_SATTN_TRACE
// dev instrumentation (tools/sattn_trace.py): clock64 stamps of CTA 0's pipeline events
constexpr int kTrEv = 16, kTrN = 1024;
__device__ long long g_sattn_trace[kTrEv][kTrN];
#define SATTN_TR(ev, idx)                                                                           \
  do {                                                                                              \
    if (blockIdx.x == 0 && (idx) < kTrN) g_sattn_trace[ev][idx] = clock64();                        \
  } while (0)
#else
#define SATTN_TR(ev, idx) \
  do {                    \
  } while (0)
#endif

template <int DQK, int DV>
__global__ void __launch_bounds__(kSattnThreads, 1) sattn_kernel(const __grid_constant__ CUtensorMap tmap_q, const SattnArgs a) {
  using C = SattnCfg<DQK>;
  constexpr int STAGES = C::STAGES;
  // P in TMEM after S0 | S1 | O (DV columns) when 64 more columns fit: the softmax writes it
  // with one tcgen05.st per 32 tokens and P V reads it as a TMEM A operand (no smem round
  // trip, no async-proxy fence); otherwise P goes through shared memory (K-major SW128)
  constexpr bool PT = MISA_SATTN_PTMEM && 256 + DV + 64 <= 512;
  constexpr uint32_t kPCol = 256 + DV;
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
  uint64_t* pfull = tempty + 2;           // P written (and O rescaled if needed)
  uint64_t* pempty = pfull + 1;           // P consumed by the PV MMA (O is stable)
  uint64_t* qfull = pempty + 1;           // Q of the row landed
  uint64_t* qempty = qfull + 1;           // the row's MMAs are done with Q
  uint64_t* ofull = qempty + 1;           // O of the row complete
  uint64_t* oempty = ofull + 1;           // O read by the epilogue
  uint64_t* nfull = oempty + 1;           // [8] a row's token count published (ring by row)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // selected tokens of row t: the length of its non-negative prefix, warp-collective, in two
  // dependent rounds (the last slot of each of 32 segments, then the first partial segment's
  // slots) instead of a binary search's eleven; each warp role looks one row ahead, the MMA
  // thread reads the count the Q loader publishes with the row's Q
  auto row_count = [&](int t) {
    if (t >= a.T) return 0;
    const int32_t* sel = a.topk + (int64_t)t * a.topk_ld;
    const int seg = (a.k + 31) / 32;
    const bool full = lane * seg < a.k && __ldg(sel + min((lane + 1) * seg, a.k) - 1) >= 0;
    const int base = __popc(__ballot_sync(~0u, full)) * seg;
    int cnt = 0;
    for (int i = lane; i < seg; i += 32) cnt += (base + i < a.k && __ldg(sel + base + i) >= 0) ? 1 : 0;
    return min(base + (int)__reduce_add_sync(~0u, (unsigned)cnt), a.k);
  };
  // row counts, Q loader -> MMA and softmax: a ring of 8 rows (the loader runs at most a few
  // rows ahead: each of its Q loads waits for the previous row's QKs, which wait for the
  // softmax of the tile before)
  __shared__ int sRowN[8];

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmap_q);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 32);  // one producer warp fills a stage
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kSattnSoftThreads);
    }
    ptx::mbar_init(pfull, kSattnSoftThreads);
    ptx::mbar_init(pempty, 1);
    ptx::mbar_init(qfull, 1);
    ptx::mbar_init(qempty, 1);
    ptx::mbar_init(ofull, 1);
    ptx::mbar_init(oempty, kSattnSoftThreads);
    for (int i = 0; i < 8; ++i) ptx::mbar_init(&nfull[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == kSattnMma) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;  // S buffers at columns 0 / 128, O at 256

  if (warp < kSattnProd) {
    // ------------------------------------------------------------ gather producers
    // warp w gathers the CTA-global tiles g == w (mod GROUPS) of the (row, tile) sequence
    const int grp = warp;
    int g = 0;  // tiles of the sequence so far: stage g % STAGES
    int rr = 0;
    int n_nxt = grp < C::GROUPS ? row_count(blockIdx.x) : 0;
    for (int t = blockIdx.x; t < a.T && grp < C::GROUPS; t += gridDim.x, ++rr) {
      const int32_t* sel = a.topk + (int64_t)t * a.topk_ld;
      const int n = n_nxt;
      n_nxt = row_count(t + gridDim.x);
      const int nt = (n + 127) / 128;
      for (int j = 0; j < nt; ++j, ++g) {
        if (g % C::GROUPS != grp) continue;
        const int s = g % STAGES;
        ptx::mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
        if (lane == 0) SATTN_TR(0, g);
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
        if (lane == 0) SATTN_TR(1, g);
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(ptx::smem_u32(&full[s]))
                     : "memory");
      }
    }
  } else if (warp == kSattnQ) {
    // ------------------------------------------------------------ Q loader
    // a row's Q lands as soon as the previous row's last QK is done; the next row's Q and
    // selection are prefetched into L2 a row ahead so that neither that load nor the next row's
    // index reads (its count, its tiles' token lists) go to HBM
    int rr = 0;
    int n_nxt = row_count(blockIdx.x);
    for (int t = blockIdx.x; t < a.T; t += gridDim.x, ++rr) {
      const int n = n_nxt;
      n_nxt = row_count(t + gridDim.x);
      const int tn = t + (int)gridDim.x;
      if (tn < a.T) {
        const char* seln = reinterpret_cast<const char*>(a.topk + (int64_t)tn * a.topk_ld);
        for (int off = lane * 128; off < a.k * 4; off += 32 * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(seln + off));
      }
      if (lane == 0) {
        sRowN[rr & 7] = n;
        ptx::mbar_arrive(&nfull[rr & 7]);
        ptx::mbar_wait(qempty, (rr & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(qfull, C::Q_BYTES);
#pragma unroll
        for (int at = 0; at < DQK / 64; ++at) ptx::tma_load_2d(sQ + at * C::ATOM, &tmap_q, qfull, at * 64, t * 128);
        if (tn < a.T)
          for (int at = 0; at < DQK / 64; ++at)
            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                             reinterpret_cast<uint64_t>(&tmap_q)),
                         "r"(at * 64), "r"(tn * 128)
                         : "memory");
        SATTN_TR(9, rr);
      }
      __syncwarp();
    }
  } else if (warp == kSattnMma) {
    // ------------------------------------------------------------ MMA issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, 128);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(128, DV) | (1u << 16);  // B (V) read MN-major
      int g = 0, rr = 0;
      const uint32_t q_base = ptx::smem_u32(sQ), p_base = ptx::smem_u32(sP);
      const uint32_t o_tmem = tmem_base + 256;
      auto issue_qk = [&](int gg) {  // S[gg & 1] = Q K_gg^T
        const int s = gg % STAGES, b = gg & 1;
        const uint32_t kv_base = ptx::smem_u32(sKV + s * C::KV_BYTES);
        ptx::mbar_wait(&tempty[b], ((gg >> 1) & 1) ^ 1);
        ptx::mbar_wait(&full[s], (gg / STAGES) & 1);
        SATTN_TR(2, gg);
        ptx::fence_proxy_async_smem();  // cp.async writes -> tensor-core reads
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DQK / 16; ++kk) {
          const uint32_t koff = (kk & 3) * 32;
          ptx::mma_bf16(tmem_base + b * 128, ptx::sw128_kmajor_desc(q_base + (kk >> 2) * C::ATOM + koff),
                        ptx::sw128_kmajor_desc(kv_base + (kk >> 2) * C::ATOM + koff), idesc_s, kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit(&tfull[b]);
      };
      for (int t = blockIdx.x; t < a.T; t += gridDim.x, ++rr) {
        ptx::mbar_wait(&nfull[rr & 7], (rr >> 3) & 1);
        const int nt = (sRowN[rr & 7] + 127) / 128;
        ptx::mbar_wait(qfull, rr & 1);
        SATTN_TR(10, rr);
        ptx::tc_fence_after();
        // sQ is released as soon as the row's last QK is done (its next Q load then overlaps the
        // last tile's softmax, PV and the epilogue)
        if (nt > 0) issue_qk(g);
        if (nt <= 1) ptx::mma_commit(qempty);
        for (int j = 0; j < nt; ++j, ++g) {
          // the next S overlaps this tile's softmax (with one stage the next tile's gather needs
          // this tile's PV done first: it is issued after it)
          if (STAGES > 1 && j + 1 < nt) {
            issue_qk(g + 1);
            if (j + 2 == nt) ptx::mma_commit(qempty);
          }
          const int s = g % STAGES;
          const uint32_t kv_base = ptx::smem_u32(sKV + s * C::KV_BYTES);
          if (j == 0) {
            ptx::mbar_wait(oempty, (rr & 1) ^ 1);  // the previous row's O was read
            SATTN_TR(13, rr);
          }
          ptx::mbar_wait(pfull, g & 1);
          SATTN_TR(3, g);
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 128 / 16; ++kk) {  // K = this tile's 128 tokens
            const uint32_t koff = (kk & 3) * 32;
            if constexpr (PT)
              ptx::mma_bf16_ts(o_tmem, tmem_base + kPCol + kk * 8, sw128_mnmajor_desc(kv_base + kk * 2048, kLbo, kSbo),
                               idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
            else
              ptx::mma_bf16(o_tmem, ptx::sw128_kmajor_desc(p_base + (kk >> 2) * C::ATOM + koff),
                            sw128_mnmajor_desc(kv_base + kk * 2048, kLbo, kSbo), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&empty[s]);
          ptx::mma_commit(pempty);
          if (STAGES == 1 && j + 1 < nt) {
            issue_qk(g + 1);
            if (j + 2 == nt) ptx::mma_commit(qempty);
          }
        }
        ptx::mma_commit(ofull);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    // kSattnSplit warps per TMEM lane quadrant: part p of a head's 128 tile columns (and of
    // O's DV columns) each; the partial maxima meet in shared memory once per tile
    constexpr int CW = 128 / kSattnSplit;  // tile columns per warp
    constexpr int OP = DV / kSattnSplit;   // O columns per warp
    constexpr int EC = C::P_BYTES / (4 * kSattnSplit) / (32 * 4);  // epilogue: staged columns per pass
    constexpr int OC = OP < EC ? OP : EC;  // O columns per TMEM load / store (16 or 32)
    const int quad = warp & 3;
    const int part = (warp - kSattnSoft0) >> 2;
    // the max / sum exchanges are per head: only the kSattnSplit warps of one lane quadrant
    // meet (one named barrier per quadrant), so quadrants never wait for each other
#if MISA_SATTN_QBAR
    const uint32_t kQBarId = 1 + quad, kQBarThreads = 32 * kSattnSplit;
#else
    const uint32_t kQBarId = 1, kQBarThreads = kSattnSoftThreads;
#endif
    const int head = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t o_addr = tmem_base + lane_off + 256 + part * OP;
    __shared__ float sMax[2][kSattnSplit][128];  // [tile parity][part][head]
    __shared__ float sL[kSattnSplit][128];
    const float sl = a.scale_log2;
    const float2 sl2 = make_float2(sl, sl);
    auto ld_o = [&](uint32_t addr, uint32_t* r) {
      if constexpr (OC == 32) {
        ptx::tmem_ld_x32p(addr, r);
        ptx::tmem_wait_ld_dep32p(r);
      } else {
        ptx::tmem_ld_x16(addr, r);
        ptx::tmem_wait_ld_dep16(r);
      }
    };
    int g = 0, rr = 0;
    for (int t = blockIdx.x; t < a.T; t += gridDim.x, ++rr) {
      ptx::mbar_wait(&nfull[rr & 7], (rr >> 3) & 1);
      const int n = sRowN[rr & 7];
      const int nt = (n + 127) / 128;
      float m = -INFINITY;               // running (lazy) max in log2 units
      float2 l2 = make_float2(0.f, 0.f);  // this part's sum of P (two lanes of columns)
      for (int j = 0; j < nt; ++j, ++g) {
        const int b = g & 1;
        const int nv = n - j * 128 - part * CW;  // valid columns of this part of the tile
        const uint32_t s_addr = tmem_base + lane_off + b * 128 + part * CW;
        ptx::mbar_wait(&tfull[b], (g >> 1) & 1);
        if (warp == kSattnSoft0 && lane == 0) SATTN_TR(4, g);
        __syncwarp();
        ptx::tc_fence_after();
        float mt = -INFINITY;  // this part's max: its 32-column loads in flight at once
        {
          uint32_t x[CW / 32][32];
#pragma unroll
          for (int u = 0; u < CW / 32; ++u) ptx::tmem_ld_x32p(s_addr + 32 * u, x[u]);
#pragma unroll
          for (int u = 0; u < CW / 32; ++u) ptx::tmem_wait_ld_dep32p(x[u]);
          if (nv >= CW) {  // a full part (all but a row's last tile): no per-column masks
            float m2[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int u = 0; u < CW / 32; ++u)
#pragma unroll
              for (int c = 0; c < 32; ++c) m2[c & 3] = fmaxf(m2[c & 3], __uint_as_float(x[u][c]));
            mt = fmaxf(fmaxf(m2[0], m2[1]), fmaxf(m2[2], m2[3]));
          } else {
#pragma unroll
            for (int u = 0; u < CW / 32; ++u)
#pragma unroll
              for (int c = 0; c < 32; ++c)
                if (32 * u + c < nv) mt = fmaxf(mt, __uint_as_float(x[u][c]));
          }
        }
        sMax[b][part][head] = mt;
        ptx::named_bar_sync(kQBarId, kQBarThreads);
#pragma unroll
        for (int u = 0; u < kSattnSplit; ++u) mt = fmaxf(mt, sMax[b][u][head]);
        mt *= sl;  // scale > 0
        if (warp == kSattnSoft0 && lane == 0) SATTN_TR(5, g);
        // P of the previous tile consumed: O is stable and sP free
        ptx::mbar_wait(pempty, (g & 1) ^ 1);
        if (warp == kSattnSoft0 && lane == 0) SATTN_TR(7, g);
        __syncwarp();
        if (mt > m + kLazy) {  // raise the max; rescale this part of O and l (not on the first tile)
          const float alpha = fast_exp2(m - mt);
          l2 = __fmul2_rn(l2, make_float2(alpha, alpha));
          if (j > 0) {
            ptx::tc_fence_after();
#pragma unroll
            for (int c = 0; c < OP; c += OC) {
              uint32_t o[OC];
              ld_o(o_addr + c, o);
#pragma unroll
              for (int e = 0; e < OC; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              if constexpr (OC == 32) tmem_st_x32(o_addr + c, o);
              else tmem_st_x16(o_addr + c, o);
            }
            tmem_wait_st();
          }
          m = mt;
        }
        // P (this head, this part's tokens) in bf16 from a second read of S: packed f32x2
        // scale-and-shift and sum; l sums the unrounded P (as flash attention does)
        {
          const float2 nm2 = make_float2(-m, -m);
          float2 lb2 = make_float2(0.f, 0.f);  // a second accumulator: two shorter FADD2 chains
#pragma unroll
          for (int c0 = 0; c0 < CW; c0 += 32) {
            uint32_t x[32];
            ptx::tmem_ld_x32p(s_addr + c0, x);
            ptx::tmem_wait_ld_dep32p(x);
            const bool full_chunk = nv >= c0 + 32;
            uint32_t pk16[16];  // PT: this chunk's 32 probabilities, two bf16 per TMEM column
#pragma unroll
            for (int c = 0; c < 32; c += 8) {
              uint32_t pk[4];
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                const float2 y = __ffma2_rn(make_float2(__uint_as_float(x[c + e]), __uint_as_float(x[c + e + 1])),
                                            sl2, nm2);
                float p0, p1;
                if ((e >> 1) < MISA_SATTN_EMU) {
                  const float2 q = exp2_fma2(y);
                  p0 = q.x, p1 = q.y;
                } else {
                  p0 = fast_exp2(y.x), p1 = fast_exp2(y.y);
                }
                if (!full_chunk) {
                  p0 = c0 + c + e < nv ? p0 : 0.f;
                  p1 = c0 + c + e + 1 < nv ? p1 : 0.f;
                }
                if (e & 2) lb2 = __fadd2_rn(lb2, make_float2(p0, p1));
                else l2 = __fadd2_rn(l2, make_float2(p0, p1));
                const __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                pk[e / 2] = *reinterpret_cast<const uint32_t*>(&h2);
              }
              if constexpr (PT) {
#pragma unroll
                for (int u = 0; u < 4; ++u) pk16[c / 2 + u] = pk[u];
              } else {
                *reinterpret_cast<uint4*>(sP + ptx::sw128_offset(head, part * CW + c0 + c, C::ATOM)) =
                    make_uint4(pk[0], pk[1], pk[2], pk[3]);
              }
            }
            if constexpr (PT) tmem_st_x16(tmem_base + lane_off + kPCol + (part * CW + c0) / 2, pk16);
          }
          l2 = __fadd2_rn(l2, lb2);
          if constexpr (PT) tmem_wait_st();
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[b]);  // S read twice (max, then P): the buffer can be refilled
        if (warp == kSattnSoft0 && lane == 0) SATTN_TR(6, g);
        if constexpr (!PT) ptx::fence_proxy_async_smem();  // generic P writes -> the PV MMA's operand reads
        ptx::tc_fence_before();         // the O rescale (tcgen05.st) before the next MMA
        ptx::mbar_arrive(pfull);
        if (warp == kSattnSoft0 && lane == 0) SATTN_TR(8, g);
      }
      // epilogue: O row / l of this head (this part of its DV columns) -> out[t][head]
      sL[part][head] = l2.x + l2.y;
      ptx::named_bar_sync(kQBarId, kQBarThreads);
      float lt = 0.f;
#pragma unroll
      for (int u = 0; u < kSattnSplit; ++u) lt += sL[u][head];
      const float inv_l = lt > 0.f ? 1.f / lt : 0.f;
      ptx::mbar_wait(ofull, rr & 1);
      if (warp == kSattnSoft0 && lane == 0) SATTN_TR(11, rr);
      __syncwarp();
      ptx::tc_fence_after();
      // O / l through this warp's share of sP (free: the row's PVs are complete) — 32 heads x
      // EC columns, 16-byte chunks XOR-swizzled by row — so each global store writes whole
      // row segments (4 x 128 B or 8 x 64 B) instead of 32 scattered 16-byte pieces
      constexpr int NC = EC / 4;                                       // 16-byte chunks per row
      constexpr int RPI = 32 / NC;                                     // rows per warp instruction
      static_assert(OP % EC == 0 && EC % OC == 0, "epilogue staging tiles O's columns");
      const uint32_t stg_a = ptx::smem_u32(sP + (warp - kSattnSoft0) * (C::P_BYTES / (4 * kSattnSplit)));
      auto swz = [](int r, int c4) { return (r * NC + (c4 ^ ((r / (8 / NC)) & (NC - 1)))) * 16; };
      const float f = n > 0 ? inv_l : 0.f;  // a row without tokens: O was never written, its output is 0
#pragma unroll
      for (int c = 0; c < OP; c += EC) {
#pragma unroll
        for (int cc = 0; cc < EC; cc += OC) {
          uint32_t o[OC];
          ld_o(o_addr + c + cc, o);
#pragma unroll
          for (int q4 = 0; q4 < OC / 4; ++q4) {
            const int c4 = cc / 4 + q4;
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stg_a + swz(lane, c4)),
                         "f"(__uint_as_float(o[4 * q4]) * f), "f"(__uint_as_float(o[4 * q4 + 1]) * f),
                         "f"(__uint_as_float(o[4 * q4 + 2]) * f), "f"(__uint_as_float(o[4 * q4 + 3]) * f)
                         : "memory");
          }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 32 / RPI; ++i) {
          const int r = i * RPI + lane / NC, c4 = lane % NC;
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "r"(stg_a + swz(r, c4))
                       : "memory");
          const int hr = quad * 32 + r;
          if (hr < a.H)
            *reinterpret_cast<float4*>(a.out + ((int64_t)t * a.H + hr) * DV + part * OP + c + c4 * 4) = v;
        }
        __syncwarp();  // the staging tile is rewritten by the next pass
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(oempty);
      if (warp == kSattnSoft0 && lane == 0) SATTN_TR(12, rr);
      ptx::named_bar_sync(kQBarId, kQBarThreads);  // sL is rewritten by the next row
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

#ifdef MISA_SATTN_TRACE
extern "C" int misa_sattn_trace_copy(long long* host) {
  return cudaMemcpyFromSymbol(host, g_sattn_trace, sizeof(g_sattn_trace)) == cudaSuccess ? 0 : -1;
}
#endif

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
  MISA_REQUIRE(scale > 0.f, "scale must be positive");
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
