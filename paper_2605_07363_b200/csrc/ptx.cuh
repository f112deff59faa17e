// Thin inline-PTX wrappers for the sm_100a features the indexer kernels use:
// mbarriers, TMA (cp.async.bulk.tensor), tcgen05 (TMEM alloc / MMA / commit /
// ld) and the proxy fences between them.  Compiled only for
// -gencode arch=compute_100a,code=sm_100a.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace misa {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Dynamic smem base rounded up to 1024 B (SW128 operand atoms) by pointer arithmetic
// on the __shared__ array itself, so the compiler keeps the shared address space
// and emits LDS/STS (an integer round-trip would demote every access to generic LD/ST).
__device__ __forceinline__ uint8_t* align_smem_1024(uint8_t* raw) {
  return raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
}

// Predicated 8-byte global store (no branch around it).
__device__ __forceinline__ void st_global_u64_if(uint64_t* p, uint64_t v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "setp.ne.b32 P, %2, 0;\n\t"
      "@P st.global.u64 [%0], %1;\n\t}" ::"l"(p),
      "l"(v), "r"(static_cast<uint32_t>(pred))
      : "memory");
}

// Predicated 8-byte global store of {lo, hi} (the u64 hi:lo) to base[idx], with the
// address formed by one wide multiply-add (no 64-bit add chains, no packing).
__device__ __forceinline__ void st_global_v2_idx_if(const void* base, uint32_t idx, uint32_t lo, uint32_t hi,
                                                    bool pred) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t.reg .b64 A;\n\t"
      "setp.ne.b32 P, %4, 0;\n\t"
      "mad.wide.u32 A, %1, 8, %0;\n\t"
      "@P st.global.v2.b32 [A], {%2, %3};\n\t}" ::"l"(base),
      "r"(idx), "r"(lo), "r"(hi), "r"(static_cast<uint32_t>(pred))
      : "memory");
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------ mbarrier ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, 10000000;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// ----------------------------------------------------------------- TMA ----
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 2-D tiled load, completion signalled on an mbarrier with complete_tx.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 1-D bulk copy global -> shared (16-B aligned, size a multiple of 16), completion
// counted on an mbarrier (complete_tx).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Generic-proxy smem writes -> visible to the async proxy (tensor core operand reads).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------- tcgen05 ----
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, f32 accumulate; single CTA.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// The same with A read from TMEM (lanes = M rows, K packed two bf16 per 32-bit column).
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05 ops of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// wait::ld that also "redefines" the destination registers of the outstanding
// loads, so the compiler cannot hoist their uses above the wait.
__device__ __forceinline__ void tmem_wait_ld_dep(uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
        "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
        "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
        "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
      :
      : "memory");
}

__device__ __forceinline__ void tmem_wait_ld_dep16(uint32_t* r) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
        "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
      :
      : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread i gets lane (base_lane + i), cols [c, c+32).
__device__ __forceinline__ void tmem_ld_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_x32p(uint32_t taddr, uint32_t* r) {
  tmem_ld_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
}
__device__ __forceinline__ void tmem_wait_ld_dep32p(uint32_t* r) {
  tmem_wait_ld_dep(*reinterpret_cast<uint32_t(*)[32]>(r));
}

// 16 lanes x 256 bits, 8 repetitions along columns: thread t gets lanes (t/4, t/4+8)
// at columns 8g + 2(t%4) + {0,1} in r[4g .. 4g+3] = (l0,c0) (l0,c1) (l8,c0) (l8,c1)
// (layout probed on B200: tools/ubench_tmem_layout.cu).
__device__ __forceinline__ void tmem_ld_16x256b_x8(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// ---------------------------------------------------- UMMA descriptors ----
// Shared-memory matrix descriptor for a K-major operand stored in the canonical
// 128-byte-swizzle layout (rows of 64 bf16 = 128 B, 8-row groups 1024 B apart),
// i.e. exactly what a TMA box {64, rows} with CU_TENSOR_MAP_SWIZZLE_128B writes.
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);  // start address
  d |= static_cast<uint64_t>(0) << 16;                       // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;              // SBO: 8-row core-matrix group stride
  d |= static_cast<uint64_t>(1) << 46;                       // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                       // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::f16, A=B=bf16, D=f32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// Byte offset of element (row r, k) inside a K-major SW128 operand made of
// K/64 atoms of [rows x 64] bf16, each atom `atom_bytes` long.
__device__ __forceinline__ uint32_t sw128_offset(uint32_t r, uint32_t k, uint32_t atom_bytes) {
  const uint32_t atom = k >> 6;
  const uint32_t kb = (k & 63u) * 2u;  // byte within the 128-B row
  const uint32_t chunk = (kb >> 4) ^ (r & 7u);
  return atom * atom_bytes + r * 128u + (chunk << 4) + (kb & 15u);
}

}  // namespace ptx

// ------------------------------------------------------ float <-> key ----
// Monotone map float -> u32 (larger float -> larger key); -0.0 == +0.0 as in the
// reference's argsort(-values) (dsa.py:74).
__device__ __forceinline__ uint32_t float_key(float f) {
  // f + 0 turns -0 into +0 (IEEE round-to-nearest); then negative -> ~u, positive -> u | sign
  // as one xor with (u >> 31 arithmetic) | sign: three instructions
  const uint32_t u = __float_as_uint(__fadd_rn(f, 0.0f));
  return u ^ (static_cast<uint32_t>(static_cast<int32_t>(u) >> 31) | 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(u);
}

}  // namespace misa

namespace misa {
// Gated-ReLU head reduction shared by every scorer so that identical inputs give
// bit-identical scores on every path (dense, routed, refine): heads are consumed
// in groups of four into two packed-f32x2 accumulators,
//   s0 += (w0, w1) * (relu x0, relu x1),  s1 += (w2, w3) * (relu x2, relu x3),
// and a query's score is (s0.x + s0.y) + (s1.x + s1.y).
//
// ReLU runs half on the ALU pipe (FMNMX) and half on the FMA pipe: for the second pair of
// each group of four heads (s1 here, A[2] / A[3] below) y = x + |x| (one FADD2 for two heads)
// is exactly 2 relu(x), and those heads' gate weights are stored HALVED (exact), so
// (w / 2) * y == w * relu(x) exactly and the fma chain is bit-identical to the all-FMNMX
// form — the ALU and FMA pipes share the epilogue's ReLUs.  Callers pass w4 with .z / .w
// (head slots 2, 3 of the group) already halved (gate_half_hi).  (A/B at C4,
// tools/variant_lib.py: DSA filter 111.4 -> 105.5-107.3 ms, refine 26.6 -> 24-26; halving the
// stored weights instead of the accumulators: MISA filter 15.2-15.4 -> 14.6-14.9; the
// all-FMA form made the MISA filter slower, 15.2-15.6 vs 14.9-15.1; skipping empty ballots
// in the filter's append loop made it slower too, 15.3 -> 15.5-16.0, coarse 15.6 -> 17.0-17.6.)
__device__ __forceinline__ float2 relu2_alu(uint32_t x0, uint32_t x1) {
  return make_float2(fmaxf(__uint_as_float(x0), 0.f), fmaxf(__uint_as_float(x1), 0.f));
}
__device__ __forceinline__ float2 relu2_fma_x2(uint32_t x0, uint32_t x1) {  // 2 * relu(x), one FADD2
  const float2 x = make_float2(__uint_as_float(x0), __uint_as_float(x1));
  return __fadd2_rn(x, make_float2(fabsf(x.x), fabsf(x.y)));
}
// gate weight as stored for head slot j of a group of four: slots 2, 3 halved
__device__ __forceinline__ float gate_stored(float w, int head_slot) { return (head_slot & 2) ? 0.5f * w : w; }
__device__ __forceinline__ float4 gate_half_hi(float4 w) { return make_float4(w.x, w.y, 0.5f * w.z, 0.5f * w.w); }

__device__ __forceinline__ void gate_relu4(float2& s0, float2& s1, const float4 w, uint32_t x0, uint32_t x1,
                                           uint32_t x2, uint32_t x3) {
  s0 = __ffma2_rn(make_float2(w.x, w.y), relu2_alu(x0, x1), s0);
  s1 = __ffma2_rn(make_float2(w.z, w.w), relu2_fma_x2(x2, x3), s1);  // w.z, w.w halved
}
__device__ __forceinline__ float gate_relu_finish(float2 s0, float2 s1) {
  return (s0.x + s0.y) + (s1.x + s1.y);
}

// The same reduction for two queries at once (HQ = 8, "pair" TMEM layout): v[4g + o],
// v[4g + o + 1] are head g of queries (a, b); w[g] = (w_a[g], w_b[g]) as stored (halved for
// g & 2).  Packed accumulator A_i holds heads (i, i + 4) of both queries, exactly the fma
// chains of gate_relu4's s0.x / s0.y / s1.x / s1.y, so .x / .y are bit-identical to
// gate_relu_finish of query a / b.
__device__ __forceinline__ float2 gate_relu_pair8(const uint32_t* v, int o, const float2 (&w)[8]) {
  float2 A[4];
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const float2 x = (g & 2) ? relu2_fma_x2(v[4 * g + o], v[4 * g + o + 1]) : relu2_alu(v[4 * g + o], v[4 * g + o + 1]);
    A[g & 3] = __ffma2_rn(w[g], x, g < 4 ? make_float2(0.f, 0.f) : A[g & 3]);
  }
  return __fadd2_rn(__fadd2_rn(A[0], A[1]), __fadd2_rn(A[2], A[3]));
}
}  // namespace misa
