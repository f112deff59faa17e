// Random 256-byte row gather from an L2-resident table into shared-memory stages — the
// MISA-dagger refine kernel's operand path (refine.cu), measured in isolation: which copy
// mechanism reaches the most L2 -> SM bandwidth with 148 SMs pulling at once.
//
//   method 0: cp.async 16 B (half a warp per row), completion via cp.async.mbarrier.arrive
//   method 1: ld.global.v4 into registers, st.shared (synchronous per group)
//   method 2: cp.async.bulk (TMA 1-D) one 256-B row per instruction, complete_tx
//   method 3: TMA tile::gather4 (4 rows x 128 B per instruction, two per 4 rows)
//
// G producer groups of W warps; group g fills tiles g, g+G, ... (128 rows = 32 KB each)
// into a ring of S stages; one consumer warp waits each stage in order and frees it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_2605_07363_b200/csrc tools/ubench_gather.cu paper_2605_07363_b200/csrc/abi.cu -lcuda -o tools/ubench_gather.bin
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"
using namespace misa;

constexpr int kRows = 131072;  // 32 MiB table of 256-B rows
constexpr int kTileBytes = 128 * 256;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int METHOD>
__global__ void gather(const uint4* __restrict__ table, const __grid_constant__ CUtensorMap tmap, int G, int W, int S,
                       int tiles, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kTileBytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full[i], METHOD == 0 ? 32 * W : (METHOD == 1 ? 32 * W : 1));
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int nprod = G * W;
  if (warp < nprod) {
    const int g = warp / W, wi = warp % W;
    for (int t = g, n = 0; t < tiles; t += G, ++n) {
      const int s = t % S;
      const uint32_t ph = (t / S) & 1;
      ptx::mbar_wait(&empty[s], ph ^ 1);
      uint8_t* st = smem + s * kTileBytes;
      const uint32_t seed = (blockIdx.x * 977u + t) * 131u;
      if constexpr (METHOD == 0) {
        // warp wi covers rows [wi*128/W, (wi+1)*128/W), two rows per instruction
        const int rpw = 128 / W;
        for (int i = 0; i < rpw / 2; ++i) {
          const int r = wi * rpw + 2 * i + (lane >> 4);
          const uint32_t row = hash32(seed + r) % kRows;
          const int ch = lane & 15;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(st + ptx::sw128_offset(r & 127, ch * 8 % 64, 128 * 128) + (ch >= 8 ? 128 * 128 : 0))),
                       "l"(table + (size_t)row * 16 + ch) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(ptx::smem_u32(&full[s])) : "memory");
      } else if constexpr (METHOD == 1) {
        const int per = 2048 / (32 * W);  // 16-B chunks per lane
        uint4 v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i < per) {
            const int c = (wi * per + i) * 32 + lane;  // chunk id in tile
            const int r = c >> 4, ch = c & 15;
            const uint32_t row = hash32(seed + r) % kRows;
            v[i] = __ldcg(table + (size_t)row * 16 + ch);
          }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i < per) {
            const int c = (wi * per + i) * 32 + lane;
            const int r = c >> 4, ch = c & 15;
            *reinterpret_cast<uint4*>(st + ptx::sw128_offset(r, ch * 8 % 64, 128 * 128) + (ch >= 8 ? 128 * 128 : 0)) = v[i];
          }
        }
        ptx::mbar_arrive(&full[s]);
      } else if constexpr (METHOD == 2) {
        // lanes of the group's warps each issue rows; one thread sets the expected bytes first
        if (wi == 0 && lane == 0) ptx::mbar_arrive_expect_tx(&full[s], kTileBytes);
        __syncwarp();
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(32 * W) : "memory");
        for (int r = wi * 32 + lane; r < 128; r += 32 * W) {
          const uint32_t row = hash32(seed + r) % kRows;
          ptx::bulk_g2s(st + r * 256, table + (size_t)row * 16, 256, &full[s]);
        }
      } else {
        if (wi == 0 && lane == 0) ptx::mbar_arrive_expect_tx(&full[s], kTileBytes);
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(32 * W) : "memory");
        // 32 groups of 4 rows x 2 halves = 64 gather4 instructions per tile
        for (int j = wi * 32 + lane; j < 64; j += 32 * W) {
          const int q = j >> 1, half = j & 1;
          int rr[4];
          for (int u = 0; u < 4; ++u) rr[u] = hash32(seed + 4 * q + u) % kRows;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(ptx::smem_u32(st + half * 128 * 128 + q * 512)),
              "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(half * 64), "r"(rr[0]), "r"(rr[1]), "r"(rr[2]), "r"(rr[3]),
              "r"(ptx::smem_u32(&full[s]))
              : "memory");
        }
      }
    }
  } else if (warp == nprod) {
    unsigned long long acc = 0;
    for (int t = 0; t < tiles; ++t) {
      const int s = t % S;
      ptx::mbar_wait(&full[s], (t / S) & 1);
      acc += reinterpret_cast<const uint32_t*>(smem + s * kTileBytes)[lane];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
    }
    if (lane == 0) atomicAdd(sink, acc);
  }
}

template <int M>
float run(const uint4* table, const CUtensorMap& map, int G, int W, int S, int tiles, unsigned long long* sink) {
  const int threads = 32 * (G * W + 1);
  const int smem = S * kTileBytes + 2 * S * 8 + 1024;
  auto k = gather<M>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int sms = sm_count();
  k<<<sms, threads, smem>>>(table, map, G, W, S, tiles, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int rep = 0; rep < 3; ++rep) k<<<sms, threads, smem>>>(table, map, G, W, S, tiles, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  const double bytes = 3.0 * sms * (double)tiles * kTileBytes;
  return (float)(bytes / (ms * 1e-3) / 1e12);
}

int main() {
  uint4* table;
  cudaMalloc(&table, (size_t)kRows * 256);
  cudaMemset(table, 1, (size_t)kRows * 256);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  CUtensorMap map;
  make_tmap_bf16_gather(&map, table, 128, kRows);
  const int tiles = 2000;
  printf("method G W S  TB/s (L2-resident 32 MiB table, 148 SMs)\n");
  int cfgs[][3] = {{1, 4, 5}, {1, 4, 6}, {2, 2, 6}, {4, 1, 6}, {1, 8, 6}, {2, 4, 6}, {3, 4, 6}, {6, 2, 6}};
  for (auto& c : cfgs) printf("cp.async16  %d %d %d  %.2f\n", c[0], c[1], c[2], run<0>(table, map, c[0], c[1], c[2], tiles, sink));
  int cfg1[][3] = {{1, 8, 4}, {2, 8, 4}, {4, 4, 4}, {4, 8, 6}, {6, 4, 6}};
  for (auto& c : cfg1) printf("ldg+sts     %d %d %d  %.2f\n", c[0], c[1], c[2], run<1>(table, map, c[0], c[1], c[2], tiles, sink));
  int cfg2[][3] = {{1, 1, 4}, {1, 1, 6}, {1, 4, 6}, {2, 1, 6}, {2, 4, 6}, {6, 1, 6}};
  for (auto& c : cfg2) printf("bulk256     %d %d %d  %.2f\n", c[0], c[1], c[2], run<2>(table, map, c[0], c[1], c[2], tiles, sink));
  for (auto& c : cfg2) printf("gather4     %d %d %d  %.2f\n", c[0], c[1], c[2], run<3>(table, map, c[0], c[1], c[2], tiles, sink));
  return 0;
}
