// Probe TMA tile::gather4 (sm_100a): gather 4 arbitrary 128-B rows into SW128 smem.
#include <cstdio>
#include <vector>
#include "common.cuh"
#include "ptx.cuh"
using namespace misa;

__global__ void k(const __grid_constant__ CUtensorMap map, int4 rows, uint32_t* out) {
  __shared__ __align__(1024) uint8_t buf[1024];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, 512);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(ptx::smem_u32(buf + 512)),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(64), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w),
        "r"(ptx::smem_u32(&bar))
        : "memory");
  }
  ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 128; i += blockDim.x) out[i] = reinterpret_cast<uint32_t*>(buf + 512)[i];
}

int main() {
  const int R = 256, C = 128;  // bf16 [R][C]; value = row*1000 + col (as raw 16-bit)
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)((r * 7 + c) & 0xffff);
  void* d; cudaMalloc(&d, h.size() * 2); cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap map;
  int rc = make_tmap_bf16_gather(&map, d, C, R);
  printf("tmap rc=%d %s\n", rc, misa_last_error());
  uint32_t* o; cudaMalloc(&o, 512);
  int4 rows = make_int4(5, 17, 3, 100);
  k<<<1, 32>>>(map, rows, o);
  uint32_t ho[128]; cudaMemcpy(ho, o, 512, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  // expected: smem row i (128 B at 512 + 128 i) = source row rows[i] cols 64..127, 16-B chunk j stored at
  // chunk j ^ ((smem_row_index) & 7) where smem_row_index = (512 + 128 i) / 128 = 4 + i
  int rr[4] = {5, 17, 3, 100};
  int bad = 0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 8; ++j)
      for (int e = 0; e < 8; ++e) {
        const int swz = j ^ ((4 + i) & 7);
        const uint16_t got = reinterpret_cast<uint16_t*>(ho)[i * 64 + swz * 8 + e];
        const uint16_t exp = h[rr[i] * C + 64 + j * 8 + e];
        if (got != exp) ++bad;
      }
  printf("gather4 SW128 mismatches: %d of 256\n", bad);
  // print first row raw
  for (int e = 0; e < 16; ++e) printf("%u ", reinterpret_cast<uint16_t*>(ho)[e]);
  printf("\n");
}
