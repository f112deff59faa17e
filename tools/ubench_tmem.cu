// Micro-benchmark: tcgen05.ld (TMEM -> registers) throughput per SM on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_07363_b200/csrc tools/ubench_tmem.cu -o /tmp/ubt
#include <cstdio>
#include "ptx.cuh"
using namespace misa;

template <int WARPS, int X>
__global__ void __launch_bounds__(WARPS * 32, 1) k_tmem(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t base = slot;
  const int quad = warp & 3, split = warp >> 2;
  constexpr int NSPLIT = WARPS / 4;
  constexpr int COLS = 512 / NSPLIT;
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll 1
    for (int c = 0; c < COLS; c += 16 * X) {
      uint32_t r[32];
      const uint32_t ta = base + (uint32_t(quad * 32) << 16) + split * COLS + c;
      if (X == 1) ptx::tmem_ld_x16(ta, r); else ptx::tmem_ld_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(r));
      if (X == 1) ptx::tmem_wait_ld_dep16(r); else ptx::tmem_wait_ld_dep(*reinterpret_cast<uint32_t(*)[32]>(r));
#pragma unroll
      for (int j = 0; j < 16 * X; ++j) acc ^= r[j];
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(base, 512);
}

template <int WARPS, int X>
void run(int iters) {
  unsigned long long* cyc; uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 148 * WARPS * 32 * 4);
  k_tmem<WARPS, X><<<148, WARPS * 32>>>(iters, cyc, sink);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_tmem<WARPS, X><<<148, WARPS * 32>>>(iters, cyc, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  double bytes_per_sm = double(iters) * 512 * 128 * 4;
  printf("warps=%2d x%d: %.1f B/clk/SM (clock64), %.2f TB/s chip (events), err=%s\n", WARPS, 16 * X,
         bytes_per_sm / h, bytes_per_sm * 148 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc); cudaFree(sink);
}

int main() {
  run<4, 1>(2000); run<8, 1>(2000); run<16, 1>(2000); run<16, 2>(2000); run<8, 2>(2000);
  return 0;
}
