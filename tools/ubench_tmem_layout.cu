// Probe the register layout of tcgen05.ld.16x256b against a known 32x32b store.
#include <cstdio>
#include "ptx.cuh"
using namespace misa;

__global__ void k(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) ptx::tmem_alloc(&slot, 32);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t base = slot + (uint32_t(warp * 32) << 16);
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = ((warp * 32 + lane) << 16) | c;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(base), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
               "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(base + (16u << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) out[lane * 8 + i] = r[i];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(slot, 32);
}

int main() {
  uint32_t* d; cudaMalloc(&d, 32 * 8 * 4);
  k<<<1, 128>>>(d);
  uint32_t h[256]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err=%s  (warp 1 reads lanes 48..63 with 16x256b.x2; entries lane:col)\n", cudaGetErrorString(cudaGetLastError()));
  for (int t = 0; t < 32; ++t) {
    printf("t%2d:", t);
    for (int i = 0; i < 8; ++i) printf(" %3u:%2u", h[t * 8 + i] >> 16, h[t * 8 + i] & 0xffff);
    printf("\n");
  }
}
