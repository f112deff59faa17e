// C-ABI plumbing: thread-local error message, driver entry point for TMA
// tensor-map encoding, device properties.
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace misa {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t row_elems, uint64_t n_rows,
                      uint64_t row_stride_elems, uint32_t box_rows) {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return MISA_ECUDA;
  }
  MISA_REQUIRE(row_elems % 64 == 0, "tensor-map rows must be a multiple of 64 elements");
  MISA_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, "tensor-map base must be 16-byte aligned");
  cuuint64_t dims[2] = {row_elems, n_rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): dims {%llu,%llu} stride %llu box {64,%u}", (int)r,
              (unsigned long long)row_elems, (unsigned long long)n_rows, (unsigned long long)row_stride_elems * 2,
              box_rows);
    return MISA_ECUDA;
  }
  return MISA_OK;
}

int make_tmap_bf16_gather(CUtensorMap* map, const void* base, uint64_t row_elems, uint64_t n_rows) {
  // tile::gather4 uses a {64, 1} box: each instruction moves four arbitrary 128-byte rows.
  return make_tmap_bf16_2d(map, base, row_elems, n_rows, row_elems, 1);
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace misa

extern "C" int misa_abi_version(void) { return 2; }
extern "C" const char* misa_last_error(void) { return misa::g_err; }
extern "C" int misa_sm_count(void) { return misa::sm_count(); }
