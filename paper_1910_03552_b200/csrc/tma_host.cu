// Host-side TMA tensor-map helpers.
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "tma_host.h"

namespace bp {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static int g_sms = 0;

int tma_init() {
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  });
  if (!g_encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
}

int tma_num_sms() { return g_sms; }

int tma_make_2d(CUtensorMap* m, const void* ptr, CUtensorMapDataType dtype, int esize, long long rows,
                long long cols, int box_cols, int box_rows, int swz) {
  if (int e = tma_init()) return e;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * esize};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = g_encode(m, dtype, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld box=%dx%d esize=%d", (int)r, rows,
              cols, box_cols, box_rows, esize);
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
}

int tma_make_f32(CUtensorMap* m, const void* ptr, int rank, const long long* dims, const long long* strides_b,
                 const int* box) {
  if (int e = tma_init()) return e;
  cuuint64_t d[5], st[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = (cuuint64_t)dims[i];
    bx[i] = (cuuint32_t)box[i];
    es[i] = 1;
    if (i + 1 < rank) st[i] = (cuuint64_t)strides_b[i];
  }
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void*>(ptr), d, st, bx, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (f32 rank %d) failed (%d)", rank, (int)r);
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
}

}  // namespace bp
