// Shared device helpers for the sm_100a learner-step kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>

#include "../../include/beast_b200.h"

#define BP_DEVICE __device__ __forceinline__

namespace bp {

// ---------------------------------------------------------------------------
// error reporting for the C ABI (thread-local message, int status codes)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers: global -> shared without register staging
// ---------------------------------------------------------------------------
BP_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
BP_DEVICE void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
BP_DEVICE void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
BP_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
BP_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// streaming stores / loads
BP_DEVICE void st_cs(float* p, float v) { asm volatile("st.global.cs.f32 [%0], %1;\n" ::"l"(p), "f"(v)); }
BP_DEVICE void st_cs4(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}

// ---------------------------------------------------------------------------
// math: fast exp/log with ~1 ulp-class error (MUFU ex2/lg2), fine for the
// 1e-5 relative V-trace tolerance.
// ---------------------------------------------------------------------------
BP_DEVICE float fast_exp(float x) { return exp2f(x * 1.4426950408889634f); }
BP_DEVICE float fast_log(float x) { return __logf(x); }

template <typename T>
BP_DEVICE T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

BP_DEVICE void set_status(unsigned* status, unsigned bits) {
  if (status && bits) atomicOr(status, bits);
}

}  // namespace bp
