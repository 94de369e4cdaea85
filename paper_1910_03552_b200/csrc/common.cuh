// Shared device helpers for the sm_100a learner-step kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>
#include <utility>

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
BP_DEVICE void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
BP_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
BP_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------------------
// TMA bulk (non-tensor) copies + mbarrier, for contiguous spans
// ---------------------------------------------------------------------------
BP_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
BP_DEVICE void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
BP_DEVICE void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
BP_DEVICE void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
BP_DEVICE void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n"
      "@!p bra W_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
// global -> shared, completes `bytes` transactions on `bar` (bytes % 16 == 0, 16B aligned)
BP_DEVICE void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global bulk store (bulk_group completion)
BP_DEVICE void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
BP_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
BP_DEVICE void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
BP_DEVICE void bulk_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }
BP_DEVICE void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
BP_DEVICE void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// streaming stores / loads
BP_DEVICE void st_cs(float* p, float v) { asm volatile("st.global.cs.f32 [%0], %1;\n" ::"l"(p), "f"(v)); }
BP_DEVICE void st_cs4(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}

// ---------------------------------------------------------------------------
// math: fast exp/log with ~1 ulp-class error (MUFU ex2/lg2), fine for the
// 1e-5 relative V-trace tolerance.
// ---------------------------------------------------------------------------
BP_DEVICE float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
BP_DEVICE float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
BP_DEVICE float fast_exp(float x) { return ex2_approx(x * 1.4426950408889634f); }
BP_DEVICE float fast_log(float x) { return lg2_approx(x) * 0.6931471805599453f; }
BP_DEVICE void mbar_arrive_cnt(uint64_t* bar, uint32_t cnt) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}

template <typename T>
BP_DEVICE T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

BP_DEVICE void set_status(unsigned* status, unsigned bits) {
  if (status && bits) atomicOr(status, bits);
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  The learner-step kernels are launched with
// programmatic stream serialization (launch_pdl below): each CTA first signals that the
// next kernel may launch (pdl_trigger), sets up its shared memory / barriers / TMEM, and
// then waits in pdl_wait() until the previous kernel has completed and its writes are
// visible; every global read of an earlier kernel's output comes after pdl_wait().  The
// next kernel's prologue thus overlaps this kernel's tail.  Both are no-ops for a normal
// launch.  EVERY kernel of the chain executes pdl_wait() (completion is transitive).
// ---------------------------------------------------------------------------
BP_DEVICE void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
BP_DEVICE void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

bool pdl_enabled();  // env BP_PDL=0 disables (A/B)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// Action sampling: Gumbel-max with Philox4x32-10 (Salmon et al., SC'11) keyed by the
// 64-bit seed, counter (row lo, row hi, column / 4, 0) -> word column % 4.  The standalone
// sampler (bp_sample_actions_f32) and the heads-GEMM epilogue share these functions, so
// both draw the same action for the same (seed, row) (sample_actions model.py:218-221).
// ---------------------------------------------------------------------------
BP_DEVICE uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// Gumbel(0, 1) noise of uniform word w: u = (w >> 8 + 1/2) 2^-24 in (0, 1), -log(-log u)
BP_DEVICE float gumbel_of(uint32_t w) {
  const float u = ((float)(w >> 8) + 0.5f) * (1.0f / 16777216.0f);
  return -logf(-logf(u));
}

// argmax_j (logit_j + Gumbel_j) over the first A values of a row (greedy: argmax logit_j);
// ties and NaNs resolve to the lowest index, as np.argmax on finite inputs
template <int MAXA>
BP_DEVICE int gumbel_argmax(const float* v, int A, unsigned long long seed, unsigned long long row, bool greedy) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  float best = -INFINITY;
  int arg = 0;
#pragma unroll
  for (int j0 = 0; j0 < MAXA; j0 += 4) {
    if (j0 >= A) break;
    uint4 w = make_uint4(0u, 0u, 0u, 0u);
    if (!greedy) w = philox4x32_10(make_uint4((uint32_t)row, (uint32_t)(row >> 32), (uint32_t)(j0 >> 2), 0u), key);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      if (j < A) {
        const float x = greedy ? v[j] : v[j] + gumbel_of(ws[q]);
        if (x > best) {
          best = x;
          arg = j;
        }
      }
    }
  }
  return arg;
}

}  // namespace bp
