// A/B micro-benchmark: tcgen05 bf16 MMA throughput per SM for the small-N shapes of the AtariNet
// torso GEMMs (N = 32 / 64 / 128 output columns).  It compares cta_group::1 (M = 128 per CTA,
// the production engine) with cta_group::2 (a CTA pair on one TPC, M = 256, each CTA holding
// its 128 A rows and HALF of B, the leader issuing).  Operands are resident in shared memory
// (K-major, 128B swizzle, no TMA, no epilogue), so the loop measures only the tensor pipe.
// The pipe reads its operands from shared memory, so cta_group::2 should help exactly when
// operand bytes per MMA, not math, bound the pipe ("structural ceiling").
// Every SM runs one CTA; prints SM cycles per M=128-row MMA step and the per-SM MAC rate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1910_03552_b200/csrc \
//        tools/micro/umma_2cta_ab.cu -o tools/micro/umma_2cta_ab && tools/micro/umma_2cta_ab
#include <cstdio>
#include <cuda_bf16.h>
#include "sm100.cuh"

constexpr int ITER = 400;
constexpr int KATOMS = 4;  // K = 256 per pass: 4 swizzle atoms of 64

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int N, int CG>
__global__ void __launch_bounds__(128, 1) mma_rate(long long* out) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  constexpr int NB = N / CG;                       // B rows held by this CTA
  constexpr uint32_t A_ATOM = 128 * 128, B_ATOM = NB * 128;
  uint8_t* A = sm;
  uint8_t* B = A + KATOMS * A_ATOM;
  uint64_t* bar = reinterpret_cast<uint64_t*>(B + KATOMS * B_ATOM);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (int)(KATOMS * (A_ATOM + B_ATOM) / 16); i += 128)
    reinterpret_cast<uint4*>(A)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
  if (tid == 0) {
    sm100::mbar_init(bar, 1);
    sm100::fence_barrier_init();
  }
  constexpr uint32_t COLS = N < 32 ? 32 : N;
  if (warp == 0) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                   "tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::"r"(sm100::smem_addr(tslot)),
                   "n"(COLS));
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n"
                   "tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::"r"(sm100::smem_addr(tslot)),
                   "n"(COLS));
    }
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  sm100::tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = *tslot;
  constexpr uint32_t idesc = sm100::idesc_bf16(128 * CG, N, false, false);
  const uint64_t hi = sm100::smem_desc(0, 16, 1024, sm100::SWZ_128B);
  const uint32_t sa = sm100::smem_addr(A), sb = sm100::smem_addr(B);
  const bool leader = CG == 1 || cta_rank() == 0;
  long long t0 = clock64();
  if (warp == 0 && leader) {
    if (sm100::elect_one()) {
      for (int it = 0; it < ITER; ++it)
#pragma unroll
        for (int ka = 0; ka < KATOMS; ++ka)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = hi | ((sa + ka * A_ATOM + k * 32) >> 4), bd = hi | ((sb + ka * B_ATOM + k * 32) >> 4);
            const uint32_t acc = (it | ka | k) ? 1u : 0u;
            if constexpr (CG == 1) {
              sm100::umma_f16(tm, ad, bd, idesc, acc);
            } else {
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                           "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                           "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
                           : "memory");
            }
          }
      if constexpr (CG == 1) {
        sm100::umma_commit(bar);
      } else {
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                     ::"r"(sm100::smem_addr(bar)), "h"((uint16_t)3)
                     : "memory");
      }
    }
    __syncwarp();
  }
  sm100::mbar_wait(bar, 0);
  long long t1 = clock64();
  if (tid == 0 && leader) out[blockIdx.x] = t1 - t0;
  sm100::tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) {
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(COLS));
  }
}

template <int N, int CG>
static void run(long long* out, long long* host, int sms) {
  constexpr int NB = N / CG;
  const int smem = KATOMS * (128 * 128 + NB * 128) + 1024 + 64;
  auto k = mma_rate<N, CG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  const int grid = sms / 2 * 2;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaMemset(out, 0, grid * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"N\": %d, \"cta_group\": %d, \"error\": \"%s\"}\n", N, CG, cudaGetErrorString(e));
    return;
  }
  cudaMemcpy(host, out, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0, sum = 0;
  int cnt = 0;
  for (int i = 0; i < grid; ++i)
    if (host[i]) {
      mx = host[i] > mx ? host[i] : mx;
      sum += host[i];
      ++cnt;
    }
  const double steps = (double)ITER * KATOMS * 4;  // MMA instructions issued per leader
  const double cyc = (double)sum / cnt / steps;    // SM cycles per instruction (M = 128 * CG)
  const double mac_per_sm = 128.0 * N * 16 / cyc;  // each SM owns 128 rows of every instruction
  const double bytes_per_sm = 128 * 16 * 2 + (double)N / CG * 16 * 2;
  printf("{\"N\": %d, \"cta_group\": %d, \"cycles_per_mma\": %.1f, \"mac_per_clk_per_sm\": %.0f, "
         "\"smem_operand_bytes_per_sm_per_mma\": %.0f, \"operand_B_per_clk\": %.1f, \"max_cycles\": %lld}\n",
         N, CG, cyc, mac_per_sm, bytes_per_sm, bytes_per_sm / cyc, mx);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  cudaMalloc(&out, 1024 * sizeof(long long));
  static long long host[1024];
  run<32, 1>(out, host, sms);
  run<32, 2>(out, host, sms);
  run<64, 1>(out, host, sms);
  run<64, 2>(out, host, sms);
  run<128, 1>(out, host, sms);
  run<128, 2>(out, host, sms);
  run<256, 1>(out, host, sms);
  run<256, 2>(out, host, sms);
  return 0;
}
