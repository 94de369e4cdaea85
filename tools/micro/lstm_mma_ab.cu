// A/B micro-benchmark: the LSTM recurrent product on mma.sync (A = W_hh slice resident in
// registers, the production design of lstm_cluster.cu) versus tcgen05.mma (A = the slice
// resident in shared memory, accumulator in TMEM), for one CTA's 128 gate rows x K = 576
// hidden inputs x 8 batch columns.  Each iteration is one dependent recurrence step without the
// cell math or the cluster exchange: product -> (K-quarter sum) -> new h written back into the
// B operand -> barrier.  Reports SM cycles per step.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1910_03552_b200/csrc \
//        tools/micro/lstm_mma_ab.cu -o tools/micro/lstm_mma_ab && tools/micro/lstm_mma_ab
#include <cstdio>
#include <cuda_bf16.h>
#include "sm100.cuh"

constexpr int ITER = 2000;
constexpr int K = 576, KST = 36, NB = 8, M = 128;

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

// ---- (a) mma.sync, 12 warps x 3 (row tile, K-quarter) items of 9 k-steps, A in registers
constexpr int WARPS = 12, ITEMS = 3, KQ = 9, HS = K + 8;  // h row stride: conflict-free
__global__ void __launch_bounds__(384, 1) ab_mma_sync(const uint32_t* wfrag, long long* out) {
  __shared__ __align__(16) __nv_bfloat16 h[NB][HS];
  __shared__ float red[4][M][NB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tig = lane & 3;
  uint32_t af[ITEMS][KQ][4];
  for (int s = 0; s < ITEMS; ++s)
    for (int q = 0; q < KQ; ++q)
      for (int r = 0; r < 4; ++r) af[s][q][r] = wfrag[((warp * ITEMS + s) * KQ + q) * 4 * 32 + r * 32 + lane];
  for (int i = tid; i < NB * HS; i += 384) (&h[0][0])[i] = __float2bfloat16_rn(0.01f * (i % 7));
  __syncthreads();
  const uint32_t ld_base = sm100::smem_addr(&h[lane & 7][((lane >> 3) & 1) * 8 + (lane >> 4) * 16]);
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
    float acc[ITEMS][4] = {};
#pragma unroll
    for (int q = 0; q < KQ; q += 2)
#pragma unroll
      for (int s = 0; s < ITEMS; ++s) {
        const int item = warp + WARPS * s;
        if (item < 32) {
          const int ks = (item / 8) * KQ + q;
          uint32_t b0, b1, b2, b3;
          ldsm_x4(ld_base + ks * 32, b0, b1, b2, b3);
          mma16816(acc[s], af[s][q], b0, b1);
          if (q + 1 < KQ) mma16816(acc[s], af[s][q + 1], b2, b3);
        }
      }
#pragma unroll
    for (int s = 0; s < ITEMS; ++s) {
      const int item = warp + WARPS * s;
      if (item < 32) {
        const int mt = item % 8, kq = item / 8;
        *reinterpret_cast<float2*>(&red[kq][mt * 16 + g][2 * tig]) = make_float2(acc[s][0], acc[s][1]);
        *reinterpret_cast<float2*>(&red[kq][mt * 16 + g + 8][2 * tig]) = make_float2(acc[s][2], acc[s][3]);
      }
    }
    __syncthreads();
    for (int e = tid; e < M * NB; e += 384) {  // new h (dependency of the next step)
      const int m = e / NB, b = e % NB;
      const float z = (red[0][m][b] + red[1][m][b]) + (red[2][m][b] + red[3][m][b]);
      h[b][m] = __float2bfloat16_rn(tanhf(z));
    }
    __syncthreads();
  }
  if (tid == 0) out[0] = clock64() - t0;
}

// ---- (b) tcgen05: A = W slice [128][576] K-major SW128 in shared memory (147 KB), B = h
//      [16][576] (8 batch columns + 8 zero), accumulator 128 x 16 f32 in TMEM
__global__ void __launch_bounds__(128, 1) ab_tcgen05(const __nv_bfloat16* w, long long* out) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = sm;                        // 9 blocks x 16 KB
  uint8_t* B = sm + 9 * 16384;            // 9 blocks x 2 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(B + 9 * 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto sw = [](int row, int k) {  // byte offset of (row, k) in a K-major SW128 block of 64 k
    return row * 128 + ((((k & 63) >> 3) ^ (row & 7)) << 4) + (k & 7) * 2;
  };
  for (int i = tid; i < M * K; i += 128) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(A + (k >> 6) * 16384 + sw(r, k)) = w[i];
  }
  for (int i = tid; i < 16 * K; i += 128) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(B + (k >> 6) * 2048 + sw(n, k)) =
        __float2bfloat16_rn(n < NB ? 0.01f * (i % 7) : 0.f);
  }
  if (tid == 0) {
    sm100::mbar_init(bar, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(tslot, 32);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = *tslot;
  constexpr uint32_t idesc = sm100::idesc_bf16(128, 16, false, false);
  const uint64_t hi = sm100::smem_desc(0, 16, 1024, sm100::SWZ_128B);
  const uint32_t sa = sm100::smem_addr(A), sb = sm100::smem_addr(B);
  uint32_t phase = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
    if (warp == 0) {
      if (sm100::elect_one()) {
        for (int ks = 0; ks < KST; ++ks) {
          const uint32_t ao = (ks >> 2) * 16384 + (ks & 3) * 32, bo = (ks >> 2) * 2048 + (ks & 3) * 32;
          sm100::umma_f16(tm, hi | ((sa + ao) >> 4), hi | ((sb + bo) >> 4), idesc, ks > 0 ? 1u : 0u);
        }
        sm100::umma_commit(bar);
      }
      __syncwarp();
    }
    sm100::mbar_wait(bar, phase);
    phase ^= 1u;
    sm100::tc_fence_after();
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tm + ((uint32_t)(warp * 32) << 16)));
    sm100::tmem_ld_wait();
    const int m = warp * 32 + lane;  // new h (dependency of the next step): row m -> input k = m
#pragma unroll
    for (int b = 0; b < NB; ++b)
      *reinterpret_cast<__nv_bfloat16*>(B + (m >> 6) * 2048 + sw(b, m)) = __float2bfloat16_rn(tanhf(__uint_as_float(r[b])));
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
  }
  if (tid == 0) out[1] = clock64() - t0;
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tm, 32);
}

int main() {
  uint32_t* wf;
  __nv_bfloat16* w;
  long long* out;
  cudaMalloc(&wf, WARPS * ITEMS * KQ * 4 * 32 * 4);
  cudaMalloc(&w, M * K * 2);
  cudaMalloc(&out, 16);
  cudaMemset(wf, 0x3c, WARPS * ITEMS * KQ * 4 * 32 * 4);  // bf16 pairs ~ 0.011
  cudaMemset(w, 0x3c, M * K * 2);
  const int smem = 9 * 16384 + 9 * 2048 + 1024 + 64;
  cudaFuncSetAttribute(ab_tcgen05, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[2];
  for (int rep = 0; rep < 3; ++rep) {
    ab_mma_sync<<<1, 384>>>(wf, out);
    ab_tcgen05<<<1, 128, smem>>>(w, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("{\"rows\": 128, \"K\": 576, \"batch\": 8, \"mma_sync_cycles_per_step\": %.1f, "
           "\"tcgen05_cycles_per_step\": %.1f}\n", (double)h[0] / ITER, (double)h[1] / ITER);
  }
  return 0;
}
