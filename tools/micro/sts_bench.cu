// Micro-benchmark: STS.128 throughput of the conv1 converter pattern (152 rows x 8 chunks of
// 16 B, 128B-swizzled) by 8 warps, alone and with 4 extra warps streaming LDS.128 reads.
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(384, 1) sts_kernel(int iters, int readers, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < 8) {
    const int c = tid, j = c & 7;
    uint32_t x = c;
    for (int it = 0; it < iters; ++it) {
      const uint32_t st = base + (it % 6) * 20480;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int rr = (c >> 3) + k * 32;
        if (rr < 152) {
          asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};\n" ::"r"(st + rr * 128 + ((j ^ (rr & 7)) << 4)), "r"(x));
          x += 1;
        }
      }
    }
  } else if (readers) {
    uint32_t acc = 0;
    const int c = tid - 256;
    for (int it = 0; it < iters * 4; ++it) {
      const uint32_t st = base + ((it + 3) % 6) * 20480;
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        uint32_t a, b, cc, d;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(a), "=r"(b), "=r"(cc), "=r"(d) : "r"(st + (c + k * 128) * 16 % 20480));
        acc += a ^ b ^ cc ^ d;
      }
    }
    if (acc == 0x12345678) out[2] = acc;
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x * 2] = clock64() - t0;
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 2 * 8 + 64);
  cudaFuncSetAttribute(sts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 20480);
  for (int readers = 0; readers < 2; ++readers) {
    sts_kernel<<<148, 384, 6 * 20480>>>(10, readers, d);
    cudaDeviceSynchronize();
    const int iters = 1000;
    sts_kernel<<<148, 384, 6 * 20480>>>(iters, readers, d);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("readers=%d: %.1f cycles per 19.5 KB window (%.1f B/clk)\n", readers, (double)h / iters,
           152.0 * 128 * iters / (double)h);
  }
  return 0;
}
