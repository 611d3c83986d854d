// TMEM load bandwidth microbenchmark: W warps per CTA repeatedly tcgen05.ld.32x32b.x32 from TMEM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void tld(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(taddr));
}
__global__ void k(unsigned long long* out, float* sink, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int col0 = (warp >> 2) * 128 % 512;
  float acc = 0.f;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int c = 0; c < 128; c += 32) {
      uint32_t r[32];
      tld(tmem + lane_off + ((col0 + c) & 511), r);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      #pragma unroll
      for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
int main() {
  const int iters = 2000;
  unsigned long long* d; float* sink; cudaMalloc(&d, 148 * 8); cudaMalloc(&sink, 148 * 1024 * 4);
  for (int warps = 4; warps <= 16; warps *= 2) {
    k<<<148, warps * 32>>>(d, sink, iters); cudaDeviceSynchronize();
    k<<<148, warps * 32>>>(d, sink, iters); cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double bytes = (double)warps * 32 * 128 * 4 * iters;  // per CTA
    printf("warps=%2d: %s  cycles=%llu  TMEM load %.1f B/clk/SM\n", warps, cudaGetErrorString(e), h[0], bytes / h[0]);
  }
  return 0;
}
