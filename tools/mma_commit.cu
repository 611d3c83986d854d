// tcgen05.mma issue rate with a tcgen05.commit after every GEMM group of 8 K=16 MMAs
// (as the causal-family kernels do): does a commit stall the tensor pipe?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
// MODE 0: no commits; 1: one commit per group; 2: three commits per group; 3: one commit per group and
// D alternating over 3 accumulators (0/128/256) with acc=0 at each group's first K step;
// 4: as 3 and the issuing thread waits for each group's commit before the next (fully serial)
// 5: as 1 plus an mbarrier try_wait poll (already complete barrier) between groups
template <int MODE>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 40503u);
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    const uint32_t lo = 0x3F00u | (h & 0x7Fu) | ((h >> 7) & 1u) << 15, hi = 0x3F00u | ((h >> 8) & 0x7Fu) | ((h >> 15) & 1u) << 15;
    reinterpret_cast<uint32_t*>(sm)[i] = lo | (hi << 16);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(sm), b = a + 32768;
    constexpr uint32_t id = idesc(128, 128);
    unsigned long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = (MODE >= 3) ? tmem + 128 * (it % 3) : tmem;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t ad = desc(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
        const uint64_t bd = desc(b + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
        const uint32_t acc = MODE >= 3 ? (kk > 0 ? 1u : 0u) : ((it > 0 || kk > 0) ? 1u : 0u);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc));
      }
      if (MODE >= 1) {
        const int nc = MODE == 2 ? 3 : 1;
        for (int c = 0; c < nc; ++c)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[c])));
      }
      if (MODE == 4 || MODE == 5) {
        uint32_t ok = 0;
        const uint32_t want = MODE == 4 ? ph : ph ^ 1;  // 5: poll the previous phase (already complete)
        if (MODE == 5 && it == 0) { ph ^= 1; continue; }
        while (!ok) {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar[0])), "r"(want));
        }
        ph ^= 1;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[3])));
    uint32_t ok = 0;
    const uint32_t p3 = MODE >= 1 ? 0 : 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar[3])), "r"(p3));
    }
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 2000;
  const char* names[6] = {"no commit", "1 commit / group", "3 commits / group", "1 commit, D over 3 accumulators",
                          "serial: wait each group's commit", "1 commit + poll of a completed barrier"};
  void (*ks[6])(unsigned long long*, int) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>};
  for (int m = 0; m < 6; ++m) {
    cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    ks[m]<<<148, 128, 100 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    ks[m]<<<148, 128, 100 * 1024>>>(d, iters);
    e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-40s %s  %.0f cycles per 128^3 GEMM (8 MMAs; floor 512)\n", names[m], cudaGetErrorString(e),
           (double)h[0] / iters);
  }
  return 0;
}
