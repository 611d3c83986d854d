// tcgen05 rate of the dK/dV pair's per-block GEMM sequence with nothing else in the way:
//   S  = q' k'^T        (SS, both K-major)      -> D0
//   O  = q' img         (SS, B MN-major)        -> D1 (acc 0 first)
//   st += k'^T v'       (SS, both MN-major)     -> D2
//   O += P v'           (TS: A from TMEM D0)    -> D1
// MODE 0: fixed tiles; 1: tiles rotate through a 5-slot ring (3 per block); 2: as 1 + the
// kernel's commits (s_full, st_full, o_full, 3 slot releases); 3: as 2 + one thread streaming
// 32 KB bulk copies global -> shared (a TMA-like writer, L2-resident source) meanwhile.
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
__device__ __forceinline__ uint64_t dk(uint32_t t, int kk) { return desc(t + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024); }
__device__ __forceinline__ uint64_t dm(uint32_t t, int kk) { return desc(t + kk * 2048, 16384, 1024); }
__host__ __device__ constexpr uint32_t idesc(uint32_t am, uint32_t bm) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (am << 15) | (bm << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(b)));
}
template <int MODE>
__global__ void k(unsigned long long* out, const uint8_t* src, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];  // ring 5 x 32 KB, img 32 KB, scratch 32 KB
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[12];
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 7 * 32768 / 4; i += blockDim.x) {
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
    stop = 0;
    for (int i = 0; i < 12; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  if (MODE == 3 && threadIdx.x == 32) {  // bulk-copy writer into the scratch 32 KB, back to back
    uint32_t ph = 0;
    const uint32_t dst = base + 6 * 32768, mb = (uint32_t)__cvta_generic_to_shared(&bar[11]);
    while (!stop) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(32768));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src + (blockIdx.x % 64) * 32768), "r"(32768), "r"(mb) : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(mb), "r"(ph));
      ph ^= 1;
    }
  }
  if (threadIdx.x == 0) {
    const uint32_t img = base + 5 * 32768;
    constexpr uint32_t id_qk = idesc(0, 0), id_qs = idesc(0, 1), id_kv = idesc(1, 1), id_pv = idesc(0, 1);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int t = MODE == 0 ? 0 : 3 * it;
      const uint32_t q = base + (t % 5) * 32768, kt = base + ((t + 1) % 5) * 32768, v = base + ((t + 2) % 5) * 32768;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) ss(tmem, dk(q, kk), dk(kt, kk), id_qk, kk > 0);
      if (MODE >= 2) commit(&bar[0]);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) ss(tmem + 128, dk(q, kk), dm(img, kk), id_qs, kk > 0);
      if (MODE >= 2) commit(&bar[1]);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) ss(tmem + 256, dm(kt, kk), dm(v, kk), id_kv, 1);
      if (MODE >= 2) { commit(&bar[2]); commit(&bar[3]); }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) ts(tmem + 128, tmem + kk * 8 + (kk >= 4 ? 32 : 0), dm(v, kk), id_pv, 1);
      if (MODE >= 2) { commit(&bar[4]); commit(&bar[5]); }
    }
    commit(&bar[10]);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar[10])));
    out[blockIdx.x] = clock64() - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
  unsigned long long* d;
  uint8_t* src;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&src, 64 * 32768);
  cudaMemset(src, 0x3c, 64 * 32768);
  const int iters = 2000;
  const char* names[4] = {"fixed tiles", "ring-rotating tiles", "+ commits", "+ bulk-copy writer"};
  void (*ks[4])(unsigned long long*, const uint8_t*, int) = {k<0>, k<1>, k<2>, k<3>};
  const int smem = 7 * 32768;
  for (int m = 0; m < 4; ++m) {
    cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    ks[m]<<<148, 128, smem>>>(d, src, iters);
    cudaError_t e = cudaDeviceSynchronize();
    ks[m]<<<148, 128, smem>>>(d, src, iters);
    e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-22s %s  %.0f cycles per block of 4 GEMMs (floor 2048)\n", names[m], cudaGetErrorString(e),
           (double)h[0] / iters);
  }
  return 0;
}
