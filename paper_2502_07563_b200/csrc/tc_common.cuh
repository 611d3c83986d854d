// Shared device helpers of the tcgen05 kernels (tile geometry, UMMA
// descriptors for SWIZZLE_128B images, TMEM -> smem conversion).
#pragma once
#include <cuda.h>

#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

namespace lasp {
namespace tc {

using namespace ptx;

constexpr int kTile = 128;                    // tokens per block, features per tile
constexpr uint32_t kTileBytes = 128 * 128 * 2;  // 32 KB
constexpr uint32_t kBoxBytes = 128 * 64 * 2;    // 16 KB (one SW128 box)

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// K-major operand descriptor for k-step kk (16 elements along the feature axis).
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t tile, int kk) {
  return umma_desc_sw128(tile + (kk >> 2) * kBoxBytes + (kk & 3) * 32, 16, 1024);
}
// MN-major operand descriptor for k-step kk (16 tokens = two 8-row atoms).
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t tile, int kk) {
  return umma_desc_sw128(tile + kk * 2048, kBoxBytes, 1024);
}

// Byte offset of element (row, col) in a 128x128 bf16 SW128 tile image.
__device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t col) {
  const uint32_t chunk = col >> 6, cc = col & 63;
  const uint32_t unit = (cc >> 3) ^ (row & 7);
  return chunk * kBoxBytes + row * 128 + unit * 16 + (cc & 7) * 2;
}

// Store 32 fp32 values (columns c0..c0+31 of `row`) as bf16 into a SW128 image.
__device__ __forceinline__ void st_row32_bf16(uint8_t* img, uint32_t row, uint32_t c0, const float* v) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint32_t w0 = pack_bf16x2(v[8 * u + 0], v[8 * u + 1]);
    uint32_t w1 = pack_bf16x2(v[8 * u + 2], v[8 * u + 3]);
    uint32_t w2 = pack_bf16x2(v[8 * u + 4], v[8 * u + 5]);
    uint32_t w3 = pack_bf16x2(v[8 * u + 6], v[8 * u + 7]);
    const uint32_t off = sw128_offset(row, c0 + 8 * u);
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(img + off)), "r"(w0), "r"(w1), "r"(w2),
                 "r"(w3)
                 : "memory");
  }
}

// v[i] += bf16 element (row, c0 + i) of a SW128 image (the read side of st_row32_bf16).
__device__ __forceinline__ void ld_row32_add_bf16(const uint8_t* img, uint32_t row, uint32_t c0, float* v) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint32_t w[4];
    const uint32_t off = sw128_offset(row, c0 + 8 * u);
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "r"(smem_u32(img + off))
                 : "memory");
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[8 * u + 2 * j] += __uint_as_float(w[j] << 16);
      v[8 * u + 2 * j + 1] += __uint_as_float(w[j] & 0xffff0000u);
    }
  }
}

// Columns [c_begin, c_begin + ncols) (multiple of 32) of this thread's TMEM lane
// -> bf16 -> SW128 image. MASK 1 keeps col <= row, MASK 2 keeps col >= row
// (the diagonal 128x128 block of a causal / anti-causal chunk). The mask is
// resolved per 32-column chunk and warp: fully kept / fully dropped chunks
// skip the per-element test (and dropped chunks skip the TMEM load).
template <int MASK, bool NEG = false>
__device__ __forceinline__ void tmem_cols_to_image(uint32_t taddr_lane, uint8_t* img, uint32_t row, int c_begin,
                                                   int ncols) {
  const int r_lo = (int)(row & ~31u), r_hi = r_lo + 31;  // rows of this warp
#pragma unroll 1
  for (int c0 = c_begin; c0 < c_begin + ncols; c0 += 32) {
    float v[32];
    const bool all_drop = (MASK == 1 && c0 > r_hi) || (MASK == 2 && c0 + 31 < r_lo);
    if (all_drop) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    } else {
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr_lane + c0, r);
      tmem_ld_wait();
      const bool all_keep = MASK == 0 || (MASK == 1 && c0 + 31 <= r_lo) || (MASK == 2 && c0 >= r_hi);
      if (all_keep) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = NEG ? -__uint_as_float(r[i]) : __uint_as_float(r[i]);
      } else {
        const int lim = (int)row - c0;  // column index (within chunk) of the diagonal
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const bool keep = MASK == 1 ? (i <= lim) : (i >= lim);
          v[i] = keep ? __uint_as_float(r[i]) : 0.f;
        }
      }
    }
    st_row32_bf16(img, row, c0, v);
  }
}

// Same conversion, but the bf16 result goes back to TMEM as the A operand of a
// TS-mode MMA: column pair (c, c+1) of this thread's row packed into one 32-bit
// column at taddr_dst_lane + c/2 (low half = column c). Caller: tcgen05.wait::st
// + fence before signalling the MMA warp.
// INPLACE: the packed pairs of [c_begin, c_begin + ncols) land at [c_begin, c_begin + ncols / 2) of
// taddr_dst (the caller passes the source), i.e. only over columns this thread has already read, so
// two column halves owned by different warps can convert the same TMEM tile in place.
template <int MASK, bool INPLACE = false>
__device__ __forceinline__ void tmem_cols_to_tmem_bf16(uint32_t taddr_lane, uint32_t taddr_dst_lane, uint32_t row,
                                                       int c_begin, int ncols) {
  const int r_lo = (int)(row & ~31u), r_hi = r_lo + 31;
#pragma unroll 1
  for (int c0 = c_begin; c0 < c_begin + ncols; c0 += 32) {
    uint32_t pk[16];
    const bool all_drop = (MASK == 1 && c0 > r_hi) || (MASK == 2 && c0 + 31 < r_lo) || (MASK == 3 && c0 >= r_hi);
    if (all_drop) {
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = 0u;
    } else {
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr_lane + c0, r);
      tmem_ld_wait();
      const bool all_keep = MASK == 0 || (MASK == 1 && c0 + 31 <= r_lo) || (MASK == 2 && c0 >= r_hi) ||
                            (MASK == 3 && c0 + 31 < r_lo);
      if (all_keep) {
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
      } else {
        const int lim = (int)row - c0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int a = 2 * i, b = 2 * i + 1;
          const bool ka = MASK == 1 ? (a <= lim) : MASK == 3 ? (a < lim) : (a >= lim);
          const bool kb = MASK == 1 ? (b <= lim) : MASK == 3 ? (b < lim) : (b >= lim);
          pk[i] = pack_bf16x2(ka ? __uint_as_float(r[a]) : 0.f, kb ? __uint_as_float(r[b]) : 0.f);
        }
      }
    }
    tmem_st_32x32b_x16(taddr_dst_lane + (uint32_t)(INPLACE ? c_begin + ((c0 - c_begin) >> 1) : (c0 >> 1)), pk);
  }
}

// Optional per-block timeline of CTA (0,0) for blocks [16, 24): each traced
// thread stamps clock64() into a local array and flushes it once at exit, so
// tracing costs a few cycles per point. Enabled when g_trace != nullptr.
static __device__ unsigned long long* g_trace = nullptr;  // one per translation unit
#ifdef LASP2_TRACE
struct Tracer {
  unsigned long long rec[64];
  int n = 0;
  bool on;
  __device__ Tracer() : on(g_trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0) {}
  __device__ explicit Tracer(bool cta) : on(g_trace != nullptr && cta) {}
  __device__ __forceinline__ void operator()(int ev, int blk) {
    if (on && blk >= 16 && blk < 24 && n < 64)
      rec[n++] = ((unsigned long long)ev << 56) | ((unsigned long long)blk << 48) |
                 ((unsigned long long)clock64() & 0xFFFFFFFFFFFFull);
  }
  __device__ void flush(int region) {
    if (!on) return;
    for (int i = 0; i < n; ++i) g_trace[region * 64 + i] = rec[i];
  }
};
#else
struct Tracer {  // compiled out: build with -DLASP2_TRACE to record timelines
  __device__ Tracer() {}
  __device__ explicit Tracer(bool) {}
  __device__ __forceinline__ void operator()(int, int) {}
  __device__ __forceinline__ void flush(int) {}
};
#endif

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// sm_100 paired fp32 arithmetic (FFMA2 / FADD2) and the 3-input max (FMNMX3):
// half the issue slots of the scalar forms in the softmax inner loops.
__device__ __forceinline__ void ffma2_bc(float& d0, float& d1, float a0, float a1, float b, float c) {
  uint64_t d;
  asm("{\n\t.reg .b64 pa, pb, pc;\n\tmov.b64 pa, {%1, %2};\n\tmov.b64 pb, {%3, %3};\n\t"
      "mov.b64 pc, {%4, %4};\n\tfma.rn.f32x2 %0, pa, pb, pc;\n\t}"
      : "=l"(d)
      : "f"(a0), "f"(a1), "f"(b), "f"(c));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}
__device__ __forceinline__ void fadd2(float& a0, float& a1, float b0, float b1) {
  uint64_t d;
  asm("{\n\t.reg .b64 pa, pb;\n\tmov.b64 pa, {%1, %2};\n\tmov.b64 pb, {%3, %4};\n\t"
      "add.rn.f32x2 %0, pa, pb;\n\t}"
      : "=l"(d)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(d));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x on the FMA pipe (the SFU's ex2 rate on sm_100 equals the tensor core's
// per-element rate of an attention block, so part of the exponentials move
// here): round-to-nearest split x = j + f, f in [-0.5, 0.5], degree-3
// relative-minimax polynomial for 2^f (max rel. error 7.5e-5, far below the
// bf16 rounding of P), exponent added as integer bits. x is clamped at -125 so
// the result stays a normal float (a masked-out score underflows to ~1e-38
// instead of 0; masked elements are zeroed by the caller anyway).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: round(x) lands in the low mantissa bits
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05517160520f, f, 0.24261111021f), f, 0.69326096773f), f, 0.99992805719f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

}  // namespace tc

// host: launch with programmatic stream serialization (PDL) and an optional
// cluster shape; kernels call pdl_wait() before their first global access.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              unsigned cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  static const bool pdl = std::getenv("LASP2_NO_PDL") == nullptr;  // diagnostic switch
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// host: opt a kernel into >48 KB dynamic smem once per (kernel, device).
inline cudaError_t set_smem_once(const void* kernel, uint32_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (done.count({kernel, dev})) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.insert({kernel, dev});
  return e;
}

// host: 3-D [slots][tokens][dim] and 4-D rank-major [ranks][slots][chunk][dim]
// bf16 tensor maps with 64 x 128 SWIZZLE_128B boxes (tc_host.cu)
cudaError_t make_tmap_3d(CUtensorMap* m, const void* ptr, int64_t slots, int64_t tokens, int dim);
cudaError_t make_tmap_3d_f32(CUtensorMap* m, const void* ptr, int64_t slots, int64_t tokens, int dim);
cudaError_t make_tmap_4d(CUtensorMap* m, const void* ptr, int64_t ranks, int64_t slots, int64_t chunk, int dim,
                         int64_t rank_stride_elems);

}  // namespace lasp
