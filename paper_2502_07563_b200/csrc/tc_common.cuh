// Shared device helpers of the tcgen05 kernels (tile geometry, UMMA
// descriptors for SWIZZLE_128B images, TMEM -> smem conversion).
#pragma once
#include <cuda.h>

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

// Load a 128-column fp32 row from TMEM (this thread's lane) in four x32 pieces,
// convert to bf16 (optionally causal-masked) and write into a SW128 image.
// mask: 0 none, 1 keep col<=row, 2 keep col>=row.
__device__ __forceinline__ void tmem_row_to_image(uint32_t taddr_lane, uint8_t* img, uint32_t row, int mask) {
#pragma unroll 1
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr_lane + c0, r);
    tmem_ld_wait();
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float x = __uint_as_float(r[i]);
      const int col = c0 + i;
      if (mask == 1 && col > (int)row) x = 0.f;
      if (mask == 2 && col < (int)row) x = 0.f;
      v[i] = x;
    }
    st_row32_bf16(img, row, c0, v);
  }
}

// Columns [c_begin, c_begin + ncols) (multiple of 32) of this thread's TMEM lane
// -> bf16 (optionally causal-masked: 1 keep col<=row, 2 keep col>=row) -> SW128 image.
__device__ __forceinline__ void tmem_cols_to_image(uint32_t taddr_lane, uint8_t* img, uint32_t row, int c_begin,
                                                   int ncols, int mask) {
#pragma unroll 1
  for (int c0 = c_begin; c0 < c_begin + ncols; c0 += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr_lane + c0, r);
    tmem_ld_wait();
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float x = __uint_as_float(r[i]);
      const int col = c0 + i;
      if (mask == 1 && col > (int)row) x = 0.f;
      if (mask == 2 && col < (int)row) x = 0.f;
      v[i] = x;
    }
    st_row32_bf16(img, row, c0, v);
  }
}

}  // namespace tc

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
cudaError_t make_tmap_4d(CUtensorMap* m, const void* ptr, int64_t ranks, int64_t slots, int64_t chunk, int dim,
                         int64_t rank_stride_elems);

}  // namespace lasp
