// Host-side TMA tensor-map construction (driver entry point fetched through
// the runtime, so the library needs no -lcuda at link time).
#include "tc_common.cuh"

namespace lasp {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// [slots][tokens][dim] bf16, box = 64 features x 128 tokens, SWIZZLE_128B.
cudaError_t make_tmap_3d(CUtensorMap* m, const void* ptr, int64_t slots, int64_t tokens, int dim) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t gdim[3] = {(cuuint64_t)dim, (cuuint64_t)tokens, (cuuint64_t)slots};
  cuuint64_t gstride[2] = {(cuuint64_t)dim * 2, (cuuint64_t)tokens * dim * 2};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// [slots][tokens][dim] fp32, box = 32 features x 128 tokens (128-byte rows), SWIZZLE_128B.
cudaError_t make_tmap_3d_f32(CUtensorMap* m, const void* ptr, int64_t slots, int64_t tokens, int dim) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t gdim[3] = {(cuuint64_t)dim, (cuuint64_t)tokens, (cuuint64_t)slots};
  cuuint64_t gstride[2] = {(cuuint64_t)dim * 4, (cuuint64_t)tokens * dim * 4};
  cuuint32_t box[3] = {32, 128, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// [ranks][slots][chunk][dim] with a free rank stride (elements), e.g. the
// all_gather output of T contiguous [slots][chunk][dim] contributions.
cudaError_t make_tmap_4d(CUtensorMap* m, const void* ptr, int64_t ranks, int64_t slots, int64_t chunk, int dim,
                         int64_t rank_stride_elems) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t gdim[4] = {(cuuint64_t)dim, (cuuint64_t)chunk, (cuuint64_t)slots, (cuuint64_t)ranks};
  cuuint64_t gstride[3] = {(cuuint64_t)dim * 2, (cuuint64_t)chunk * dim * 2,
                           (cuuint64_t)(ranks > 1 ? rank_stride_elems : slots * chunk * dim) * 2};
  cuuint32_t box[4] = {64, 128, 1, 1};
  cuuint32_t estride[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace lasp
