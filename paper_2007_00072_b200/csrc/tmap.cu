// TMA tensor-map encoding without linking libcuda: cuTensorMapEncodeTiled is resolved once
// through the runtime's driver entry-point query, so libencoder.so loads (and its host-side
// argument checks run) on machines without a GPU driver.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "kernels.h"

namespace enc {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUresult tmap_encode_tiled(CUtensorMap* map, CUtensorMapDataType dtype, cuuint32_t rank,
                           void* addr, const cuuint64_t* dims, const cuuint64_t* strides,
                           const cuuint32_t* box, const cuuint32_t* estrides,
                           CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                           CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) return CUDA_ERROR_NOT_FOUND;
  return fn(map, dtype, rank, addr, dims, strides, box, estrides, il, sw, l2, oob);
}

bool map_pop(CUtensorMap* m, const void* ptr, int B, int H, int rows, int P, int64_t ld,
             int box_rows) {
  const bool head_major = ld == P;
  const uint64_t sh = head_major ? (uint64_t)rows * P : (uint64_t)P;   // h
  const uint64_t sr = head_major ? (uint64_t)P : (uint64_t)ld;         // row
  const uint64_t sb = head_major ? (uint64_t)H * rows * P : (uint64_t)rows * ld;  // b
  cuuint64_t gdim[4] = {(cuuint64_t)P, (cuuint64_t)H, (cuuint64_t)rows, (cuuint64_t)B};
  cuuint64_t gstr[3] = {sh * 2, sr * 2, sb * 2};
  cuuint32_t bdim[4] = {64, 1, (cuuint32_t)box_rows, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return tmap_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), gdim,
                           gstr, bdim, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace enc
