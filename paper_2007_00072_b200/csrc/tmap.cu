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

}  // namespace enc
