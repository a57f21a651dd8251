// tmap.cuh -- host-side TMA tensor-map encoding (cuTensorMapEncodeTiled via the
// runtime's driver entry point: no libcuda link dependency).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include <cstring>

namespace splatct {

// Encode a tiled tensor map of a rank-r tensor (dims[0] innermost, strides in
// bytes for dims 1..r-1) with the given box; false when the driver entry
// point is missing, SPLATCT_NO_TMA is set, or the encoding is rejected (the
// caller then takes its non-TMA path).
inline bool encode_tiled(CUtensorMap* m, CUtensorMapDataType dtype, int rank, const void* base,
                         const cuuint64_t* dims, const cuuint64_t* strides,
                         const cuuint32_t* box, CUtensorMapSwizzle swizzle) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    memset(m, 0, sizeof(*m));
    if (!encode || ((uintptr_t)base & 15) != 0 || getenv("SPLATCT_NO_TMA")) return false;
    cuuint32_t estride[5] = {1, 1, 1, 1, 1};
    return encode(m, dtype, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace splatct
