// Host-side TMA tensor-map encoding through the driver entry point (no -lcuda).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace tmb {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            throw std::runtime_error("cuTensorMapEncodeTiled is unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 3-D tensor, dims[0] contiguous; box {box0, box1, 1}; OOB reads are zero.
inline CUtensorMap make_tmap_3d(CUtensorMapDataType dt, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                                uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1,
                                CUtensorMapSwizzle sw) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
    const cuuint32_t box[3] = {box0, box1, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_tiled_fn()(&m, dt, 3, const_cast<void*>(base), dims, strides,
                                         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

inline CUtensorMap make_tmap_3d_f32(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                                    uint64_t stride2_bytes, uint32_t box0, uint32_t box1, CUtensorMapSwizzle sw) {
    return make_tmap_3d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, d0, d1, d2, stride1_bytes, stride2_bytes, box0, box1,
                        sw);
}

inline CUtensorMap make_tmap_3d_f16(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                                    uint64_t stride2_bytes, uint32_t box0, uint32_t box1, CUtensorMapSwizzle sw) {
    return make_tmap_3d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, base, d0, d1, d2, stride1_bytes, stride2_bytes, box0, box1,
                        sw);
}

}  // namespace tmb
