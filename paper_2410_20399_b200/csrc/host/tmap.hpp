// tmap.hpp — host-side CUtensorMap construction (the `gl` global-layout
// descriptor). The driver entry point is resolved through the runtime so the
// library does not link libcuda directly.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

namespace tkb {
namespace host {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || p == nullptr)
            return (EncodeTiledFn) nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// Row-major tensor of `rank` dims (dims[0] innermost, contiguous), element
// strides for dims 1..rank-1 in ELEMENTS. Box sizes per dim; swizzle 128B
// requires box[0] * elem_bytes == 128 (one atom wide).
inline bool make_tmap(CUtensorMap* out, const void* base, CUtensorMapDataType dtype, int elem_bytes, int rank,
                      const uint64_t* dims, const uint64_t* strides_elems, const uint32_t* box,
                      CUtensorMapSwizzle swz, std::string* err) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) {
        if (err) *err = "cuTensorMapEncodeTiled unavailable (driver too old?)";
        return false;
    }
    cuuint64_t gdim[5];
    cuuint64_t gstride[4];
    cuuint32_t bdim[5];
    cuuint32_t estride[5];
    for (int i = 0; i < rank; ++i) {
        gdim[i] = dims[i];
        bdim[i] = box[i];
        estride[i] = 1;
    }
    for (int i = 1; i < rank; ++i) gstride[i - 1] = strides_elems[i] * (uint64_t)elem_bytes;
    std::memset(out, 0, sizeof(*out));
    CUresult r = fn(out, dtype, (cuuint32_t)rank, const_cast<void*>(base), gdim, gstride, bdim, estride,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        if (err) *err = "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r);
        return false;
    }
    return true;
}

}  // namespace host
}  // namespace tkb
