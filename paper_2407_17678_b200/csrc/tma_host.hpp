// Host-side TMA tensor-map construction (driver entry point fetched through
// the runtime, so nothing links against libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace s2host {

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D bf16 tensor [outer][rows][inner] (inner contiguous), box
// {box_inner, box_rows, 1}, 128-byte swizzle, out-of-bounds rows read as 0.
inline CUtensorMap make_map_bf16_3d(const void* base, uint64_t inner, uint64_t rows,
                                    uint64_t outer, uint32_t box_inner, uint32_t box_rows,
                                    CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {inner, rows, outer};
    const cuuint64_t strides[2] = {inner * 2, inner * rows * 2};
    const cuuint32_t box[3] = {box_inner, box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = tensor_map_encoder()(
        &m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

// The same [outer][rows][inner] bf16 tensor viewed 4-D as [outer][inner/64][rows][64]
// (strides: row inner*2 B, 64-column slice 128 B): one box {64, box_rows,
// inner/64, 1} moves box_rows full rows and lands in shared memory as
// [inner/64][box_rows][64] with 128-byte swizzle -- the SW128 K-major layout of
// the MMA operands, slices box_rows*128 B apart.  One 16-32 KB box per load
// instead of inner/64 boxes of 8-16 KB: per-SM TMA throughput grows with the
// box size (tools/probe_tma2.cu: 64-row chunk of D=128 as one box 32-45
// B/cycle/SM vs 23-27 as two).
inline CUtensorMap make_map_bf16_kmajor(const void* base, uint64_t inner, uint64_t rows,
                                        uint64_t outer, uint32_t box_rows) {
    if (inner % 64 != 0) throw std::runtime_error("make_map_bf16_kmajor: inner % 64 != 0");
    CUtensorMap m;
    const cuuint64_t dims[4] = {64, rows, inner / 64, outer};
    const cuuint64_t strides[3] = {inner * 2, 128, inner * rows * 2};
    const cuuint32_t box[4] = {64, box_rows, static_cast<cuuint32_t>(inner / 64), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = tensor_map_encoder()(
        &m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw std::runtime_error("cuTensorMapEncodeTiled (4-D) failed: " + std::to_string(int(r)));
    return m;
}

}  // namespace s2host
