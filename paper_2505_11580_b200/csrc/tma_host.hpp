// Host-side TMA tensor-map construction (cuTensorMapEncodeTiled fetched through the
// runtime's driver entry point, so the library needs no -lcuda at link time).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace fipa_b200 {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        if (e != cudaSuccess || p == nullptr || q != cudaDriverEntryPointSuccess) {
            throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
        }
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// Row-major bf16 matrix [rows, cols] (cols contiguous, row stride `ld` elements),
// box {box_cols (inner, must be 64 for SWIZZLE_128B), box_rows}.
inline CUtensorMap make_map_2d_bf16(const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                                    uint32_t box_cols, uint32_t box_rows) {
    CUtensorMap m{};
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(2d) failed: " + std::to_string(int(r)));
    }
    return m;
}

// fp32 tensor [d2, d1, d0] (d0 contiguous, rows of `ld` elements), box {box0, box1, 1},
// SWIZZLE_128B (box0 = 32: one 128-byte row).
inline CUtensorMap make_map_3d_f32(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t ld,
                                   uint32_t box0, uint32_t box1) {
    CUtensorMap m{};
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {ld * 4, ld * 4 * d1};
    cuuint32_t box[3] = {box0, box1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled(3d f32) failed: " + std::to_string(int(r)));
    return m;
}

// bf16 tensor [d2, d1, d0] (d0 contiguous, rows of `ld` elements), box {box0, box1, 1}.
inline CUtensorMap make_map_3d_bf16(const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                                    uint64_t ld, uint32_t box0, uint32_t box1) {
    CUtensorMap m{};
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {ld * 2, ld * 2 * d1};
    cuuint32_t box[3] = {box0, box1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base),
                                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(3d) failed: " + std::to_string(int(r)));
    }
    return m;
}

// bf16 tensor [d2][rows][ld] viewed as 128-byte column blocks: 4-D map
// {64 elements, rows, ld/64 blocks, d2} with strides {ld*2, 128, rows*ld*2}, so a single box
// {64, box_rows, nblk, 1} lands in shared memory as nblk consecutive [box_rows][128 B] blocks --
// exactly the SWIZZLE_128B K-major operand layout -- in ONE TMA instruction.  ld % 64 == 0.
inline CUtensorMap make_map_blocks_bf16(const void* base, uint64_t rows, uint64_t d2, uint64_t ld,
                                        uint32_t box_rows, uint32_t nblk) {
    CUtensorMap m{};
    cuuint64_t dims[4] = {64, rows, ld / 64, d2};
    cuuint64_t strides[3] = {ld * 2, 128, rows * ld * 2};
    cuuint32_t box[4] = {64, box_rows, nblk, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base),
                                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(4d blocks) failed: " + std::to_string(int(r)));
    }
    return m;
}

// fp32 matrix [rows][ld] viewed as 128-byte (32-float) column blocks, one box = {32, box_rows,
// nblk}: nblk consecutive SWIZZLE_128B [box_rows][128 B] blocks in shared memory.  ld % 32 == 0.
inline CUtensorMap make_map_blocks_f32(const void* base, uint64_t rows, uint64_t ld, uint32_t box_rows,
                                       uint32_t nblk) {
    CUtensorMap m{};
    cuuint64_t dims[3] = {32, rows, ld / 32};
    cuuint64_t strides[2] = {ld * 4, 128};
    cuuint32_t box[3] = {32, box_rows, nblk};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base),
                                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(f32 blocks) failed: " + std::to_string(int(r)));
    }
    return m;
}

// Key/value rows gathered from G shards: bf16 [G][d2][rows][ld] (row i of shard g is global key
// g*rows + i).  5-D block map {64, rows, ld/64, d2, G}: one box {64, box_rows, nblk, 1, 1} is the
// same 128-byte-block operand tile as make_map_blocks_bf16.  G = 1 is the unsharded layout.
inline CUtensorMap make_map_blocks_bf16_sharded(const void* base, uint64_t rows, uint64_t d2, uint64_t G,
                                                uint64_t ld, uint32_t box_rows, uint32_t nblk) {
    CUtensorMap m{};
    cuuint64_t dims[5] = {64, rows, ld / 64, d2, G};
    cuuint64_t strides[4] = {ld * 2, 128, rows * ld * 2, d2 * rows * ld * 2};
    cuuint32_t box[5] = {64, box_rows, nblk, 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(5d sharded blocks) failed: " + std::to_string(int(r)));
    }
    return m;
}

// bf16 [G][d2][rows][ld] as a 4-D map {ld, rows, d2, G} with box {box0, box1, 1, 1}.
inline CUtensorMap make_map_4d_bf16_sharded(const void* base, uint64_t ld, uint64_t rows, uint64_t d2, uint64_t G,
                                            uint32_t box0, uint32_t box1) {
    CUtensorMap m{};
    cuuint64_t dims[4] = {ld, rows, d2, G};
    cuuint64_t strides[3] = {ld * 2, rows * ld * 2, d2 * rows * ld * 2};
    cuuint32_t box[4] = {box0, box1, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(4d sharded) failed: " + std::to_string(int(r)));
    }
    return m;
}

// fp32 matrix [rows, cols] (row stride ld elements), box {box_cols (<= 32: 128 B), box_rows}, SWIZZLE_128B.
inline CUtensorMap make_map_2d_f32(const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_cols,
                                   uint32_t box_rows) {
    CUtensorMap m{};
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * 4};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(2d f32) failed: " + std::to_string(int(r)));
    }
    return m;
}

// fp32 [d3][d2][d1][d0] (d0 contiguous), box {box0, box1, box2, box3}, SWIZZLE_128B (box0 * 4 <= 128).
inline CUtensorMap make_map_4d_f32(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3,
                                   uint32_t box0, uint32_t box1, uint32_t box2, uint32_t box3) {
    CUtensorMap m{};
    cuuint64_t dims[4] = {d0, d1, d2, d3};
    cuuint64_t strides[3] = {d0 * 4, d0 * d1 * 4, d0 * d1 * d2 * 4};
    cuuint32_t box[4] = {box0, box1, box2, box3};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(4d f32) failed: " + std::to_string(int(r)));
    }
    return m;
}

// fp32 4-D tensor with explicit byte strides of dims 1..3, box {box0, box1, box2, box3}, SWIZZLE_128B.
inline CUtensorMap make_map_4d_f32_strided(const void* base, const uint64_t dims_in[4], const uint64_t strides_in[3],
                                           const uint32_t box_in[4]) {
    CUtensorMap m{};
    cuuint64_t dims[4] = {dims_in[0], dims_in[1], dims_in[2], dims_in[3]};
    cuuint64_t strides[3] = {strides_in[0], strides_in[1], strides_in[2]};
    cuuint32_t box[4] = {box_in[0], box_in[1], box_in[2], box_in[3]};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(4d f32 strided) failed: " + std::to_string(int(r)));
    }
    return m;
}

// bf16 4-D tensor with explicit byte strides of dims 1..3, box {box0 (64: one 128-byte row), ...},
// SWIZZLE_128B.
inline CUtensorMap make_map_4d_bf16_strided(const void* base, const uint64_t dims_in[4], const uint64_t strides_in[3],
                                            const uint32_t box_in[4]) {
    CUtensorMap m{};
    cuuint64_t dims[4] = {dims_in[0], dims_in[1], dims_in[2], dims_in[3]};
    cuuint64_t strides[3] = {strides_in[0], strides_in[1], strides_in[2]};
    cuuint32_t box[4] = {box_in[0], box_in[1], box_in[2], box_in[3]};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(4d bf16 strided) failed: " + std::to_string(int(r)));
    }
    return m;
}

// bf16 5-D tensor with explicit byte strides of dims 1..4, box {box0 (64: one 128-byte row), ...},
// SWIZZLE_128B.
inline CUtensorMap make_map_5d_bf16_strided(const void* base, const uint64_t dims_in[5], const uint64_t strides_in[4],
                                            const uint32_t box_in[5]) {
    CUtensorMap m{};
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    for (int i = 0; i < 5; ++i) {
        dims[i] = dims_in[i];
        box[i] = box_in[i];
    }
    for (int i = 0; i < 4; ++i) strides[i] = strides_in[i];
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(5d bf16 strided) failed: " + std::to_string(int(r)));
    }
    return m;
}

// fp32 5-D tensor with explicit byte strides of dims 1..4, box {box0..box4}, SWIZZLE_128B
// (box0 * 4 == 128: one 128-byte row per box row).
inline CUtensorMap make_map_5d_f32_strided(const void* base, const uint64_t dims_in[5], const uint64_t strides_in[4],
                                           const uint32_t box_in[5]) {
    CUtensorMap m{};
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    for (int i = 0; i < 5; ++i) {
        dims[i] = dims_in[i];
        box[i] = box_in[i];
    }
    for (int i = 0; i < 4; ++i) strides[i] = strides_in[i];
    CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        throw std::runtime_error("cuTensorMapEncodeTiled(5d f32 strided) failed: " + std::to_string(int(r)));
    }
    return m;
}

}  // namespace fipa_b200
