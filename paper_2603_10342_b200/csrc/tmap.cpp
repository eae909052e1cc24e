// TMA tensor-map creation through the driver entry point (no link-time libcuda
// dependency, so the C-ABI library also loads on GPU-less hosts).
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "gemm.h"

namespace asb {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess) {
            fn = reinterpret_cast<EncodeFn>(p);
        }
    });
    return fn;
}
}  // namespace

bool make_tmap_bf16(CUtensorMap* out, const void* base, int rows, int cols, int row_stride_elems,
                    int box_rows) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride_elems) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tmap_bf16_3d(CUtensorMap* out, const void* base, int d0, int d1, int d2, int b1, int b2) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(d0), static_cast<cuuint64_t>(d1),
                          static_cast<cuuint64_t>(d2)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(d0) * 2, static_cast<cuuint64_t>(d0) * d1 * 2};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(b1), static_cast<cuuint32_t>(b2)};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tmap_packed(CUtensorMap* out, const void* base, int rows_padded, int cols, int box_tiles,
                      int box_kb) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    const int kb = cols / 64, nt = rows_padded / 128;
    cuuint64_t dims[4] = {64, 128, static_cast<cuuint64_t>(kb), static_cast<cuuint64_t>(nt)};
    cuuint64_t strides[3] = {128, 128 * 128, static_cast<cuuint64_t>(kb) * 128 * 128};
    cuuint32_t box[4] = {64, 128, static_cast<cuuint32_t>(box_kb), static_cast<cuuint32_t>(box_tiles)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tmap_kv_sub(CUtensorMap* out, const void* base, long pages, int hd, int page_rows, int box_rows) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    const int halves = hd / 64;
    // (col within a 64-col half, row within a K or V page, half, K|V, page)
    cuuint64_t dims[5] = {64, static_cast<cuuint64_t>(page_rows), static_cast<cuuint64_t>(halves), 2,
                          static_cast<cuuint64_t>(pages)};
    const cuuint64_t row_b = static_cast<cuuint64_t>(hd) * 2;
    cuuint64_t strides[4] = {row_b, 128, row_b * page_rows, row_b * page_rows * 2};
    cuuint32_t box[5] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(halves), 2, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tmap_act_kpair(CUtensorMap* out, const void* base, int rows, int cols, int box_rows) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>((cols + 63) / 64)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 2, 128};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace asb
