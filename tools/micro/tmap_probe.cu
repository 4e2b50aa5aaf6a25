// Probe which 1-D tensor-map encodings the driver accepts (development aid).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
int main() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    printf("entry point: err=%d q=%d p=%p\n", (int)e, (int)q, p);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    float* buf;
    cudaMalloc(&buf, 1 << 26);
    CUtensorMap m;
    cuuint64_t dims[] = {264ull * 7680, 264ull * 4194304, 1ull << 20};
    for (cuuint64_t d : dims) {
        for (int strides_null = 0; strides_null < 2; ++strides_null)
            for (int l2 = 0; l2 < 2; ++l2) {
                cuuint64_t dim[1] = {d};
                cuuint64_t st[1] = {d * 4};
                cuuint32_t box[1] = {128};
                cuuint32_t es[1] = {1};
                CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, buf, dim, strides_null ? nullptr : st, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                printf("rank1 dim=%llu strides_null=%d l2=%d -> %d\n", (unsigned long long)d, strides_null, l2, (int)r);
            }
        // rank 2: (d/64) x 64? no: dim0 = 128-multiple rows
        cuuint64_t dim2[2] = {1024, d / 1024};
        cuuint64_t st2[1] = {1024 * 4};
        cuuint32_t box2[2] = {128, 1};
        cuuint32_t es2[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dim2, st2, box2, es2,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("rank2 -> %d\n", (int)r);
    }
    return 0;
}
