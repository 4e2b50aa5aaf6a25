// Minimal 1-D TMA tile load test (development aid): which coordinates and
// which ways of passing the tensor map work.  Usage: tma1d_test <case>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, int c0, float* out, int mode) {
    __shared__ __align__(128) float buf0[256];
    float* buf = buf0 + (mode == 1 ? 4 : 0);  // mode 1: 16-byte (not 128-byte) aligned destination
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(512) : "memory");
        const void* pm = &m;
        if (mode == 2)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    smem_u32(buf)), "l"(pm), "r"(c0), "r"(1), "r"(smem_u32(&bar)) : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
                    smem_u32(buf)), "l"(pm), "r"(c0), "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
    out[threadIdx.x] = buf[threadIdx.x];
}

int main(int argc, char** argv) {
    int c0 = argc > 1 ? atoi(argv[1]) : 0;
    int mode = argc > 2 ? atoi(argv[2]) : 0;  // 0: 1-D, 1: 1-D to a 16-B aligned slot, 2: 2-D (500 x 2)
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    const int n = 1000;
    float* d;
    cudaMalloc(&d, n * 4);
    float h[n];
    for (int i = 0; i < n; ++i) h[i] = (float)i;
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    CUtensorMap m;
    cuuint64_t dim[1] = {(cuuint64_t)n};
    cuuint64_t st[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[1] = {128}, es[1] = {1};
    cuuint64_t dim2[2] = {500, 2};
    cuuint64_t st2[1] = {500 * 4};
    cuuint32_t box2[2] = {128, 1}, es2[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, mode == 2 ? 2 : 1, d, mode == 2 ? dim2 : dim, mode == 2 ? st2 : st,
                     mode == 2 ? box2 : box, mode == 2 ? es2 : es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    float* o;
    cudaMalloc(&o, 128 * 4);
    k<<<1, 128>>>(m, c0, o, mode);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[128];
    cudaMemcpy(ho, o, 512, cudaMemcpyDeviceToHost);
    printf("mode=%d c0=%d encode=%d kernel=%s  out[0]=%g out[1]=%g out[127]=%g\n", mode, c0, (int)r, cudaGetErrorString(e), ho[0],
           ho[1], ho[127]);
    return e != cudaSuccess;
}
