// Throughput of the warp-level TF32 tensor-core MMA (mma.sync.m16n8k8.tf32,
// fp32 accumulate) on B200 (sm_100a), for sizing a tensor-core NLM gather.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tf32_mma_rate tf32_mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(float* out, int iters) {
    unsigned a0 = __float_as_uint(1.0f + threadIdx.x * 1e-7f), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    unsigned b0 = __float_as_uint(0.5f), b1 = b0 + 5;
    float c[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * sms * 1024 * 4);
    const int iters = 20000;
    for (int warps : {4, 8, 16, 32}) {
        dim3 grid(sms), block(32 * warps);
        k<<<grid, block>>>(out, 10);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<grid, block>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double fma = (double)sms * warps * iters * 4 * 16 * 8 * 8;
        printf("warps/SM=%2d: %.1f T FMA/s (%.0f FMA/clk/SM at 1.965 GHz)\n", warps, fma / ms / 1e9,
               fma / (ms * 1e-3) / sms / 1.965e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
