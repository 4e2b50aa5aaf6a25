// Microbenchmark: FP64 tensor-core MMA (mma.sync m8n8k4 f64) throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 0.999;
    double acc[C][2];
#pragma unroll
    for (int c = 0; c < C; ++c) { acc[c][0] = c; acc[c][1] = -c; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
    if (s == 12345.0) out[0] = s;
}

template <int C>
void run(int warps, double* d) {
    int iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<C><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e0);
    k<C><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = 148.0 * warps * (double)iters * C * 256;
    printf("chains=%d warps/SM=%2d : %.2f TFLOP/s (%.1f FMA/clk/SM at 1.965 GHz)\n", C, warps,
           2 * fma / (ms * 1e-3) / 1e12, fma / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
    double* d; cudaMalloc(&d, 8);
    for (int w : {4, 8, 16, 32}) { run<1>(w, d); run<2>(w, d); run<4>(w, d); run<8>(w, d); }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
