// Microbenchmark: DFMA issue rate on B200 vs warps per SM and independent
// chains per thread (informs the FP64-bound window kernel design).
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k(double* out, int iters, double a, double b) {
    double x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) x[c] = __fma_rn(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c];
    if (s == 12345.0) out[0] = s;
}

template <int C>
void run(int warps, double* d) {
    int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<C><<<148, warps * 32>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    k<C><<<148, warps * 32>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dfma = 148.0 * warps * 32 * (double)iters * C;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double per_clk_sm = dfma / (ms * 1e-3) / 148 / (clk * 1e3);
    printf("chains=%d warps/SM=%2d : %.2f TFLOP/s  %.1f DFMA/clk/SM (at %d MHz nominal)\n", C, warps,
           2 * dfma / (ms * 1e-3) / 1e12, per_clk_sm, clk / 1000);
}

int main() {
    double* d; cudaMalloc(&d, 8);
    for (int w : {4, 8, 12, 16, 24, 32}) { run<1>(w, d); run<2>(w, d); run<4>(w, d); run<8>(w, d); }
    return 0;
}
