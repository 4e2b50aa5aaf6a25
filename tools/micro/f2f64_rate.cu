// Microbenchmark: F2F.F64.F32 (float -> double widening) throughput on B200,
// alone and interleaved with DFMA, to see which pipe it uses.
#include <cstdio>
#include <cuda_runtime.h>

template <int NC, int NF>
__global__ void k(float* out, int iters, double a, double b) {
    float f[8];
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { f[c] = threadIdx.x * 1e-3f + c; x[c] = c; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            double d = (double)f[c & 7];             // F2F.F64.F32
            f[c & 7] = (float)__int_as_float(__double2hiint(d) ^ (i & 1));  // keep the chain alive cheaply
        }
#pragma unroll
        for (int c = 0; c < NF; ++c) x[c & 7] = __fma_rn(x[c & 7], a, b);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += f[c] + (float)x[c];
    if (s == 12345.0f) out[0] = s;
}

template <int NC, int NF>
void run(const char* name, double* dummy, float* d) {
    int iters = 4000, warps = 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<NC, NF><<<148, warps * 32>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    k<NC, NF><<<148, warps * 32>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lanes = 148.0 * warps * 32 * (double)iters;
    printf("%-18s: %.1f F2F/clk/SM, %.1f DFMA/clk/SM at 1.965 GHz (%.3f ms)\n", name,
           lanes * NC / (ms * 1e-3) / 148 / 1.965e9, lanes * NF / (ms * 1e-3) / 148 / 1.965e9, ms);
}

int main() {
    float* d; cudaMalloc(&d, 8);
    run<8, 0>("F2F.F64.F32 x8", nullptr, d);
    run<0, 8>("DFMA x8", nullptr, d);
    run<8, 8>("F2F x8 + DFMA x8", nullptr, d);
    run<4, 16>("F2F x4 + DFMA x16", nullptr, d);
    run<8, 16>("F2F x8 + DFMA x16", nullptr, d);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
