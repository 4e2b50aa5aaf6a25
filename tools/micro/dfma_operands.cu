// Microbenchmark: DFMA throughput when all three operands are distinct
// registers (no uniform / constant operands), versus one shared operand.
#include <cstdio>
#include <cuda_runtime.h>

template <int C, int MODE>
__global__ void k(double* out, int iters) {
    double x[C], y[C], w[C];
#pragma unroll
    for (int c = 0; c < C; ++c) { x[c] = threadIdx.x * 1e-3 + c; y[c] = 0.999 - c * 1e-6; w[c] = 1e-3 * c; }
    double s = 0.5 + threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (MODE == 0) x[c] = __fma_rn(x[c], y[c], w[c]);        // 3 distinct registers
            else if (MODE == 1) x[c] = __fma_rn(x[c], s, w[c]);      // one operand shared by all chains
            else x[c] = __dadd_rn(x[c], w[c]);                       // DADD, 2 registers
        }
#pragma unroll
        for (int c = 0; c < C; ++c) { double t = y[c]; y[c] = w[c]; w[c] = t; }
    }
    double r = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) r += x[c] + y[c] + w[c];
    if (r == 12345.0) out[0] = r;
}

template <int C, int MODE>
void run(int warps, double* d) {
    int iters = 10000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<C, MODE><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e0);
    k<C, MODE><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 148.0 * warps * 32 * (double)iters * C;
    printf("mode=%d (%s) chains=%d warps/SM=%2d : %.1f lane-ops/clk/SM at 1.965 GHz\n", MODE,
           MODE == 0 ? "DFMA 3 reg" : (MODE == 1 ? "DFMA shared" : "DADD"), C, warps,
           ops / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
    double* d; cudaMalloc(&d, 8);
    for (int w : {8, 16, 32}) {
        run<8, 0>(w, d); run<8, 1>(w, d); run<8, 2>(w, d);
    }
    return 0;
}
