// Microbenchmark: B200 FP64 pipe rate for DFMA, DADD, DMUL and a mix like
// the window kernel's pair (9 DADD : 6 DMUL : 14 DFMA), 16 warps/SM, 4 chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int C>
__global__ void k(double* out, int iters, double a, double b) {
    double x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (OP == 0) x[c] = __fma_rn(x[c], a, b);
            if (OP == 1) x[c] = __dadd_rn(x[c], b);
            if (OP == 2) x[c] = __dmul_rn(x[c], a);
            if (OP == 3) {  // 29-op mix: 9 add, 6 mul, 14 fma
#pragma unroll
                for (int j = 0; j < 9; ++j) x[c] = __dadd_rn(x[c], b);
#pragma unroll
                for (int j = 0; j < 6; ++j) x[c] = __dmul_rn(x[c], a);
#pragma unroll
                for (int j = 0; j < 14; ++j) x[c] = __fma_rn(x[c], a, b);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c];
    if (s == 12345.0) out[0] = s;
}

template <int OP, int C>
void run(const char* name, int warps, double* d) {
    int iters = OP == 3 ? 1000 : 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<OP, C><<<148, warps * 32>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    k<OP, C><<<148, warps * 32>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 148.0 * warps * 32 * (double)iters * C * (OP == 3 ? 29 : 1);
    printf("%-5s chains=%d warps/SM=%2d : %.1f ops/clk/SM at 1965 MHz (%.3f ms)\n", name, C, warps,
           ops / (ms * 1e-3) / 148 / 1.965e9, ms);
}

int main() {
    double* d; cudaMalloc(&d, 8);
    for (int w : {8, 16, 32}) {
        run<0, 4>("DFMA", w, d); run<1, 4>("DADD", w, d); run<2, 4>("DMUL", w, d); run<3, 4>("mix", w, d);
        run<0, 8>("DFMA", w, d); run<1, 8>("DADD", w, d); run<2, 8>("DMUL", w, d);
    }
    return 0;
}
