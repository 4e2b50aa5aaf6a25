// Microbenchmark: do FP64 tensor-core MMAs (DMMA.8x8x4) and scalar DFMAs share
// one pipe on B200?  Runs DMMA alone, DFMA alone, and both interleaved in
// each warp; reports FP64 FMA/clk/SM (DMMA = 256 FMA per warp instruction,
// DFMA = 32).  If the mix exceeds either alone, the pipes are separate.
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int NF>
__global__ void k(double* out, int iters, double a, double b) {
    double acc[4][2];
    double x[8];
#pragma unroll
    for (int c = 0; c < 4; ++c) { acc[c][0] = c; acc[c][1] = -c; }
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
    const double ma = threadIdx.x * 1e-3, mb = 0.999;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < NM; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[c & 3][0]), "+d"(acc[c & 3][1]) : "d"(ma), "d"(mb));
#pragma unroll
        for (int c = 0; c < NF; ++c) x[c & 7] = __fma_rn(x[c & 7], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) s += acc[c][0] + acc[c][1];
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.0) out[0] = s;
}

template <int NM, int NF>
void run(const char* name, int warps, double* d) {
    int iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<NM, NF><<<148, warps * 32>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    k<NM, NF><<<148, warps * 32>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = 148.0 * warps * (double)iters * (NM * 256.0 + NF * 32.0);
    printf("%-22s warps/SM=%2d : %.1f FP64 FMA/clk/SM at 1.965 GHz (%.3f ms)\n", name, warps,
           fma / (ms * 1e-3) / 148 / 1.965e9, ms);
}

int main() {
    double* d; cudaMalloc(&d, 8);
    for (int w : {8, 16}) {
        run<4, 0>("DMMA x4", w, d);
        run<0, 32>("DFMA x32", w, d);
        run<4, 32>("DMMA x4 + DFMA x32", w, d);
        run<2, 32>("DMMA x2 + DFMA x32", w, d);
        run<4, 16>("DMMA x4 + DFMA x16", w, d);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
