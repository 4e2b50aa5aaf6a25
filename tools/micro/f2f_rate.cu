// Microbenchmark: F2F.F32.F64 (double -> float) and MUFU.RCP throughput, and
// their cost when mixed with DFMA (does F2F occupy the FP64 pipe?).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
    double x[8];
    float acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { x[c] = threadIdx.x * 1e-3 + c; acc[c] = 0.f; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (MODE == 0) acc[c] += (float)x[c];                 // F2F only
            else if (MODE == 1) { x[c] = __fma_rn(x[c], 0.999, 1e-3); }  // DFMA only
            else if (MODE == 2) { x[c] = __fma_rn(x[c], 0.999, 1e-3); acc[c] += (float)x[c]; }  // 1 DFMA + 1 F2F
            else if (MODE == 4) {  // 4 DFMA + 1 F2F
                x[c] = __fma_rn(x[c], 0.999, 1e-3); x[c] = __fma_rn(x[c], 0.999, 1e-3);
                x[c] = __fma_rn(x[c], 0.999, 1e-3); x[c] = __fma_rn(x[c], 0.999, 1e-3);
                acc[c] += (float)x[c]; }
            else if (MODE == 5) {  // 4 DFMA + 1 MUFU
                x[c] = __fma_rn(x[c], 0.999, 1e-3); x[c] = __fma_rn(x[c], 0.999, 1e-3);
                x[c] = __fma_rn(x[c], 0.999, 1e-3); x[c] = __fma_rn(x[c], 0.999, 1e-3);
                float f = acc[c] + 1.0f; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"(f)); acc[c] = f; }
            else { float f = acc[c] + 1.0f; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"(f)); acc[c] = f; }  // MUFU
        }
        if (MODE == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] += 1.0;  // keep x changing (DADD, 1 per F2F)
        }
    }
    float r = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) r += acc[c] + (float)x[c];
    if (r == 12345.f) out[0] = r;
}

template <int MODE>
void run(int warps, float* d, const char* name) {
    int iters = 10000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e0);
    k<MODE><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double it = 148.0 * warps * 32 * (double)iters * 8;
    printf("%-28s warps/SM=%2d : %.1f iterations(lane)/clk/SM\n", name, warps, it / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
    float* d; cudaMalloc(&d, 8);
    for (int w : {16, 32}) {
        run<4>(w, d, "4 DFMA + 1 F2F");
        run<5>(w, d, "4 DFMA + 1 MUFU");
        run<0>(w, d, "F2F.F32.F64 + DADD");
        run<1>(w, d, "DFMA");
        run<2>(w, d, "DFMA + F2F.F32.F64");
        run<3>(w, d, "MUFU.RCP (+FADD)");
    }
    return 0;
}
