// K1's I/O at the c2 size (1024^2 fp32 pixels, 84 MB per pass, L2 flushed by a
// 512 MB read before each launch): one 4-pixel group per thread (the product
// form) against G groups per thread with all loads issued first.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void alg2(const double* m, double* o) {
    double a = m[0], br = m[1], bi = m[2], cr = m[3], ci = m[4], d = m[5], er = m[6], ei = m[7], f = m[8];
    double ai = __fma_rn(d, f, -__fma_rn(er, er, ei * ei));
    double bir = __fma_rn(cr, er, __fma_rn(ci, ei, -br * f));
    double bii = __fma_rn(ci, er, -__fma_rn(cr, ei, bi * f));
    double cir = __fma_rn(br, er, -__fma_rn(bi, ei, cr * d));
    double cii = __fma_rn(br, ei, __fma_rn(bi, er, -ci * d));
    double di = __fma_rn(a, f, -__fma_rn(cr, cr, ci * ci));
    double eir = __fma_rn(cr, br, __fma_rn(ci, bi, -a * er));
    double eii = __fma_rn(ci, br, -__fma_rn(cr, bi, a * ei));
    double fi = __fma_rn(a, d, -__fma_rn(br, br, bi * bi));
    double det = __fma_rn(a, ai, __fma_rn(br, bir, __fma_rn(bi, bii, __fma_rn(cr, cir, ci * cii))));
    double t = __drcp_rn(det);
    o[0] = t * ai; o[1] = t * bir; o[2] = t * bii; o[3] = t * cir; o[4] = t * cii;
    o[5] = t * di; o[6] = t * eir; o[7] = t * eii; o[8] = t * fi; o[9] = det; o[10] = t;
}

template <int G, int TB>
__global__ void __launch_bounds__(TB) k(const float* __restrict__ z, float* __restrict__ out,
                                        uint8_t* __restrict__ st, int64_t ng, int64_t ld) {
    const int64_t g0 = blockIdx.x * (int64_t)TB * G + threadIdx.x;
    float4 in[G][9];
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const int64_t g = g0 + q * TB;
        if (g < ng) {
#pragma unroll
            for (int k = 0; k < 9; ++k) in[q][k] = reinterpret_cast<const float4*>(z + k * ld)[g];
        }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const int64_t g = g0 + q * TB;
        if (g >= ng) break;
        float res[11][4];
        uint32_t sw = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            double m[9], o[11];
            const float* iv = reinterpret_cast<const float*>(&in[q][0]);
#pragma unroll
            for (int kk = 0; kk < 9; ++kk) m[kk] = reinterpret_cast<const float*>(&in[q][kk])[v];
            alg2(m, o);
#pragma unroll
            for (int kk = 0; kk < 11; ++kk) res[kk][v] = (float)o[kk];
            sw |= (uint32_t)(o[9] > 0 ? 0 : 1) << (8 * v);
            (void)iv;
        }
#pragma unroll
        for (int kk = 0; kk < 11; ++kk)
            reinterpret_cast<float4*>(out + kk * ld)[g] = make_float4(res[kk][0], res[kk][1], res[kk][2], res[kk][3]);
        reinterpret_cast<uint32_t*>(st)[g] = sw;
    }
}

template <int G, int TB>
void run(const char* name, const float* z, float* out, uint8_t* st, int64_t n, char* flush, int64_t* sink) {
    const int64_t ng = n / 4;
    const int64_t grid = (ng + (int64_t)TB * G - 1) / ((int64_t)TB * G);
    for (int i = 0; i < 3; ++i) k<G, TB><<<grid, TB>>>(z, out, st, ng, n);
    float tot = 0;
    const int reps = 50;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < reps; ++i) {
        cudaMemsetAsync(flush, i, 1);  // touch
        // a 512 MB read flush
        extern void flush_read(const char*, int64_t*);
        flush_read(flush, sink);
        cudaEventRecord(e0);
        k<G, TB><<<grid, TB>>>(z, out, st, ng, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
    }
    const double ms = tot / reps;
    printf("%-28s %.2f us  %.1f GB/s\n", name, ms * 1e3, n * 81.0 / (ms * 1e-3) / 1e9);
}

__global__ void kflush(const int4* p, int64_t n, int64_t* sink) {
    int64_t s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += p[i].x;
    if (s == 42) *sink = s;
}
void flush_read(const char* f, int64_t* sink) { kflush<<<148 * 8, 256>>>((const int4*)f, (512ll << 20) / 16, sink); }

int main() {
    const int64_t n = 1 << 20;
    float *z, *out; uint8_t* st; char* flush; int64_t* sink;
    cudaMalloc(&z, 9 * n * 4); cudaMalloc(&out, 11 * n * 4); cudaMalloc(&st, n);
    cudaMalloc(&flush, 512ll << 20); cudaMalloc(&sink, 8);
    cudaMemset(z, 0, 9 * n * 4); cudaMemset(flush, 1, 512ll << 20);
    for (int r = 0; r < 2; ++r) {
        run<1, 128>("G=1 TB=128 (product)", z, out, st, n, flush, sink);
        run<2, 128>("G=2 TB=128", z, out, st, n, flush, sink);
        run<4, 128>("G=4 TB=128", z, out, st, n, flush, sink);
        run<1, 256>("G=1 TB=256", z, out, st, n, flush, sink);
        run<2, 64>("G=2 TB=64", z, out, st, n, flush, sink);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
