// Tuning sweep for the K1 streaming structure on c3-sized buffers (4e8 px,
// fp32 storage, fp64 Alg. 2 arithmetic).  Not the product kernel: the same
// I/O pattern with knobs (block size, grid cap, pixels per thread, cache
// hints) to find the fastest configuration on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ldnc(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ldplain(const float4* p) { return *p; }
__device__ __forceinline__ float4 ldcs(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ void stcs(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void stplain(float4* p, float4 v) { *p = v; }

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

template <int LD, int ST, int G>  // LD: 0 nc, 1 plain, 2 cs; ST: 0 cs, 1 plain; G groups/thread/iter
__global__ void k(const float* __restrict__ z, float* __restrict__ out, uint8_t* __restrict__ st, int64_t ng, int64_t ld) {
    for (int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); g0 < ng; g0 += (int64_t)gridDim.x * blockDim.x * G) {
        float4 in[G][9];
#pragma unroll
        for (int q = 0; q < G; ++q) {
            int64_t g = g0 + (int64_t)q * gridDim.x * blockDim.x;
            if (g < ng) {
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const float4* p = reinterpret_cast<const float4*>(z + k * ld) + g;
                    in[q][k] = LD == 0 ? ldnc(p) : (LD == 1 ? ldplain(p) : ldcs(p));
                }
            }
        }
#pragma unroll
        for (int q = 0; q < G; ++q) {
            int64_t g = g0 + (int64_t)q * gridDim.x * blockDim.x;
            if (g >= ng) break;
            float res[11][4];
            uint32_t sw = 0;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                double m[9], o[11];
#pragma unroll
                for (int k = 0; k < 9; ++k) m[k] = (&in[q][k].x)[v];
                alg2(m, o);
#pragma unroll
                for (int k = 0; k < 11; ++k) res[k][v] = (float)o[k];
                sw |= (o[9] > 1e-30 ? 0u : 1u) << (8 * v);
            }
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                float4* p = reinterpret_cast<float4*>(out + k * ld) + g;
                float4 v4 = make_float4(res[k][0], res[k][1], res[k][2], res[k][3]);
                if (ST == 0) stcs(p, v4); else stplain(p, v4);
            }
            reinterpret_cast<uint32_t*>(st)[g] = sw;
        }
    }
}

__global__ void fill(float* z, int64_t n, int64_t ld) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        float s = 1.0f + (p % 97) * 1e-3f;
        z[0 * ld + p] = 2 * s; z[1 * ld + p] = 0.1f; z[2 * ld + p] = 0.2f; z[3 * ld + p] = 0.05f; z[4 * ld + p] = -0.1f;
        z[5 * ld + p] = 1.5f * s; z[6 * ld + p] = 0.3f; z[7 * ld + p] = 0.01f; z[8 * ld + p] = 1.2f;
    }
}

template <int LD, int ST, int G>
void run(const char* name, const float* z, float* out, uint8_t* st, int64_t n, int block, int grid_cap) {
    int64_t ng = n / 4;
    int64_t need = (ng + block - 1) / block;
    int grid = (int)(need < grid_cap ? need : grid_cap);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) k<LD, ST, G><<<grid, block>>>(z, out, st, ng, n);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) k<LD, ST, G><<<grid, block>>>(z, out, st, ng, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-28s block=%4d grid=%8d : %.3f ms  %.1f GB/s\n", name, block, grid, ms, n * 81.0 / ms / 1e6);
}

int main() {
    const int64_t n = 400000000;
    float *z, *out; uint8_t* st;
    cudaMalloc(&z, 9 * n * 4); cudaMalloc(&out, 11 * n * 4); cudaMalloc(&st, n);
    fill<<<148 * 16, 256>>>(z, n, n);
    cudaDeviceSynchronize();
    const int FULL = 1 << 30;
    for (int rep = 0; rep < 2; ++rep) {
        run<0, 0, 1>("nc/cs full", z, out, st, n, 256, FULL);
        run<1, 0, 1>("plain/cs full", z, out, st, n, 256, FULL);
        run<1, 1, 1>("plain/plain full", z, out, st, n, 256, FULL);
        run<0, 1, 1>("nc/plain full", z, out, st, n, 256, FULL);
        run<2, 1, 1>("cs/plain full", z, out, st, n, 256, FULL);
        run<1, 1, 1>("plain/plain full b128", z, out, st, n, 128, FULL);
        run<1, 1, 1>("plain/plain full b512", z, out, st, n, 512, FULL);
        run<1, 1, 1>("plain/plain cap9472", z, out, st, n, 256, 148 * 64);
        run<0, 0, 1>("nc/cs cap9472", z, out, st, n, 256, 148 * 64);
    }
    // pure copy reference (9 in -> 11 out planes, no math): same traffic
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
