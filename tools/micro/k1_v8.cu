// K1's I/O with 256-bit vectors (8 fp32 pixels per plane per thread:
// ld.global.v8.f32 / st.global.v8.f32, sm_100) against the product's 128-bit
// form, on c3-sized buffers (4e8 px): does B200 stream the 9-in / 11-out
// pattern faster with wider accesses?  Alg. 2 in fp64 as in K1 (plain form).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct f8 { float v[8]; };
__device__ __forceinline__ f8 ld8(const float* p) {
    f8 r;
    asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                   "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
    return r;
}
__device__ __forceinline__ void st8(float* p, const f8& r) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "f"(r.v[0]), "f"(r.v[1]),
                 "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7]) : "memory");
}

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

template <int W>  // pixels per thread per plane: 4 (128-bit) or 8 (256-bit)
__global__ void __launch_bounds__(128) k(const float* __restrict__ z, float* __restrict__ out,
                                         uint8_t* __restrict__ st, int64_t ng, int64_t ld) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    float in[9][W];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const float* p = z + k * ld + g * W;
        if constexpr (W == 8) {
            f8 r = ld8(p);
#pragma unroll
            for (int v = 0; v < 8; ++v) in[k][v] = r.v[v];
        } else {
            float4 r = *reinterpret_cast<const float4*>(p);
            in[k][0] = r.x; in[k][1] = r.y; in[k][2] = r.z; in[k][3] = r.w;
        }
    }
    float res[11][W];
    uint64_t sw = 0;
#pragma unroll
    for (int v = 0; v < W; ++v) {
        double m[9], o[11];
#pragma unroll
        for (int k = 0; k < 9; ++k) m[k] = in[k][v];
        alg2(m, o);
#pragma unroll
        for (int k = 0; k < 11; ++k) res[k][v] = (float)o[k];
        sw |= (uint64_t)(o[9] > 0 ? 0 : 1) << (8 * v);
    }
#pragma unroll
    for (int k = 0; k < 11; ++k) {
        float* p = out + k * ld + g * W;
        if constexpr (W == 8) {
            f8 r;
#pragma unroll
            for (int v = 0; v < 8; ++v) r.v[v] = res[k][v];
            st8(p, r);
        } else {
            *reinterpret_cast<float4*>(p) = make_float4(res[k][0], res[k][1], res[k][2], res[k][3]);
        }
    }
    if constexpr (W == 8) *reinterpret_cast<uint64_t*>(st + g * 8) = sw;
    else *reinterpret_cast<uint32_t*>(st + g * 4) = (uint32_t)sw;
}

template <int W>
void run(const char* name, const float* z, float* out, uint8_t* st, int64_t n) {
    const int64_t ng = n / W;
    const int64_t grid = (ng + 127) / 128;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k<W><<<grid, 128>>>(z, out, st, ng, n);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) k<W><<<grid, 128>>>(z, out, st, ng, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-24s %.3f ms  %.1f GB/s  (%s)\n", name, ms, n * 81.0 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int64_t n = 400000000;
    float *z, *out; uint8_t* st;
    cudaMalloc(&z, 9 * n * 4); cudaMalloc(&out, 11 * n * 4); cudaMalloc(&st, n);
    cudaMemset(z, 0, 9 * n * 4);
    for (int r = 0; r < 2; ++r) {
        run<4>("128-bit (product form)", z, out, st, n);
        run<8>("256-bit", z, out, st, n);
    }
    return 0;
}
