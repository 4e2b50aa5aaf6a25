// window_core.cuh -- part of libpolsar.so (B200, sm_100a); arXiv 1807.08084.
// Layout, ownership and error conventions: include/polsar.h.  Design notes:
// DESIGN.md.  Nothing here is shared with oracle/.
//
// The search-window machinery shared by window.cu (K3 polsar_window_distance,
// K6 polsar_window_kl and the workspace queries) and nlm.cu (K4
// polsar_nlm_filter): the pair determinant and weights, the shared-memory
// records, pass 1 of the symmetric form (k_window_fwd) with its pair policies
// and both backward-sum forms, the direct and expansion forms, and the KL
// prepass.  Included once per translation unit (anonymous namespace).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "alg.cuh"

namespace polsar_impl {
namespace {

// ==================================================== K3: window distance
// K3a: per-pixel g_i = 1/(8 det Z_i) (det by Eq. 6) into the workspace.
// K3b: one CTA per TY x TX output tile; the (TY+2R) x (TX+2R) halo of Z (9
// planes, type T) and g (1 plane) is staged in shared memory once.  Each
// thread owns RB vertically adjacent output pixels of one column and walks
// the window's columns; every staged Z_j it loads is paired with all of its
// RB pixels that reach it (RB-fold reuse of each shared-memory load, RB
// independent dependency chains for the FP64 pipe).  Per pair (R-12,
// BASELINE configs[4]):
//   S = Z_i + Z_j            (9 adds; exact in fp64 for fp32 storage)
//   ds = det(S) by Eq. 6     (only a_c, b_c, c_c needed: 20 fp64 ops)
//   r = (ds g_i)(ds g_j) = D_S^2 / (D_i D_j),  D_S = det((Z_i+Z_j)/2)
//   exp(-d_ij/h) = r^(-L/(2h))   (L/(2h) = 2: 1/(r r), no transcendental)
// Rows of the window that reach all RB pixels run branch-free; the RB-1 rows
// at each vertical end take a warp-uniform branch per pixel.  Columns outside
// the image read zero-filled cells and are masked by a select.
constexpr int K3_TX = 32;  // tile width; tile height TY in {32, 16, 8} (the largest
                           // whose halo fits in shared memory); K3_RB output rows per thread

template <typename T>
__device__ __forceinline__ T det_eq6(T a, T br, T bi, T cr, T ci, T d, T er, T ei, T f) {
    T ac = FMA(d, f, -FMA(er, er, MUL(ei, ei)));
    T bcr = FMA(cr, er, FMA(ci, ei, -MUL(br, f)));
    T bci = FMA(ci, er, -FMA(cr, ei, MUL(bi, f)));
    T ccr = FMA(br, er, -FMA(bi, ei, MUL(cr, d)));
    T cci = FMA(br, ei, FMA(bi, er, -MUL(ci, d)));
    return FMA(a, ac, FMA(br, bcr, FMA(bi, bci, FMA(cr, ccr, MUL(ci, cci)))));
}

// K3a: g_i = 1 / (8 det Z_i) per slab pixel (det by Eq. 6 in T).
template <typename S, typename T, typename WT>
__global__ void __launch_bounds__(256)
k_window_prep(const S* __restrict__ z, int64_t ld, int64_t n, WT* __restrict__ g) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        T v[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) v[k] = (T)z[k * ld + p];
        T dz = det_eq6<T>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8]);
        // NaN marks a pixel that is not positive definite (or not finite): every
        // weight it enters becomes NaN, and so does W of every pixel whose
        // window holds it
        const WT gv = (WT)(T(1) / MUL(T(8), dz));
        g[p] = (dz > T(0) && gv < WT(INFINITY)) ? gv : WT(NAN);
    }
}

__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// w = r^(-alpha), alpha = L/(2h).  alpha == 2 (L = 4, h = 1): w = 1/(r r),
// no transcendental.
__device__ __forceinline__ float fast_log2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// (MUFU lg2 / ex2: absolute error ~2^-22 in log2 r, i.e. a relative error of
// about alpha * 1e-7 in w -- far inside the 2e-5 budget for the fp32 weight.)
__device__ __forceinline__ float pair_weight(float r, float alpha, bool alpha_is_2) {
    if (alpha_is_2) return fast_rcp(r * r);
    return fast_exp2(-alpha * fast_log2(r));
}
// 1/x for the fp64 weight: MUFU's ~23-bit reciprocal and two Newton steps
// (error squared each step: <= 2 ulp), against div.rn.f64's longer sequence
// with its special-case branch.  x = r^2 > 0 and finite for valid pixels; a
// NaN or 0 propagates as NaN / inf (the NaN marks of R-19 survive).
__device__ __forceinline__ double fast_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = __fma_rn(-x, y, 1.0);
    y = __fma_rn(y, e, y);
    e = __fma_rn(-x, y, 1.0);
    return __fma_rn(y, e, y);
}
__device__ __forceinline__ double pair_weight(double r, double alpha, bool alpha_is_2) {
    if (alpha_is_2) return fast_rcp(r * r);
    return exp(-alpha * log(r));
}

template <typename T, typename WT>
__device__ __forceinline__ WT pair_w(const T* zi, WT gi, const T* zj, WT gj, WT alpha, bool a2) {
    T ds = det_eq6<T>(ADD(zi[0], zj[0]), ADD(zi[1], zj[1]), ADD(zi[2], zj[2]), ADD(zi[3], zj[3]),
                      ADD(zi[4], zj[4]), ADD(zi[5], zj[5]), ADD(zi[6], zj[6]), ADD(zi[7], zj[7]),
                      ADD(zi[8], zj[8]));
    WT fds = (WT)ds;
    WT rr = (fds * gi) * (fds * gj);
    return pair_weight(rr, alpha, a2);
}

// Shared-memory halo pixel (symmetric pass 1, NLM): the 9 planes and g in one 10-slot record
// (stride 10 T: 16-byte aligned for T = double, 8-byte for float), read with
// five 2-wide loads from one address.  Record strides of 5 (double2) / 5
// (float2) bank units are odd, so a warp's loads are conflict-free.
template <typename T>
struct Vec2Of;
template <>
struct Vec2Of<double> { using type = double2; };
template <>
struct Vec2Of<float> { using type = float2; };

// g (WT) carried in the record's T slot, bit-exact.
template <typename T, typename WT>
__device__ __forceinline__ T pack_g(WT v) {
    if constexpr (sizeof(T) == sizeof(WT)) return (T)v;
    else return __longlong_as_double((long long)__float_as_uint(v));
}
template <typename T, typename WT>
__device__ __forceinline__ WT unpack_g(T v) {
    if constexpr (sizeof(T) == sizeof(WT)) return (WT)v;
    else return __uint_as_float((unsigned)__double_as_longlong(v));
}

template <typename T, typename WT>
__device__ __forceinline__ void load_rec(const T* rec, T (&zj)[9], WT& gj) {
    using V = typename Vec2Of<T>::type;
    const V* p = reinterpret_cast<const V*>(rec);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const V v = p[k];
        zj[2 * k] = v.x;
        zj[2 * k + 1] = v.y;
    }
    const V v = p[4];
    zj[8] = v.x;
    gj = unpack_g<T, WT>(v.y);
}

#ifndef POLSAR_K3_RB
#define POLSAR_K3_RB 2
#endif
template <int TY>
struct K3_RB_FOR {
    static constexpr int v = (TY >= 16) ? POLSAR_K3_RB : 4;
};

// K3b.  r = D_S^2 / (D_i D_j) with D_S = det(Z_i + Z_j)/8 = (ds g_i)(ds g_j).
template <typename S, typename T, typename WT, int K3_TY, int K3_RB>
__global__ void __launch_bounds__(K3_TX * K3_TY / K3_RB, 1)
k_window_sum(const S* __restrict__ z, int64_t ld, int64_t width, int64_t slab_rows,
             int64_t row_begin, int64_t row_end, int R, const WT* __restrict__ g, double alpha_d,
             int alpha_is_2, S* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int HW = K3_TX + 2 * R;        // halo tile width
    const int HH = K3_TY + 2 * R;        // halo tile height
    const int HP = HW * HH;              // pixels in the halo tile
    T* sz = reinterpret_cast<T*>(smem_raw);        // 9 planes of Z (type T)
    WT* sg = reinterpret_cast<WT*>(sz + 9 * HP);   // 1 plane of g

    const int64_t x0 = (int64_t)blockIdx.x * K3_TX;
    const int64_t y0 = row_begin + (int64_t)blockIdx.y * K3_TY;
    // stage the halo; cells outside the slab are zero-filled (masked later)
    for (int q = threadIdx.x; q < HP; q += blockDim.x) {
        int hy = q / HW, hx = q % HW;
        int64_t gy = y0 - R + hy, gx = x0 - R + hx;
        bool in = gy >= 0 && gy < slab_rows && gx >= 0 && gx < width;
        int64_t p = in ? gy * width + gx : 0;
#pragma unroll
        for (int k = 0; k < 9; ++k) sz[k * HP + q] = in ? (T)z[k * ld + p] : T(0);
        sg[q] = in ? g[p] : WT(0);
    }
    __syncthreads();

    const int tx = threadIdx.x % K3_TX;
    const int ty0 = (threadIdx.x / K3_TX) * K3_RB;
    const int64_t gx = x0 + tx;
    T zi[K3_RB][9];
    WT gi[K3_RB];
    double acc[K3_RB];
#pragma unroll
    for (int r = 0; r < K3_RB; ++r) {
        int q = (ty0 + r + R) * HW + (tx + R);
#pragma unroll
        for (int k = 0; k < 9; ++k) zi[r][k] = sz[k * HP + q];
        gi[r] = sg[q];
        acc[r] = 0.0;
    }
    const WT alpha = (WT)alpha_d;
    const bool a2 = alpha_is_2 != 0;
    // the CTA's window columns all lie inside the image: no column masks
    const bool interior_x = (x0 - R >= 0) && (x0 + K3_TX + R <= width);

    for (int wy = -R; wy <= R + K3_RB - 1; ++wy) {
        const int64_t gyj = y0 + ty0 + wy;
        if (gyj < 0 || gyj >= slab_rows) continue;  // warp-uniform
        const int hy = ty0 + wy + R;
        const T* rowz = sz + hy * HW + tx + R;
        const WT* rowg = sg + hy * HW + tx + R;
        WT row[K3_RB];
#pragma unroll
        for (int r = 0; r < K3_RB; ++r) row[r] = WT(0);
        if ((wy >= K3_RB - 1 - R) && (wy <= R)) {
            // this window row reaches every owned pixel: straight-line RB pairs
            if (interior_x) {
#pragma unroll 2
                for (int wx = -R; wx <= R; ++wx) {
                    T zj[9];
                    POLSAR_CHECK(hy >= 0 && hy < HH && tx + wx + R >= 0 && tx + wx + R < HW);
#pragma unroll
                    for (int k = 0; k < 9; ++k) zj[k] = rowz[k * HP + wx];
                    const WT gj = rowg[wx];
#pragma unroll
                    for (int r = 0; r < K3_RB; ++r) row[r] += pair_w<T, WT>(zi[r], gi[r], zj, gj, alpha, a2);
                }
            } else {
                for (int wx = -R; wx <= R; ++wx) {
                    T zj[9];
                    POLSAR_CHECK(hy >= 0 && hy < HH && tx + wx + R >= 0 && tx + wx + R < HW);
#pragma unroll
                    for (int k = 0; k < 9; ++k) zj[k] = rowz[k * HP + wx];
                    const WT gj = rowg[wx];
                    const bool colok = gx + wx >= 0 && gx + wx < width;
#pragma unroll
                    for (int r = 0; r < K3_RB; ++r) {
                        WT w = pair_w<T, WT>(zi[r], gi[r], zj, gj, alpha, a2);
                        row[r] += colok ? w : WT(0);
                    }
                }
            }
        } else {
            // one of the RB-1 rows at either end: only some owned pixels reach it
            for (int wx = -R; wx <= R; ++wx) {
                T zj[9];
                POLSAR_CHECK(hy >= 0 && hy < HH && tx + wx + R >= 0 && tx + wx + R < HW);
#pragma unroll
                for (int k = 0; k < 9; ++k) zj[k] = rowz[k * HP + wx];
                const WT gj = rowg[wx];
                const bool colok = interior_x || (gx + wx >= 0 && gx + wx < width);
#pragma unroll
                for (int r = 0; r < K3_RB; ++r) {
                    const int dy = wy - r;
                    if (dy >= -R && dy <= R) {  // warp-uniform
                        WT w = pair_w<T, WT>(zi[r], gi[r], zj, gj, alpha, a2);
                        row[r] += colok ? w : WT(0);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < K3_RB; ++r) acc[r] += (double)row[r];
    }
#pragma unroll
    for (int r = 0; r < K3_RB; ++r) {
        const int64_t gy = y0 + ty0 + r;
        if (gx < width && gy < row_end) out[(gy - row_begin) * width + gx] = (S)acc[r];
    }
}

template <typename S, typename T, typename WT, int TY>
int launch_window_ty(const S* z, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb,
                     int64_t re, int R, double alpha, const WT* g, S* out, size_t smem,
                     cudaStream_t s) {
    constexpr int K3_RB = K3_RB_FOR<TY>::v;
    auto kern = k_window_sum<S, T, WT, TY, K3_RB>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return fail(POLSAR_ENOTSUP, "polsar_window_distance: shared memory request too large");
    dim3 grid((unsigned)((width + K3_TX - 1) / K3_TX), (unsigned)((re - rb + TY - 1) / TY));
    kern<<<grid, K3_TX * TY / K3_RB, smem, s>>>(z, ld, width, slab_rows, rb, re, R, g, alpha,
                                                alpha == 2.0 ? 1 : 0, out);
    return launch_check("polsar_window_distance: launch failed");
}

constexpr size_t K3_SMEM_MAX = 227 * 1024;

template <typename T, typename WT>
size_t window_smem(int TY, int R) {
    return (size_t)(K3_TX + 2 * R) * (TY + 2 * R) * (9 * sizeof(T) + sizeof(WT));
}

template <typename S, typename T, typename WT>
int launch_window(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb,
                  int64_t re, int R, double looks, double h, void* ws, void* outv,
                  cudaStream_t s) {
    const S* z = (const S*)zv;
    WT* g = (WT*)ws;
    int64_t n = slab_rows * width;
    k_window_prep<S, T, WT><<<grid_for(n, 256), 256, 0, s>>>(z, ld, n, g);
    const double alpha = looks / (2.0 * h);
    S* out = (S*)outv;
    if (window_smem<T, WT>(32, R) <= K3_SMEM_MAX)
        return launch_window_ty<S, T, WT, 32>(z, ld, width, slab_rows, rb, re, R, alpha, g, out,
                                              window_smem<T, WT>(32, R), s);
    if (window_smem<T, WT>(16, R) <= K3_SMEM_MAX)
        return launch_window_ty<S, T, WT, 16>(z, ld, width, slab_rows, rb, re, R, alpha, g, out,
                                              window_smem<T, WT>(16, R), s);
    if (window_smem<T, WT>(8, R) <= K3_SMEM_MAX)
        return launch_window_ty<S, T, WT, 8>(z, ld, width, slab_rows, rb, re, R, alpha, g, out,
                                             window_smem<T, WT>(8, R), s);
    return fail(POLSAR_ENOTSUP, "polsar_window_distance: radius too large for shared memory");
}

// ------------------------------------------------------------------------
// Shared by the symmetric forms: the largest radius whose tiles fit shared
// memory (the paper's R = 11) and the KL prepass's plane count.
constexpr int V3_NP = 20;        // prepass planes per pixel (KL: Z | w Z^-1 | 0 | 0)
constexpr int V3_RMAX = 12;      // radius limit of the symmetric and tensor-core forms

// KL prepass: planes 9..17 hold w * Z^-1 from Alg. 2
// (K1's device function: cofactors, Eq. 6 det, t = 1/det, scale), plane 18
// holds 0, so the pair sum T = <X_i, Z_j> + <Z_i, X_j> = tr(Z_i^-1 Z_j) +
// tr(Z_j^-1 Z_i).
template <typename S>
__global__ void __launch_bounds__(256)
k_window_prep_kl(const S* __restrict__ z, int64_t ld, int64_t n, double* __restrict__ ws) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        H9<double> m;
        m.a = (double)z[0 * ld + p];
        m.br = (double)z[1 * ld + p];
        m.bi = (double)z[2 * ld + p];
        m.cr = (double)z[3 * ld + p];
        m.ci = (double)z[4 * ld + p];
        m.d = (double)z[5 * ld + p];
        m.er = (double)z[6 * ld + p];
        m.ei = (double)z[7 * ld + p];
        m.f = (double)z[8 * ld + p];
        double x[9], det, t;
        alg2_plain<double>(m, x, det, t);
        const int64_t P = n;
        ws[0 * P + p] = m.a;  ws[1 * P + p] = m.br; ws[2 * P + p] = m.bi;
        ws[3 * P + p] = m.cr; ws[4 * P + p] = m.ci; ws[5 * P + p] = m.d;
        ws[6 * P + p] = m.er; ws[7 * P + p] = m.ei; ws[8 * P + p] = m.f;
        const double wk[9] = {1, 2, 2, 2, 2, 1, 2, 2, 1};
        // X = NaN marks a pixel that is not positive definite (as g in k_window_prep)
        const bool ok = det > 0.0 && t < INFINITY;
#pragma unroll
        for (int k = 0; k < 9; ++k) ws[(9 + k) * P + p] = ok ? wk[k] * x[k] : NAN;
        ws[18 * P + p] = 0.0;
        ws[19 * P + p] = 0.0;
    }
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    int src_bytes = valid ? 8 : 0;  // 0: zero-fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(sa), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

// plane 19 holds g as fp64 (fp64 weights) or as fp32 bits in the low word
// Weight of a pair for the symmetric Wishart KL distance:
// T = tr(Z_i^-1 Z_j) + tr(Z_j^-1 Z_i), d = L (T/2 - 3), w = exp(-d/h);
// lk = L/h.  The subtraction is done in fp64 (T/2 ~ 3 for similar pixels).
template <typename WT>
__device__ __forceinline__ WT weight_kl(double T, WT lk);
template <>
__device__ __forceinline__ float weight_kl<float>(double T, float lk) {
    const float d = (float)__fma_rn(T, 0.5, -3.0);
    return fast_exp2(-lk * d * 1.4426950408889634f);
}
template <>
__device__ __forceinline__ double weight_kl<double>(double T, double lk) {
    return exp(-lk * __fma_rn(T, 0.5, -3.0));
}

// ------------------------------------------------------------------------
// K3 (symmetric, default for R <= V3_RMAX): d_ij = d_ji (the window is
// symmetric and det((Z_i+Z_j)/2) is), so each unordered pair is evaluated
// once.  Pass 1 (k_window_fwd) computes, for every pixel i, the weights of its
// 2R(R+1) "forward" neighbours j = i + delta (delta_y > 0, or delta_y = 0 and
// delta_x > 0) and their sum F_i.  Each weight must also reach W_j:
//  * ACC form (default for the window and KL): added to j's backward sum in
//    shared memory as an exact fixed-point integer (acc_add below); pass 2
//    (k_window_bwd_acc) adds the <= 4 tile sums of each pixel.
//  * plane form (NLM, whose gather reads the weights; POLSAR_WINDOW_PLANES=1):
//    stored at wbuf[delta][i]; pass 2 (k_window_bwd) adds, for every output
//    pixel j, W_j = 1 + F_j + sum_delta wbuf[delta][j - delta] (1068 B/pixel
//    of workspace traffic at R = 11, fp32 weights).
// d_jj = 0 contributes exactly 1.  Half the FP64 work of k_window_sum; every
// sum is exact or in a fixed order, so results are bit-reproducible and slab
// decompositions are exact.
__host__ __device__ __forceinline__ int fwd_count(int R) { return 2 * R * (R + 1); }
// Row pitch of the weight planes: width rounded up to 16 bytes, so every row
// of every plane starts 16-byte aligned (the TMA tiles of the NLM gather need
// 16-byte aligned starts: measured, tools/micro/tma1d_test.cu).
template <typename WT>
__host__ __device__ __forceinline__ int64_t weight_pitch(int64_t width) {
    constexpr int64_t a = 16 / sizeof(WT);
    return (width + a - 1) / a * a;
}
__device__ __forceinline__ int fwd_index(int dy, int dx, int R) {
    return dy == 0 ? dx - 1 : R + (dy - 1) * (2 * R + 1) + (dx + R);
}

#ifndef POLSAR_SYM_TY
#define POLSAR_SYM_TY 32
#endif
#ifndef POLSAR_SYM_RB
#define POLSAR_SYM_RB 2
#endif
#ifndef POLSAR_SYM_UNROLL
#define POLSAR_SYM_UNROLL 2
#endif
constexpr int kSymUnroll = POLSAR_SYM_UNROLL;

// Pair policies of pass 1: what a shared-memory record holds (RS slots of T)
// and how a pair weight is computed from two records.
//
// Log-det distance (R-12): 9 planes + g = 1/(8 det Z); w from Eq. 6 on
// S = Z_i + Z_j (pair_w).
template <typename S_, typename T_, typename WT_, int A2_ = -1>
struct LogDetPair {
    // A2_: 1 / 0 fix "alpha == 2" at compile time (the weight is 1/r^2, or
    // MUFU lg2/ex2); -1 reads the runtime flag a2
    using S = S_;
    using T = T_;
    using WT = WT_;
    static constexpr int RS = 10;
    struct Rec {
        T z[9];
        WT g;
    };
    const S* z;
    int64_t ld;
    const WT* g;
    WT alpha;
    bool a2;
    __device__ __forceinline__ void fill(T* rec, int64_t p, bool in) const {
#pragma unroll
        for (int k = 0; k < 9; ++k) rec[k] = in ? (T)z[k * ld + p] : T(0);
        rec[9] = pack_g<T, WT>(in ? g[p] : WT(0));
    }
    __device__ __forceinline__ static void load(const T* rec, Rec& r) { load_rec(rec, r.z, r.g); }
    // (k_window_prep's NaN mark)
    __device__ __forceinline__ static bool invalid(const Rec& r) { return !(r.g > WT(0)); }
    // weight = post(pre(i, j), i, aux(j)): pre is the FP64 part (det of
    // S = Z_i + Z_j by Eq. 6), post the fp32 weight (same arithmetic as pair_w)
#ifndef POLSAR_LOGDET_PIPELINE
#define POLSAR_LOGDET_PIPELINE 0
#endif
    static constexpr bool kPipeline = POLSAR_LOGDET_PIPELINE;  // measured: pipelining costs 4 % here
    using Q = T;
    using Aux = WT;
    __device__ __forceinline__ Q pre(const Rec& i, const Rec& j) const {
        return det_eq6<T>(ADD(i.z[0], j.z[0]), ADD(i.z[1], j.z[1]), ADD(i.z[2], j.z[2]),
                          ADD(i.z[3], j.z[3]), ADD(i.z[4], j.z[4]), ADD(i.z[5], j.z[5]),
                          ADD(i.z[6], j.z[6]), ADD(i.z[7], j.z[7]), ADD(i.z[8], j.z[8]));
    }
    __device__ __forceinline__ static Aux aux(const Rec& j) { return j.g; }
    __device__ __forceinline__ WT post(Q ds, const Rec& i, Aux gj) const {
        WT fds = (WT)ds;
        WT rr = (fds * i.g) * (fds * gj);
        return pair_weight(rr, alpha, A2_ < 0 ? a2 : A2_ == 1);
    }
    __device__ __forceinline__ WT weight(const Rec& i, const Rec& j) const {
        return post(pre(i, j), i, aux(j));
    }
};

// Symmetric Wishart KL (K6): Z and X = w * Z^-1 (Alg. 2 in k_window_prep_kl,
// w the Hermitian trace weights), T = <X_i, Z_j> + <Z_i, X_j>
// = tr(Z_i^-1 Z_j) + tr(Z_j^-1 Z_i), w = exp(-L (T/2 - 3) / h).
template <typename WT_>
struct KLPair {
    using T = double;
    using WT = WT_;
    static constexpr int RS = 18;
    struct Rec {
        double z[9];
        double x[9];
    };
    const double* ws;  // prep planes 0..8 = Z, 9..17 = X, plane stride P
    int64_t P;
    WT lk;             // L / h
    __device__ __forceinline__ void fill(double* rec, int64_t p, bool in) const {
#pragma unroll
        for (int k = 0; k < 18; ++k) rec[k] = in ? ws[k * P + p] : 0.0;
    }
    __device__ __forceinline__ static void load(const double* rec, Rec& r) {
        const double2* v = reinterpret_cast<const double2*>(rec);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            const double2 u = v[k];
            const int a = 2 * k, b = 2 * k + 1;
            (a < 9 ? r.z[a] : r.x[a - 9]) = u.x;
            (b < 9 ? r.z[b] : r.x[b - 9]) = u.y;
        }
    }
    static constexpr bool kPipeline = true;  // measured: 4.79 -> 4.43 ms on c5
    __device__ __forceinline__ static bool invalid(const Rec& r) { return r.x[0] != r.x[0]; }  // NaN mark
    using Q = double;
    using Aux = int;
    __device__ __forceinline__ Q pre(const Rec& i, const Rec& j) const {
        double A = __dmul_rn(i.x[0], j.z[0]);
        double B = __dmul_rn(i.z[0], j.x[0]);
#pragma unroll
        for (int k = 1; k < 9; ++k) {
            A = __fma_rn(i.x[k], j.z[k], A);
            B = __fma_rn(i.z[k], j.x[k], B);
        }
        return __dadd_rn(A, B);
    }
    __device__ __forceinline__ static Aux aux(const Rec&) { return 0; }
    __device__ __forceinline__ WT post(Q T, const Rec&, Aux) const { return weight_kl<WT>(T, lk); }
    __device__ __forceinline__ WT weight(const Rec& i, const Rec& j) const {
        return post(pre(i, j), i, aux(j));
    }
};

// KL with fp32 storage: Z is exact in fp32, so the record keeps X (9 fp64)
// and Z (9 fp32, widened on load): 112 bytes instead of 144 (KL's pass 1 is
// bound by shared-memory bandwidth).  Same arithmetic as KLPair.
template <typename WT_>
struct KLPairF {
    using T = double;
    using WT = WT_;
    static constexpr int RS = 14;  // 112 bytes: X0..X8 (fp64), Z0..Z8 (fp32) at byte 72, pad
    using Rec = typename KLPair<WT_>::Rec;
    const double* ws;  // prep planes 0..8 = Z, 9..17 = X, plane stride P
    int64_t P;
    WT lk;             // L / h
    __device__ __forceinline__ void fill(double* rec, int64_t p, bool in) const {
#pragma unroll
        for (int k = 0; k < 9; ++k) rec[k] = in ? ws[(9 + k) * P + p] : 0.0;
        float* zf = reinterpret_cast<float*>(rec + 9);
#pragma unroll
        for (int k = 0; k < 9; ++k) zf[k] = in ? (float)ws[k * P + p] : 0.0f;  // exact: Z came from fp32
        zf[9] = 0.0f;
    }
    __device__ __forceinline__ static void load(const double* rec, Rec& r) {
        const double2* v = reinterpret_cast<const double2*>(rec);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 u = v[k];
            r.x[2 * k] = u.x;
            r.x[2 * k + 1] = u.y;
        }
        r.x[8] = rec[8];
        const float2 a = *reinterpret_cast<const float2*>(rec + 9);          // byte 72
        const float4 b = *reinterpret_cast<const float4*>(rec + 10);         // byte 80
        const float4 c = *reinterpret_cast<const float4*>(rec + 12);         // byte 96
        r.z[0] = a.x; r.z[1] = a.y; r.z[2] = b.x; r.z[3] = b.y;
        r.z[4] = b.z; r.z[5] = b.w; r.z[6] = c.x; r.z[7] = c.y; r.z[8] = c.z;
    }
    static constexpr bool kPipeline = true;
    __device__ __forceinline__ static bool invalid(const Rec& r) { return r.x[0] != r.x[0]; }  // NaN mark
    using Q = double;
    using Aux = int;
    __device__ __forceinline__ Q pre(const Rec& i, const Rec& j) const {
        double A = __dmul_rn(i.x[0], j.z[0]);
        double B = __dmul_rn(i.z[0], j.x[0]);
#pragma unroll
        for (int k = 1; k < 9; ++k) {
            A = __fma_rn(i.x[k], j.z[k], A);
            B = __fma_rn(i.z[k], j.x[k], B);
        }
        return __dadd_rn(A, B);
    }
    __device__ __forceinline__ static Aux aux(const Rec&) { return 0; }
    __device__ __forceinline__ WT post(Q T, const Rec&, Aux) const { return weight_kl<WT>(T, lk); }
    __device__ __forceinline__ WT weight(const Rec& i, const Rec& j) const {
        return post(pre(i, j), i, aux(j));
    }
};

#ifndef POLSAR_KLF_TY
#define POLSAR_KLF_TY 24
#endif
#ifndef POLSAR_KLF_RB
#define POLSAR_KLF_RB 2
#endif

// Backward sums in shared memory (ACC forms of pass 1, window and KL): each
// pair weight w(i, j) is added to j's backward sum as the fixed-point integer
// round(w 2^44), split over two 32-bit counters (bits 22 and up, bits 0-21)
// so the native shared-memory ATOMS.ADD serves: integer addition is exact
// and associative, so the sums are bit-reproducible in any order and any
// tiling.  Per target and tile at most 2R(R+1) <= 312 weights <= 1 arrive
// (positive-definite inputs: d >= 0): the high counter stays below 2^31, and
// the low one, fed < 2^22 per add, below 2^30.1.  Bit 31 of the low counter
// is a NaN flag: a pixel marked invalid by the prepass (NaN g or X) sets it on
// its own slot and on all its forward targets, so W comes out NaN exactly on
// the pixels whose window holds it (its forward-pair weights are NaN too and
// make F NaN; the integers they add to flagged slots are discarded).
constexpr float kFix = 17592186044416.0f;  // 2^44
constexpr unsigned kBadBit = 0x80000000u;
constexpr long long kBadSum = (long long)(1ull << 63);  // a flagged tile sum in part[]
__device__ __forceinline__ long long fixed_w(float w) { return __float2ll_rn(w * kFix); }
__device__ __forceinline__ long long fixed_w(double w) { return __double2ll_rn(w * (double)kFix); }
__device__ __forceinline__ void acc_add(unsigned* ah, int hp, int q, long long v) {
    atomicAdd(ah + q, (unsigned)((unsigned long long)v >> 22));
    atomicAdd(ah + hp + q, (unsigned)(v & 0x3fffff));
}

// Pass 1, one full window row (all 2R+1 neighbours valid for every owned
// row): weights into row[] and, for owned in-image pairs, into the planes
// wp[r] (advanced by one plane per neighbour), or (ACC) into the neighbours'
// backward sums ah[qj + wx + R].
template <typename Pair, int RB, bool FULL, bool ACC>
__device__ __forceinline__ void fwd_full_row(const Pair& pr, const typename Pair::Rec (&ri)[RB],
                                             const typename Pair::T* rec, int R, int64_t gx,
                                             int64_t width, bool interior_x, const bool (&own)[RB],
                                             typename Pair::WT* (&wp)[RB], int64_t N,
                                             typename Pair::WT (&row)[RB], unsigned* ah, int hp, int qj) {
    // FULL: the CTA's whole tile is inside the image and the output rows, so
    // every pair is in-image and owned: no masks, unconditional stores
    using WT = typename Pair::WT;
#pragma unroll kSymUnroll
    for (int wx = -R; wx <= R; ++wx, rec += Pair::RS, ++qj) {
        typename Pair::Rec rj;
        Pair::load(rec, rj);
        const bool colok = FULL || interior_x || (gx + wx >= 0 && gx + wx < width);
        long long v = 0;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            WT w = pr.weight(ri[r], rj);
            if constexpr (ACC) {
                if (!FULL) w = colok ? w : WT(0);
                row[r] += w;
                if (FULL || own[r]) v += fixed_w(w);
            } else if constexpr (FULL) {
                row[r] += w;
                *wp[r] = w;
            } else {
                w = colok ? w : WT(0);
                row[r] += w;
                if (colok && own[r]) *wp[r] = w;
            }
            if constexpr (!ACC) wp[r] += N;
        }
        if constexpr (ACC) acc_add(ah, hp, qj, v);
    }
}

// The same row software-pipelined by one neighbour: the FP64 part (pre) of
// neighbour wx and the weight, sum and store (post) of wx - 1 form one basic
// block, so the scheduler overlaps them.  The first post is a no-op
// (ok = false) and the sums keep wx order, so results equal fwd_full_row's.
template <typename Pair, int RB, bool ACC>
__device__ __forceinline__ void fwd_full_row_pipelined(
    const Pair& pr, const typename Pair::Rec (&ri)[RB], const typename Pair::T* rec, int R,
    int64_t gx, int64_t width, bool interior_x, const bool (&own)[RB], typename Pair::WT* (&wp)[RB],
    int64_t N, typename Pair::WT (&row)[RB], unsigned* ah, int hp, int qj) {
    using WT = typename Pair::WT;
    typename Pair::Q qp[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        wp[r] -= N;
        qp[r] = typename Pair::Q(1);
    }
    typename Pair::Aux ap = Pair::aux(ri[0]);
    bool okp = false;
#pragma unroll kSymUnroll
    for (int wx = -R; wx <= R; ++wx, rec += Pair::RS) {
        typename Pair::Rec rj;
        Pair::load(rec, rj);
        const bool colok = interior_x || (gx + wx >= 0 && gx + wx < width);
        typename Pair::Q q[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) q[r] = pr.pre(ri[r], rj);
        long long v = 0;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            WT w = pr.post(qp[r], ri[r], ap);
            w = okp ? w : WT(0);
            row[r] += w;
            if constexpr (ACC) {
                if (own[r]) v += fixed_w(w);
            } else {
                if (okp && own[r]) *wp[r] = w;
                wp[r] += N;
            }
            qp[r] = q[r];
        }
        if constexpr (ACC) {
            if (wx > -R) acc_add(ah, hp, qj + wx + R - 1, v);  // neighbour wx - 1
        }
        ap = Pair::aux(rj);
        okp = colok;
    }
    long long v = 0;
#pragma unroll
    for (int r = 0; r < RB; ++r) {  // the last neighbour's post
        WT w = pr.post(qp[r], ri[r], ap);
        w = okp ? w : WT(0);
        row[r] += w;
        if constexpr (ACC) {
            if (own[r]) v += fixed_w(w);
        } else {
            if (okp && own[r]) *wp[r] = w;
        }
    }
    if constexpr (ACC) acc_add(ah, hp, qj + 2 * R, v);
}

// Pass 1, generic over the pair policy.  ACC: instead of storing the pair
// weights, accumulate every in-tile-halo neighbour's backward sum in shared
// memory (fixed point, acc_add) and write the tile's halo-region sums to
// part[tile][HP] (int64) at the end; pass 2 (k_window_bwd_acc) adds the <= 4
// tiles' sums of each pixel.
template <typename Pair, int TY, int RB, bool ACC = false>
__global__ void __launch_bounds__(K3_TX * TY / RB, 1)
k_window_fwd(Pair pr, int64_t width, int64_t slab_rows, int64_t row_begin, int64_t row_end, int R,
             int64_t wpitch, typename Pair::WT* __restrict__ wbuf, double* __restrict__ fbuf,
             long long* __restrict__ part) {
    using T = typename Pair::T;
    using WT = typename Pair::WT;
    using Rec = typename Pair::Rec;
    constexpr int RS = Pair::RS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int HW = K3_TX + 2 * R;   // halo columns x0-R .. x0+TX-1+R
    const int HH = TY + R;          // halo rows y0 .. y0+TY-1+R (forward only)
    const int HP = HW * HH;
    T* sz = reinterpret_cast<T*>(smem_raw);  // HP records of RS T
    const int64_t N = slab_rows * wpitch;    // weight-plane stride (row pitch wpitch >= width)

    const int64_t x0 = (int64_t)blockIdx.x * K3_TX;
    const int64_t y0 = row_begin + (int64_t)blockIdx.y * TY;
    // ACC: the backward-sum counters follow the records (high words, then low)
    unsigned* ah = reinterpret_cast<unsigned*>(sz + (size_t)RS * HP);
    for (int q = threadIdx.x; q < HP; q += blockDim.x) {
        int hy = q / HW, hx = q % HW;
        int64_t gy = y0 + hy, gx = x0 - R + hx;
        bool in = gy < slab_rows && gx >= 0 && gx < width;
        pr.fill(sz + RS * q, in ? gy * width + gx : 0, in);
        if constexpr (ACC) {
            ah[q] = 0u;
            ah[HP + q] = 0u;
        }
    }
    __syncthreads();

    const int tx = threadIdx.x % K3_TX;
    const int ty0 = (threadIdx.x / K3_TX) * RB;
    const int64_t gx = x0 + tx;
    Rec ri[RB];
    double acc[RB];
    bool own[RB];
    int64_t pi[RB];  // weight-plane index of the owned pixel (F is indexed gy * width + gx)
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int64_t gy = y0 + ty0 + r;
        own[r] = gx < width && gy < row_end;
        pi[r] = gy * wpitch + gx;
        Pair::load(sz + RS * ((ty0 + r) * HW + (tx + R)), ri[r]);
        acc[r] = 0.0;
    }
    const bool interior_x = (x0 - R >= 0) && (x0 + K3_TX + R <= width);
    const bool full = interior_x && y0 + TY <= row_end;  // CTA-uniform
    if constexpr (ACC) {
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            if (own[r] && Pair::invalid(ri[r])) {  // rare: flag the pixel and its forward targets
                const int q0 = (ty0 + r) * HW + (tx + R);
                atomicOr(ah + HP + q0, kBadBit);
                for (int dy = 0; dy <= R; ++dy)
                    for (int dx = (dy == 0 ? 1 : -R); dx <= R; ++dx)
                        atomicOr(ah + HP + q0 + dy * HW + dx, kBadBit);
            }
        }
    }

    // window rows wy: the full rows RB..R (every owned pixel at dy = wy - r in
    // [1, R]) in loops of their own (no per-row branch between the full and the
    // edge forms; measured on the tensor-core pass 1), the edge rows around them
    auto full_row = [&](int wy, auto fullc) {
        const int hy = ty0 + wy;
        const T* rec = sz + RS * (hy * HW + tx);  // neighbour wx = -R
        WT row[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) row[r] = WT(0);
        // wp[r] walks the weight planes delta = (wy - r, wx), consecutive in wx.
        WT* wp[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) wp[r] = wbuf + (int64_t)fwd_index(wy - r, -R, R) * N + pi[r];
        POLSAR_CHECK(hy >= 0 && hy < HH && tx + 2 * R < HW);  // records wx = -R..R
        const int qj = hy * HW + tx;  // backward-sum slot of neighbour wx = -R
        if constexpr (Pair::kPipeline)
            fwd_full_row_pipelined<Pair, RB, ACC>(pr, ri, rec, R, gx, width, interior_x, own, wp, N, row, ah, HP,
                                                  qj);
        else
            fwd_full_row<Pair, RB, decltype(fullc)::value, ACC>(pr, ri, rec, R, gx, width, interior_x, own, wp, N,
                                                                 row, ah, HP, qj);
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[r] += (double)row[r];
    };
    auto edge_row = [&](int wy) {
        const int hy = ty0 + wy;
        const T* rec = sz + RS * (hy * HW + tx);  // neighbour wx = -R
        WT row[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) row[r] = WT(0);
        for (int wx = -R; wx <= R; ++wx, rec += RS) {
            POLSAR_CHECK(hy >= 0 && hy < HH && tx + wx + R >= 0 && tx + wx + R < HW);
            Rec rj;
            Pair::load(rec, rj);
            const bool colok = interior_x || (gx + wx >= 0 && gx + wx < width);
            long long v = 0;
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const int dy = wy - r;
                if (dy >= 0 && dy <= R && (dy > 0 || wx > 0)) {  // warp-uniform
                    WT w = pr.weight(ri[r], rj);
                    w = colok ? w : WT(0);
                    row[r] += w;
                    if constexpr (ACC) {
                        if (own[r]) v += fixed_w(w);
                    } else {
                        if (colok && own[r]) wbuf[(int64_t)fwd_index(dy, wx, R) * N + pi[r]] = w;
                    }
                }
            }
            if constexpr (ACC) acc_add(ah, HP, hy * HW + tx + wx + R, v);
        }
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[r] += (double)row[r];
    };
    // (rows past the slab end are skipped: warp-uniform)
    const int wmax = (int)(slab_rows - y0 - ty0 - 1 < R + RB - 1 ? slab_rows - y0 - ty0 - 1 : R + RB - 1);
    for (int wy = 0; wy < RB && wy <= wmax; ++wy) edge_row(wy);
    const int wf = R < wmax ? R : wmax;
    if (full) {
        for (int wy = RB; wy <= wf; ++wy) full_row(wy, std::true_type{});
    } else {
        for (int wy = RB; wy <= wf; ++wy) full_row(wy, std::false_type{});
    }
    for (int wy = R + 1 > RB ? R + 1 : RB; wy <= wmax; ++wy) edge_row(wy);
#pragma unroll
    for (int r = 0; r < RB; ++r)
        if (gx < width && y0 + ty0 + r < row_end) fbuf[(y0 + ty0 + r) * width + gx] = acc[r];
    if constexpr (ACC) {
        __syncthreads();
        long long* dst = part + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * HP;
        for (int q = threadIdx.x; q < HP; q += blockDim.x) {
            const unsigned lo = ah[HP + q];
            dst[q] = (lo & kBadBit) ? kBadSum : (long long)(((unsigned long long)ah[q] << 22) + lo);
        }
    }
}

// Pass 2 of the ACC forms: W_j = 1 + F_j + 2^-44 (sum of the backward sums of
// the <= 4 pass-1 tiles whose halo region holds j; integer, exact).  Tile
// (bx, by) covers rows p0 + by TY .. + TY + R - 1 and columns 32 bx - R ..
// 32 bx + 31 + R of its halo region.
template <typename S>
__global__ void __launch_bounds__(256)
k_window_bwd_acc(const long long* __restrict__ part, const double* __restrict__ fbuf, int64_t width,
                 int64_t row_begin, int64_t row_end, int64_t p0, int R, int TY, int nbx, int nby,
                 S* __restrict__ out) {
    // a 2D grid (columns x rows, rows grid-strided): no 64-bit division per pixel
    const int HW = K3_TX + 2 * R;
    const int HP = HW * (TY + R);
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= width) return;
    // bx: 32 bx - R <= x < 32 bx + 32 + R
    const int bx_hi = (int)((x + R) / K3_TX < nbx - 1 ? (x + R) / K3_TX : nbx - 1);
    const int bx_lo = (int)(x - K3_TX - R + 1 > 0 ? (x - K3_TX - R + 1 + K3_TX - 1) / K3_TX : 0);
    for (int64_t y = row_begin + blockIdx.y; y < row_end; y += gridDim.y) {
        const int64_t yr = y - p0;  // >= 0
        // by: p0 + by TY <= y < p0 + by TY + TY + R
        const int64_t by_hi = yr / TY;
        const int64_t by_lo = yr - TY - R + 1 > 0 ? (yr - TY - R + 1 + TY - 1) / TY : 0;
        long long sum = 0;
        bool bad = false;
        for (int64_t by = by_lo; by <= by_hi && by < nby; ++by)
            for (int bx = bx_lo; bx <= bx_hi; ++bx) {
                const int64_t hy = yr - by * TY, hx = x - K3_TX * bx + R;
                POLSAR_CHECK(hy >= 0 && hy < TY + R && hx >= 0 && hx < HW);
                const long long t = part[(by * nbx + bx) * HP + hy * HW + hx];
                bad = bad || t == kBadSum;
                sum += t;
            }
        const double wb = bad ? __longlong_as_double(0x7ff8000000000000ll) : (double)sum * (1.0 / (double)kFix);
        out[(y - row_begin) * width + x] = (S)__dadd_rn(__dadd_rn(1.0, fbuf[y * width + x]), wb);
    }
}

// Pass 2: W_j = 1 + F_j + sum over backward neighbours, one thread per pixel.
// Each (delta_y) row of weights is summed in WT, then added in double.  RC > 0
// fixes R at compile time (the paper's R = 11), so a row's 2R+1 independent
// loads are all in flight at once.
template <typename S, typename WT, int RC>
__global__ void __launch_bounds__(256)
k_window_bwd(const WT* __restrict__ wbuf, const double* __restrict__ fbuf, int64_t width,
             int64_t wpitch, int64_t slab_rows, int64_t row_begin, int64_t row_end, int R_rt,
             S* __restrict__ out) {
    const int R = RC > 0 ? RC : R_rt;
    const int64_t N = slab_rows * wpitch;  // weight-plane stride
    const int64_t m = (row_end - row_begin) * width;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = row_begin + q / width, x = q % width;
        const int64_t p = y * width + x;
        double acc = 1.0 + fbuf[p];
        const bool inx = x - R >= 0 && x + R < width;
        for (int dy = 0; dy <= R; ++dy) {
            if (y - dy < 0) break;
            const int dx0 = dy == 0 ? 1 : -R;
            const WT* base = wbuf + (int64_t)fwd_index(dy, dx0, R) * N + (y - dy) * wpitch + x - dx0;
            WT rowp = WT(0);
            if (inx) {
                if (RC > 0 && dy > 0) {
#pragma unroll
                    for (int k = 0; k < 2 * RC + 1; ++k) rowp += base[(int64_t)k * (N - 1)];
                } else {
                    for (int dx = dx0; dx <= R; ++dx) rowp += base[(int64_t)(dx - dx0) * (N - 1)];
                }
            } else {
                for (int dx = dx0; dx <= R; ++dx)
                    if (x - dx >= 0 && x - dx < width) rowp += base[(int64_t)(dx - dx0) * (N - 1)];
            }
            acc += (double)rowp;
        }
        out[q] = (S)acc;
    }
}

template <typename Pair>
size_t window_fwd_smem(int TY, int R) {
    return (size_t)(K3_TX + 2 * R) * (TY + R) * Pair::RS * sizeof(typename Pair::T);
}

// Launch pass 1 over rows [p0, re) (p0 = max(0, rb - R): the R rows above the
// output rows hold the forward pairs that are their backward pairs).
// Pass-1 tile grid over rows [p0, re): (nbx, nby) and the halo-region size
// HP of a tile (also the ACC forms' backward-sum slots per tile).
struct FwdGrid {
    int64_t p0;
    int nbx, nby, HP;
};
inline FwdGrid fwd_grid(int64_t width, int64_t rb, int64_t re, int R, int TY) {
    FwdGrid g;
    g.p0 = rb - R > 0 ? rb - R : 0;
    g.nbx = (int)((width + K3_TX - 1) / K3_TX);
    g.nby = (int)((re - g.p0 + TY - 1) / TY);
    g.HP = (K3_TX + 2 * R) * (TY + R);
    return g;
}

template <typename Pair, int TY, int RB, bool ACC = false>
int launch_fwd(const Pair& pr, int64_t width, int64_t slab_rows, int64_t rb, int64_t re, int R,
               typename Pair::WT* wbuf, double* fbuf, cudaStream_t s, const char* who,
               long long* part = nullptr) {
    const FwdGrid fg = fwd_grid(width, rb, re, R, TY);
    const size_t smem = window_fwd_smem<Pair>(TY, R) + (ACC ? 2 * sizeof(unsigned) * (size_t)fg.HP : 0);
    auto kern = k_window_fwd<Pair, TY, RB, ACC>;
    if (smem > K3_SMEM_MAX ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return fail(POLSAR_ENOTSUP, who);
    dim3 grid((unsigned)fg.nbx, (unsigned)fg.nby);
    kern<<<grid, K3_TX * TY / RB, smem, s>>>(pr, width, slab_rows, fg.p0, re, R, weight_pitch<typename Pair::WT>(width),
                                             wbuf, fbuf, part);
    return POLSAR_OK;
}

// shared memory of pass 1 in the ACC form (records + two counters per slot)
template <typename Pair>
size_t acc_fwd_smem(int TY, int R) {
    return window_fwd_smem<Pair>(TY, R) + 2 * sizeof(unsigned) * (size_t)(K3_TX + 2 * R) * (TY + R);
}

template <typename S>
void launch_bwd_acc(const long long* part, const double* fbuf, int64_t width, int64_t rb, int64_t re,
                    int R, int TY, void* outv, cudaStream_t s) {
    const FwdGrid fg = fwd_grid(width, rb, re, R, TY);
    const int64_t rows = re - rb;
    if (rows <= 0 || width <= 0) return;
    dim3 grid((unsigned)((width + 255) / 256), (unsigned)(rows < 65535 ? rows : 65535));
    k_window_bwd_acc<S><<<grid, 256, 0, s>>>(part, fbuf, width, rb, re, fg.p0, R, TY, fg.nbx, fg.nby, (S*)outv);
}

// workspace of the ACC forms: the prepass planes (pre_bytes) | F | the tiles'
// backward sums (int64, HP per tile, over the whole slab's row range)
inline size_t acc_sym_bytes(size_t pre_bytes, int64_t slab_rows, int64_t width, int R, int TY) {
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const FwdGrid fg = fwd_grid(width, 0, slab_rows, R, TY);
    return up(pre_bytes) + up((size_t)slab_rows * width * sizeof(double)) +
           up((size_t)fg.nbx * fg.nby * fg.HP * sizeof(long long));
}

// Compile-time A/B switch (tools/build_variant.sh -DPOLSAR_WINDOW_PLANES=1;
// the product never reads the environment): route the window sums through
// the weight-plane form even where the shared-memory backward sums fit.
#ifndef POLSAR_WINDOW_PLANES
#define POLSAR_WINDOW_PLANES 0
#endif
constexpr bool window_planes() { return POLSAR_WINDOW_PLANES != 0; }

template <typename S, typename WT>
void launch_bwd(const WT* wbuf, const double* fbuf, int64_t width, int64_t slab_rows, int64_t rb,
                int64_t re, int R, void* outv, cudaStream_t s) {
    if (R == 11)
        k_window_bwd<S, WT, 11><<<grid_for((re - rb) * width, 256), 256, 0, s>>>(
            wbuf, fbuf, width, weight_pitch<WT>(width), slab_rows, rb, re, R, (S*)outv);
    else
        k_window_bwd<S, WT, 0><<<grid_for((re - rb) * width, 256), 256, 0, s>>>(
            wbuf, fbuf, width, weight_pitch<WT>(width), slab_rows, rb, re, R, (S*)outv);
}

// workspace: g (N x WT) | F (N x double) | wbuf (fwd_count(R) weight planes
// of slab_rows x weight_pitch(width) WT; see weight_pitch)
template <typename WT>
size_t window_sym_bytes(int64_t slab_rows, int64_t width, int R) {
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const int64_t n = slab_rows * width;
    return up(n * sizeof(WT)) + up(n * sizeof(double)) +
           up((size_t)fwd_count(R) * slab_rows * weight_pitch<WT>(width) * sizeof(WT));
}

template <typename S, typename T, typename WT>
int launch_window_sym(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb,
                      int64_t re, int R, double looks, double h, void* wsv, void* outv,
                      cudaStream_t s) {
    const S* z = (const S*)zv;
    const int64_t n = slab_rows * width;
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    unsigned char* ws = (unsigned char*)wsv;
    WT* g = (WT*)ws;
    double* fbuf = (double*)(ws + up(n * sizeof(WT)));
    WT* wbuf = (WT*)(ws + up(n * sizeof(WT)) + up(n * sizeof(double)));
    k_window_prep<S, T, WT><<<grid_for(n, 256), 256, 0, s>>>(z, ld, n, g);
    const double alpha = looks / (2.0 * h);
    const char* who = "polsar_window_distance: shared memory request too large";
    if (!window_planes() && acc_fwd_smem<LogDetPair<S, T, WT, 1>>(POLSAR_SYM_TY, R) <= K3_SMEM_MAX) {
        long long* part = (long long*)wbuf;  // (same offset: g | F | tile sums)
        int rc = alpha == 2.0
                     ? launch_fwd<LogDetPair<S, T, WT, 1>, POLSAR_SYM_TY, POLSAR_SYM_RB, true>(
                           LogDetPair<S, T, WT, 1>{z, ld, g, (WT)alpha, true}, width, slab_rows, rb, re, R,
                           nullptr, fbuf, s, who, part)
                     : launch_fwd<LogDetPair<S, T, WT, 0>, POLSAR_SYM_TY, POLSAR_SYM_RB, true>(
                           LogDetPair<S, T, WT, 0>{z, ld, g, (WT)alpha, false}, width, slab_rows, rb, re, R,
                           nullptr, fbuf, s, who, part);
        if (rc != POLSAR_OK) return rc;
        launch_bwd_acc<S>(part, fbuf, width, rb, re, R, POLSAR_SYM_TY, outv, s);
        return launch_check("polsar_window_distance: launch failed");
    }
    int rc = alpha == 2.0
                 ? launch_fwd<LogDetPair<S, T, WT, 1>, POLSAR_SYM_TY, POLSAR_SYM_RB>(
                       LogDetPair<S, T, WT, 1>{z, ld, g, (WT)alpha, true}, width, slab_rows, rb, re, R,
                       wbuf, fbuf, s, who)
                 : launch_fwd<LogDetPair<S, T, WT, 0>, POLSAR_SYM_TY, POLSAR_SYM_RB>(
                       LogDetPair<S, T, WT, 0>{z, ld, g, (WT)alpha, false}, width, slab_rows, rb, re, R,
                       wbuf, fbuf, s, who);
    if (rc != POLSAR_OK) return rc;
    launch_bwd<S, WT>(wbuf, fbuf, width, slab_rows, rb, re, R, outv, s);
    return launch_check("polsar_window_distance: launch failed");
}

// K6, symmetric form: the KL prepass planes | F | weight planes.
template <typename WT>
size_t kl_sym_bytes(int64_t slab_rows, int64_t width, int R) {
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const int64_t n = slab_rows * width;
    return up((size_t)n * V3_NP * sizeof(double)) + up(n * sizeof(double)) +
           up((size_t)fwd_count(R) * slab_rows * weight_pitch<WT>(width) * sizeof(WT));
}

template <typename S, typename WT>
int launch_window_kl_sym(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb,
                         int64_t re, int R, double looks, double h, void* wsv, void* outv,
                         cudaStream_t s) {
    const int64_t n = slab_rows * width;
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    unsigned char* ws = (unsigned char*)wsv;
    double* prep = (double*)ws;
    double* fbuf = (double*)(ws + up((size_t)n * V3_NP * sizeof(double)));
    WT* wbuf = (WT*)(ws + up((size_t)n * V3_NP * sizeof(double)) + up(n * sizeof(double)));
    k_window_prep_kl<S><<<grid_for(n, 256), 256, 0, s>>>((const S*)zv, ld, n, prep);
    KLPair<WT> pr{prep, n, (WT)(looks / h)};
    if constexpr (sizeof(S) == 4) {  // fp32 storage: the 112-byte records
        constexpr int TYF = POLSAR_KLF_TY;
        KLPairF<WT> pf{prep, n, (WT)(looks / h)};
        if (!window_planes() && acc_fwd_smem<KLPairF<WT>>(TYF, R) <= K3_SMEM_MAX) {
            long long* part = (long long*)wbuf;
            int rc = launch_fwd<KLPairF<WT>, TYF, POLSAR_KLF_RB, true>(pf, width, slab_rows, rb, re, R, nullptr, fbuf, s,
                                                            "polsar_window_kl: shared memory request too large",
                                                            part);
            if (rc != POLSAR_OK) return rc;
            launch_bwd_acc<S>(part, fbuf, width, rb, re, R, TYF, outv, s);
            return launch_check("polsar_window_kl: launch failed");
        }
    }
    // (KL at R = 12: records + counters exceed shared memory; the plane form serves)
    if (!window_planes() && acc_fwd_smem<KLPair<WT>>(16, R) <= K3_SMEM_MAX) {
        long long* part = (long long*)wbuf;
        int rc = launch_fwd<KLPair<WT>, 16, 2, true>(pr, width, slab_rows, rb, re, R, nullptr, fbuf, s,
                                                      "polsar_window_kl: shared memory request too large", part);
        if (rc != POLSAR_OK) return rc;
        launch_bwd_acc<S>(part, fbuf, width, rb, re, R, 16, outv, s);
        return launch_check("polsar_window_kl: launch failed");
    }
    int rc = launch_fwd<KLPair<WT>, 16, 2>(pr, width, slab_rows, rb, re, R, wbuf, fbuf, s,
                                            "polsar_window_kl: shared memory request too large");
    if (rc != POLSAR_OK) return rc;
    launch_bwd<S, WT>(wbuf, fbuf, width, slab_rows, rb, re, R, outv, s);
    return launch_check("polsar_window_kl: launch failed");
}

// NLM form: symmetric (pass 1 + gather, the product for 1 <= R <= V3_RMAX) or
// the direct form (always for R = 0 and R > V3_RMAX; compile-time A/B switch
// -DPOLSAR_NLM_DIRECT=1 for every radius).
#ifndef POLSAR_NLM_DIRECT
#define POLSAR_NLM_DIRECT 0
#endif
constexpr bool nlm_direct() { return POLSAR_NLM_DIRECT != 0; }

// The NLM gather's CTA width (threads = TMA tile length); here because the
// workspace query applies the gather's dispatch conditions.
constexpr int NLM_TX = 128;

// Workspace of launch_window_sym / launch_window_kl_sym for (dtype, R): the
// same form choice those launchers make.
template <typename S, typename T, typename WT>
size_t window_sym_need_t(int64_t slab_rows, int64_t width, int R) {
    if (!window_planes() && acc_fwd_smem<LogDetPair<S, T, WT, 1>>(POLSAR_SYM_TY, R) <= K3_SMEM_MAX)
        return acc_sym_bytes((size_t)slab_rows * width * sizeof(WT), slab_rows, width, R, POLSAR_SYM_TY);
    return window_sym_bytes<WT>(slab_rows, width, R);
}
inline size_t window_sym_need(int dtype, int64_t slab_rows, int64_t width, int R) {
    switch (dtype) {
        case POLSAR_F32: return window_sym_need_t<float, double, float>(slab_rows, width, R);
        case POLSAR_F32_PLAIN: return window_sym_need_t<float, float, float>(slab_rows, width, R);
        default: return window_sym_need_t<double, double, double>(slab_rows, width, R);
    }
}
inline size_t kl_sym_need(int dtype, int64_t slab_rows, int64_t width, int R) {
    const size_t pre = (size_t)slab_rows * width * V3_NP * sizeof(double);
    if (dtype == POLSAR_F32) {
        if (!window_planes() && acc_fwd_smem<KLPairF<float>>(POLSAR_KLF_TY, R) <= K3_SMEM_MAX)
            return acc_sym_bytes(pre, slab_rows, width, R, POLSAR_KLF_TY);
        if (!window_planes() && acc_fwd_smem<KLPair<float>>(16, R) <= K3_SMEM_MAX)
            return acc_sym_bytes(pre, slab_rows, width, R, 16);
        return kl_sym_bytes<float>(slab_rows, width, R);
    }
    if (!window_planes() && acc_fwd_smem<KLPair<double>>(16, R) <= K3_SMEM_MAX)
        return acc_sym_bytes(pre, slab_rows, width, R, 16);
    return kl_sym_bytes<double>(slab_rows, width, R);
}

// NLM bands.  The symmetric NLM keeps every forward weight of its slab in
// weight planes (2R(R+1) values per pixel: 1.07 KB at R = 11 in fp32), so
// polsar_nlm_filter walks the output rows in bands of at most NLM_BAND rows,
// each band a sub-slab with its own R-row halos (the slab decomposition is
// bit-exact): the workspace covers one band's sub-slab, not
// the image -- ~2.3 GB at a 2048-pixel width, ~46 GB for a 40000-pixel-wide
// UAVSAR image of any height -- at the cost of recomputing R halo rows of
// forward weights per band (1 % at R = 11) and one launch ramp per band.
#ifndef POLSAR_NLM_BAND
#define POLSAR_NLM_BAND 1024
#endif
constexpr int64_t NLM_BAND = POLSAR_NLM_BAND;
inline bool nlm_sym_ok(int R) { return R >= 1 && R <= V3_RMAX && !nlm_direct(); }
inline int64_t nlm_band_slab_rows(int64_t slab_rows, int R) {
    const int64_t b = NLM_BAND + 2 * (int64_t)R;
    return slab_rows < b ? slab_rows : b;
}


}  // namespace
}  // namespace polsar_impl
