// polsar.cu -- B200 (sm_100a) kernels and C-ABI for arXiv 1807.08084:
// batched inverse + determinant of 3x3 Hermitian PD PolSAR matrices.
//
//   K1  polsar_inv_det           Alg. 2, HBM-streaming
//   K2  polsar_inv_det_cholesky  Alg. 1, l21 corrected
//   K3  polsar_window_distance   23x23 search-window log-det distance sum
//   R1  polsar_checksum          order-independent output hash + status counts
//   E2E polsar_inv_det_host      chunked H2D / kernel / D2H pipeline
//
// Layout, ownership and error conventions: include/polsar.h.  Design and
// roofline notes: DESIGN.md.  Nothing here is shared with oracle/.
//
// Bit-stability: every floating-point operation of the per-matrix device
// functions is an explicit round-to-nearest intrinsic (__fma_rn, __dmul_rn,
// __dadd_rn, ...), so ptxas cannot contract or reassociate differently in the
// vector body and the scalar tail: both yield identical bits.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <type_traits>

#include "../../include/polsar.h"

namespace {

// ------------------------------------------------------------------ errors
thread_local const char* g_last_error = "";

int fail(int code, const char* msg) {
    g_last_error = msg;
    return code;
}

int launch_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_last_error = what;
        return POLSAR_ECUDA;
    }
    g_last_error = "";
    return POLSAR_OK;
}

// ----------------------------------------------------- rounding intrinsics
// Overloads so one template body serves fp32 and fp64 arithmetic.
__device__ __forceinline__ double MUL(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float MUL(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double ADD(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float ADD(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double SUB(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float SUB(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double FMA(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float FMA(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double RCP(double a) { return __drcp_rn(a); }
__device__ __forceinline__ float RCP(float a) { return __frcp_rn(a); }
__device__ __forceinline__ double SQRT(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float SQRT(float a) { return __fsqrt_rn(a); }

// ------------------------------------------------------ streaming HBM I/O
// Plain 16-byte global loads and stores (LDG.E.128 / STG.E.128).  Measured
// on B200 at c3 size (tools/micro/k1_tune.cu): the default cache policy beats
// ld.global.nc.L1::no_allocate + st.global.cs by ~5 % for this 9-in / 11-out
// stream, reaching 103 % of the driver's copy peak with one 16-B vector per
// plane per thread and 128-thread CTAs over the whole batch.
__device__ __forceinline__ float4 ld_stream(const float4* p) { return *p; }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return *p; }
__device__ __forceinline__ float ld_stream(const float* p) { return *p; }
__device__ __forceinline__ double ld_stream(const double* p) { return *p; }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { *p = v; }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { *p = v; }
__device__ __forceinline__ void st_stream(float* p, float v) { *p = v; }
__device__ __forceinline__ void st_stream(double* p, double v) { *p = v; }

// ------------------------------------------------------------ matrix types
template <typename T>
struct H9 {  // packed Hermitian
    T a, br, bi, cr, ci, d, er, ei, f;
};

template <typename T>
struct R11 {  // 9 inverse components, det, det^-1, status
    T v[11];
    uint8_t status;
};

// tau * a*d*f, tau = 16 u_in (R-5)
template <typename S>
struct Tau;
template <>
struct Tau<float> {
    static constexpr double v = 16.0 * 5.9604644775390625e-08;  // 16 * 2^-24
};
template <>
struct Tau<double> {
    static constexpr double v = 16.0 * 1.1102230246251565e-16;  // 16 * 2^-53
};

template <typename T>
__device__ __forceinline__ bool finite_pos(T x) {
    return x > T(0) && x < T(INFINITY);
}

// ====================================================== Alg. 2 (proposed)
// PAPER.md:480-545.  Step 1 cofactors (495-503, Eq. 3), step 2 determinant
// from real parts only (505-517, Eq. 6), step 3 t = 1/det (519-520), step 4
// scale the six entries by t (523-528).  Arithmetic type T, one rounding per
// operation, FMA where the hardware fuses.
template <typename T>
__device__ __forceinline__ void alg2_plain(const H9<T>& m, T* o, T& det, T& t) {
    // step 1: cofactors (stored in the output slots, as Alg. 2 does)
    T ai = FMA(m.d, m.f, -FMA(m.er, m.er, MUL(m.ei, m.ei)));       // d f - |e|^2
    T bir = FMA(m.cr, m.er, FMA(m.ci, m.ei, -MUL(m.br, m.f)));      // Re(c conj e - b f)
    T bii = FMA(m.ci, m.er, -FMA(m.cr, m.ei, MUL(m.bi, m.f)));      // Im(c conj e - b f)
    T cir = FMA(m.br, m.er, -FMA(m.bi, m.ei, MUL(m.cr, m.d)));      // Re(b e - c d)
    T cii = FMA(m.br, m.ei, FMA(m.bi, m.er, -MUL(m.ci, m.d)));      // Im(b e - c d)
    T di = FMA(m.a, m.f, -FMA(m.cr, m.cr, MUL(m.ci, m.ci)));        // a f - |c|^2
    T eir = FMA(m.cr, m.br, FMA(m.ci, m.bi, -MUL(m.a, m.er)));      // Re(c conj b - a e)
    T eii = FMA(m.ci, m.br, -FMA(m.cr, m.bi, MUL(m.a, m.ei)));      // Im(c conj b - a e)
    T fi = FMA(m.a, m.d, -FMA(m.br, m.br, MUL(m.bi, m.bi)));        // a d - |b|^2
    // step 2: det = a a_i + Re b Re b_i + Im b Im b_i + Re c Re c_i + Im c Im c_i
    det = FMA(m.a, ai, FMA(m.br, bir, FMA(m.bi, bii, FMA(m.cr, cir, MUL(m.ci, cii)))));
    // step 3
    t = RCP(det);
    // step 4
    o[0] = MUL(t, ai);
    o[1] = MUL(t, bir);
    o[2] = MUL(t, bii);
    o[3] = MUL(t, cir);
    o[4] = MUL(t, cii);
    o[5] = MUL(t, di);
    o[6] = MUL(t, eir);
    o[7] = MUL(t, eii);
    o[8] = MUL(t, fi);
}

// ---- error-free transformations (fp64) for the accurate Alg. 2 (R-16)
struct dd {
    double hi, lo;
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
    s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// x1 y1 + x2 y2 + x3 y3 as an unevaluated sum hi + lo (Dot2 of Ogita, Rump &
// Oishi 2005 with FMA two-products): |hi + lo - exact| <= ~3u^2 sum|x y|.
__device__ __forceinline__ dd dot3(double x1, double y1, double x2, double y2, double x3,
                                   double y3) {
    double p1 = __dmul_rn(x1, y1), e1 = __fma_rn(x1, y1, -p1);
    double p2 = __dmul_rn(x2, y2), e2 = __fma_rn(x2, y2, -p2);
    double p3 = __dmul_rn(x3, y3), e3 = __fma_rn(x3, y3, -p3);
    double s, t1, s2, t2;
    two_sum(p1, p2, s, t1);
    two_sum(s, p3, s2, t2);
    double lo = __dadd_rn(__dadd_rn(e1, e2), __dadd_rn(e3, __dadd_rn(t1, t2)));
    dd r;
    two_sum(s2, lo, r.hi, r.lo);
    return r;
}

// x1 y1 + x2 y2 + x3 y3 rounded to ~2u of the exact value (no low part):
// exact products of the first two terms, an exact sum of their high parts,
// the third product fused exactly into one rounding, then the corrections.
__device__ __forceinline__ double dot3_hi(double x1, double y1, double x2, double y2, double x3,
                                          double y3) {
    double p1 = __dmul_rn(x1, y1), e1 = __fma_rn(x1, y1, -p1);
    double p2 = __dmul_rn(x2, y2), e2 = __fma_rn(x2, y2, -p2);
    double s, t;
    two_sum(p1, p2, s, t);
    double r = __fma_rn(x3, y3, s);
    return __dadd_rn(r, __dadd_rn(__dadd_rn(e1, e2), t));
}

// Alg. 2 with the five cofactors that enter Eq. 6 carried as hi + lo, the
// other four to ~2u (dot3_hi), and the step-2 determinant summed with Dot2
// over (x_k, hi_k) plus the x_k lo_k terms: det and every inverse entry come
// out within a few ulp, independent of the cancellation (the plain form loses
// ~kappa^2 u for matrices with one dominant eigenvalue).
__device__ __forceinline__ void alg2_accurate(const H9<double>& m, double* o, double& det,
                                              double& t) {
    // step 1 (Eq. 3), each cofactor as a 3-term dot product
    dd ai = dot3(m.d, m.f, -m.er, m.er, -m.ei, m.ei);
    dd bir = dot3(m.cr, m.er, m.ci, m.ei, -m.br, m.f);
    dd bii = dot3(m.ci, m.er, -m.cr, m.ei, -m.bi, m.f);
    dd cir = dot3(m.br, m.er, -m.bi, m.ei, -m.cr, m.d);
    dd cii = dot3(m.br, m.ei, m.bi, m.er, -m.ci, m.d);
    // d_c, e_c, f_c do not enter the determinant: the high part suffices
    const double di = dot3_hi(-m.cr, m.cr, -m.ci, m.ci, m.a, m.f);
    const double eir = dot3_hi(m.cr, m.br, m.ci, m.bi, -m.a, m.er);
    const double eii = dot3_hi(m.ci, m.br, -m.cr, m.bi, -m.a, m.ei);
    const double fi = dot3_hi(-m.br, m.br, -m.bi, m.bi, m.a, m.d);
    // step 2 (Eq. 6): det = sum_k x_k (hi_k + lo_k), compensated
    double p0 = __dmul_rn(m.a, ai.hi), q0 = __fma_rn(m.a, ai.hi, -p0);
    double p1 = __dmul_rn(m.br, bir.hi), q1 = __fma_rn(m.br, bir.hi, -p1);
    double p2 = __dmul_rn(m.bi, bii.hi), q2 = __fma_rn(m.bi, bii.hi, -p2);
    double p3 = __dmul_rn(m.cr, cir.hi), q3 = __fma_rn(m.cr, cir.hi, -p3);
    double p4 = __dmul_rn(m.ci, cii.hi), q4 = __fma_rn(m.ci, cii.hi, -p4);
    double s, r1, r2, r3, r4;
    two_sum(p0, p1, s, r1);
    two_sum(s, p2, s, r2);
    two_sum(s, p3, s, r3);
    two_sum(s, p4, s, r4);
    double err = __dadd_rn(__dadd_rn(__dadd_rn(q0, q1), __dadd_rn(q2, q3)),
                           __dadd_rn(q4, __dadd_rn(__dadd_rn(r1, r2), __dadd_rn(r3, r4))));
    err = __fma_rn(m.a, ai.lo, err);
    err = __fma_rn(m.br, bir.lo, err);
    err = __fma_rn(m.bi, bii.lo, err);
    err = __fma_rn(m.cr, cir.lo, err);
    err = __fma_rn(m.ci, cii.lo, err);
    det = __dadd_rn(s, err);
    // step 3
    t = __drcp_rn(det);
    // step 4
    o[0] = __dmul_rn(t, ai.hi);
    o[1] = __dmul_rn(t, bir.hi);
    o[2] = __dmul_rn(t, bii.hi);
    o[3] = __dmul_rn(t, cir.hi);
    o[4] = __dmul_rn(t, cii.hi);
    o[5] = __dmul_rn(t, di);
    o[6] = __dmul_rn(t, eir);
    o[7] = __dmul_rn(t, eii);
    o[8] = __dmul_rn(t, fi);
}

// ===================================================== Alg. 1 (Cholesky)
// PAPER.md:279-378 with l21 = (conj(e) - l20 conj(l10)) v1 (R-1).  Complex
// quantities as (re, im) pairs; l_kk real positive (R-4).
template <typename T>
__device__ __forceinline__ bool alg1(const H9<T>& m, T* o, T& det, T& tdet) {
    // step 1: L and v_k
    T l00 = SQRT(m.a);
    T v0 = RCP(l00);
    T l10r = MUL(m.br, v0), l10i = MUL(-m.bi, v0);  // conj(b) v0
    T l20r = MUL(m.cr, v0), l20i = MUL(-m.ci, v0);  // conj(c) v0
    T r1 = FMA(-l10r, l10r, FMA(-l10i, l10i, m.d));  // d - |l10|^2
    T l11 = SQRT(r1);
    T v1 = RCP(l11);
    // conj(e) - l20 conj(l10)
    T ur = SUB(m.er, FMA(l20r, l10r, MUL(l20i, l10i)));
    T ui = SUB(-m.ei, FMA(l20i, l10r, -MUL(l20r, l10i)));
    T l21r = MUL(ur, v1), l21i = MUL(ui, v1);
    T r2 = FMA(-l21r, l21r, FMA(-l21i, l21i, FMA(-l20r, l20r, FMA(-l20i, l20i, m.f))));
    T l22 = SQRT(r2);
    T v2 = RCP(l22);
    // step 2: T = L^-1
    T v01 = MUL(v0, v1);
    T t10r = MUL(-l10r, v01), t10i = MUL(-l10i, v01);
    T wr = FMA(l21r, l10r, -MUL(l21i, l10i));  // l21 l10
    T wi = FMA(l21r, l10i, MUL(l21i, l10r));
    T v02 = MUL(v2, v0);
    T t20r = MUL(v02, FMA(wr, v1, -l20r));
    T t20i = MUL(v02, FMA(wi, v1, -l20i));
    T v12 = MUL(v1, v2);
    T t21r = MUL(-l21r, v12), t21i = MUL(-l21i, v12);
    // step 3: det = (l00 l11 l22)^2; det^-1 = (v0 v1 v2)^2 (R-14)
    T pl = MUL(MUL(l00, l11), l22);
    det = MUL(pl, pl);
    T pv = MUL(v01, v2);
    tdet = MUL(pv, pv);
    // step 4: A^-1 = T^H T
    o[0] = FMA(v0, v0, FMA(t10r, t10r, FMA(t10i, t10i, FMA(t20r, t20r, MUL(t20i, t20i)))));
    o[1] = FMA(t10r, v1, FMA(t20r, t21r, MUL(t20i, t21i)));    // Re(conj t10 v1 + conj t20 t21)
    o[2] = FMA(-t10i, v1, FMA(t20r, t21i, -MUL(t20i, t21r)));  // Im
    o[3] = MUL(t20r, v2);                                      // conj(t20) v2
    o[4] = MUL(-t20i, v2);
    o[5] = FMA(v1, v1, FMA(t21r, t21r, MUL(t21i, t21i)));
    o[6] = MUL(t21r, v2);  // conj(t21) v2
    o[7] = MUL(-t21i, v2);
    o[8] = MUL(v2, v2);
    // radicands must be positive and finite (R-5)
    return finite_pos(m.a) && finite_pos(r1) && finite_pos(r2);
}

// ------------------------------------------------------------------ modes
// storage S, arithmetic per dtype code (include/polsar.h)
enum { ALGO_ADJ = 0, ALGO_CHOL = 1 };
enum { MATH_F64 = 0, MATH_F64_EFT = 1, MATH_F32 = 2 };

template <int MATH>
struct MathT {
    typedef typename std::conditional<MATH == MATH_F32, float, double>::type type;
};

// One matrix: inverse (9 values in the arithmetic type), det, t, status.
template <typename S, int ALGO, int MATH>
__device__ __forceinline__ uint8_t solve_core(const S* in, typename MathT<MATH>::type* o,
                                              typename MathT<MATH>::type& det,
                                              typename MathT<MATH>::type& t) {
    typedef typename MathT<MATH>::type T;
    H9<T> m;
    m.a = (T)in[0];
    m.br = (T)in[1];
    m.bi = (T)in[2];
    m.cr = (T)in[3];
    m.ci = (T)in[4];
    m.d = (T)in[5];
    m.er = (T)in[6];
    m.ei = (T)in[7];
    m.f = (T)in[8];
    bool pd = true;
    if constexpr (ALGO == ALGO_ADJ) {
        if constexpr (MATH == MATH_F64_EFT)
            alg2_accurate(m, o, det, t);
        else
            alg2_plain<T>(m, o, det, t);
    } else {
        pd = alg1<T>(m, o, det, t);
    }
    // full-rank check as a scaled threshold (R-5)
    T thr = MUL(MUL(MUL((T)Tau<S>::v, m.a), m.d), m.f);
    bool ok = (det > thr) && finite_pos(det) && finite_pos(t);
    return !pd ? (uint8_t)POLSAR_STATUS_NOT_PD
               : (ok ? (uint8_t)POLSAR_STATUS_OK : (uint8_t)POLSAR_STATUS_SINGULAR);
}

template <typename S, int ALGO, int MATH>
__device__ __forceinline__ void solve_one(const S* in, S* out, uint8_t& st) {
    typedef typename MathT<MATH>::type T;
    T o[9], det, t;
    st = solve_core<S, ALGO, MATH>(in, o, det, t);
#pragma unroll
    for (int k = 0; k < 9; ++k) out[k] = (S)o[k];
    out[9] = (S)det;
    out[10] = (S)t;
}

// --------------------------------------------------------------- K1 / K2
// Vector body: each thread owns VEC consecutive pixels, reads one 16-byte
// vector per input plane (9 x LDG.128) and writes one per output plane
// (11 x STG.128), plus VEC status bytes.  Grid-stride over groups.
template <typename S>
struct Vec;
template <>
struct Vec<float> {
    typedef float4 type;
    static constexpr int n = 4;
};
template <>
struct Vec<double> {
    typedef double2 type;
    static constexpr int n = 2;
};

template <typename V, typename S>
__device__ __forceinline__ void unpack(const V& v, S* x);
template <>
__device__ __forceinline__ void unpack<float4, float>(const float4& v, float* x) {
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}
template <>
__device__ __forceinline__ void unpack<double2, double>(const double2& v, double* x) {
    x[0] = v.x; x[1] = v.y;
}
__device__ __forceinline__ float4 pack4(const float* x) { return make_float4(x[0], x[1], x[2], x[3]); }
__device__ __forceinline__ double2 pack2(const double* x) { return make_double2(x[0], x[1]); }
__device__ __forceinline__ float4 packv(const float* x, float4*) { return pack4(x); }
__device__ __forceinline__ double2 packv(const double* x, double2*) { return pack2(x); }

constexpr int K1_THREADS = 128;

template <typename S, int ALGO, int MATH>
__global__ void __launch_bounds__(K1_THREADS)
k_inv_det_vec(const S* __restrict__ z, S* __restrict__ out, uint8_t* __restrict__ status,
              int64_t n_groups, int64_t ld) {
    typedef typename Vec<S>::type V;
    constexpr int W = Vec<S>::n;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_groups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = g * W;
        S in[9][W];
#pragma unroll
        for (int k = 0; k < 9; ++k) unpack<V, S>(ld_stream(reinterpret_cast<const V*>(z + k * ld + p)), in[k]);
        S res[11][W];
        uint8_t st[W];
#pragma unroll
        for (int v = 0; v < W; ++v) {
            S x[9], y[11];
#pragma unroll
            for (int k = 0; k < 9; ++k) x[k] = in[k][v];
            solve_one<S, ALGO, MATH>(x, y, st[v]);
#pragma unroll
            for (int k = 0; k < 11; ++k) res[k][v] = y[k];
        }
#pragma unroll
        for (int k = 0; k < 11; ++k)
            st_stream(reinterpret_cast<V*>(out + k * ld + p), packv(res[k], (V*)nullptr));
        if (status) {
            if (W == 4) {
                uint32_t w = (uint32_t)st[0] | ((uint32_t)st[1 % W] << 8) |
                             ((uint32_t)st[2 % W] << 16) | ((uint32_t)st[3 % W] << 24);
                *reinterpret_cast<uint32_t*>(status + p) = w;
            } else {
                uint16_t w = (uint16_t)(st[0] | (st[1 % W] << 8));
                *reinterpret_cast<uint16_t*>(status + p) = w;
            }
        }
    }
}

// Scalar path: misaligned planes and the ragged tail; same solve_one.
template <typename S, int ALGO, int MATH>
__global__ void __launch_bounds__(256)
k_inv_det_scalar(const S* __restrict__ z, S* __restrict__ out, uint8_t* __restrict__ status,
                 int64_t begin, int64_t end, int64_t ld) {
    for (int64_t p = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < end;
         p += (int64_t)gridDim.x * blockDim.x) {
        S x[9], y[11];
        uint8_t st;
#pragma unroll
        for (int k = 0; k < 9; ++k) x[k] = ld_stream(z + k * ld + p);
        solve_one<S, ALGO, MATH>(x, y, st);
#pragma unroll
        for (int k = 0; k < 11; ++k) st_stream(out + k * ld + p, y[k]);
        if (status) status[p] = st;
    }
}

int g_num_sms = 0;

int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

// one thread per work item, the whole batch in one grid (capped at 2^31-1
// CTAs; the kernels' grid-stride loops take any remainder)
int grid_full(int64_t work, int threads) {
    int64_t need = (work + threads - 1) / threads;
    if (need > 0x7fffffff) need = 0x7fffffff;
    return (int)(need < 1 ? 1 : need);
}

int grid_for(int64_t work, int threads) {
    // enough CTAs for every SM to hold its resident maximum several times
    // over; beyond that the grid-stride loop takes over
    int64_t need = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * 64;
    if (need > cap) need = cap;
    return (int)(need < 1 ? 1 : need);
}

template <typename S, int ALGO, int MATH>
int launch_inv_det(const void* zv, void* outv, uint8_t* status, int64_t n, int64_t ld,
                   cudaStream_t s) {
    const S* z = (const S*)zv;
    S* out = (S*)outv;
    constexpr int W = Vec<S>::n;
    bool aligned = ((uintptr_t)z % 16 == 0) && ((uintptr_t)out % 16 == 0) && (ld % W == 0) &&
                   (status == nullptr || (uintptr_t)status % W == 0);
    int64_t n_vec = aligned ? (n / W) * W : 0;
    if (n_vec > 0) {
        int64_t groups = n_vec / W;
        k_inv_det_vec<S, ALGO, MATH><<<grid_full(groups, K1_THREADS), K1_THREADS, 0, s>>>(z, out, status, groups, ld);
    }
    if (n > n_vec) {
        k_inv_det_scalar<S, ALGO, MATH>
            <<<grid_for(n - n_vec, 256), 256, 0, s>>>(z, out, status, n_vec, n, ld);
    }
    return launch_check(ALGO == ALGO_ADJ ? "polsar_inv_det: launch failed"
                                         : "polsar_inv_det_cholesky: launch failed");
}

// ------------------------------------------------ multi-frequency blocks
// PAPER.md:1043-1055 [§V]: a pixel holds nblocks Hermitian 3x3 diagonal
// blocks (one per frequency band).  Alg. 2 runs on each block; the whole
// matrix's det and det^-1 are the products of the blocks' (in the arithmetic
// type, rounded once); status is the worst block status.  Planes: input block
// b at 9b..9b+8; output block inverses at 9b..9b+8, det at 9B, det^-1 at 9B+1.
template <typename S, int MATH>
__global__ void __launch_bounds__(K1_THREADS)
k_inv_det_blocks_vec(const S* __restrict__ z, S* __restrict__ out, uint8_t* __restrict__ status,
                     int64_t n_groups, int64_t ld, int nblocks) {
    typedef typename Vec<S>::type V;
    typedef typename MathT<MATH>::type T;
    constexpr int W = Vec<S>::n;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_groups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = g * W;
        T det_all[W], t_all[W];
        uint8_t st[W];
#pragma unroll
        for (int v = 0; v < W; ++v) {
            det_all[v] = T(1);
            t_all[v] = T(1);
            st[v] = 0;
        }
        for (int b = 0; b < nblocks; ++b) {
            const S* zb = z + (int64_t)9 * b * ld;
            S* ob = out + (int64_t)9 * b * ld;
            S in[9][W];
#pragma unroll
            for (int k = 0; k < 9; ++k) unpack<V, S>(ld_stream(reinterpret_cast<const V*>(zb + k * ld + p)), in[k]);
            S res[9][W];
#pragma unroll
            for (int v = 0; v < W; ++v) {
                S x[9];
                T o[9], det, t;
#pragma unroll
                for (int k = 0; k < 9; ++k) x[k] = in[k][v];
                uint8_t s1 = solve_core<S, ALGO_ADJ, MATH>(x, o, det, t);
                st[v] = s1 > st[v] ? s1 : st[v];
                det_all[v] = MUL(det_all[v], det);
                t_all[v] = MUL(t_all[v], t);
#pragma unroll
                for (int k = 0; k < 9; ++k) res[k][v] = (S)o[k];
            }
#pragma unroll
            for (int k = 0; k < 9; ++k)
                st_stream(reinterpret_cast<V*>(ob + k * ld + p), packv(res[k], (V*)nullptr));
        }
        S dd[W], tt[W];
#pragma unroll
        for (int v = 0; v < W; ++v) {
            dd[v] = (S)det_all[v];
            tt[v] = (S)t_all[v];
        }
        S* oe = out + (int64_t)9 * nblocks * ld;
        st_stream(reinterpret_cast<V*>(oe + p), packv(dd, (V*)nullptr));
        st_stream(reinterpret_cast<V*>(oe + ld + p), packv(tt, (V*)nullptr));
        if (status) {
#pragma unroll
            for (int v = 0; v < W; ++v) status[p + v] = st[v];
        }
    }
}

template <typename S, int MATH>
__global__ void __launch_bounds__(256)
k_inv_det_blocks_scalar(const S* __restrict__ z, S* __restrict__ out, uint8_t* __restrict__ status,
                        int64_t begin, int64_t end, int64_t ld, int nblocks) {
    typedef typename MathT<MATH>::type T;
    for (int64_t p = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < end;
         p += (int64_t)gridDim.x * blockDim.x) {
        T det_all = T(1), t_all = T(1);
        uint8_t st = 0;
        for (int b = 0; b < nblocks; ++b) {
            S x[9];
            T o[9], det, t;
#pragma unroll
            for (int k = 0; k < 9; ++k) x[k] = ld_stream(z + ((int64_t)9 * b + k) * ld + p);
            uint8_t s1 = solve_core<S, ALGO_ADJ, MATH>(x, o, det, t);
            st = s1 > st ? s1 : st;
            det_all = MUL(det_all, det);
            t_all = MUL(t_all, t);
#pragma unroll
            for (int k = 0; k < 9; ++k) st_stream(out + ((int64_t)9 * b + k) * ld + p, (S)o[k]);
        }
        st_stream(out + (int64_t)9 * nblocks * ld + p, (S)det_all);
        st_stream(out + ((int64_t)9 * nblocks + 1) * ld + p, (S)t_all);
        if (status) status[p] = st;
    }
}

template <typename S, int MATH>
int launch_blocks(const void* zv, void* outv, uint8_t* status, int64_t n, int64_t ld, int nb,
                  cudaStream_t s) {
    const S* z = (const S*)zv;
    S* out = (S*)outv;
    constexpr int W = Vec<S>::n;
    bool aligned = ((uintptr_t)z % 16 == 0) && ((uintptr_t)out % 16 == 0) && (ld % W == 0);
    int64_t n_vec = aligned ? (n / W) * W : 0;
    if (n_vec > 0) {
        int64_t groups = n_vec / W;
        k_inv_det_blocks_vec<S, MATH><<<grid_full(groups, K1_THREADS), K1_THREADS, 0, s>>>(
            z, out, status, groups, ld, nb);
    }
    if (n > n_vec)
        k_inv_det_blocks_scalar<S, MATH><<<grid_for(n - n_vec, 256), 256, 0, s>>>(z, out, status, n_vec,
                                                                              n, ld, nb);
    return launch_check("polsar_inv_det_blocks: launch failed");
}

template <int ALGO>
int dispatch_inv_det(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld, int dtype,
                     void* stream) {
    if (n < 0) return fail(POLSAR_EINVAL, "n < 0");
    if (ld < n) return fail(POLSAR_EINVAL, "ld < n");
    if (n == 0) return POLSAR_OK;
    if (!z || !out) return fail(POLSAR_EINVAL, "null z or out");
    cudaStream_t s = (cudaStream_t)stream;
    switch (dtype) {
        case POLSAR_F32: return launch_inv_det<float, ALGO, MATH_F64>(z, out, status, n, ld, s);
        case POLSAR_F64:
            return ALGO == ALGO_ADJ ? launch_inv_det<double, ALGO, MATH_F64_EFT>(z, out, status, n, ld, s)
                                    : launch_inv_det<double, ALGO, MATH_F64>(z, out, status, n, ld, s);
        case POLSAR_F32_PLAIN: return launch_inv_det<float, ALGO, MATH_F32>(z, out, status, n, ld, s);
        case POLSAR_F64_PLAIN: return launch_inv_det<double, ALGO, MATH_F64>(z, out, status, n, ld, s);
        default: return fail(POLSAR_EINVAL, "bad dtype");
    }
}

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
        g[p] = (WT)(T(1) / MUL(T(8), dz));
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
__device__ __forceinline__ double pair_weight(double r, double alpha, bool alpha_is_2) {
    if (alpha_is_2) return 1.0 / (r * r);
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
    extern __shared__ unsigned char smem_raw[];
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
#pragma unroll
                    for (int k = 0; k < 9; ++k) zj[k] = rowz[k * HP + wx];
                    const WT gj = rowg[wx];
#pragma unroll
                    for (int r = 0; r < K3_RB; ++r) row[r] += pair_w<T, WT>(zi[r], gi[r], zj, gj, alpha, a2);
                }
            } else {
                for (int wx = -R; wx <= R; ++wx) {
                    T zj[9];
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
// K4: non-local-means filter output (the NLM filter with
// stochastic distances of PAPER.md:77-80 [§I]).  Same pair weights as K3 and
// in the same pass, accumulated with the window pixels themselves:
//   W_i = sum_j w_ij,   Zhat_i = sum_j w_ij Z_j / W_i   (9 packed planes).
// Layout and staging as k_window_sum; the weighted sums accumulate in the
// pair-determinant type (fp64 for the default modes: one F2F, one DADD and
// nine DFMA per pair on top of the determinant).
template <typename S, typename T, typename WT, int TY, int RB>
__global__ void __launch_bounds__(K3_TX * TY / RB, 1)
k_nlm_sum(const S* __restrict__ z, int64_t ld, int64_t width, int64_t slab_rows,
          int64_t row_begin, int64_t row_end, int R, const WT* __restrict__ g, double alpha_d,
          int alpha_is_2, S* __restrict__ out_w, S* __restrict__ out_z, int64_t ld_out) {
    extern __shared__ unsigned char smem_raw[];
    const int HW = K3_TX + 2 * R;
    const int HH = TY + 2 * R;
    const int HP = HW * HH;
    T* sz = reinterpret_cast<T*>(smem_raw);
    WT* sg = reinterpret_cast<WT*>(sz + 9 * HP);

    const int64_t x0 = (int64_t)blockIdx.x * K3_TX;
    const int64_t y0 = row_begin + (int64_t)blockIdx.y * TY;
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
    const int ty0 = (threadIdx.x / K3_TX) * RB;
    const int64_t gx = x0 + tx;
    T zi[RB][9], accz[RB][9], accw[RB];
    WT gi[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        int q = (ty0 + r + R) * HW + (tx + R);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            zi[r][k] = sz[k * HP + q];
            accz[r][k] = T(0);
        }
        gi[r] = sg[q];
        accw[r] = T(0);
    }
    const WT alpha = (WT)alpha_d;
    const bool a2 = alpha_is_2 != 0;
    const bool interior_x = (x0 - R >= 0) && (x0 + K3_TX + R <= width);

    for (int wy = -R; wy <= R + RB - 1; ++wy) {
        const int64_t gyj = y0 + ty0 + wy;
        if (gyj < 0 || gyj >= slab_rows) continue;  // warp-uniform
        const int hy = ty0 + wy + R;
        const T* rowz = sz + hy * HW + tx + R;
        const WT* rowg = sg + hy * HW + tx + R;
        bool rok[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) rok[r] = (wy - r >= -R) && (wy - r <= R);  // warp-uniform
        for (int wx = -R; wx <= R; ++wx) {
            T zj[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) zj[k] = rowz[k * HP + wx];
            const WT gj = rowg[wx];
            const bool colok = interior_x || (gx + wx >= 0 && gx + wx < width);
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if (rok[r]) {
                    WT w = pair_w<T, WT>(zi[r], gi[r], zj, gj, alpha, a2);
                    const T wt = colok ? (T)w : T(0);
                    accw[r] = ADD(accw[r], wt);
#pragma unroll
                    for (int k = 0; k < 9; ++k) accz[r][k] = FMA(wt, zj[k], accz[r][k]);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int64_t gy = y0 + ty0 + r;
        if (gx < width && gy < row_end) {
            const int64_t o = (gy - row_begin) * width + gx;
            if (out_w) out_w[o] = (S)accw[r];
#pragma unroll
            for (int k = 0; k < 9; ++k) out_z[k * ld_out + o] = (S)(accz[r][k] / accw[r]);
        }
    }
}

template <typename S, typename T, typename WT>
int launch_nlm(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb, int64_t re,
               int R, double looks, double h, void* ws, void* out_w, void* out_z, int64_t ld_out,
               cudaStream_t s) {
    const S* z = (const S*)zv;
    WT* g = (WT*)ws;
    const int64_t n = slab_rows * width;
    k_window_prep<S, T, WT><<<grid_for(n, 256), 256, 0, s>>>(z, ld, n, g);
    const double alpha = looks / (2.0 * h);
    dim3 block(K3_TX * 16 / 2);
    int TY = 16;
    size_t smem = window_smem<T, WT>(16, R);
    if (smem > K3_SMEM_MAX) {
        TY = 8;
        smem = window_smem<T, WT>(8, R);
        if (smem > K3_SMEM_MAX)
            return fail(POLSAR_ENOTSUP, "polsar_nlm_filter: radius too large for shared memory");
    }
    auto kern = TY == 16 ? k_nlm_sum<S, T, WT, 16, 2> : k_nlm_sum<S, T, WT, 8, 2>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return fail(POLSAR_ENOTSUP, "polsar_nlm_filter: shared memory request too large");
    dim3 grid((unsigned)((width + K3_TX - 1) / K3_TX), (unsigned)((re - rb + TY - 1) / TY));
    kern<<<grid, K3_TX * TY / 2, smem, s>>>(z, ld, width, slab_rows, rb, re, R, g, alpha,
                                            alpha == 2.0 ? 1 : 0, (S*)out_w, (S*)out_z, ld_out);
    return launch_check("polsar_nlm_filter: launch failed");
}

// ------------------------------------------------------------------------
// K3 (v3, the fp64-determinant modes): the pair determinant by the 3x3
// expansion  det(A + B) = det A + det B + <adj A, B> + <A, adj B>,
// <X, Y> = tr(X Y) = sum_k w_k x_k y_k over the packed components with
// w = (1, 2, 2, 2, 2, 1, 2, 2, 1).  Alg. 2's cofactors (Eq. 3) and
// determinant (Eq. 6) are evaluated ONCE per pixel in the prepass; each pair
// then costs one add and 18 FMAs instead of 9 adds and 20 multiply-adds
// (S = Z_i + Z_j, then Eq. 6 on S).  All four terms are >= 0 for positive-
// definite pixels, so the sum itself cannot cancel.
//
// Prepass (K3a v3) writes 20 fp64 planes per slab pixel:
//   0..8   z   (the packed Z)
//   9..17  u = w * adj(Z) (cofactors a_c, b_c, c_c, d_c, e_c, f_c, weighted)
//   18     D = det Z (Eq. 6)
//   19     g = 1 / (8 D) as float in the low 4 bytes
// Main pass (K3b v3): a CTA owns a 256-column x RB-row output block (each
// thread one column, RB rows).  The window rows it needs stream through
// shared memory V3_CH rows at a time (all 20 planes, 256 + 2R' columns),
// double-buffered with cp.async so the next rows load while the current ones
// are consumed.  Every thread of the CTA pairs each staged row with the same
// owned rows, so the per-row work is identical across warps (no barrier
// imbalance), and each staged Z_j serves RB pairs.
constexpr int V3_TX = 256;
constexpr int V3_RB = 4;
constexpr int V3_CH = 2;
constexpr int V3_NP = 20;        // planes per pixel
constexpr int V3_THREADS = V3_TX;
constexpr int V3_RMAX = 12;      // radius limit of this kernel (the paper's R = 11)
constexpr int V3_XOFF = V3_RMAX; // column of x0 inside a staged row (even)
constexpr int V3_SW = V3_TX + 2 * V3_XOFF;  // staged row width (compile-time strides)
constexpr int V3_CHP = V3_CH * V3_SW;       // pixels per chunk plane

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
#pragma unroll
        for (int k = 0; k < 9; ++k) ws[(9 + k) * P + p] = wk[k] * x[k];
        ws[18 * P + p] = 0.0;
        ws[19 * P + p] = 0.0;
    }
}

template <typename S, typename WT>
__global__ void __launch_bounds__(256)
k_window_prep_v3(const S* __restrict__ z, int64_t ld, int64_t n, double* __restrict__ ws) {
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
        // Eq. 3 cofactors (Alg. 2 step 1) and Eq. 6 determinant (step 2)
        double ac = FMA(m.d, m.f, -FMA(m.er, m.er, MUL(m.ei, m.ei)));
        double bcr = FMA(m.cr, m.er, FMA(m.ci, m.ei, -MUL(m.br, m.f)));
        double bci = FMA(m.ci, m.er, -FMA(m.cr, m.ei, MUL(m.bi, m.f)));
        double ccr = FMA(m.br, m.er, -FMA(m.bi, m.ei, MUL(m.cr, m.d)));
        double cci = FMA(m.br, m.ei, FMA(m.bi, m.er, -MUL(m.ci, m.d)));
        double dc = FMA(m.a, m.f, -FMA(m.cr, m.cr, MUL(m.ci, m.ci)));
        double ecr = FMA(m.cr, m.br, FMA(m.ci, m.bi, -MUL(m.a, m.er)));
        double eci = FMA(m.ci, m.br, -FMA(m.cr, m.bi, MUL(m.a, m.ei)));
        double fc = FMA(m.a, m.d, -FMA(m.br, m.br, MUL(m.bi, m.bi)));
        double det = FMA(m.a, ac, FMA(m.br, bcr, FMA(m.bi, bci, FMA(m.cr, ccr, MUL(m.ci, cci)))));
        const int64_t P = n;  // plane stride of the workspace
        ws[0 * P + p] = m.a;  ws[1 * P + p] = m.br; ws[2 * P + p] = m.bi;
        ws[3 * P + p] = m.cr; ws[4 * P + p] = m.ci; ws[5 * P + p] = m.d;
        ws[6 * P + p] = m.er; ws[7 * P + p] = m.ei; ws[8 * P + p] = m.f;
        ws[9 * P + p] = ac;
        ws[10 * P + p] = 2.0 * bcr; ws[11 * P + p] = 2.0 * bci;
        ws[12 * P + p] = 2.0 * ccr; ws[13 * P + p] = 2.0 * cci;
        ws[14 * P + p] = dc;
        ws[15 * P + p] = 2.0 * ecr; ws[16 * P + p] = 2.0 * eci;
        ws[17 * P + p] = fc;
        ws[18 * P + p] = det;
        const double g = 1.0 / (8.0 * det);
        if constexpr (std::is_same<WT, float>::value)
            ws[19 * P + p] = __longlong_as_double((long long)(unsigned)__float_as_uint((float)g));
        else
            ws[19 * P + p] = g;
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
template <typename WT>
__device__ __forceinline__ WT load_g(double v);
template <>
__device__ __forceinline__ float load_g<float>(double v) {
    return __uint_as_float((unsigned)__double_as_longlong(v));
}
template <>
__device__ __forceinline__ double load_g<double>(double v) { return v; }

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

template <typename WT>
__device__ __forceinline__ WT weight_v3(double T, WT gi, WT gj, WT alpha, bool a2) {
    WT ft = (WT)T;
    WT rr = (ft * gi) * (ft * gj);
    return pair_weight(rr, alpha, a2);
}

// one pair: T = det(Z_i + Z_j) = D_i + D_j + <u_i, z_j> + <z_i, u_j>
__device__ __forceinline__ double pair_T(const double* ui, const double* zi, double Di,
                                         const double* uj, const double* zj, double Dj) {
    double a = __fma_rn(ui[0], zj[0], __dadd_rn(Di, Dj));
    double b = __dmul_rn(ui[6], zj[6]);
    double c = __dmul_rn(zi[3], uj[3]);
    a = __fma_rn(ui[1], zj[1], a);
    b = __fma_rn(ui[7], zj[7], b);
    c = __fma_rn(zi[4], uj[4], c);
    a = __fma_rn(ui[2], zj[2], a);
    b = __fma_rn(ui[8], zj[8], b);
    c = __fma_rn(zi[5], uj[5], c);
    a = __fma_rn(ui[3], zj[3], a);
    b = __fma_rn(zi[0], uj[0], b);
    c = __fma_rn(zi[6], uj[6], c);
    a = __fma_rn(ui[4], zj[4], a);
    b = __fma_rn(zi[1], uj[1], b);
    c = __fma_rn(zi[7], uj[7], c);
    a = __fma_rn(ui[5], zj[5], a);
    b = __fma_rn(zi[2], uj[2], b);
    c = __fma_rn(zi[8], uj[8], c);
    return __dadd_rn(a, __dadd_rn(b, c));
}


// T_r = det(Z_{i_r} + Z_j) for the RB owned pixels at once, written as
// 2*RB independent FMA chains (k-outer, pixel-inner) so the FP64 pipe always
// has independent work in flight.
template <int RB>
__device__ __forceinline__ void pair_T_block(const double (&ui)[RB][9], const double (&zi)[RB][9],
                                             const double (&Di)[RB], const double* uj,
                                             const double* zj, double Dj, double (&T)[RB]) {
    double A[RB], B[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        A[r] = __fma_rn(ui[r][0], zj[0], Di[r]);
        B[r] = __fma_rn(zi[r][0], uj[0], Dj);
    }
#pragma unroll
    for (int k = 1; k < 9; ++k) {
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            A[r] = __fma_rn(ui[r][k], zj[k], A[r]);
            B[r] = __fma_rn(zi[r][k], uj[k], B[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) T[r] = __dadd_rn(A[r], B[r]);
}

enum { DIST_LOGDET = 0, DIST_KL = 1 };

template <int KIND, typename WT>
__device__ __forceinline__ WT weight_kind(double T, WT gi, WT gj, WT alpha, bool a2) {
    if constexpr (KIND == DIST_KL)
        return weight_kl<WT>(T, alpha);
    else
        return weight_v3<WT>(T, gi, gj, alpha, a2);
}

template <typename S, typename WT, bool A2, int KIND = DIST_LOGDET>
__global__ void __launch_bounds__(V3_THREADS, 1)
k_window_sum_v3(const double* __restrict__ ws, int64_t width, int64_t slab_rows, int64_t row_begin,
                int64_t row_end, int R, double alpha_d, S* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int XOFF = V3_XOFF, SW = V3_SW, CHP = V3_CHP;
    double* buf = reinterpret_cast<double*>(smem_raw);  // [2][V3_NP][V3_CH][SW]
    const int64_t P = slab_rows * width;                // workspace plane stride

    const int64_t x0 = (int64_t)blockIdx.x * V3_TX;
    const int64_t y0 = row_begin + (int64_t)blockIdx.y * V3_RB;
    // window rows of the block, clipped to the slab
    const int64_t ja = y0 - R > 0 ? y0 - R : 0;
    const int64_t jb = (y0 + V3_RB - 1 + R) < slab_rows - 1 ? (y0 + V3_RB - 1 + R) : slab_rows - 1;
    const int nrows = (int)(jb - ja + 1);
    const int nchunks = (nrows + V3_CH - 1) / V3_CH;

    auto load_chunk = [&](int c, int b) {
        double* dst = buf + (size_t)b * V3_NP * CHP;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int pr = warp; pr < V3_NP * V3_CH; pr += V3_THREADS / 32) {
            const int pl = pr / V3_CH, row = pr % V3_CH;  // compile-time divisors
            const int64_t gy = ja + (int64_t)c * V3_CH + row;
            const bool rok = gy <= jb;
            const double* srow = ws + pl * P + (rok ? gy : 0) * width;
            double* drow = dst + pl * CHP + row * SW;
            for (int col = lane; col < SW; col += 32) {
                const int64_t gxx = x0 - XOFF + col;
                const bool ok = rok && gxx >= 0 && gxx < width;
                cp_async8(drow + col, srow + (ok ? gxx : 0), ok);
            }
        }
        cp_async_commit();
    };
    load_chunk(0, 0);

    // owned pixels: column gx, rows y0 .. y0 + RB - 1
    const int tx = threadIdx.x;
    const int64_t gx = x0 + tx;
    double ui[V3_RB][9], zi[V3_RB][9], Di[V3_RB];
    WT gi[V3_RB];
    double acc[V3_RB];
#pragma unroll
    for (int r = 0; r < V3_RB; ++r) {
        const int64_t gy = y0 + r;
        const bool ok = gx < width && gy < slab_rows;
        const int64_t p = ok ? gy * width + gx : 0;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            zi[r][k] = ok ? ws[k * P + p] : 0.0;
            ui[r][k] = ok ? ws[(9 + k) * P + p] : 0.0;
        }
        Di[r] = ok ? ws[18 * P + p] : 0.0;
        gi[r] = ok ? load_g<WT>(ws[19 * P + p]) : WT(0);
        acc[r] = 0.0;
    }
    const WT alpha = (WT)alpha_d;
    constexpr bool a2 = A2;
    const bool interior_x = (x0 - R >= 0) && (x0 + V3_TX + R <= width);

    for (int c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) {
            load_chunk(c + 1, (c + 1) & 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* cb = buf + (size_t)(c & 1) * V3_NP * CHP;
#pragma unroll 1
        for (int row = 0; row < V3_CH; ++row) {
            const int64_t gyj = ja + (int64_t)c * V3_CH + row;
            if (gyj > jb) break;
            const int dy0 = (int)(gyj - y0);  // dy of owned row r is dy0 - r (CTA-uniform)
            const double* rb = cb + row * SW + XOFF + tx;
            WT rowacc[V3_RB];
#pragma unroll
            for (int r = 0; r < V3_RB; ++r) rowacc[r] = WT(0);
            const bool all = (dy0 - (V3_RB - 1) >= -R) && (dy0 <= R);
            if (all) {
                // software-pipelined: the weights of column wx-1 (F2F / FMUL /
                // MUFU, long-latency) are evaluated alongside the FMA chains of
                // column wx, so the FP64 pipe never waits on the weight tail
                double Tp[V3_RB];
                WT gp = WT(0);
                bool okp = false;
#pragma unroll
                for (int r = 0; r < V3_RB; ++r) Tp[r] = 1.0;
#pragma unroll 1
                for (int wx = -R; wx <= R; ++wx) {
                    double zj[9], uj[9];
#pragma unroll
                    for (int k = 0; k < 9; ++k) {
                        zj[k] = rb[k * CHP + wx];
                        uj[k] = rb[(9 + k) * CHP + wx];
                    }
                    const double Dj = rb[18 * CHP + wx];
                    const WT gj = load_g<WT>(rb[19 * CHP + wx]);
                    const bool colok = interior_x || (gx + wx >= 0 && gx + wx < width);
                    double T[V3_RB];
                    pair_T_block<V3_RB>(ui, zi, Di, uj, zj, Dj, T);
#pragma unroll
                    for (int r = 0; r < V3_RB; ++r) {
                        WT w = weight_kind<KIND, WT>(Tp[r], gi[r], gp, alpha, a2);
                        rowacc[r] += okp ? w : WT(0);
                        Tp[r] = T[r];
                    }
                    gp = gj;
                    okp = colok;
                }
#pragma unroll
                for (int r = 0; r < V3_RB; ++r) {
                    WT w = weight_kind<KIND, WT>(Tp[r], gi[r], gp, alpha, a2);
                    rowacc[r] += okp ? w : WT(0);
                }
            } else {
#pragma unroll 1
                for (int wx = -R; wx <= R; ++wx) {
                    double zj[9], uj[9];
#pragma unroll
                    for (int k = 0; k < 9; ++k) {
                        zj[k] = rb[k * CHP + wx];
                        uj[k] = rb[(9 + k) * CHP + wx];
                    }
                    const double Dj = rb[18 * CHP + wx];
                    const WT gj = load_g<WT>(rb[19 * CHP + wx]);
                    const bool colok = interior_x || (gx + wx >= 0 && gx + wx < width);
#pragma unroll
                    for (int r = 0; r < V3_RB; ++r) {
                        const int dy = dy0 - r;
                        if (dy >= -R && dy <= R) {  // CTA-uniform
                            WT w = weight_kind<KIND, WT>(pair_T(ui[r], zi[r], Di[r], uj, zj, Dj), gi[r], gj, alpha, a2);
                            rowacc[r] += colok ? w : WT(0);
                        }
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < V3_RB; ++r) acc[r] += (double)rowacc[r];
        }
        __syncthreads();  // buffer (c & 1) is refilled by the prefetch of chunk c + 2
    }
#pragma unroll
    for (int r = 0; r < V3_RB; ++r) {
        const int64_t gy = y0 + r;
        if (gx < width && gy < row_end) out[(gy - row_begin) * width + gx] = (S)acc[r];
    }
}

template <typename S, typename WT>
int launch_window_v3(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb,
                     int64_t re, int R, double looks, double h, void* wsv, void* outv,
                     cudaStream_t s) {
    const int64_t n = slab_rows * width;
    double* ws = (double*)wsv;
    k_window_prep_v3<S, WT><<<grid_for(n, 256), 256, 0, s>>>((const S*)zv, ld, n, ws);
    size_t smem = (size_t)2 * V3_NP * V3_CHP * sizeof(double);
    const double alpha = looks / (2.0 * h);
    auto kern = alpha == 2.0 ? k_window_sum_v3<S, WT, true> : k_window_sum_v3<S, WT, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return fail(POLSAR_ENOTSUP, "polsar_window_distance: shared memory request too large");
    dim3 grid((unsigned)((width + V3_TX - 1) / V3_TX), (unsigned)((re - rb + V3_RB - 1) / V3_RB));
    kern<<<grid, V3_THREADS, smem, s>>>(ws, width, slab_rows, rb, re, R, alpha, (S*)outv);
    return launch_check("polsar_window_distance: launch failed");
}

template <typename S, typename WT>
int launch_window_kl(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb,
                     int64_t re, int R, double looks, double h, void* wsv, void* outv,
                     cudaStream_t s) {
    const int64_t n = slab_rows * width;
    double* ws = (double*)wsv;
    k_window_prep_kl<S><<<grid_for(n, 256), 256, 0, s>>>((const S*)zv, ld, n, ws);
    size_t smem = (size_t)2 * V3_NP * V3_CHP * sizeof(double);
    auto kern = k_window_sum_v3<S, WT, false, DIST_KL>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return fail(POLSAR_ENOTSUP, "polsar_window_kl: shared memory request too large");
    dim3 grid((unsigned)((width + V3_TX - 1) / V3_TX), (unsigned)((re - rb + V3_RB - 1) / V3_RB));
    kern<<<grid, V3_THREADS, smem, s>>>(ws, width, slab_rows, rb, re, R, looks / h, (S*)outv);
    return launch_check("polsar_window_kl: launch failed");
}

// ======================================================= R1: checksums
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

template <typename U>
__global__ void __launch_bounds__(256)
k_checksum(const U* __restrict__ planes, int64_t n, int64_t ld, int nplanes, int64_t pix_offset,
           const uint8_t* __restrict__ status, unsigned long long* __restrict__ result) {
    uint64_t h = 0;
    unsigned long long c0 = 0, c1 = 0, c2 = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = (uint64_t)(pix_offset + p) * 0x9E3779B97F4A7C15ull;
        for (int k = 0; k < nplanes; ++k)
            h += mix64((uint64_t)planes[k * ld + p] ^ (key + (uint64_t)k * 0xD6E8FEB86659FD93ull));
        if (status) {
            uint8_t s = status[p];
            c0 += s == 0;
            c1 += s == 1;
            c2 += s == 2;
        }
    }
    // warp reduction, then one atomic per warp (wrapping uint64 sums commute)
    for (int o = 16; o > 0; o >>= 1) {
        h += __shfl_down_sync(0xffffffffu, h, o);
        c0 += __shfl_down_sync(0xffffffffu, c0, o);
        c1 += __shfl_down_sync(0xffffffffu, c1, o);
        c2 += __shfl_down_sync(0xffffffffu, c2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(result + 0, (unsigned long long)h);
        if (status) {
            atomicAdd(result + 1, c0);
            atomicAdd(result + 2, c1);
            atomicAdd(result + 3, c2);
        }
    }
}

}  // namespace

// Window kernel variant for the fp64-determinant modes: 2 (direct Eq. 6 on
// S = Z_i + Z_j, default: fastest measured on B200) or 3 (cubic expansion
// over per-pixel adjugates, fewer FP64 ops but smem/register bound);
// POLSAR_WINDOW_VARIANT=3 selects the latter (A/B runs; both are parity-tested).
int window_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("POLSAR_WINDOW_VARIANT");
        v = (e && e[0] == '3') ? 3 : 2;
    }
    return v;
}

// ============================================================== C-ABI
extern "C" {

int polsar_inv_det(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld, int dtype,
                   void* cuda_stream) {
    return dispatch_inv_det<ALGO_ADJ>(z, out, status, n, ld, dtype, cuda_stream);
}

int polsar_inv_det_cholesky(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld,
                            int dtype, void* cuda_stream) {
    return dispatch_inv_det<ALGO_CHOL>(z, out, status, n, ld, dtype, cuda_stream);
}

int polsar_inv_det_blocks(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld,
                          int nblocks, int dtype, void* cuda_stream) {
    if (n < 0) return fail(POLSAR_EINVAL, "n < 0");
    if (ld < n) return fail(POLSAR_EINVAL, "ld < n");
    if (nblocks < 1 || nblocks > 64) return fail(POLSAR_EINVAL, "nblocks out of [1, 64]");
    if (n == 0) return POLSAR_OK;
    if (!z || !out) return fail(POLSAR_EINVAL, "null z or out");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    switch (dtype) {
        case POLSAR_F32: return launch_blocks<float, MATH_F64>(z, out, status, n, ld, nblocks, s);
        case POLSAR_F64: return launch_blocks<double, MATH_F64_EFT>(z, out, status, n, ld, nblocks, s);
        case POLSAR_F32_PLAIN: return launch_blocks<float, MATH_F32>(z, out, status, n, ld, nblocks, s);
        case POLSAR_F64_PLAIN: return launch_blocks<double, MATH_F64>(z, out, status, n, ld, nblocks, s);
        default: return fail(POLSAR_EINVAL, "bad dtype");
    }
}

size_t polsar_window_workspace_bytes(int64_t slab_rows, int64_t width, int dtype) {
    if (slab_rows < 0 || width < 0) return 0;
    // fp64-determinant modes: 20 fp64 planes per pixel (z, weighted adj(Z),
    // det, g); F32_PLAIN: one fp32 plane of g (rounded up to 256 bytes)
    size_t per = (dtype == POLSAR_F32_PLAIN) ? 4 : 20 * 8;
    return (((size_t)(slab_rows * width) * per) + 255) / 256 * 256;
}

int polsar_window_distance(const void* z, int64_t ld, int64_t width, int64_t slab_rows,
                           int64_t out_row_begin, int64_t out_row_end, int radius, double looks,
                           double h, void* workspace, void* out, int dtype, void* cuda_stream) {
    if (width < 0 || slab_rows < 0) return fail(POLSAR_EINVAL, "negative size");
    if (out_row_begin < 0 || out_row_end < out_row_begin || out_row_end > slab_rows)
        return fail(POLSAR_EINVAL, "bad output row range");
    if (radius < 0 || radius > 16) return fail(POLSAR_EINVAL, "radius out of [0, 16]");
    if (!(looks > 0) || !(h > 0)) return fail(POLSAR_EINVAL, "looks and h must be > 0");
    if (ld < slab_rows * width) return fail(POLSAR_EINVAL, "ld < slab_rows*width");
    if (width == 0 || out_row_end == out_row_begin) return POLSAR_OK;
    if (!z || !workspace || !out) return fail(POLSAR_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    switch (dtype) {
        case POLSAR_F32:
            if (radius <= V3_RMAX && window_variant() == 3)
                return launch_window_v3<float, float>(z, ld, width, slab_rows, out_row_begin,
                                                      out_row_end, radius, looks, h, workspace, out, s);
            return launch_window<float, double, float>(z, ld, width, slab_rows, out_row_begin,
                                                       out_row_end, radius, looks, h, workspace, out, s);
        case POLSAR_F64:
        case POLSAR_F64_PLAIN:
            if (radius <= V3_RMAX && window_variant() == 3)
                return launch_window_v3<double, double>(z, ld, width, slab_rows, out_row_begin,
                                                        out_row_end, radius, looks, h, workspace, out, s);
            return launch_window<double, double, double>(z, ld, width, slab_rows, out_row_begin,
                                                         out_row_end, radius, looks, h, workspace, out, s);
        case POLSAR_F32_PLAIN:
            return launch_window<float, float, float>(z, ld, width, slab_rows, out_row_begin,
                                                      out_row_end, radius, looks, h, workspace, out, s);
        default: return fail(POLSAR_EINVAL, "bad dtype");
    }
}

int polsar_window_kl(const void* z, int64_t ld, int64_t width, int64_t slab_rows,
                     int64_t out_row_begin, int64_t out_row_end, int radius, double looks,
                     double h, void* workspace, void* out, int dtype, void* cuda_stream) {
    if (width < 0 || slab_rows < 0) return fail(POLSAR_EINVAL, "negative size");
    if (out_row_begin < 0 || out_row_end < out_row_begin || out_row_end > slab_rows)
        return fail(POLSAR_EINVAL, "bad output row range");
    if (radius < 0 || radius > V3_RMAX) return fail(POLSAR_EINVAL, "radius out of [0, 12]");
    if (!(looks > 0) || !(h > 0)) return fail(POLSAR_EINVAL, "looks and h must be > 0");
    if (ld < slab_rows * width) return fail(POLSAR_EINVAL, "ld < slab_rows*width");
    if (width == 0 || out_row_end == out_row_begin) return POLSAR_OK;
    if (!z || !workspace || !out) return fail(POLSAR_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    switch (dtype) {
        case POLSAR_F32:
            return launch_window_kl<float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                  radius, looks, h, workspace, out, s);
        case POLSAR_F64:
        case POLSAR_F64_PLAIN:
            return launch_window_kl<double, double>(z, ld, width, slab_rows, out_row_begin,
                                                    out_row_end, radius, looks, h, workspace, out, s);
        default: return fail(POLSAR_ENOTSUP, "polsar_window_kl: fp32-arithmetic mode not provided");
    }
}

int polsar_nlm_filter(const void* z, int64_t ld, int64_t width, int64_t slab_rows,
                      int64_t out_row_begin, int64_t out_row_end, int radius, double looks,
                      double h, void* workspace, void* out_w, void* out_z, int64_t ld_out,
                      int dtype, void* cuda_stream) {
    if (width < 0 || slab_rows < 0) return fail(POLSAR_EINVAL, "negative size");
    if (out_row_begin < 0 || out_row_end < out_row_begin || out_row_end > slab_rows)
        return fail(POLSAR_EINVAL, "bad output row range");
    if (radius < 0 || radius > 16) return fail(POLSAR_EINVAL, "radius out of [0, 16]");
    if (!(looks > 0) || !(h > 0)) return fail(POLSAR_EINVAL, "looks and h must be > 0");
    if (ld < slab_rows * width) return fail(POLSAR_EINVAL, "ld < slab_rows*width");
    if (ld_out < (out_row_end - out_row_begin) * width) return fail(POLSAR_EINVAL, "ld_out too small");
    if (width == 0 || out_row_end == out_row_begin) return POLSAR_OK;
    if (!z || !workspace || !out_z) return fail(POLSAR_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    switch (dtype) {
        case POLSAR_F32:
            return launch_nlm<float, double, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                    radius, looks, h, workspace, out_w, out_z, ld_out, s);
        case POLSAR_F64:
        case POLSAR_F64_PLAIN:
            return launch_nlm<double, double, double>(z, ld, width, slab_rows, out_row_begin,
                                                      out_row_end, radius, looks, h, workspace, out_w,
                                                      out_z, ld_out, s);
        case POLSAR_F32_PLAIN:
            return launch_nlm<float, float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                   radius, looks, h, workspace, out_w, out_z, ld_out, s);
        default: return fail(POLSAR_EINVAL, "bad dtype");
    }
}

int polsar_checksum(const void* planes, int64_t n, int64_t ld, int nplanes, int dtype,
                    int64_t pix_offset, const uint8_t* status, uint64_t* result, void* cuda_stream) {
    if (n < 0 || ld < n || nplanes < 0 || !result) return fail(POLSAR_EINVAL, "bad checksum args");
    if (n == 0) return POLSAR_OK;
    if (nplanes > 0 && !planes) return fail(POLSAR_EINVAL, "null planes");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    int grid = grid_for(n, 256);
    if (dtype == POLSAR_F32 || dtype == POLSAR_F32_PLAIN)
        k_checksum<uint32_t><<<grid, 256, 0, s>>>((const uint32_t*)planes, n, ld, nplanes, pix_offset,
                                                  status, (unsigned long long*)result);
    else if (dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN)
        k_checksum<uint64_t><<<grid, 256, 0, s>>>((const uint64_t*)planes, n, ld, nplanes, pix_offset,
                                                  status, (unsigned long long*)result);
    else
        return fail(POLSAR_EINVAL, "bad dtype");
    return launch_check("polsar_checksum: launch failed");
}

int64_t polsar_host_chunk_pixels(size_t ws_bytes, int dtype) {
    size_t es = (dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN) ? 8 : 4;
    // 3 slots x (9 in + 11 out planes + 1 status byte) per pixel, chunk a
    // multiple of 64 pixels so every device plane stays 256-byte aligned
    size_t per = 3 * (20 * es + 1);
    int64_t c = (int64_t)(ws_bytes / per);
    return (c / 64) * 64;
}

int polsar_inv_det_host(const void* z_host, void* out_host, uint8_t* status_host, int64_t n,
                        int64_t ld_host, int dtype, int algo, void* dev_ws, size_t ws_bytes,
                        void* stream_h2d, void* stream_compute, void* stream_d2h) {
    if (n < 0 || ld_host < n) return fail(POLSAR_EINVAL, "bad n / ld_host");
    if (n == 0) return POLSAR_OK;
    if (!z_host || !out_host || !dev_ws) return fail(POLSAR_EINVAL, "null pointer");
    if ((uintptr_t)dev_ws % 256) return fail(POLSAR_EINVAL, "dev_ws must be 256-byte aligned");
    if (algo != 0 && algo != 1) return fail(POLSAR_EINVAL, "bad algo");
    if (dtype < POLSAR_F32 || dtype > POLSAR_F64_PLAIN) return fail(POLSAR_EINVAL, "bad dtype");
    if (!stream_h2d || !stream_compute || !stream_d2h || stream_h2d == stream_compute ||
        stream_h2d == stream_d2h || stream_compute == stream_d2h)
        return fail(POLSAR_EINVAL, "three distinct non-null streams required");
    const size_t es = (dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN) ? 8 : 4;
    const int64_t chunk = polsar_host_chunk_pixels(ws_bytes, dtype);
    if (chunk <= 0) return fail(POLSAR_EINVAL, "workspace too small");
    cudaStream_t sh = (cudaStream_t)stream_h2d, sc = (cudaStream_t)stream_compute,
                 sd = (cudaStream_t)stream_d2h;
    // slot layout: [9 in planes][11 out planes][status], each plane `chunk` elements
    const size_t slot_bytes = (size_t)chunk * (20 * es + 1);
    cudaEvent_t ev_in[3], ev_k[3], ev_out[3];
    for (int i = 0; i < 3; ++i) {
        cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_k[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming);
    }
    int rc = POLSAR_OK;
    const int64_t n_chunks = (n + chunk - 1) / chunk;
    for (int64_t c = 0; c < n_chunks && rc == POLSAR_OK; ++c) {
        const int slot = (int)(c % 3);
        const int64_t p0 = c * chunk;
        const int64_t m = (n - p0) < chunk ? (n - p0) : chunk;
        unsigned char* base = (unsigned char*)dev_ws + slot * slot_bytes;
        unsigned char* din = base;
        unsigned char* dout = base + (size_t)9 * chunk * es;
        uint8_t* dst = (uint8_t*)(base + (size_t)20 * chunk * es);
        if (c >= 3) cudaStreamWaitEvent(sh, ev_out[slot], 0);  // slot drained by its D2H
        if (cudaMemcpy2DAsync(din, chunk * es, (const unsigned char*)z_host + p0 * es, ld_host * es,
                              m * es, 9, cudaMemcpyHostToDevice, sh) != cudaSuccess) {
            rc = fail(POLSAR_ECUDA, "polsar_inv_det_host: H2D copy failed");
            break;
        }
        cudaEventRecord(ev_in[slot], sh);
        cudaStreamWaitEvent(sc, ev_in[slot], 0);
        rc = (algo == 0 ? polsar_inv_det : polsar_inv_det_cholesky)(
            din, dout, status_host ? dst : nullptr, m, chunk, dtype, sc);
        if (rc != POLSAR_OK) break;
        cudaEventRecord(ev_k[slot], sc);
        cudaStreamWaitEvent(sd, ev_k[slot], 0);
        if (cudaMemcpy2DAsync((unsigned char*)out_host + p0 * es, ld_host * es, dout, chunk * es,
                              m * es, 11, cudaMemcpyDeviceToHost, sd) != cudaSuccess) {
            rc = fail(POLSAR_ECUDA, "polsar_inv_det_host: D2H copy failed");
            break;
        }
        if (status_host &&
            cudaMemcpyAsync(status_host + p0, dst, m, cudaMemcpyDeviceToHost, sd) != cudaSuccess) {
            rc = fail(POLSAR_ECUDA, "polsar_inv_det_host: D2H status copy failed");
            break;
        }
        cudaEventRecord(ev_out[slot], sd);
    }
    if (cudaStreamSynchronize(sd) != cudaSuccess && rc == POLSAR_OK)
        rc = fail(POLSAR_ECUDA, "polsar_inv_det_host: stream error");
    for (int i = 0; i < 3; ++i) {
        cudaEventDestroy(ev_in[i]);
        cudaEventDestroy(ev_k[i]);
        cudaEventDestroy(ev_out[i]);
    }
    return rc;
}

const char* polsar_last_error(void) { return g_last_error; }

int polsar_version(void) { return 0x000100; }

}  // extern "C"
