// alg.cuh -- part of libpolsar.so (B200, sm_100a); arXiv 1807.08084.
// Layout, ownership and error conventions: include/polsar.h.  Design notes:
// DESIGN.md.  Nothing here is shared with oracle/.
//
// The per-matrix device functions of the method: Alg. 2 (plain and
// error-free-transformation forms), Alg. 1 (l21 corrected), and the
// status rule.  Included by the kernels of inv_det.cu and window.cu.
#pragma once
#include "common.cuh"

namespace polsar_impl {

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

// p q - x^2 - y^2 for p q >= x^2 + y^2 (a diagonal cofactor of a positive
// definite matrix: a principal 2x2 minor) to ~2u: as dot3_hi, but RN(p q) >=
// RN(x^2) lets the exact sum of the first two products use FastTwoSum.
__device__ __forceinline__ double diag_hi(double p, double q, double x, double y) {
    double p1 = __dmul_rn(p, q), e1 = __fma_rn(p, q, -p1);
    double p2 = __dmul_rn(x, x), e2 = __fma_rn(x, x, -p2);
    double s = __dsub_rn(p1, p2);
    double t = __dsub_rn(__dsub_rn(p1, s), p2);  // FastTwoSum error of p1 - p2
    double r = __fma_rn(-y, y, s);
    return __dadd_rn(r, __dadd_rn(__dsub_rn(e1, e2), t));
}

// Alg. 2 with every cofactor to ~2u (FMA two-products and one exact sum per
// 3-term cofactor) and the step-2 determinant as a compensated dot over
// (x_k, c_k): the cofactors' own ~2u errors, amplified by the row-0
// expansion's condition (~kappa), are what is left.  Measured on c4's law
// (tools/forms/f64_forms.py, host emulation): <= 2.5e-13 at kappa <= 1e4,
// 6.3e-13 on matrices with kappa = 1e4 exactly; ~171 FP64 operations per
// matrix against the error-free form's ~255, which on full-size c4 is the
// difference between 99 % and 103 % of the HBM copy peak.  POLSAR_F64.
__device__ __forceinline__ void alg2_comp(const H9<double>& m, double* o, double& det, double& t) {
    // step 1 (Eq. 3)
    const double ai = diag_hi(m.d, m.f, m.er, m.ei);
    const double bir = dot3_hi(m.cr, m.er, m.ci, m.ei, -m.br, m.f);
    const double bii = dot3_hi(m.ci, m.er, -m.cr, m.ei, -m.bi, m.f);
    const double cir = dot3_hi(m.br, m.er, -m.bi, m.ei, -m.cr, m.d);
    const double cii = dot3_hi(m.br, m.ei, m.bi, m.er, -m.ci, m.d);
    const double di = diag_hi(m.a, m.f, m.cr, m.ci);
    const double eir = dot3_hi(m.cr, m.br, m.ci, m.bi, -m.a, m.er);
    const double eii = dot3_hi(m.ci, m.br, -m.cr, m.bi, -m.a, m.ei);
    const double fi = diag_hi(m.a, m.d, m.br, m.bi);
    // step 2 (Eq. 6), compensated
    double p0 = __dmul_rn(m.a, ai), q0 = __fma_rn(m.a, ai, -p0);
    double p1 = __dmul_rn(m.br, bir), q1 = __fma_rn(m.br, bir, -p1);
    double p2 = __dmul_rn(m.bi, bii), q2 = __fma_rn(m.bi, bii, -p2);
    double p3 = __dmul_rn(m.cr, cir), q3 = __fma_rn(m.cr, cir, -p3);
    double p4 = __dmul_rn(m.ci, cii), q4 = __fma_rn(m.ci, cii, -p4);
    double s, r1, r2, r3, r4;
    two_sum(p0, p1, s, r1);
    two_sum(s, p2, s, r2);
    two_sum(s, p3, s, r3);
    two_sum(s, p4, s, r4);
    double err = __dadd_rn(__dadd_rn(__dadd_rn(q0, q1), __dadd_rn(q2, q3)),
                           __dadd_rn(q4, __dadd_rn(__dadd_rn(r1, r2), __dadd_rn(r3, r4))));
    det = __dadd_rn(s, err);
    // step 3
    t = __drcp_rn(det);
    // step 4
    o[0] = __dmul_rn(t, ai);
    o[1] = __dmul_rn(t, bir);
    o[2] = __dmul_rn(t, bii);
    o[3] = __dmul_rn(t, cir);
    o[4] = __dmul_rn(t, cii);
    o[5] = __dmul_rn(t, di);
    o[6] = __dmul_rn(t, eir);
    o[7] = __dmul_rn(t, eii);
    o[8] = __dmul_rn(t, fi);
}

// Alg. 2 with the five cofactors that enter Eq. 6 carried as hi + lo, the
// other four to ~2u (dot3_hi), and the step-2 determinant summed with Dot2
// over (x_k, hi_k) plus the x_k lo_k terms: det and every inverse entry come
// out within a few ulp, independent of the cancellation (the plain form loses
// ~kappa^2 u for matrices with one dominant eigenvalue).  POLSAR_F64_EFT.
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
enum { MATH_F64 = 0, MATH_F64_COMP = 1, MATH_F32 = 2, MATH_F64_EFT = 3 };

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
        else if constexpr (MATH == MATH_F64_COMP)
            alg2_comp(m, o, det, t);
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

}  // namespace polsar_impl
