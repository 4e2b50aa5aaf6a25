/* f64_forms.c -- host emulation of candidate fp64 evaluations of Alg. 2
 * for the K1 POLSAR_F64 mode, to choose the cheapest form
 * that holds BASELINE's 1e-12 (R-16).  IEEE double with explicit
 * fma() and -ffp-contract=off reproduces the device's __dmul_rn / __dadd_rn /
 * __fma_rn / __drcp_rn bit for bit.  Development tool: not part of the
 * product, never linked into libpolsar.so.
 *   form 0: the round-1 error-free form (5 Dot2 cofactors as hi+lo, 4 at ~2u,
 *           compensated Eq. 6)
 *   form 1: 9 cofactors at ~2u (dot3_hi; the diagonal ones with FastTwoSum),
 *           Eq. 6 as a plain FMA chain
 *   form 2: as 1, Eq. 6 compensated (TwoProd + TwoSum cascade)
 *   form 3: plain Alg. 2 (FMA, as printed)
 *   form 4: as 2, diagonal cofactors through dot3_hi too (no FastTwoSum)
 */
#include <math.h>
#include <stdint.h>

typedef struct { double hi, lo; } dd;
static int nops;  /* FP64 operations of the last form evaluated (one matrix) */
#define OP(x) (nops++, (x))
static double mul(double a, double b) { return OP(a * b); }
static double add(double a, double b) { return OP(a + b); }
static double sub(double a, double b) { return OP(a - b); }
static double fm(double a, double b, double c) { return OP(fma(a, b, c)); }

static void two_sum(double a, double b, double* s, double* e) {
    *s = add(a, b);
    double bb = sub(*s, a);
    *e = add(sub(a, sub(*s, bb)), sub(b, bb));
}
static void fast_two_sum(double a, double b, double* s, double* e) {  /* |a| >= |b| */
    *s = add(a, b);
    *e = sub(b, sub(*s, a));
}
static dd dot3(double x1, double y1, double x2, double y2, double x3, double y3) {
    double p1 = mul(x1, y1), e1 = fm(x1, y1, -p1);
    double p2 = mul(x2, y2), e2 = fm(x2, y2, -p2);
    double p3 = mul(x3, y3), e3 = fm(x3, y3, -p3);
    double s, t1, s2, t2;
    two_sum(p1, p2, &s, &t1);
    two_sum(s, p3, &s2, &t2);
    double lo = add(add(e1, e2), add(e3, add(t1, t2)));
    dd r;
    two_sum(s2, lo, &r.hi, &r.lo);
    return r;
}
static double dot3_hi(double x1, double y1, double x2, double y2, double x3, double y3) {
    double p1 = mul(x1, y1), e1 = fm(x1, y1, -p1);
    double p2 = mul(x2, y2), e2 = fm(x2, y2, -p2);
    double s, t;
    two_sum(p1, p2, &s, &t);
    double r = fm(x3, y3, s);
    return add(r, add(add(e1, e2), t));
}
/* p*q - x^2 - y^2 with p*q >= x^2 (a diagonal cofactor of a PD matrix) */
static double diag_hi(double p, double q, double x, double y) {
    double p1 = mul(p, q), e1 = fm(p, q, -p1);
    double p2 = mul(x, x), e2 = fm(x, x, -p2);
    double s, t;
    fast_two_sum(p1, -p2, &s, &t);
    double r = fm(-y, y, s);
    return add(r, add(sub(e1, e2), t));
}

void form_eval(int form, const double* z, int64_t ld, double* out, int64_t ldo, int64_t n, int* ops) {
    for (int64_t p = 0; p < n; ++p) {
        double a = z[p], br = z[ld + p], bi = z[2 * ld + p], cr = z[3 * ld + p], ci = z[4 * ld + p];
        double d = z[5 * ld + p], er = z[6 * ld + p], ei = z[7 * ld + p], f = z[8 * ld + p];
        double c[9], det;
        nops = 0;
        if (form == 0) {
            dd ai = dot3(d, f, -er, er, -ei, ei), bir = dot3(cr, er, ci, ei, -br, f);
            dd bii = dot3(ci, er, -cr, ei, -bi, f), cir = dot3(br, er, -bi, ei, -cr, d);
            dd cii = dot3(br, ei, bi, er, -ci, d);
            c[5] = dot3_hi(-cr, cr, -ci, ci, a, f);
            c[6] = dot3_hi(cr, br, ci, bi, -a, er);
            c[7] = dot3_hi(ci, br, -cr, bi, -a, ei);
            c[8] = dot3_hi(-br, br, -bi, bi, a, d);
            double x[5] = {a, br, bi, cr, ci};
            dd h[5] = {ai, bir, bii, cir, cii};
            double s = 0, err = 0;
            for (int k = 0; k < 5; ++k) {
                double pk = mul(x[k], h[k].hi), qk = fm(x[k], h[k].hi, -pk);
                if (k == 0) s = pk; else { double r; two_sum(s, pk, &s, &r); err = add(err, r); }
                err = add(err, qk);
            }
            for (int k = 0; k < 5; ++k) err = fm(x[k], h[k].lo, err);
            det = add(s, err);
            for (int k = 0; k < 5; ++k) c[k] = h[k].hi;
        } else if (form == 3) {
            c[0] = fm(d, f, -fm(er, er, mul(ei, ei)));
            c[1] = fm(cr, er, fm(ci, ei, -mul(br, f)));
            c[2] = fm(ci, er, -fm(cr, ei, mul(bi, f)));
            c[3] = fm(br, er, -fm(bi, ei, mul(cr, d)));
            c[4] = fm(br, ei, fm(bi, er, -mul(ci, d)));
            c[5] = fm(a, f, -fm(cr, cr, mul(ci, ci)));
            c[6] = fm(cr, br, fm(ci, bi, -mul(a, er)));
            c[7] = fm(ci, br, -fm(cr, bi, mul(a, ei)));
            c[8] = fm(a, d, -fm(br, br, mul(bi, bi)));
            det = fm(a, c[0], fm(br, c[1], fm(bi, c[2], fm(cr, c[3], mul(ci, c[4])))));
        } else {
            if (form == 4) {
                c[0] = dot3_hi(-er, er, -ei, ei, d, f);
                c[5] = dot3_hi(-cr, cr, -ci, ci, a, f);
                c[8] = dot3_hi(-br, br, -bi, bi, a, d);
            } else {
                c[0] = diag_hi(d, f, er, ei);
                c[5] = diag_hi(a, f, cr, ci);
                c[8] = diag_hi(a, d, br, bi);
            }
            c[1] = dot3_hi(cr, er, ci, ei, -br, f);
            c[2] = dot3_hi(ci, er, -cr, ei, -bi, f);
            c[3] = dot3_hi(br, er, -bi, ei, -cr, d);
            c[4] = dot3_hi(br, ei, bi, er, -ci, d);
            c[6] = dot3_hi(cr, br, ci, bi, -a, er);
            c[7] = dot3_hi(ci, br, -cr, bi, -a, ei);
            if (form == 1) {
                det = fm(a, c[0], fm(br, c[1], fm(bi, c[2], fm(cr, c[3], mul(ci, c[4])))));
            } else {
                double x[5] = {a, br, bi, cr, ci};
                double s = 0, err = 0;
                for (int k = 0; k < 5; ++k) {
                    double pk = mul(x[k], c[k]), qk = fm(x[k], c[k], -pk);
                    if (k == 0) s = pk; else { double r; two_sum(s, pk, &s, &r); err = add(err, r); }
                    err = add(err, qk);
                }
                det = add(s, err);
            }
        }
        double t = OP(1.0 / det);
        for (int k = 0; k < 9; ++k) out[k * ldo + p] = mul(t, c[k]);
        out[9 * ldo + p] = det;
        out[10 * ldo + p] = t;
        *ops = nops;
    }
}
