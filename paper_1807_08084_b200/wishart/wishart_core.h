/*
 * wishart_core.h -- seeded, counter-based generator of multilook PolSAR
 * covariance matrices (SUPPORT, untimed).  Compiled twice from this one
 * header: by nvcc into libpolsar_gen.so (GPU) and by gcc into
 * libpolsar_gen_cpu.so (host twin).  Both builds disable FMA contraction
 * (-fmad=false / -ffp-contract=off) and use only IEEE-754 correctly rounded
 * operations (+ - * / sqrt, and explicit fma), so the two produce
 * bit-identical matrices for the same (seed, pixel) -- the host twin lets
 * tests regenerate any sampled pixel of a 4e8-pixel image independently.
 *
 * This module holds none of the method's arithmetic (no inverse, no
 * determinant); it is the input generator that the CUDA path and the oracle
 * both consume.
 *
 * Model (Eq. (2) [§I], read as Z = (1/L) sum_l s_l s_l^H,
 * DESIGN.md reading R-3): s_l = C z_l with Sigma = C C^H (C lower
 * triangular, from a per-config table), z_l ~ CN(0, I) with Re and Im iid
 * N(0, 1/2) (reading R-9).  Normals by Box-Muller from Philox4x32-10
 * (Salmon et al., SC'11), keyed by (seed, stream), counter = (global pixel,
 * look, draw).  Mode PAPER_SIM is the paper's simulated law (PAPER.md:715-723
 * [§IV-B1]): G with Re/Im uniform on [-1, 1], Z = G G^H.
 */
#ifndef POLSAR_WISHART_CORE_H
#define POLSAR_WISHART_CORE_H

#include <stdint.h>

#ifdef __CUDACC__
#define WG_FN static __host__ __device__ __forceinline__
#else
#define WG_FN static inline
#include <math.h>
#include <string.h>
#endif

enum {
    WG_MODE_SINGLE = 0,    /* one Sigma for the whole image (c1)              */
    WG_MODE_QUADRANT = 1,  /* table[2*(y >= H/2) + (x >= W/2)] (c2)           */
    WG_MODE_ROW = 2,       /* table[y], y the global row (c3, c4)              */
    WG_MODE_CHECKER = 3,   /* table[((y>>6) + (x>>6)) & 7], 64-px tiles (c5)   */
    WG_MODE_PAPER_SIM = 4  /* G G^H, Re/Im(G) ~ U[-1, 1]    */
};

typedef struct {
    uint64_t seed;
    uint32_t stream;
    int32_t looks;
    int32_t mode;
    int64_t height, width;
    const double* table;      /* n_table x 9 doubles: c00, Re c10, Im c10, c11,
                                 Re c20, Im c20, Re c21, Im c21, c22          */
    int64_t n_table;
    uint32_t near_singular_threshold; /* pixel replaced iff u32 < threshold   */
} wg_params;

/* ----------------------------------------------------------- Philox4x32-10 */
WG_FN void wg_mulhilo(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

WG_FN void wg_philox(const uint32_t ctr_in[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        wg_mulhilo(0xD2511F53u, c0, &hi0, &lo0);
        wg_mulhilo(0xCD9E8D57u, c2, &hi1, &lo1);
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 53-bit uniform in (0, 1]: (x + 1) 2^-53, exact. */
WG_FN double wg_u53(uint32_t hi, uint32_t lo) {
    uint64_t x = ((uint64_t)hi << 21) | (uint64_t)(lo >> 11);
    return (double)(x + 1) * 1.1102230246251565404236316680908203125e-16;
}

/* --------------------------------------------- deterministic elementary fns */
WG_FN uint64_t wg_bits(double x) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t b;
    memcpy(&b, &x, 8);
    return b;
#endif
}

WG_FN double wg_from_bits(uint64_t b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)b);
#else
    double x;
    memcpy(&x, &b, 8);
    return x;
#endif
}

/* natural log for x in (0, 1] (normal numbers); atanh series, |err| ~ 1 ulp */
WG_FN double wg_log(double x) {
    uint64_t b = wg_bits(x);
    int e = (int)((b >> 52) & 0x7ff) - 1023;
    double m = wg_from_bits((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull);
    if (m > 1.4142135623730951) { m = m * 0.5; e += 1; }
    double s = (m - 1.0) / (m + 1.0);
    double s2 = s * s;
    double p = 0.04;                                   /* 1/25 */
    p = fma(p, s2, 0.043478260869565216);              /* 1/23 */
    p = fma(p, s2, 0.047619047619047616);              /* 1/21 */
    p = fma(p, s2, 0.052631578947368418);              /* 1/19 */
    p = fma(p, s2, 0.058823529411764705);              /* 1/17 */
    p = fma(p, s2, 0.066666666666666666);              /* 1/15 */
    p = fma(p, s2, 0.076923076923076927);              /* 1/13 */
    p = fma(p, s2, 0.090909090909090912);              /* 1/11 */
    p = fma(p, s2, 0.11111111111111110);               /* 1/9  */
    p = fma(p, s2, 0.14285714285714285);               /* 1/7  */
    p = fma(p, s2, 0.20000000000000001);               /* 1/5  */
    p = fma(p, s2, 0.33333333333333331);               /* 1/3  */
    double lnm = 2.0 * s + 2.0 * s * s2 * p;
    double ed = (double)e;
    return fma(ed, 6.93147180369123816490e-01, fma(ed, 1.90821492927058770002e-10, lnm));
}

/* (cos, sin)(2 pi u) for u in [0, 1): quadrant split, Taylor on [0, pi/2) */
WG_FN void wg_cossin_2pi(double u, double* c_out, double* s_out) {
    double t = u * 4.0;
    int q = (int)t;
    double f = t - (double)q;
    double ph = f * 1.5707963267948966;
    double p2 = ph * ph;
    /* sin: ph * (1 - p2/3! + p2^2/5! - ... ) up to ph^21 */
    double sp = -1.9572941063391263e-20;               /* -1/21! */
    sp = fma(sp, p2, 8.2206352466243295e-18);          /*  1/19! */
    sp = fma(sp, p2, -2.8114572543455206e-15);         /* -1/17! */
    sp = fma(sp, p2, 7.6471637318198164e-13);          /*  1/15! */
    sp = fma(sp, p2, -1.6059043836821613e-10);         /* -1/13! */
    sp = fma(sp, p2, 2.5052108385441720e-08);          /*  1/11! */
    sp = fma(sp, p2, -2.7557319223985893e-06);         /* -1/9!  */
    sp = fma(sp, p2, 1.9841269841269841e-04);          /*  1/7!  */
    sp = fma(sp, p2, -8.3333333333333332e-03);         /* -1/5!  */
    sp = fma(sp, p2, 1.6666666666666666e-01);          /*  1/3!  */
    double sn = fma(-ph * p2, sp, ph);
    /* cos: 1 - p2/2! + p2^2/4! - ... up to ph^22 */
    double cp = -8.8967913924505741e-22;               /* -1/22! */
    cp = fma(cp, p2, 4.1103176233121648e-19);          /*  1/20! */
    cp = fma(cp, p2, -1.5619206968586225e-16);         /* -1/18! */
    cp = fma(cp, p2, 4.7794773323873853e-14);          /*  1/16! */
    cp = fma(cp, p2, -1.1470745597729725e-11);         /* -1/14! */
    cp = fma(cp, p2, 2.0876756987868100e-09);          /*  1/12! */
    cp = fma(cp, p2, -2.7557319223985888e-07);         /* -1/10! */
    cp = fma(cp, p2, 2.4801587301587302e-05);          /*  1/8!  */
    cp = fma(cp, p2, -1.3888888888888889e-03);         /* -1/6!  */
    cp = fma(cp, p2, 4.1666666666666664e-02);          /*  1/4!  */
    cp = fma(cp, p2, -0.5);                            /* -1/2!  */
    double cs = fma(p2, cp, 1.0);
    switch (q & 3) {
        case 0: *c_out = cs;  *s_out = sn;  break;
        case 1: *c_out = -sn; *s_out = cs;  break;
        case 2: *c_out = -cs; *s_out = -sn; break;
        default: *c_out = sn; *s_out = -cs; break;
    }
}

/* 2^x for x in [-1000, 0]: integer split, Taylor of e^(f ln 2) on [0, ln 2) */
WG_FN double wg_exp2(double x) {
    double k = floor(x);
    double f = x - k;
    double y = f * 0.69314718055994531;
    double p = 4.1103176233121648e-19;                 /* 1/20! */
    p = fma(p, y, 8.2206352466243295e-18);             /* 1/19! */
    p = fma(p, y, 1.5619206968586225e-16);             /* 1/18! */
    p = fma(p, y, 2.8114572543455206e-15);             /* 1/17! */
    p = fma(p, y, 4.7794773323873853e-14);             /* 1/16! */
    p = fma(p, y, 7.6471637318198164e-13);             /* 1/15! */
    p = fma(p, y, 1.1470745597729725e-11);             /* 1/14! */
    p = fma(p, y, 1.6059043836821613e-10);             /* 1/13! */
    p = fma(p, y, 2.0876756987868100e-09);             /* 1/12! */
    p = fma(p, y, 2.5052108385441720e-08);             /* 1/11! */
    p = fma(p, y, 2.7557319223985888e-07);             /* 1/10! */
    p = fma(p, y, 2.7557319223985893e-06);             /* 1/9!  */
    p = fma(p, y, 2.4801587301587302e-05);             /* 1/8!  */
    p = fma(p, y, 1.9841269841269841e-04);             /* 1/7!  */
    p = fma(p, y, 1.3888888888888889e-03);             /* 1/6!  */
    p = fma(p, y, 8.3333333333333332e-03);             /* 1/5!  */
    p = fma(p, y, 4.1666666666666664e-02);             /* 1/4!  */
    p = fma(p, y, 1.6666666666666666e-01);             /* 1/3!  */
    p = fma(p, y, 0.5);                                /* 1/2!  */
    p = fma(p, y, 1.0);
    p = fma(p, y, 1.0);
    int ki = (int)k;
    if (ki < -1022) { p = p * wg_from_bits((uint64_t)(ki + 1022 + 1023) << 52); ki = -1022; }
    return p * wg_from_bits((uint64_t)(ki + 1023) << 52);
}

/* ---------------------------------------------------------- random draws */
typedef struct { double re, im; } wg_cx;

WG_FN void wg_draw(const wg_params* P, uint64_t pix, uint32_t look, uint32_t draw, uint32_t out[4]) {
    uint32_t ctr[4] = {(uint32_t)pix, (uint32_t)(pix >> 32), look, draw};
    wg_philox(ctr, (uint32_t)P->seed ^ P->stream, (uint32_t)(P->seed >> 32), out);
}

/* one circular complex normal CN(0, 1): Re, Im iid N(0, 1/2) (Box-Muller) */
WG_FN wg_cx wg_cnormal(const wg_params* P, uint64_t pix, uint32_t look, uint32_t draw) {
    uint32_t r[4];
    wg_draw(P, pix, look, draw, r);
    double u1 = wg_u53(r[0], r[1]);
    double u2 = wg_u53(r[2], r[3]) - 1.1102230246251565404236316680908203125e-16; /* [0,1) */
    double rad = sqrt(-wg_log(u1));
    double c, s;
    wg_cossin_2pi(u2, &c, &s);
    wg_cx z;
    z.re = rad * c;
    z.im = rad * s;
    return z;
}

WG_FN double wg_uniform(const wg_params* P, uint64_t pix, uint32_t look, uint32_t draw, int half) {
    uint32_t r[4];
    wg_draw(P, pix, look, draw, r);
    return half ? wg_u53(r[2], r[3]) : wg_u53(r[0], r[1]);
}

/* Accumulator for Z = sum_k w_k v_k v_k^H (upper triangle, 9 reals). */
typedef struct { double a, br, bi, cr, ci, d, er, ei, f; } wg_herm;

WG_FN void wg_rank1_add(wg_herm* z, wg_cx s0, wg_cx s1, wg_cx s2, double w) {
    /* a += w|s0|^2, b += w s0 conj(s1), c += w s0 conj(s2), d += w|s1|^2,
       e += w s1 conj(s2), f += w|s2|^2 */
    z->a  += w * (s0.re * s0.re + s0.im * s0.im);
    z->br += w * (s0.re * s1.re + s0.im * s1.im);
    z->bi += w * (s0.im * s1.re - s0.re * s1.im);
    z->cr += w * (s0.re * s2.re + s0.im * s2.im);
    z->ci += w * (s0.im * s2.re - s0.re * s2.im);
    z->d  += w * (s1.re * s1.re + s1.im * s1.im);
    z->er += w * (s1.re * s2.re + s1.im * s2.im);
    z->ei += w * (s1.im * s2.re - s1.re * s2.im);
    z->f  += w * (s2.re * s2.re + s2.im * s2.im);
}

WG_FN int64_t wg_table_index(const wg_params* P, int64_t y, int64_t x) {
    switch (P->mode) {
        case WG_MODE_QUADRANT: return 2 * (y >= P->height / 2) + (x >= P->width / 2);
        case WG_MODE_ROW: return y;
        case WG_MODE_CHECKER: return ((y >> 6) + (x >> 6)) & 7;
        default: return 0;
    }
}

/* Haar unitary Q by Gram-Schmidt of three CN(0, I) columns; returns Z =
   Q diag(lam) Q^H.  Used for the c4 near-singular pixels (kappa = 1e6). */
WG_FN wg_herm wg_near_singular(const wg_params* P, uint64_t pix) {
    wg_cx v[3][3];
    for (int k = 0; k < 3; ++k)
        for (int i = 0; i < 3; ++i)
            v[k][i] = wg_cnormal(P, pix, 0xFFFFFFFEu, (uint32_t)(3 * k + i));
    for (int k = 0; k < 3; ++k) {
        for (int j = 0; j < k; ++j) {
            /* v_k -= (q_j^H v_k) q_j */
            double pr = 0.0, pi = 0.0;
            for (int i = 0; i < 3; ++i) {
                pr += v[j][i].re * v[k][i].re + v[j][i].im * v[k][i].im;
                pi += v[j][i].re * v[k][i].im - v[j][i].im * v[k][i].re;
            }
            for (int i = 0; i < 3; ++i) {
                v[k][i].re -= pr * v[j][i].re - pi * v[j][i].im;
                v[k][i].im -= pr * v[j][i].im + pi * v[j][i].re;
            }
        }
        double nrm = 0.0;
        for (int i = 0; i < 3; ++i) nrm += v[k][i].re * v[k][i].re + v[k][i].im * v[k][i].im;
        double inv = 1.0 / sqrt(nrm);
        for (int i = 0; i < 3; ++i) { v[k][i].re *= inv; v[k][i].im *= inv; }
    }
    /* mu log-uniform on [1e-6, 1]: mu = 2^(-6 log2(10) u) */
    double u = wg_uniform(P, pix, 0xFFFFFFFDu, 0, 0);
    double mu = wg_exp2(-19.931568569324174 * u);
    wg_herm z = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    wg_rank1_add(&z, v[0][0], v[0][1], v[0][2], 1.0);
    wg_rank1_add(&z, v[1][0], v[1][1], v[1][2], mu);
    wg_rank1_add(&z, v[2][0], v[2][1], v[2][2], 1e-6);
    return z;
}

/* The matrix of global pixel (y, x). */
WG_FN wg_herm wg_pixel(const wg_params* P, int64_t y, int64_t x) {
    uint64_t pix = (uint64_t)(y * P->width + x);
    wg_herm z = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (P->mode == WG_MODE_PAPER_SIM) {
        /* G with Re, Im ~ U[-1, 1]; Z = G G^H (rows g_i: Z_ij = g_i . conj(g_j)) */
        wg_cx g[3][3];
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k) {
                uint32_t r[4];
                wg_draw(P, pix, 0, (uint32_t)(3 * i + k), r);
                g[i][k].re = 2.0 * wg_u53(r[0], r[1]) - 1.0;
                g[i][k].im = 2.0 * wg_u53(r[2], r[3]) - 1.0;
            }
        /* G G^H = sum_k (column k)(column k)^H */
        for (int k = 0; k < 3; ++k) wg_rank1_add(&z, g[0][k], g[1][k], g[2][k], 1.0);
        return z;
    }
    if (P->near_singular_threshold) {
        uint32_t r[4];
        wg_draw(P, pix, 0xFFFFFFFFu, 0, r);
        if (r[0] < P->near_singular_threshold) return wg_near_singular(P, pix);
    }
    const double* C = P->table + 9 * wg_table_index(P, y, x);
    for (int l = 0; l < P->looks; ++l) {
        wg_cx z0 = wg_cnormal(P, pix, (uint32_t)l, 0);
        wg_cx z1 = wg_cnormal(P, pix, (uint32_t)l, 1);
        wg_cx z2 = wg_cnormal(P, pix, (uint32_t)l, 2);
        /* s = C z, C lower triangular */
        wg_cx s0, s1, s2;
        s0.re = C[0] * z0.re;
        s0.im = C[0] * z0.im;
        s1.re = (C[1] * z0.re - C[2] * z0.im) + C[3] * z1.re;
        s1.im = (C[1] * z0.im + C[2] * z0.re) + C[3] * z1.im;
        s2.re = ((C[4] * z0.re - C[5] * z0.im) + (C[6] * z1.re - C[7] * z1.im)) + C[8] * z2.re;
        s2.im = ((C[4] * z0.im + C[5] * z0.re) + (C[6] * z1.im + C[7] * z1.re)) + C[8] * z2.im;
        wg_rank1_add(&z, s0, s1, s2, 1.0);
    }
    double invl = 1.0 / (double)P->looks;
    z.a *= invl; z.br *= invl; z.bi *= invl; z.cr *= invl; z.ci *= invl;
    z.d *= invl; z.er *= invl; z.ei *= invl; z.f *= invl;
    return z;
}

#endif /* POLSAR_WISHART_CORE_H */
