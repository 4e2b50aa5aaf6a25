/*
 * polsar_oracle.c -- CPU ORACLE for arXiv 1807.08084 (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library (the latter two time the storage-
 * precision instantiation at the end of this file).  The product path
 * (paper_1807_08084_b200/) never links, imports or calls it, and this file
 * shares no code, header, table or constant with the CUDA path.
 *
 * Everything here is the plain definition, evaluated in extended precision
 * (binary128 `__float128` for the inverse/det oracle, x87 `long double` for
 * the window oracle) from the exactly upcast inputs and rounded once to
 * double on output.  Each function cites the passage it follows
 * (PAPER.md line numbers; section / equation / algorithm in brackets).
 *
 * Packed Hermitian layout (PAPER.md:136-153 [§II-A]): a, d, f real; b, c, e
 * complex; A = [[a, b, c], [conj b, d, e], [conj c, conj e, f]].  Inputs are
 * 9 planes (structure of arrays, plane stride `ld`) in the field order
 *     0 a, 1 Re b, 2 Im b, 3 Re c, 4 Im c, 5 d, 6 Re e, 7 Im e, 8 f.
 *
 * Pins (tests/test_oracle.py, `-m "not gpu"`): identity, diagonal and
 * block-diagonal closed forms; the golden matrix (tests/golden/); exact
 * rational Gauss-Jordan on random inputs; numpy/LAPACK special case;
 * Z*Z^-1 = I by an independent dense multiply; det(2^m Z) = 2^{3m} det Z.
 * The window oracle is pinned by the constant-image closed form (W_i =
 * clipped window count), the two-class closed form, d_ii = 0, d_ij = d_ji,
 * and a brute-force Python evaluation on tiny images.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

typedef long double ld_t;   /* window oracle: 64-bit mantissa          */
typedef __float128  q_t;    /* inverse/det oracle: 113-bit mantissa    */

/* ---------------------------------------------------------------------------
 * Cofactors of the packed Hermitian matrix: Eq. (3)
 * [§II-A]:
 *   a_c = d f - |e|^2,  b_c = c conj(e) - b f,  c_c = b e - c d,
 *   d_c = a f - |c|^2,  e_c = c conj(b) - a e,  f_c = a d - |b|^2.
 * (The adjoint's (i,j) entry is the cofactor of A's (j,i) entry.)
 *
 * Determinant by the row-0 cofactor expansion, the FULL complex form of
 * Eq. (5), PAPER.md:399-409 [§III-A]:  det A = a a_c + conj(b) b_c + conj(c) c_c.
 * The real part is det A; the imaginary part must vanish for Hermitian A
 * and is returned for checking.
 *
 * Written once as a macro and instantiated in two evaluation types.  The
 * cofactor expansion's rounding error grows like kappa^2 * u for matrices
 * with one dominant eigenvalue ("oracle precision"), so the
 * inverse/det oracle runs in binary128 (u = 2^-113), which keeps the oracle's
 * own error below 1e-25 at kappa = 1e4; the window oracle, compared at 2e-5,
 * runs in x87 long double.
 * ------------------------------------------------------------------------- */
#define DEFINE_HERM(T, SFX)                                                   \
typedef struct { T a, br, bi, cr, ci, d, er, ei, f; } herm_##SFX;            \
                                                                              \
static herm_##SFX load_##SFX##_f64(const double* z, int64_t ld, int64_t p) { \
    herm_##SFX m;                                                             \
    m.a  = (T)z[0 * ld + p]; m.br = (T)z[1 * ld + p];                        \
    m.bi = (T)z[2 * ld + p]; m.cr = (T)z[3 * ld + p];                        \
    m.ci = (T)z[4 * ld + p]; m.d  = (T)z[5 * ld + p];                        \
    m.er = (T)z[6 * ld + p]; m.ei = (T)z[7 * ld + p];                        \
    m.f  = (T)z[8 * ld + p];                                                  \
    return m;                                                                 \
}                                                                             \
static herm_##SFX load_##SFX##_f32(const float* z, int64_t ld, int64_t p) {  \
    herm_##SFX m;                                                             \
    m.a  = (T)z[0 * ld + p]; m.br = (T)z[1 * ld + p];                        \
    m.bi = (T)z[2 * ld + p]; m.cr = (T)z[3 * ld + p];                        \
    m.ci = (T)z[4 * ld + p]; m.d  = (T)z[5 * ld + p];                        \
    m.er = (T)z[6 * ld + p]; m.ei = (T)z[7 * ld + p];                        \
    m.f  = (T)z[8 * ld + p];                                                  \
    return m;                                                                 \
}                                                                             \
static herm_##SFX cofactors_##SFX(herm_##SFX m) {                            \
    herm_##SFX c;                                                             \
    /* a_c = d*f - |e|^2 */                                                   \
    c.a = m.d * m.f - (m.er * m.er + m.ei * m.ei);                            \
    /* b_c = c*conj(e) - b*f */                                               \
    c.br = (m.cr * m.er + m.ci * m.ei) - m.br * m.f;                          \
    c.bi = (m.ci * m.er - m.cr * m.ei) - m.bi * m.f;                          \
    /* c_c = b*e - c*d */                                                     \
    c.cr = (m.br * m.er - m.bi * m.ei) - m.cr * m.d;                          \
    c.ci = (m.br * m.ei + m.bi * m.er) - m.ci * m.d;                          \
    /* d_c = a*f - |c|^2 */                                                   \
    c.d = m.a * m.f - (m.cr * m.cr + m.ci * m.ci);                            \
    /* e_c = c*conj(b) - a*e */                                               \
    c.er = (m.cr * m.br + m.ci * m.bi) - m.a * m.er;                          \
    c.ei = (m.ci * m.br - m.cr * m.bi) - m.a * m.ei;                          \
    /* f_c = a*d - |b|^2 */                                                   \
    c.f = m.a * m.d - (m.br * m.br + m.bi * m.bi);                            \
    return c;                                                                 \
}                                                                             \
static void det_full_##SFX(herm_##SFX m, herm_##SFX c, T* re, T* im) {       \
    /* conj(b)*b_c = (br - i bi)(bcr + i bci);  conj(c)*c_c likewise */       \
    T t1r = m.br * c.br + m.bi * c.bi;                                        \
    T t1i = m.br * c.bi - m.bi * c.br;                                        \
    T t2r = m.cr * c.cr + m.ci * c.ci;                                        \
    T t2i = m.cr * c.ci - m.ci * c.cr;                                        \
    *re = m.a * c.a + t1r + t2r;                                              \
    *im = t1i + t2i;                                                          \
}

DEFINE_HERM(q_t, q)
DEFINE_HERM(ld_t, ld)

static void store_inv(double* out, int64_t ldo, int64_t p, herm_q c, q_t det,
                      double* det_imag, q_t im) {
    /* Eq. (4), PAPER.md:390-397 [§III-A]: A^-1 = adj(A) / det A, every entry
     * divided (the plain definition; Alg. 2's t = 1/det scaling is the
     * kernel's business, not the oracle's). */
    out[0 * ldo + p]  = (double)(c.a / det);
    out[1 * ldo + p]  = (double)(c.br / det);
    out[2 * ldo + p]  = (double)(c.bi / det);
    out[3 * ldo + p]  = (double)(c.cr / det);
    out[4 * ldo + p]  = (double)(c.ci / det);
    out[5 * ldo + p]  = (double)(c.d / det);
    out[6 * ldo + p]  = (double)(c.er / det);
    out[7 * ldo + p]  = (double)(c.ei / det);
    out[8 * ldo + p]  = (double)(c.f / det);
    /* det Z and det Z^-1 = 1/det Z (PAPER.md:66-76 [§I], 460-468 [§III-A]). */
    out[9 * ldo + p]  = (double)det;
    out[10 * ldo + p] = (double)((q_t)1 / det);
    if (det_imag) det_imag[p] = (double)im;
}

/* oracle_inv_det_f64 / _f32: per pixel Z^-1 (upper triangle, 9 reals),
 * det Z and det Z^-1, for n pixels.
 *   z   : 9 planes, plane stride ldz (>= n), input dtype double / float
 *   out : 11 planes of double, plane stride ldo (>= n): planes 0..8 the
 *         inverse in the input field order, 9 det Z, 10 det Z^-1
 *   det_imag : nullable, n doubles, Im of the Eq. (5) expansion.
 * Singular inputs give inf/nan entries (no status is computed here). */
void oracle_inv_det_f64(const double* z, int64_t ldz, double* out, int64_t ldo,
                        double* det_imag, int64_t n) {
    for (int64_t p = 0; p < n; ++p) {
        herm_q m = load_q_f64(z, ldz, p);
        herm_q c = cofactors_q(m);
        q_t re, im;
        det_full_q(m, c, &re, &im);
        store_inv(out, ldo, p, c, re, det_imag, im);
    }
}

void oracle_inv_det_f32(const float* z, int64_t ldz, double* out, int64_t ldo,
                        double* det_imag, int64_t n) {
    for (int64_t p = 0; p < n; ++p) {
        herm_q m = load_q_f32(z, ldz, p);
        herm_q c = cofactors_q(m);
        q_t re, im;
        det_full_q(m, c, &re, &im);
        store_inv(out, ldo, p, c, re, det_imag, im);
    }
}

/* Multi-frequency block-diagonal matrices (PAPER.md:1043-1055 [§V]): a pixel
 * holds nblocks Hermitian 3x3 diagonal blocks; its inverse is the block
 * diagonal of the block inverses and its determinant the product of the block
 * determinants ("obtained after applications of the proposed method to each of
 * the diagonal blocks").  z: 9*nblocks planes (block b at planes 9b..9b+8);
 * out: 9*nblocks + 2 planes (block inverses, then det and det^-1 of the whole
 * matrix).  Block values by the cofactor definition above, in binary128. */
void oracle_inv_det_blocks_f64(const double* z, int64_t ldz, int nblocks, double* out,
                               int64_t ldo, int64_t n) {
    for (int64_t p = 0; p < n; ++p) {
        q_t det_all = 1, inv_all = 1;
        for (int b = 0; b < nblocks; ++b) {
            herm_q m = load_q_f64(z + (int64_t)9 * b * ldz, ldz, p);
            herm_q c = cofactors_q(m);
            q_t re, im;
            det_full_q(m, c, &re, &im);
            double* o = out + (int64_t)9 * b * ldo;
            o[0 * ldo + p] = (double)(c.a / re);  o[1 * ldo + p] = (double)(c.br / re);
            o[2 * ldo + p] = (double)(c.bi / re); o[3 * ldo + p] = (double)(c.cr / re);
            o[4 * ldo + p] = (double)(c.ci / re); o[5 * ldo + p] = (double)(c.d / re);
            o[6 * ldo + p] = (double)(c.er / re); o[7 * ldo + p] = (double)(c.ei / re);
            o[8 * ldo + p] = (double)(c.f / re);
            det_all *= re;
            inv_all /= re;
        }
        out[((int64_t)9 * nblocks) * ldo + p] = (double)det_all;
        out[((int64_t)9 * nblocks + 1) * ldo + p] = (double)inv_all;
    }
}

void oracle_inv_det_blocks_f32(const float* z, int64_t ldz, int nblocks, double* out,
                               int64_t ldo, int64_t n) {
    for (int64_t p = 0; p < n; ++p) {
        q_t det_all = 1, inv_all = 1;
        for (int b = 0; b < nblocks; ++b) {
            herm_q m = load_q_f32(z + (int64_t)9 * b * ldz, ldz, p);
            herm_q c = cofactors_q(m);
            q_t re, im;
            det_full_q(m, c, &re, &im);
            double* o = out + (int64_t)9 * b * ldo;
            o[0 * ldo + p] = (double)(c.a / re);  o[1 * ldo + p] = (double)(c.br / re);
            o[2 * ldo + p] = (double)(c.bi / re); o[3 * ldo + p] = (double)(c.cr / re);
            o[4 * ldo + p] = (double)(c.ci / re); o[5 * ldo + p] = (double)(c.d / re);
            o[6 * ldo + p] = (double)(c.er / re); o[7 * ldo + p] = (double)(c.ei / re);
            o[8 * ldo + p] = (double)(c.f / re);
            det_all *= re;
            inv_all /= re;
        }
        out[((int64_t)9 * nblocks) * ldo + p] = (double)det_all;
        out[((int64_t)9 * nblocks + 1) * ldo + p] = (double)inv_all;
    }
}

/* ---------------------------------------------------------------------------
 * Brute force: complex Gauss-Jordan elimination with partial pivoting on the
 * full 3x3 matrix (no cofactors involved).  Independent check of the
 * cofactor oracle for tiny inputs.  Textbook algorithm (Golub & Van Loan,
 * the reference the paper cites for its matrix facts).
 *   m18 : row-major 3x3 complex matrix, (re, im) interleaved (18 doubles)
 *   inv18 : the full inverse, same layout
 *   det2 : complex determinant (product of pivots times permutation sign)
 * Returns 0, or 1 if a zero pivot was met.
 * ------------------------------------------------------------------------- */
int oracle_gauss_jordan(const double* m18, double* inv18, double* det2) {
    ld_t ar[3][6], ai[3][6];
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 6; ++k) {
            if (k < 3) {
                ar[r][k] = (ld_t)m18[2 * (3 * r + k)];
                ai[r][k] = (ld_t)m18[2 * (3 * r + k) + 1];
            } else {
                ar[r][k] = (k - 3 == r) ? 1.0L : 0.0L;
                ai[r][k] = 0.0L;
            }
        }
    ld_t dr = 1.0L, di = 0.0L;
    for (int col = 0; col < 3; ++col) {
        int piv = col;
        ld_t best = -1.0L;
        for (int r = col; r < 3; ++r) {
            ld_t mag = ar[r][col] * ar[r][col] + ai[r][col] * ai[r][col];
            if (mag > best) { best = mag; piv = r; }
        }
        if (best <= 0.0L) return 1;
        if (piv != col) {
            for (int k = 0; k < 6; ++k) {
                ld_t tr = ar[col][k], ti = ai[col][k];
                ar[col][k] = ar[piv][k]; ai[col][k] = ai[piv][k];
                ar[piv][k] = tr; ai[piv][k] = ti;
            }
            dr = -dr; di = -di;
        }
        /* det *= pivot */
        ld_t pr = ar[col][col], pi = ai[col][col];
        ld_t ndr = dr * pr - di * pi, ndi = dr * pi + di * pr;
        dr = ndr; di = ndi;
        /* row /= pivot */
        ld_t den = pr * pr + pi * pi;
        ld_t qr = pr / den, qi = -pi / den; /* 1/pivot */
        for (int k = 0; k < 6; ++k) {
            ld_t xr = ar[col][k], xi = ai[col][k];
            ar[col][k] = xr * qr - xi * qi;
            ai[col][k] = xr * qi + xi * qr;
        }
        /* eliminate the column from every other row */
        for (int r = 0; r < 3; ++r) {
            if (r == col) continue;
            ld_t fr = ar[r][col], fi = ai[r][col];
            for (int k = 0; k < 6; ++k) {
                ld_t xr = ar[col][k], xi = ai[col][k];
                ar[r][k] -= fr * xr - fi * xi;
                ai[r][k] -= fr * xi + fi * xr;
            }
        }
    }
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) {
            inv18[2 * (3 * r + k)] = (double)ar[r][k + 3];
            inv18[2 * (3 * r + k) + 1] = (double)ai[r][k + 3];
        }
    det2[0] = (double)dr;
    det2[1] = (double)di;
    return 0;
}

/* ---------------------------------------------------------------------------
 * Search-window log-det distance sum (BASELINE.json configs[4]; the NLM
 * workload of PAPER.md:77-80 [§I]).  For pixel i and every j in the
 * (2R+1)x(2R+1) window centred on i, clipped to the image (DESIGN.md
 * reading R-12):
 *   S_ij = (Z_i + Z_j) / 2,
 *   d_ij = L * [ ln det S_ij - (ln det Z_i + ln det Z_j) / 2 ],
 *   W_i  = sum_j exp(-d_ij / h).
 * det is the plain Eq. (5) expansion above, in long double.
 * ------------------------------------------------------------------------- */
static ld_t det_plain(herm_ld m) {
    ld_t re, im;
    det_full_ld(m, cofactors_ld(m), &re, &im);
    return re;
}

static herm_ld half_sum(herm_ld x, herm_ld y) {
    herm_ld s;
    s.a  = (x.a  + y.a)  / 2.0L;
    s.br = (x.br + y.br) / 2.0L;
    s.bi = (x.bi + y.bi) / 2.0L;
    s.cr = (x.cr + y.cr) / 2.0L;
    s.ci = (x.ci + y.ci) / 2.0L;
    s.d  = (x.d  + y.d)  / 2.0L;
    s.er = (x.er + y.er) / 2.0L;
    s.ei = (x.ei + y.ei) / 2.0L;
    s.f  = (x.f  + y.f)  / 2.0L;
    return s;
}

static ld_t pair_distance(herm_ld zi, herm_ld zj, ld_t looks) {
    ld_t ds = det_plain(half_sum(zi, zj));
    ld_t di = det_plain(zi), dj = det_plain(zj);
    return looks * (logl(ds) - 0.5L * (logl(di) + logl(dj)));
}

/* d_ij for two packed matrices given as 9 doubles each (field order above). */
double oracle_pair_distance(const double* zi9, const double* zj9, double looks) {
    herm_ld x = load_ld_f64(zi9, 1, 0);
    herm_ld y = load_ld_f64(zj9, 1, 0);
    return (double)pair_distance(x, y, (ld_t)looks);
}

/* W_i for the m pixels listed in idx (row-major index y*width + x) of a
 * height x width image stored as 9 double planes with stride ld. */
void oracle_window_f64(const double* z, int64_t ld, int64_t height, int64_t width,
                       int radius, double looks, double h,
                       const int64_t* idx, int64_t m, double* out) {
    for (int64_t q = 0; q < m; ++q) {
        int64_t yi = idx[q] / width, xi = idx[q] % width;
        herm_ld zi = load_ld_f64(z, ld, idx[q]);
        ld_t acc = 0.0L;
        for (int64_t yj = yi - radius; yj <= yi + radius; ++yj) {
            if (yj < 0 || yj >= height) continue;
            for (int64_t xj = xi - radius; xj <= xi + radius; ++xj) {
                if (xj < 0 || xj >= width) continue;
                herm_ld zj = load_ld_f64(z, ld, yj * width + xj);
                acc += expl(-pair_distance(zi, zj, (ld_t)looks) / (ld_t)h);
            }
        }
        out[q] = (double)acc;
    }
}

void oracle_window_f32(const float* z, int64_t ld, int64_t height, int64_t width,
                       int radius, double looks, double h,
                       const int64_t* idx, int64_t m, double* out) {
    for (int64_t q = 0; q < m; ++q) {
        int64_t yi = idx[q] / width, xi = idx[q] % width;
        herm_ld zi = load_ld_f32(z, ld, idx[q]);
        ld_t acc = 0.0L;
        for (int64_t yj = yi - radius; yj <= yi + radius; ++yj) {
            if (yj < 0 || yj >= height) continue;
            for (int64_t xj = xi - radius; xj <= xi + radius; ++xj) {
                if (xj < 0 || xj >= width) continue;
                herm_ld zj = load_ld_f32(z, ld, yj * width + xj);
                acc += expl(-pair_distance(zi, zj, (ld_t)looks) / (ld_t)h);
            }
        }
        out[q] = (double)acc;
    }
}

/* Window sum with the symmetric Wishart Kullback-Leibler distance (the
 * divergences of PAPER.md:70-76 [§I] that need Z^-1):
 *   d_ij = L [ (tr(Z_i^-1 Z_j) + tr(Z_j^-1 Z_i)) / 2 - 3 ],  W_i = sum_j exp(-d_ij / h).
 * Z^-1 by the cofactor definition (Eq. 3/4), traces by the plain definition
 * tr(X Y) = sum_k sum_l X_kl Y_lk over the full complex 3x3 matrices; long
 * double. */
typedef struct { ld_t re, im; } cld;

static void full_ld(herm_ld m, cld M[3][3]) {
    M[0][0].re = m.a;  M[0][0].im = 0;
    M[1][1].re = m.d;  M[1][1].im = 0;
    M[2][2].re = m.f;  M[2][2].im = 0;
    M[0][1].re = m.br; M[0][1].im = m.bi;  M[1][0].re = m.br; M[1][0].im = -m.bi;
    M[0][2].re = m.cr; M[0][2].im = m.ci;  M[2][0].re = m.cr; M[2][0].im = -m.ci;
    M[1][2].re = m.er; M[1][2].im = m.ei;  M[2][1].re = m.er; M[2][1].im = -m.ei;
}

static herm_ld inverse_ld(herm_ld m) {
    herm_ld c = cofactors_ld(m), x;
    ld_t re, im;
    det_full_ld(m, c, &re, &im);
    x.a = c.a / re;   x.br = c.br / re; x.bi = c.bi / re; x.cr = c.cr / re; x.ci = c.ci / re;
    x.d = c.d / re;   x.er = c.er / re; x.ei = c.ei / re; x.f = c.f / re;
    return x;
}

static ld_t trace_prod(herm_ld x, herm_ld y) {
    cld X[3][3], Y[3][3];
    full_ld(x, X);
    full_ld(y, Y);
    ld_t t = 0;  /* real part of sum_k sum_l X_kl Y_lk (the trace is real) */
    for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) t += X[k][l].re * Y[l][k].re - X[k][l].im * Y[l][k].im;
    return t;
}

static void window_kl_any(const void* z, int is32, int64_t ld, int64_t height, int64_t width,
                          int radius, double looks, double h, const int64_t* idx, int64_t m,
                          double* out) {
    for (int64_t q = 0; q < m; ++q) {
        int64_t yi = idx[q] / width, xi = idx[q] % width;
        herm_ld zi = is32 ? load_ld_f32((const float*)z, ld, idx[q]) : load_ld_f64((const double*)z, ld, idx[q]);
        herm_ld xinv = inverse_ld(zi);
        ld_t acc = 0.0L;
        for (int64_t yj = yi - radius; yj <= yi + radius; ++yj) {
            if (yj < 0 || yj >= height) continue;
            for (int64_t xj = xi - radius; xj <= xi + radius; ++xj) {
                if (xj < 0 || xj >= width) continue;
                int64_t pj = yj * width + xj;
                herm_ld zj = is32 ? load_ld_f32((const float*)z, ld, pj) : load_ld_f64((const double*)z, ld, pj);
                ld_t d = (ld_t)looks * ((trace_prod(xinv, zj) + trace_prod(inverse_ld(zj), zi)) / 2.0L - 3.0L);
                acc += expl(-d / (ld_t)h);
            }
        }
        out[q] = (double)acc;
    }
}

void oracle_window_kl_f64(const double* z, int64_t ld, int64_t height, int64_t width, int radius,
                          double looks, double h, const int64_t* idx, int64_t m, double* out) {
    window_kl_any(z, 0, ld, height, width, radius, looks, h, idx, m, out);
}

void oracle_window_kl_f32(const float* z, int64_t ld, int64_t height, int64_t width, int radius,
                          double looks, double h, const int64_t* idx, int64_t m, double* out) {
    window_kl_any(z, 1, ld, height, width, radius, looks, h, idx, m, out);
}

/* d_KL for two packed matrices (9 doubles each). */
double oracle_kl_distance(const double* zi9, const double* zj9, double looks) {
    herm_ld x = load_ld_f64(zi9, 1, 0), y = load_ld_f64(zj9, 1, 0);
    return (double)((ld_t)looks * ((trace_prod(inverse_ld(x), y) + trace_prod(inverse_ld(y), x)) / 2.0L - 3.0L));
}

/* Non-local-means filter output with the window weights (the NLM filter of
 * PAPER.md:77-80 [§I]):
 *   W_i = sum_j w_ij,  Zhat_i = sum_j w_ij Z_j / W_i,  w_ij = exp(-d_ij / h),
 * N(i) the clipped window.  Long double.  out: 10 x m doubles, row q = pixel
 * idx[q]: out[k*m + q] = Zhat_k (k < 9), out[9*m + q] = W. */
static void nlm_pixel(herm_ld zi, ld_t looks, ld_t h, const void* z, int is32, int64_t ld,
                      int64_t height, int64_t width, int radius, int64_t yi, int64_t xi,
                      ld_t acc[10]) {
    for (int k = 0; k < 10; ++k) acc[k] = 0.0L;
    for (int64_t yj = yi - radius; yj <= yi + radius; ++yj) {
        if (yj < 0 || yj >= height) continue;
        for (int64_t xj = xi - radius; xj <= xi + radius; ++xj) {
            if (xj < 0 || xj >= width) continue;
            herm_ld zj = is32 ? load_ld_f32((const float*)z, ld, yj * width + xj)
                              : load_ld_f64((const double*)z, ld, yj * width + xj);
            ld_t w = expl(-pair_distance(zi, zj, looks) / h);
            acc[0] += w * zj.a;  acc[1] += w * zj.br; acc[2] += w * zj.bi;
            acc[3] += w * zj.cr; acc[4] += w * zj.ci; acc[5] += w * zj.d;
            acc[6] += w * zj.er; acc[7] += w * zj.ei; acc[8] += w * zj.f;
            acc[9] += w;
        }
    }
}

void oracle_nlm_f64(const double* z, int64_t ld, int64_t height, int64_t width, int radius,
                    double looks, double h, const int64_t* idx, int64_t m, double* out) {
    for (int64_t q = 0; q < m; ++q) {
        ld_t acc[10];
        herm_ld zi = load_ld_f64(z, ld, idx[q]);
        nlm_pixel(zi, (ld_t)looks, (ld_t)h, z, 0, ld, height, width, radius, idx[q] / width,
                  idx[q] % width, acc);
        for (int k = 0; k < 9; ++k) out[k * m + q] = (double)(acc[k] / acc[9]);
        out[9 * m + q] = (double)acc[9];
    }
}

void oracle_nlm_f32(const float* z, int64_t ld, int64_t height, int64_t width, int radius,
                    double looks, double h, const int64_t* idx, int64_t m, double* out) {
    for (int64_t q = 0; q < m; ++q) {
        ld_t acc[10];
        herm_ld zi = load_ld_f32(z, ld, idx[q]);
        nlm_pixel(zi, (ld_t)looks, (ld_t)h, z, 1, ld, height, width, radius, idx[q] / width,
                  idx[q] % width, acc);
        for (int k = 0; k < 9; ++k) out[k * m + q] = (double)(acc[k] / acc[9]);
        out[9 * m + q] = (double)acc[9];
    }
}

/* ---------------------------------------------------------------------------
 * The same definition in the STORAGE precision: float for fp32 storage,
 * double for fp64 -- the plain CPU implementation of SURVEY §8(d), used only
 * as bench.py's cpu_baseline (and the --impl reference arm).  Eq. (3)
 * cofactors, the Eq. (5) row-0 expansion (real part), Eq. (4) entrywise
 * division and 1/det, all in type T.  bench.py times a separate
 * -O3 -march=native build of this file (oracle.build_plain()); the accuracy
 * oracle above stays binary128.  Pinned in tests/test_oracle.py (worked
 * examples exactly; the binary128 oracle within kappa^2-scaled rounding).
 * ------------------------------------------------------------------------- */
DEFINE_HERM(float, s)
DEFINE_HERM(double, d)

#define DEFINE_PLAIN(T, SFX, IN, LOAD)                                         \
void oracle_inv_det_plain_##SFX(const IN* z, int64_t ldz, T* out, int64_t ldo, \
                                int64_t n) {                                   \
    for (int64_t p = 0; p < n; ++p) {                                          \
        herm_##SFX m = LOAD(z, ldz, p);                                        \
        herm_##SFX c = cofactors_##SFX(m);                                     \
        T re, im;                                                              \
        det_full_##SFX(m, c, &re, &im);                                        \
        out[0 * ldo + p] = c.a / re;  out[1 * ldo + p] = c.br / re;            \
        out[2 * ldo + p] = c.bi / re; out[3 * ldo + p] = c.cr / re;            \
        out[4 * ldo + p] = c.ci / re; out[5 * ldo + p] = c.d / re;             \
        out[6 * ldo + p] = c.er / re; out[7 * ldo + p] = c.ei / re;            \
        out[8 * ldo + p] = c.f / re;                                           \
        out[9 * ldo + p] = re;                                                 \
        out[10 * ldo + p] = (T)1 / re;                                         \
        (void)im;                                                              \
    }                                                                          \
}
DEFINE_PLAIN(float, s, float, load_s_f32)
DEFINE_PLAIN(double, d, double, load_d_f64)

/* Mantissa digits of the evaluation type, so tests can assert the oracle
 * really runs in extended precision on the host it is built on. */
int oracle_ldbl_mant_dig(void) { return __LDBL_MANT_DIG__; }
int oracle_quad_mant_dig(void) { return __FLT128_MANT_DIG__; }
