/*
 * polsar_gen.h -- C-ABI of the seeded multilook-covariance generator
 * (support for the hot path; never timed).  Two builds of one source
 * (paper_1807_08084_b200/wishart/wishart_core.h):
 *   libpolsar_gen.so      polsar_gen_wishart          (device pointers, async on a stream)
 *   libpolsar_gen_cpu.so  polsar_gen_wishart_cpu      (host pointers)
 *                         polsar_gen_wishart_pixels_cpu (host, listed global pixels)
 * Both produce bit-identical matrices for the same arguments.
 *
 * What is generated (Eq. (2) [§I]; readings R-3,
 * R-9, R-13): for global pixel (y, x) of a height x width image,
 *   Z = (1/L) sum_{l<L} s_l s_l^H,  s_l = C z_l,  z_l ~ CN(0, I) (Re, Im iid N(0, 1/2)),
 * with C the lower-triangular Cholesky factor of Sigma selected by `mode`
 * from `table` (n_table rows of 9 doubles: c00, Re c10, Im c10, c11, Re c20,
 * Im c20, Re c21, Im c21, c22).  mode 4 (paper-sim) ignores the table and
 * returns Z = G G^H with Re/Im(G) ~ U[-1, 1] (PAPER.md:715-723 [§IV-B1]).
 * With near_singular_frac > 0 each pixel is, with that probability, replaced
 * by Q diag(1, mu, 1e-6) Q^H (Q Haar, mu log-uniform on [1e-6, 1]): kappa_2 = 1e6.
 * Randomness: Philox4x32-10 keyed by (seed, stream_id), counter (pixel, look, draw).
 *
 * Output layout: 9 planes (field order a, Re b, Im b, Re c, Im c, d, Re e,
 * Im e, f), plane k at z + k*ld elements; pixel (y, x) of rows
 * [row_begin, row_end) at offset (y - row_begin)*width + x.  dtype 0 = fp32
 * (each value rounded once from fp64), 1 = fp64.  The caller owns z (and
 * table: device memory for the GPU build, host memory for the CPU build).
 *
 * Return: 0 ok, 1 EINVAL (bad pointer / range / mode / dtype, ld too small),
 * 2 ECUDA (launch failed; asynchronous faults surface at the next sync).
 */
#ifndef POLSAR_GEN_H
#define POLSAR_GEN_H
#include <stdint.h>

#define POLSAR_GEN_EINVAL 1
#define POLSAR_GEN_ECUDA 2

#ifdef __cplusplus
extern "C" {
#endif

int polsar_gen_wishart(void* z, int64_t ld, int dtype, int64_t row_begin, int64_t row_end,
                       int64_t width, int64_t height, int looks, uint64_t seed,
                       uint32_t stream_id, int mode, const double* table, int64_t n_table,
                       double near_singular_frac, void* cuda_stream);

int polsar_gen_wishart_cpu(void* z, int64_t ld, int dtype, int64_t row_begin, int64_t row_end,
                           int64_t width, int64_t height, int looks, uint64_t seed,
                           uint32_t stream_id, int mode, const double* table, int64_t n_table,
                           double near_singular_frac);

int polsar_gen_wishart_pixels_cpu(const int64_t* pix, int64_t m, void* z, int64_t ld, int dtype,
                                  int64_t width, int64_t height, int looks, uint64_t seed,
                                  uint32_t stream_id, int mode, const double* table,
                                  int64_t n_table, double near_singular_frac);

#ifdef __cplusplus
}
#endif

/* probability -> u32 threshold (shared by both builds; exact) */
static inline uint32_t polsar_gen_threshold(double frac) {
    if (!(frac > 0.0)) return 0u;
    if (frac >= 1.0) return 0xFFFFFFFFu;
    return (uint32_t)(frac * 4294967296.0);
}

#endif
