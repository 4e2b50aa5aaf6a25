/* wishart_gen_cpu.c -- host twin of the seeded Wishart generator.  Same
 * arithmetic as the GPU build (wishart_core.h), compiled with
 * -ffp-contract=off, so any pixel of any image can be regenerated on the host
 * bit-identically (tests use it to feed the oracle sampled pixels of the
 * 4e8-pixel configs without copying the image back). */
#include "wishart_core.h"
#include "../../include/polsar_gen.h"

static void store(void* z, int64_t ld, int dtype, int64_t q, wg_herm m) {
    if (dtype == 0) {
        float* o = (float*)z;
        o[0 * ld + q] = (float)m.a;  o[1 * ld + q] = (float)m.br; o[2 * ld + q] = (float)m.bi;
        o[3 * ld + q] = (float)m.cr; o[4 * ld + q] = (float)m.ci; o[5 * ld + q] = (float)m.d;
        o[6 * ld + q] = (float)m.er; o[7 * ld + q] = (float)m.ei; o[8 * ld + q] = (float)m.f;
    } else {
        double* o = (double*)z;
        o[0 * ld + q] = m.a;  o[1 * ld + q] = m.br; o[2 * ld + q] = m.bi;
        o[3 * ld + q] = m.cr; o[4 * ld + q] = m.ci; o[5 * ld + q] = m.d;
        o[6 * ld + q] = m.er; o[7 * ld + q] = m.ei; o[8 * ld + q] = m.f;
    }
}

static int fill_params(wg_params* P, int64_t width, int64_t height, int looks, uint64_t seed,
                       uint32_t stream_id, int mode, const double* table, int64_t n_table,
                       double near_singular_frac) {
    if (width <= 0 || height <= 0) return POLSAR_GEN_EINVAL;
    if (mode < WG_MODE_SINGLE || mode > WG_MODE_PAPER_SIM) return POLSAR_GEN_EINVAL;
    if (mode != WG_MODE_PAPER_SIM && (!table || looks < 1)) return POLSAR_GEN_EINVAL;
    P->seed = seed; P->stream = stream_id; P->looks = looks; P->mode = mode;
    P->height = height; P->width = width; P->table = table; P->n_table = n_table;
    P->near_singular_threshold = polsar_gen_threshold(near_singular_frac);
    return 0;
}

int polsar_gen_wishart_cpu(void* z, int64_t ld, int dtype, int64_t row_begin, int64_t row_end,
                           int64_t width, int64_t height, int looks, uint64_t seed,
                           uint32_t stream_id, int mode, const double* table, int64_t n_table,
                           double near_singular_frac) {
    wg_params P;
    int rc = fill_params(&P, width, height, looks, seed, stream_id, mode, table, n_table,
                         near_singular_frac);
    if (rc) return rc;
    if (!z || row_begin < 0 || row_end < row_begin || row_end > height) return POLSAR_GEN_EINVAL;
    if (dtype != 0 && dtype != 1) return POLSAR_GEN_EINVAL;
    int64_t n_pix = (row_end - row_begin) * width;
    if (ld < n_pix) return POLSAR_GEN_EINVAL;
    for (int64_t q = 0; q < n_pix; ++q)
        store(z, ld, dtype, q, wg_pixel(&P, row_begin + q / width, q % width));
    return 0;
}

int polsar_gen_wishart_pixels_cpu(const int64_t* pix, int64_t m, void* z, int64_t ld, int dtype,
                                  int64_t width, int64_t height, int looks, uint64_t seed,
                                  uint32_t stream_id, int mode, const double* table,
                                  int64_t n_table, double near_singular_frac) {
    wg_params P;
    int rc = fill_params(&P, width, height, looks, seed, stream_id, mode, table, n_table,
                         near_singular_frac);
    if (rc) return rc;
    if (!z || !pix || ld < m || (dtype != 0 && dtype != 1)) return POLSAR_GEN_EINVAL;
    for (int64_t q = 0; q < m; ++q) {
        if (pix[q] < 0 || pix[q] >= width * height) return POLSAR_GEN_EINVAL;
        store(z, ld, dtype, q, wg_pixel(&P, pix[q] / width, pix[q] % width));
    }
    return 0;
}

/* self-test hooks for the deterministic elementary functions */
double polsar_gen_cpu_log(double x) { return wg_log(x); }
double polsar_gen_cpu_exp2(double x) { return wg_exp2(x); }
void polsar_gen_cpu_cossin(double u, double* c, double* s) { wg_cossin_2pi(u, c, s); }
