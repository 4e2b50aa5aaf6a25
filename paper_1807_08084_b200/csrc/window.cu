// window.cu -- part of libpolsar.so (B200, sm_100a); arXiv 1807.08084.
// Layout, ownership and error conventions: include/polsar.h.  Design notes:
// DESIGN.md.  Nothing here is shared with oracle/.
//
//   K3  polsar_window_distance   23x23 search-window log-det distance sum
//   K6  polsar_window_kl         window sum with the symmetric Wishart KL distance
//   the window workspace queries (all three entry points, K4 included)
// Kernels and launchers: window_core.cuh.
#include "window_core.cuh"
#include "window_mma.cuh"

using namespace polsar_impl;

extern "C" {

size_t polsar_window_workspace_bytes_for(int entry, int64_t slab_rows, int64_t width, int radius,
                                         int dtype) {
    if (!slab_size_ok(slab_rows, width) || radius < 0 || entry < 0 || entry > 2) return 0;
    if (dtype != POLSAR_F32 && dtype != POLSAR_F64 && dtype != POLSAR_F32_PLAIN && dtype != POLSAR_F64_PLAIN)
        return 0;
    const int64_t n = slab_rows * width;
    const bool wt64 = dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN;
    const size_t wt = wt64 ? 8 : 4;
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const bool sym_ok = radius <= V3_RMAX;
    // the need of the form this entry point runs for (dtype, radius) -- the
    // dispatch below, fixed at compile time (no environment switches)
    if (entry == 0) {  // polsar_window_distance
        if (!sym_ok) return up((size_t)n * wt);  // the direct form: one plane of g
        if (use_window_mma(dtype, radius, false)) return mma_sym_bytes(slab_rows, width, radius);
        return window_sym_need(dtype, slab_rows, width, radius);
    }
    if (entry == 1) {  // polsar_nlm_filter
        if (!nlm_sym_ok(radius)) return up((size_t)n * wt);
        const int64_t rows = nlm_band_slab_rows(slab_rows, radius);
        return wt64 ? window_sym_bytes<double>(rows, width, radius) : window_sym_bytes<float>(rows, width, radius);
    }
    // polsar_window_kl (radius <= 12; no fp32-arithmetic mode)
    if (dtype == POLSAR_F32_PLAIN || !sym_ok) return 0;
    if (use_window_mma(dtype, radius, true)) return mma_sym_bytes(slab_rows, width, radius);
    return kl_sym_need(dtype, slab_rows, width, radius);
}

size_t polsar_window_workspace_bytes(int64_t slab_rows, int64_t width, int radius, int dtype) {
    size_t b = 0;
    for (int e = 0; e < 3; ++e)
        b = std::max(b, polsar_window_workspace_bytes_for(e, slab_rows, width, radius, dtype));
    return b;
}

int polsar_window_distance(const void* z, int64_t ld, int64_t width, int64_t slab_rows,
                           int64_t out_row_begin, int64_t out_row_end, int radius, double looks,
                           double h, void* workspace, void* out, int dtype, void* cuda_stream) {
    if (!slab_size_ok(slab_rows, width)) return fail(POLSAR_EINVAL, "negative size or slab_rows*width > 2^40");
    if (out_row_begin < 0 || out_row_end < out_row_begin || out_row_end > slab_rows)
        return fail(POLSAR_EINVAL, "bad output row range");
    if (radius < 0 || radius > 16) return fail(POLSAR_EINVAL, "radius out of [0, 16]");
    if (!(looks > 0) || !(h > 0)) return fail(POLSAR_EINVAL, "looks and h must be > 0");
    if (ld < slab_rows * width) return fail(POLSAR_EINVAL, "ld < slab_rows*width");
    if (width == 0 || out_row_end == out_row_begin) return POLSAR_OK;
    if (!z || !workspace || !out) return fail(POLSAR_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (use_window_mma(dtype, radius, false))
        return dtype == POLSAR_F32
                   ? launch_window_mma<float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end, radius,
                                                     looks, h, workspace, out, s)
                   : launch_window_mma<double, double>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                       radius, looks, h, workspace, out, s);
    // the symmetric two-pass form for R <= V3_RMAX, else the direct form
    const bool sym = radius <= V3_RMAX;
    switch (dtype) {
        case POLSAR_F32:
            return sym ? launch_window_sym<float, double, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                                 radius, looks, h, workspace, out, s)
                       : launch_window<float, double, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                             radius, looks, h, workspace, out, s);
        case POLSAR_F64:
        case POLSAR_F64_PLAIN:
            return sym ? launch_window_sym<double, double, double>(z, ld, width, slab_rows, out_row_begin,
                                                                   out_row_end, radius, looks, h, workspace, out, s)
                       : launch_window<double, double, double>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                               radius, looks, h, workspace, out, s);
        case POLSAR_F32_PLAIN:
            return sym ? launch_window_sym<float, float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                                radius, looks, h, workspace, out, s)
                       : launch_window<float, float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                            radius, looks, h, workspace, out, s);
        case POLSAR_F64_EFT: return fail(POLSAR_ENOTSUP, "POLSAR_F64_EFT: inverse/det entry points only");
        default: return fail(POLSAR_EINVAL, "bad dtype");
    }
}

int polsar_window_kl(const void* z, int64_t ld, int64_t width, int64_t slab_rows,
                     int64_t out_row_begin, int64_t out_row_end, int radius, double looks,
                     double h, void* workspace, void* out, int dtype, void* cuda_stream) {
    if (!slab_size_ok(slab_rows, width)) return fail(POLSAR_EINVAL, "negative size or slab_rows*width > 2^40");
    if (out_row_begin < 0 || out_row_end < out_row_begin || out_row_end > slab_rows)
        return fail(POLSAR_EINVAL, "bad output row range");
    if (radius < 0 || radius > V3_RMAX) return fail(POLSAR_EINVAL, "radius out of [0, 12]");
    if (!(looks > 0) || !(h > 0)) return fail(POLSAR_EINVAL, "looks and h must be > 0");
    if (ld < slab_rows * width) return fail(POLSAR_EINVAL, "ld < slab_rows*width");
    if (width == 0 || out_row_end == out_row_begin) return POLSAR_OK;
    if (!z || !workspace || !out) return fail(POLSAR_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (use_window_mma(dtype, radius, true))
        return dtype == POLSAR_F32
                   ? launch_window_kl_mma<float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end, radius,
                                                        looks, h, workspace, out, s)
                   : launch_window_kl_mma<double, double>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                          radius, looks, h, workspace, out, s);
    switch (dtype) {
        case POLSAR_F32:
            return launch_window_kl_sym<float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end, radius,
                                                      looks, h, workspace, out, s);
        case POLSAR_F64:
        case POLSAR_F64_PLAIN:
            return launch_window_kl_sym<double, double>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                        radius, looks, h, workspace, out, s);
        case POLSAR_F64_EFT: return fail(POLSAR_ENOTSUP, "POLSAR_F64_EFT: inverse/det entry points only");
        default: return fail(POLSAR_ENOTSUP, "polsar_window_kl: fp32-arithmetic mode not provided");
    }
}

}  // extern "C"
