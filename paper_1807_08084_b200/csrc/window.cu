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
    const int64_t n = slab_rows * width;
    const bool wt64 = dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN;
    const size_t wt = wt64 ? 8 : 4;
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const bool sym_ok = radius <= V3_RMAX;
    const int v = window_variant();
    // the largest need of the kernels this entry point may run (with this
    // process's POLSAR_* A/B settings, which the library reads the same way)
    size_t b = up((size_t)n * wt);  // direct forms: one plane of g
    if (entry == 0) {                // polsar_window_distance
        if (sym_ok && v == 3 && dtype != POLSAR_F32_PLAIN) b = std::max(b, up((size_t)n * 160));
        if (use_window_mma(dtype, radius))
            b = std::max(b, mma_sym_bytes(slab_rows, width, radius));
        if (sym_ok && v == 4) {
            b = std::max(b, acc_sym_bytes((size_t)n * wt, slab_rows, width, radius, POLSAR_SYM_TY));
            if (window_planes())
                b = std::max(b, wt64 ? window_sym_bytes<double>(slab_rows, width, radius)
                                     : window_sym_bytes<float>(slab_rows, width, radius));
        }
    } else if (entry == 1) {         // polsar_nlm_filter (the dispatch conditions of the gather form)
        if (sym_ok && radius >= 1 && !nlm_direct() && slab_rows * (width + 4) + 2 * NLM_TX < ((int64_t)1 << 31))
            b = std::max(b, wt64 ? window_sym_bytes<double>(slab_rows, width, radius)
                                 : window_sym_bytes<float>(slab_rows, width, radius));
    } else {                         // polsar_window_kl (radius <= 12; no fp32-arithmetic mode)
        if (dtype == POLSAR_F32_PLAIN || !sym_ok) return 0;
        if (use_window_mma(dtype, radius))  // the tensor-core form: F | tile sums only
            return std::max(b, mma_sym_bytes(slab_rows, width, radius));
        b = std::max(b, up((size_t)n * 160));  // prepass planes (the streaming form's too)
        if (v == 4) {  // the choice of launch_window_kl_sym
            const size_t pre = (size_t)n * V3_NP * sizeof(double);
            const bool planes = window_planes();
            if (!wt64 && !planes && acc_fwd_smem<KLPairF<float>>(POLSAR_KLF_TY, radius) <= K3_SMEM_MAX)
                b = std::max(b, acc_sym_bytes(pre, slab_rows, width, radius, POLSAR_KLF_TY));
            else if (!planes && acc_fwd_smem<KLPair<float>>(16, radius) <= K3_SMEM_MAX)
                b = std::max(b, acc_sym_bytes(pre, slab_rows, width, radius, 16));
            else  // the weight-plane form (POLSAR_WINDOW_PLANES=1, or R = 12)
                b = std::max(b, wt64 ? kl_sym_bytes<double>(slab_rows, width, radius)
                                     : kl_sym_bytes<float>(slab_rows, width, radius));
        }
    }
    return b;
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
    if (use_window_mma(dtype, radius))
        return dtype == POLSAR_F32
                   ? launch_window_mma<float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end, radius,
                                                     looks, h, workspace, out, s)
                   : launch_window_mma<double, double>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                       radius, looks, h, workspace, out, s);
    switch (dtype) {
        case POLSAR_F32:
            if (radius <= V3_RMAX && window_variant() == 3)
                return launch_window_v3<float, float>(z, ld, width, slab_rows, out_row_begin,
                                                      out_row_end, radius, looks, h, workspace, out, s);
            if (radius <= V3_RMAX && window_variant() == 4)
                return launch_window_sym<float, double, float>(z, ld, width, slab_rows, out_row_begin,
                                                               out_row_end, radius, looks, h, workspace,
                                                               out, s);
            return launch_window<float, double, float>(z, ld, width, slab_rows, out_row_begin,
                                                       out_row_end, radius, looks, h, workspace, out, s);
        case POLSAR_F64:
        case POLSAR_F64_PLAIN:
            if (radius <= V3_RMAX && window_variant() == 3)
                return launch_window_v3<double, double>(z, ld, width, slab_rows, out_row_begin,
                                                        out_row_end, radius, looks, h, workspace, out, s);
            if (radius <= V3_RMAX && window_variant() == 4)
                return launch_window_sym<double, double, double>(z, ld, width, slab_rows, out_row_begin,
                                                                 out_row_end, radius, looks, h,
                                                                 workspace, out, s);
            return launch_window<double, double, double>(z, ld, width, slab_rows, out_row_begin,
                                                         out_row_end, radius, looks, h, workspace, out, s);
        case POLSAR_F32_PLAIN:
            if (radius <= V3_RMAX && window_variant() == 4)
                return launch_window_sym<float, float, float>(z, ld, width, slab_rows, out_row_begin,
                                                              out_row_end, radius, looks, h, workspace,
                                                              out, s);
            return launch_window<float, float, float>(z, ld, width, slab_rows, out_row_begin,
                                                      out_row_end, radius, looks, h, workspace, out, s);
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
    if (use_window_mma(dtype, radius))
        return dtype == POLSAR_F32
                   ? launch_window_kl_mma<float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end, radius,
                                                        looks, h, workspace, out, s)
                   : launch_window_kl_mma<double, double>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                          radius, looks, h, workspace, out, s);
    switch (dtype) {
        case POLSAR_F32:
            if (window_variant() == 4)
                return launch_window_kl_sym<float, float>(z, ld, width, slab_rows, out_row_begin,
                                                          out_row_end, radius, looks, h, workspace, out, s);
            return launch_window_kl<float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                  radius, looks, h, workspace, out, s);
        case POLSAR_F64:
        case POLSAR_F64_PLAIN:
            if (window_variant() == 4)
                return launch_window_kl_sym<double, double>(z, ld, width, slab_rows, out_row_begin,
                                                            out_row_end, radius, looks, h, workspace,
                                                            out, s);
            return launch_window_kl<double, double>(z, ld, width, slab_rows, out_row_begin,
                                                    out_row_end, radius, looks, h, workspace, out, s);
        default: return fail(POLSAR_ENOTSUP, "polsar_window_kl: fp32-arithmetic mode not provided");
    }
}

}  // extern "C"
