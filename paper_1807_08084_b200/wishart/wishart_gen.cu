// wishart_gen.cu -- GPU build of the seeded Wishart generator (support,
// untimed).  All arithmetic is in wishart_core.h, shared verbatim with the
// host twin wishart_gen_cpu.c; compiled with -fmad=false so both builds
// evaluate the same IEEE operation sequence (bit-identical output).
#include <cuda_runtime.h>
#include "wishart_core.h"
#include "../../include/polsar_gen.h"

template <typename T>
__global__ void __launch_bounds__(256) k_gen_wishart(T* __restrict__ z, int64_t ld, int64_t row_begin,
                                                     int64_t n_pix, wg_params P) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_pix;
         q += (int64_t)gridDim.x * blockDim.x) {
        int64_t y = row_begin + q / P.width;
        int64_t x = q % P.width;
        wg_herm m = wg_pixel(&P, y, x);
        z[0 * ld + q] = (T)m.a;
        z[1 * ld + q] = (T)m.br;
        z[2 * ld + q] = (T)m.bi;
        z[3 * ld + q] = (T)m.cr;
        z[4 * ld + q] = (T)m.ci;
        z[5 * ld + q] = (T)m.d;
        z[6 * ld + q] = (T)m.er;
        z[7 * ld + q] = (T)m.ei;
        z[8 * ld + q] = (T)m.f;
    }
}

extern "C" int polsar_gen_wishart(void* z, int64_t ld, int dtype, int64_t row_begin, int64_t row_end,
                                  int64_t width, int64_t height, int looks, uint64_t seed,
                                  uint32_t stream_id, int mode, const double* table, int64_t n_table,
                                  double near_singular_frac, void* cuda_stream) {
    if (!z || width <= 0 || height <= 0 || row_begin < 0 || row_end < row_begin || row_end > height)
        return POLSAR_GEN_EINVAL;
    if (mode < WG_MODE_SINGLE || mode > WG_MODE_PAPER_SIM) return POLSAR_GEN_EINVAL;
    if (mode != WG_MODE_PAPER_SIM && (!table || looks < 1)) return POLSAR_GEN_EINVAL;
    if (dtype != 0 && dtype != 1) return POLSAR_GEN_EINVAL;
    int64_t n_pix = (row_end - row_begin) * width;
    if (ld < n_pix) return POLSAR_GEN_EINVAL;
    if (n_pix == 0) return 0;
    wg_params P;
    P.seed = seed; P.stream = stream_id; P.looks = looks; P.mode = mode;
    P.height = height; P.width = width; P.table = table; P.n_table = n_table;
    P.near_singular_threshold = polsar_gen_threshold(near_singular_frac);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    int grid = (int)((n_pix + 255) / 256);
    if (grid > 148 * 64) grid = 148 * 64;
    if (dtype == 0)
        k_gen_wishart<float><<<grid, 256, 0, s>>>((float*)z, ld, row_begin, n_pix, P);
    else
        k_gen_wishart<double><<<grid, 256, 0, s>>>((double*)z, ld, row_begin, n_pix, P);
    return cudaGetLastError() == cudaSuccess ? 0 : POLSAR_GEN_ECUDA;
}
