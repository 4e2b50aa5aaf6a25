// nlm_fused_mma.cuh -- EXPERIMENT, not part of libpolsar.so (arXiv 1807.08084).
// Measured on B200 in round 2 and dropped: parity green against
// the oracle (W 1.7e-7, Zhat 1.9e-7 over the NLM test shapes), but c5 takes
// 7.50 ms against the product's 5.81 (ncu: per 1024-row band the pass is
// 3.57 ms, tensor pipe 25 %, issue 59 % at 16 warps/SM; ~100 instructions per
// 8x8 block against the window pass's ~35).  To try it: copy to
// paper_1807_08084_b200/csrc/, #include it from nlm.cu and window.cu, and
// dispatch polsar_nlm_filter / the NLM workspace query through
// nlm_fused_ok() / launch_nlm_fused() / nm_bytes() (build with
// -DPOLSAR_NLM_FUSED=1).
//
// K4, fused form: the NLM filter output (the NLM filter with stochastic
// distances of PAPER.md:77-80 [§I])
//   W_i = sum_j w_ij,   Zhat_i = sum_j w_ij Z_j / W_i,
// accumulated inside the tensor-core pass 1 of the window sum (window_mma.cuh):
// no weight planes, no gather pass.  Each unordered pair's weight is computed
// once (8x8 DMMA blocks of pair determinants, as K3b) and used twice:
//   forward  (owner i, window pixel j):  F_i += w [1, Z_j]   -- registers
//   backward (window pixel j, owner i):  B_j += w [1, Z_i]   -- shared memory
// Lane (m, q) of a block holds the weights of window pixel m against owned
// pixels 2q, 2q+1; the four lanes of m exchange them (8 shuffles), and lane q
// then takes the Z components c = q, q + 4 (and 8 for q = 0) of window pixel
// m for all 8 owned pixels: 24 FFMAs forward into its registers and 24 FFMAs
// backward, whose 3 sums go to m's shared-memory counters without a
// cross-lane reduction.  Every shared-memory sum is an exact fixed-point
// integer (W: 2^-44 as K3b; Z: 2^(44 - e) with 2^e >= max |Z| over the slab,
// from a prepass), so the result is bit-reproducible run to run.  Tiles are
// 16 x 8 owned pixels (one warp per 8 pixels x 1 row, 16 warps): the records
// (160 B), an fp32 copy of Z (36 B) and 20 counters (80 B) per halo slot
// take 224 KB at R = 11 (R = 12 does not fit: the banded plane form serves).
// Pass 2 adds each pixel's forward sums, the <= 3 x 3 tiles' backward sums
// that hold it, and Z_i itself (d_ii = 0, weight 1).
#pragma once
#include "window_mma.cuh"

namespace polsar_impl {
namespace {

constexpr int NM_TX = 16;                              // owned columns per tile
constexpr int NM_TY = 8;                               // owned rows per tile
constexpr int NM_THREADS = 32 * (NM_TX / 8) * NM_TY;   // one warp per 8 owned pixels x 1 row
constexpr int NM_NC = 10;                              // counter components: W, then Z_0..Z_8
#ifndef POLSAR_NM_CHUNK
#define POLSAR_NM_CHUNK 16
#endif
constexpr int NM_CHUNK = POLSAR_NM_CHUNK;              // tiles per CTA (a column of them)

__host__ __device__ constexpr int nm_hwe(int R) { return NM_TX - 8 + 8 * mma_nt(R); }
__host__ __device__ constexpr int nm_hw(int R) { return NM_TX + 2 * R; }  // pass 2's halo width
inline size_t nm_smem(int R) {
    const size_t slots = (size_t)nm_hwe(R) * (NM_TY + R);
    return slots * (MMA_RS * sizeof(double) + sizeof(float) + 9 * sizeof(float) + 2 * NM_NC * sizeof(unsigned)) +
           (size_t)NM_TY * nm_hwe(R) * 9 * sizeof(float);
}
inline bool nm_fits(int R) { return R >= 1 && R <= V3_RMAX && nm_smem(R) <= K3_SMEM_MAX; }
#ifndef POLSAR_NLM_FUSED
#define POLSAR_NLM_FUSED 0
#endif
// Does polsar_nlm_filter run the fused form?  (fp32 storage; the workspace
// query asks the same question)
inline bool nlm_fused_ok(int dtype, int R) {
    return POLSAR_NLM_FUSED && dtype == POLSAR_F32 && nm_fits(R) && !nlm_direct();
}

// the slab's largest |Z| entry (as uint bits of a non-negative float; atomicMax
// on the bits orders non-negative floats), for the Z counters' fixed point
__global__ void __launch_bounds__(256)
k_nm_maxabs(const float* __restrict__ z, int64_t ld, int64_t n, unsigned* __restrict__ out) {
    unsigned m = 0u;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            const float a = fabsf(z[k * ld + p]);
            m = a < INFINITY && __float_as_uint(a) > m ? __float_as_uint(a) : m;  // (NaN / inf skipped)
        }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__device__ __forceinline__ float nm_zscale(unsigned maxbits) {
    int e = 0;
    const float m = __uint_as_float(maxbits);
    if (m > 0.0f && m < INFINITY) frexpf(m, &e);  // m < 2^e
    return ldexpf(1.0f, 44 - e);
}

__device__ __forceinline__ void nm_add(unsigned* cnt, int HPe, int comp, int q, long long v) {
    atomicAdd(cnt + comp * HPe + q, (unsigned)((unsigned long long)v >> 22));
    atomicAdd(cnt + (NM_NC + comp) * HPe + q, (unsigned)(v & 0x3fffff));
}

// Pass 1: CTA = a column of NM_CHUNK tiles of 16 x 8 owned pixels, records in
// a ring of HH = 8 + R rows (window_mma.cuh's walk).  Outputs: fbuf (the W
// forward sums, double), fz (the Z forward sums, 9 planes of float, pixel
// stride N), and per tile the halo region's backward sums: partw (int64, W
// in 2^-44 units or kBadSum) and partz (9 floats per slot).
template <typename Pair, int NT>
__global__ void __launch_bounds__(NM_THREADS, 1)
k_nlm_fwd_mma(Pair pr, const float* __restrict__ z, int64_t ld, int64_t width, int64_t slab_rows,
              int64_t row_begin, int64_t row_end, int R, int nby, const unsigned* __restrict__ maxbits,
              double* __restrict__ fbuf, float* __restrict__ fz, long long* __restrict__ partw,
              float* __restrict__ partz) {
    using WT = float;
    constexpr int TY = NM_TY;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int HWe = NM_TX - 8 + 8 * NT;
    const int HH = TY + R;
    const int HPe = HWe * HH;
    const int HW = NM_TX + 2 * R;
    const int HP = HW * HH;
    const int64_t N = slab_rows * width;
    double* rec = reinterpret_cast<double*>(smem_raw);
    float* gs = reinterpret_cast<float*>(rec + (size_t)MMA_RS * HPe);
    float* zf = gs + HPe;                                           // 9 floats per slot
    unsigned* cnt = reinterpret_cast<unsigned*>(zf + (size_t)9 * HPe);  // [2][NM_NC][HPe] (tile-relative)
    float* stg = reinterpret_cast<float*>(cnt + (size_t)2 * NM_NC * HPe);

    const float zscale = nm_zscale(*maxbits);
    const float zinv = 1.0f / zscale;  // (a power of two: exact)
    const int64_t x0 = (int64_t)blockIdx.x * NM_TX;
    const int by0 = blockIdx.y * NM_CHUNK;
    const int by1 = by0 + NM_CHUNK < nby ? by0 + NM_CHUNK : nby;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cg = warp % (NM_TX / 8), rg = warp / (NM_TX / 8);  // rg = the owned row (RB = 1)
    const int am = lane >> 2, kq = lane & 3, b0 = 2 * kq;
    const int c0 = kq, c1 = kq + 4;  // this lane's Z components (plus 8 if kq == 0)
    unsigned mfull = 0u, mzero = 0u;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int64_t gxj = x0 + 8 * cg - R + 8 * t + am;
        const bool col = gxj >= 0 && gxj < width;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int dx = 8 * t + am - b0 - e - R;
            mfull |= (unsigned)(col && dx >= -R && dx <= R) << (2 * t + e);
            mzero |= (unsigned)(col && dx >= 1 && dx <= R) << (2 * t + e);
        }
    }

    // the first tile: every halo row from global memory
    {
        const int64_t y0 = row_begin + (int64_t)by0 * TY;
        for (int q = threadIdx.x; q < HPe; q += NM_THREADS) {
            const int hy = q / HWe, hx = q % HWe;
            const int64_t gy = y0 + hy, gx = x0 - R + hx;
            const bool in = gy < slab_rows && gx >= 0 && gx < width;
            const int64_t p = in ? gy * width + gx : 0;
            double v[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const float s = in ? z[k * ld + p] : 0.0f;
                v[k] = (double)s;
                zf[(size_t)9 * q + k] = s;
            }
            Pair::fill(rec + (size_t)MMA_RS * q, gs + q, v, in);
        }
        for (int q = threadIdx.x; q < 2 * NM_NC * HPe; q += NM_THREADS) cnt[q] = 0u;
    }

    for (int by = by0; by < by1; ++by) {
        const int64_t y0 = row_begin + (int64_t)by * TY;
        const int roff = ((by - by0) * TY) % HH;
        if (by > by0) {
            asm volatile("cp.async.wait_all;" ::: "memory");
            for (int q = threadIdx.x; q < TY * HWe; q += NM_THREADS) {
                const int hy = R + q / HWe, hx = q % HWe;
                const int64_t gy = y0 + hy, gx = x0 - R + hx;
                const bool in = gy < slab_rows && gx >= 0 && gx < width;
                const int slot = mma_ring(hy + roff, HH) * HWe + hx;
                POLSAR_CHECK(slot >= 0 && slot < HPe);
                double v[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const float s = in ? stg[q * 9 + k] : 0.0f;
                    v[k] = (double)s;
                    zf[(size_t)9 * slot + k] = s;
                }
                Pair::fill(rec + (size_t)MMA_RS * slot, gs + slot, v, in);
            }
        }
        __syncthreads();
        if (by + 1 < by1) {
            const int64_t yn = y0 + TY;
            for (int q = threadIdx.x; q < TY * HWe; q += NM_THREADS) {
                const int hy = R + q / HWe, hx = q % HWe;
                const int64_t gy = yn + hy, gx = x0 - R + hx;
                if (gy < slab_rows && gx >= 0 && gx < width) {
#pragma unroll
                    for (int k = 0; k < 9; ++k) mma_cp_async(stg + q * 9 + k, z + k * ld + gy * width + gx);
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }

        // the owned row: B fragments, g, ownership, and Z of the 8 owned pixels
        // in this lane's components
        const int ty = rg;
        const int hr = mma_ring(ty + roff, HH) * HWe + R + 8 * cg;  // slot of the group's first owned pixel
        const int64_t gy = y0 + ty;
        double bo[1][5];
        WT gi[1][2];
        bool own[2];
#pragma unroll
        for (int s = 0; s < 5; ++s) bo[0][s] = rec[(size_t)MMA_RS * (hr + am) + mma_perm(4 * s + kq)];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            gi[0][e] = gs[hr + b0 + e];
            own[e] = x0 + 8 * cg + b0 + e < width && gy < row_end;
        }
        float zo[8][3];
#pragma unroll
        for (int o = 0; o < 8; ++o) {
            const float* zp = zf + (size_t)9 * (hr + o);
            zo[o][0] = zp[c0];
            zo[o][1] = zp[c1];
            zo[o][2] = zp[8];
        }
        const bool bad = x0 + 8 * cg + am < width && gy < row_end && !(gs[hr + am] > WT(0));
        if (bad && kq == 0) {  // rare: flag an invalid owned pixel and its forward targets (R-19)
            const int qa = ty * HWe + R + 8 * cg + am;
            for (int dy = 0; dy <= R; ++dy)
                for (int dx = (dy == 0 ? 0 : -R); dx <= R; ++dx)
                    atomicOr(cnt + NM_NC * HPe + qa + dy * HWe + dx, kBadBit);
        }
        unsigned mask[1][2];
        {
            unsigned ob = 0u;
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int e = 0; e < 2; ++e) ob |= (unsigned)own[e] << (2 * t + e);
            mask[0][0] = mfull & ob;
            mask[0][1] = mzero & ob;
        }
        long long accw[2] = {0ll, 0ll};  // forward W sums, fixed point (as K3b)
        unsigned fnan = 0u;
        float fzs[8][3];  // forward Z sums of the 8 owned pixels, this lane's components and window pixels
#pragma unroll
        for (int o = 0; o < 8; ++o) fzs[o][0] = fzs[o][1] = fzs[o][2] = 0.0f;

        auto row = [&](int wy, auto full) {
            constexpr bool FULL = decltype(full)::value;
            const int dy = wy;  // the owned row is tile row rg; window tile row rg + wy
            const int hy = rg + wy;
            const int jrow = mma_ring(hy + roff, HH) * HWe + 8 * cg;
            const int jcnt = hy * HWe + 8 * cg;
            WT rp[2] = {WT(0), WT(0)};
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int jb = jrow + 8 * t;
                POLSAR_CHECK(jb + am >= 0 && jb + am < HPe && jcnt + 8 * t + am < HPe);
                const double* ra = rec + (size_t)MMA_RS * (jb + am) + kq;
                double aw[5];
#pragma unroll
                for (int s = 0; s < 5; ++s) aw[s] = ra[4 * s];
                const WT gj = gs[jb + am];
                const float* zm = zf + (size_t)9 * (jb + am);
                const float zm0 = zm[c0], zm1 = zm[c1], zm2 = zm[8];
                double c[2] = {0.0, 0.0};
#pragma unroll
                for (int s = 0; s < 5; ++s) dmma_884(c, aw[s], bo[0][s]);
                const unsigned mk = (FULL || dy > 0) ? mask[0][0] : mask[0][1];
                WT w[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    WT x = pr.weight(c[e], gj, gi[0][e]);
                    w[e] = ((mk >> (2 * t + e)) & 1u) ? x : WT(0);
                    rp[e] += w[e];
                }
                long long vw = fixed_w(w[0] + w[1]);
                vw += __shfl_xor_sync(0xffffffffu, vw, 1);
                vw += __shfl_xor_sync(0xffffffffu, vw, 2);
                // the 8 owned weights of window pixel am, from the 4 lanes of its row
                float wall[8];
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    wall[2 * s] = __shfl_sync(0xffffffffu, w[0], (lane & ~3) | s);
                    wall[2 * s + 1] = __shfl_sync(0xffffffffu, w[1], (lane & ~3) | s);
                }
                float bz0 = 0.0f, bz1 = 0.0f, bz2 = 0.0f;
#pragma unroll
                for (int o = 0; o < 8; ++o) {
                    fzs[o][0] = __fmaf_rn(wall[o], zm0, fzs[o][0]);
                    fzs[o][1] = __fmaf_rn(wall[o], zm1, fzs[o][1]);
                    fzs[o][2] = __fmaf_rn(wall[o], zm2, fzs[o][2]);
                    bz0 = __fmaf_rn(wall[o], zo[o][0], bz0);
                    bz1 = __fmaf_rn(wall[o], zo[o][1], bz1);
                    bz2 = __fmaf_rn(wall[o], zo[o][2], bz2);
                }
                const int qj = jcnt + 8 * t + am;
                if (kq == 0) nm_add(cnt, HPe, 0, qj, vw);
                nm_add(cnt, HPe, 1 + c0, qj, __float2ll_rn(bz0 * zscale));
                nm_add(cnt, HPe, 1 + c1, qj, __float2ll_rn(bz1 * zscale));
                if (kq == 0) nm_add(cnt, HPe, 1 + 8, qj, __float2ll_rn(bz2 * zscale));
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                accw[e] += fixed_w(rp[e]);
                fnan |= (unsigned)(rp[e] != rp[e]) << e;
            }
        };
        const int wmax = (int)(slab_rows - y0 - rg - 1 < R ? slab_rows - y0 - rg - 1 : R);
        if (wmax >= 0) row(0, std::false_type{});
        for (int wy = 1; wy <= wmax; ++wy) row(wy, std::true_type{});

        // forward W sums: as K3b (the 8 lanes of a C column hold disjoint window pixels)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            long long a = accw[e];
            a += __shfl_xor_sync(0xffffffffu, a, 4);
            a += __shfl_xor_sync(0xffffffffu, a, 8);
            a += __shfl_xor_sync(0xffffffffu, a, 16);
            const unsigned nanl = __ballot_sync(0xffffffffu, (fnan >> e) & 1u);
            const bool isnan_f = (nanl & (0x11111111u << kq)) != 0u;
            if (am == 0 && own[e])
                fbuf[gy * width + x0 + 8 * cg + b0 + e] =
                    isnan_f ? __longlong_as_double(0x7ff8000000000000ll) : (double)a * (1.0 / (double)kFix);
        }
        // forward Z sums: reduce over the 8 window-pixel lanes of each component
#pragma unroll
        for (int o = 0; o < 8; ++o)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                float a = fzs[o][i];
                a += __shfl_xor_sync(0xffffffffu, a, 4);
                a += __shfl_xor_sync(0xffffffffu, a, 8);
                a += __shfl_xor_sync(0xffffffffu, a, 16);
                fzs[o][i] = a;
            }
        if (am == 0 && gy < row_end) {
#pragma unroll
            for (int o = 0; o < 8; ++o) {
                const int64_t gx = x0 + 8 * cg + o;
                if (gx < width) {
                    const int64_t p = gy * width + gx;
                    fz[(int64_t)c0 * N + p] = fzs[o][0];
                    fz[(int64_t)c1 * N + p] = fzs[o][1];
                    if (kq == 0) fz[(int64_t)8 * N + p] = fzs[o][2];
                }
            }
        }
        __syncthreads();
        // the tile's halo-region backward sums (pass 2's layout); each slot is
        // cleared by the thread that writes it out
        const int64_t tile = (int64_t)by * gridDim.x + blockIdx.x;
        long long* dw = partw + tile * HP;
        float* dz = partz + tile * HP * 9;
        for (int q = threadIdx.x; q < HP; q += NM_THREADS) {
            const int sq = (q / HW) * HWe + q % HW;
            POLSAR_CHECK(sq < HPe);
            const unsigned hi = cnt[sq], lo = cnt[NM_NC * HPe + sq];
            dw[q] = (lo & kBadBit) ? kBadSum : (long long)(((unsigned long long)hi << 22) + lo);
            cnt[sq] = 0u;
            cnt[NM_NC * HPe + sq] = 0u;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const unsigned zh = cnt[(1 + k) * HPe + sq], zl = cnt[(NM_NC + 1 + k) * HPe + sq];
                const long long v = ((long long)(int)zh << 22) + (long long)zl;
                dz[(int64_t)q * 9 + k] = (float)v * zinv;
                cnt[(1 + k) * HPe + sq] = 0u;
                cnt[(NM_NC + 1 + k) * HPe + sq] = 0u;
            }
        }
    }
}

// Pass 2: W_j = 1 + F_j + 2^-44 (sum of the <= 3 x 3 tile sums holding j);
// Zhat_j = (Z_j + Fz_j + sum of the tiles' backward Z sums) / W_j.
template <typename S>
__global__ void __launch_bounds__(256)
k_nlm_fused_bwd(const S* __restrict__ z, int64_t ld, const long long* __restrict__ partw,
                const float* __restrict__ partz, const double* __restrict__ fbuf, const float* __restrict__ fz,
                int64_t width, int64_t slab_rows, int64_t row_begin, int64_t row_end, int64_t p0, int R, int nbx,
                int nby, S* __restrict__ out_w, S* __restrict__ out_z, int64_t ld_out) {
    const int HW = NM_TX + 2 * R;
    const int HP = HW * (NM_TY + R);
    const int64_t N = slab_rows * width;
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= width) return;
    const int bx_hi = (int)((x + R) / NM_TX < nbx - 1 ? (x + R) / NM_TX : nbx - 1);
    const int bx_lo = (int)(x - NM_TX - R + 1 > 0 ? (x - NM_TX - R + 1 + NM_TX - 1) / NM_TX : 0);
    for (int64_t y = row_begin + blockIdx.y; y < row_end; y += gridDim.y) {
        const int64_t yr = y - p0;
        const int64_t by_hi = yr / NM_TY;
        const int64_t by_lo = yr - NM_TY - R + 1 > 0 ? (yr - NM_TY - R + 1 + NM_TY - 1) / NM_TY : 0;
        const int64_t p = y * width + x;
        long long sw = 0;
        bool bad = false;
        double zs[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) zs[k] = (double)z[k * ld + p] + (double)fz[k * N + p];
        for (int64_t by = by_lo; by <= by_hi && by < nby; ++by)
            for (int bx = bx_lo; bx <= bx_hi; ++bx) {
                const int64_t hy = yr - by * NM_TY, hx = x - NM_TX * bx + R;
                POLSAR_CHECK(hy >= 0 && hy < NM_TY + R && hx >= 0 && hx < HW);
                const int64_t q = (by * nbx + bx) * HP + hy * HW + hx;
                const long long t = partw[q];
                bad = bad || t == kBadSum;
                sw += t;
#pragma unroll
                for (int k = 0; k < 9; ++k) zs[k] += (double)partz[q * 9 + k];
            }
        const double wsum = bad ? __longlong_as_double(0x7ff8000000000000ll)
                                : __dadd_rn(__dadd_rn(1.0, fbuf[p]), (double)sw * (1.0 / (double)kFix));
        const int64_t o = (y - row_begin) * width + x;
        if (out_w) out_w[o] = (S)wsum;
#pragma unroll
        for (int k = 0; k < 9; ++k) out_z[k * ld_out + o] = (S)__ddiv_rn(zs[k], wsum);
    }
}

// workspace: maxbits (256 B) | F (N doubles) | Fz (9 N floats) | partw (int64,
// HP per tile) | partz (9 HP floats per tile), each region 256-byte aligned
inline size_t nm_bytes(int64_t slab_rows, int64_t width, int R) {
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const int64_t n = slab_rows * width;
    const int64_t p0 = 0;
    const int64_t nbx = (width + NM_TX - 1) / NM_TX, nby = (slab_rows - p0 + NM_TY - 1) / NM_TY;
    const size_t tiles = (size_t)nbx * nby, hp = (size_t)nm_hw(R) * (NM_TY + R);
    return 256 + up((size_t)n * 8) + up((size_t)n * 36) + up(tiles * hp * 8) + up(tiles * hp * 36);
}

template <int NT, typename Pair>
int launch_nm_fwd(const Pair& pr, const float* z, int64_t ld, int64_t width, int64_t slab_rows, int64_t p0,
                  int64_t re, int R, int nby, const unsigned* maxbits, double* fbuf, float* fz, long long* partw,
                  float* partz, cudaStream_t s) {
    const size_t smem = nm_smem(R);
    auto kern = k_nlm_fwd_mma<Pair, NT>;
    if (smem > K3_SMEM_MAX ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return fail(POLSAR_ENOTSUP, "polsar_nlm_filter: fused form does not fit shared memory");
    const int nbx = (int)((width + NM_TX - 1) / NM_TX);
    dim3 grid((unsigned)nbx, (unsigned)((nby + NM_CHUNK - 1) / NM_CHUNK));
    kern<<<grid, NM_THREADS, smem, s>>>(pr, z, ld, width, slab_rows, p0, re, R, nby, maxbits, fbuf, fz, partw,
                                        partz);
    return POLSAR_OK;
}

// The fused NLM over output rows [rb, re) of a slab (fp32 storage).
template <typename Pair>
int launch_nlm_fused_pair(const Pair& pr, const float* z, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb,
                          int64_t re, int R, void* wsv, float* out_w, float* out_z, int64_t ld_out, cudaStream_t s) {
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const int64_t n = slab_rows * width;
    unsigned char* ws = (unsigned char*)wsv;
    unsigned* maxbits = (unsigned*)ws;
    double* fbuf = (double*)(ws + 256);
    float* fz = (float*)(ws + 256 + up((size_t)n * 8));
    const int64_t p0 = rb - R > 0 ? rb - R : 0;
    const int nbx = (int)((width + NM_TX - 1) / NM_TX);
    const int nby = (int)((re - p0 + NM_TY - 1) / NM_TY);
    const size_t hp = (size_t)nm_hw(R) * (NM_TY + R);
    long long* partw = (long long*)(ws + 256 + up((size_t)n * 8) + up((size_t)n * 36));
    float* partz = (float*)((unsigned char*)partw + up((size_t)nbx * nby * hp * 8));
    cudaMemsetAsync(maxbits, 0, sizeof(unsigned), s);
    k_nm_maxabs<<<grid_for(n, 256), 256, 0, s>>>(z, ld, n, maxbits);
    int rc;
    switch (mma_nt(R)) {
        case 1: rc = launch_nm_fwd<1>(pr, z, ld, width, slab_rows, p0, re, R, nby, maxbits, fbuf, fz, partw, partz, s); break;
        case 2: rc = launch_nm_fwd<2>(pr, z, ld, width, slab_rows, p0, re, R, nby, maxbits, fbuf, fz, partw, partz, s); break;
        case 3: rc = launch_nm_fwd<3>(pr, z, ld, width, slab_rows, p0, re, R, nby, maxbits, fbuf, fz, partw, partz, s); break;
        default: rc = launch_nm_fwd<4>(pr, z, ld, width, slab_rows, p0, re, R, nby, maxbits, fbuf, fz, partw, partz, s);
    }
    if (rc != POLSAR_OK) return rc;
    const int64_t rows = re - rb;
    dim3 grid2((unsigned)((width + 255) / 256), (unsigned)(rows < 65535 ? rows : 65535));
    k_nlm_fused_bwd<float><<<grid2, 256, 0, s>>>(z, ld, partw, partz, fbuf, fz, width, slab_rows, rb, re, p0, R, nbx,
                                                 nby, out_w, out_z, ld_out);
    return launch_check("polsar_nlm_filter: launch failed");
}

inline int launch_nlm_fused(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb, int64_t re,
                            int R, double looks, double h, void* wsv, void* out_w, void* out_z, int64_t ld_out,
                            cudaStream_t s) {
    const double alpha = looks / (2.0 * h);
    const float* z = (const float*)zv;
    if (alpha == 2.0)
        return launch_nlm_fused_pair(MmaLogDet<float, float, true>{(float)alpha}, z, ld, width, slab_rows, rb, re, R,
                                     wsv, (float*)out_w, (float*)out_z, ld_out, s);
    return launch_nlm_fused_pair(MmaLogDet<float, float, false>{(float)alpha}, z, ld, width, slab_rows, rb, re, R,
                                 wsv, (float*)out_w, (float*)out_z, ld_out, s);
}

}  // namespace
}  // namespace polsar_impl
