// window_mma.cuh -- part of libpolsar.so (B200, sm_100a); arXiv 1807.08084.
// Pass 1 of the window sums on the FP64 tensor cores: K3b (log-det distance)
// and K6 (symmetric Wishart KL), the product for fp32 storage.
//
// The pair determinant of the log-det window (BASELINE
// configs[4]) through the 3x3 identity
//   det(A + B) = det A + det B + <adj A, B> + <A, adj B>,   <X, Y> = tr(X Y),
// (the expansion form of K3 v3) is the dot product of two
// 20-vectors,
//   a_i = [adj2(Z_i), Z_i, D_i, 1],   b_j = [Z_j, adj2(Z_j), 1, D_j],
// adj2 = the adjugate of Eq. 3 with its off-diagonal entries doubled (the
// Hermitian inner product counts each off-diagonal pair twice), D = det by
// Eq. 6.  So an 8 x 8 block of pair determinants (8 window pixels of a row x
// 8 owned pixels of a row) is one 8 x 8 x 20 fp64 matrix product: five
// mma.sync.m8n8k4.f64 (DMMA).  The KL distance's T - 6 = <X_i, Z_j> +
// <Z_i, X_j> - 6 (X = w Z^-1, Alg. 2) has the same shape (MmaKL).  Each warp
// keeps the fragments of its 2 rows x 8 owned pixels in registers (the B
// operand: 5 doubles per row per lane) and streams the window pixels' records
// from shared memory (the A operand).  The symmetric two-pass structure of
// the ACC form (window_core.cuh) is kept: pass 1 covers the forward
// half-window (dy = 1..R, and dy = 0 with dx = 1..R) and adds every weight to
// the neighbour's fixed-point backward sum in shared memory; pass 2 is
// k_window_bwd_acc unchanged (tile height 8).  A CTA walks a column of
// MMA_CHUNK tiles with the halo records in a ring (k_window_fwd_mma).
//
// Per 8-pixel group and window row the 8 + 2R window columns are covered by
// NT = ceil((8 + 2R) / 8) column blocks of 8 (72 % of the computed pairs are
// inside the window at R = 11): 47 blocks x 5 DMMA x 256 FMA per 8 pixels, an
// FP64 floor of 1.69 ms at c5, the same as the scalar form's 29 operations per
// pair (1.72 ms) -- the gain is the tensor pipe's issue efficiency (62.6 of
// 64 FMA/clk/SM at 16 warps, profiles/r01_micro_dmma_rate.txt; 67 % busy in
// this kernel) against the scalar pair loop's 57 % of the FP64 pipe.
#pragma once
#include <type_traits>

#include "window_core.cuh"

namespace polsar_impl {
namespace {

#ifndef POLSAR_MMA_TY
#define POLSAR_MMA_TY 8
#endif
#ifndef POLSAR_MMA_PROBE
#define POLSAR_MMA_PROBE 0  // development probe: 1 = tile fill and writeout only; 2 = no weight arithmetic
#endif
#ifndef POLSAR_MMA_CHUNK
#define POLSAR_MMA_CHUNK 16
#endif
constexpr int MMA_CHUNK = POLSAR_MMA_CHUNK;  // tiles per CTA (a column of them)
#ifndef POLSAR_MMA_UNROLL
#define POLSAR_MMA_UNROLL 1
#endif
constexpr int kMmaUnroll = POLSAR_MMA_UNROLL;  // full window rows per loop iteration
constexpr int MMA_TY = POLSAR_MMA_TY;  // tile rows (pass 2 takes the same TY)
#ifndef POLSAR_MMA_RB
#define POLSAR_MMA_RB 1
#endif
constexpr int MMA_RB = POLSAR_MMA_RB;  // owned rows per warp
constexpr int MMA_THREADS = 32 * (K3_TX / 8) * (MMA_TY / MMA_RB);  // one warp per 8 x RB pixels
constexpr int MMA_RS = 20;             // record doubles: Z (9) | adj2 (9) | 1 | D  (160 B:
                                       // a warp's b-fragment loads hit 32 distinct banks per half)

// POLSAR_WINDOW_MMA (compile time; tools/build_variant.sh): -1 (the product) =
// the tensor-core pass 1 for fp32 storage, and for the fp64 KL window (see
// use_window_mma); 1 = for every call; 0 = never.
#ifndef POLSAR_WINDOW_MMA
#define POLSAR_WINDOW_MMA -1
#endif
constexpr int window_mma_mode() { return POLSAR_WINDOW_MMA; }

__host__ __device__ constexpr int mma_nt(int R) { return (2 * R + 15) / 8; }
// halo columns: x0 - R .. x0 - R + HWe - 1 (the last group's NT blocks may
// reach 2 columns past the window; those pairs are masked)
__host__ __device__ constexpr int mma_hwe(int R) { return K3_TX - 8 + 8 * mma_nt(R); }

template <typename S, typename WT>
size_t mma_fwd_smem(int R) {
    const size_t slots = (size_t)mma_hwe(R) * (MMA_TY + R);
    return slots * (MMA_RS * sizeof(double) + sizeof(WT) + 2 * sizeof(unsigned)) +
           (size_t)MMA_TY * mma_hwe(R) * 9 * sizeof(S);  // + the staging buffer
}

// Does polsar_window_distance (kl = false) / polsar_window_kl (kl = true) run
// the tensor-core form for this call?  (The workspace query asks the same
// question.)  fp32 storage: both.  fp64 storage: the KL window (4.78 vs 5.33 ms
// on c5: its per-pair weight is one exp, so the DMMAs keep the FP64 datapath),
// not the log-det window (3.84 vs 3.49 ms: its fp64 weight's DFMA Newton
// steps share the datapath with the DMMAs); POLSAR_WINDOW_MMA=1 forces both.
bool use_window_mma(int dtype, int radius, bool kl) {
    if (radius > V3_RMAX || window_planes()) return false;
    const int m = window_mma_mode();
    if (m == 0) return false;
    if (dtype == POLSAR_F32) return mma_fwd_smem<float, float>(radius) <= K3_SMEM_MAX;
    return (m == 1 || kl) && (dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN) &&
           mma_fwd_smem<double, double>(radius) <= K3_SMEM_MAX;  // (fp64 at R = 12: 229,376 B, fits)
}

__device__ __forceinline__ void dmma_884(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

// Pair policies: fill() writes one halo slot's 20-double record (from the 9
// planes) and its validity/g value; weight() maps the pair's dot product c to
// the weight.  Invalid pixels (not positive definite, or non-finite) get a NaN
// g, which the kernel turns into NaN W on every pixel whose window holds them
// (R-19); out-of-image slots get g = 0 and are always masked.

// The log-det window: record [Z, adj2, 1, D] (adjugate of Eq. 3, off-diagonal
// entries doubled; D by Eq. 6, the same det_eq6 as k_window_prep, so g =
// 1/(8D) is bit-identical to it); c = det(Z_i + Z_j).
template <typename S_, typename WT_, bool A2_>
struct MmaLogDet {
    using S = S_;
    using WT = WT_;
    WT alpha;  // L / (2h): w = ((c/8)^2 / (D_i D_j))^-alpha
    __device__ __forceinline__ static void fill(double* rec, WT* gs, const double (&v)[9], bool in) {
        const double a = v[0], br = v[1], bi = v[2], cr = v[3], ci = v[4], d = v[5], er = v[6], ei = v[7],
                     f = v[8];
        const double A00 = FMA(d, f, -FMA(er, er, MUL(ei, ei)));
        const double A01r = FMA(cr, er, FMA(ci, ei, -MUL(br, f)));  // c conj(e) - b f
        const double A01i = FMA(ci, er, -FMA(cr, ei, MUL(bi, f)));
        const double A02r = FMA(br, er, -FMA(bi, ei, MUL(cr, d)));  // b e - c d
        const double A02i = FMA(br, ei, FMA(bi, er, -MUL(ci, d)));
        const double A11 = FMA(a, f, -FMA(cr, cr, MUL(ci, ci)));
        const double A12r = FMA(br, cr, FMA(bi, ci, -MUL(a, er)));  // conj(b) c - a e
        const double A12i = FMA(br, ci, -FMA(bi, cr, MUL(a, ei)));
        const double A22 = FMA(a, d, -FMA(br, br, MUL(bi, bi)));
        const double D = det_eq6<double>(a, br, bi, cr, ci, d, er, ei, f);
        const double r[MMA_RS] = {a,    br,         bi,         cr,         ci,         d,   er,
                                  ei,   f,          A00,        2.0 * A01r, 2.0 * A01i, 2.0 * A02r, 2.0 * A02i,
                                  A11,  2.0 * A12r, 2.0 * A12i, A22,        1.0,        D};
        double2* o = reinterpret_cast<double2*>(rec);
#pragma unroll
        for (int k = 0; k < MMA_RS / 2; ++k) o[k] = make_double2(r[2 * k], r[2 * k + 1]);
        const WT gv = (WT)(1.0 / MUL(8.0, D));
        *gs = in ? ((D > 0.0 && gv < WT(INFINITY)) ? gv : WT(NAN)) : WT(0);
    }
    __device__ __forceinline__ WT weight(double c, WT gj, WT gi) const {
#if POLSAR_MMA_PROBE == 2
        return (WT)c * gi;  // development probe: the epilogue without the weight arithmetic
#endif
        const WT fds = (WT)c;
        const WT rr = (fds * gj) * (fds * gi);
        return pair_weight(rr, alpha, A2_);
    }
};

// The symmetric Wishart KL window (K6): record [Z, X, 1, -3] with X = w Z^-1
// (Alg. 2, the Hermitian trace weights w as k_window_prep_kl), so
// c = tr(Z_i^-1 Z_j) + tr(Z_j^-1 Z_i) - 6 and d = L c / 2 (the -6 rides in the
// dot product: no FP64 instruction outside the DMMAs).
template <typename S_, typename WT_>
struct MmaKL {
    using S = S_;
    using WT = WT_;
    WT lk;  // L / h
    __device__ __forceinline__ static void fill(double* rec, WT* gs, const double (&v)[9], bool in) {
        H9<double> m;
        m.a = v[0]; m.br = v[1]; m.bi = v[2]; m.cr = v[3]; m.ci = v[4];
        m.d = v[5]; m.er = v[6]; m.ei = v[7]; m.f = v[8];
        double x[9], det, t;
        alg2_plain<double>(m, x, det, t);
        const bool ok = det > 0.0 && t < INFINITY;
        const double wk[9] = {1, 2, 2, 2, 2, 1, 2, 2, 1};
        double r[MMA_RS];
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            r[k] = v[k];
            r[9 + k] = in ? (ok ? wk[k] * x[k] : (double)NAN) : 0.0;
        }
        r[18] = 1.0;
        r[19] = -3.0;
        double2* o = reinterpret_cast<double2*>(rec);
#pragma unroll
        for (int k = 0; k < MMA_RS / 2; ++k) o[k] = make_double2(r[2 * k], r[2 * k + 1]);
        *gs = in ? (ok ? WT(1) : WT(NAN)) : WT(0);
    }
    __device__ __forceinline__ WT weight(double c, WT, WT) const;
};
template <>
__device__ __forceinline__ float MmaKL<float, float>::weight(double c, float, float) const {
    return fast_exp2(-lk * 0.5f * 1.4426950408889634f * (float)c);
}
template <>
__device__ __forceinline__ double MmaKL<double, double>::weight(double c, double, double) const {
    return exp(-lk * 0.5 * c);
}

// the owned operand's k -> record slot: [adj2, Z, D, 1] against the window
// pixel's record [Z, adj2, 1, D]
__device__ __forceinline__ int mma_perm(int k) { return k < 9 ? k + 9 : k < 18 ? k - 9 : (k == 18 ? 19 : 18); }

// Fragment roles: the window pixels are the MMA's A operand (rows m, streamed
// from shared memory per 8-pixel block) and the owned pixels its B operand
// (columns n, register-resident), so lane (m = lane/4, q = lane%4) holds the
// pairs (window pixel m, owned pixels 2q and 2q+1).  A window pixel's
// backward sum then needs a reduction over only the 4 lanes of its row, and
// the forward sums are reduced once, at the end of the kernel.
template <typename WT>
struct MmaLane {
    int am, kq, b0;         // fragment row / k, first C column
    unsigned mfull, mzero;  // window-and-image masks over (block t, column e): dy > 0, dy == 0
};

// One window row (slot jrow = its first block's first pixel) against the
// warp's RB owned rows: per 8-pixel block, the A fragment, RB chains of 5
// DMMA, the weights into rp (forward) and the row's fixed-point sums into
// the backward counters.  FULL: dy = wy - r in [1, R] for every r (no
// branches, so the scheduler interleaves the chains).
template <typename Pair, int NT, bool FULL, typename WT = typename Pair::WT>
__device__ __forceinline__ void mma_row(const Pair& pr, const double* rec, const WT* gs, unsigned* ah, int HPe,
                                        int jrow, int jcnt, const double (&bo)[MMA_RB][5], const WT (&gi)[MMA_RB][2],
                                        const unsigned (&mask)[MMA_RB][2], int wy, int R, const MmaLane<WT>& ln,
                                        WT (&rp)[MMA_RB][2]) {
#pragma unroll
    for (int r = 0; r < MMA_RB; ++r) rp[r][0] = rp[r][1] = WT(0);
    long long vs[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int jb = jrow + 8 * t;  // slot of the block's first window pixel
        POLSAR_CHECK(jb + ln.am >= 0 && jb + ln.am < HPe && jcnt + 8 * t + ln.am < HPe);
        const double* ra = rec + (size_t)MMA_RS * (jb + ln.am) + ln.kq;
        double aw[5];
#pragma unroll
        for (int s = 0; s < 5; ++s) aw[s] = ra[4 * s];
        const WT gj = gs[jb + ln.am];
        long long v = 0ll;
#pragma unroll
        for (int r = 0; r < MMA_RB; ++r) {
            const int dy = wy - r;
            if (!FULL && (dy < 0 || dy > R)) continue;  // warp-uniform
            double c[2] = {0.0, 0.0};
#pragma unroll
            for (int s = 0; s < 5; ++s) dmma_884(c, aw[s], bo[r][s]);
            // the window/image masks with the owned-pixel test folded in (the
            // forward sums of pixels that are not owned are never written)
            const unsigned m = (FULL || dy > 0) ? mask[r][0] : mask[r][1];
            WT wb = WT(0);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                WT w = pr.weight(c[e], gj, gi[r][e]);
                w = ((m >> (2 * t + e)) & 1u) ? w : WT(0);
                rp[r][e] += w;
                wb += w;
            }
            // the two owned columns 2q, 2q+1 are fixed by x mod 8, so this
            // float sum is the same under any row decomposition; the rest is
            // integer (exact, order-free)
            v += fixed_w(wb);
        }
        // sum over the 4 lanes of the window pixel's fragment row
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        vs[t] = v;
    }
    // one shared-memory add per window pixel, after all blocks (a branch per
    // block would split the row into basic blocks the scheduler cannot overlap)
    if (ln.kq == 0) {
#pragma unroll
        for (int t = 0; t < NT; ++t) acc_add(ah, HPe, jcnt + 8 * t + ln.am, vs[t]);
    }
}

// ring row of tile row + offset, both < HH (no division)
__device__ __forceinline__ int mma_ring(int r, int HH) { return r >= HH ? r - HH : r; }

// cp.async of one plane element (4 or 8 bytes) into the staging buffer
template <typename S>
__device__ __forceinline__ void mma_cp_async(S* smem, const S* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(sa), "l"(gmem), "n"(sizeof(S)) : "memory");
}

// Pass 1, persistent over a column of MMA_CHUNK tiles: tile by's halo rows
// overlap tile by + 1's in HH - TY = R rows, so the records live in a ring of
// HH rows and each later tile computes only its TY new rows -- from planes
// that cp.async staged during the previous tile's DMMA work.  The backward-sum
// counters are tile-relative: written out (and cleared) after each tile.
template <typename Pair, int NT>
__global__ void __launch_bounds__(MMA_THREADS, 1)
k_window_fwd_mma(Pair pr, const typename Pair::S* __restrict__ z, int64_t ld, int64_t width, int64_t slab_rows,
                 int64_t row_begin, int64_t row_end, int R, int nby, double* __restrict__ fbuf,
                 long long* __restrict__ part) {
    using S = typename Pair::S;
    using WT = typename Pair::WT;
    constexpr int TY = MMA_TY, RB = MMA_RB;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int HWe = K3_TX - 8 + 8 * NT;
    const int HH = TY + R;
    const int HPe = HWe * HH;
    const int HW = K3_TX + 2 * R;  // pass 2's tile layout
    const int HP = HW * HH;
    double* rec = reinterpret_cast<double*>(smem_raw);
    WT* gs = reinterpret_cast<WT*>(rec + (size_t)MMA_RS * HPe);
    unsigned* ah = reinterpret_cast<unsigned*>(gs + HPe);  // high counters, then low (tile-relative)
    S* stg = reinterpret_cast<S*>(ah + 2 * HPe);           // staged planes of the next tile's TY new rows

    const int64_t x0 = (int64_t)blockIdx.x * K3_TX;
    const int by0 = blockIdx.y * MMA_CHUNK;
    const int by1 = by0 + MMA_CHUNK < nby ? by0 + MMA_CHUNK : nby;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cg = warp % (K3_TX / 8), rg = warp / (K3_TX / 8);
    const int am = lane >> 2;  // A row (window pixel of a block) / B column (owned pixel of the B fragment)
    const int kq = lane & 3;   // fragment k / C column pair
    const int b0 = 2 * kq;     // this lane's C columns: owned pixels b0, b0 + 1
    // per-lane masks over (t, e): the window column test for dy > 0 and dy == 0,
    // and the image column test of the window pixel
    unsigned mfull = 0u, mzero = 0u;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int64_t gxj = x0 + 8 * cg - R + 8 * t + am;
        const bool col = gxj >= 0 && gxj < width;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int dx = 8 * t + am - b0 - e - R;  // window pixel column - owned pixel column
            mfull |= (unsigned)(col && dx >= -R && dx <= R) << (2 * t + e);
            mzero |= (unsigned)(col && dx >= 1 && dx <= R) << (2 * t + e);
        }
    }
    const MmaLane<WT> ln{am, kq, b0, mfull, mzero};

    // the first tile: every halo row from global memory (all loads issued first)
    {
        constexpr int MAXQ = (56 * (MMA_TY + V3_RMAX) + MMA_THREADS - 1) / MMA_THREADS;
        const int64_t y0 = row_begin + (int64_t)by0 * TY;
        double v[MAXQ][9];
        bool in[MAXQ];
#pragma unroll
        for (int i = 0; i < MAXQ; ++i) {
            const int q = threadIdx.x + i * MMA_THREADS;
            const int hy = q / HWe, hx = q % HWe;
            const int64_t gy = y0 + hy, gx = x0 - R + hx;
            in[i] = q < HPe && gy < slab_rows && gx >= 0 && gx < width;
            const int64_t p = in[i] ? gy * width + gx : 0;
#pragma unroll
            for (int k = 0; k < 9; ++k) v[i][k] = in[i] ? (double)z[k * ld + p] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < MAXQ; ++i) {
            const int q = threadIdx.x + i * MMA_THREADS;
            if (q < HPe) {
                Pair::fill(rec + (size_t)MMA_RS * q, gs + q, v[i], in[i]);
                ah[q] = 0u;
                ah[HPe + q] = 0u;
            }
        }
    }

    for (int by = by0; by < by1; ++by) {
        const int64_t y0 = row_begin + (int64_t)by * TY;
        const int roff = ((by - by0) * TY) % HH;  // ring row of tile row 0
        if (by > by0) {
            // the TY new rows (tile rows R .. HH-1) from the staged planes; each
            // thread fills the slots whose planes it staged itself
            asm volatile("cp.async.wait_all;" ::: "memory");
            for (int q = threadIdx.x; q < TY * HWe; q += MMA_THREADS) {
                const int hy = R + q / HWe, hx = q % HWe;
                const int64_t gy = y0 + hy, gx = x0 - R + hx;
                const bool in = gy < slab_rows && gx >= 0 && gx < width;
                double v[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) v[k] = in ? (double)stg[q * 9 + k] : 0.0;
                const int slot = mma_ring(hy + roff, HH) * HWe + hx;
                POLSAR_CHECK(slot >= 0 && slot < HPe && q * 9 + 8 < MMA_TY * HWe * 9);
                Pair::fill(rec + (size_t)MMA_RS * slot, gs + slot, v, in);
            }
        }
        __syncthreads();
        // stage the next tile's new rows while this tile computes
        if (by + 1 < by1) {
            const int64_t yn = y0 + TY;  // the next tile's y0
            for (int q = threadIdx.x; q < TY * HWe; q += MMA_THREADS) {
                const int hy = R + q / HWe, hx = q % HWe;
                const int64_t gy = yn + hy, gx = x0 - R + hx;
                if (gy < slab_rows && gx >= 0 && gx < width) {
#pragma unroll
                    for (int k = 0; k < 9; ++k) mma_cp_async(stg + q * 9 + k, z + k * ld + gy * width + gx);
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }

        double bo[RB][5];
        WT gi[RB][2];
        bool own[RB][2];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            const int ty = rg * RB + r;
            const int hr = mma_ring(ty + roff, HH) * HWe + R + 8 * cg;  // record slot of the group's first owned pixel
            POLSAR_CHECK(hr + 7 < HPe && roff >= 0 && roff < HH);
            const int64_t gy = y0 + ty;
#pragma unroll
            for (int s = 0; s < 5; ++s) bo[r][s] = rec[(size_t)MMA_RS * (hr + am) + mma_perm(4 * s + kq)];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                gi[r][e] = gs[hr + b0 + e];
                own[r][e] = x0 + 8 * cg + b0 + e < width && gy < row_end;
            }
            // rare: flag an invalid owned pixel and its forward targets (R-19)
            const bool bad = x0 + 8 * cg + am < width && gy < row_end && !(gs[hr + am] > WT(0));
            if (bad && kq == 0) {
                const int qa = ty * HWe + R + 8 * cg + am;  // counter slot (tile-relative)
                POLSAR_CHECK(qa - R >= 0 && qa + R * HWe + R < HPe);
                atomicOr(ah + HPe + qa, kBadBit);
                for (int dy = 0; dy <= R; ++dy)
                    for (int dx = (dy == 0 ? 1 : -R); dx <= R; ++dx)
                        atomicOr(ah + HPe + qa + dy * HWe + dx, kBadBit);
            }
        }

        unsigned mask[RB][2];  // per owned row: (dy > 0, dy == 0) masks over (t, e), owned pixels only
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            unsigned ob = 0u;
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int e = 0; e < 2; ++e) ob |= (unsigned)own[r][e] << (2 * t + e);
            mask[r][0] = mfull & ob;
            mask[r][1] = mzero & ob;
        }
        // forward sums as fixed-point integers too (each row's float sum rounded
        // to 2^-44): integer adds keep them off the FP64 datapath the DMMAs use
        long long acc[RB][2];
        unsigned fnan = 0u;  // (r, e) bits: a NaN weight entered that forward sum (R-19)
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[r][0] = acc[r][1] = 0ll;
        // window rows wy = hy - (first owned row): the full rows RB..R (every owned
        // row at dy in [1, R]) in a loop of their own, the edge rows around it
        auto row = [&](int wy, auto full) {
            const int hy = rg * RB + wy;
            WT rp[RB][2];
            const int jrow = mma_ring(hy + roff, HH) * HWe + 8 * cg;  // record slots (ring)
            const int jcnt = hy * HWe + 8 * cg;                      // counter slots (tile-relative)
            mma_row<Pair, NT, decltype(full)::value>(pr, rec, gs, ah, HPe, jrow, jcnt, bo, gi, mask, wy, R, ln, rp);
#pragma unroll
            for (int r = 0; r < RB; ++r)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    acc[r][e] += fixed_w(rp[r][e]);
                    fnan |= (unsigned)(rp[r][e] != rp[r][e]) << (2 * r + e);
                }
        };
        // (rows past the slab end are skipped: warp-uniform)
        const int wmax = (int)(slab_rows - y0 - rg * RB - 1 < R + RB - 1 ? slab_rows - y0 - rg * RB - 1 : R + RB - 1);
        if (POLSAR_MMA_PROBE != 1) {
            for (int wy = 0; wy < RB && wy <= wmax; ++wy) row(wy, std::false_type{});
            const int wf = R < wmax ? R : wmax;
#pragma unroll kMmaUnroll
            for (int wy = RB; wy <= wf; ++wy) row(wy, std::true_type{});
            for (int wy = R + 1 > RB ? R + 1 : RB; wy <= wmax; ++wy) row(wy, std::false_type{});
        }
        // forward sums: the 8 lanes of a C column hold disjoint window pixels
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                long long a = acc[r][e];
                a += __shfl_xor_sync(0xffffffffu, a, 4);
                a += __shfl_xor_sync(0xffffffffu, a, 8);
                a += __shfl_xor_sync(0xffffffffu, a, 16);
                const unsigned nanl = __ballot_sync(0xffffffffu, (fnan >> (2 * r + e)) & 1u);
                const bool isnan_f = (nanl & (0x11111111u << kq)) != 0u;
                if (am == 0 && own[r][e])
                    fbuf[(y0 + rg * RB + r) * width + x0 + 8 * cg + b0 + e] =
                        isnan_f ? __longlong_as_double(0x7ff8000000000000ll) : (double)a * (1.0 / (double)kFix);
            }
        __syncthreads();
        // the tile's halo-region sums in pass 2's layout; each slot is cleared
        // by the thread that writes it out (the columns HW..HWe-1 only ever hold
        // zeros: masked pairs add 0, and no flag reaches past dx = R)
        long long* dst = part + ((int64_t)by * gridDim.x + blockIdx.x) * HP;
        for (int q = threadIdx.x; q < HP; q += MMA_THREADS) {
            const int sq = (q / HW) * HWe + q % HW;
            POLSAR_CHECK(sq < HPe);
            const unsigned hi = ah[sq], lo = ah[HPe + sq];
            dst[q] = (lo & kBadBit) ? kBadSum : (long long)(((unsigned long long)hi << 22) + lo);
            ah[sq] = 0u;
            ah[HPe + sq] = 0u;
        }
    }
}

// workspace: F (N doubles) | the tiles' backward sums (pass-1 grid of tile height MMA_TY)
inline size_t mma_sym_bytes(int64_t slab_rows, int64_t width, int R) {
    return acc_sym_bytes(0, slab_rows, width, R, MMA_TY);
}

template <typename Pair, int NT>
int launch_fwd_mma(const Pair& pr, const typename Pair::S* z, int64_t ld, int64_t width, int64_t slab_rows,
                   int64_t rb, int64_t re, int R, double* fbuf, long long* part, cudaStream_t s, const char* who) {
    const FwdGrid fg = fwd_grid(width, rb, re, R, MMA_TY);
    const size_t smem = mma_fwd_smem<typename Pair::S, typename Pair::WT>(R);
    auto kern = k_window_fwd_mma<Pair, NT>;
    if (smem > K3_SMEM_MAX ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return fail(POLSAR_ENOTSUP, who);
    dim3 grid((unsigned)fg.nbx, (unsigned)((fg.nby + MMA_CHUNK - 1) / MMA_CHUNK));
    kern<<<grid, MMA_THREADS, smem, s>>>(pr, z, ld, width, slab_rows, fg.p0, re, R, fg.nby, fbuf, part);
    return POLSAR_OK;
}

// Pass 1 (NT from R) + pass 2: workspace F | the tiles' backward sums (mma_sym_bytes).
template <typename Pair>
int launch_window_mma_pair(const Pair& pr, const void* zv, int64_t ld, int64_t width, int64_t slab_rows,
                           int64_t rb, int64_t re, int R, void* wsv, void* outv, cudaStream_t s, const char* who) {
    using S = typename Pair::S;
    const S* z = (const S*)zv;
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    unsigned char* ws = (unsigned char*)wsv;
    double* fbuf = (double*)ws;
    long long* part = (long long*)(ws + up((size_t)slab_rows * width * sizeof(double)));
    int rc;
    switch (mma_nt(R)) {
        case 1: rc = launch_fwd_mma<Pair, 1>(pr, z, ld, width, slab_rows, rb, re, R, fbuf, part, s, who); break;
        case 2: rc = launch_fwd_mma<Pair, 2>(pr, z, ld, width, slab_rows, rb, re, R, fbuf, part, s, who); break;
        case 3: rc = launch_fwd_mma<Pair, 3>(pr, z, ld, width, slab_rows, rb, re, R, fbuf, part, s, who); break;
        default: rc = launch_fwd_mma<Pair, 4>(pr, z, ld, width, slab_rows, rb, re, R, fbuf, part, s, who);
    }
    if (rc != POLSAR_OK) return rc;
    launch_bwd_acc<S>(part, fbuf, width, rb, re, R, MMA_TY, outv, s);
    return launch_check(who);
}

// The log-det window (K3) with the tensor-core pass 1 (R <= V3_RMAX).
template <typename S, typename WT>
int launch_window_mma(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb, int64_t re,
                      int R, double looks, double h, void* wsv, void* outv, cudaStream_t s) {
    const double alpha = looks / (2.0 * h);
    const char* who = "polsar_window_distance: tensor-core pass 1 failed";
    if (alpha == 2.0)
        return launch_window_mma_pair(MmaLogDet<S, WT, true>{(WT)alpha}, zv, ld, width, slab_rows, rb, re, R, wsv,
                                      outv, s, who);
    return launch_window_mma_pair(MmaLogDet<S, WT, false>{(WT)alpha}, zv, ld, width, slab_rows, rb, re, R, wsv,
                                  outv, s, who);
}

// The KL window (K6) with the tensor-core pass 1 (R <= V3_RMAX).
template <typename S, typename WT>
int launch_window_kl_mma(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb, int64_t re,
                         int R, double looks, double h, void* wsv, void* outv, cudaStream_t s) {
    return launch_window_mma_pair(MmaKL<S, WT>{(WT)(looks / h)}, zv, ld, width, slab_rows, rb, re, R, wsv, outv, s,
                                  "polsar_window_kl: tensor-core pass 1 failed");
}

}  // namespace
}  // namespace polsar_impl
