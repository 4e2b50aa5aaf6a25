// nlm.cu -- part of libpolsar.so (B200, sm_100a); arXiv 1807.08084.
// Layout, ownership and error conventions: include/polsar.h.  Design notes:
// DESIGN.md.  Nothing here is shared with oracle/.
//
//   K4  polsar_nlm_filter   non-local-means filter output: the symmetric form
//                           (pass 1 of window_core.cuh + the TMA-fed gather)
//                           and the direct form
#include <vector>

#include "window_core.cuh"

namespace polsar_impl {
namespace {

// ------------------------------------------------------------------------
// K4: non-local-means filter output (the NLM filter with
// stochastic distances of PAPER.md:77-80 [§I]).  Same pair weights as K3 and
// in the same pass, accumulated with the window pixels themselves:
//   W_i = sum_j w_ij,   Zhat_i = sum_j w_ij Z_j / W_i   (9 packed planes).
// Layout and staging as k_window_sum; the weighted sums accumulate in the
// pair-determinant type (fp64 for the default modes: one F2F, one DADD and
// nine DFMA per pair on top of the determinant).
template <typename S, typename T, typename WT, int TY, int RB>
__global__ void __launch_bounds__(K3_TX * TY / RB, 1)
k_nlm_sum(const S* __restrict__ z, int64_t ld, int64_t width, int64_t slab_rows,
          int64_t row_begin, int64_t row_end, int R, const WT* __restrict__ g, double alpha_d,
          int alpha_is_2, S* __restrict__ out_w, S* __restrict__ out_z, int64_t ld_out) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int HW = K3_TX + 2 * R;
    const int HH = TY + 2 * R;
    const int HP = HW * HH;
    T* sz = reinterpret_cast<T*>(smem_raw);  // HP records of 10 T (load_rec)

    const int64_t x0 = (int64_t)blockIdx.x * K3_TX;
    const int64_t y0 = row_begin + (int64_t)blockIdx.y * TY;
    for (int q = threadIdx.x; q < HP; q += blockDim.x) {
        int hy = q / HW, hx = q % HW;
        int64_t gy = y0 - R + hy, gx = x0 - R + hx;
        bool in = gy >= 0 && gy < slab_rows && gx >= 0 && gx < width;
        int64_t p = in ? gy * width + gx : 0;
        T* rec = sz + 10 * q;
#pragma unroll
        for (int k = 0; k < 9; ++k) rec[k] = in ? (T)z[k * ld + p] : T(0);
        rec[9] = pack_g<T, WT>(in ? g[p] : WT(0));
    }
    __syncthreads();

    const int tx = threadIdx.x % K3_TX;
    const int ty0 = (threadIdx.x / K3_TX) * RB;
    const int64_t gx = x0 + tx;
    T zi[RB][9], accz[RB][9], accw[RB];
    WT gi[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        load_rec(sz + 10 * ((ty0 + r + R) * HW + (tx + R)), zi[r], gi[r]);
#pragma unroll
        for (int k = 0; k < 9; ++k) accz[r][k] = T(0);
        accw[r] = T(0);
    }
    const WT alpha = (WT)alpha_d;
    const bool a2 = alpha_is_2 != 0;
    const bool interior_x = (x0 - R >= 0) && (x0 + K3_TX + R <= width);

    for (int wy = -R; wy <= R + RB - 1; ++wy) {
        const int64_t gyj = y0 + ty0 + wy;
        if (gyj < 0 || gyj >= slab_rows) continue;  // warp-uniform
        const int hy = ty0 + wy + R;
        const T* rec = sz + 10 * (hy * HW + tx);  // neighbour wx = -R
        bool rok[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) rok[r] = (wy - r >= -R) && (wy - r <= R);  // warp-uniform
        for (int wx = -R; wx <= R; ++wx, rec += 10) {
            T zj[9];
            WT gj;
            POLSAR_CHECK(hy >= 0 && hy < HH && tx + wx + R >= 0 && tx + wx + R < HW);
            load_rec(rec, zj, gj);
            const bool colok = interior_x || (gx + wx >= 0 && gx + wx < width);
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if (rok[r]) {
                    WT w = pair_w<T, WT>(zi[r], gi[r], zj, gj, alpha, a2);
                    const T wt = colok ? (T)w : T(0);
                    accw[r] = ADD(accw[r], wt);
#pragma unroll
                    for (int k = 0; k < 9; ++k) accz[r][k] = FMA(wt, zj[k], accz[r][k]);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int64_t gy = y0 + ty0 + r;
        if (gx < width && gy < row_end) {
            const int64_t o = (gy - row_begin) * width + gx;
            if (out_w) out_w[o] = (S)accw[r];
#pragma unroll
            for (int k = 0; k < 9; ++k) out_z[k * ld_out + o] = (S)(accz[r][k] / accw[r]);
        }
    }
}

template <typename S, typename T, typename WT>
int launch_nlm(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb, int64_t re,
               int R, double looks, double h, void* ws, void* out_w, void* out_z, int64_t ld_out,
               cudaStream_t s) {
    const S* z = (const S*)zv;
    WT* g = (WT*)ws;
    const int64_t n = slab_rows * width;
    k_window_prep<S, T, WT><<<grid_for(n, 256), 256, 0, s>>>(z, ld, n, g);
    const double alpha = looks / (2.0 * h);
    auto nlm_smem = [R](int ty) { return (size_t)(K3_TX + 2 * R) * (ty + 2 * R) * 10 * sizeof(T); };
    int TY = 16;
    size_t smem = nlm_smem(16);
    if (smem > K3_SMEM_MAX) {
        TY = 8;
        smem = nlm_smem(8);
        if (smem > K3_SMEM_MAX)
            return fail(POLSAR_ENOTSUP, "polsar_nlm_filter: radius too large for shared memory");
    }
    auto kern = TY == 16 ? k_nlm_sum<S, T, WT, 16, 2> : k_nlm_sum<S, T, WT, 8, 2>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return fail(POLSAR_ENOTSUP, "polsar_nlm_filter: shared memory request too large");
    dim3 grid((unsigned)((width + K3_TX - 1) / K3_TX), (unsigned)((re - rb + TY - 1) / TY));
    kern<<<grid, K3_TX * TY / 2, smem, s>>>(z, ld, width, slab_rows, rb, re, R, g, alpha,
                                            alpha == 2.0 ? 1 : 0, (S*)out_w, (S*)out_z, ld_out);
    return launch_check("polsar_nlm_filter: launch failed");
}

// ------------------------------------------------------------------------
// K4, symmetric form (default for R <= V3_RMAX): pass 1 (k_window_fwd with
// the log-det pair policy) stores every unordered pair's weight once; this
// gather pass then forms, for every output pixel i,
//   W_i = sum_j w_ij,   Zhat_i = sum_j w_ij Z_j / W_i
// reading w_ij from the weight planes: with j = i + (dy, dx),
//   forward  (dy > 0, or dy = 0 and dx > 0): w_ij = wbuf[fwd_index(dy, dx)][i]
//   backward (the mirror):                   w_ij = wbuf[fwd_index(-dy, -dx)][j]
//   j = i:                                   w_ii = 1 (d_ii = 0)
// Along a neighbour row both offsets are linear in dx: forward
// fwd_index(dy, 0) N + i + dx N, backward fwd_index(-dy, 0) N + j0 + dx (1 - N)
// (j0 = the neighbour at dx = 0; for dy = 0, fwd_index(0, 0) = -1 and j0 = i).
// So the pass is pure data movement plus 9 FMAs per ordered pair in the
// storage precision: no FP64 determinant work at all (the direct form
// k_nlm_sum evaluates every ordered pair's determinant, 29 FP64 ops, plus 10
// FP64 accumulations).
//
// A CTA owns NLM_COLS = NLM_TX - AL columns x RB rows (AL = 16 / sizeof(WT));
// each thread one column and RB rows, and the CTA walks the window rows its
// pixels share.  For each window row:
//  * the weights: for every owned row r and dx, the CTA's weights form one
//    contiguous run of a weight plane (at i for forward pairs, at j = i +
//    (dy, dx) for backward ones), fetched by TMA as one 1-D tile of NLM_TX
//    elements of a tensor map over the whole weight buffer.  TMA needs a
//    16-byte aligned start (measured, tools/micro/tma1d_test.cu); with the
//    padded plane layout (weight_pitch) forward runs start aligned and a
//    backward run at dx starts m(dx) = dx mod AL elements past an aligned
//    point, so its tile is fetched from there and read at offset m(dx).
//    Tiles of rows that do not pair with this window row, and the j = i
//    tile, are fetched from an out-of-range coordinate: TMA zero-fills them.
//    RB (2R + 1) tiles per row, one per thread, completing on the stage's
//    mbarrier; NLM_NS row stages in flight.
//  * the neighbours Z_j: the row's 9 planes over NLM_TX + 2 V3_RMAX columns
//    (zero-filled outside the image), staged by cp.async into a ring of
//    NLM_NZ rows; each Z_j is read from shared memory once per thread and
//    serves its RB pairs.
// Window rows above the owned rows are all-backward, rows below all-forward
// (fully unrolled, branch-free); the RB rows in between mix both laws and
// the self pair, whose w_ii = 1 is added after the row.  Columns within R of
// the image edge mask the out-of-image pairs.  Shared-memory reads are
// conflict-free (consecutive lanes, consecutive columns).  Per window row the
// pairs are summed in WT (2R + 1 terms), then added to fp64 totals in a fixed
// order per pixel: bit-reproducible, and slab decompositions are exact.
#ifndef POLSAR_NLM_RB
#define POLSAR_NLM_RB 2
#endif
#ifndef POLSAR_NLM_NS
#define POLSAR_NLM_NS 2
#endif
constexpr int NLM_NZ = 3;                      // Z row buffers
constexpr int NLM_ZW = NLM_TX + 2 * V3_RMAX;   // staged Z columns x0 - 12 .. x0 + 139
// Z record of one staged column: the 9 planes padded to 16-byte vectors
// (12 floats / 10 doubles; strides of 12 and 20 words keep the 16-byte
// loads of 8 consecutive lanes on distinct banks)
template <typename S>
#ifndef POLSAR_NLM_REC9
#define POLSAR_NLM_REC9 1
#endif
struct NlmRec {
    // (POLSAR_NLM_REC9: fp32 records unpadded, 9 words, read as 9 scalars)
    static constexpr int n = sizeof(S) == 4 ? (POLSAR_NLM_REC9 ? 9 : 12) : 10;
};
constexpr int NLM_OOB = -(1 << 30);            // a TMA coordinate whose tile is all zero-fill

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    int src_bytes = valid ? 4 : 0;  // 0: zero-fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" :: "r"(sa), "l"(gmem), "r"(src_bytes)
                 : "memory");
}

// stage window row gy (9 planes, columns x0 - V3_RMAX .. x0 + NLM_TX + V3_RMAX - 1)
template <typename S>
__device__ __forceinline__ void nlm_stage_row(S* dst, const S* __restrict__ z, int64_t ld,
                                              int64_t width, int64_t gy, int64_t x0) {
    const S* src = z + gy * width;
    constexpr int ZR = NlmRec<S>::n;
    for (int c = threadIdx.x; c < NLM_ZW; c += NLM_TX) {
        const int64_t gx = x0 - V3_RMAX + c;
        const bool ok = gx >= 0 && gx < width;
        const S* sp = src + (ok ? gx : 0);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            if constexpr (sizeof(S) == 4)
                cp_async4(dst + c * ZR + k, sp + k * ld, ok);
            else
                cp_async8(dst + c * ZR + k, sp + k * ld, ok);
        }
    }
}

template <int AL>
__host__ __device__ __forceinline__ int nlm_mis(int wx) { return wx & (AL - 1); }

// TMA coordinates (pixel index within the plane, a multiple of AL; plane)
// of the tile of owned row yi at dx for window row gy; plane NLM_OOB when
// the row does not pair (the tile zero-fills).
template <int AL>
__device__ __forceinline__ int2 nlm_tile_coord(int64_t gy, int64_t yi, int wx, int R, int64_t wp,
                                               int64_t x0, int64_t row_end) {
    const int64_t dy = gy - yi;
    if (yi >= row_end || dy < -R || dy > R || (dy == 0 && wx == 0)) return make_int2(0, NLM_OOB);
    const int ad = (int)(dy < 0 ? -dy : dy);
    const int fi = ad == 0 ? -1 : R + (ad - 1) * (2 * R + 1) + R;  // fwd_index(|dy|, 0)
    if (dy > 0 || (dy == 0 && wx > 0)) return make_int2((int)(yi * wp + x0), fi + wx);  // forward: at i
    return make_int2((int)(gy * wp + x0 + wx - nlm_mis<AL>(wx)), fi - wx);           // backward: at j
}

template <typename WT>
size_t nlm_smem_bytes(int R, int RB, int NS, size_t s_bytes) {
    return 128 + (size_t)NS * RB * (2 * R + 1) * NLM_TX * sizeof(WT) +
           (size_t)NLM_NZ * NLM_ZW * (s_bytes == 4 ? NlmRec<float>::n : NlmRec<double>::n) * s_bytes;
}

// One window row for one thread: K = 0 all rows backward, 1 all forward,
// 2 mixed (cls[r]: 0 backward, 1 forward, 2 the pixel's own row, backward for
// dx < 0 and forward for dx > 0; its dx = 0 tile is zero); EDGE masks
// out-of-image columns.
__device__ __forceinline__ void nlm_load_rec(const float* p, float (&zj)[9]) {
#if POLSAR_NLM_REC9
#pragma unroll
    for (int k = 0; k < 9; ++k) zj[k] = p[k];
#else
    const float4 a = reinterpret_cast<const float4*>(p)[0];
    const float4 b = reinterpret_cast<const float4*>(p)[1];
    zj[0] = a.x; zj[1] = a.y; zj[2] = a.z; zj[3] = a.w;
    zj[4] = b.x; zj[5] = b.y; zj[6] = b.z; zj[7] = b.w;
    zj[8] = p[8];
#endif
}
__device__ __forceinline__ void nlm_load_rec(const double* p, double (&zj)[9]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double2 v = reinterpret_cast<const double2*>(p)[k];
        zj[2 * k] = v.x;
        zj[2 * k + 1] = v.y;
    }
    zj[8] = p[8];
}

#ifndef POLSAR_NLM_UNROLL
#define POLSAR_NLM_UNROLL 4
#endif
constexpr int kNlmUnroll = POLSAR_NLM_UNROLL;
template <typename WT, int AL, int RB, int K, bool EDGE, int RC>
__device__ __forceinline__ void nlm_row(const WT* __restrict__ wrow, const WT* __restrict__ zrowT, int R,
                                        const int (&cls)[RB], int64_t x, int64_t width, WT (&pw)[RB],
                                        WT (&pz)[RB][9]) {
    // wrow: w(r, dx) tile at wrow[(r * (2R + 1) + dx) * NLM_TX] (+ m(dx) for backward tiles)
    // zrowT: the record of Z_j(dx) at zrowT + dx * ZR
    // (a rolled loop: the per-dx body is 9 + RB loads and 10 RB FMA/adds; a
    // fully unrolled row measured slower, instruction-fetch bound)
    const int WX = RC > 0 ? 2 * RC + 1 : 2 * R + 1;
    constexpr int ZR = NlmRec<WT>::n;
    const WT* zp = zrowT - R * ZR;
    const WT* wp = wrow - R * NLM_TX;
#pragma unroll(kNlmUnroll)
    for (int wx = -R; wx <= R; ++wx, zp += ZR, wp += NLM_TX) {
        WT zj[9];
        nlm_load_rec(zp, zj);
        const bool colok = !EDGE || (x + wx >= 0 && x + wx < width);
        const int m = nlm_mis<AL>(wx);
        const WT* wpm = wp + (K == 1 ? 0 : m);
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            const WT* a;
            if constexpr (K == 2)
                a = (cls[r] == 0 || (cls[r] == 2 && wx < 0)) ? wpm : wp;
            else
                a = wpm;
            WT w = a[r * WX * NLM_TX];
            if constexpr (EDGE) w = colok ? w : WT(0);
            pw[r] = ADD(pw[r], w);
#pragma unroll
            for (int k = 0; k < 9; ++k) pz[r][k] = FMA(w, zj[k], pz[r][k]);
        }
    }
}

template <typename S, typename WT, int RC, int RB, int NS>
__global__ void __launch_bounds__(NLM_TX)
k_nlm_gather(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap wmap2,
             const S* __restrict__ z, int64_t ld,
             int64_t width, int64_t slab_rows, int64_t row_begin, int64_t row_end, int R_rt,
             S* __restrict__ out_w, S* __restrict__ out_z, int64_t ld_out) {
    constexpr int AL = 16 / sizeof(WT);
    constexpr int COLS = NLM_TX - AL;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int R = RC > 0 ? RC : R_rt;
    const int WX = 2 * R + 1;
    const int SW = RB * WX * NLM_TX;  // weights per stage
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    WT* wst = reinterpret_cast<WT*>(smem_raw + 128);
    S* zs = reinterpret_cast<S*>(smem_raw + 128 + (size_t)NS * SW * sizeof(WT));
    const CUtensorMap* pmap = &wmap;
    const CUtensorMap* pmap2 = &wmap2;
    constexpr int ZREC = NLM_ZW * NlmRec<S>::n;  // one staged row

    const int64_t wp = weight_pitch<WT>(width);
    const int64_t x0 = (int64_t)blockIdx.x * COLS;
    const int tx = threadIdx.x;
    const int64_t x = x0 + tx;
    const int64_t y0 = row_begin + (int64_t)blockIdx.y * RB;
    const bool colin = tx < COLS && x < width;  // (other threads still stage rows)
    const bool inx = x - R >= 0 && x + R < width;
    const int64_t ga = y0 - R > 0 ? y0 - R : 0;
    const int64_t gb = (y0 + RB - 1 + R) < slab_rows - 1 ? (y0 + RB - 1 + R) : slab_rows - 1;
    const int nrows = (int)(gb - ga + 1);

    if (tx == 0) {
        for (int st = 0; st < NS; ++st) mbar_init(&bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // weights of window row q -> stage q % NS: thread t fetches tile t = (r, dx)
    auto issue = [&](int q) {
        const int64_t gy = ga + q;
        const int st = q % NS;
        if (tx == 0) mbar_expect_tx(&bar[st], (uint32_t)(SW * sizeof(WT)));
        for (int t = tx; t < RB * WX; t += NLM_TX) {
            const int r = t / WX, wx = t - r * WX - R;
            const int64_t yi = y0 + r, dy = gy - yi;
            if (yi >= row_end || dy < -R || dy > R || dy > 0) {
                // a whole forward row (the 2R + 1 planes fwd_index(dy, -R..R) at i: one
                // 2-D box), or a row that does not pair (one out-of-range box: zeros)
                if (wx == -R) {
                    const bool act = yi < row_end && dy >= -R && dy <= R;
                    const int c0 = act ? (int)(yi * wp + x0) : 0;
                    const int c1 = act ? R + (int)(dy - 1) * (2 * R + 1) : NLM_OOB;
                    tma_load_2d(wst + (size_t)st * SW + (size_t)t * NLM_TX, pmap2, c0, c1, &bar[st]);
                }
            } else {
                const int2 c = nlm_tile_coord<AL>(gy, yi, wx, R, wp, x0, row_end);
                tma_load_2d(wst + (size_t)st * SW + (size_t)t * NLM_TX, pmap, c.x, c.y, &bar[st]);
            }
        }
    };
#pragma unroll
    for (int q = 0; q < NS - 1; ++q)
        if (q < nrows) issue(q);
#pragma unroll
    for (int q = 0; q < NLM_NZ - 1; ++q) {
        if (q < nrows) nlm_stage_row<S>(zs + (size_t)q * ZREC, z, ld, width, ga + q, x0);
        cp_async_commit();
    }

    double tw[RB], tz[RB][9];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        tw[r] = 0.0;
#pragma unroll
        for (int k = 0; k < 9; ++k) tz[r][k] = 0.0;
    }
    for (int q = 0; q < nrows; ++q) {
        const int64_t gy = ga + q;
        // refill the stage and ring slot row q - 1 used (released by the barrier that ended it)
        if (q + NS - 1 < nrows) issue(q + NS - 1);
        if (q + NLM_NZ - 1 < nrows)
            nlm_stage_row<S>(zs + (size_t)((q + NLM_NZ - 1) % NLM_NZ) * ZREC, z, ld, width,
                             gy + NLM_NZ - 1, x0);
        cp_async_commit();
        cp_async_wait<NLM_NZ - 1>();
        __syncthreads();
        mbar_wait(&bar[q % NS], (uint32_t)((q / NS) & 1));
        if (colin) {
            // records dx = -R..R of column tx, and tile elements tx + m(dx) (m < AL)
            POLSAR_CHECK(tx + V3_RMAX - R >= 0 && tx + V3_RMAX + R < NLM_ZW && tx + AL - 1 < NLM_TX);
            const S* zrow = zs + (size_t)(q % NLM_NZ) * ZREC + (tx + V3_RMAX) * NlmRec<S>::n;
            const WT* wrow = wst + (size_t)(q % NS) * SW + tx + R * NLM_TX;
            WT pw[RB], pz[RB][9];
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                pw[r] = WT(0);
#pragma unroll
                for (int k = 0; k < 9; ++k) pz[r][k] = WT(0);
            }
            int cls[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) cls[r] = gy < y0 + r ? 0 : (gy > y0 + r ? 1 : 2);
            const int K = gy < y0 ? 0 : (gy >= y0 + RB ? 1 : 2);  // CTA-uniform
            static_assert(sizeof(S) == sizeof(WT), "the gather reads Z in the weight type");
            const WT* zr = reinterpret_cast<const WT*>(zrow);
            if (inx) {
                if (K == 0) nlm_row<WT, AL, RB, 0, false, RC>(wrow, zr, R, cls, x, width, pw, pz);
                else if (K == 1) nlm_row<WT, AL, RB, 1, false, RC>(wrow, zr, R, cls, x, width, pw, pz);
                else nlm_row<WT, AL, RB, 2, false, RC>(wrow, zr, R, cls, x, width, pw, pz);
            } else {
                if (K == 0) nlm_row<WT, AL, RB, 0, true, RC>(wrow, zr, R, cls, x, width, pw, pz);
                else if (K == 1) nlm_row<WT, AL, RB, 1, true, RC>(wrow, zr, R, cls, x, width, pw, pz);
                else nlm_row<WT, AL, RB, 2, true, RC>(wrow, zr, R, cls, x, width, pw, pz);
            }
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if (gy == y0 + r && y0 + r < row_end) {  // the self pair: w_ii = 1 (d_ii = 0)
                    pw[r] = ADD(pw[r], WT(1));
#pragma unroll
                    for (int k = 0; k < 9; ++k) pz[r][k] = ADD(pz[r][k], zr[k]);
                }
                // a row that does not pair with this window row ran on zero weights
                // but its Z (0 * NaN): skip it
                const int64_t dyr = gy - (y0 + r);
                if (y0 + r < row_end && dyr >= -R && dyr <= R) {
                    tw[r] = __dadd_rn(tw[r], (double)pw[r]);
#pragma unroll
                    for (int k = 0; k < 9; ++k) tz[r][k] = __dadd_rn(tz[r][k], (double)pz[r][k]);
                }
            }
        }
        __syncthreads();  // stage q % NS and ring slot q % NLM_NZ are refilled from row q + 1
    }
    if (!colin) return;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int64_t yi = y0 + r;
        if (yi < row_end) {
            const int64_t o = (yi - row_begin) * width + x;
            if (out_w) out_w[o] = (S)tw[r];
#pragma unroll
            for (int k = 0; k < 9; ++k) out_z[k * ld_out + o] = (S)__ddiv_rn(tz[r][k], tw[r]);
        }
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        return (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                   ? (PFN_cuTensorMapEncodeTiled_v12000)p
                   : nullptr;
    }();
    return fn;
}

// 2-D view of the weight planes (P x planes, row stride P) with a box of
// NLM_TX x rows: rows = 1 for single tiles, 2R + 1 for a forward row's
// consecutive planes in one transfer.  False if the driver call is
// unavailable or refuses.  (A 1-D map over the flattened buffer also works
// but caps the buffer at 2^31 elements of 32-bit coordinates.)
template <typename WT>
bool nlm_weight_map2(CUtensorMap* m, const WT* wbuf, int64_t P, int planes, int rows) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dim[2] = {(cuuint64_t)P, (cuuint64_t)planes};
    cuuint64_t st[1] = {(cuuint64_t)P * sizeof(WT)};
    cuuint32_t box[2] = {(cuuint32_t)NLM_TX, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, sizeof(WT) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                     (void*)wbuf, dim, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <typename S, typename T, typename WT>
int launch_nlm_sym(const void* zv, int64_t ld, int64_t width, int64_t slab_rows, int64_t rb,
                   int64_t re, int R, double looks, double h, void* wsv, void* out_w, void* out_z,
                   int64_t ld_out, cudaStream_t s) {
    const S* z = (const S*)zv;
    const int64_t n = slab_rows * width;
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    unsigned char* ws = (unsigned char*)wsv;
    WT* g = (WT*)ws;
    double* fbuf = (double*)(ws + up(n * sizeof(WT)));
    WT* wbuf = (WT*)(ws + up(n * sizeof(WT)) + up(n * sizeof(double)));
    constexpr int RB = sizeof(WT) == 4 ? POLSAR_NLM_RB : 2;
    constexpr int NS = POLSAR_NLM_NS;
    CUtensorMap wmap, wmap2;
    const int64_t P = slab_rows * weight_pitch<WT>(width);
    if (!nlm_weight_map2<WT>(&wmap, wbuf, P, fwd_count(R), 1) ||
        !nlm_weight_map2<WT>(&wmap2, wbuf, P, fwd_count(R), 2 * R + 1))
        return fail(POLSAR_ECUDA, "polsar_nlm_filter: cuTensorMapEncodeTiled failed");
    const size_t smem = nlm_smem_bytes<WT>(R, RB, NS, sizeof(S));
    auto kern = R == 11 ? k_nlm_gather<S, WT, 11, RB, NS> : k_nlm_gather<S, WT, 0, RB, NS>;
    if (smem > K3_SMEM_MAX ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return fail(POLSAR_ENOTSUP, "polsar_nlm_filter: shared memory request too large");
    k_window_prep<S, T, WT><<<grid_for(n, 256), 256, 0, s>>>(z, ld, n, g);
    const double alpha = looks / (2.0 * h);
    int rc = alpha == 2.0
                 ? launch_fwd<LogDetPair<S, T, WT, 1>, POLSAR_SYM_TY, POLSAR_SYM_RB>(
                       LogDetPair<S, T, WT, 1>{z, ld, g, (WT)alpha, true}, width, slab_rows, rb, re, R,
                       wbuf, fbuf, s, "polsar_nlm_filter: shared memory request too large")
                 : launch_fwd<LogDetPair<S, T, WT, 0>, POLSAR_SYM_TY, POLSAR_SYM_RB>(
                       LogDetPair<S, T, WT, 0>{z, ld, g, (WT)alpha, false}, width, slab_rows, rb, re, R,
                       wbuf, fbuf, s, "polsar_nlm_filter: shared memory request too large");
    if (rc != POLSAR_OK) return rc;
    constexpr int COLS = NLM_TX - 16 / (int)sizeof(WT);
    dim3 grid((unsigned)((width + COLS - 1) / COLS), (unsigned)((re - rb + RB - 1) / RB));
    kern<<<grid, NLM_TX, smem, s>>>(wmap, wmap2, z, ld, width, slab_rows, rb, re, R, (S*)out_w, (S*)out_z, ld_out);
    return launch_check("polsar_nlm_filter: launch failed");
}

}  // namespace
}  // namespace polsar_impl

using namespace polsar_impl;

extern "C" {

int polsar_nlm_filter(const void* z, int64_t ld, int64_t width, int64_t slab_rows,
                      int64_t out_row_begin, int64_t out_row_end, int radius, double looks,
                      double h, void* workspace, void* out_w, void* out_z, int64_t ld_out,
                      int dtype, void* cuda_stream) {
    if (!slab_size_ok(slab_rows, width)) return fail(POLSAR_EINVAL, "negative size or slab_rows*width > 2^40");
    if (out_row_begin < 0 || out_row_end < out_row_begin || out_row_end > slab_rows)
        return fail(POLSAR_EINVAL, "bad output row range");
    if (radius < 0 || radius > 16) return fail(POLSAR_EINVAL, "radius out of [0, 16]");
    if (!(looks > 0) || !(h > 0)) return fail(POLSAR_EINVAL, "looks and h must be > 0");
    if (ld < slab_rows * width) return fail(POLSAR_EINVAL, "ld < slab_rows*width");
    if (ld_out < (out_row_end - out_row_begin) * width) return fail(POLSAR_EINVAL, "ld_out too small");
    if (width == 0 || out_row_end == out_row_begin) return POLSAR_OK;
    if (!z || !workspace || !out_z) return fail(POLSAR_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (dtype == POLSAR_F64_EFT) return fail(POLSAR_ENOTSUP, "POLSAR_F64_EFT: inverse/det entry points only");
    // the symmetric form, band by band (NLM_BAND output rows, each band a
    // sub-slab with its R-row halos; the workspace covers one band); its
    // gather addresses a weight plane with 32-bit TMA coordinates
    const int64_t band_rows = nlm_band_slab_rows(slab_rows, radius);
    if (nlm_sym_ok(radius) && tensor_map_encoder() &&
        band_rows * (width + 4) + 2 * NLM_TX < ((int64_t)1 << 31)) {
        const size_t es = (dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN) ? 8 : 4;
        for (int64_t b0 = out_row_begin; b0 < out_row_end; b0 += NLM_BAND) {
            const int64_t b1 = b0 + NLM_BAND < out_row_end ? b0 + NLM_BAND : out_row_end;
            const int64_t s0 = b0 - radius > 0 ? b0 - radius : 0;
            const int64_t s1 = b1 + radius < slab_rows ? b1 + radius : slab_rows;
            const void* zb = (const unsigned char*)z + (size_t)(s0 * width) * es;
            void* wb = out_w ? (void*)((unsigned char*)out_w + (size_t)((b0 - out_row_begin) * width) * es) : nullptr;
            void* ob = (unsigned char*)out_z + (size_t)((b0 - out_row_begin) * width) * es;
            int rc;
            switch (dtype) {
                case POLSAR_F32:
                    rc = launch_nlm_sym<float, double, float>(zb, ld, width, s1 - s0, b0 - s0, b1 - s0, radius, looks,
                                                              h, workspace, wb, ob, ld_out, s);
                    break;
                case POLSAR_F64:
                case POLSAR_F64_PLAIN:
                    rc = launch_nlm_sym<double, double, double>(zb, ld, width, s1 - s0, b0 - s0, b1 - s0, radius,
                                                                looks, h, workspace, wb, ob, ld_out, s);
                    break;
                case POLSAR_F32_PLAIN:
                    rc = launch_nlm_sym<float, float, float>(zb, ld, width, s1 - s0, b0 - s0, b1 - s0, radius, looks,
                                                             h, workspace, wb, ob, ld_out, s);
                    break;
                default: return fail(POLSAR_EINVAL, "bad dtype");
            }
            if (rc != POLSAR_OK) return rc;
        }
        return POLSAR_OK;
    }
    switch (dtype) {
        case POLSAR_F32:
            return launch_nlm<float, double, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                    radius, looks, h, workspace, out_w, out_z, ld_out, s);
        case POLSAR_F64:
        case POLSAR_F64_PLAIN:
            return launch_nlm<double, double, double>(z, ld, width, slab_rows, out_row_begin,
                                                      out_row_end, radius, looks, h, workspace, out_w,
                                                      out_z, ld_out, s);
        case POLSAR_F32_PLAIN:
            return launch_nlm<float, float, float>(z, ld, width, slab_rows, out_row_begin, out_row_end,
                                                   radius, looks, h, workspace, out_w, out_z, ld_out, s);
        default: return fail(POLSAR_EINVAL, "bad dtype");
    }
}

}  // extern "C"
