// inv_det.cu -- part of libpolsar.so (B200, sm_100a); arXiv 1807.08084.
// Layout, ownership and error conventions: include/polsar.h.  Design notes:
// DESIGN.md.  Nothing here is shared with oracle/.
//
//   K1  polsar_inv_det           Alg. 2, HBM-streaming
//   K2  polsar_inv_det_cholesky  Alg. 1, l21 corrected
//   K5  polsar_inv_det_blocks    multi-frequency block-diagonal pixels (§V)
//   E2E polsar_inv_det_host      chunked H2D / kernel / D2H pipeline
#include "alg.cuh"

namespace polsar_impl {
namespace {

// --------------------------------------------------------------- K1 / K2
// Vector body: each thread owns VEC consecutive pixels, reads one 16-byte
// vector per input plane (9 x LDG.128) and writes one per output plane
// (11 x STG.128), plus VEC status bytes.  Grid-stride over groups.
template <typename S>
struct Vec;
template <>
struct Vec<float> {
    typedef float4 type;
    static constexpr int n = 4;
};
template <>
struct Vec<double> {
    typedef double2 type;
    static constexpr int n = 2;
};

#ifndef K2_VEC
#define K2_VEC Vec2f
#endif
// Alg. 1 (K2) takes 2 fp32 pixels per thread instead of 4: its DSQRT / DRCP
// sequences are latency-bound, and twice the threads hide more of it
// (measured on B200).
struct Vec2f {
    typedef float2 type;
    static constexpr int n = 2;
};
template <typename S, int ALGO>
struct VecSel {
    typedef Vec<S> V;
};
template <>
struct VecSel<float, 1> {
    typedef K2_VEC V;
};

template <typename V, typename S>
__device__ __forceinline__ void unpack(const V& v, S* x);
template <>
__device__ __forceinline__ void unpack<float2, float>(const float2& v, float* x) {
    x[0] = v.x; x[1] = v.y;
}
template <>
__device__ __forceinline__ void unpack<float4, float>(const float4& v, float* x) {
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}
template <>
__device__ __forceinline__ void unpack<double2, double>(const double2& v, double* x) {
    x[0] = v.x; x[1] = v.y;
}
__device__ __forceinline__ float4 pack4(const float* x) { return make_float4(x[0], x[1], x[2], x[3]); }
__device__ __forceinline__ double2 pack2(const double* x) { return make_double2(x[0], x[1]); }
__device__ __forceinline__ float4 packv(const float* x, float4*) { return pack4(x); }
__device__ __forceinline__ double2 packv(const double* x, double2*) { return pack2(x); }
__device__ __forceinline__ float2 packv(const float* x, float2*) { return make_float2(x[0], x[1]); }

constexpr int K1_THREADS = 128;

// (POLSAR_K2_MINB: an A/B register cap for Alg. 1 through __launch_bounds__'
// min-blocks argument; 0 = none -- an explicit 1 alone changes ptxas's register
// budget: 82 instead of 76 registers, 5 instead of 6 CTAs per SM, K2 6 % slower)
#ifndef POLSAR_K2_MINB
#define POLSAR_K2_MINB 0
#endif
#if POLSAR_K2_MINB > 0
#define K1_LAUNCH_BOUNDS(ALGO) __launch_bounds__(K1_THREADS, (ALGO) == 1 ? POLSAR_K2_MINB : 1)
#else
#define K1_LAUNCH_BOUNDS(ALGO) __launch_bounds__(K1_THREADS)
#endif
template <typename S, int ALGO, int MATH>
__device__ __forceinline__ void store_status(uint8_t* status, int64_t p, const uint8_t* st) {
    constexpr int W = VecSel<S, ALGO>::V::n;
    if constexpr (W == 4) {
        uint32_t w = (uint32_t)st[0] | ((uint32_t)st[1] << 8) | ((uint32_t)st[2] << 16) | ((uint32_t)st[3] << 24);
        *reinterpret_cast<uint32_t*>(status + p) = w;
    } else if constexpr (W == 2) {
        *reinterpret_cast<uint16_t*>(status + p) = (uint16_t)(st[0] | (st[1] << 8));
    } else {
        status[p] = st[0];
    }
}

// The product body: each thread one vector group (VEC pixels), one 16-byte
// vector per input plane (9 x LDG.128) and per output plane (11 x STG.128) +
// VEC status bytes, over a whole-batch grid (grid-stride for the remainder).
template <typename S, int ALGO, int MATH>
__global__ void K1_LAUNCH_BOUNDS(ALGO)
k_inv_det_vec(const S* __restrict__ z, S* __restrict__ out, uint8_t* __restrict__ status,
              int64_t n_groups, int64_t ld) {
    typedef typename VecSel<S, ALGO>::V VV;
    typedef typename VV::type V;
    constexpr int W = VV::n;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_groups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = g * W;
        POLSAR_CHECK(p + W <= n_groups * W && p % W == 0);
        S in[9][W];
#pragma unroll
        for (int k = 0; k < 9; ++k) unpack<V, S>(ld_stream(reinterpret_cast<const V*>(z + k * ld + p)), in[k]);
        S res[11][W];
        uint8_t st[W];
#pragma unroll
        for (int v = 0; v < W; ++v) {
            S x[9], y[11];
#pragma unroll
            for (int k = 0; k < 9; ++k) x[k] = in[k][v];
            solve_one<S, ALGO, MATH>(x, y, st[v]);
#pragma unroll
            for (int k = 0; k < 11; ++k) res[k][v] = y[k];
        }
#pragma unroll
        for (int k = 0; k < 11; ++k)
            st_stream(reinterpret_cast<V*>(out + k * ld + p), packv(res[k], (V*)nullptr));
        if (status) store_status<S, ALGO, MATH>(status, p, st);
    }
}

// Scalar path: misaligned planes and the ragged tail; same solve_one.
template <typename S, int ALGO, int MATH>
__global__ void __launch_bounds__(256)
k_inv_det_scalar(const S* __restrict__ z, S* __restrict__ out, uint8_t* __restrict__ status,
                 int64_t begin, int64_t end, int64_t ld) {
    for (int64_t p = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < end;
         p += (int64_t)gridDim.x * blockDim.x) {
        S x[9], y[11];
        uint8_t st;
#pragma unroll
        for (int k = 0; k < 9; ++k) x[k] = ld_stream(z + k * ld + p);
        solve_one<S, ALGO, MATH>(x, y, st);
#pragma unroll
        for (int k = 0; k < 11; ++k) st_stream(out + k * ld + p, y[k]);
        if (status) status[p] = st;
    }
}


template <typename S, int ALGO, int MATH>
int launch_inv_det(const void* zv, void* outv, uint8_t* status, int64_t n, int64_t ld,
                   cudaStream_t s) {
    const S* z = (const S*)zv;
    S* out = (S*)outv;
    constexpr int W = VecSel<S, ALGO>::V::n;
    bool aligned = ((uintptr_t)z % 16 == 0) && ((uintptr_t)out % 16 == 0) && (ld % W == 0) &&
                   (status == nullptr || (uintptr_t)status % W == 0);
    int64_t n_vec = aligned ? (n / W) * W : 0;
    if (n_vec > 0) {
        int64_t groups = n_vec / W;
        k_inv_det_vec<S, ALGO, MATH><<<grid_full(groups, K1_THREADS), K1_THREADS, 0, s>>>(z, out, status, groups, ld);
    }
    if (n > n_vec) {
        k_inv_det_scalar<S, ALGO, MATH>
            <<<grid_for(n - n_vec, 256), 256, 0, s>>>(z, out, status, n_vec, n, ld);
    }
    return launch_check(ALGO == ALGO_ADJ ? "polsar_inv_det: launch failed"
                                         : "polsar_inv_det_cholesky: launch failed");
}

// ------------------------------------------------ multi-frequency blocks
// PAPER.md:1043-1055 [§V]: a pixel holds nblocks Hermitian 3x3 diagonal
// blocks (one per frequency band).  Alg. 2 runs on each block; the whole
// matrix's det and det^-1 are the products of the blocks' (in the arithmetic
// type, rounded once); status is the worst block status.  Planes: input block
// b at 9b..9b+8; output block inverses at 9b..9b+8, det at 9B, det^-1 at 9B+1.
template <typename S, int MATH>
__global__ void __launch_bounds__(K1_THREADS)
k_inv_det_blocks_vec(const S* __restrict__ z, S* __restrict__ out, uint8_t* __restrict__ status,
                     int64_t n_groups, int64_t ld, int nblocks) {
    typedef typename Vec<S>::type V;
    typedef typename MathT<MATH>::type T;
    constexpr int W = Vec<S>::n;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_groups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = g * W;
        T det_all[W], t_all[W];
        uint8_t st[W];
#pragma unroll
        for (int v = 0; v < W; ++v) {
            det_all[v] = T(1);
            t_all[v] = T(1);
            st[v] = 0;
        }
        for (int b = 0; b < nblocks; ++b) {
            const S* zb = z + (int64_t)9 * b * ld;
            S* ob = out + (int64_t)9 * b * ld;
            S in[9][W];
#pragma unroll
            for (int k = 0; k < 9; ++k) unpack<V, S>(ld_stream(reinterpret_cast<const V*>(zb + k * ld + p)), in[k]);
            S res[9][W];
#pragma unroll
            for (int v = 0; v < W; ++v) {
                S x[9];
                T o[9], det, t;
#pragma unroll
                for (int k = 0; k < 9; ++k) x[k] = in[k][v];
                uint8_t s1 = solve_core<S, ALGO_ADJ, MATH>(x, o, det, t);
                st[v] = s1 > st[v] ? s1 : st[v];
                det_all[v] = MUL(det_all[v], det);
                t_all[v] = MUL(t_all[v], t);
#pragma unroll
                for (int k = 0; k < 9; ++k) res[k][v] = (S)o[k];
            }
#pragma unroll
            for (int k = 0; k < 9; ++k)
                st_stream(reinterpret_cast<V*>(ob + k * ld + p), packv(res[k], (V*)nullptr));
        }
        S dd[W], tt[W];
#pragma unroll
        for (int v = 0; v < W; ++v) {
            dd[v] = (S)det_all[v];
            tt[v] = (S)t_all[v];
        }
        S* oe = out + (int64_t)9 * nblocks * ld;
        st_stream(reinterpret_cast<V*>(oe + p), packv(dd, (V*)nullptr));
        st_stream(reinterpret_cast<V*>(oe + ld + p), packv(tt, (V*)nullptr));
        if (status) {
#pragma unroll
            for (int v = 0; v < W; ++v) status[p + v] = st[v];
        }
    }
}

template <typename S, int MATH>
__global__ void __launch_bounds__(256)
k_inv_det_blocks_scalar(const S* __restrict__ z, S* __restrict__ out, uint8_t* __restrict__ status,
                        int64_t begin, int64_t end, int64_t ld, int nblocks) {
    typedef typename MathT<MATH>::type T;
    for (int64_t p = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < end;
         p += (int64_t)gridDim.x * blockDim.x) {
        T det_all = T(1), t_all = T(1);
        uint8_t st = 0;
        for (int b = 0; b < nblocks; ++b) {
            S x[9];
            T o[9], det, t;
#pragma unroll
            for (int k = 0; k < 9; ++k) x[k] = ld_stream(z + ((int64_t)9 * b + k) * ld + p);
            uint8_t s1 = solve_core<S, ALGO_ADJ, MATH>(x, o, det, t);
            st = s1 > st ? s1 : st;
            det_all = MUL(det_all, det);
            t_all = MUL(t_all, t);
#pragma unroll
            for (int k = 0; k < 9; ++k) st_stream(out + ((int64_t)9 * b + k) * ld + p, (S)o[k]);
        }
        st_stream(out + (int64_t)9 * nblocks * ld + p, (S)det_all);
        st_stream(out + ((int64_t)9 * nblocks + 1) * ld + p, (S)t_all);
        if (status) status[p] = st;
    }
}

template <typename S, int MATH>
int launch_blocks(const void* zv, void* outv, uint8_t* status, int64_t n, int64_t ld, int nb,
                  cudaStream_t s) {
    const S* z = (const S*)zv;
    S* out = (S*)outv;
    constexpr int W = Vec<S>::n;
    bool aligned = ((uintptr_t)z % 16 == 0) && ((uintptr_t)out % 16 == 0) && (ld % W == 0);
    int64_t n_vec = aligned ? (n / W) * W : 0;
    if (n_vec > 0) {
        int64_t groups = n_vec / W;
        k_inv_det_blocks_vec<S, MATH><<<grid_full(groups, K1_THREADS), K1_THREADS, 0, s>>>(
            z, out, status, groups, ld, nb);
    }
    if (n > n_vec)
        k_inv_det_blocks_scalar<S, MATH><<<grid_for(n - n_vec, 256), 256, 0, s>>>(z, out, status, n_vec,
                                                                              n, ld, nb);
    return launch_check("polsar_inv_det_blocks: launch failed");
}

template <int ALGO>
int dispatch_inv_det(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld, int dtype,
                     void* stream) {
    if (n < 0) return fail(POLSAR_EINVAL, "n < 0");
    if (ld < n) return fail(POLSAR_EINVAL, "ld < n");
    if (n == 0) return POLSAR_OK;
    if (!z || !out) return fail(POLSAR_EINVAL, "null z or out");
    cudaStream_t s = (cudaStream_t)stream;
    switch (dtype) {
        case POLSAR_F32: return launch_inv_det<float, ALGO, MATH_F64>(z, out, status, n, ld, s);
        case POLSAR_F64:
            return ALGO == ALGO_ADJ ? launch_inv_det<double, ALGO, MATH_F64_COMP>(z, out, status, n, ld, s)
                                    : launch_inv_det<double, ALGO, MATH_F64>(z, out, status, n, ld, s);
        case POLSAR_F64_EFT:
            if constexpr (ALGO == ALGO_ADJ) return launch_inv_det<double, ALGO, MATH_F64_EFT>(z, out, status, n, ld, s);
            return fail(POLSAR_ENOTSUP, "POLSAR_F64_EFT: Alg. 2 only");
        case POLSAR_F32_PLAIN: return launch_inv_det<float, ALGO, MATH_F32>(z, out, status, n, ld, s);
        case POLSAR_F64_PLAIN: return launch_inv_det<double, ALGO, MATH_F64>(z, out, status, n, ld, s);
        default: return fail(POLSAR_EINVAL, "bad dtype");
    }
}

}  // namespace
}  // namespace polsar_impl

using namespace polsar_impl;

extern "C" {

int polsar_inv_det(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld, int dtype,
                   void* cuda_stream) {
    return dispatch_inv_det<ALGO_ADJ>(z, out, status, n, ld, dtype, cuda_stream);
}

int polsar_inv_det_cholesky(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld,
                            int dtype, void* cuda_stream) {
    return dispatch_inv_det<ALGO_CHOL>(z, out, status, n, ld, dtype, cuda_stream);
}

int polsar_inv_det_blocks(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld,
                          int nblocks, int dtype, void* cuda_stream) {
    if (n < 0) return fail(POLSAR_EINVAL, "n < 0");
    if (ld < n) return fail(POLSAR_EINVAL, "ld < n");
    if (nblocks < 1 || nblocks > 64) return fail(POLSAR_EINVAL, "nblocks out of [1, 64]");
    if (n == 0) return POLSAR_OK;
    if (!z || !out) return fail(POLSAR_EINVAL, "null z or out");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    switch (dtype) {
        case POLSAR_F32: return launch_blocks<float, MATH_F64>(z, out, status, n, ld, nblocks, s);
        case POLSAR_F64: return launch_blocks<double, MATH_F64_COMP>(z, out, status, n, ld, nblocks, s);
        case POLSAR_F64_EFT: return launch_blocks<double, MATH_F64_EFT>(z, out, status, n, ld, nblocks, s);
        case POLSAR_F32_PLAIN: return launch_blocks<float, MATH_F32>(z, out, status, n, ld, nblocks, s);
        case POLSAR_F64_PLAIN: return launch_blocks<double, MATH_F64>(z, out, status, n, ld, nblocks, s);
        default: return fail(POLSAR_EINVAL, "bad dtype");
    }
}

int64_t polsar_host_chunk_pixels(size_t ws_bytes, int dtype) {
    size_t es = (dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN || dtype == POLSAR_F64_EFT) ? 8 : 4;
    // 3 slots x (9 in + 11 out planes + 1 status byte) per pixel, chunk a
    // multiple of 64 pixels so every device plane stays 256-byte aligned
    size_t per = 3 * (20 * es + 1);
    int64_t c = (int64_t)(ws_bytes / per);
    return (c / 64) * 64;
}

int polsar_inv_det_host(const void* z_host, void* out_host, uint8_t* status_host, int64_t n,
                        int64_t ld_host, int dtype, int algo, void* dev_ws, size_t ws_bytes,
                        void* stream_h2d, void* stream_compute, void* stream_d2h) {
    if (n < 0 || ld_host < n) return fail(POLSAR_EINVAL, "bad n / ld_host");
    if (n == 0) return POLSAR_OK;
    if (!z_host || !out_host || !dev_ws) return fail(POLSAR_EINVAL, "null pointer");
    if ((uintptr_t)dev_ws % 256) return fail(POLSAR_EINVAL, "dev_ws must be 256-byte aligned");
    if (algo != 0 && algo != 1) return fail(POLSAR_EINVAL, "bad algo");
    if (dtype < POLSAR_F32 || dtype > POLSAR_F64_EFT) return fail(POLSAR_EINVAL, "bad dtype");
    if (algo == 1 && dtype == POLSAR_F64_EFT) return fail(POLSAR_ENOTSUP, "POLSAR_F64_EFT: Alg. 2 only");
    if (!stream_h2d || !stream_compute || !stream_d2h || stream_h2d == stream_compute ||
        stream_h2d == stream_d2h || stream_compute == stream_d2h)
        return fail(POLSAR_EINVAL, "three distinct non-null streams required");
    const size_t es = (dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN || dtype == POLSAR_F64_EFT) ? 8 : 4;
    const int64_t chunk = polsar_host_chunk_pixels(ws_bytes, dtype);
    if (chunk <= 0) return fail(POLSAR_EINVAL, "workspace too small");
    cudaStream_t sh = (cudaStream_t)stream_h2d, sc = (cudaStream_t)stream_compute,
                 sd = (cudaStream_t)stream_d2h;
    // 2D copies take the host plane stride as their pitch, which CUDA caps at
    // cudaDevAttrMaxPitch (2^31 - 1 B): a plane stride beyond it (fp64 with
    // ld_host >= 2^28, e.g. a UAVSAR-scale c4 image) is copied plane by plane.
    int dev = 0, max_pitch = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&max_pitch, cudaDevAttrMaxPitch, dev) != cudaSuccess)
        return fail(POLSAR_ECUDA, "polsar_inv_det_host: device query failed");
    const bool use_2d = (uint64_t)ld_host * es <= (uint64_t)max_pitch;
    auto copy_planes = [&](void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                           int planes, cudaMemcpyKind kind, cudaStream_t st) -> bool {
        if (use_2d) return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, planes, kind, st) == cudaSuccess;
        for (int k = 0; k < planes; ++k)
            if (cudaMemcpyAsync((unsigned char*)dst + k * dpitch, (const unsigned char*)src + k * spitch,
                                width, kind, st) != cudaSuccess)
                return false;
        return true;
    };
    // slot layout: [9 in planes][11 out planes][status], each plane `chunk` elements
    const size_t slot_bytes = (size_t)chunk * (20 * es + 1);
    cudaEvent_t ev[9];
    int n_ev = 0;
    for (; n_ev < 9; ++n_ev)
        if (cudaEventCreateWithFlags(&ev[n_ev], cudaEventDisableTiming) != cudaSuccess) break;
    int rc = n_ev == 9 ? POLSAR_OK : fail(POLSAR_ECUDA, "polsar_inv_det_host: event creation failed");
    cudaEvent_t *ev_in = ev, *ev_k = ev + 3, *ev_out = ev + 6;
    const int64_t n_chunks = (n + chunk - 1) / chunk;
    for (int64_t c = 0; c < n_chunks && rc == POLSAR_OK; ++c) {
        const int slot = (int)(c % 3);
        const int64_t p0 = c * chunk;
        const int64_t m = (n - p0) < chunk ? (n - p0) : chunk;
        unsigned char* base = (unsigned char*)dev_ws + slot * slot_bytes;
        unsigned char* din = base;
        unsigned char* dout = base + (size_t)9 * chunk * es;
        uint8_t* dst = (uint8_t*)(base + (size_t)20 * chunk * es);
        if (c >= 3) cudaStreamWaitEvent(sh, ev_out[slot], 0);  // slot drained by its D2H
        if (!copy_planes(din, chunk * es, (const unsigned char*)z_host + p0 * es, ld_host * es, m * es, 9,
                         cudaMemcpyHostToDevice, sh)) {
            rc = fail(POLSAR_ECUDA, "polsar_inv_det_host: H2D copy failed");
            break;
        }
        cudaEventRecord(ev_in[slot], sh);
        cudaStreamWaitEvent(sc, ev_in[slot], 0);
        rc = (algo == 0 ? polsar_inv_det : polsar_inv_det_cholesky)(
            din, dout, status_host ? dst : nullptr, m, chunk, dtype, sc);
        if (rc != POLSAR_OK) break;
        cudaEventRecord(ev_k[slot], sc);
        cudaStreamWaitEvent(sd, ev_k[slot], 0);
        if (!copy_planes((unsigned char*)out_host + p0 * es, ld_host * es, dout, chunk * es, m * es, 11,
                         cudaMemcpyDeviceToHost, sd)) {
            rc = fail(POLSAR_ECUDA, "polsar_inv_det_host: D2H copy failed");
            break;
        }
        if (status_host &&
            cudaMemcpyAsync(status_host + p0, dst, m, cudaMemcpyDeviceToHost, sd) != cudaSuccess) {
            rc = fail(POLSAR_ECUDA, "polsar_inv_det_host: D2H status copy failed");
            break;
        }
        cudaEventRecord(ev_out[slot], sd);
    }
    // Synchronous on every path: nothing this call enqueued may still read the
    // caller's host buffers or write dev_ws after it returns, so all three
    // streams are drained, error paths included.
    const cudaStream_t all[3] = {sh, sc, sd};
    for (int i = 0; i < 3; ++i)
        if (cudaStreamSynchronize(all[i]) != cudaSuccess && rc == POLSAR_OK)
            rc = fail(POLSAR_ECUDA, "polsar_inv_det_host: stream error");
    for (int i = 0; i < n_ev; ++i) cudaEventDestroy(ev[i]);
    return rc;
}

}  // extern "C"
