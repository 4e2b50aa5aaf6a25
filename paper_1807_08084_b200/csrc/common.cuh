// common.cuh -- part of libpolsar.so (B200, sm_100a); arXiv 1807.08084.
// Layout, ownership and error conventions: include/polsar.h.  Design notes:
// DESIGN.md.  Nothing here is shared with oracle/.
//
// Shared device helpers: round-to-nearest arithmetic overloads, streaming
// 16-byte I/O, the packed Hermitian type, launch-geometry and error helpers.
//
// Bit-stability: every floating-point operation of the per-matrix device
// functions is an explicit round-to-nearest intrinsic (__fma_rn, __dmul_rn,
// __dadd_rn, ...), so ptxas cannot contract or reassociate differently in the
// vector body and the scalar tail: both yield identical bits.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/polsar.h"

// Bounds checks for debug builds (-DPOLSAR_DEBUG_BOUNDS, tools/debug_build.sh):
// device-side asserts on shared-memory and global indexing.  Compiled out of
// the product library.
#ifdef POLSAR_DEBUG_BOUNDS
#include <assert.h>
#define POLSAR_CHECK(c) assert(c)
#else
#define POLSAR_CHECK(c) \
    do {                \
    } while (0)
#endif

namespace polsar_impl {

// ------------------------------------------------------------------ errors
// (defined in abi.cu; thread-local, read back by polsar_last_error)
int fail(int code, const char* msg);
int launch_check(const char* what);

// Image extents the window-family entry points accept: slab_rows * width <=
// 2^40 pixels (far beyond any HBM; keeps every byte count below in int64)
constexpr int64_t kMaxSlabPixels = (int64_t)1 << 40;
__host__ __forceinline__ bool slab_size_ok(int64_t slab_rows, int64_t width) {
    return slab_rows >= 0 && width >= 0 && (width == 0 || slab_rows <= kMaxSlabPixels / width);
}

// --------------------------------------------------------- launch geometry
int num_sms();
// one thread per work item, the whole batch in one grid (capped at 2^31-1
// CTAs; the kernels' grid-stride loops take any remainder)
int grid_full(int64_t work, int threads);
// enough CTAs for every SM to hold its resident maximum several times over
int grid_for(int64_t work, int threads);

// ----------------------------------------------------- rounding intrinsics
// Overloads so one template body serves fp32 and fp64 arithmetic.
__device__ __forceinline__ double MUL(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float MUL(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double ADD(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float ADD(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double SUB(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float SUB(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double FMA(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float FMA(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double RCP(double a) { return __drcp_rn(a); }
__device__ __forceinline__ float RCP(float a) { return __frcp_rn(a); }
__device__ __forceinline__ double SQRT(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float SQRT(float a) { return __fsqrt_rn(a); }

// ------------------------------------------------------ streaming HBM I/O
// Plain 16-byte global loads and stores (LDG.E.128 / STG.E.128).  Measured
// on B200 at c3 size (tools/micro/k1_tune.cu): the default cache policy beats
// ld.global.nc.L1::no_allocate + st.global.cs by ~5 % for this 9-in / 11-out
// stream, reaching 103 % of the driver's copy peak with one 16-B vector per
// plane per thread and 128-thread CTAs over the whole batch.
__device__ __forceinline__ float4 ld_stream(const float4* p) { return *p; }
__device__ __forceinline__ float2 ld_stream(const float2* p) { return *p; }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return *p; }
__device__ __forceinline__ float ld_stream(const float* p) { return *p; }
__device__ __forceinline__ double ld_stream(const double* p) { return *p; }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { *p = v; }
__device__ __forceinline__ void st_stream(float2* p, float2 v) { *p = v; }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { *p = v; }
__device__ __forceinline__ void st_stream(float* p, float v) { *p = v; }
__device__ __forceinline__ void st_stream(double* p, double v) { *p = v; }

// ------------------------------------------------------------ matrix types
template <typename T>
struct H9 {  // packed Hermitian
    T a, br, bi, cr, ci, d, er, ei, f;
};

// tau * a*d*f, tau = 16 u_in (R-5)
template <typename S>
struct Tau;
template <>
struct Tau<float> {
    static constexpr double v = 16.0 * 5.9604644775390625e-08;  // 16 * 2^-24
};
template <>
struct Tau<double> {
    static constexpr double v = 16.0 * 1.1102230246251565e-16;  // 16 * 2^-53
};

template <typename T>
__device__ __forceinline__ bool finite_pos(T x) {
    return x > T(0) && x < T(INFINITY);
}

// ------------------------------------------- mbarrier, bulk copies and TMA
// (the NLM gather in nlm.cu)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA: one 2-D box of a tensor map into shared memory, completion on bar
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace polsar_impl
