// checksum.cu -- part of libpolsar.so (B200, sm_100a); arXiv 1807.08084.
// Layout, ownership and error conventions: include/polsar.h.  Design notes:
// DESIGN.md.  Nothing here is shared with oracle/.
//
//   R1  polsar_checksum          order-independent output hash + status counts
#include "common.cuh"

namespace polsar_impl {
namespace {

// ======================================================= R1: checksums
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

template <typename U>
__global__ void __launch_bounds__(256)
k_checksum(const U* __restrict__ planes, int64_t n, int64_t ld, int nplanes, int64_t pix_offset,
           const uint8_t* __restrict__ status, unsigned long long* __restrict__ result) {
    uint64_t h = 0;
    unsigned long long c0 = 0, c1 = 0, c2 = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = (uint64_t)(pix_offset + p) * 0x9E3779B97F4A7C15ull;
        for (int k = 0; k < nplanes; ++k)
            h += mix64((uint64_t)planes[k * ld + p] ^ (key + (uint64_t)k * 0xD6E8FEB86659FD93ull));
        if (status) {
            uint8_t s = status[p];
            c0 += s == 0;
            c1 += s == 1;
            c2 += s == 2;
        }
    }
    // warp reduction, then one atomic per warp (wrapping uint64 sums commute)
    for (int o = 16; o > 0; o >>= 1) {
        h += __shfl_down_sync(0xffffffffu, h, o);
        c0 += __shfl_down_sync(0xffffffffu, c0, o);
        c1 += __shfl_down_sync(0xffffffffu, c1, o);
        c2 += __shfl_down_sync(0xffffffffu, c2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(result + 0, (unsigned long long)h);
        if (status) {
            atomicAdd(result + 1, c0);
            atomicAdd(result + 2, c1);
            atomicAdd(result + 3, c2);
        }
    }
}

}  // namespace
}  // namespace polsar_impl

using namespace polsar_impl;

extern "C" {

int polsar_checksum(const void* planes, int64_t n, int64_t ld, int nplanes, int dtype,
                    int64_t pix_offset, const uint8_t* status, uint64_t* result, void* cuda_stream) {
    if (n < 0 || ld < n || nplanes < 0 || !result) return fail(POLSAR_EINVAL, "bad checksum args");
    if (n == 0) return POLSAR_OK;
    if (nplanes > 0 && !planes) return fail(POLSAR_EINVAL, "null planes");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    int grid = grid_for(n, 256);
    if (dtype == POLSAR_F32 || dtype == POLSAR_F32_PLAIN)
        k_checksum<uint32_t><<<grid, 256, 0, s>>>((const uint32_t*)planes, n, ld, nplanes, pix_offset,
                                                  status, (unsigned long long*)result);
    else if (dtype == POLSAR_F64 || dtype == POLSAR_F64_PLAIN || dtype == POLSAR_F64_EFT)
        k_checksum<uint64_t><<<grid, 256, 0, s>>>((const uint64_t*)planes, n, ld, nplanes, pix_offset,
                                                  status, (unsigned long long*)result);
    else
        return fail(POLSAR_EINVAL, "bad dtype");
    return launch_check("polsar_checksum: launch failed");
}

}  // extern "C"
