// abi.cu -- part of libpolsar.so (B200, sm_100a); arXiv 1807.08084.
// Layout, ownership and error conventions: include/polsar.h.  Design notes:
// DESIGN.md.  Nothing here is shared with oracle/.
//
// Library-wide state and helpers: the thread-local error string, launch
// geometry, and the diagnostic entry points.
#include "common.cuh"

namespace polsar_impl {

thread_local const char* g_last_error = "";

int fail(int code, const char* msg) {
    g_last_error = msg;
    return code;
}

int launch_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_last_error = what;
        return POLSAR_ECUDA;
    }
    g_last_error = "";
    return POLSAR_OK;
}

int num_sms() {  // of the device current at first use (read once, thread-safe)
    static const int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return n;
}

// one thread per work item, the whole batch in one grid (capped at 2^31-1
// CTAs; the kernels' grid-stride loops take any remainder)
int grid_full(int64_t work, int threads) {
    int64_t need = (work + threads - 1) / threads;
    if (need > 0x7fffffff) need = 0x7fffffff;
    return (int)(need < 1 ? 1 : need);
}

int grid_for(int64_t work, int threads) {
    // enough CTAs for every SM to hold its resident maximum several times
    // over; beyond that the grid-stride loop takes over
    int64_t need = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * 64;
    if (need > cap) need = cap;
    return (int)(need < 1 ? 1 : need);
}

}  // namespace polsar_impl

extern "C" {

const char* polsar_last_error(void) { return polsar_impl::g_last_error; }

int polsar_version(void) { return 0x000200; }

}  // extern "C"
