// Check of the mma.sync.m8n8k4 f64 fragment layout assumed by window_mma.cuh:
// A[m = lane/4][k = lane%4], B[k = lane%4][n = lane/4], C[m = lane/4][n = 2(lane%4) + i].
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* A, const double* B, double* C) {
    int lane = threadIdx.x;
    double a = A[(lane >> 2) * 4 + (lane & 3)];
    double b = B[(lane & 3) * 8 + (lane >> 2)];
    double c0 = 0, c1 = 0;
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    C[(lane >> 2) * 8 + 2 * (lane & 3)] = c0;
    C[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = c1;
}
int main() {
    double hA[32], hB[32], hC[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = i * 0.5 + 1; hB[i] = (i % 7) - 3 + i * 0.25; }
    for (int m = 0; m < 8; ++m) for (int n = 0; n < 8; ++n) {
        double s = 0; for (int kk = 0; kk < 4; ++kk) s += hA[m * 4 + kk] * hB[kk * 8 + n]; ref[m * 8 + n] = s; }
    double *A, *B, *C; cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512);
    cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(A, B, C); cudaMemcpy(hC, C, 512, cudaMemcpyDeviceToHost);
    double e = 0; for (int i = 0; i < 64; ++i) e = fmax(e, fabs(hC[i] - ref[i]));
    printf("max abs err %g (%s)\n", e, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
