// Conversion throughput probe: FP64 -> FP32 -> FP64 round trips (the per-gate rounding of
// FP32 storage, kernels.py:36-40), independent chains, all SMs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, double a) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = (double)__double2float_rn(__dmul_rn(x[i], a));
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}
int main() {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int threads : {256, 512, 1024}) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        int iters = 20000; int blocks = sms * (2048 / threads);
        k<<<blocks, threads>>>(d, iters, 1.0000001);
        cudaEventRecord(e0); k<<<blocks, threads>>>(d, iters, 1.0000001); cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * iters * 8;
        printf("DMUL+F2F.F32.F64+F2F.F64.F32 threads/blk %4d: %.2f T round-trips/s (%.1f /clk/SM)\n", threads,
               ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
    }
    return 0;
}
