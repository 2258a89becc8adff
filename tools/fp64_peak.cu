// FP64 throughput probe: independent DFMA / DMUL / DADD chains, all SMs.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = __fma_rn(x[i], a, b);
            else if (OP == 1) x[i] = __dmul_rn(x[i], a);
            else x[i] = __dadd_rn(x[i], b);
        }
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}
int main() {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[3] = {"DFMA", "DMUL", "DADD"};
    for (int threads : {256, 512, 1024}) for (int op = 0; op < 3; ++op) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        int iters = 20000; int blocks = sms * (2048 / threads);
        auto launch = [&]() {
            if (op == 0) k<0><<<blocks, threads>>>(d, iters, 1.0000001, 1e-7);
            else if (op == 1) k<1><<<blocks, threads>>>(d, iters, 1.0000001, 1e-7);
            else k<2><<<blocks, threads>>>(d, iters, 1.0000001, 1e-7);
        };
        launch(); cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * iters * 8;
        printf("%s threads/blk %4d: %.2f Tops/s (%.1f ops/clk/SM at 1.965GHz)\n", names[op], threads, ops / ms / 1e9,
               ops / (ms * 1e-3) / sms / 1.965e9);
    }
    return 0;
}
