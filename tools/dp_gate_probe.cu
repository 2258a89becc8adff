// How fast can an SM run the fused kernel's in-register 2x2 gate body?
// Same arithmetic as reg_1q<R,J> (numpy operand order), no memory traffic.
#include <cstdio>
#include "../paper_2511_03359_b200/csrc/sv_common.cuh"
using namespace sv;

template <int R, int J>
__device__ __forceinline__ void g1(cplx (&r)[R], const double* md) {
    const cplx m0 = {md[0], md[1]}, m1 = {md[2], md[3]}, m2 = {md[4], md[5]}, m3 = {md[6], md[7]};
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i & (1 << J)) continue;
        const cplx a0 = r[i], a1 = r[i | (1 << J)];
        r[i] = row2(m0, m1, a0, a1);
        r[i | (1 << J)] = row2(m2, m3, a0, a1);
    }
}

template <int R>
__global__ void k(double* out, const double* __restrict__ mats, int iters, int nmat) {
    cplx r[R];
#pragma unroll
    for (int i = 0; i < R; ++i) r[i] = {threadIdx.x * 1e-3 + i, 0.5};
    for (int it = 0; it < iters; ++it) {
        const double* md = mats + 8 * (it % nmat);
        switch (it & 3) {
            case 0: g1<R, 0>(r, md); break;
            case 1: g1<R, 1>(r, md); break;
            case 2: g1<R, 2>(r, md); break;
            default: if constexpr (R >= 16) g1<R, 3>(r, md); else g1<R, 0>(r, md); break;
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) s += r[i].re + r[i].im;
    if (s == 1.2345) out[0] = s;
}

int main() {
    double* d; cudaMalloc(&d, 8);
    double hm[64];
    for (int i = 0; i < 64; ++i) hm[i] = 0.7071067811865476 * ((i % 3) - 1) + 1e-3 * i;
    double* dm; cudaMalloc(&dm, sizeof(hm)); cudaMemcpy(dm, hm, sizeof(hm), cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps_per_sm : {4, 8, 16, 32}) {
        for (int rr : {8, 16}) {
            const int threads = 128;
            const int blocks = sms * warps_per_sm * 32 / threads;
            const int iters = 4000;
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            auto launch = [&]() {
                if (rr == 8) k<8><<<blocks, threads>>>(d, dm, iters, 8);
                else k<16><<<blocks, threads>>>(d, dm, iters, 8);
            };
            launch(); cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double dp = (double)blocks * threads * iters * (rr / 2) * 20.0;
            printf("warps/SM %2d R=%2d: %.2f T DP/s = %.0f%% of 18.5T\n", warps_per_sm, rr, dp / ms / 1e9,
                   dp / ms / 1e9 / 18.5 * 100);
        }
    }
    return 0;
}
