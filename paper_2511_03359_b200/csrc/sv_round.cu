// Device check of the FP32-storage rounding used by the specialised passes
// (sv_jit_dev.cuh r32_split / r32_f2f): every value of a host array rounded on the
// B200 with the chosen method, so tests can compare the split against the float
// conversion bit for bit over tie / carry / exponent-edge patterns.
#include "sv_common.cuh"
#include "sv_kernels.cuh"
#include "sv_jit_dev.cuh"
#include "svb200.h"

namespace sv {
int capi_fail(int code, const char* msg);
int capi_cuda_fail(cudaError_t e, const char* what);

namespace {
__global__ void k_f32_round(const double* in, double* out, uint64_t n, int mode) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = mode == 1 ? svj::r32_split(in[i]) : (mode == 2 ? svj::r32_int(in[i]) : svj::r32_f2f(in[i]));
}
}  // namespace
}  // namespace sv

extern "C" int svk_f32_round(const double* host_in, double* host_out, uint64_t n, int mode) {
    if (mode < 0 || mode > 2) return sv::capi_fail(SV_EVALUE, "rounding mode must be 0 (F2F), 1 (split) or 2 (integer)");
    if (n == 0) return SV_OK;
    double *d_in = nullptr, *d_out = nullptr;
    cudaError_t e = cudaMalloc(&d_in, 8 * n);
    if (e == cudaSuccess) e = cudaMalloc(&d_out, 8 * n);
    if (e == cudaSuccess) e = cudaMemcpy(d_in, host_in, 8 * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        sv::k_f32_round<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256>>>(d_in, d_out, n, mode);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(host_out, d_out, 8 * n, cudaMemcpyDeviceToHost);
    cudaFree(d_in);
    cudaFree(d_out);
    return e == cudaSuccess ? SV_OK : sv::capi_cuda_fail(e, "f32 round check");
}
