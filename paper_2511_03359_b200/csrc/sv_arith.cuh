// Reference arithmetic (numpy order, svsim/kernels.py:1-15): include-free so the
// same text compiles under nvcc (sv_common.cuh) and NVRTC (sv_jit.cu pass kernels).
#pragma once

namespace sv {

struct cplx { double re, im; };

__device__ __forceinline__ cplx cmul(cplx a, cplx b) {   // a first (numpy order)
    return { __fma_rn(a.re, b.re, -__dmul_rn(a.im, b.im)),
             __fma_rn(a.re, b.im, __dmul_rn(a.im, b.re)) };
}
__device__ __forceinline__ cplx cadd(cplx a, cplx b) {
    return { __dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im) };
}

// 2x2 row: m0*a0 + m1*a1 (matrix entry first, left-to-right sum; kernels.py:39-40)
__device__ __forceinline__ cplx row2(cplx m0, cplx m1, cplx a0, cplx a1) {
    return cadd(cmul(m0, a0), cmul(m1, a1));
}
// 4x4 row: ((m0*a0 + m1*a1) + m2*a2) + m3*a3 (kernels.py:60-64)
__device__ __forceinline__ cplx row4(const cplx* m, cplx a0, cplx a1, cplx a2, cplx a3) {
    return cadd(cadd(cadd(cmul(m[0], a0), cmul(m[1], a1)), cmul(m[2], a2)), cmul(m[3], a3));
}

}  // namespace sv
