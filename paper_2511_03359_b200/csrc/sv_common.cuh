// Common device helpers for the B200 state-vector kernels (sm_100a).
//
// Arithmetic contract (bit-identical to the reference's numpy arithmetic,
// /root/reference/pkg/src/svsim/kernels.py:1-15):
//   * complex product a*b with `a` the FIRST operand:
//       re = fma(ar, br, -(ai*bi)),  im = fma(ar, bi, ai*br)
//   * complex sum: IEEE add per component
//   * all arithmetic in FP64; FP32 storage widens exactly on load and rounds
//     once (round-to-nearest-even) on store (kernels.py:36-40).
// Every product/sum below is written with explicit __fma_rn/__dmul_rn/__dadd_rn
// so nvcc cannot contract or reassociate them.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "sv_arith.cuh"  // cplx, cmul, cadd, row2, row4 (shared with the NVRTC pass kernels)

namespace sv {

// ---- storage element types ------------------------------------------------
// FP64: 16 B per amplitude; FP32: 8 B per amplitude.  A "vector" is 32 B, the
// widest global access sm_100a has (LDG.E.ENL2.256 / STG.E.ENL2.256).
struct __align__(16) c64s { double re, im; };
struct __align__(8) c32s { float re, im; };

template <typename S> struct Store;
template <> struct Store<c64s> {
    static constexpr int V = 2;                   // amplitudes per 32 B vector
    // value as it would read back after a store (identity for FP64 storage)
    __device__ __forceinline__ static cplx round(cplx c) { return c; }
    __device__ __forceinline__ static cplx get(c64s s) { return {s.re, s.im}; }
    __device__ __forceinline__ static c64s put(cplx c) { return {c.re, c.im}; }
};
template <> struct Store<c32s> {
    static constexpr int V = 4;
    // FP32 storage rounds after every gate (kernels.py:36-40 store into complex64)
    __device__ __forceinline__ static cplx round(cplx c) {
        return {(double)__double2float_rn(c.re), (double)__double2float_rn(c.im)};
    }
    __device__ __forceinline__ static cplx get(c32s s) { return {(double)s.re, (double)s.im}; }
    __device__ __forceinline__ static c32s put(cplx c) {
        return {__double2float_rn(c.re), __double2float_rn(c.im)};
    }
};

template <typename S> struct __align__(32) Vec { S a[Store<S>::V]; };

template <typename S>
__device__ __forceinline__ Vec<S> vload(const S* p) {
    return *reinterpret_cast<const Vec<S>*>(p);
}
template <typename S>
__device__ __forceinline__ void vstore(S* p, const Vec<S>& v) {
    *reinterpret_cast<Vec<S>*>(p) = v;
}

// ---- index helpers ---------------------------------------------------------
// insert a zero bit at position q: the low member of pair number t (kernels.py:21-27)
__device__ __forceinline__ uint64_t insert0(uint64_t t, int q) {
    const uint64_t lowmask = (1ull << q) - 1ull;
    return ((t & ~lowmask) << 1) | (t & lowmask);
}
// scatter the low bits of x into the set bits of mask (software PDEP)
__device__ __forceinline__ uint64_t pdep64(uint64_t x, uint64_t mask) {
    uint64_t r = 0;
    while (mask) {
        const uint64_t bit = mask & (~mask + 1ull);
        if (x & 1ull) r |= bit;
        x >>= 1;
        mask &= mask - 1ull;
    }
    return r;
}

// insert a zero at every set bit of `mask` (ascending) == pdep64(x, ~mask):
// cost is popcount(mask) steps instead of the width of the free mask
__device__ __forceinline__ uint64_t insert_zeros(uint64_t x, uint64_t mask) {
    while (mask) {
        const int q = __ffsll((long long)mask) - 1;
        x = insert0(x, q);
        mask &= mask - 1ull;
    }
    return x;
}

}  // namespace sv
