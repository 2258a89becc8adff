// Device side of the specialised fused-pass kernels (compiled at run time by
// NVRTC from sv_jit.cu; include-free apart from sv_arith.cuh).
//
// A generated pass kernel is k_fused3 (sv_fused2.cu) with every pass constant
// folded in: tile positions, segment register/thread positions, shared-memory
// swizzle offsets, op kinds, register bits, monomial codes and diagonal masks
// are literals, so the per-op dispatch (switches, selects, register moves at
// the join points, LDC of the op tables) disappears and the matrices are read
// as constant-bank operands of the DFMA/DMUL instructions.  The arithmetic is
// the same sequence as k_fused3 (sv_arith.cuh, reference operand order), so a
// specialised pass is bit-identical to the generic one.
#pragma once

#include "sv_arith.cuh"

namespace svj {

using sv::cadd;
using sv::cmul;
using sv::cplx;
using sv::row2;
using sv::row4;
typedef unsigned long long u64;

struct __align__(16) c64s { double re, im; };
struct __align__(8) c32s { float re, im; };

// ---- FP32 storage: the reference stores every gate's result into complex64
// (kernels.py:36-40), i.e. one round-to-nearest-even to float after each gate:
// F2F there and back (exact widening).  F2F runs at ~16/clk/SM on B200
// (tools/f2f_probe.cu: 2.2 T FP64->FP32->FP64 round trips/s), the cost floor of FP32
// passes with many gates.
// SVJ_F32_ROUND (set by the generated source): 0 = F2F there and back for every value,
// 1 = Veltkamp split on the FP64 pipe for every value, 2 = real parts Veltkamp, imaginary
// parts F2F (both pipes busy).  Veltkamp with C = 2^29 + 1 in round-to-nearest-even
// FP64: g = C x, hi = g + (x - g) is x rounded to 24 significant bits, ties to even --
// identical to the float rounding for 2^-126 <= |x| < 2^127 (tests/test_fp32_round.py:
// every tie / carry / exponent-edge pattern, random values; tools/f32_round_check.cu on
// the device).  Outside that range (float subnormals, overflow, NaN / Inf, double
// subnormals) the F2F path runs; +-0 is returned as is (the split would drop the sign).
#ifndef SVJ_F32_ROUND
#define SVJ_F32_ROUND 0
#endif
__device__ __forceinline__ double r32_f2f(double x) { return (double)__double2float_rn(x); }
__device__ __forceinline__ double r32_split(double x) {
    const double g = __dmul_rn(536870913.0, x);             // 2^29 + 1
    const double v = __dadd_rn(g, __dadd_rn(x, -g));
    const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
    if (e - 897u < 253u) return v;                          // 2^-126 <= |x| < 2^127
    if (x == 0.0) return x;
    return r32_f2f(x);
}
// integer pipe: add half an ulp of the float mantissa (ties to even) to the double's bits
// and clear the 29 dropped bits -- the same rounding, no FP64 or conversion instruction
__device__ __forceinline__ double r32_int(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const unsigned e = (unsigned)(b >> 52) & 0x7ffu;
    if (e - 897u < 253u)
        return __longlong_as_double((long long)((b + 0x0FFFFFFFull + ((b >> 29) & 1ull)) & ~0x1FFFFFFFull));
    if ((b << 1) == 0ull) return x;
    return r32_f2f(x);
}
// SVJ_F32_ROUND: 0 F2F, 1 split, 2 re split / im F2F, 3 re integer / im F2F, 4 integer
__device__ __forceinline__ double r32(double x) {
#if SVJ_F32_ROUND == 1
    return r32_split(x);
#elif SVJ_F32_ROUND == 4
    return r32_int(x);
#else
    return r32_f2f(x);
#endif
}
__device__ __forceinline__ double r32_re(double x) {
#if SVJ_F32_ROUND == 1 || SVJ_F32_ROUND == 2
    return r32_split(x);
#elif SVJ_F32_ROUND == 3 || SVJ_F32_ROUND == 4
    return r32_int(x);
#else
    return r32_f2f(x);
#endif
}
template <int R>
__device__ __forceinline__ void rnd_all(cplx (&r)[R]) {
#pragma unroll
    for (int i = 0; i < R; ++i) r[i] = {r32_re(r[i].re), r32(r[i].im)};
}
template <int R, unsigned MR>
__device__ __forceinline__ void rnd_mask(cplx (&r)[R]) {
#pragma unroll
    for (int i = 0; i < R; ++i)
        if ((i & MR) == MR) r[i] = {r32_re(r[i].re), r32(r[i].im)};
}

// shared-memory swizzle of k_fused3 (linear in the element index)
__device__ __forceinline__ int swz(int e) {
    const int g = (((e >> 3) & 1) * 7) ^ (((e >> 4) & 1) * 3) ^ (((e >> 5) & 1) * 5) ^ (((e >> 6) & 1) * 6);
    return e ^ g;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
// the same with a source size: 0 fills the 16 shared-memory bytes with zeros, reading nothing
__device__ __forceinline__ void cp_async16_z(void* smem_dst, const void* gsrc, unsigned bytes) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---- bulk tile loads (FP64 passes): one cp.async.bulk (TMA engine, SASS UBLKCP) per
// 256-byte run of 16 contiguous amplitudes (tile positions 0..3 = qubits 0..3), completion
// counted in bytes on an mbarrier, instead of 16 cp.async (LDGSTS) per thread.  A bulk
// copy cannot permute inside a run, so bank conflicts are avoided by PADDING between runs
// instead of the XOR swizzle: slot(e) = e + D0 (e >> 4) + D1 (e >> 7) + D2 (e >> 10)
// (additive over disjoint bit sets, so a thread's slot + a register's slot is the element's
// slot); sv_jit.cu picks D0..D2 and the thread-bit order per pass.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SVJ_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SVJ_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on `bar` once every cp.async this thread issued so far has landed (the barrier
// counts one arrival per issuing thread: .noinc)
__device__ __forceinline__ void cp_async_mbar_arrive(u64* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// named barrier of one warp group (ring passes: two groups of `n` threads per CTA)
__device__ __forceinline__ void bar_group(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// generic-proxy reads of the buffer (earlier tile) ordered before the async-proxy writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, u64* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// p + off amplitudes, computed where it is used: the 16 prefetch / store addresses of
// a tile are loop-invariant offsets from the tile base, and hoisting them out of the
// tile loop (32 live 64-bit pointers) is what made the compiler spill
template <typename T>
__device__ __forceinline__ T* at(T* p, u64 off) {
    T* r;
    asm volatile("add.s64 %0, %1, %2;" : "=l"(r) : "l"(p), "l"(off * sizeof(T)));
    return r;
}

__device__ __forceinline__ void stg(c64s* p, cplx v) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.re), "d"(v.im) : "memory");
}
// value already float-representable (rounded after its last gate): the narrowing is exact
__device__ __forceinline__ void stg(c32s* p, cplx v) {
    asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"((float)v.re), "f"((float)v.im) : "memory");
}

// direct tile input (no shared-memory staging): 16-byte load, not kept in L1 (read once)
__device__ __forceinline__ cplx ldg(const c64s* p) {
    double re, im;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(re), "=d"(im) : "l"(p));
    return {re, im};
}

template <int U>
__device__ __forceinline__ cplx mu(cplx a) {   // U: 0 -> 1, 1 -> i, 2 -> -1, 3 -> -i
    if constexpr (U == 0) return a;
    else if constexpr (U == 1) return {-a.im, a.re};
    else if constexpr (U == 2) return {-a.re, -a.im};
    else return {a.im, -a.re};
}

__device__ __forceinline__ cplx rmul(double m, cplx a) { return {__dmul_rn(m, a.re), __dmul_rn(m, a.im)}; }

// Matrix entries of the pass live in kernel parameter 1 (Args::m).  They are read
// at the point of use through a parameter-space address that the generated kernel
// rebuilds every tile from an opaque zero (tile >> 62): with plain (or volatile)
// constant loads ptxas hoists every matrix of the pass out of the tile loop, the
// uniform registers overflow into ~130 regular registers for a few U4 gates and the
// kernel spills; a per-use LDC costs one instruction per entry per tile.
constexpr int kArgsM = 48;   // byte offset of Args::m (after n_tiles, cmask, cpat, vinit, pfix, pval)

// tile index t of a chunked launch -> full tile index: zeros inserted at the bits of cm,
// then the chunk pattern
__device__ __forceinline__ u64 chunk_tile(u64 t, u64 cm, u64 cp) {
    while (cm) {
        const int q = __ffsll((long long)cm) - 1;
        t = ((t >> q) << (q + 1)) | (t & ((1ull << q) - 1ull));
        cm &= cm - 1ull;
    }
    return t | cp;
}

__device__ __forceinline__ u64 mbase(u64 tile) {
    u64 b;
    asm("mov.u64 %0, sv_pass_param_1;" : "=l"(b));
    return b + ((tile >> 62) << 3);
}
template <int OFF>
__device__ __forceinline__ double ldm(u64 mb) {
    double v;
    asm volatile("ld.param.f64 %0, [%1+%2];" : "=d"(v) : "l"(mb), "n"(kArgsM + 8 * OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ cplx ldc2(u64 mb) { return {ldm<OFF>(mb), ldm<OFF + 1>(mb)}; }

// ---- single-qubit ops on register bit J ------------------------------------------
template <int R, int J, int OFF>
__device__ __forceinline__ void g1(cplx (&r)[R], u64 mb) {
    const cplx m0 = ldc2<OFF>(mb), m1 = ldc2<OFF + 2>(mb), m2 = ldc2<OFF + 4>(mb), m3 = ldc2<OFF + 6>(mb);
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i & (1 << J)) continue;
        const cplx a0 = r[i], a1 = r[i | (1 << J)];
        r[i] = row2(m0, m1, a0, a1);
        r[i | (1 << J)] = row2(m2, m3, a0, a1);
    }
}

template <int R, int J, int OFF>
__device__ __forceinline__ void g1r(cplx (&r)[R], u64 mb) {   // real matrix (H)
    const double m0 = ldm<OFF>(mb), m1 = ldm<OFF + 2>(mb), m2 = ldm<OFF + 4>(mb), m3 = ldm<OFF + 6>(mb);
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i & (1 << J)) continue;
        const cplx a0 = r[i], a1 = r[i | (1 << J)];
        r[i] = cadd(rmul(m0, a0), rmul(m1, a1));
        r[i | (1 << J)] = cadd(rmul(m2, a0), rmul(m3, a1));
    }
}

// monomial rows: per row 2-bit source selector | 2-bit unit << 2 (k_fused3's mono code)
template <int R, int J, unsigned MONO>
__device__ __forceinline__ void g1m(cplx (&r)[R]) {
    constexpr int s0 = MONO & 3, u0 = (MONO >> 2) & 3, s1 = (MONO >> 4) & 3, u1 = (MONO >> 6) & 3;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i & (1 << J)) continue;
        const cplx a0 = r[i], a1 = r[i | (1 << J)];
        r[i] = mu<u0>(s0 ? a1 : a0);
        r[i | (1 << J)] = mu<u1>(s1 ? a1 : a0);
    }
}

// ---- two-qubit ops: JA = register bit of qa, JB = of qb; basis bit(qa) + 2 bit(qb) -----
template <int R, int JA, int JB, int OFF>
__device__ __forceinline__ void g2(cplx (&r)[R], u64 mb) {
    const cplx mm[4][4] = {
        {ldc2<OFF + 0>(mb), ldc2<OFF + 2>(mb), ldc2<OFF + 4>(mb), ldc2<OFF + 6>(mb)},
        {ldc2<OFF + 8>(mb), ldc2<OFF + 10>(mb), ldc2<OFF + 12>(mb), ldc2<OFF + 14>(mb)},
        {ldc2<OFF + 16>(mb), ldc2<OFF + 18>(mb), ldc2<OFF + 20>(mb), ldc2<OFF + 22>(mb)},
        {ldc2<OFF + 24>(mb), ldc2<OFF + 26>(mb), ldc2<OFF + 28>(mb), ldc2<OFF + 30>(mb)}};
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i & ((1 << JA) | (1 << JB))) continue;
        const int idx[4] = {i, i | (1 << JA), i | (1 << JB), i | (1 << JA) | (1 << JB)};
        const cplx a[4] = {r[idx[0]], r[idx[1]], r[idx[2]], r[idx[3]]};
#pragma unroll
        for (int row = 0; row < 4; ++row) r[idx[row]] = row4(mm[row], a[0], a[1], a[2], a[3]);
    }
}

template <int R, int JA, int JB, unsigned MONO>
__device__ __forceinline__ void g2m(cplx (&r)[R]) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i & ((1 << JA) | (1 << JB))) continue;
        const int idx[4] = {i, i | (1 << JA), i | (1 << JB), i | (1 << JA) | (1 << JB)};
        const cplx a[4] = {r[idx[0]], r[idx[1]], r[idx[2]], r[idx[3]]};
        r[idx[0]] = mu<(MONO >> 2) & 3>(a[MONO & 3]);
        r[idx[1]] = mu<(MONO >> 6) & 3>(a[(MONO >> 4) & 3]);
        r[idx[2]] = mu<(MONO >> 10) & 3>(a[(MONO >> 8) & 3]);
        r[idx[3]] = mu<(MONO >> 14) & 3>(a[(MONO >> 12) & 3]);
    }
}

// ---- diagonal factor on the registers whose bits cover MR (amplitude first) --------
// cmul() in place, the same roundings: t1 = a.im*f.im, t2 = a.im*f.re, then
// im = fma(a.re, f.im, t2) before re = fma(a.re, f.re, -t1) so both results can take
// the operand registers.  Written as cmul(), ptxas renamed the 16 amplitudes on every
// multiply block and merged them back with ~2 MOVs per amplitude (pass SASS -20 %).
__device__ __forceinline__ void cmul_inplace(cplx& a, cplx f) {
    asm("{\n\t.reg .f64 t1, t2;\n\t"
        "mul.rn.f64 t1, %1, %3;\n\t"
        "mul.rn.f64 t2, %1, %2;\n\t"
        "fma.rn.f64 %1, %0, %3, t2;\n\t"
        "neg.f64 t1, t1;\n\t"
        "fma.rn.f64 %0, %0, %2, t1;\n\t}"
        : "+d"(a.re), "+d"(a.im) : "d"(f.re), "d"(f.im));
}
template <int R, unsigned MR, int OFF>
__device__ __forceinline__ void gd(cplx (&r)[R], u64 mb) {
    const cplx f = ldc2<OFF>(mb);
#pragma unroll
    for (int i = 0; i < R; ++i)
        if ((i & MR) == MR) cmul_inplace(r[i], f);
}

// ---- long runs of diagonal ops: one compact loop over a descriptor table -----------
// Straight-line code for ~100 diagonal ops (the adder's CPHASE runs) overflows the
// instruction cache (ncu: no_instruction stalls 5.8 per issue).  A run is instead a
// loop over 4-double descriptors in the kernel parameters: [out-of-tile mask bits,
// thread mask | register mask << 16, factor re, factor im]; the register mask picks
// one of 16 straight-line multiply blocks (compile-time register indices), so the
// code is one switch regardless of the run length.  Same multiplies in the same
// order as gd<> (amplitude first), the Z factor (-1, 0) included: numpy's product.
__device__ __forceinline__ double ldp_at(u64 mb, int idx) {
    double v;
    asm volatile("ld.param.f64 %0, [%1];" : "=d"(v) : "l"(mb + (u64)kArgsM + 8ull * (u64)idx));
    return v;
}
template <int R, unsigned MR>
__device__ __forceinline__ void gdf(cplx (&r)[R], cplx f) {
#pragma unroll
    for (int i = 0; i < R; ++i)
        if ((i & MR) == MR) cmul_inplace(r[i], f);
}
template <int R, unsigned MR, bool F32>
__device__ __forceinline__ void gdf_r(cplx (&r)[R], cplx f) {
    gdf<R, MR>(r, f);
    if constexpr (F32) rnd_mask<R, MR>(r);
}
constexpr unsigned kDiagAllRegs = 1u << 31;   // descriptor flag: register mask 0 (set by sv_jit.cu)
template <int R, bool F32>
__device__ __forceinline__ void diag_apply(cplx (&r)[R], unsigned w, cplx f) {
    if (w & kDiagAllRegs) {   // no register bit in the mask: the common case, one test
        gdf_r<R, 0, F32>(r, f);
        return;
    }
    switch ((w >> 16) & 0xfu) {
        case 1: gdf_r<R, 1, F32>(r, f); break;
        case 2: gdf_r<R, 2, F32>(r, f); break;
        case 3: gdf_r<R, 3, F32>(r, f); break;
        case 4: gdf_r<R, 4, F32>(r, f); break;
        case 5: gdf_r<R, 5, F32>(r, f); break;
        case 6: gdf_r<R, 6, F32>(r, f); break;
        case 7: gdf_r<R, 7, F32>(r, f); break;
        case 8: gdf_r<R, 8, F32>(r, f); break;
        case 9: gdf_r<R, 9, F32>(r, f); break;
        case 10: gdf_r<R, 10, F32>(r, f); break;
        case 11: gdf_r<R, 11, F32>(r, f); break;
        case 12: gdf_r<R, 12, F32>(r, f); break;
        case 13: gdf_r<R, 13, F32>(r, f); break;
        case 14: gdf_r<R, 14, F32>(r, f); break;
        default: gdf_r<R, 15, F32>(r, f); break;
    }
}
// The out-of-tile test is uniform over the tile: lane j of each warp tests
// descriptor k0 + j and one ballot leaves the ops that touch this tile, so the
// loop below visits only those (in order) instead of a load -> test -> branch
// chain per descriptor (adder 124-op passes 90 -> 78 ms at N=32; loading the next
// descriptor ahead of the multiplies measured slower).
template <int R, bool F32 = false>
__device__ __forceinline__ void diag_run(cplx (&r)[R], int tb, u64 base, u64 mb, int off, int cnt) {
    const int lane = threadIdx.x & 31;
    for (int k0 = 0; k0 < cnt; k0 += 32) {
        bool hit = false;
        if (k0 + lane < cnt) {
            const u64 dout = (u64)__double_as_longlong(ldp_at(mb, off + 4 * (k0 + lane)));
            hit = (base & dout) == dout;
        }
        unsigned act = __ballot_sync(0xffffffffu, hit);
        while (act) {
            const int d = off + 4 * (k0 + __ffs(act) - 1);
            act &= act - 1;
            const unsigned w = (unsigned)__double_as_longlong(ldp_at(mb, d + 1));
            const unsigned dthr = w & 0xffffu;
            if (((unsigned)tb & dthr) != dthr) continue;
            diag_apply<R, F32>(r, w, cplx{ldp_at(mb, d + 2), ldp_at(mb, d + 3)});
        }
    }
}

template <int R, unsigned MR>
__device__ __forceinline__ void gdn(cplx (&r)[R]) {   // factor exactly -1 (Z): exact negation
#pragma unroll
    for (int i = 0; i < R; ++i)
        if ((i & MR) == MR) r[i] = {-r[i].re, -r[i].im};
}

}  // namespace svj
