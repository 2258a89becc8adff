// Fused tile passes, v3: register-resident amplitudes + cp.async double buffering
// (sm_100a, FP64 storage).
//
// One persistent CTA per SM (256 threads) walks tiles of 2^12 amplitudes whose
// local index differs only in the 12 tile qubits (positions 0..b-1 are the
// contiguous low qubits, so HBM is touched in runs of >= 2^5 amplitudes).
//
// Pipeline per CTA: while tile i is computed, tile i+1 is already streaming
// from HBM into the other shared-memory buffer with cp.async (16-byte
// LDGSTS per amplitude, 64 KB per tile in flight per SM); results leave from
// registers with STG.128.  So HBM reads, FP64 math and HBM writes overlap
// inside one CTA instead of relying on several CTAs per SM.
//
// Compute: each thread holds 16 amplitudes in registers spanning 4 "register
// positions" of the tile index (its thread id spans the other 8).  A pass is
// cut into segments; inside a segment every gate acts on register positions
// only and is applied in registers with no shared-memory traffic.  Between
// segments the tile is transposed through shared memory (write, barrier,
// read).  Shared memory uses a linear XOR swizzle of the low 3 index bits
// (columns 7,3,5,6 for bits 3..6, found by exhaustive search: every 8-lane
// quarter-warp touches >= 4 distinct 16-byte bank groups for any register
// choice), applied already by the cp.async destinations.
//
// Gates keep the reference arithmetic (svsim/kernels.py: matrix entry first,
// left-to-right sums in the (qa, qb) basis order), so a fused pass is
// bit-identical to one kernel per gate.  Exact shortcuts (results differ from
// numpy at most in the sign of an exact zero):
//   1Q real matrices (H): the +-0 imaginary products are dropped;
//   monomial matrices with entries in {+-1, +-i} (X, Y, CNOT): exact moves;
//   diagonal factor exactly -1 (Z): exact negation.
#include <algorithm>

#include "sv_common.cuh"
#include "sv_kernels.cuh"

namespace sv {

namespace {

__device__ __forceinline__ int swz(int e) {
    const int g = (((e >> 3) & 1) * 7) ^ (((e >> 4) & 1) * 3) ^ (((e >> 5) & 1) * 5) ^ (((e >> 6) & 1) * 6);
    return e ^ g;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ cplx mul_unit(cplx a, int u) {    // u: 0 -> 1, 1 -> i, 2 -> -1, 3 -> -i
    switch (u) {
        case 0: return a;
        case 1: return {-a.im, a.re};
        case 2: return {-a.re, -a.im};
        default: return {a.im, -a.re};
    }
}

__device__ __forceinline__ cplx rmul(double m, cplx a) { return {__dmul_rn(m, a.re), __dmul_rn(m, a.im)}; }

template <int R, int J>
__device__ __forceinline__ void reg_1q(cplx (&r)[R], int kind, const double* md, uint32_t mono) {
    if (kind == F2_1Q_MONO) {
        const int s0 = mono & 3, u0 = (mono >> 2) & 3, s1 = (mono >> 4) & 3, u1 = (mono >> 6) & 3;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (i & (1 << J)) continue;
            const cplx a0 = r[i], a1 = r[i | (1 << J)];
            r[i] = mul_unit(s0 ? a1 : a0, u0);
            r[i | (1 << J)] = mul_unit(s1 ? a1 : a0, u1);
        }
    } else if (kind == F2_1Q_REAL) {
        const double m0 = md[0], m1 = md[2], m2 = md[4], m3 = md[6];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (i & (1 << J)) continue;
            const cplx a0 = r[i], a1 = r[i | (1 << J)];
            r[i] = cadd(rmul(m0, a0), rmul(m1, a1));
            r[i | (1 << J)] = cadd(rmul(m2, a0), rmul(m3, a1));
        }
    } else {
        const cplx m0 = {md[0], md[1]}, m1 = {md[2], md[3]}, m2 = {md[4], md[5]}, m3 = {md[6], md[7]};
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (i & (1 << J)) continue;
            const cplx a0 = r[i], a1 = r[i | (1 << J)];
            r[i] = row2(m0, m1, a0, a1);
            r[i | (1 << J)] = row2(m2, m3, a0, a1);
        }
    }
}

// JA = register bit of qa, JB = register bit of qb; basis bit(qa) + 2*bit(qb)
template <int R, int JA, int JB>
__device__ __forceinline__ void reg_2q(cplx (&r)[R], int kind, const double* md, uint32_t mono) {
    if (kind == F2_2Q_MONO) {
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (i & ((1 << JA) | (1 << JB))) continue;
            const int idx[4] = {i, i | (1 << JA), i | (1 << JB), i | (1 << JA) | (1 << JB)};
            const cplx a[4] = {r[idx[0]], r[idx[1]], r[idx[2]], r[idx[3]]};
#pragma unroll
            for (int row = 0; row < 4; ++row) {
                const int code = (mono >> (4 * row)) & 15;
                const int src = code & 3;
                const cplx x = src == 0 ? a[0] : (src == 1 ? a[1] : (src == 2 ? a[2] : a[3]));
                r[idx[row]] = mul_unit(x, code >> 2);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (i & ((1 << JA) | (1 << JB))) continue;
            const int idx[4] = {i, i | (1 << JA), i | (1 << JB), i | (1 << JA) | (1 << JB)};
            const cplx a[4] = {r[idx[0]], r[idx[1]], r[idx[2]], r[idx[3]]};
#pragma unroll
            for (int row = 0; row < 4; ++row) {
                const double* m = md + 8 * row;
                const cplx mm[4] = {{m[0], m[1]}, {m[2], m[3]}, {m[4], m[5]}, {m[6], m[7]}};
                r[idx[row]] = row4(mm, a[0], a[1], a[2], a[3]);
            }
        }
    }
}

template <int R>
__device__ __forceinline__ void dispatch_1q(cplx (&r)[R], int j, int kind, const double* md, uint32_t mono) {
    switch (j) {
        case 0: reg_1q<R, 0>(r, kind, md, mono); break;
        case 1: reg_1q<R, 1>(r, kind, md, mono); break;
        case 2: reg_1q<R, 2>(r, kind, md, mono); break;
        default:
            if constexpr (R >= 16) reg_1q<R, 3>(r, kind, md, mono);
            break;
    }
}

template <int R>
__device__ __forceinline__ void dispatch_2q(cplx (&r)[R], int ja, int jb, int kind, const double* md,
                                            uint32_t mono) {
    switch (ja * 4 + jb) {
        case 1: reg_2q<R, 0, 1>(r, kind, md, mono); break;
        case 2: reg_2q<R, 0, 2>(r, kind, md, mono); break;
        case 4: reg_2q<R, 1, 0>(r, kind, md, mono); break;
        case 6: reg_2q<R, 1, 2>(r, kind, md, mono); break;
        case 8: reg_2q<R, 2, 0>(r, kind, md, mono); break;
        case 9: reg_2q<R, 2, 1>(r, kind, md, mono); break;
        default:
            if constexpr (R >= 16) {
                switch (ja * 4 + jb) {
                    case 3: reg_2q<R, 0, 3>(r, kind, md, mono); break;
                    case 7: reg_2q<R, 1, 3>(r, kind, md, mono); break;
                    case 11: reg_2q<R, 2, 3>(r, kind, md, mono); break;
                    case 12: reg_2q<R, 3, 0>(r, kind, md, mono); break;
                    case 13: reg_2q<R, 3, 1>(r, kind, md, mono); break;
                    default: reg_2q<R, 3, 2>(r, kind, md, mono); break;
                }
            }
            break;
    }
}

}  // namespace

template <int KB, int RB, int MINB>
__global__ void __launch_bounds__(1 << (KB - RB), MINB)
    k_fused3(c64s* __restrict__ psi, const __grid_constant__ Fused2Params p) {
    constexpr int TILE = 1 << KB;
    constexpr int R = 1 << RB;                 // amplitudes per thread
    constexpr int NT = TILE / R;               // threads per CTA
    constexpr int TB = KB - RB;                // thread-id bits
    constexpr int CHUNKS = R;                  // 16-byte copies per thread per tile
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cplx* bufs = reinterpret_cast<cplx*>(smem_raw);                       // 2 x TILE, swizzled
    const int tid = threadIdx.x;
    // HBM offset of this thread's chunk bits (prefetch) and of its last-segment bits (direct store)
    uint64_t go_tid = 0, go_last = 0;
    {
        const uint8_t* thr = p.seg_thr[p.n_segs - 1];
#pragma unroll
        for (int j = 0; j < TB; ++j) {
            if ((tid >> j) & 1) {
                go_tid += 1ull << p.tq[j];
                go_last += 1ull << p.tq[thr[j]];
            }
        }
    }
    const int sw_tid = swz(tid);
    __syncthreads();

    auto tile_base = [&](uint64_t t) {
        t = insert_zeros(t, p.cmask_t) | p.cpat_t;       // chunked pass (remap overlap): fixed tile bits
        return p.base_tab[0][t & 255] | p.base_tab[1][(t >> 8) & 255] | p.base_tab[2][(t >> 16) & 255] |
               p.base_tab[3][(t >> 24) & 255];
    };
    auto prefetch = [&](uint64_t t, cplx* dst) {
        const c64s* g = psi + tile_base(t) + go_tid;
#pragma unroll
        for (int j = 0; j < CHUNKS; ++j) cp_async16(dst + (sw_tid + j * NT), g + p.pf_go[j]);
    };

    uint64_t tile = blockIdx.x;
    if (tile < p.n_tiles) prefetch(tile, bufs);
    cp_commit();
    for (int it = 0; tile < p.n_tiles; ++it, tile += gridDim.x) {
        cplx* S = bufs + (it & 1) * TILE;
        const uint64_t next = tile + gridDim.x;
        if (next < p.n_tiles) prefetch(next, bufs + ((it + 1) & 1) * TILE);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const uint64_t base = tile_base(tile);
        cplx r[R];
        int o = 0;
        for (int seg = 0; seg < p.n_segs; ++seg) {
            int tb_seg = 0;
#pragma unroll
            for (int j = 0; j < TB; ++j) tb_seg |= ((tid >> j) & 1) << p.seg_thr[seg][j];
            const int tsw = swz(tb_seg);
            const uint16_t* rsw = p.seg_rsw[seg];
#pragma unroll
            for (int i = 0; i < R; ++i) r[i] = S[tsw ^ rsw[i]];
            const int end = p.seg_end[seg];
            for (; o < end; ++o) {
                const int kind = p.kind[o];
                const double* md = p.mdata + p.moff[o];
                if (kind <= F2_1Q_MONO) {
                    dispatch_1q<R>(r, p.ra[o], kind, md, p.mono[o]);
                } else if (kind <= F2_2Q_MONO) {
                    dispatch_2q<R>(r, p.ra[o], p.rb[o], kind, md, p.mono[o]);
                } else {
                    // thread-position bits of the mask: compare against the unswizzled thread base
                    if ((base & p.dout[o]) != p.dout[o] || (tb_seg & p.dthr[o]) != p.dthr[o]) continue;
                    const int mr = p.dreg[o];
                    if (kind == F2_DIAG_NEG) {
#pragma unroll
                        for (int i = 0; i < R; ++i)
                            if ((i & mr) == mr) r[i] = {-r[i].re, -r[i].im};
                    } else {
                        const cplx f = {md[0], md[1]};
#pragma unroll
                        for (int i = 0; i < R; ++i)
                            if ((i & mr) == mr) r[i] = cmul(r[i], f);
                    }
                }
            }
            if (seg == p.n_segs - 1 && p.direct_out) {
                c64s* gt = psi + base + go_last;
#pragma unroll
                for (int i = 0; i < R; ++i) gt[p.last_rgo[i]] = Store<c64s>::put(r[i]);
            } else {
                __syncthreads();   // every thread has read S for this segment
#pragma unroll
                for (int i = 0; i < R; ++i) S[tsw ^ rsw[i]] = r[i];
                __syncthreads();
            }
        }
        if (!p.direct_out) {
            c64s* gt = psi + base + go_tid;
#pragma unroll
            for (int j = 0; j < CHUNKS; ++j) gt[p.pf_go[j]] = Store<c64s>::put(S[sw_tid + j * NT]);
        }
        __syncthreads();   // S is the prefetch target two tiles from now
    }
    cp_wait<0>();
}

template <int KB, int RB, int MINB>
static cudaError_t fused3_cfg(void* psi, const Fused2Params& p, cudaStream_t st) {
    constexpr int TILE = 1 << KB;
    const size_t smem = 2 * sizeof(cplx) * TILE;
    static bool configured[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k_fused3<KB, RB, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    const uint64_t cap = (uint64_t)sm_count(dev) * MINB;
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(p.n_tiles, cap));
    k_fused3<KB, RB, MINB><<<g, TILE >> RB, smem, st>>>(static_cast<c64s*>(psi), p);
    count_launch();
    return cudaGetLastError();
}

// cfg: 1 = 2^12 tile, 16 amplitudes/thread, 1 CTA/SM; 2 = 2^11 tile, 8/thread, 2 CTAs/SM;
//      3 = 2^12 tile, 8/thread (512 threads), 1 CTA/SM
cudaError_t launch_fused2(void* psi, int mode, const Fused2Params& p, cudaStream_t st) {
    static_assert(sizeof(Fused2Params) < 32700, "kernel parameter block too large");
    if (mode != SV_FP64) return cudaErrorInvalidValue;
    switch (p.cfg) {
        case 2: return fused3_cfg<11, 3, 2>(psi, p, st);
        case 3: return fused3_cfg<12, 3, 1>(psi, p, st);
        case 4: return fused3_cfg<11, 3, 3>(psi, p, st);
        case 5: return fused3_cfg<10, 3, 4>(psi, p, st);
        case 6: return fused3_cfg<11, 4, 3>(psi, p, st);
        case 7: return fused3_cfg<10, 4, 6>(psi, p, st);
        case 8: return fused3_cfg<12, 4, 1>(psi, p, st);   // generic stand-in for the JIT-only config 8
        case 10: return cudaErrorNotSupported;               // 2^13 tiles: specialised kernel only
        default: return fused3_cfg<12, 4, 1>(psi, p, st);
    }
}

}  // namespace sv
