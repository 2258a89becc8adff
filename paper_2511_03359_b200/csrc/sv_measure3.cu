// All-qubit measurement reductions, register-resident form (FP64 storage, sm_100a).
//
// Same sums as k_measure (sv_measure.cu; reference svsim/measure.py:51-56):
//   norm, ones_q = sum_{bit q = 1} |a|^2, cross_q = sum_{bit q = 0} conj(a_i) a_{i + 2^q}
// but organised like the fused gate pass k_fused3 (sv_fused2.cu): tiles of
// 2^KB amplitudes stream into swizzled shared memory with cp.async (double
// buffered), and each thread then reads 16 amplitudes spanning 4 "register
// positions" of the tile per segment.  Every cross term of a register position
// is a register-register product, so a segment reads each amplitude from shared
// memory once (k_measure read it twice per tile qubit: 24 LDS.128 per amplitude
// at KB = 12, shared-memory bound at ~2.8 TB/s).  A pass needs ceil(#cross
// positions / 4) segments.
//
// Results are deterministic: per-CTA partial rows (warp shuffles, fixed-order
// sums over warps), summed on the host in CTA order.  The reference sums with
// numpy (pairwise), so reports agree within the 1e-12 the north star allows,
// not bit for bit (test_gpu_fp.py).
#include <algorithm>

#include "sv_common.cuh"
#include "sv_kernels.cuh"

namespace sv {

namespace {

// swizzle with the pass's columns (chosen on the host so that every segment's quarter-warp
// loads are conflict-free)
__device__ __forceinline__ int swz3(int e, const uint8_t (&c)[4]) {
    const int g = (((e >> 3) & 1) * c[0]) ^ (((e >> 4) & 1) * c[1]) ^ (((e >> 5) & 1) * c[2]) ^ (((e >> 6) & 1) * c[3]);
    return e ^ g;
}

__device__ __forceinline__ void cp_async16m(void* smem_dst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit_m() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_m() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// with a source size (0: 16 zero bytes, nothing read) -- a dirty support's unwritten HBM
__device__ __forceinline__ void cp_async16mz(void* smem_dst, const void* gsrc, unsigned bytes) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(bytes) : "memory");
}

constexpr int kOutMax = 52;

}  // namespace

// BYTE = true: the state is two uint8 planes (sv_byte.cu); each thread loads 16
// consecutive magnitude / phase bytes of the tile (tile positions 0..3 are qubits 0..3),
// decodes them with the reference's single rounding (codec.py:203-206) into the
// shared-memory tile, and the next tile's bytes are already in flight in registers.
// NSEG: register segments per tile (3 for the first pass, whose 12 tile positions are all
// new; later passes keep 5 done low positions for coalescing and need 2); ONES: the first
// pass also sums |a|^2 per qubit.  The 2-segment form without ONES fits 128 registers,
// i.e. 2 CTAs per SM (16 warps instead of 8 to hide the HBM latency).
// RB: register bits per segment (R = 2^RB amplitudes per thread, 2^(KB-RB) threads).
// RB = 3 (8 amplitudes per thread, 4 segments per 12-bit tile, 16 warps per SM) was
// measured slower than the 2-CTA RB = 4 variants (N=33: 126 vs 108 ms) and is not launched.
// DIRECT (FP64): segment 0 loads its 16 registers straight from HBM -- its lanes are tile
// positions 0..4 = qubits 0..4, so a warp load is 512 contiguous bytes -- and stores them
// into the shared-memory tile only for the later segments: one shared-memory sweep less per
// tile (the 3-segment first pass is shared-memory bound: cp.async write + 3 reads = 4 sweeps
// of the tile at 128 B/clk vs its HBM read).  The next tile is prefetched into L2.
template <int KB, int MINB, bool BYTE, int NSEG, bool ONES, int RB = 4, bool DIRECT = false>
__global__ void __launch_bounds__(1 << (KB - RB), MINB)
    k_measure3(const c64s* __restrict__ psi, const __grid_constant__ Measure3Params p, double* __restrict__ partials,
               const MeasureBytes bsrc) {
    constexpr int TILE = 1 << KB, R = 1 << RB, NT = TILE / R, TB = KB - RB, NW = NT / 32;
    static_assert(!BYTE || RB == 4, "BYTE decode: 16 bytes per thread");
    // FP64 with 2 CTAs per SM: one tile buffer (2 x 2 x 64 KB would not fit); the next tile is
    // requested once the last segment holds the tile in registers, the other CTA covers the gap
    static_assert(!(DIRECT && BYTE), "direct loads read FP64 tiles");
    constexpr bool SINGLE = !BYTE && MINB >= 2 && !DIRECT;
    constexpr int NBUF = (BYTE || SINGLE || DIRECT) ? 1 : 2;
    // 2 CTAs per SM with 3 segments: segment 0 accumulates in registers, segments 1, 2 add
    // their per-tile sums to thread-private shared-memory slots (16 doubles per thread)
    constexpr bool ACC_SMEM = !BYTE && MINB >= 2 && NSEG >= 3;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cplx* bufs = reinterpret_cast<cplx*>(smem_raw);
    double* ow = reinterpret_cast<double*>(smem_raw + NBUF * sizeof(cplx) * TILE);  // [NW][kOutMax]
    double* red = ow + NW * kOutMax;                                                 // [NW][1 + 3 KB]
    constexpr int NSL = 1 + 3 * KB;
    double* dtab = red + NW * NSL;                                                   // BYTE: dmag, dux, duy
    // BYTE: ring of NSTAGE raw tiles (magnitude bytes, phase bytes) filled by cp.async, so that
    // NSTAGE - 1 tiles of bytes are in flight while one is decoded
    constexpr int NSTAGE = 4;
    unsigned char* stage = reinterpret_cast<unsigned char*>(dtab + 768);                // [NSTAGE][2][TILE]
    double* accs = red + NW * NSL;   // ACC_SMEM: slot k of thread t at accs[k * NT + t]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if constexpr (ACC_SMEM)
        for (int i = tid; i < (NSEG - 1) * 2 * RB * NT; i += NT) accs[i] = 0.0;
    for (int i = tid; i < NW * kOutMax; i += NT) ow[i] = 0.0;
    for (int i = tid; i < NW * NSL; i += NT) red[i] = 0.0;
    if constexpr (BYTE)
        for (int i = tid; i < 768; i += NT) dtab[i] = bsrc.tab[i];
    uint64_t go_tid = 0;
#pragma unroll
    for (int j = 0; j < TB; ++j)
        if ((tid >> j) & 1) go_tid += 1ull << p.tq[j];
    const int sw_tid = swz3(tid, p.swz_cols);
    __syncthreads();

    auto tile_base = [&](uint64_t t) {
        return p.base_tab[0][t & 255] | p.base_tab[1][(t >> 8) & 255] | p.base_tab[2][(t >> 16) & 255] |
               p.base_tab[3][(t >> 24) & 255] | p.base_const;
    };
    auto prefetch = [&](uint64_t t, cplx* dst) {
        const uint64_t gb = tile_base(t) + go_tid;
        const c64s* g = psi + gb;
        if (p.pfix) {   // amplitudes outside the support were never written: zeros
#pragma unroll
            for (int j = 0; j < R; ++j)
                cp_async16mz(dst + (sw_tid + j * NT), g + p.pf_go[j],
                             ((gb + p.pf_go[j]) & p.pfix) == p.pval ? 16u : 0u);
            return;
        }
#pragma unroll
        for (int j = 0; j < R; ++j) cp_async16m(dst + (sw_tid + j * NT), g + p.pf_go[j]);
    };
    uint64_t go0 = 0;   // DIRECT: HBM offset of this thread's segment-0 registers
    if constexpr (DIRECT) {
#pragma unroll
        for (int j = 0; j < TB; ++j)
            if ((tid >> j) & 1) go0 += 1ull << p.tq[p.seg_thr[0][j]];
    }

    double tw_all = 0.0, twr[RB];
    double out_acc0 = 0.0, out_acc1 = 0.0;   // ONES: out-of-tile qubits lane, lane + 32
    const int oq0 = lane < p.n_out ? p.oq[lane] : 0, oq1 = lane + 32 < p.n_out ? p.oq[lane + 32] : 0;
    double cr[NSEG][RB], ci[NSEG][RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) twr[j] = 0.0;
#pragma unroll
    for (int s = 0; s < NSEG; ++s)
#pragma unroll
        for (int j = 0; j < RB; ++j) cr[s][j] = ci[s][j] = 0.0;

    // BYTE: this thread's 16-byte chunk of the tile (elements 16 tid .. 16 tid + 15)
    uint64_t go_chunk = 0;
    if constexpr (BYTE) {
#pragma unroll
        for (int j = 0; j < KB - 4; ++j)
            if ((tid >> j) & 1) go_chunk += 1ull << p.tq[4 + j];
    }
    auto fetch_bytes = [&](uint64_t t, int sidx) {
        const uint64_t a = tile_base(t) + go_chunk;
        unsigned char* st = stage + (size_t)sidx * 2 * TILE;
        cp_async16m(st + 16 * tid, bsrc.mi + a);
        cp_async16m(st + TILE + 16 * tid, bsrc.pi + a);
    };

    uint64_t tile = blockIdx.x;
    if constexpr (BYTE) {
#pragma unroll
        for (int k = 0; k < NSTAGE - 1; ++k) {
            const uint64_t tk = tile + (uint64_t)k * gridDim.x;
            if (tk < p.n_tiles) fetch_bytes(tk, k);
            cp_commit_m();
        }
    } else if constexpr (!DIRECT) {
        if (tile < p.n_tiles) prefetch(tile, bufs);
        cp_commit_m();
    }
    for (int it = 0; tile < p.n_tiles; ++it, tile += gridDim.x) {
        cplx* S = bufs + (NBUF == 1 ? 0 : (it & 1) * TILE);
        const uint64_t next = tile + gridDim.x;
        if constexpr (BYTE) {
            cp_wait_m<NSTAGE - 2>();      // this tile's bytes landed (the newer ones may not)
            __syncthreads();
            const uint64_t ahead = tile + (uint64_t)(NSTAGE - 1) * gridDim.x;
            if (ahead < p.n_tiles) fetch_bytes(ahead, (it + NSTAGE - 1) % NSTAGE);
            cp_commit_m();
            const unsigned char* st = stage + (size_t)(it % NSTAGE) * 2 * TILE;
            const uint4 cm = *reinterpret_cast<const uint4*>(st + 16 * tid);
            const uint4 cpp = *reinterpret_cast<const uint4*>(st + TILE + 16 * tid);
            const unsigned wm[4] = {cm.x, cm.y, cm.z, cm.w}, wp[4] = {cpp.x, cpp.y, cpp.z, cpp.w};
            auto uniform = [](const uint4& v) {
                return v.x == v.y && v.x == v.z && v.x == v.w && v.x == (v.x & 255u) * 0x01010101u;
            };
            if (uniform(cm) && uniform(cpp)) {   // structured states: one decode for 16 amplitudes
                const unsigned mi = cm.x & 255u, pi = cpp.x & 255u;
                const double m = dtab[mi];
                const cplx v = mi == 0 ? cplx{0.0, 0.0} : cplx{__dmul_rn(m, dtab[256 + pi]), __dmul_rn(m, dtab[512 + pi])};
#pragma unroll
                for (int i = 0; i < 16; ++i) S[swz3(16 * tid + i, p.swz_cols)] = v;
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const unsigned mi = (wm[i >> 2] >> (8 * (i & 3))) & 255u, pi = (wp[i >> 2] >> (8 * (i & 3))) & 255u;
                    const double m = dtab[mi];
                    const cplx v =
                        mi == 0 ? cplx{0.0, 0.0} : cplx{__dmul_rn(m, dtab[256 + pi]), __dmul_rn(m, dtab[512 + pi])};
                    S[swz3(16 * tid + i, p.swz_cols)] = v;
                }
            }
        } else if constexpr (DIRECT) {
            if (next < p.n_tiles) {   // the next tile's lines into L2 while this one is reduced
                const c64s* g = psi + tile_base(next) + go0;
#pragma unroll
                for (int i = 0; i < R; ++i)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(g + p.seg0_go[i]));
            }
        } else if constexpr (SINGLE) {
            cp_wait_m<0>();
        } else {
            if (next < p.n_tiles) prefetch(next, bufs + ((it + 1) & 1) * TILE);
            cp_commit_m();
            cp_wait_m<1>();
        }
        if constexpr (!DIRECT) __syncthreads();
#pragma unroll
        for (int s = 0; s < NSEG; ++s) {
            if (s >= p.n_segs) break;
            int tb = 0;
#pragma unroll
            for (int j = 0; j < TB; ++j) tb |= ((tid >> j) & 1) << p.seg_thr[s][j];
            const int tsw = swz3(tb, p.swz_cols);
            cplx r[R];
            if (DIRECT && s == 0) {
                const c64s* g = psi + tile_base(tile) + go0;
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    double re, im;
                    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                                 : "=d"(re), "=d"(im) : "l"(g + p.seg0_go[i]));
                    r[i] = {re, im};
                }
                if (p.n_segs > 1) {   // the later segments read the tile from shared memory
                    __syncthreads();  // (the previous tile's last segment has read it)
#pragma unroll
                    for (int i = 0; i < R; ++i) S[tsw ^ p.seg_rsw[0][i]] = r[i];
                    __syncthreads();
                }
            } else {
#pragma unroll
                for (int i = 0; i < R; ++i) r[i] = S[tsw ^ p.seg_rsw[s][i]];
            }
            if constexpr (SINGLE) {
                if (s == p.n_segs - 1) {   // tile in registers: the buffer takes the next tile
                    __syncthreads();
                    if (next < p.n_tiles) prefetch(next, S);
                    cp_commit_m();
                }
            }
            if (ONES && s == 0) {
                double tt = 0.0;
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    const double w = r[i].re * r[i].re + r[i].im * r[i].im;
                    tt += w;
#pragma unroll
                    for (int j = 0; j < RB; ++j)
                        if ((i >> j) & 1) twr[j] += w;
                }
                tw_all += tt;
                // out-of-tile qubits: bit constant over the tile.  Every lane gets the warp's
                // tile sum and lane j adds it for out-of-tile qubit j (and j + 32): no serial
                // per-qubit loop in lane 0 (a chain of shared-memory read-modify-writes per tile)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, o);
                const uint64_t base = tile_base(tile);
                if (lane < p.n_out && ((base >> oq0) & 1)) out_acc0 += tt;
                if (lane + 32 < p.n_out && ((base >> oq1) & 1)) out_acc1 += tt;
            }
            const uint32_t cm = p.cross_reg[s];
            if (ACC_SMEM && s > 0) {
#pragma unroll
                for (int j = 0; j < RB; ++j) {
                    if (!((cm >> j) & 1)) continue;
                    double lr = 0.0, li = 0.0;
#pragma unroll
                    for (int i = 0; i < R; ++i) {
                        if ((i >> j) & 1) continue;
                        const cplx a0 = r[i], a1 = r[i | (1 << j)];
                        lr = __fma_rn(a0.im, a1.im, __fma_rn(a0.re, a1.re, lr));
                        li = __fma_rn(-a0.im, a1.re, __fma_rn(a0.re, a1.im, li));
                    }
                    const int k = ((s - 1) * RB + j) * 2;
                    accs[k * NT + tid] += lr;
                    accs[(k + 1) * NT + tid] += li;
                }
                continue;
            }
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                if (!((cm >> j) & 1)) continue;
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    if ((i >> j) & 1) continue;
                    const cplx a0 = r[i], a1 = r[i | (1 << j)];
                    // conj(a0) a1 accumulated with two fused multiply-adds per part (reports
                    // are compared within 1e-12, not bit for bit; one rounding per product)
                    cr[s][j] = __fma_rn(a0.im, a1.im, __fma_rn(a0.re, a1.re, cr[s][j]));
                    ci[s][j] = __fma_rn(-a0.im, a1.re, __fma_rn(a0.re, a1.im, ci[s][j]));
                }
            }
        }
        if constexpr (!SINGLE) __syncthreads();   // S is the prefetch target two tiles from now (BYTE: the next tile)
    }
    cp_wait_m<0>();

    // ---- deterministic reduction: warp shuffles, then fixed-order sum over warps ----
    // slots: [0] norm, [1 + pos] ones of tile position pos, [1 + KB + 2 pos (+1)] cross of pos
    auto wsum = [&](double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        return v;
    };
    double v = wsum(tw_all);
    if (lane == 0) red[warp * NSL + 0] = v;
    if (ONES) {
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            v = wsum(twr[j]);
            if (lane == 0) red[warp * NSL + 1 + p.seg_reg[0][j]] = v;
        }
#pragma unroll
        for (int j = 0; j < TB; ++j) {
            v = wsum(((tid >> j) & 1) ? tw_all : 0.0);
            if (lane == 0) red[warp * NSL + 1 + p.seg_thr[0][j]] = v;
        }
        if (lane < p.n_out) ow[warp * kOutMax + lane] = out_acc0;
        if (lane + 32 < p.n_out) ow[warp * kOutMax + lane + 32] = out_acc1;
    }
#pragma unroll
    for (int s = 0; s < NSEG; ++s)
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            if (s >= p.n_segs || !((p.cross_reg[s] >> j) & 1)) continue;
            const int k = ((s - 1) * RB + j) * 2;
            const double a = wsum((ACC_SMEM && s > 0) ? accs[k * NT + tid] : cr[s][j]);
            const double b = wsum((ACC_SMEM && s > 0) ? accs[(k + 1) * NT + tid] : ci[s][j]);
            if (lane == 0) {
                red[warp * NSL + 1 + KB + 2 * p.seg_reg[s][j]] = a;
                red[warp * NSL + 2 + KB + 2 * p.seg_reg[s][j]] = b;
            }
        }
    __syncthreads();
    const int nslots = 1 + p.n + 2 * KB;
    double* row = partials + (uint64_t)blockIdx.x * nslots;
    for (int sl = tid; sl < NSL; sl += NT) {
        double acc = 0.0;
        for (int w = 0; w < NW; ++w) acc += red[w * NSL + sl];
        const int dst = sl <= KB ? sl : sl + p.n_out;   // tile ones, then out ones, then cross
        row[dst] = acc;
    }
    for (int j = tid; j < p.n_out; j += NT) {
        double acc = 0.0;
        for (int w = 0; w < NW; ++w) acc += ow[w * kOutMax + j];
        row[1 + KB + j] = acc;
    }
}

template <int KB, int MINB, bool BYTE, int NSEG, bool ONES, int RB = 4, bool DIRECT = false>
static cudaError_t measure3_cfg(const c64s* psi, const Measure3Params& p, double* partials, int grid,
                                cudaStream_t st, const MeasureBytes& b) {
    constexpr int TILE = 1 << KB, NW = (TILE >> RB) / 32;
    constexpr bool ACC_SMEM = !BYTE && MINB >= 2 && NSEG >= 3;
    const size_t smem = (ACC_SMEM ? sizeof(double) * (NSEG - 1) * 2 * RB * (TILE >> RB) : 0) +
                        ((BYTE || MINB >= 2 || DIRECT) ? 1 : 2) * sizeof(cplx) * TILE + sizeof(double) * NW * (kOutMax + 1 + 3 * KB) +
                        (BYTE ? sizeof(double) * 768 + 4 * 2 * TILE : 0);
    static bool configured[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k_measure3<KB, MINB, BYTE, NSEG, ONES, RB, DIRECT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    k_measure3<KB, MINB, BYTE, NSEG, ONES, RB, DIRECT><<<grid, TILE >> RB, smem, st>>>(psi, p, partials, b);
    count_launch();
    return cudaGetLastError();
}

// CTAs per SM of the variant a pass runs (grid = that x SMs)
static bool light_pass(const Measure3Params& p) { return !p.want_ones && p.n_segs <= 2; }
int measure3_ctas_per_sm(int kb, bool byte, const Measure3Params& p) {
    if (kb != 12) return 3;
    if (byte) return light_pass(p) ? 2 : 1;
    return 2;   // light passes, and the 3-segment pass with shared-memory accumulators
}
int measure3_grid(int device, int kb, bool byte) { return sm_count(device) * (kb == 12 ? 2 : 3); }   // max over variants

cudaError_t launch_measure3(const void* psi, const Measure3Params& p, double* partials, int grid, cudaStream_t st) {
    const MeasureBytes none{nullptr, nullptr, nullptr};
    const c64s* s = static_cast<const c64s*>(psi);
    if (p.kbits != 12) return measure3_cfg<11, 3, false, 3, true>(s, p, partials, grid, st, none);
    if (p.direct)
        return light_pass(p) ? measure3_cfg<12, 2, false, 2, false, 4, true>(s, p, partials, grid, st, none)
                             : measure3_cfg<12, 2, false, 3, true, 4, true>(s, p, partials, grid, st, none);
    return light_pass(p) ? measure3_cfg<12, 2, false, 2, false>(s, p, partials, grid, st, none)
                         : measure3_cfg<12, 2, false, 3, true>(s, p, partials, grid, st, none);
}

cudaError_t launch_measure3_byte(const MeasureBytes& b, const Measure3Params& p, double* partials, int grid,
                                 cudaStream_t st) {
    return light_pass(p) ? measure3_cfg<12, 2, true, 2, false>(nullptr, p, partials, grid, st, b)
                         : measure3_cfg<12, 1, true, 3, true>(nullptr, p, partials, grid, st, b);
}

}  // namespace sv
