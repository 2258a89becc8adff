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

constexpr int kOutMax = 52;

}  // namespace

// BYTE = true: the state is two uint8 planes (sv_byte.cu); each thread loads 16
// consecutive magnitude / phase bytes of the tile (tile positions 0..3 are qubits 0..3),
// decodes them with the reference's single rounding (codec.py:203-206) into the
// shared-memory tile, and the next tile's bytes are already in flight in registers.
template <int KB, int MINB, bool BYTE>
__global__ void __launch_bounds__(1 << (KB - 4), MINB)
    k_measure3(const c64s* __restrict__ psi, const __grid_constant__ Measure3Params p, double* __restrict__ partials,
               const MeasureBytes bsrc) {
    constexpr int TILE = 1 << KB, R = 16, NT = TILE / R, TB = KB - 4, NW = NT / 32;
    constexpr int NBUF = BYTE ? 1 : 2;
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
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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
               p.base_tab[3][(t >> 24) & 255];
    };
    auto prefetch = [&](uint64_t t, cplx* dst) {
        const c64s* g = psi + tile_base(t) + go_tid;
#pragma unroll
        for (int j = 0; j < R; ++j) cp_async16m(dst + (sw_tid + j * NT), g + p.pf_go[j]);
    };

    double tw_all = 0.0, twr[4] = {0.0, 0.0, 0.0, 0.0};
    double cr[3][4], ci[3][4];
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
        for (int j = 0; j < 4; ++j) cr[s][j] = ci[s][j] = 0.0;

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
    } else {
        if (tile < p.n_tiles) prefetch(tile, bufs);
        cp_commit_m();
    }
    for (int it = 0; tile < p.n_tiles; ++it, tile += gridDim.x) {
        cplx* S = bufs + (BYTE ? 0 : (it & 1) * TILE);
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
        } else {
            if (next < p.n_tiles) prefetch(next, bufs + ((it + 1) & 1) * TILE);
            cp_commit_m();
            cp_wait_m<1>();
        }
        __syncthreads();
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            if (s >= p.n_segs) break;
            int tb = 0;
#pragma unroll
            for (int j = 0; j < TB; ++j) tb |= ((tid >> j) & 1) << p.seg_thr[s][j];
            const int tsw = swz3(tb, p.swz_cols);
            cplx r[R];
#pragma unroll
            for (int i = 0; i < R; ++i) r[i] = S[tsw ^ p.seg_rsw[s][i]];
            if (s == 0 && p.want_ones) {
                double tt = 0.0;
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    const double w = r[i].re * r[i].re + r[i].im * r[i].im;
                    tt += w;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if ((i >> j) & 1) twr[j] += w;
                }
                tw_all += tt;
                // out-of-tile qubits: bit constant over the tile
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) tt += __shfl_down_sync(0xffffffffu, tt, o);
                if (lane == 0) {
                    const uint64_t base = tile_base(tile);
                    for (int j = 0; j < p.n_out; ++j)
                        if ((base >> p.oq[j]) & 1) ow[warp * kOutMax + j] += tt;
                }
            }
            const uint32_t cm = p.cross_reg[s];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (!((cm >> j) & 1)) continue;
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    if ((i >> j) & 1) continue;
                    const cplx a0 = r[i], a1 = r[i | (1 << j)];
                    cr[s][j] += a0.re * a1.re + a0.im * a1.im;
                    ci[s][j] += a0.re * a1.im - a0.im * a1.re;
                }
            }
        }
        __syncthreads();   // S is the prefetch target two tiles from now (BYTE: the next tile)
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
    if (p.want_ones) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v = wsum(twr[j]);
            if (lane == 0) red[warp * NSL + 1 + p.seg_reg[0][j]] = v;
        }
#pragma unroll
        for (int j = 0; j < TB; ++j) {
            v = wsum(((tid >> j) & 1) ? tw_all : 0.0);
            if (lane == 0) red[warp * NSL + 1 + p.seg_thr[0][j]] = v;
        }
    }
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (s >= p.n_segs || !((p.cross_reg[s] >> j) & 1)) continue;
            const double a = wsum(cr[s][j]), b = wsum(ci[s][j]);
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

template <int KB, int MINB, bool BYTE>
static cudaError_t measure3_cfg(const c64s* psi, const Measure3Params& p, double* partials, int grid,
                                cudaStream_t st, const MeasureBytes& b) {
    constexpr int TILE = 1 << KB, NW = (TILE / 16) / 32;
    const size_t smem = (BYTE ? 1 : 2) * sizeof(cplx) * TILE + sizeof(double) * NW * (kOutMax + 1 + 3 * KB) +
                        (BYTE ? sizeof(double) * 768 + 4 * 2 * TILE : 0);
    static bool configured[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k_measure3<KB, MINB, BYTE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    k_measure3<KB, MINB, BYTE><<<grid, TILE / 16, smem, st>>>(psi, p, partials, b);
    count_launch();
    return cudaGetLastError();
}

int measure3_grid(int device, int kb, bool byte) { return sm_count(device) * (byte ? 1 : (kb == 12 ? 1 : 3)); }

cudaError_t launch_measure3(const void* psi, const Measure3Params& p, double* partials, int grid, cudaStream_t st) {
    const MeasureBytes none{nullptr, nullptr, nullptr};
    const c64s* s = static_cast<const c64s*>(psi);
    return p.kbits == 12 ? measure3_cfg<12, 1, false>(s, p, partials, grid, st, none)
                         : measure3_cfg<11, 3, false>(s, p, partials, grid, st, none);
}

cudaError_t launch_measure3_byte(const MeasureBytes& b, const Measure3Params& p, double* partials, int grid,
                                 cudaStream_t st) {
    return measure3_cfg<12, 1, true>(nullptr, p, partials, grid, st, b);   // 2 CTAs/SM spill (128 regs)
}

}  // namespace sv
