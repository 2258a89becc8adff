// All-qubit three-axis measurement reductions (sm_100a).
//
// Reference: /root/reference/pkg/src/svsim/measure.py
//   _pair_sums_local 51-56: ones_q  = sum_{bit q = 1} |a|^2
//                           cross_q = sum_{bit q = 0} conj(a_i) * a_{i + 2^q}
//   measure_all 59-109:      N full passes over the state (one per qubit)
// Here a pass stages tiles of 2^k amplitudes (tile qubits T) in shared memory
// and produces, per CTA, the norm, ones_q for EVERY local qubit (first pass
// only: for q outside T the bit is constant over the tile) and cross_q for
// every requested q in T.  ceil((n - k) / (k - b)) + 1 passes cover all
// qubits instead of n.  Partials are written per CTA and summed on the host
// in a fixed order, so results are deterministic (no float atomics) and
// independent of scheduling (test_engine.py:147-153).
#include <algorithm>

#include "sv_common.cuh"
#include "sv_kernels.cuh"

namespace sv {

int measure_slots(int k, int n) { return 1 + n + 2 * k; }

constexpr int kMaxOut = 40;

// BYTE storage (two uint8 planes) is decoded on the fly: mags[mi] * (ux[pi], uy[pi])
// with the same single rounding as codec.py:203-206, so a BYTE state is measured
// without ever materialising it in FP64.
struct ByteSrc {
    const uint8_t* mi;
    const uint8_t* pi;
    const double* tab;      // dmag[256], dux[256], duy[256] (ByteTables prefix)
};

template <typename S, int K, bool BYTE>
__global__ void __launch_bounds__(256) k_measure(const S* __restrict__ psi,
                                                 const __grid_constant__ MeasureParams p,
                                                 double* __restrict__ partials, const ByteSrc bsrc) {
    constexpr int NT = 256;
    constexpr int TILE = 1 << K;
    constexpr int V = Store<S>::V;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* s = reinterpret_cast<cplx*>(smem_raw);
    uint64_t* off_hi = reinterpret_cast<uint64_t*>(smem_raw + sizeof(cplx) * TILE);
    // per-warp one-weights of the out-of-tile qubits (constant bit per tile)
    double* ow = reinterpret_cast<double*>(smem_raw + sizeof(cplx) * TILE + sizeof(uint64_t) * TILE);
    double* red = ow + (NT / 32) * kMaxOut;             // block-reduction scratch
    double* dtab = red + 8 * (1 + 64 + 2 * 12);         // BYTE decode tables (768 doubles)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (NT / 32) * kMaxOut; i += NT) ow[i] = 0.0;
    if constexpr (BYTE)
        for (int i = threadIdx.x; i < 768; i += NT) dtab[i] = bsrc.tab[i];

    const int b = p.b;
    const int nhi = 1 << (K - b);
    for (int h = threadIdx.x; h < nhi; h += NT) {
        uint64_t o = 0;
        for (int j = 0; j < K - b; ++j)
            if ((h >> j) & 1) o |= 1ull << p.tq[b + j];
        off_hi[h] = o;
    }
    __syncthreads();
    const uint32_t lowmask = (1u << b) - 1u;
    const int n_out = p.n - K;

    double norm = 0.0;
    double onesT[K];
    double cre[K], cim[K];
#pragma unroll
    for (int i = 0; i < K; ++i) onesT[i] = cre[i] = cim[i] = 0.0;

    for (uint64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        const uint64_t base = insert_zeros(tile, p.tile_mask);
        if constexpr (BYTE) {
            for (int e = threadIdx.x; e < TILE; e += NT) {
                const uint64_t i = base + off_hi[e >> b] + (e & lowmask);
                const uint8_t mi = bsrc.mi[i], pi = bsrc.pi[i];
                s[e] = mi == 0 ? cplx{0.0, 0.0}
                               : cplx{__dmul_rn(dtab[mi], dtab[256 + pi]), __dmul_rn(dtab[mi], dtab[512 + pi])};
            }
        } else if constexpr (TILE >= NT * V) {
            constexpr int PER = TILE / (NT * V);
            Vec<S> buf[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const uint32_t e = (threadIdx.x + j * NT) * V;
                buf[j] = vload(psi + base + off_hi[e >> b] + (e & lowmask));
            }
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const uint32_t e = (threadIdx.x + j * NT) * V;
#pragma unroll
                for (int v = 0; v < V; ++v) s[e + v] = Store<S>::get(buf[j].a[v]);
            }
        } else {
            for (int e = threadIdx.x; e < TILE; e += NT)
                s[e] = Store<S>::get(psi[base + off_hi[e >> b] + (e & lowmask)]);
        }
        __syncthreads();
        if (p.want_ones) {
            double tn = 0.0;
            for (int e = threadIdx.x; e < TILE; e += NT) {
                const cplx a = s[e];
                const double w = a.re * a.re + a.im * a.im;
                tn += w;
#pragma unroll
                for (int i = 0; i < K; ++i)
                    if ((e >> i) & 1) onesT[i] += w;
            }
            norm += tn;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tn += __shfl_down_sync(0xffffffffu, tn, o);
            if (lane == 0)
                for (int j = 0; j < n_out; ++j)
                    if ((base >> p.oq[j]) & 1) ow[warp * kMaxOut + j] += tn;
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (!((p.cross_pos >> i) & 1)) continue;
            for (int w = threadIdx.x; w < TILE / 2; w += NT) {
                const int e0 = (int)insert0((uint64_t)w, i);
                const cplx a0 = s[e0], a1 = s[e0 | (1 << i)];
                cre[i] += a0.re * a1.re + a0.im * a1.im;
                cim[i] += a0.re * a1.im - a0.im * a1.re;
            }
        }
        __syncthreads();
    }

    // ---- deterministic block reduction: warp shuffle, then fixed-order sum of warps ----
    // slot layout: [norm][ones over tile positions: K][ones over out-of-tile qubits: n-K]
    //              [cross (re, im) over tile positions: 2K]
    const int nslots = 1 + p.n + 2 * K;
    double* rowv = partials + (uint64_t)blockIdx.x * nslots;
    auto wsum = [&](double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        return v;
    };
    const int nreg = 1 + 3 * K;                 // register-held slots
    double v0 = wsum(norm);
    if (lane == 0) red[0 * (NT / 32) + warp] = v0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const double a = wsum(onesT[i]), c = wsum(cre[i]), d = wsum(cim[i]);
        if (lane == 0) {
            red[(1 + i) * (NT / 32) + warp] = a;
            red[(1 + K + 2 * i) * (NT / 32) + warp] = c;
            red[(2 + K + 2 * i) * (NT / 32) + warp] = d;
        }
    }
    __syncthreads();
    for (int sl = threadIdx.x; sl < nreg; sl += NT) {
        double v = 0.0;
        for (int w = 0; w < NT / 32; ++w) v += red[sl * (NT / 32) + w];
        const int dst = sl == 0 ? 0 : (sl <= K ? sl : sl + n_out);
        rowv[dst] = v;
    }
    for (int j = threadIdx.x; j < n_out; j += NT) {
        double v = 0.0;
        for (int w = 0; w < NT / 32; ++w) v += ow[w * kMaxOut + j];
        rowv[1 + K + j] = v;
    }
}

int measure_grid(int device) { return sm_count(device) * 2; }

template <typename S, int K, bool BYTE>
static cudaError_t measure_k(const S* psi, const MeasureParams& p, double* partials, int grid,
                             cudaStream_t st, const ByteSrc& bsrc) {
    const size_t tile_bytes = sizeof(cplx) * (1u << K) + sizeof(uint64_t) * (1u << K) +
                              sizeof(double) * 8 * kMaxOut;
    const size_t red_bytes = sizeof(double) * (size_t)(1 + 64 + 2 * 12) * 8;
    const size_t smem = tile_bytes + red_bytes + (BYTE ? sizeof(double) * 768 : 0);
    static bool configured[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k_measure<S, K, BYTE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(tile_bytes + red_bytes + sizeof(double) * 768));
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    k_measure<S, K, BYTE><<<grid, 256, smem, st>>>(psi, p, partials, bsrc);
    count_launch();
    return cudaGetLastError();
}

template <typename S, bool BYTE>
static cudaError_t measure_t(const S* psi, const MeasureParams& p, double* partials, int grid,
                             cudaStream_t st, const ByteSrc& bsrc) {
    switch (p.k) {
        case 1: return measure_k<S, 1, BYTE>(psi, p, partials, grid, st, bsrc);
        case 2: return measure_k<S, 2, BYTE>(psi, p, partials, grid, st, bsrc);
        case 3: return measure_k<S, 3, BYTE>(psi, p, partials, grid, st, bsrc);
        case 4: return measure_k<S, 4, BYTE>(psi, p, partials, grid, st, bsrc);
        case 5: return measure_k<S, 5, BYTE>(psi, p, partials, grid, st, bsrc);
        case 6: return measure_k<S, 6, BYTE>(psi, p, partials, grid, st, bsrc);
        case 7: return measure_k<S, 7, BYTE>(psi, p, partials, grid, st, bsrc);
        case 8: return measure_k<S, 8, BYTE>(psi, p, partials, grid, st, bsrc);
        case 9: return measure_k<S, 9, BYTE>(psi, p, partials, grid, st, bsrc);
        case 10: return measure_k<S, 10, BYTE>(psi, p, partials, grid, st, bsrc);
        case 11: return measure_k<S, 11, BYTE>(psi, p, partials, grid, st, bsrc);
        case 12: return measure_k<S, 12, BYTE>(psi, p, partials, grid, st, bsrc);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_measure(const void* psi, int mode, const MeasureParams& p, double* partials,
                           int grid, cudaStream_t st) {
    const ByteSrc none{nullptr, nullptr, nullptr};
    if (mode == SV_BYTE) {
        const ByteSrc* b = static_cast<const ByteSrc*>(psi);
        return measure_t<c64s, true>(nullptr, p, partials, grid, st, *b);
    }
    return mode == SV_FP32 ? measure_t<c32s, false>(static_cast<const c32s*>(psi), p, partials, grid, st, none)
                           : measure_t<c64s, false>(static_cast<const c64s*>(psi), p, partials, grid, st, none);
}

// BYTE measurement entry: planes + decode tables
cudaError_t launch_measure_byte(const uint8_t* mi, const uint8_t* pi, const double* tab, const MeasureParams& p,
                                double* partials, int grid, cudaStream_t st) {
    const ByteSrc b{mi, pi, tab};
    return measure_t<c64s, true>(nullptr, p, partials, grid, st, b);
}

}  // namespace sv
