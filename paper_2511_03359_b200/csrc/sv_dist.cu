// Cross-GPU kernels over NVLink 5 / NVSwitch peer memory (sm_100a).
//
// Rank r owns the 2^n' amplitudes whose top index bits equal r
// (svsim/layout.py:26-47).  Peer buffers are mapped with CUDA IPC, so one
// kernel reads and writes the partner GPU's HBM directly (LDG/STG on peer
// addresses; the transfer overlaps the arithmetic element by element).
//
//   k_swap_peer  global<->local qubit swap (the remap planner's move):
//                rank with global bit c exchanges its amplitudes whose local
//                bit l is 1-c with the partner's amplitudes whose bit l is c.
//                Each rank of the pair moves one half of them (reads the peer's
//                element, writes its own into the peer), so every amplitude
//                crosses NVLink exactly once: L/2 elements per direction per
//                rank pair, the minimum for making the qubit local.
//   k_pair_dot   sum conj(a0) * a1 across a rank pair (measure.py:83-101:
//                cross term of a global qubit), deterministic block partials.
// The exchange-fused 2x2 update of the reference choreography
// (engine.py:246-269) is svk_pair_update with one peer pointer.
#include <algorithm>

#include "sv_common.cuh"
#include "sv_kernels.cuh"

namespace sv {

namespace {
__device__ __forceinline__ uint64_t insert_bit(uint64_t t, int l, uint64_t b) {
    const uint64_t low = t & ((1ull << l) - 1ull);
    return ((t >> l) << (l + 1)) | (b << l) | low;
}
}  // namespace

template <typename S, int U>
__global__ void __launch_bounds__(256) k_swap_peer_vec(S* __restrict__ own, S* __restrict__ peer, uint64_t t0,
                                                       uint64_t n_vec, int l, int c) {
    constexpr int V = Store<S>::V;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w0 < n_vec; w0 += U * step) {
        Vec<S> a[U], b[U];
        uint64_t x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t w = w0 + u * step;
            if (w < n_vec) {
                const uint64_t t = t0 + w * V;
                x[u] = insert_bit(t, l, (uint64_t)(1 - c));
                y[u] = insert_bit(t, l, (uint64_t)c);
                a[u] = vload(own + x[u]);
                b[u] = vload(peer + y[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t w = w0 + u * step;
            if (w < n_vec) {
                vstore(own + x[u], b[u]);
                vstore(peer + y[u], a[u]);
            }
        }
    }
}

template <typename S>
__global__ void __launch_bounds__(256) k_swap_peer_scalar(S* own, S* peer, uint64_t t0, uint64_t n, int l, int c) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n; w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = t0 + w;
        const uint64_t x = insert_bit(t, l, (uint64_t)(1 - c)), y = insert_bit(t, l, (uint64_t)c);
        const S a = own[x];
        own[x] = peer[y];
        peer[y] = a;
    }
}

// Batched swap of k global qubits with k local victims (one member pair of the
// 2^k-rank group): this rank's amplitudes whose victim bits read `own_pat` trade
// places with the member's amplitudes whose victim bits read `peer_pat` (same
// remaining bits).  t runs over the remaining-bit space [t0, t0 + n).
template <typename S>
__global__ void __launch_bounds__(256) k_swap_group(S* __restrict__ own, S* __restrict__ peer, uint64_t t0,
                                                    uint64_t n, uint64_t vmask, uint64_t own_pat,
                                                    uint64_t peer_pat, uint64_t cmask, uint64_t cpat) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n; w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t base = insert_zeros(t0 + w, vmask | cmask) | cpat;
        const uint64_t x = base | own_pat, y = base | peer_pat;
        const S a = own[x];
        own[x] = peer[y];
        peer[y] = a;
    }
}

template <typename S, int U>
__global__ void __launch_bounds__(256) k_swap_group_vec(S* __restrict__ own, S* __restrict__ peer, uint64_t t0,
                                                        uint64_t n_vec, uint64_t vmask, uint64_t own_pat,
                                                        uint64_t peer_pat, uint64_t cmask, uint64_t cpat) {
    constexpr int V = Store<S>::V;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w0 < n_vec; w0 += U * step) {
        Vec<S> a[U], b[U];
        uint64_t x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t w = w0 + u * step;
            if (w < n_vec) {
                const uint64_t base = insert_zeros(t0 + w * V, vmask | cmask) | cpat;
                x[u] = base | own_pat;
                y[u] = base | peer_pat;
                a[u] = vload(own + x[u]);
                b[u] = vload(peer + y[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t w = w0 + u * step;
            if (w < n_vec) {
                vstore(own + x[u], b[u]);
                vstore(peer + y[u], a[u]);
            }
        }
    }
}

int g_swap_blocks = 0;   // > 0: grid cap of the group-swap kernel (overlapped swaps leave SMs to the pass)

template <typename S>
static cudaError_t swap_group_t(S* own, S* peer, uint64_t t0, uint64_t n, uint64_t vmask, uint64_t op, uint64_t pp,
                                uint64_t cmask, uint64_t cpat, cudaStream_t st) {
    constexpr int V = Store<S>::V;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t cap = g_swap_blocks > 0 ? (uint64_t)g_swap_blocks : (uint64_t)sm_count(dev) * 8;
    const bool vec = ((vmask | cmask) & (uint64_t)(V - 1)) == 0 && (t0 % V) == 0 && (n % V) == 0;
    if (vec) {
        const uint64_t nv = n / V;
        const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nv + 1023) / 1024, cap));
        k_swap_group_vec<S, 4><<<g, 256, 0, st>>>(own, peer, t0, nv, vmask, op, pp, cmask, cpat);
    } else {
        const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, cap));
        k_swap_group<S><<<g, 256, 0, st>>>(own, peer, t0, n, vmask, op, pp, cmask, cpat);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_swap_group(void* own, void* peer, uint64_t t0, uint64_t n, int mode, uint64_t vmask,
                              uint64_t own_pat, uint64_t peer_pat, uint64_t cmask, uint64_t cpat, cudaStream_t st) {
    return mode == SV_FP32 ? swap_group_t(static_cast<c32s*>(own), static_cast<c32s*>(peer), t0, n, vmask, own_pat,
                                          peer_pat, cmask, cpat, st)
                           : swap_group_t(static_cast<c64s*>(own), static_cast<c64s*>(peer), t0, n, vmask, own_pat,
                                          peer_pat, cmask, cpat, st);
}

// 4 independent 32-byte loads of each side per iteration: the remote side is an NVLink read,
// so enough requests must be in flight per thread to cover its latency
// deterministic block partial of (re, im): warp shuffles, then warp 0's thread 0 in order
__device__ __forceinline__ void block_partials(double re, double im, double* partials) {
    __shared__ double sr[8], si[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_down_sync(0xffffffffu, re, o);
        im += __shfl_down_sync(0xffffffffu, im, o);
    }
    if ((threadIdx.x & 31) == 0) { sr[threadIdx.x >> 5] = re; si[threadIdx.x >> 5] = im; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += sr[w]; b += si[w]; }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
    }
}

template <typename S>
__global__ void __launch_bounds__(256) k_pair_dot(const S* __restrict__ a0, const S* __restrict__ a1, uint64_t n,
                                                  double* __restrict__ partials) {
    constexpr int V = Store<S>::V, U = 4;
    double re = 0.0, im = 0.0;
    const bool aligned = ((reinterpret_cast<uintptr_t>(a0) | reinterpret_cast<uintptr_t>(a1)) & 31) == 0;
    const uint64_t nv = aligned ? n / V : 0, step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w0 < nv; w0 += U * step) {
        Vec<S> x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t w = w0 + u * step;
            if (w < nv) {
                x[u] = vload(a0 + w * V);
                y[u] = vload(a1 + w * V);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (w0 + u * step >= nv) continue;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const cplx a = Store<S>::get(x[u].a[v]), b = Store<S>::get(y[u].a[v]);
                re += a.re * b.re + a.im * b.im;
                im += a.re * b.im - a.im * b.re;
            }
        }
    }
    for (uint64_t i = nv * V + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += step) {   // tail
        const cplx a = Store<S>::get(a0[i]), b = Store<S>::get(a1[i]);
        re += a.re * b.re + a.im * b.im;
        im += a.re * b.im - a.im * b.re;
    }
    block_partials(re, im, partials);
}

// the same over the amplitudes whose bits under cmask read cpat (a tracked support's fixed
// bits): element t0 + w of the rest indices is insert_zeros(t0 + w, cmask) | cpat
template <typename S>
__global__ void __launch_bounds__(256) k_pair_dot_chunk(const S* __restrict__ a0, const S* __restrict__ a1,
                                                        uint64_t t0, uint64_t n, uint64_t cmask, uint64_t cpat,
                                                        double* __restrict__ partials) {
    double re = 0.0, im = 0.0;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n; w += step) {
        const uint64_t i = insert_zeros(t0 + w, cmask) | cpat;
        const cplx a = Store<S>::get(a0[i]), b = Store<S>::get(a1[i]);
        re += a.re * b.re + a.im * b.im;
        im += a.re * b.im - a.im * b.re;
    }
    block_partials(re, im, partials);
}

template <typename S>
static cudaError_t swap_t(S* own, S* peer, uint64_t n_local_elems, int l, int c, cudaStream_t st) {
    constexpr int V = Store<S>::V;
    constexpr int LOGV = V == 2 ? 1 : 2;
    const uint64_t quarter = n_local_elems / 4;     // this rank's share of the L/2 rest indices
    const uint64_t t0 = (uint64_t)c * quarter;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t cap = (uint64_t)sm_count(dev) * 8;
    if (l >= LOGV && quarter % V == 0) {
        const uint64_t n_vec = quarter / V;
        const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_vec + 1023) / 1024, cap));
        k_swap_peer_vec<S, 4><<<g, 256, 0, st>>>(own, peer, t0, n_vec, l, c);
    } else {
        const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((quarter + 255) / 256, cap));
        k_swap_peer_scalar<S><<<g, 256, 0, st>>>(own, peer, t0, quarter, l, c);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_swap_peer(void* own, void* peer, uint64_t n_local_elems, int mode, int l, int c, cudaStream_t st) {
    return mode == SV_FP32 ? swap_t(static_cast<c32s*>(own), static_cast<c32s*>(peer), n_local_elems, l, c, st)
                           : swap_t(static_cast<c64s*>(own), static_cast<c64s*>(peer), n_local_elems, l, c, st);
}

cudaError_t launch_pair_dot(const void* a0, const void* a1, uint64_t n, int mode, double* partials, int grid,
                            cudaStream_t st) {
    if (mode == SV_FP32)
        k_pair_dot<c32s><<<grid, 256, 0, st>>>(static_cast<const c32s*>(a0), static_cast<const c32s*>(a1), n, partials);
    else
        k_pair_dot<c64s><<<grid, 256, 0, st>>>(static_cast<const c64s*>(a0), static_cast<const c64s*>(a1), n, partials);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_pair_dot_chunk(const void* a0, const void* a1, uint64_t t0, uint64_t n, uint64_t cmask,
                                  uint64_t cpat, int mode, double* partials, int grid, cudaStream_t st) {
    if (mode == SV_FP32)
        k_pair_dot_chunk<c32s><<<grid, 256, 0, st>>>(static_cast<const c32s*>(a0), static_cast<const c32s*>(a1), t0, n,
                                                     cmask, cpat, partials);
    else
        k_pair_dot_chunk<c64s><<<grid, 256, 0, st>>>(static_cast<const c64s*>(a0), static_cast<const c64s*>(a1), t0, n,
                                                     cmask, cpat, partials);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sv
