// Gate kernels for the FP64 / FP32 state vector on B200 (sm_100a).
//
// Reference semantics: /root/reference/pkg/src/svsim/kernels.py
//   apply_single      30-40   -> k_gate1_hi / k_gate1_lo (streaming, one HBM pass)
//   apply_two         43-64   -> k_gate2 (streaming)
//   apply_diagonal    67-81   -> k_diag (touches only the active subcube)
//   apply_pair_arrays 84-88   -> k_pair (two buffers; one may live on a peer GPU)
//   apply_quad_arrays 91-98   -> k_quad
//   a run of local gates      -> k_fused (tile staged in shared memory, every
//                                 gate of the run applied in order per tile)
//
// All of it is HBM-bandwidth bound (0.44 FLOP/B for a 2x2 in FP64), so the
// design rules are: 32-byte vector accesses (LDG/STG.E.ENL2.256), enough
// independent loads in flight per thread, grids sized in multiples of the
// 148 SMs, and as few HBM passes per gate as possible (fusion).
#include <algorithm>
#include <atomic>
#include <cstring>

#include "sv_common.cuh"
#include "sv_kernels.cuh"

namespace sv {

namespace {
int g_sm_count[64] = {0};
std::atomic<uint64_t> g_launches{0};
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
uint64_t launch_total() { return g_launches.load(std::memory_order_relaxed); }

int sm_count(int device) {
    if (device < 0 || device >= 64) return 148;
    if (g_sm_count[device] == 0) {
        int c = 0;
        if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || c <= 0)
            c = 148;
        g_sm_count[device] = c;
    }
    return g_sm_count[device];
}

static int current_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    return sm_count(dev);
}

static unsigned grid_for(uint64_t items, int threads, int per_sm) {
    const uint64_t want = (items + threads - 1) / threads;
    const uint64_t cap = (uint64_t)current_sms() * per_sm;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, cap));
}

struct Mat2 { cplx m[4]; };
struct Mat4 { cplx m[16]; };

static Mat2 mat2_from(const double* d) {
    Mat2 r;
    for (int i = 0; i < 4; ++i) r.m[i] = {d[2 * i], d[2 * i + 1]};
    return r;
}
static Mat4 mat4_from(const double* d) {
    Mat4 r;
    for (int i = 0; i < 16; ++i) r.m[i] = {d[2 * i], d[2 * i + 1]};
    return r;
}

// ---------------------------------------------------------------------------
// single-qubit gate, q >= log2(V): each item is V consecutive low members.
// U items are issued back to back so every thread has 2*U 32-byte loads in
// flight before the first use.
template <typename S, int U>
__global__ void __launch_bounds__(256) k_gate1_hi(S* __restrict__ psi, uint64_t n_items, int q,
                                                  Mat2 m) {
    constexpr int V = Store<S>::V;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t off = 1ull << q;
    for (uint64_t w0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w0 < n_items; w0 += U * step) {
        Vec<S> x[U], y[U];
        uint64_t i0[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t w = w0 + u * step;
            if (w < n_items) {
                i0[u] = insert0(w * V, q);
                x[u] = vload(psi + i0[u]);
                y[u] = vload(psi + i0[u] + off);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t w = w0 + u * step;
            if (w < n_items) {
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const cplx a0 = Store<S>::get(x[u].a[j]);
                    const cplx a1 = Store<S>::get(y[u].a[j]);
                    x[u].a[j] = Store<S>::put(row2(m.m[0], m.m[1], a0, a1));
                    y[u].a[j] = Store<S>::put(row2(m.m[2], m.m[3], a0, a1));
                }
                vstore(psi + i0[u], x[u]);
                vstore(psi + i0[u] + off, y[u]);
            }
        }
    }
}

// single-qubit gate, q < log2(V): the pair partners share a 32-byte vector.
template <typename S, int U, int Q>
__global__ void __launch_bounds__(256) k_gate1_lo(S* __restrict__ psi, uint64_t n_vecs, Mat2 m) {
    constexpr int V = Store<S>::V;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    constexpr int off = 1 << Q;
    for (uint64_t w0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w0 < n_vecs; w0 += U * step) {
        Vec<S> x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t w = w0 + u * step;
            if (w < n_vecs) x[u] = vload(psi + w * V);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t w = w0 + u * step;
            if (w < n_vecs) {
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    if (j & off) continue;
                    const cplx a0 = Store<S>::get(x[u].a[j]);
                    const cplx a1 = Store<S>::get(x[u].a[j + off]);
                    x[u].a[j] = Store<S>::put(row2(m.m[0], m.m[1], a0, a1));
                    x[u].a[j + off] = Store<S>::put(row2(m.m[2], m.m[3], a0, a1));
                }
                vstore(psi + w * V, x[u]);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// two-qubit gate: one thread per quadruple (scalar 16/8-byte accesses; the
// four members are 2^lo apart so consecutive threads stay coalesced for
// lo >= 1).  Basis order bit(qa) + 2*bit(qb) (kernels.py:46).
template <typename S>
__global__ void __launch_bounds__(256) k_gate2(S* __restrict__ psi, uint64_t n_quads, int lo, int hi,
                                               uint64_t ba, uint64_t bb, Mat4 m) {
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_quads; w += step) {
        const uint64_t e = insert0(insert0(w, lo), hi);
        const uint64_t idx[4] = {e, e | ba, e | bb, e | ba | bb};
        cplx a[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = Store<S>::get(psi[idx[c]]);
#pragma unroll
        for (int r = 0; r < 4; ++r) psi[idx[r]] = Store<S>::put(row4(&m.m[4 * r], a[0], a[1], a[2], a[3]));
    }
}

// ---------------------------------------------------------------------------
// diagonal: the active set {i : i & mask == mask} is a subcube; enumerate it
// directly (no full-array mask as in kernels.py:77-80).  Vector granularity
// when the mask has no bit inside a 32-byte vector.
template <typename S>
__global__ void __launch_bounds__(256) k_diag_vec(S* __restrict__ psi, uint64_t n_items,
                                                  uint64_t free_mask, uint64_t mask, cplx f) {
    constexpr int V = Store<S>::V;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_items; w += step) {
        const uint64_t i = insert_zeros(w * V, mask) | mask;
        Vec<S> x = vload(psi + i);
#pragma unroll
        for (int j = 0; j < V; ++j) x.a[j] = Store<S>::put(cmul(Store<S>::get(x.a[j]), f));
        vstore(psi + i, x);
    }
}

template <typename S>
__global__ void __launch_bounds__(256) k_diag_scalar(S* __restrict__ psi, uint64_t n_items,
                                                     uint64_t free_mask, uint64_t mask, cplx f) {
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_items; w += step) {
        const uint64_t i = insert_zeros(w, mask) | mask;
        psi[i] = Store<S>::put(cmul(Store<S>::get(psi[i]), f));
    }
}

// ---------------------------------------------------------------------------
// two / four aligned buffers (exchange rounds, engine.py:246-363)
template <typename S>
__global__ void __launch_bounds__(256) k_pair(S* __restrict__ a0, S* __restrict__ a1, uint64_t count,
                                              Mat2 m) {
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += step) {
        const cplx x = Store<S>::get(a0[i]);
        const cplx y = Store<S>::get(a1[i]);
        a0[i] = Store<S>::put(row2(m.m[0], m.m[1], x, y));
        a1[i] = Store<S>::put(row2(m.m[2], m.m[3], x, y));
    }
}

template <typename S>
__global__ void __launch_bounds__(256) k_quad(S* p0, S* p1, S* p2, S* p3, uint64_t count, Mat4 m) {
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += step) {
        const cplx a0 = Store<S>::get(p0[i]), a1 = Store<S>::get(p1[i]);
        const cplx a2 = Store<S>::get(p2[i]), a3 = Store<S>::get(p3[i]);
        p0[i] = Store<S>::put(row4(&m.m[0], a0, a1, a2, a3));
        p1[i] = Store<S>::put(row4(&m.m[4], a0, a1, a2, a3));
        p2[i] = Store<S>::put(row4(&m.m[8], a0, a1, a2, a3));
        p3[i] = Store<S>::put(row4(&m.m[12], a0, a1, a2, a3));
    }
}

// two buffers, a two-qubit gate whose qubits are an in-buffer bit `lo` and the
// buffer choice (b0 / b1): the tier executor's chunk pairs (tier.py "mid" groups).
// Basis index = bit(qa) + 2 bit(qb) (kernels.py:56-58); hi_is_b: the buffer choice
// is qb, else qa.  Same row4 arithmetic as k_gate2 / k_quad.
template <typename S>
__global__ void __launch_bounds__(256) k_pair2q(S* __restrict__ b0, S* __restrict__ b1, uint64_t n_quads, int lo,
                                                int hi_is_b, Mat4 m) {
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t bl = 1ull << lo;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_quads; t += step) {
        const uint64_t i = insert0(t, lo);
        S* p[4];
        uint64_t o[4];
        if (hi_is_b) {   // (qa = lo, qb = buffer): members (b0[i], b0[i|l], b1[i], b1[i|l])
            p[0] = b0; o[0] = i; p[1] = b0; o[1] = i | bl; p[2] = b1; o[2] = i; p[3] = b1; o[3] = i | bl;
        } else {         // (qa = buffer, qb = lo): members (b0[i], b1[i], b0[i|l], b1[i|l])
            p[0] = b0; o[0] = i; p[1] = b1; o[1] = i; p[2] = b0; o[2] = i | bl; p[3] = b1; o[3] = i | bl;
        }
        cplx a[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = Store<S>::get(p[c][o[c]]);
#pragma unroll
        for (int r = 0; r < 4; ++r) p[r][o[r]] = Store<S>::put(row4(&m.m[4 * r], a[0], a[1], a[2], a[3]));
    }
}

// ---------------------------------------------------------------------------
// Fused pass.  A tile is the 2^k amplitudes whose local index differs only
// in the tile qubits T (tq[0..k-1], with tq[i] == i for i < b so that runs of
// 2^b amplitudes are contiguous in HBM).  Each CTA stages a tile in shared
// memory as FP64, applies every op of the run in order (the reference's
// per-gate arithmetic, so results are bit-identical to one pass per gate),
// and writes the tile back: one HBM read + one HBM write for the whole run.
template <typename S, int K>
__global__ void __launch_bounds__(256) k_fused(S* __restrict__ psi, const __grid_constant__ FusedParams p) {
    constexpr int NT = 256;
    constexpr int TILE = 1 << K;
    constexpr int V = Store<S>::V;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* s = reinterpret_cast<cplx*>(smem_raw);
    uint64_t* off_hi = reinterpret_cast<uint64_t*>(smem_raw + sizeof(cplx) * TILE);

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

    for (uint64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        const uint64_t base = insert_zeros(tile, p.tile_mask);
        // ---- load (32-byte vectors when the tile is large: b >= 5 >= log2 V) ----
        if constexpr (TILE >= NT * V) {
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
        // ---- ops, in circuit order ----
        int prev_kind = 0;
        for (int o = 0; o < p.n_ops; ++o) {
            const int kind = p.kind[o];
            const double* md = p.mdata + p.moff[o];
            if (kind == SV_OP_1Q) {
                if (prev_kind != 0) __syncthreads();
                const int pos = p.pa[o];
                const cplx m0 = {md[0], md[1]}, m1 = {md[2], md[3]}, m2 = {md[4], md[5]}, m3 = {md[6], md[7]};
                for (int w = threadIdx.x; w < TILE / 2; w += NT) {
                    const int e0 = (int)insert0((uint64_t)w, pos);
                    const int e1 = e0 | (1 << pos);
                    const cplx a0 = s[e0], a1 = s[e1];
                    s[e0] = Store<S>::round(row2(m0, m1, a0, a1));
                    s[e1] = Store<S>::round(row2(m2, m3, a0, a1));
                }
            } else if (kind == SV_OP_2Q) {
                if (prev_kind != 0) __syncthreads();
                const int pa = p.pa[o], pb = p.pb[o];
                const int lo = pa < pb ? pa : pb, hi = pa < pb ? pb : pa;
                cplx m[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) m[i] = {md[2 * i], md[2 * i + 1]};
                for (int w = threadIdx.x; w < TILE / 4; w += NT) {
                    const int e = (int)insert0(insert0((uint64_t)w, lo), hi);
                    const int idx[4] = {e, e | (1 << pa), e | (1 << pb), e | (1 << pa) | (1 << pb)};
                    const cplx a0 = s[idx[0]], a1 = s[idx[1]], a2 = s[idx[2]], a3 = s[idx[3]];
#pragma unroll
                    for (int r = 0; r < 4; ++r) s[idx[r]] = Store<S>::round(row4(&m[4 * r], a0, a1, a2, a3));
                }
            } else {  // SV_OP_DIAG: elementwise; same element->thread map as other diags
                if (prev_kind != 0 && prev_kind != SV_OP_DIAG) __syncthreads();
                if ((base & p.dmask_o[o]) == p.dmask_o[o]) {
                    const uint32_t mt = p.dmask_t[o];
                    const cplx f = {md[0], md[1]};
                    for (int e = threadIdx.x; e < TILE; e += NT)
                        if (((uint32_t)e & mt) == mt) s[e] = Store<S>::round(cmul(s[e], f));
                }
            }
            prev_kind = kind;
        }
        __syncthreads();
        // ---- store ----
        if constexpr (TILE >= NT * V) {
            constexpr int PER = TILE / (NT * V);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const uint32_t e = (threadIdx.x + j * NT) * V;
                Vec<S> vv;
#pragma unroll
                for (int v = 0; v < V; ++v) vv.a[v] = Store<S>::put(s[e + v]);
                vstore(psi + base + off_hi[e >> b] + (e & lowmask), vv);
            }
        } else {
            for (int e = threadIdx.x; e < TILE; e += NT)
                psi[base + off_hi[e >> b] + (e & lowmask)] = Store<S>::put(s[e]);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// launchers
template <typename S>
static cudaError_t gate1_t(S* psi, uint64_t n, int q, const Mat2& m, cudaStream_t st) {
    constexpr int V = Store<S>::V;
    constexpr int LOGV = V == 2 ? 1 : 2;
    constexpr int U = 2;
    if (q >= LOGV) {
        const uint64_t items = n / 2 / V;
        k_gate1_hi<S, U><<<grid_for(items, 256 * U, 8), 256, 0, st>>>(psi, items, q, m);
    } else {
        const uint64_t vecs = n / V;
        if (q == 0)
            k_gate1_lo<S, 4, 0><<<grid_for(vecs, 256 * 4, 8), 256, 0, st>>>(psi, vecs, m);
        else
            k_gate1_lo<S, 4, 1><<<grid_for(vecs, 256 * 4, 8), 256, 0, st>>>(psi, vecs, m);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gate1(void* psi, uint64_t n, int mode, int q, const double* m8, cudaStream_t st) {
    const Mat2 m = mat2_from(m8);
    return mode == SV_FP32 ? gate1_t(static_cast<c32s*>(psi), n, q, m, st)
                           : gate1_t(static_cast<c64s*>(psi), n, q, m, st);
}

cudaError_t launch_gate2(void* psi, uint64_t n, int mode, int qa, int qb, const double* m32,
                         cudaStream_t st) {
    const Mat4 m = mat4_from(m32);
    const int lo = std::min(qa, qb), hi = std::max(qa, qb);
    const uint64_t quads = n / 4;
    const unsigned g = grid_for(quads, 256, 8);
    if (mode == SV_FP32)
        k_gate2<c32s><<<g, 256, 0, st>>>(static_cast<c32s*>(psi), quads, lo, hi, 1ull << qa, 1ull << qb, m);
    else
        k_gate2<c64s><<<g, 256, 0, st>>>(static_cast<c64s*>(psi), quads, lo, hi, 1ull << qa, 1ull << qb, m);
    count_launch();
    return cudaGetLastError();
}

template <typename S>
static cudaError_t diag_t(S* psi, uint64_t n, uint64_t mask, cplx f, cudaStream_t st) {
    constexpr int V = Store<S>::V;
    const uint64_t all = n - 1;                     // n is a power of two here
    const uint64_t free_mask = all & ~mask;
    const uint64_t active = n >> __builtin_popcountll(mask);
    if ((mask & (uint64_t)(V - 1)) == 0) {
        const uint64_t items = active / V;
        k_diag_vec<S><<<grid_for(items, 256, 8), 256, 0, st>>>(psi, items, free_mask, mask, f);
    } else {
        k_diag_scalar<S><<<grid_for(active, 256, 8), 256, 0, st>>>(psi, active, free_mask, mask, f);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_diag(void* psi, uint64_t n, int mode, uint64_t mask, const double* f2,
                        cudaStream_t st) {
    const cplx f = {f2[0], f2[1]};
    return mode == SV_FP32 ? diag_t(static_cast<c32s*>(psi), n, mask, f, st)
                           : diag_t(static_cast<c64s*>(psi), n, mask, f, st);
}

cudaError_t launch_pair(void* a0, void* a1, uint64_t count, int mode, const double* m8,
                        cudaStream_t st) {
    const Mat2 m = mat2_from(m8);
    const unsigned g = grid_for(count, 256, 8);
    if (mode == SV_FP32)
        k_pair<c32s><<<g, 256, 0, st>>>(static_cast<c32s*>(a0), static_cast<c32s*>(a1), count, m);
    else
        k_pair<c64s><<<g, 256, 0, st>>>(static_cast<c64s*>(a0), static_cast<c64s*>(a1), count, m);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_quad(void* const* parts, uint64_t count, int mode, const double* m32,
                        cudaStream_t st) {
    const Mat4 m = mat4_from(m32);
    const unsigned g = grid_for(count, 256, 8);
    if (mode == SV_FP32)
        k_quad<c32s><<<g, 256, 0, st>>>(static_cast<c32s*>(parts[0]), static_cast<c32s*>(parts[1]),
                                        static_cast<c32s*>(parts[2]), static_cast<c32s*>(parts[3]), count, m);
    else
        k_quad<c64s><<<g, 256, 0, st>>>(static_cast<c64s*>(parts[0]), static_cast<c64s*>(parts[1]),
                                        static_cast<c64s*>(parts[2]), static_cast<c64s*>(parts[3]), count, m);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_pair2q(void* b0, void* b1, uint64_t count, int mode, int lo, int hi_is_b, const double* m32,
                          cudaStream_t st) {
    const Mat4 m = mat4_from(m32);
    const uint64_t quads = count / 2;
    const unsigned g = grid_for(quads, 256, 8);
    if (mode == SV_FP32)
        k_pair2q<c32s><<<g, 256, 0, st>>>(static_cast<c32s*>(b0), static_cast<c32s*>(b1), quads, lo, hi_is_b, m);
    else
        k_pair2q<c64s><<<g, 256, 0, st>>>(static_cast<c64s*>(b0), static_cast<c64s*>(b1), quads, lo, hi_is_b, m);
    count_launch();
    return cudaGetLastError();
}

template <typename S, int K>
static cudaError_t fused_k(S* psi, const FusedParams& p, cudaStream_t st) {
    const size_t smem = sizeof(cplx) * (1u << K) + sizeof(uint64_t) * (1u << (K - p.b));
    static bool configured[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k_fused<S, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(sizeof(cplx) * (1u << K) + sizeof(uint64_t) * (1u << K)));
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused<S, K>, 256, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t cap = (uint64_t)current_sms() * per_sm;
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(p.n_tiles, cap));
    k_fused<S, K><<<g, 256, smem, st>>>(psi, p);
    count_launch();
    return cudaGetLastError();
}

template <typename S>
static cudaError_t fused_t(S* psi, const FusedParams& p, cudaStream_t st) {
    switch (p.k) {
        case 1: return fused_k<S, 1>(psi, p, st);
        case 2: return fused_k<S, 2>(psi, p, st);
        case 3: return fused_k<S, 3>(psi, p, st);
        case 4: return fused_k<S, 4>(psi, p, st);
        case 5: return fused_k<S, 5>(psi, p, st);
        case 6: return fused_k<S, 6>(psi, p, st);
        case 7: return fused_k<S, 7>(psi, p, st);
        case 8: return fused_k<S, 8>(psi, p, st);
        case 9: return fused_k<S, 9>(psi, p, st);
        case 10: return fused_k<S, 10>(psi, p, st);
        case 11: return fused_k<S, 11>(psi, p, st);
        case 12: return fused_k<S, 12>(psi, p, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_fused(void* psi, int mode, const FusedParams& p, cudaStream_t st) {
    return mode == SV_FP32 ? fused_t(static_cast<c32s*>(psi), p, st)
                           : fused_t(static_cast<c64s*>(psi), p, st);
}

}  // namespace sv
