// extern "C" boundary of libsvb200.so (declared in include/svb200.h).
//
// Validation and error texts follow the reference operators they replace
// (/root/reference/pkg/src/svsim/kernels.py:23-24, 34-35, 49-52) so the
// Python layer can re-raise the same exception types with the same messages.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <algorithm>
#include <atomic>
#include <mutex>

#include "sv_common.cuh"
#include "sv_kernels.cuh"

using namespace sv;

namespace sv { uint64_t launch_total(); }

namespace {

thread_local std::string g_err;

std::atomic<uint64_t> g_h2d{0}, g_d2h{0};
inline void count_h2d(uint64_t b) { g_h2d.fetch_add(b, std::memory_order_relaxed); }
inline void count_d2h(uint64_t b) { g_d2h.fetch_add(b, std::memory_order_relaxed); }

struct TimedPass { cudaEvent_t a, b; double bytes; };
bool g_timing = false;
int g_fused_v2 = 9;      // default: auto (config 6 = 2^11 tiles, 3 CTAs/SM; config 8 = 2^12 single-buffer tiles when they save a pass)
int g_seg_limit = 0;        // > 0: passes needing more segments fall back to v1
std::mutex g_timing_mu;
std::vector<TimedPass> g_timed;
std::atomic<unsigned long long> g_support_tiles_skipped{0};   // tiles support tracking left out

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();  // clear sticky-free errors
    return fail(e == cudaErrorMemoryAllocation ? SV_ENOMEM : SV_ECUDA, "%s: %s (%s)", what,
                cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CUDA_TRY(expr, what)                               \
    do {                                                   \
        cudaError_t _e = (expr);                           \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

inline bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }
inline int log2u(uint64_t x) { return 63 - __builtin_clzll(x); }
inline size_t elem_bytes(int mode) { return mode == SV_FP32 ? 8 : 16; }
inline bool valid_fp_mode(int mode) { return mode == SV_FP64 || mode == SV_FP32; }

// ---- scalar fallbacks for tiny / unaligned / non-power-of-two buffers -----
template <typename S>
__global__ void k_gate1_scalar(S* psi, uint64_t n_pairs, int q, cplx m0, cplx m1, cplx m2, cplx m3) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_pairs;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i0 = insert0(t, q), i1 = i0 | (1ull << q);
        const cplx a0 = Store<S>::get(psi[i0]), a1 = Store<S>::get(psi[i1]);
        psi[i0] = Store<S>::put(row2(m0, m1, a0, a1));
        psi[i1] = Store<S>::put(row2(m2, m3, a0, a1));
    }
}

template <typename S>
__global__ void k_diag_all(S* psi, uint64_t n, uint64_t mask, cplx f) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if ((i & mask) == mask) psi[i] = Store<S>::put(cmul(Store<S>::get(psi[i]), f));
}

unsigned small_grid(uint64_t items) {
    uint64_t g = (items + 255) / 256;
    if (g < 1) g = 1;
    if (g > 4096) g = 4096;
    return (unsigned)g;
}

int check_1q(uint64_t n, int q) {
    if (q < 0 || q >= 63 || (1ull << q) >= n)
        return fail(SV_EINDEX, "qubit %d outside local array of %llu amplitudes", q,
                    (unsigned long long)n);
    if (n % (2ull << q))
        return fail(SV_EVALUE, "array of %llu amplitudes does not split into pairs of stride %llu",
                    (unsigned long long)n, (unsigned long long)(1ull << q));
    return SV_OK;
}

int check_2q(uint64_t n, int qa, int qb) {
    if (qa == qb) return fail(SV_EVALUE, "two-qubit gate requires distinct qubits");
    if (qa < 0 || qb < 0 || qa >= 63 || qb >= 63 || (1ull << qa) >= n || (1ull << qb) >= n)
        return fail(SV_EINDEX, "qubits (%d, %d) outside local array of %llu amplitudes", qa, qb,
                    (unsigned long long)n);
    const int hi = qa > qb ? qa : qb;
    if (n % (2ull << hi))
        return fail(SV_EVALUE, "array of %llu amplitudes does not split into quadruples",
                    (unsigned long long)n);
    return SV_OK;
}

// ---------------------------------------------------------------------------
// fused-pass planning: greedy grouping of consecutive ops whose non-diagonal
// qubits fit one tile of 2^k amplitudes; the tile always contains the lowest
// qubits so HBM runs stay contiguous (>= 2^5 amplitudes = 512 B in FP64).
struct PassPlan {
    std::vector<int> ops;       // indices into the op list
    uint64_t qmask = 0;         // qubits that must be in the tile
    int mdata = 0;
    int ndiag = 0;              // diagonal ops among them
};

// low qubits every fused-pass tile keeps (contiguous HBM runs of 2^b amplitudes):
// SVB200_LOW_BITS, default 4 (256-byte runs in FP64, full 32-byte sectors).  One more free
// tile qubit per pass: the C2 layers at N=33 plan 3.35 instead of 3.55 passes per layer and
// run 1553 instead of 1639 ms per 9 layers (per-pass efficiency 0.823 vs 0.832).
int low_bits() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("SVB200_LOW_BITS");
        const int x = e ? std::atoi(e) : 4;
        v = (x >= 2 && x <= 5) ? x : 4;
    }
    return v;
}

int op_mdata(int kind) { return kind == SV_OP_2Q ? 32 : (kind == SV_OP_1Q ? 8 : 2); }

int popcount64(uint64_t x) { return __builtin_popcountll(x); }

uint64_t tile_mask_for(uint64_t qmask, int n, int k) {
    // required qubits plus the lowest ones, k in total
    uint64_t t = qmask;
    for (int q = 0; q < n && popcount64(t) < k; ++q) t |= 1ull << q;
    return t;
}

int build_params(const sv_op* ops, const PassPlan& pp, int n, int k, FusedParams& P) {
    std::memset(&P, 0, sizeof(P));
    const uint64_t tmask = tile_mask_for(pp.qmask, n, k);
    P.n = n;
    P.k = k;
    P.tile_mask = tmask;
    P.out_mask = ((n == 64) ? ~0ull : ((1ull << n) - 1ull)) & ~tmask;
    P.n_tiles = 1ull << (n - k);
    int pos_of[64];
    int j = 0;
    for (int q = 0; q < n; ++q) {
        pos_of[q] = -1;
        if ((tmask >> q) & 1) {
            pos_of[q] = j;
            P.tq[j++] = (int8_t)q;
        }
    }
    int b = 0;
    while (b < k && P.tq[b] == b) ++b;
    P.b = b;
    int md = 0;
    P.n_ops = (int)pp.ops.size();
    for (int i = 0; i < P.n_ops; ++i) {
        const sv_op& o = ops[pp.ops[i]];
        P.kind[i] = (uint8_t)o.kind;
        P.moff[i] = (uint16_t)md;
        const int cnt = op_mdata(o.kind);
        for (int c = 0; c < cnt; ++c) P.mdata[md + c] = o.m[c];
        md += cnt;
        if (o.kind == SV_OP_1Q) {
            P.pa[i] = (uint8_t)pos_of[o.qa];
        } else if (o.kind == SV_OP_2Q) {
            P.pa[i] = (uint8_t)pos_of[o.qa];
            P.pb[i] = (uint8_t)pos_of[o.qb];
        } else {
            uint32_t mt = 0;
            for (int q = 0; q < n; ++q)
                if (((o.diag_mask >> q) & 1) && pos_of[q] >= 0) mt |= 1u << pos_of[q];
            P.dmask_t[i] = mt;
            P.dmask_o[i] = o.diag_mask & ~tmask;
        }
    }
    return SV_OK;
}

// ---- v2 planner: 12-bit register-resident tiles (sv_fused2.cu) -----------------
// unit code of a matrix entry: 0 -> 1, 1 -> i, 2 -> -1, 3 -> -i, -1 -> not a unit
int unit_code(double re, double im) {
    if (im == 0.0 && re == 1.0) return 0;
    if (re == 0.0 && im == 1.0) return 1;
    if (im == 0.0 && re == -1.0) return 2;
    if (re == 0.0 && im == -1.0) return 3;
    return -1;
}

// classify a dim x dim row-major complex matrix: 0 generic, 1 real, 2 monomial (units)
int classify(const double* m, int dim, uint32_t* mono) {
    bool real = true;
    for (int i = 0; i < dim * dim; ++i) real = real && m[2 * i + 1] == 0.0;
    uint32_t code = 0;
    bool monomial = true;
    for (int r = 0; r < dim && monomial; ++r) {
        int src = -1, u = -1, nz = 0;
        for (int c = 0; c < dim; ++c) {
            const double re = m[2 * (r * dim + c)], im = m[2 * (r * dim + c) + 1];
            if (re != 0.0 || im != 0.0) {
                ++nz;
                src = c;
                u = unit_code(re, im);
            }
        }
        if (nz != 1 || u < 0) monomial = false;
        else code |= (uint32_t)(src | (u << 2)) << (4 * r);
    }
    if (monomial) {
        *mono = code;
        return 2;
    }
    return real ? 1 : 0;
}

// ---- support tracking (sv_set_support_tracking) ---------------------------------------------
// Amplitudes outside {i : (i & ~free) == val} are exactly zero: a state starts as a basis state
// (free = 0), a non-monomial gate frees its qubits, a monomial on fixed qubits moves val, a
// diagonal gate changes nothing.  A fused pass then runs only the tiles whose fixed
// out-of-tile bits equal val (the chunked-launch path): the others hold zeros and stay zeros
// (+-0: identical under np.array_equal, the parity tests' comparison).
struct Support {
    bool on = false;
    uint64_t free = 0, val = 0;
    // dirty: HBM outside the support was never written (a lazy basis state whose first pass
    // generated only the support's tiles); passes then load it as zeros (Fused2Params::pfix),
    // every other reader first zero-fills it (clean_support)
    bool dirty = false;
};
__global__ void k_zero_outside(c64s* __restrict__ psi, uint64_t n, uint64_t fixed, uint64_t val) {
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 4; i < n; i += step) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (i + k < n && ((i + k) & fixed) != val) psi[i + k] = c64s{0.0, 0.0};
    }
}
// the support's amplitudes {deposit(t, free) | val} to / from a compact buffer
__global__ void k_support_copy(c64s* __restrict__ psi, c64s* __restrict__ buf, uint64_t m, uint64_t freem,
                               uint64_t val, int to_buf) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < m; t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t i = val, f = freem, tt = t;
        while (f) {
            const uint64_t b = f & (~f + 1ull);
            if (tt & 1ull) i |= b;
            tt >>= 1;
            f &= f - 1ull;
        }
        if (to_buf) buf[t] = psi[i];
        else psi[i] = buf[t];
    }
}
// zeros into the never-written part of a dirty FP64 state.  A small support (<= 2^24
// amplitudes): saved, the whole state memset (the copy engine's write rate), restored;
// otherwise a zero-fill kernel over the complement
static int clean_support(void* psi, uint64_t n_elems, Support& s, cudaStream_t st) {
    if (!s.on || !s.dirty) return SV_OK;
    const uint64_t all = n_elems - 1, freem = s.free & all, fixed = ~s.free & all, val = s.val & fixed;
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned grid = (unsigned)sm_count(dev) * 8;
    const int nf = __builtin_popcountll(freem);
    cudaError_t e = cudaSuccess;
    if (nf <= 24) {
        const uint64_t m = 1ull << nf;
        c64s* buf = nullptr;
        e = cudaMallocAsync(reinterpret_cast<void**>(&buf), m * sizeof(c64s), st);
        if (e == cudaSuccess) {
            const unsigned g = (unsigned)std::min<uint64_t>(grid, (m + 255) / 256);
            k_support_copy<<<g, 256, 0, st>>>(static_cast<c64s*>(psi), buf, m, freem, val, 1);
            e = cudaMemsetAsync(psi, 0, n_elems * sizeof(c64s), st);
            if (e == cudaSuccess) k_support_copy<<<g, 256, 0, st>>>(static_cast<c64s*>(psi), buf, m, freem, val, 0);
            cudaFreeAsync(buf, st);
            count_launch();
            count_launch();
        }
    } else {
        k_zero_outside<<<grid, 256, 0, st>>>(static_cast<c64s*>(psi), n_elems, fixed, val);
        count_launch();
    }
    s.dirty = false;
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? SV_OK : cuda_fail(e, "zero-fill outside the support");
}
static thread_local Support* g_support = nullptr;   // the handle's, for one fused_impl call
struct SupportScope {
    Support* prev;
    explicit SupportScope(Support* s) : prev(g_support) { g_support = (s && s->on) ? s : nullptr; }
    ~SupportScope() { g_support = prev; }
};
static bool czero(const double* m, int idx) { return m[2 * idx] == 0.0 && m[2 * idx + 1] == 0.0; }
static void support_apply(Support& s, const sv_op& o) {
    if (!s.on || (o.kind != SV_OP_1Q && o.kind != SV_OP_2Q)) return;   // diagonal: support unchanged
    if (o.kind == SV_OP_1Q) {
        const uint64_t b = 1ull << o.qa;
        if (s.free & b) return;
        const int c = (s.val & b) ? 1 : 0;                 // the column the fixed bit selects
        const bool r0 = !czero(o.m, 0 * 2 + c), r1 = !czero(o.m, 1 * 2 + c);
        if (r0 && r1) s.free |= b;
        else if (r1) s.val |= b;
        else if (r0) s.val &= ~b;
        else s.free |= b;                                  // a zero column: conservative
        return;
    }
    const uint64_t ba = 1ull << o.qa, bb = 1ull << o.qb;
    if ((s.free & ba) || (s.free & bb)) { s.free |= ba | bb; return; }
    const int c = ((s.val & ba) ? 1 : 0) + ((s.val & bb) ? 2 : 0);   // basis index bit(qa) + 2 bit(qb)
    int rows = 0, r = -1;
    for (int row = 0; row < 4; ++row)
        if (!czero(o.m, row * 4 + c)) { ++rows; r = row; }
    if (rows != 1) { s.free |= ba | bb; return; }
    s.val = (s.val & ~(ba | bb)) | ((r & 1) ? ba : 0) | ((r & 2) ? bb : 0);
}

// combined diagonal runs (sv_set_diag_combine): set by the C entry points for the duration of
// one fused_impl call; diagonal ops then cost one conditional multiply into a per-mask factor,
// so mostly-diagonal passes are no longer closed at kDiagPassOps
static thread_local int g_combine_diag = 0;
struct CombineScope {
    int prev;
    explicit CombineScope(int on) : prev(g_combine_diag) { g_combine_diag = on; }
    ~CombineScope() { g_combine_diag = prev; }
};
int build_params2(const sv_op* ops, const PassPlan& pp, int n, int cfg, Fused2Params& P) {
    std::memset(&P, 0, sizeof(P));
    P.combine_diag = g_combine_diag;
    P.vinit = -2;                       // read the tiles (see fused_impl for lazy basis states)
    const int K = (cfg == 2 || cfg == 4 || cfg == 6) ? 11 : ((cfg == 5 || cfg == 7) ? 10 : (cfg == 10 ? 13 : 12));
    const int RB = (cfg == 1 || cfg == 6 || cfg == 7 || cfg == 8 || cfg == 10 || cfg == 11) ? 4 : 3;
    const int NTH = 1 << (K - RB);
    P.cfg = cfg;
    P.kbits = K;
    P.rbits = RB;
    // Tile = the pass's non-diagonal qubits + the fixed low qubits (HBM runs) + fillers.  The
    // fillers avoid qubits the pass's diagonal ops test: a diagonal mask bit outside the tile
    // is a tile-uniform condition (the whole tile skips the op), inside the tile it would be
    // a thread position, where a lane condition still issues the warp's multiplies
    // (SVB200_TILE_FILL=0: lowest qubits first, as before).
    static const int fill_env = [] {
        const char* e = std::getenv("SVB200_TILE_FILL");
        return e ? std::atoi(e) : 1;
    }();
    uint64_t diag_used = 0;
    for (int i : pp.ops)
        if (ops[i].kind != SV_OP_1Q && ops[i].kind != SV_OP_2Q) diag_used |= ops[i].diag_mask;
    uint64_t tmask = pp.qmask;
    for (int q = 0; q < n && q < low_bits() && popcount64(tmask) < K; ++q) tmask |= 1ull << q;
    for (int pass = fill_env ? 0 : 1; pass < 2; ++pass)
        for (int q = 0; q < n && popcount64(tmask) < K; ++q)
            if (pass == 1 || !((diag_used >> q) & 1)) tmask |= 1ull << q;
    P.n = n;
    P.tile_mask = tmask;
    P.n_tiles = 1ull << (n - K);
    int pos_of[64];
    int j = 0;
    for (int q = 0; q < n; ++q) {
        pos_of[q] = -1;
        if ((tmask >> q) & 1) { pos_of[q] = j; P.tq[j++] = (int8_t)q; }
    }
    int b = 0;
    while (b < K && P.tq[b] == b) ++b;
    P.b = b;
    // segments: greedy, at most 4 distinct tile positions in registers
    const int nops = (int)pp.ops.size();
    std::vector<uint32_t> seg_sets;
    std::vector<int> seg_end;
    uint32_t cur = 0;
    for (int i = 0; i < nops; ++i) {
        const sv_op& o = ops[pp.ops[i]];
        uint32_t need = 0;
        if (o.kind == SV_OP_1Q) need = 1u << pos_of[o.qa];
        if (o.kind == SV_OP_2Q) need = (1u << pos_of[o.qa]) | (1u << pos_of[o.qb]);
        if (__builtin_popcount(cur | need) > RB) {
            seg_sets.push_back(cur);
            seg_end.push_back(i);
            cur = 0;
        }
        cur |= need;
    }
    seg_sets.push_back(cur);
    seg_end.push_back(nops);
    if ((int)seg_sets.size() > kMaxSegs) return -1;
    P.n_segs = (int)seg_sets.size();
    P.n_ops = nops;
    std::vector<int> seg_of(nops);
    for (int sgi = 0, i = 0; sgi < P.n_segs; ++sgi)
        for (; i < seg_end[sgi]; ++i) seg_of[i] = sgi;
    int regbit_of[kMaxSegs][13];
    for (int sgi = 0; sgi < P.n_segs; ++sgi) {
        uint32_t set = seg_sets[sgi];
        // free register slots take the tile positions the segment's diagonal masks use most:
        // a diagonal op on register bits multiplies an exact subset of the registers, on a
        // lane bit it runs on every register with part of the warp masked off (the adder's
        // CPHASE passes).  Ties (and segments without diagonal ops): from the top, as before.
        int use[16] = {0};
        for (int i = (sgi ? seg_end[sgi - 1] : 0); i < seg_end[sgi]; ++i) {
            const sv_op& o = ops[pp.ops[i]];
            if (o.kind == SV_OP_1Q || o.kind == SV_OP_2Q) continue;
            for (int q = 0; q < n; ++q)
                if (((o.diag_mask >> q) & 1) && pos_of[q] >= 0) ++use[pos_of[q]];
        }
        while (__builtin_popcount(set) < RB) {
            int best = -1;
            for (int pos = K - 1; pos >= 0; --pos)
                if (!((set >> pos) & 1) && (best < 0 || use[pos] > use[best])) best = pos;
            set |= 1u << best;
        }
        int r = 0, t = 0;
        for (int pos = 0; pos < K; ++pos) {
            regbit_of[sgi][pos] = -1;
            if ((set >> pos) & 1) { P.seg_reg[sgi][r] = (uint8_t)pos; regbit_of[sgi][pos] = r; ++r; }
            else P.seg_thr[sgi][t++] = (uint8_t)pos;
        }
        P.seg_end[sgi] = (uint16_t)seg_end[sgi];
    }
    auto lanes_contiguous = [&](int sgi) {
        // lanes = tile positions 0..4, the low_bits() lowest of them contiguous qubits: every
        // warp access covers whole runs of >= 2^low_bits amplitudes (full 32-byte sectors)
        return b >= low_bits() && P.seg_reg[sgi][0] >= 5;
    };
    // linear helpers: shared-memory swizzle and HBM offset of a set of tile positions
    auto swz_h = [](int e) {
        const int g = (((e >> 3) & 1) * 7) ^ (((e >> 4) & 1) * 3) ^ (((e >> 5) & 1) * 5) ^ (((e >> 6) & 1) * 6);
        return e ^ g;
    };
    auto gofs = [&](int e) {
        uint64_t o = 0;
        for (int pos = 0; pos < K; ++pos)
            if ((e >> pos) & 1) o += 1ull << P.tq[pos];
        return o;
    };
    for (int sgi = 0; sgi < P.n_segs; ++sgi)
        for (int i = 0; i < (1 << RB); ++i) {
            int e = 0;
            for (int bit = 0; bit < RB; ++bit)
                if ((i >> bit) & 1) e |= 1 << P.seg_reg[sgi][bit];
            P.seg_rsw[sgi][i] = (uint16_t)swz_h(e);
            if (sgi == P.n_segs - 1) P.last_rgo[i] = gofs(e);
        }
    for (int jj = 0; jj < (1 << RB); ++jj) P.pf_go[jj] = gofs(jj * NTH);
    {
        // deposit tables: tile index byte -> local index bits outside the tile
        int outpos[64], no = 0;
        for (int q = 0; q < n; ++q)
            if (!((tmask >> q) & 1)) outpos[no++] = q;
        if (no > 32) return -1;
        for (int byte = 0; byte < 4; ++byte)
            for (int v = 0; v < 256; ++v) {
                uint64_t d = 0;
                for (int bit = 0; bit < 8; ++bit) {
                    const int src = byte * 8 + bit;
                    if (((v >> bit) & 1) && src < no) d |= 1ull << outpos[src];
                }
                P.base_tab[byte][v] = d;
            }
    }
    // direct stores of the last segment from registers: coalesced when the lanes are the
    // contiguous low positions.  Single-buffered tiles (configs 8, 10) store directly for
    // any other lane layout too (a warp's 16-byte stores then cover 32-byte sectors in
    // halves that the write-back L2 merges; DRAM bytes unchanged): it saves the tile's
    // round trip through shared memory and lets the next tile's loads start as soon as the
    // last segment holds the tile in registers.  Measured on the C2 layers at N=33: passes
    // whose last segment keeps a low qubit in registers 62-71 -> 48-59 ms; double-buffered
    // tiles lose ~2 ms with scattered stores and keep the shared-memory path.
    // SVB200_DIRECT_OUT: 0 contiguous only, 1 (default) single-buffered too, 2 always.
    static const int dout_all = [] {
        const char* e = std::getenv("SVB200_DIRECT_OUT");
        return e ? std::atoi(e) : 1;
    }();
    static const int din_all = [] {
        const char* e = std::getenv("SVB200_DIRECT_IN");
        return e ? std::atoi(e) : 0;
    }();
    P.direct_in = din_all >= 2 ? 1 : lanes_contiguous(0);
    const bool single_buf = cfg == 8 || cfg == 10 || cfg == 11;
    P.direct_out = (dout_all >= 2 || (dout_all == 1 && single_buf)) ? 1 : lanes_contiguous(P.n_segs - 1);
    int md = 0;
    for (int i = 0; i < nops; ++i) {
        const sv_op& o = ops[pp.ops[i]];
        const int sgi = seg_of[i];
        P.moff[i] = (uint16_t)md;
        if (o.kind == SV_OP_1Q) {
            uint32_t mono = 0;
            const int cls = classify(o.m, 2, &mono);
            P.kind[i] = (uint8_t)(cls == 2 ? F2_1Q_MONO : (cls == 1 ? F2_1Q_REAL : F2_1Q));
            P.mono[i] = (uint16_t)mono;
            P.ra[i] = (uint8_t)regbit_of[sgi][pos_of[o.qa]];
            for (int c = 0; c < 8; ++c) P.mdata[md + c] = o.m[c];
            md += 8;
        } else if (o.kind == SV_OP_2Q) {
            uint32_t mono = 0;
            const int cls = classify(o.m, 4, &mono);
            P.kind[i] = (uint8_t)(cls == 2 ? F2_2Q_MONO : F2_2Q);   // real 4x4: generic path (exact)
            P.mono[i] = (uint16_t)mono;
            P.ra[i] = (uint8_t)regbit_of[sgi][pos_of[o.qa]];
            P.rb[i] = (uint8_t)regbit_of[sgi][pos_of[o.qb]];
            for (int c = 0; c < 32; ++c) P.mdata[md + c] = o.m[c];
            md += 32;
        } else {
            const bool neg = o.m[0] == -1.0 && o.m[1] == 0.0;
            P.kind[i] = (uint8_t)(neg ? F2_DIAG_NEG : F2_DIAG);
            uint32_t dreg = 0, dthr = 0;
            for (int q = 0; q < n; ++q) {
                if (!((o.diag_mask >> q) & 1) || pos_of[q] < 0) continue;
                const int rb = regbit_of[sgi][pos_of[q]];
                if (rb >= 0) dreg |= 1u << rb;
                else dthr |= 1u << pos_of[q];
            }
            P.dreg[i] = (uint8_t)dreg;
            P.dthr[i] = (uint16_t)dthr;
            P.dout[i] = o.diag_mask & ~tmask;
            P.mdata[md] = o.m[0];
            P.mdata[md + 1] = o.m[1];
            md += 2;
        }
    }
    return 0;
}

// greedy pass count of an op list with tiles of 2^K amplitudes (the 5 lowest qubits fixed)
// ops per fused pass: 128, or fewer (SVB200_MAX_PASS_OPS, tuning of diagonal-heavy passes);
// combined diagonal runs cost one factor multiply per op, so those passes take up to kMaxOps
constexpr int kDefaultPassOps = 128;
static int max_pass_ops() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("SVB200_MAX_PASS_OPS");
        const int x = e ? std::atoi(e) : kDefaultPassOps;
        v = (x >= 8 && x <= kMaxOps) ? x : kDefaultPassOps;
    }
    return g_combine_diag ? kMaxOps : v;
}
// A pass of mostly diagonal ops is closed at 80 ops: the specialised kernel then keeps
// them as straight-line code, which beats the descriptor loop that >= 96 diagonal ops
// need (adder N=32: two 124-op passes of 78 ms became 80 + 44 ops; 0.348 -> 0.305 s).
constexpr int kDiagPassOps = 80;
static bool pass_full(int n, int ndiag) {
    if (g_combine_diag) return n >= max_pass_ops();
    return n >= max_pass_ops() || (n >= kDiagPassOps && 4 * ndiag >= 3 * n);
}
static bool is_diag_kind(int kind) { return kind != SV_OP_1Q && kind != SV_OP_2Q; }

int count_passes(const sv_op* ops, int n_ops, int n, int K) {
    const uint64_t low = (1ull << low_bits()) - 1ull;
    uint64_t qm = 0;
    int passes = 0, cnt = 0, md = 0, nd = 0;
    for (int i = 0; i < n_ops; ++i) {
        const sv_op& o = ops[i];
        uint64_t need = 0;
        if (o.kind == SV_OP_1Q) need = 1ull << o.qa;
        if (o.kind == SV_OP_2Q) need = (1ull << o.qa) | (1ull << o.qb);
        if (cnt == 0 || popcount64(qm | need | low) > K || pass_full(cnt, nd) || md + op_mdata(o.kind) > kMaxMData) {
            if (cnt) ++passes;
            qm = 0; cnt = 0; md = 0; nd = 0;
        }
        qm |= need; ++cnt; md += op_mdata(o.kind); nd += is_diag_kind(o.kind);
    }
    (void)n;
    return passes + (cnt ? 1 : 0);
}

// configuration 9 ("auto"): 2^12 single-buffer tiles (config 8) when they save a pass over
// 2^11 tiles (config 6) for this op list -- fewer HBM passes at a lower per-pass efficiency
// (77 % vs 83 % of HBM measured), otherwise config 6
int choose_cfg(const sv_op* ops, int n_ops, int n) {
    if (n < 12 || !jit_enabled()) return 6;
    static const int ring = [] {   // SVB200_RING=1: 2^12 tiles as config 11 (two warp groups, 3 buffers)
        const char* e = std::getenv("SVB200_RING");
        return e ? std::atoi(e) : 0;
    }();
    if (count_passes(ops, n_ops, n, 12) < count_passes(ops, n_ops, n, 11)) return ring ? 11 : 8;
    return 6;
}

// prepare != nullptr: plan only and queue the specialised kernels of the v3 passes for
// compilation (sv_jit_prepare); *prepare counts them.  Nothing is launched.
// init != nullptr (*init != -2): the buffer holds |*init> (-1: zeros) only virtually; the first
// pass generates its tiles if its specialised kernel is ready, otherwise materialize() writes
// the state first.  *init is set to -2 once the state is real.
// sv_plan_pass_costs: the planning walk also records each pass's FP64 instructions per amplitude
static thread_local std::vector<double>* g_plan_costs = nullptr;

int fused_impl(void* psi, uint64_t n_elems, int mode, const sv_op* ops, int n_ops, int tile_bits,
               cudaStream_t st, int* prepare = nullptr, uint64_t chunk_mask = 0, uint64_t chunk_pat = 0,
               std::vector<int>* pass_ends = nullptr, int64_t* init = nullptr,
               const std::function<int()>& materialize_fn = nullptr) {
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "fused passes need FP64 or FP32 storage");
    if (!is_pow2(n_elems)) return fail(SV_EVALUE, "fused pass needs a power-of-two buffer");
    if (!prepare && (reinterpret_cast<uintptr_t>(psi) & 31) != 0)
        return fail(SV_EVALUE, "fused pass needs a 32-byte aligned buffer");
    const int n = log2u(n_elems);
    if (tile_bits <= 0) tile_bits = 12;
    int cfg = g_fused_v2 == 9 ? choose_cfg(ops, n_ops, n) : g_fused_v2;
    if (cfg == 11 && mode != SV_FP64) cfg = 8;   // the ring form exists for FP64 tiles only
    const int kv3 = (cfg == 2 || cfg == 4 || cfg == 6) ? 11 : ((cfg == 5 || cfg == 7) ? 10 : (cfg == 10 ? 13 : 12));
    // FP32 storage takes the v3 planning only when the specialised kernel can run it
    const bool use_v3 = cfg != 0 && (mode == SV_FP64 || (mode == SV_FP32 && jit_enabled())) &&
                        n >= kv3 && tile_bits >= kv3;
    const int k = use_v3 ? kv3 : (tile_bits < n ? tile_bits : n);
    if (k < 1 || k > (use_v3 ? 13 : kMaxTileBits)) return fail(SV_EVALUE, "tile bits %d out of range", tile_bits);
    const int bmin = k >= low_bits() ? low_bits() : k;
    const uint64_t lowfix = (1ull << bmin) - 1ull;
    for (int i = 0; i < n_ops; ++i) {
        const sv_op& o = ops[i];
        if (o.kind == SV_OP_1Q) {
            if (int rc = check_1q(n_elems, o.qa)) return rc;
        } else if (o.kind == SV_OP_2Q) {
            if (int rc = check_2q(n_elems, o.qa, o.qb)) return rc;
        } else if (o.kind == SV_OP_DIAG) {
            if (n < 64 && (o.diag_mask >> n))
                return fail(SV_EINDEX, "diagonal mask 0x%llx outside local array of %llu amplitudes",
                            (unsigned long long)o.diag_mask, (unsigned long long)n_elems);
        } else {
            return fail(SV_EVALUE, "unknown op kind %d", o.kind);
        }
    }
    PassPlan cur;
    auto flush = [&]() -> int {
        if (cur.ops.empty()) return SV_OK;
        if (pass_ends) pass_ends->push_back(cur.ops.back() + 1);
        if (prepare) {
            static thread_local Fused2Params Pp;
            if (use_v3 && build_params2(ops, cur, n, cfg, Pp) == 0 &&
                (g_seg_limit <= 0 || Pp.n_segs <= g_seg_limit)) {
                Pp.storage = mode;
                if (g_plan_costs) g_plan_costs->push_back(jit_fp64_per_amp(Pp));
                else *prepare += jit_prepare_fused(Pp);
            } else if (g_plan_costs) {
                g_plan_costs->push_back(-1.0);   // generic kernel (no specialised pass)
            }
            cur = PassPlan();
            return SV_OK;
        }
        cudaEvent_t ev0 = nullptr, ev1 = nullptr;
        if (g_timing) {
            cudaEventCreate(&ev0);
            cudaEventCreate(&ev1);
            cudaEventRecord(ev0, st);
        }
        cudaError_t e;
        static thread_local Fused2Params P2;
        if (chunk_mask) {   // chunked pass: only the specialised / register-resident kernels take it
            if (!use_v3 || build_params2(ops, cur, n, cfg, P2) != 0 || (P2.tile_mask & chunk_mask))
                return fail(SV_EVALUE, "chunked pass needs the v3 kernel and chunk bits outside its tile");
            // chunk bits in tile-index space: tile index bit j <-> j-th out-of-tile qubit
            uint64_t cm = 0, cp = 0;
            int j = 0;
            for (int q = 0; q < n; ++q) {
                if ((P2.tile_mask >> q) & 1) continue;
                if ((chunk_mask >> q) & 1) {
                    cm |= 1ull << j;
                    if ((chunk_pat >> q) & 1) cp |= 1ull << j;
                }
                ++j;
            }
            P2.cmask_t = cm;
            P2.cpat_t = cp;
            P2.n_tiles >>= __builtin_popcountll(cm);
            P2.storage = mode;
            const int jr = jit_launch_fused(psi, P2, st);
            e = jr < 0 ? cudaErrorLaunchFailure
                       : (jr == 0 ? cudaSuccess : (mode == SV_FP64 ? launch_fused2(psi, mode, P2, st)
                                                                     : cudaErrorNotSupported));
            if (e != cudaSuccess) return cuda_fail(e, "chunked fused pass launch");
            cur = PassPlan();
            return SV_OK;
        }
        auto v1 = [&]() {
            static thread_local FusedParams P;
            build_params(ops, cur, n, k, P);
            count_h2d(sizeof(FusedParams));
            return launch_fused(psi, mode, P, st);
        };
        // after a launch: the support moves through the pass's ops (in order)
        auto advance_support = [&]() {
            if (g_support)
                for (int i : cur.ops) support_apply(*g_support, ops[i]);
        };
        double pass_bytes = 2.0 * (double)n_elems * (mode == SV_FP32 ? 8.0 : 16.0);
        if (use_v3 && build_params2(ops, cur, n, cfg, P2) == 0 &&
            (g_seg_limit <= 0 || P2.n_segs <= g_seg_limit)) {
            P2.storage = mode;
            P2.vinit = -2;
            static const bool lazy_memset = [] {
                const char* e = std::getenv("SVB200_LAZY_MEMSET");
                return !e || std::atoi(e) != 0;
            }();
            static const bool lazy_pred = [] {
                const char* e = std::getenv("SVB200_LAZY_PRED");
                return !e || std::atoi(e) != 0;
            }();
            const uint64_t allq = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
            // tile-index bits of the support's fixed out-of-tile qubits and their values
            auto restrict_tiles = [&](uint64_t fixed_out, uint64_t* cm, uint64_t* cp) {
                *cm = *cp = 0;
                int j = 0;
                for (int q = 0; q < n; ++q) {
                    if ((P2.tile_mask >> q) & 1) continue;
                    if ((fixed_out >> q) & 1) {
                        *cm |= 1ull << j;
                        if ((g_support->val >> q) & 1) *cp |= 1ull << j;
                    }
                    ++j;
                }
            };
            if (lazy_memset && g_support && init && *init != -2 && materialize_fn) {
                // a lazy basis state under support tracking.  FP64 specialised passes: generate
                // only the support's tiles and leave the rest of HBM unwritten (dirty: later
                // passes load it as zeros, other readers zero-fill it first).  Otherwise write
                // the state (memset + the unit amplitude) and run the pass over the support's
                // tiles only -- either way no pass generates every tile through its arithmetic
                const uint64_t fixed_out = ~g_support->free & ~P2.tile_mask & allq;
                if (fixed_out) {
                    if (lazy_pred && mode == SV_FP64 && jit_predicable(P2)) {
                        uint64_t cm, cp;
                        restrict_tiles(fixed_out, &cm, &cp);
                        const uint64_t full_tiles = P2.n_tiles;
                        P2.cmask_t = cm;
                        P2.cpat_t = cp;
                        P2.n_tiles >>= __builtin_popcountll(cm);
                        P2.vinit = *init;
                        const int jr = jit_launch_fused(psi, P2, st);
                        if (jr < 0) return cuda_fail(cudaErrorLaunchFailure, "fused pass launch");
                        if (jr == 0) {
                            *init = -2;
                            g_support->dirty = true;
                            g_support_tiles_skipped += full_tiles - P2.n_tiles;
                            if (g_timing) {
                                cudaEventRecord(ev1, st);
                                std::lock_guard<std::mutex> lk(g_timing_mu);
                                g_timed.push_back({ev0, ev1, 0.5 * pass_bytes * (double)P2.n_tiles / (double)full_tiles});
                            }
                            advance_support();
                            cur = PassPlan();
                            return SV_OK;
                        }
                        P2.cmask_t = 0;   // not compiled yet: write the state
                        P2.cpat_t = 0;
                        P2.n_tiles = full_tiles;
                        P2.vinit = -2;
                    }
                    if (int rc = materialize_fn()) return rc;
                    *init = -2;
                }
            }
            // a dirty support (unwritten HBM outside it): the plain specialised FP64 passes load
            // those amplitudes as zeros; any other kernel needs them written first
            auto predicate = [&]() -> int {
                if (!g_support || !g_support->dirty) return SV_OK;
                if (mode == SV_FP64 && jit_predicable(P2)) {
                    P2.pfix = ~g_support->free & allq;
                    P2.pval = g_support->val & P2.pfix;
                    return SV_OK;
                }
                return clean_support(psi, n_elems, *g_support, st);
            };
            auto unpredicate = [&]() -> int {   // before a generic-kernel fallback
                P2.pfix = P2.pval = 0;
                return g_support ? clean_support(psi, n_elems, *g_support, st) : SV_OK;
            };
            if (g_support && !(init && *init != -2)) {
                // only the tiles whose fixed out-of-tile bits read val can be nonzero
                const uint64_t all = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
                const uint64_t fixed_out = ~g_support->free & ~P2.tile_mask & all;
                if (fixed_out) {
                    uint64_t cm, cp;
                    restrict_tiles(fixed_out, &cm, &cp);
                    const uint64_t full_tiles = P2.n_tiles;
                    P2.cmask_t = cm;
                    P2.cpat_t = cp;
                    P2.n_tiles >>= __builtin_popcountll(cm);
                    if (int rc = predicate()) return rc;
                    int jr = jit_launch_fused(psi, P2, st);
                    if (jr < 0) return cuda_fail(cudaErrorLaunchFailure, "fused pass launch");
                    if (jr != 0 && mode == SV_FP64) {   // not compiled yet: the generic kernel takes chunks too
                        if (int rc = unpredicate()) return rc;
                        count_h2d(sizeof(Fused2Params));
                        const cudaError_t eg = launch_fused2(psi, mode, P2, st);
                        if (eg != cudaSuccess) return cuda_fail(eg, "fused pass launch");
                        jr = 0;
                    }
                    if (jr == 0) {
                        g_support_tiles_skipped += full_tiles - P2.n_tiles;
                        if (g_timing) {
                            cudaEventRecord(ev1, st);
                            std::lock_guard<std::mutex> lk(g_timing_mu);
                            g_timed.push_back({ev0, ev1, pass_bytes * (double)P2.n_tiles / (double)full_tiles});
                        }
                        advance_support();
                        cur = PassPlan();
                        return SV_OK;
                    }
                    // FP32, specialised kernel not compiled yet: the whole state through v1
                    if (int rc = unpredicate()) return rc;
                    P2.cmask_t = 0;
                    P2.cpat_t = 0;
                    P2.n_tiles = full_tiles;
                }
            }
            if (init && *init != -2) {
                P2.vinit = *init;
                const int jr0 = jit_launch_fused(psi, P2, st);
                if (jr0 < 0) return cuda_fail(cudaErrorLaunchFailure, "fused pass launch");
                if (jr0 == 0) {          // generated its input: the state is real from here on
                    *init = -2;
                    if (g_timing) {
                        cudaEventRecord(ev1, st);
                        std::lock_guard<std::mutex> lk(g_timing_mu);
                        g_timed.push_back({ev0, ev1, 1.0 * (double)n_elems * (mode == SV_FP32 ? 8.0 : 16.0)});
                    }
                    advance_support();
                    cur = PassPlan();
                    return SV_OK;
                }
                if (int rc = materialize_fn ? materialize_fn() : SV_OK) return rc;   // not compiled yet
                *init = -2;
                P2.vinit = -2;
            }
            if (int rc = predicate()) return rc;
            const int jr = jit_launch_fused(psi, P2, st);
            count_h2d(sizeof(Fused2Params));
            if (jr < 0) e = cudaErrorLaunchFailure;
            else if (jr == 0) {
                e = cudaSuccess;
                if (P2.pfix) g_support->dirty = false;   // every tile written
            } else {                                     // not compiled yet
                if (int rc = unpredicate()) return rc;
                e = mode == SV_FP64 ? launch_fused2(psi, mode, P2, st) : v1();
            }
        } else if (mode == SV_FP32 && use_v3) {
            if (g_support)
                if (int rc = clean_support(psi, n_elems, *g_support, st)) return rc;
            if (init && *init != -2) {
                if (int rc = materialize_fn ? materialize_fn() : SV_OK) return rc;
                *init = -2;
            }
            e = v1();
        } else {
            if (g_support)
                if (int rc = clean_support(psi, n_elems, *g_support, st)) return rc;
            if (init && *init != -2) {
                if (int rc = materialize_fn ? materialize_fn() : SV_OK) return rc;
                *init = -2;
            }
            static thread_local FusedParams P;
            build_params(ops, cur, n, k, P);
            e = launch_fused(psi, mode, P, st);
            count_h2d(sizeof(FusedParams));
        }
        if (g_timing) {
            cudaEventRecord(ev1, st);
            std::lock_guard<std::mutex> lk(g_timing_mu);
            g_timed.push_back({ev0, ev1, pass_bytes});
        }
        if (e != cudaSuccess) return cuda_fail(e, "fused pass launch");
        advance_support();
        cur = PassPlan();
        return SV_OK;
    };
    for (int i = 0; i < n_ops; ++i) {
        const sv_op& o = ops[i];
        uint64_t need = 0;
        if (o.kind == SV_OP_1Q) need = 1ull << o.qa;
        if (o.kind == SV_OP_2Q) need = (1ull << o.qa) | (1ull << o.qb);
        const uint64_t merged = cur.qmask | need;
        const bool fits = popcount64(merged | (lowfix & ((n >= 64) ? ~0ull : ((1ull << n) - 1)))) <= k;
        if (!fits || pass_full((int)cur.ops.size(), cur.ndiag) || cur.mdata + op_mdata(o.kind) > kMaxMData) {
            if (int rc = flush()) return rc;
        }
        cur.qmask |= need;
        cur.ops.push_back(i);
        cur.mdata += op_mdata(o.kind);
        cur.ndiag += is_diag_kind(o.kind);
    }
    return flush();
}

// CTA slots the measurement passes leave free (sv_measure_reserve): the distributed
// measurement runs the global-qubit pair dots on a second stream at the same time, and a
// measurement grid that fills every slot (2 x 128-register CTAs per SM) would run first
// and serialise the two.
int g_measure_reserve = 0;

// FP64 measurement with the register-resident pass (sv_measure3.cu): tiles of 2^K
// (K = 12: 1 + ceil((n - 12) / 7) passes), segments of 4 register positions cover the
// cross terms of the pass's new tile qubits.
// sup (tracked support, FP64): amplitudes outside {i : (i & ~free) == val} are zero, so the
// passes read only the tiles inside it, cross terms are formed for the free qubits only (a
// fixed qubit's partner amplitudes are zero) and a fixed qubit's Qz is the norm or 0.
int measure3_impl(const void* psi, int n, double* norm, double* ones, double* cross, double* dev_partials,
                  size_t partial_cap, cudaStream_t st, bool byte = false, const Support* sup = nullptr) {
    const uint64_t all = (n >= 64) ? ~0ull : ((1ull << n) - 1ull);
    const bool tracked = sup && sup->on;
    const uint64_t freem = tracked ? (sup->free & all) : all, fixv = tracked ? (sup->val & ~sup->free & all) : 0;
    int dev = 0;
    cudaGetDevice(&dev);
    static int kenv = -1;
    if (kenv < 0) {
        const char* e = std::getenv("SVB200_MEASURE_K");
        kenv = (e && std::atoi(e) == 11) ? 11 : 12;
    }
    static int benv = -1;   // low index bits every later pass keeps in its tile (contiguous runs)
    if (benv < 0) {
        const char* e = std::getenv("SVB200_MEASURE_BMIN");
        benv = e ? std::max(1, std::min(5, std::atoi(e))) : 5;
    }
    const int K = byte ? 12 : kenv, bmin = benv;
    const int grid_cap = measure3_grid(dev, K, byte);
    const int slots = measure_slots(K, n);
    double* partials = dev_partials;
    const size_t need = (size_t)grid_cap * slots;
    bool owned = false;
    if (partials == nullptr || partial_cap < need) {
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&partials), need * sizeof(double), st), "measure scratch");
        owned = true;
    }
    std::vector<double> host(need);
    for (int q = 0; q < n; ++q) { ones[q] = 0; cross[2 * q] = cross[2 * q + 1] = 0; }
    *norm = 0;
    std::vector<uint64_t> passes;
    passes.push_back((1ull << K) - 1ull);
    for (int q = K; q < n;) {
        uint64_t t = (1ull << bmin) - 1ull;
        int c = 0;
        while (q < n && c < K - bmin) {
            if ((freem >> q) & 1) { t |= 1ull << q; ++c; }   // fixed qubits need no cross term
            ++q;
        }
        if (!c) break;
        for (int f = bmin; popcount64(t) < K; ++f) t |= 1ull << f;
        passes.push_back(t);
    }
    uint64_t done = ~freem & all;   // fixed qubits: cross terms are zero
    int rc = SV_OK;
    static thread_local Measure3Params P;
    for (size_t pi = 0; pi < passes.size() && rc == SV_OK; ++pi) {
        std::memset(&P, 0, sizeof(P));
        const uint64_t tmask = passes[pi];
        const int RB = 4, NT = 1 << (K - RB);   // register bits per segment (RB = 3 measured slower)
        P.n = n;
        P.kbits = K;
        P.rbits = RB;
        P.n_tiles = 1ull << (n - K);
        P.want_ones = pi == 0;
        int j = 0, o = 0;
        for (int q = 0; q < n; ++q) {
            if ((tmask >> q) & 1) P.tq[j++] = (int8_t)q;
            else if ((freem >> q) & 1) P.oq[o++] = (int8_t)q;   // tiles vary in the free out-of-tile bits
        }
        P.n_out = o;
        P.base_const = fixv & ~tmask;                             // and carry the fixed ones
        if (tracked && sup->dirty && !byte) {                     // unwritten HBM outside the support
            P.pfix = ~freem & all;
            P.pval = fixv;
        }
        P.n_tiles = 1ull << o;
        int b = 0;
        while (b < K && P.tq[b] == b) ++b;
        P.b = b;
        std::vector<int> cpos;
        for (int i = 0; i < K; ++i)
            if (!((done >> P.tq[i]) & 1)) cpos.push_back(i);
        // direct segment 0 (sv_measure3.cu DIRECT): its registers take cross positions >= 5 so
        // that its lanes are tile positions 0..4 = qubits 0..4 (512-byte warp loads)
        static int denv = -1;
        if (denv < 0) {
            const char* e = std::getenv("SVB200_MEASURE_DIRECT");
            denv = e ? std::atoi(e) : 0;   // measured slower (N=33: 108.9 vs 99.2 ms)
        }
        int n_hi = 0;
        for (int i : cpos) n_hi += i >= 5;
        P.direct = (denv && !byte && !P.pfix && K == 12 && b >= 5 && n_hi >= RB) ? 1 : 0;
        if (P.direct) std::stable_partition(cpos.begin(), cpos.end(), [](int i) { return i >= 5; });
        P.n_segs = (int)((cpos.size() + RB - 1) / RB);
        if (P.n_segs < 1) P.n_segs = 1;
        for (int sg = 0; sg < P.n_segs; ++sg) {
            uint32_t regs = 0;
            int cnt = 0;
            for (size_t c = (size_t)RB * sg; c < cpos.size() && cnt < RB; ++c, ++cnt) {
                P.seg_reg[sg][cnt] = (uint8_t)cpos[c];
                P.cross_reg[sg] |= 1u << cnt;
                regs |= 1u << cpos[c];
            }
            for (int pos = K - 1; pos >= 0 && cnt < RB; --pos)    // fill from the top
                if (!((regs >> pos) & 1)) { P.seg_reg[sg][cnt++] = (uint8_t)pos; regs |= 1u << pos; }
            // registers ascending by position within the segment keep the slot order simple
            int t = 0;
            for (int pos = 0; pos < K; ++pos)
                if (!((regs >> pos) & 1)) P.seg_thr[sg][t++] = (uint8_t)pos;
        }
        // swizzle columns with a conflict-free quarter-warp in every segment (as sv_jit.cu):
        // segment 0 of the first pass has registers at positions 0..3, where the fixed
        // columns 7,3,5,6 give 2-way conflicts
        {
            auto contrib = [](int pos, const int* c) { return pos < 3 ? (1 << pos) : (pos < 7 ? c[pos - 3] : 0); };
            auto ok = [&](const int* c) {
                for (int sg = 0; sg < P.n_segs; ++sg) {
                    const int a = contrib(P.seg_thr[sg][0], c), b2 = contrib(P.seg_thr[sg][1], c),
                              d = contrib(P.seg_thr[sg][2], c);
                    if (!a || !b2 || !d || a == b2 || a == d || b2 == d || (a ^ b2) == d) return false;
                }
                return true;
            };
            int cols[4] = {7, 3, 5, 6};
            if (!ok(cols)) {
                bool found = false;
                int c[4];
                for (c[0] = 1; c[0] < 8 && !found; ++c[0])
                    for (c[1] = 1; c[1] < 8 && !found; ++c[1])
                        for (c[2] = 1; c[2] < 8 && !found; ++c[2])
                            for (c[3] = 1; c[3] < 8 && !found; ++c[3])
                                if (ok(c)) {
                                    for (int i = 0; i < 4; ++i) cols[i] = c[i];
                                    found = true;
                                }
            }
            for (int i = 0; i < 4; ++i) P.swz_cols[i] = (uint8_t)cols[i];
            auto swz_h = [&](int e) {
                int g = 0;
                for (int bb = 3; bb < 7; ++bb)
                    if ((e >> bb) & 1) g ^= cols[bb - 3];
                return e ^ g;
            };
            for (int sg = 0; sg < P.n_segs; ++sg)
                for (int i = 0; i < (1 << RB); ++i) {
                    int e = 0;
                    for (int bit = 0; bit < RB; ++bit)
                        if ((i >> bit) & 1) e |= 1 << P.seg_reg[sg][bit];
                    P.seg_rsw[sg][i] = (uint16_t)swz_h(e);
                }
        }
        for (int jj = 0; jj < (1 << RB); ++jj) {
            uint64_t off = 0;
            for (int pos = 0; pos < K; ++pos)
                if (((jj * NT) >> pos) & 1) off += 1ull << P.tq[pos];
            P.pf_go[jj] = off;
            uint64_t o0 = 0;
            for (int bit = 0; bit < RB; ++bit)
                if ((jj >> bit) & 1) o0 += 1ull << P.tq[P.seg_reg[0][bit]];
            P.seg0_go[jj] = o0;
        }
        for (int byte = 0; byte < 4; ++byte)
            for (int v = 0; v < 256; ++v) {
                uint64_t d = 0;
                for (int bit = 0; bit < 8; ++bit) {
                    const int src = byte * 8 + bit;
                    if (((v >> bit) & 1) && src < o) d |= 1ull << P.oq[src];
                }
                P.base_tab[byte][v] = d;
            }
        // <= grid_cap; g_measure_reserve CTA slots stay free for a concurrent pair dot
        const int gcap = std::max(sm_count(dev), sm_count(dev) * measure3_ctas_per_sm(K, byte, P) - g_measure_reserve);
        const int grid = (int)((P.n_tiles < (uint64_t)gcap) ? P.n_tiles : gcap);
        cudaError_t e = byte ? launch_measure3_byte(*static_cast<const MeasureBytes*>(psi), P, partials, grid, st)
                             : launch_measure3(psi, P, partials, grid, st);
        if (e != cudaSuccess) { rc = cuda_fail(e, "measure launch"); break; }
        e = cudaMemcpyAsync(host.data(), partials, sizeof(double) * grid * slots, cudaMemcpyDeviceToHost, st);
        count_d2h(sizeof(double) * grid * slots);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { rc = cuda_fail(e, "measure readback"); break; }
        for (int g = 0; g < grid; ++g) {
            const double* row = host.data() + (size_t)g * slots;
            if (pi == 0) {
                *norm += row[0];
                for (int i = 0; i < K; ++i) ones[P.tq[i]] += row[1 + i];
                for (int jj = 0; jj < o; ++jj) ones[P.oq[jj]] += row[1 + K + jj];
            }
            for (int i : cpos) {   // the kernel's row: norm, K tile ones, n_out outside ones, cross
                cross[2 * P.tq[i]] += row[1 + K + o + 2 * i];
                cross[2 * P.tq[i] + 1] += row[2 + K + o + 2 * i];
            }
        }
        for (int i : cpos) done |= 1ull << P.tq[i];
    }
    if (tracked && rc == SV_OK)   // fixed qubits outside the first pass's tile: every amplitude shares the bit
        for (int q = 0; q < n; ++q)
            if (!((freem >> q) & 1) && !((passes[0] >> q) & 1)) ones[q] = ((fixv >> q) & 1) ? *norm : 0.0;
    if (owned) cudaFreeAsync(partials, st);
    return rc;
}

int measure_impl(const void* psi, uint64_t n_elems, int mode, double* norm, double* ones,
                 double* cross, double* dev_partials, size_t partial_cap, cudaStream_t st,
                 const Support* sup = nullptr) {
    if (!valid_fp_mode(mode) && mode != SV_BYTE) return fail(SV_EVALUE, "unknown storage mode");
    if (!is_pow2(n_elems)) return fail(SV_EVALUE, "measurement needs a power-of-two buffer");
    const int n = log2u(n_elems);
    if (n > 52) return fail(SV_EVALUE, "buffer too large");
    int dev = 0;
    cudaGetDevice(&dev);
    const int k = n < 12 ? n : 12;
    if (n == 0 && mode == SV_BYTE) return fail(SV_EVALUE, "BYTE measurement needs >= 2 amplitudes");
    if (n == 0) {  // a single amplitude: no qubits, just the norm
        double h[2];
        CUDA_TRY(cudaMemcpyAsync(h, psi, 16, cudaMemcpyDeviceToHost, st), "measure copy");
        CUDA_TRY(cudaStreamSynchronize(st), "measure sync");
        *norm = h[0] * h[0] + h[1] * h[1];
        return SV_OK;
    }
    static int use3 = -1;
    if (use3 < 0) {
        const char* e = std::getenv("SVB200_MEASURE3");
        use3 = (e && std::atoi(e) == 0) ? 0 : 1;
    }
    if (use3 && mode == SV_FP64 && n >= 16 && (reinterpret_cast<uintptr_t>(psi) & 15) == 0)
        return measure3_impl(psi, n, norm, ones, cross, dev_partials, partial_cap, st, false, sup);
    if (use3 && mode == SV_BYTE && n >= 16)
        return measure3_impl(psi, n, norm, ones, cross, dev_partials, partial_cap, st, true, sup);
    const int bmin = k >= 5 ? 5 : k;
    const int grid_cap = measure_grid(dev);
    const int slots_max = measure_slots(k, n);
    double* partials = dev_partials;
    const size_t need = (size_t)grid_cap * slots_max;
    bool owned = false;
    if (partials == nullptr || partial_cap < need) {
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&partials), need * sizeof(double), st),
                 "measure scratch");
        owned = true;
    }
    std::vector<double> host(need);
    for (int q = 0; q < n; ++q) { ones[q] = 0; cross[2 * q] = cross[2 * q + 1] = 0; }
    *norm = 0;
    // pass list: first {0..k-1}, then blocks of (k - bmin) higher qubits
    std::vector<uint64_t> passes;
    passes.push_back((1ull << k) - 1ull);
    for (int q = k; q < n;) {
        uint64_t t = (1ull << bmin) - 1ull;
        int c = 0;
        while (q < n && c < k - bmin) { t |= 1ull << q; ++q; ++c; }
        for (int f = bmin; popcount64(t) < k; ++f) t |= 1ull << f;   // fill (always < first new q)
        passes.push_back(t);
    }
    uint64_t done = 0;
    int rc = SV_OK;
    for (size_t pi = 0; pi < passes.size() && rc == SV_OK; ++pi) {
        MeasureParams P;
        std::memset(&P, 0, sizeof(P));
        const uint64_t tmask = passes[pi];
        P.n = n; P.k = k;
        P.tile_mask = tmask;
        P.out_mask = ((1ull << n) - 1ull) & ~tmask;
        P.n_tiles = 1ull << (n - k);
        P.want_ones = pi == 0;
        int j = 0, o = 0;
        int tq[64];
        for (int q = 0; q < n; ++q) {
            if ((tmask >> q) & 1) { P.tq[j] = (int8_t)q; tq[j] = q; ++j; }
            else P.oq[o++] = (int8_t)q;
        }
        int b = 0;
        while (b < k && P.tq[b] == b) ++b;
        P.b = b;
        uint32_t cp = 0;
        for (int i = 0; i < k; ++i)
            if (!((done >> tq[i]) & 1)) cp |= 1u << i;
        P.cross_pos = cp;
        const int grid = (int)((P.n_tiles < (uint64_t)grid_cap) ? P.n_tiles : grid_cap);
        const int slots = measure_slots(k, n);
        cudaError_t e = launch_measure(psi, mode, P, partials, grid, st);
        if (e != cudaSuccess) { rc = cuda_fail(e, "measure launch"); break; }
        e = cudaMemcpyAsync(host.data(), partials, sizeof(double) * grid * slots, cudaMemcpyDeviceToHost, st);
        count_d2h(sizeof(double) * grid * slots);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { rc = cuda_fail(e, "measure readback"); break; }
        // fixed-order host reduction over CTAs
        for (int g = 0; g < grid; ++g) {
            const double* row = host.data() + (size_t)g * slots;
            if (pi == 0) {
                *norm += row[0];
                for (int i = 0; i < k; ++i) ones[tq[i]] += row[1 + i];
                for (int jj = 0; jj < n - k; ++jj) ones[P.oq[jj]] += row[1 + k + jj];
            }
            for (int i = 0; i < k; ++i) {
                if (!((cp >> i) & 1)) continue;
                cross[2 * tq[i]] += row[1 + n + 2 * i];
                cross[2 * tq[i] + 1] += row[2 + n + 2 * i];
            }
        }
        for (int i = 0; i < k; ++i)
            if ((cp >> i) & 1) done |= 1ull << tq[i];
    }
    if (owned) cudaFreeAsync(partials, st);
    return rc;
}

}  // namespace

namespace sv {
int capi_fail(int code, const char* msg) { return fail(code, "%s", msg); }
int capi_cuda_fail(cudaError_t e, const char* what) { return cuda_fail(e, what); }
int capi_measure(const void* psi, uint64_t n, int mode, double* norm, double* ones, double* cross,
                 cudaStream_t st) {
    return measure_impl(psi, n, mode, norm, ones, cross, nullptr, 0, st);
}
// psi = host pointer to {mi plane, pi plane, decode tables} (sv_measure.cu ByteSrc)
int capi_measure_byte(const void* src, uint64_t n, double* norm, double* ones, double* cross, cudaStream_t st) {
    return measure_impl(src, n, SV_BYTE, norm, ones, cross, nullptr, 0, st);
}
// BYTE states with a tracked support (byte_state.py): the passes read only its tiles
int capi_measure_byte_sup(const void* src, uint64_t n, uint64_t sup_fixed, uint64_t sup_val, double* norm,
                          double* ones, double* cross, cudaStream_t st) {
    Support sp;
    sp.on = true;
    sp.free = ~sup_fixed & (n - 1ull);
    sp.val = sup_val & sup_fixed & (n - 1ull);
    return measure_impl(src, n, SV_BYTE, norm, ones, cross, nullptr, 0, st, &sp);
}
}  // namespace sv

// ---------------------------------------------------------------------------
struct sv_state {
    int device;
    int n;
    int mode;
    void* ptr;
    size_t bytes;
    cudaStream_t stream;
    double* partials;
    size_t partial_cap;
    int64_t lazy = -2;      // sv_zero_state_lazy: -1 all zeros / unit index not yet written, -2 none
    int diag_combine = 0;   // sv_set_diag_combine
    int track = 0;          // sv_set_support_tracking
    Support sup;            // valid while sup.on
};
extern "C" {
static int materialize(sv_handle h);
}

namespace {
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};
cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

int sv_abi_version(void) { return SV_ABI_VERSION; }
const char* sv_last_error(void) { return g_err.c_str(); }

int sv_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        *count = 0;
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    *count = c;
    return SV_OK;
}

int sv_set_device(int device) {
    CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");
    return SV_OK;
}

int sv_mem_info(int device, uint64_t* free_bytes, uint64_t* total_bytes) {
    DeviceGuard g(device);
    size_t f = 0, t = 0;
    CUDA_TRY(cudaMemGetInfo(&f, &t), "cudaMemGetInfo");
    *free_bytes = f;
    *total_bytes = t;
    return SV_OK;
}

int sv_sm_count(int device, int* count) {
    *count = sm_count(device);
    return SV_OK;
}

int svk_apply_1q(void* psi, uint64_t n, int mode, int q, const double* m8, void* stream) {
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "apply_1q needs FP64 or FP32 storage");
    if (int rc = check_1q(n, q)) return rc;
    const bool vec_ok = is_pow2(n) && n >= 64 && (reinterpret_cast<uintptr_t>(psi) & 31) == 0;
    cudaError_t e;
    if (vec_ok) {
        e = launch_gate1(psi, n, mode, q, m8, as_stream(stream));
    } else {
        const cplx m0 = {m8[0], m8[1]}, m1 = {m8[2], m8[3]}, m2 = {m8[4], m8[5]}, m3 = {m8[6], m8[7]};
        if (mode == SV_FP32)
            k_gate1_scalar<c32s><<<small_grid(n / 2), 256, 0, as_stream(stream)>>>(
                static_cast<c32s*>(psi), n / 2, q, m0, m1, m2, m3);
        else
            k_gate1_scalar<c64s><<<small_grid(n / 2), 256, 0, as_stream(stream)>>>(
                static_cast<c64s*>(psi), n / 2, q, m0, m1, m2, m3);
        e = cudaGetLastError();
        count_launch();
    }
    return e == cudaSuccess ? SV_OK : cuda_fail(e, "apply_1q launch");
}

int svk_apply_2q(void* psi, uint64_t n, int mode, int qa, int qb, const double* m32, void* stream) {
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "apply_2q needs FP64 or FP32 storage");
    if (int rc = check_2q(n, qa, qb)) return rc;
    cudaError_t e = launch_gate2(psi, n, mode, qa, qb, m32, as_stream(stream));
    return e == cudaSuccess ? SV_OK : cuda_fail(e, "apply_2q launch");
}

int svk_apply_diag(void* psi, uint64_t n, int mode, uint64_t mask, const double* f2, void* stream) {
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "apply_diag needs FP64 or FP32 storage");
    if (n == 0) return SV_OK;
    const bool structured = is_pow2(n) && n >= 64 && (reinterpret_cast<uintptr_t>(psi) & 31) == 0;
    if (structured && (mask & ~(n - 1)))
        return fail(SV_EINDEX, "diagonal mask 0x%llx outside local array of %llu amplitudes",
                    (unsigned long long)mask, (unsigned long long)n);
    cudaError_t e;
    if (structured) {
        e = launch_diag(psi, n, mode, mask, f2, as_stream(stream));
    } else {
        const cplx f = {f2[0], f2[1]};
        if (mode == SV_FP32)
            k_diag_all<c32s><<<small_grid(n), 256, 0, as_stream(stream)>>>(static_cast<c32s*>(psi), n, mask, f);
        else
            k_diag_all<c64s><<<small_grid(n), 256, 0, as_stream(stream)>>>(static_cast<c64s*>(psi), n, mask, f);
        e = cudaGetLastError();
        count_launch();
    }
    return e == cudaSuccess ? SV_OK : cuda_fail(e, "apply_diag launch");
}

int svk_pair_update(void* a0, void* a1, uint64_t count, int mode, const double* m8, void* stream) {
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "pair update needs FP64 or FP32 storage");
    if (count == 0) return SV_OK;
    cudaError_t e = launch_pair(a0, a1, count, mode, m8, as_stream(stream));
    return e == cudaSuccess ? SV_OK : cuda_fail(e, "pair update launch");
}

int svk_quad_update(void* const* parts, uint64_t count, int mode, const double* m32, void* stream) {
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "quad update needs FP64 or FP32 storage");
    if (count == 0) return SV_OK;
    cudaError_t e = launch_quad(parts, count, mode, m32, as_stream(stream));
    return e == cudaSuccess ? SV_OK : cuda_fail(e, "quad update launch");
}

int svk_apply_fused(void* psi, uint64_t n, int mode, const sv_op* ops, int n_ops, int tile_bits,
                    void* stream) {
    if (n_ops <= 0) return SV_OK;
    return fused_impl(psi, n, mode, ops, n_ops, tile_bits, as_stream(stream));
}

int svk_measure(const void* psi, uint64_t n, int mode, double* norm, double* ones, double* cross,
                void* stream) {
    return measure_impl(psi, n, mode, norm, ones, cross, nullptr, 0, as_stream(stream));
}

// ---- handles ---------------------------------------------------------------
int sv_create(int device, int n_qubits, int mode, sv_handle* out) {
    *out = nullptr;
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "handle storage mode %d not supported here", mode);
    if (n_qubits < 0 || n_qubits > 40) return fail(SV_EVALUE, "n_qubits %d out of range", n_qubits);
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(SV_EVALUE, "device %d not present (%d visible)", device, ndev);
    DeviceGuard g(device);
    keep_scratch_pool(device);
    sv_state* h = new sv_state();
    h->device = device;
    h->n = n_qubits;
    h->mode = mode;
    h->partials = nullptr;
    h->partial_cap = 0;
    const size_t bytes = (size_t)elem_bytes(mode) << n_qubits;
    h->bytes = bytes < 256 ? 256 : bytes;
    cudaError_t e = slab_alloc(&h->ptr, h->bytes);
    if (e != cudaSuccess) {
        delete h;
        return cuda_fail(e, "state allocation");
    }
    e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        slab_free(h->ptr, h->bytes);
        delete h;
        return cuda_fail(e, "stream creation");
    }
    const size_t cap = (size_t)measure_grid(device) * measure_slots(12, 40 > n_qubits ? n_qubits : 40);
    e = cudaMalloc(reinterpret_cast<void**>(&h->partials), cap * sizeof(double));
    if (e == cudaSuccess) h->partial_cap = cap;
    else { h->partials = nullptr; cudaGetLastError(); }
    *out = h;
    return SV_OK;
}

int sv_destroy(sv_handle h) {
    if (!h) return SV_OK;
    DeviceGuard g(h->device);
    cudaStreamSynchronize(h->stream);
    if (h->partials) cudaFree(h->partials);
    slab_free(h->ptr, h->bytes);
    cudaStreamDestroy(h->stream);
    delete h;
    return SV_OK;
}

int sv_info(sv_handle h, int* device, int* n_qubits, int* mode, void** dev_ptr, void** stream) {
    if (!h) return fail(SV_EVALUE, "null handle");
    if (dev_ptr) {   // the caller may touch the buffer directly
        DeviceGuard g(h->device);
        if (int rc = materialize(h)) return rc;
    }
    if (device) *device = h->device;
    if (n_qubits) *n_qubits = h->n;
    if (mode) *mode = h->mode;
    if (dev_ptr) *dev_ptr = h->ptr;
    if (stream) *stream = reinterpret_cast<void*>(h->stream);
    return SV_OK;
}

int sv_zero_state(sv_handle h, int64_t unit) {
    DeviceGuard g(h->device);
    // a basis state's support (materialize() writes the pending lazy |unit>, the same point)
    h->sup.on = h->track && unit >= 0;
    h->sup.free = 0;
    h->sup.val = unit >= 0 ? (uint64_t)unit : 0;
    h->sup.dirty = false;
    h->lazy = -2;
    const size_t eb = elem_bytes(h->mode);
    const uint64_t n = 1ull << h->n;
    CUDA_TRY(cudaMemsetAsync(h->ptr, 0, eb * n, h->stream), "zero state");
    if (unit >= 0) {
        if ((uint64_t)unit >= n) return fail(SV_EINDEX, "unit index %lld outside %llu amplitudes",
                                             (long long)unit, (unsigned long long)n);
        static const double one64[2] = {1.0, 0.0};
        static const float one32[2] = {1.0f, 0.0f};
        const void* src = h->mode == SV_FP32 ? static_cast<const void*>(one32) : static_cast<const void*>(one64);
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(h->ptr) + eb * unit, src, eb, cudaMemcpyHostToDevice,
                                 h->stream), "unit amplitude");
        count_h2d(eb);
    }
    return SV_OK;
}

// |unit> (or all zeros) recorded but not written: the first fused pass generates its tiles
// instead of reading them (saves the memset and one full read); any other use writes it now
int sv_zero_state_lazy(sv_handle h, int64_t unit) {
    if (unit >= (int64_t)(1ull << h->n)) return fail(SV_EINDEX, "unit index %lld outside the state", (long long)unit);
    h->lazy = unit < 0 ? -1 : unit;
    h->sup.on = h->track && unit >= 0;
    h->sup.free = 0;
    h->sup.val = unit >= 0 ? (uint64_t)unit : 0;
    h->sup.dirty = false;
    return SV_OK;
}

int sv_set_support_tracking(sv_handle h, int on) {
    h->track = on ? 1 : 0;
    if (!on) {
        DeviceGuard g(h->device);
        if (int rc = clean_support(h->ptr, 1ull << h->n, h->sup, h->stream)) return rc;
        h->sup.on = false;
    }
    return SV_OK;
}

// a support the caller derived itself (the distributed layer: its rank slice of the global
// support, re-derived after every remap swap); the handle then tracks it from here
int sv_set_support(sv_handle h, uint64_t free_mask, uint64_t val) {
    const uint64_t all = h->n >= 64 ? ~0ull : ((1ull << h->n) - 1ull);
    h->track = 1;
    h->sup.on = true;
    if (int rc = clean_support(h->ptr, 1ull << h->n, h->sup, h->stream)) return rc;
    h->sup.free = free_mask & all;
    h->sup.val = val & ~free_mask & all;
    return SV_OK;
}

// the support rule of the fused passes and sv_apply_1q/2q, without a state: *free_mask / *val
// move through ops in order (host-side bookkeeping of the distributed layer, and tests)
int sv_support_advance(const sv_op* ops, int n_ops, uint64_t* free_mask, uint64_t* val) {
    if (n_ops < 0 || (n_ops && !ops) || !free_mask || !val) return fail(SV_EVALUE, "bad support arguments");
    Support s;
    s.on = true;
    s.free = *free_mask;
    s.val = *val & ~*free_mask;
    for (int i = 0; i < n_ops; ++i) {
        if (ops[i].qa < 0 || ops[i].qa >= 64 || ops[i].qb < 0 || ops[i].qb >= 64)
            return fail(SV_EINDEX, "op %d: qubit outside 0..63", i);
        support_apply(s, ops[i]);
    }
    *free_mask = s.free;
    *val = s.val & ~s.free;
    return SV_OK;
}

int sv_support_info(sv_handle h, int* on, uint64_t* free_mask, uint64_t* val, uint64_t* tiles_skipped) {
    if (on) *on = h->sup.on ? 1 : 0;
    if (free_mask) *free_mask = h->sup.free;
    if (val) *val = h->sup.val;
    if (tiles_skipped) *tiles_skipped = g_support_tiles_skipped.load();
    return SV_OK;
}

static int materialize(sv_handle h) {
    if (h->lazy == -2) return clean_support(h->ptr, 1ull << h->n, h->sup, h->stream);
    const int64_t u = h->lazy;
    return sv_zero_state(h, u);   // clears h->lazy
}

int sv_apply_1q(sv_handle h, int q, const double* m8) {
    DeviceGuard g(h->device);
    if (int rc = materialize(h)) return rc;
    const int rc = svk_apply_1q(h->ptr, 1ull << h->n, h->mode, q, m8, h->stream);
    if (rc == SV_OK && h->sup.on) {
        sv_op o{};
        o.kind = SV_OP_1Q;
        o.qa = q;
        std::memcpy(o.m, m8, 8 * sizeof(double));
        support_apply(h->sup, o);
    }
    return rc;
}
int sv_apply_2q(sv_handle h, int qa, int qb, const double* m32) {
    DeviceGuard g(h->device);
    if (int rc = materialize(h)) return rc;
    const int rc = svk_apply_2q(h->ptr, 1ull << h->n, h->mode, qa, qb, m32, h->stream);
    if (rc == SV_OK && h->sup.on) {
        sv_op o{};
        o.kind = SV_OP_2Q;
        o.qa = qa;
        o.qb = qb;
        std::memcpy(o.m, m32, 32 * sizeof(double));
        support_apply(h->sup, o);
    }
    return rc;
}
int sv_apply_diag(sv_handle h, uint64_t mask, const double* f2) {
    DeviceGuard g(h->device);
    if (int rc = materialize(h)) return rc;
    return svk_apply_diag(h->ptr, 1ull << h->n, h->mode, mask, f2, h->stream);
}
int sv_jit_probe(const sv_op* ops, int n_ops, int n_qubits, char* src_out, size_t cap, double* compile_ms) {
    // plan the FIRST fused pass of `ops` on 2^n_qubits amplitudes exactly as fused_impl
    // does, print its specialised source, optionally compile it (CPU only)
    const char* pc = std::getenv("SVB200_PROBE_CFG");      // debugging: another tile configuration
    CombineScope cs(std::getenv("SVB200_PROBE_COMBINE") ? 1 : 0);   // debugging: combined diagonal runs
    const int pcfg = pc ? std::atoi(pc) : 6;
    const int K = (pcfg == 1 || pcfg == 3 || pcfg == 8 || pcfg == 11) ? 12 : (pcfg == 10 ? 13 : 11);
    if (n_qubits < K || n_qubits > 62 || n_ops <= 0) return fail(SV_EVALUE, "probe needs n >= 11 and ops");
    const uint64_t lowfix = (1ull << low_bits()) - 1ull;
    PassPlan cur;
    for (int i = 0; i < n_ops; ++i) {
        const sv_op& o = ops[i];
        uint64_t need = 0;
        if (o.kind == SV_OP_1Q) need = 1ull << o.qa;
        if (o.kind == SV_OP_2Q) need = (1ull << o.qa) | (1ull << o.qb);
        if (popcount64(cur.qmask | need | lowfix) > K || pass_full((int)cur.ops.size(), cur.ndiag) ||
            cur.mdata + op_mdata(o.kind) > kMaxMData)
            break;
        cur.qmask |= need;
        cur.ops.push_back(i);
        cur.mdata += op_mdata(o.kind);
        cur.ndiag += is_diag_kind(o.kind);
    }
    static thread_local Fused2Params P2;
    if (build_params2(ops, cur, n_qubits, pcfg, P2) != 0) return fail(SV_EVALUE, "pass does not fit the v3 kernel");
    std::string src, log;
    double ms = 0.0;
    const int rc = sv::jit_probe(P2, &src, compile_ms != nullptr, &ms, &log);
    if (compile_ms) *compile_ms = ms;
    if (src_out && cap) {
        std::strncpy(src_out, src.c_str(), cap - 1);
        src_out[cap - 1] = 0;
    }
    if (rc) return fail(SV_EVALUE, "NVRTC compile failed: %s", log.c_str());
    return (int)cur.ops.size();
}

int sv_plan_pass_costs(int n_qubits, int mode, const sv_op* ops, int n_ops, int tile_bits, int* ends,
                       double* fp64_per_amp, int cap, int flags) {
    if (n_qubits < 1 || n_qubits > 62) return fail(SV_EVALUE, "qubit count %d out of range", n_qubits);
    if ((flags & 1) && mode != SV_FP64) return fail(SV_EVALUE, "combined diagonal runs need FP64 storage");
    CombineScope cs(flags & 1);
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "passes are planned for FP64 / FP32 storage");
    if (n_ops <= 0) return 0;
    int queued = 0;
    std::vector<int> e;
    std::vector<double> c;
    g_plan_costs = &c;
    const int rc = fused_impl(nullptr, 1ull << n_qubits, mode, ops, n_ops, tile_bits, nullptr, &queued, 0, 0, &e);
    g_plan_costs = nullptr;
    if (rc) return rc;
    for (size_t i = 0; i < e.size() && (int)i < cap; ++i) {
        ends[i] = e[i];
        fp64_per_amp[i] = i < c.size() ? c[i] : -1.0;
    }
    return (int)e.size();
}

int sv_plan_passes(int n_qubits, int mode, const sv_op* ops, int n_ops, int tile_bits, int* ends, int cap) {
    if (n_qubits < 1 || n_qubits > 62) return fail(SV_EVALUE, "qubit count %d out of range", n_qubits);
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "passes are planned for FP64 / FP32 storage");
    if (n_ops <= 0) return 0;
    int queued = 0;
    std::vector<int> e;
    if (int rc = fused_impl(nullptr, 1ull << n_qubits, mode, ops, n_ops, tile_bits, nullptr, &queued, 0, 0, &e))
        return rc;
    for (size_t i = 0; i < e.size() && (int)i < cap; ++i) ends[i] = e[i];
    return (int)e.size();
}

int sv_jit_prepare(int n_qubits, const sv_op* ops, int n_ops, int tile_bits) {
    return sv_jit_prepare_mode(n_qubits, SV_FP64, ops, n_ops, tile_bits);
}

int sv_jit_prepare_opts(int n_qubits, int mode, const sv_op* ops, int n_ops, int tile_bits, int flags) {
    if ((flags & 1) && mode != SV_FP64) return fail(SV_EVALUE, "combined diagonal runs need FP64 storage");
    CombineScope cs(flags & 1);
    return sv_jit_prepare_mode(n_qubits, mode, ops, n_ops, tile_bits);
}

int sv_jit_prepare_mode(int n_qubits, int mode, const sv_op* ops, int n_ops, int tile_bits) {
    if (n_qubits < 1 || n_qubits > 62) return fail(SV_EVALUE, "qubit count %d out of range", n_qubits);
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "specialised passes exist for FP64 / FP32 storage");
    int queued = 0;
    if (int rc = fused_impl(nullptr, 1ull << n_qubits, mode, ops, n_ops, tile_bits, nullptr, &queued)) return rc;
    return queued;
}

int sv_apply_fused_chunk(sv_handle h, const sv_op* ops, int n_ops, int tile_bits, uint64_t chunk_mask,
                         uint64_t chunk_pattern) {
    DeviceGuard g(h->device);
    if (int rc = materialize(h)) return rc;
    if (n_ops <= 0) return SV_OK;
    if ((chunk_pattern & ~chunk_mask) || (chunk_mask >> h->n)) return fail(SV_EINDEX, "chunk mask outside the state");
    h->sup.on = false;   // chunked passes belong to the distributed layer (peers write this buffer)
    return fused_impl(h->ptr, 1ull << h->n, h->mode, ops, n_ops, tile_bits, h->stream, nullptr, chunk_mask,
                      chunk_pattern);
}

int sv_set_diag_combine(sv_handle h, int on) {
    if (on && h->mode != SV_FP64) return fail(SV_EVALUE, "combined diagonal runs need FP64 storage");
    h->diag_combine = on ? 1 : 0;
    return SV_OK;
}

int sv_apply_fused(sv_handle h, const sv_op* ops, int n_ops, int tile_bits) {
    DeviceGuard g(h->device);
    if (n_ops <= 0) return SV_OK;
    CombineScope cs(h->diag_combine);
    SupportScope ss(&h->sup);
    if (h->lazy != -2) {   // lazy |unit>: the first pass generates its input tiles
        int64_t init = h->lazy;
        const int rc = fused_impl(h->ptr, 1ull << h->n, h->mode, ops, n_ops, tile_bits, h->stream, nullptr, 0, 0,
                                  nullptr, &init, [&]() { return materialize(h); });
        if (rc == SV_OK) h->lazy = -2;
        return rc;
    }
    return svk_apply_fused(h->ptr, 1ull << h->n, h->mode, ops, n_ops, tile_bits, h->stream);
}
int sv_measure(sv_handle h, double* norm, double* ones, double* cross) {
    DeviceGuard g(h->device);
    // a dirty support (never-written HBM outside it) is read through zero-filled loads by
    // the register-resident FP64 measurement; any other form writes the zeros first
    const char* m3 = std::getenv("SVB200_MEASURE3");
    const bool zfill = h->lazy == -2 && h->sup.on && h->sup.dirty && h->mode == SV_FP64 && h->n >= 16 &&
                       !(m3 && std::atoi(m3) == 0);
    if (!zfill)
        if (int rc = materialize(h)) return rc;
    return measure_impl(h->ptr, 1ull << h->n, h->mode, norm, ones, cross, h->partials, h->partial_cap,
                        h->stream, h->sup.on ? &h->sup : nullptr);
}

int sv_export(sv_handle h, void* host, uint64_t first, uint64_t count) {
    DeviceGuard g(h->device);
    if (int rc = materialize(h)) return rc;
    const uint64_t n = 1ull << h->n;
    if (first > n || count > n - first) return fail(SV_EINDEX, "export range outside the state");
    const size_t eb = elem_bytes(h->mode);
    CUDA_TRY(cudaMemcpyAsync(host, static_cast<char*>(h->ptr) + eb * first, eb * count,
                             cudaMemcpyDeviceToHost, h->stream), "export");
    count_d2h(eb * count);
    CUDA_TRY(cudaStreamSynchronize(h->stream), "export sync");
    return SV_OK;
}

int sv_import(sv_handle h, const void* host, uint64_t first, uint64_t count) {
    DeviceGuard g(h->device);
    if (int rc = materialize(h)) return rc;
    h->sup.on = false;   // arbitrary values
    const uint64_t n = 1ull << h->n;
    if (first > n || count > n - first) return fail(SV_EINDEX, "import range outside the state");
    const size_t eb = elem_bytes(h->mode);
    CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(h->ptr) + eb * first, host, eb * count,
                             cudaMemcpyHostToDevice, h->stream), "import");
    count_h2d(eb * count);
    CUDA_TRY(cudaStreamSynchronize(h->stream), "import sync");
    return SV_OK;
}

int sv_synchronize(sv_handle h) {
    DeviceGuard g(h->device);
    // a pending lazy basis state is written; a dirty support's unwritten HBM stays unwritten
    // (synchronising reads nothing; every reader zero-fills it first)
    if (h->lazy != -2)
        if (int rc = materialize(h)) return rc;
    CUDA_TRY(cudaStreamSynchronize(h->stream), "synchronize");
    return SV_OK;
}

int sv_launch_count(uint64_t* count) {
    *count = sv::launch_total();
    return SV_OK;
}

int sv_transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
    *h2d = g_h2d.load();
    *d2h = g_d2h.load();
    return SV_OK;
}

int sv_fused_variant(int v2) {
    if (v2 < 0 || v2 > 11) return fail(SV_EVALUE, "fused variant %d not in 0..11", v2);
    g_fused_v2 = v2;
    return SV_OK;
}

int sv_fused_segment_limit(int limit) {
    g_seg_limit = limit;
    return SV_OK;
}

int sv_pass_timing(int enable) {
    g_timing = enable != 0;
    return SV_OK;
}

int sv_pass_timing_read(uint64_t* passes, double* ms, double* bytes) {
    std::vector<TimedPass> v;
    {
        std::lock_guard<std::mutex> lk(g_timing_mu);
        v.swap(g_timed);
    }
    double tot = 0.0, by = 0.0;
    for (auto& t : v) {
        float m = 0.f;
        cudaEventSynchronize(t.b);
        if (cudaEventElapsedTime(&m, t.a, t.b) == cudaSuccess) tot += m;
        by += t.bytes;
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    *passes = v.size();
    *ms = tot;
    *bytes = by;
    return SV_OK;
}

int sv_ipc_handle(sv_handle h, void* out64) {
    DeviceGuard g(h->device);
    if (int rc = materialize(h)) return rc;
    cudaIpcMemHandle_t ih;
    CUDA_TRY(cudaIpcGetMemHandle(&ih, h->ptr), "cudaIpcGetMemHandle");
    slab_mark_exported(h->ptr);
    static_assert(sizeof(ih) == 64, "IPC handle size");
    std::memcpy(out64, &ih, 64);
    return SV_OK;
}

int sv_ipc_open(int device, const void* handle64, void** peer_ptr) {
    DeviceGuard g(device);
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, handle64, 64);
    CUDA_TRY(cudaIpcOpenMemHandle(peer_ptr, ih, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    return SV_OK;
}

int sv_ipc_close(int device, void* peer_ptr) {
    DeviceGuard g(device);
    CUDA_TRY(cudaIpcCloseMemHandle(peer_ptr), "cudaIpcCloseMemHandle");
    return SV_OK;
}

int svk_swap_peer(void* own, void* peer, uint64_t n_local_elems, int mode, int l, int side, void* stream) {
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "swap needs FP64 or FP32 storage");
    if (!is_pow2(n_local_elems) || n_local_elems < 4) return fail(SV_EVALUE, "swap needs a power-of-two slice >= 4");
    if (l < 0 || (1ull << l) >= n_local_elems) return fail(SV_EINDEX, "swap qubit %d outside the slice", l);
    if (side != 0 && side != 1) return fail(SV_EVALUE, "side must be 0 or 1");
    cudaError_t e = launch_swap_peer(own, peer, n_local_elems, mode, l, side, as_stream(stream));
    return e == cudaSuccess ? SV_OK : cuda_fail(e, "swap launch");
}

int svk_swap_group(void* own, void* peer, uint64_t n_local_elems, int mode, uint64_t victim_mask,
                   uint64_t own_pattern, uint64_t peer_pattern, uint64_t t_begin, uint64_t t_count, void* stream) {
    return svk_swap_group_chunk(own, peer, n_local_elems, mode, victim_mask, own_pattern, peer_pattern, 0, 0, t_begin,
                                t_count, stream);
}

int sv_measure_reserve(int ctas) {
    const int prev = g_measure_reserve;
    if (ctas >= 0) g_measure_reserve = ctas;
    return prev;
}

int sv_swap_blocks(int blocks) {
    const int prev = sv::g_swap_blocks;
    if (blocks >= 0) sv::g_swap_blocks = blocks;
    return prev;
}

int svk_swap_group_chunk(void* own, void* peer, uint64_t n_local_elems, int mode, uint64_t victim_mask,
                         uint64_t own_pattern, uint64_t peer_pattern, uint64_t chunk_mask, uint64_t chunk_pattern,
                         uint64_t t_begin, uint64_t t_count, void* stream) {
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "swap needs FP64 or FP32 storage");
    if (!is_pow2(n_local_elems)) return fail(SV_EVALUE, "swap needs a power-of-two slice");
    if (((victim_mask | chunk_mask) & ~(n_local_elems - 1)) || ((own_pattern | peer_pattern) & ~victim_mask) ||
        (victim_mask & chunk_mask) || (chunk_pattern & ~chunk_mask))
        return fail(SV_EINDEX, "victim / chunk masks or patterns outside the slice or overlapping");
    const uint64_t rest = n_local_elems >> __builtin_popcountll(victim_mask | chunk_mask);
    if (t_begin > rest || t_count > rest - t_begin) return fail(SV_EINDEX, "rest range outside the slice");
    if (t_count == 0) return SV_OK;
    cudaError_t e = launch_swap_group(own, peer, t_begin, t_count, mode, victim_mask, own_pattern, peer_pattern,
                                      chunk_mask, chunk_pattern, as_stream(stream));
    return e == cudaSuccess ? SV_OK : cuda_fail(e, "group swap launch");
}

static int pair_dot_impl(const void* a0, const void* a1, uint64_t t_begin, uint64_t count, uint64_t cmask,
                         uint64_t cpat, bool chunk, int mode, int max_blocks, double* out2, void* stream) {
    if (!valid_fp_mode(mode)) return fail(SV_EVALUE, "pair dot needs FP64 or FP32 storage");
    out2[0] = out2[1] = 0.0;
    if (count == 0) return SV_OK;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t cap = max_blocks > 0 ? (uint64_t)max_blocks : (uint64_t)sm_count(dev) * 2;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((count + 1023) / 1024, cap));
    double* part = nullptr;
    cudaStream_t st = as_stream(stream);
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&part), 16 * grid, st), "pair dot scratch");
    cudaError_t e = chunk ? launch_pair_dot_chunk(a0, a1, t_begin, count, cmask, cpat, mode, part, grid, st)
                          : launch_pair_dot(a0, a1, count, mode, part, grid, st);
    std::vector<double> h(2 * grid);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), part, 16 * grid, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(part, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "pair dot");
    for (int b = 0; b < grid; ++b) { out2[0] += h[2 * b]; out2[1] += h[2 * b + 1]; }
    return SV_OK;
}

int svk_pair_dot(const void* a0, const void* a1, uint64_t count, int mode, int max_blocks, double* out2,
                 void* stream) {
    return pair_dot_impl(a0, a1, 0, count, 0, 0, false, mode, max_blocks, out2, stream);
}

int svk_pair_dot_chunk(const void* a0, const void* a1, uint64_t n_elems, int mode, uint64_t chunk_mask,
                       uint64_t chunk_pattern, uint64_t t_begin, uint64_t t_count, int max_blocks, double* out2,
                       void* stream) {
    if (!is_pow2(n_elems) || (chunk_mask & ~(n_elems - 1)) || (chunk_pattern & ~chunk_mask))
        return fail(SV_EINDEX, "chunk mask / pattern outside the buffer");
    const uint64_t rest = n_elems >> __builtin_popcountll(chunk_mask);
    if (t_begin > rest || t_count > rest - t_begin) return fail(SV_EINDEX, "rest range outside the buffer");
    return pair_dot_impl(a0, a1, t_begin, t_count, chunk_mask, chunk_pattern, true, mode, max_blocks, out2, stream);
}

int sv_buffer_alloc(int device, uint64_t bytes, void** ptr) {
    DeviceGuard g(device);
    CUDA_TRY(cudaMalloc(ptr, bytes ? bytes : 256), "buffer allocation");
    return SV_OK;
}
int sv_buffer_free(int device, void* ptr) {
    DeviceGuard g(device);
    CUDA_TRY(cudaFree(ptr), "buffer free");
    return SV_OK;
}
int sv_copy_h2d(void* dst, const void* src, uint64_t bytes, void* stream) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)), "h2d copy");
    count_h2d(bytes);
    CUDA_TRY(cudaStreamSynchronize(as_stream(stream)), "h2d sync");
    return SV_OK;
}
int sv_copy_d2h(void* dst, const void* src, uint64_t bytes, void* stream) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)), "d2h copy");
    count_d2h(bytes);
    CUDA_TRY(cudaStreamSynchronize(as_stream(stream)), "d2h sync");
    return SV_OK;
}
int sv_stream_create(int device, void** stream) {
    DeviceGuard g(device);
    cudaStream_t s;
    CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream create");
    *stream = reinterpret_cast<void*>(s);
    return SV_OK;
}
int sv_stream_destroy(void* stream) {
    cudaStreamDestroy(as_stream(stream));
    return SV_OK;
}

int sv_event_create(void** ev) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e), "event create");
    *ev = reinterpret_cast<void*>(e);
    return SV_OK;
}
int sv_event_destroy(void* ev) {
    cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev));
    return SV_OK;
}
int sv_event_create_ipc(void** ev, void* handle_out64) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventInterprocess), "IPC event create");
    cudaIpcEventHandle_t hnd;
    static_assert(sizeof(hnd) == 64, "IPC event handle size");
    cudaError_t r = cudaIpcGetEventHandle(&hnd, e);
    if (r != cudaSuccess) {
        cudaEventDestroy(e);
        return cuda_fail(r, "cudaIpcGetEventHandle");
    }
    std::memcpy(handle_out64, &hnd, 64);
    *ev = reinterpret_cast<void*>(e);
    return SV_OK;
}
int sv_event_open_ipc(const void* handle64, void** ev) {
    cudaIpcEventHandle_t hnd;
    std::memcpy(&hnd, handle64, 64);
    cudaEvent_t e;
    CUDA_TRY(cudaIpcOpenEventHandle(&e, hnd), "cudaIpcOpenEventHandle");
    *ev = reinterpret_cast<void*>(e);
    return SV_OK;
}
int sv_stream_wait_event(void* stream, void* ev) {
    CUDA_TRY(cudaStreamWaitEvent(as_stream(stream), reinterpret_cast<cudaEvent_t>(ev), 0), "stream wait event");
    return SV_OK;
}
int sv_event_record(void* ev, void* stream) {
    CUDA_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev), as_stream(stream)), "event record");
    return SV_OK;
}
int sv_event_elapsed_ms(void* start, void* stop, float* ms) {
    CUDA_TRY(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(stop)), "event sync");
    CUDA_TRY(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(start), reinterpret_cast<cudaEvent_t>(stop)),
             "event elapsed");
    return SV_OK;
}
int sv_stream_synchronize(void* stream) {
    CUDA_TRY(cudaStreamSynchronize(as_stream(stream)), "stream synchronize");
    return SV_OK;
}

}  // extern "C"
