// Adaptive two-byte polar encoding on the B200 (sm_100a).
//
// Reference: /root/reference/pkg/src/svsim/codec.py and engine.py:186-225.
// A BYTE state is two uint8 planes (magnitude index, phase index) per
// amplitude.  One gate = one kernel pass that, per amplitude group,
//   decodes   mags[mi] * (ux[pi] + i uy[pi])           (codec.py:203-206)
//   applies   the gate with numpy's FP64 operand order  (kernels.py)
//   canonicalises each produced value                   (codec.py:33-53)
//   encodes   it against the CURRENT tables, nearest entry, ties to the
//             smaller original index                    (codec.py:56-71, 193-201)
//   proposes  values whose magnitude / phase is not representable
//             (codec.py:122-152) into per-CTA shared-memory hash sets,
//             flushed to a global candidate buffer at the end of the pass.
// so compressed amplitudes never round-trip HBM in FP64 (2 B read + 2 B
// written per amplitude).  The pass writes a second pair of planes; if the
// host-side merge of the candidates (the reference's per-gate barrier) grows
// a table, the pass is re-run from the untouched input planes with the new
// tables before the planes are swapped.
//
// Exactness.  |v| is numpy's complex abs (L*sqrt(fma(S/L,S/L,1))), ux/uy are
// IEEE divisions: bit-identical to numpy.  The angle is numpy's SVML atan2 in
// the reference, which is not reproducible on the GPU, so theta is computed
// with CUDA atan2 (<= 2 ulp) EXCEPT on the axes (im == 0 or re == 0), where
// both libraries return the exact IEEE special values.  Every decision that
// depends on theta (nearest phase entry, 1e-12 representability, the 2*pi
// wrap) is taken with a margin; amplitudes inside the margin are listed as
// "uncertain" and resolved on the host with numpy, so the produced bytes are
// the reference's bytes.
#include <algorithm>
#include <mutex>
#include <map>
#include <cstdlib>
#include <cstring>

#include "sv_byte.cuh"
#include "sv_common.cuh"
#include "sv_kernels.cuh"

namespace sv {

namespace {
constexpr double TWO_PI = 6.283185307179586;        // 2.0 * math.pi
constexpr double MAG_RTOL = 1e-12, PHASE_ATOL = 1e-12;
constexpr double TH_MARGIN = 1e-14;                 // >> |atan2_cuda - atan2_svml| (a few ulp of 2pi)
constexpr int NT = 256;

struct STables {
    double dmag[256], dux[256], duy[256];
    double smag[256], sth[256];
    double sqmid[256];      // squared midpoints of consecutive sorted magnitudes (+inf sentinel)
    double sqmag[256];      // squared sorted magnitudes
    uint8_t smag_idx[256], sth_idx[256];
    int n_mag, n_ph;
    int search_top;         // largest power of two < n_mag (branch-free search)
};

__device__ __forceinline__ cplx decode(const STables& t, uint8_t mi, uint8_t pi) {
    if (mi == 0) return {0.0, 0.0};
    const double m = t.dmag[mi];
    return {__dmul_rn(m, t.dux[pi]), __dmul_rn(m, t.duy[pi])};
}

struct Polar {
    double r, th, ux, uy;
    bool th_exact;      // theta bit-identical to numpy (axis values, zero)
    bool wrap_unsure;   // the 2*pi wrap decision is inside the margin
};

__device__ __forceinline__ Polar canon(cplx v) {
    Polar p;
    const double ax = fabs(v.re), ay = fabs(v.im);
    const double L = fmax(ax, ay), S = fmin(ax, ay);
    if (L == 0.0) {
        p.r = 0.0;
    } else {
        const double q = __ddiv_rn(S, L);
        p.r = __dmul_rn(L, __dsqrt_rn(__fma_rn(q, q, 1.0)));
    }
    p.wrap_unsure = false;
    if (p.r == 0.0) {
        p.th = 0.0; p.ux = 1.0; p.uy = 0.0; p.th_exact = true;
        return p;
    }
    double a;
    if (v.im == 0.0) {            // atan2(+-0, x): +-0 or +-pi (exact in every libm)
        a = v.re > 0.0 ? 0.0 : (signbit(v.im) ? -3.141592653589793 : 3.141592653589793);
        p.th_exact = true;
    } else if (v.re == 0.0) {     // atan2(y, +-0) = +-pi/2
        a = v.im > 0.0 ? 1.5707963267948966 : -1.5707963267948966;
        p.th_exact = true;
    } else {
        a = atan2(v.im, v.re);
        p.th_exact = false;
    }
    double th = (a == 0.0) ? 0.0 : (a < 0.0 ? __dadd_rn(a, TWO_PI) : a);   // np.mod(a, 2pi)
    const double gap = __dsub_rn(TWO_PI, th);
    if (gap < PHASE_ATOL) th = 0.0;
    if (!p.th_exact && fabs(gap - PHASE_ATOL) <= TH_MARGIN) p.wrap_unsure = true;
    p.th = th;
    p.ux = __dadd_rn(__ddiv_rn(v.re, p.r), 0.0);
    p.uy = __dadd_rn(__ddiv_rn(v.im, p.r), 0.0);
    return p;
}

// numpy.searchsorted(side='left'): first i with s[i] >= x
__device__ __forceinline__ int lower_bound(const double* s, int n, double x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// codec.py:56-71; returns index, and sets *unsure if a perturbation of x by
// `margin` could change the answer
__device__ __forceinline__ int nearest(const double* s, const uint8_t* orig, int n, double x, bool circular,
                                       double margin, bool* unsure) {
    const int pos = lower_bound(s, n, x);
    const int last = n - 1;
    // four candidates, always (duplicates of candidate 0 when the wrap entries do not apply):
    // a fixed shape keeps everything in registers
    const bool wrap = circular && last > 0;
    const int c0 = min(max(pos - 1, 0), last), c1 = min(max(pos, 0), last);
    const int cand[4] = {c0, c1, wrap ? 0 : c0, wrap ? last : c0};
    double d[4];
    double best = 1e300;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        double dd = fabs(__dsub_rn(s[cand[c]], x));
        if (circular) dd = fmin(dd, __dsub_rn(TWO_PI, dd));
        d[c] = dd;
        best = fmin(best, dd);
    }
    int idx = 1 << 30;
#pragma unroll
    for (int c = 0; c < 4; ++c)
        if (d[c] == best) idx = min(idx, (int)orig[cand[c]]);
    if (margin > 0.0) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if ((int)orig[cand[c]] != idx && d[c] - best <= 2.0 * margin) *unsure = true;
    }
    return idx;
}

// codec.py:122-135 for one value: 1 representable, 0 not, -1 inside the margin
__device__ __forceinline__ int representable(const double* s, int n, double x, bool mag, double margin) {
    const int pos = lower_bound(s, n, x);
    const int last = n - 1;
    const int c0 = min(max(pos - 1, 0), last), c1 = min(max(pos, 0), last);
    int verdict = 0;
    for (int k = 0; k < 2; ++k) {
        const double e = s[k == 0 ? c0 : c1];
        double d = fabs(__dsub_rn(e, x));
        double tol;
        if (mag) {
            tol = __dmul_rn(MAG_RTOL, fmax(fabs(x), fabs(e)));
        } else {
            d = fmin(d, __dsub_rn(TWO_PI, d));
            tol = PHASE_ATOL;
        }
        if (d <= tol - margin) return 1;
        if (d <= tol + margin) verdict = -1;
    }
    return verdict;
}

// ---- per-CTA candidate sets ----------------------------------------------------
constexpr int MAG_SLOTS = 1024;
constexpr int PH_SLOTS = 512;
constexpr unsigned long long EMPTY = ~0ull;

struct CtaSets {
    unsigned long long mag_key[MAG_SLOTS];
    unsigned long long ph_key[PH_SLOTS];
    double ph_ux[PH_SLOTS], ph_uy[PH_SLOTS], ph_re[PH_SLOTS], ph_im[PH_SLOTS];
    int ph_lock[PH_SLOTS];
    int mag_count, ph_count;
    int full;                       // a set ran out of slots: flush at the next barrier
    int mag_rs, ph_rs;              // slots per producer region (tagged collection: one region
                                    // per reference rank, so each rank's proposal stays separate)
};

__device__ __forceinline__ unsigned hash64(unsigned long long k) {
    k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
    return (unsigned)k;
}

__device__ void global_mag(ByteCand* out, double r, int prod) {
    const unsigned long long slot = atomicAdd(&out->n_mag, 1ull);
    if (slot < out->cap_mag) {
        out->mag[slot] = r;
        out->mag_tag[slot] = prod;
    } else {
        out->overflow = 1;
    }
}

__device__ void global_phase(ByteCand* out, const Polar& p, cplx v, int prod) {
    const unsigned long long slot = atomicAdd(&out->n_ph, 1ull);
    if (slot < out->cap_ph) {
        out->ph[4 * slot + 0] = v.re;
        out->ph[4 * slot + 1] = v.im;
        out->ph[4 * slot + 2] = p.ux;
        out->ph[4 * slot + 3] = p.uy;
        out->ph_tag[slot] = prod;
    } else {
        out->overflow = 1;
    }
}

// shared-memory set first; a full set spills straight to the global buffer
// (duplicates there are harmless: the host takes unique values / first per theta)
__device__ void insert_mag(CtaSets& s, ByteCand* out, double r, int prod) {
    const unsigned long long key = (unsigned long long)__double_as_longlong(r);
    const unsigned rs = (unsigned)s.mag_rs, base = (unsigned)prod * rs;
    unsigned h = hash64(key) & (rs - 1);
    for (int probe = 0; probe < 64; ++probe) {
        const unsigned long long cur = s.mag_key[base + h];
        if (cur == key) return;
        if (cur == EMPTY) {
            const unsigned long long prev = atomicCAS(&s.mag_key[base + h], EMPTY, key);
            if (prev == EMPTY) { atomicAdd(&s.mag_count, 1); return; }
            if (prev == key) return;
        }
        h = (h + 1) & (rs - 1);
    }
    global_mag(out, r, prod);
}

__device__ __forceinline__ bool lex_less(double ax, double ay, double bx, double by) {
    return ax < bx || (ax == bx && ay < by);
}

// Phase candidates.  codec.py:137-152 keeps, per exact numpy theta, the value of smallest
// (ux, uy).  Only on the axes is the device's theta bit-identical to numpy's: there values
// are grouped by theta and the smallest (ux, uy) kept.  Any other angle comes from CUDA
// atan2, which can round two angles numpy keeps apart (a few ulps) to the same double, so
// grouping by it could drop a proposal (tests/test_gpu_byte.py clustered-angle test): such
// values are kept per distinct VALUE (re, im), deduplicated exactly, and the host groups
// them by numpy's theta (codec.finalize_proposal).  Keys: theta bits (top bit 0, theta is
// in [0, 2 pi)) or a hash of the value bits with the top bit set; a value key is confirmed
// by comparing the stored (re, im) under the slot lock (hash collisions keep probing).
__device__ __forceinline__ unsigned long long value_key(cplx v) {
    const unsigned long long a = (unsigned long long)__double_as_longlong(v.re);
    const unsigned long long b = (unsigned long long)__double_as_longlong(v.im);
    unsigned long long k = a * 0x9e3779b97f4a7c15ull ^ (b + 0x632be59bd9b4e019ull + (a << 6) + (a >> 2));
    k ^= k >> 31;
    return k | (1ull << 63);
}

__device__ void insert_phase(CtaSets& s, ByteCand* out, const Polar& p, cplx v, int prod) {
    const bool by_value = !p.th_exact;
    const unsigned long long key = by_value ? value_key(v) : (unsigned long long)__double_as_longlong(p.th);
    const unsigned rs = (unsigned)s.ph_rs, base = (unsigned)prod * rs;
    unsigned h0 = hash64(key ^ 0x9e3779b97f4a7c15ull) & (rs - 1);
    for (int probe = 0; probe < 64; ++probe) {
        const unsigned h = base + h0;
        unsigned long long cur = s.ph_key[h];
        bool mine = false;
        if (cur == EMPTY) {
            cur = atomicCAS(&s.ph_key[h], EMPTY, key);
            if (cur == EMPTY) { atomicAdd(&s.ph_count, 1); cur = key; mine = true; }
        }
        if (cur == key) {
            if (by_value) {
                for (;;) {
                    while (atomicCAS(&s.ph_lock[h], 0, 1) != 0) {}
                    const double sre = *(volatile double*)&s.ph_re[h], sim = *(volatile double*)&s.ph_im[h];
                    int verdict;   // 1: this value, 0: another value (collision), -1: owner not done
                    if (mine) {
                        s.ph_ux[h] = p.ux; s.ph_uy[h] = p.uy; s.ph_re[h] = v.re; s.ph_im[h] = v.im;
                        verdict = 1;
                    } else if (sre != sre) {
                        verdict = -1;
                    } else {
                        verdict = (sre == v.re && sim == v.im) ? 1 : 0;
                    }
                    __threadfence_block();
                    atomicExch(&s.ph_lock[h], 0);
                    if (verdict == 1) return;
                    if (verdict == 0) break;
                }
            } else {
                // keep the lexicographically smallest (ux, uy) per exact theta (codec.py:144-148);
                // the stored ux only decreases, so a strictly larger ux can never win
                if (p.ux > *(volatile double*)&s.ph_ux[h]) return;
                while (atomicCAS(&s.ph_lock[h], 0, 1) != 0) {}
                if (lex_less(p.ux, p.uy, s.ph_ux[h], s.ph_uy[h])) {
                    s.ph_ux[h] = p.ux; s.ph_uy[h] = p.uy; s.ph_re[h] = v.re; s.ph_im[h] = v.im;
                }
                __threadfence_block();
                atomicExch(&s.ph_lock[h], 0);
                return;
            }
        }
        h0 = (h0 + 1) & (rs - 1);
    }
    global_phase(out, p, v, prod);
}

__device__ void sets_clear(CtaSets& s, int regions) {
    for (int i = threadIdx.x; i < MAG_SLOTS; i += blockDim.x) s.mag_key[i] = EMPTY;
    for (int i = threadIdx.x; i < PH_SLOTS; i += blockDim.x) {
        s.ph_key[i] = EMPTY; s.ph_ux[i] = 1e300; s.ph_uy[i] = 1e300; s.ph_lock[i] = 0;
        s.ph_re[i] = __longlong_as_double(0x7ff8000000000000ll);   // NaN: value slot not written yet
        s.ph_im[i] = 0.0;
    }
    if (threadIdx.x == 0) {
        s.mag_count = 0; s.ph_count = 0; s.full = 0;
        s.mag_rs = MAG_SLOTS / regions; s.ph_rs = PH_SLOTS / regions;
    }
}

__device__ void sets_flush(CtaSets& s, ByteCand* out) {
    for (int i = threadIdx.x; i < MAG_SLOTS; i += blockDim.x) {
        if (s.mag_key[i] == EMPTY) continue;
        const unsigned long long slot = atomicAdd(&out->n_mag, 1ull);
        if (slot < out->cap_mag) {
            out->mag[slot] = __longlong_as_double((long long)s.mag_key[i]);
            out->mag_tag[slot] = i / s.mag_rs;
        } else {
            out->overflow = 1;
        }
    }
    for (int i = threadIdx.x; i < PH_SLOTS; i += blockDim.x) {
        if (s.ph_key[i] == EMPTY) continue;
        const unsigned long long slot = atomicAdd(&out->n_ph, 1ull);
        if (slot < out->cap_ph) {
            out->ph[4 * slot + 0] = s.ph_re[i];
            out->ph[4 * slot + 1] = s.ph_im[i];
            out->ph[4 * slot + 2] = s.ph_ux[i];
            out->ph[4 * slot + 3] = s.ph_uy[i];
            out->ph_tag[slot] = i / s.ph_rs;
        } else {
            out->overflow = 1;
        }
    }
}

// producer rank of a work item in the reference's exchange choreography
// producer rank of a work item in the reference's exchange choreography, from the
// item's LOGICAL index (the remap planner may have permuted physical qubits):
// logical bit (n_local - 2 + j) lives at physical bit lbit[j] of phys_base | i0
__device__ __forceinline__ int producer_of(const ByteGate& g, uint64_t i0) {
    const uint64_t full = g.phys_base | i0;
    auto lb = [&](int j) -> int { return (int)((full >> g.lbit[j]) & 1ull); };
    int rank = 0;
    for (int j = 0; j < g.rank_bits; ++j) rank |= lb(2 + j) << j;
    const int top1 = g.n_local >= 1 ? lb(1) : 0;    // logical bit n_local - 1
    const int top2 = g.n_local >= 2 ? lb(0) : 0;    // logical bit n_local - 2
    switch (g.xkind) {
        case 1:     // pairwise, single-qubit gate on a global qubit: low side computes offsets [0, L/2)
            return top1 ? (rank | (int)g.xmask_a) : (rank & ~(int)g.xmask_a);
        case 2: {   // pairwise, two-qubit gate with one global qubit (engine.py:278-323)
            const int side = g.qlow_top ? top2 : top1;
            return side ? (rank | (int)g.xmask_a) : (rank & ~(int)g.xmask_a);
        }
        case 3: {   // quad: the rank at position p computes quarter p
            const int pos = (top1 << 1) | top2;
            const int base = rank & ~(int)(g.xmask_a | g.xmask_b);
            return base | ((pos & 1) ? (int)g.xmask_a : 0) | ((pos & 2) ? (int)g.xmask_b : 0);
        }
        default:
            return rank;
    }
}

// exact numpy complex abs (codec.py:41 via np.abs)
__device__ __forceinline__ double exact_abs(cplx v) {
    const double ax = fabs(v.re), ay = fabs(v.im);
    const double L = fmax(ax, ay), S = fmin(ax, ay);
    if (L == 0.0) return 0.0;
    const double q = __ddiv_rn(S, L);
    return __dmul_rn(L, __dsqrt_rn(__fma_rn(q, q, 1.0)));
}

// theta as canonicalize computes it; exact on the axes
__device__ __forceinline__ double theta_of(cplx v, bool* exact, bool* wrap_unsure) {
    double a;
    *exact = true;
    if (v.im == 0.0) {
        a = v.re > 0.0 ? 0.0 : (signbit(v.im) ? -3.141592653589793 : 3.141592653589793);
    } else if (v.re == 0.0) {
        a = v.im > 0.0 ? 1.5707963267948966 : -1.5707963267948966;
    } else {
        a = atan2(v.im, v.re);
        *exact = false;
    }
    double th = (a == 0.0) ? 0.0 : (a < 0.0 ? __dadd_rn(a, TWO_PI) : a);
    const double gap = __dsub_rn(TWO_PI, th);
    if (gap < PHASE_ATOL) th = 0.0;
    *wrap_unsure = !*exact && fabs(gap - PHASE_ATOL) <= TH_MARGIN;
    return th;
}

constexpr double SQ_EPS = 1e-13;      // relative margin on |v|^2 decisions (fast path)

struct ThreadCache {                  // last values seen by this thread
    double mre, mim, pre, pim;        // last magnitude / phase candidate
    double cre, cim;                  // last encoded value ...
    unsigned ccode;                   // ... and its (certain) code
    int prod;                         // producer region the remembered candidates belong to
};

struct Emitter {
    const STables& t;
    const ByteGate& g;
    CtaSets& sets;
    ByteCand* cand;
    uint8_t* mo;
    uint8_t* po;
    bool collect;
    bool write;

    __device__ void unsure_push(uint64_t idx, cplx v) const {
        const unsigned long long slot = atomicAdd(&cand->n_unsure, 1ull);
        if (slot < cand->cap_unsure) {   // n_unsure > cap_unsure is reported by svb_unsure
            cand->unsure_idx[slot] = idx;
            cand->unsure_val[2 * slot] = v.re;
            cand->unsure_val[2 * slot + 1] = v.im;
        }
    }

    __device__ __forceinline__ void emit(uint64_t idx, cplx v, ThreadCache& tc, int prod = 0) const {
        const unsigned c = code(idx, v, tc, nullptr, prod);
        if (write) {
            mo[idx] = (uint8_t)(c & 255);
            if (po) po[idx] = (uint8_t)(c >> 8);   // null: phase plane stays all zero (see svb_gate)
        }
    }

    // (magnitude index | phase index << 8) of a produced value; candidate and
    // uncertain-phase bookkeeping as a side effect
    __device__ __forceinline__ unsigned code(uint64_t idx, cplx v, ThreadCache& tc, bool* sure = nullptr,
                                             int prod = 0) const {
        if (sure) *sure = true;
        if (collect && prod != tc.prod) {   // candidates are remembered per producer region
            tc.mre = tc.mim = tc.pre = tc.pim = tc.cre = tc.cim = NAN;
            tc.prod = prod;
        }
        if (v.re == 0.0 && v.im == 0.0) return 0u;   // r == 0: indices (0, 0), always representable
        // structured states repeat values: reuse the last certain code (candidates of an
        // identical value were already recorded)
        if (v.re == tc.cre && v.im == tc.cim) return tc.ccode;
        const double x2 = __fma_rn(v.re, v.re, __dmul_rn(v.im, v.im));
        // ---- magnitude: nearest sorted entry from squared midpoints (branch-free search over the
        //      +inf-padded table); exact |v| only near a boundary
        bool slow = !(x2 > 1e-280);
        int k = 0;
        for (int step = t.search_top; step > 0; step >>= 1)
            k += (t.sqmid[k + step - 1] < x2) ? step : 0;
        if (k > 0 && x2 - t.sqmid[k - 1] <= SQ_EPS * x2) slow = true;
        if (k < t.n_mag - 1 && t.sqmid[k] - x2 <= SQ_EPS * x2) slow = true;
        // representability by the nearest entry: |r - m| <= 1e-12 max(r, m)  <=>  |x2 - m^2| ~ 2e-12 m^2
        const double m2 = t.sqmag[k];
        const double dd = fabs(x2 - m2);
        int mag_rep = (dd < 1.98e-12 * m2) ? 1 : ((dd > 2.02e-12 * m2) ? 0 : -1);
        if (m2 == 0.0) mag_rep = 0;
        double r = 0.0;
        bool have_r = false;
        int mi;
        if (slow) {
            r = exact_abs(v);
            have_r = true;
            bool dummy = false;
            mi = nearest(t.smag, t.smag_idx, t.n_mag, r, false, 0.0, &dummy);
            mag_rep = representable(t.smag, t.n_mag, r, true, 0.0);
        } else {
            mi = t.smag_idx[k];
            if (mag_rep < 0) {
                r = exact_abs(v);
                have_r = true;
                mag_rep = representable(t.smag, t.n_mag, r, true, 0.0);
            }
        }
        // ---- phase: a single-entry table needs no angle to encode
        bool th_exact = true, wrap_unsure = false, have_th = false;
        double th = 0.0;
        int pi = 0;
        bool unsure = false;
        if (t.n_ph > 1 && mi != 0) {
            th = theta_of(v, &th_exact, &wrap_unsure);
            have_th = true;
            unsure = wrap_unsure;
            pi = nearest(t.sth, t.sth_idx, t.n_ph, th, true, th_exact ? 0.0 : TH_MARGIN, &unsure);
        }
        if (mi == 0) pi = 0;
        if (write && unsure && mi != 0) unsure_push(idx, v);
        const unsigned result = (unsigned)mi | ((unsigned)pi << 8);
        if (!unsure) { tc.cre = v.re; tc.cim = v.im; tc.ccode = result; }
        if (sure) *sure = !unsure;
        if (!collect) return result;
        if (g.want_mag && mag_rep == 0 && !(v.re == tc.mre && v.im == tc.mim)) {
            if (!have_r) r = exact_abs(v);
            if (r < g.mag_cut) {
                cand->any_mag = 1;
                insert_mag(sets, cand, r, prod);
            }
            tc.mre = v.re; tc.mim = v.im;
        }
        if (g.want_ph && !(v.re == tc.pre && v.im == tc.pim)) {
            if (!have_th) th = theta_of(v, &th_exact, &wrap_unsure);
            if (th < g.ph_cut && representable(t.sth, t.n_ph, th, false, th_exact ? 0.0 : TH_MARGIN) != 1) {
                if (!have_r) { r = exact_abs(v); have_r = true; }
                Polar p;
                p.r = r; p.th = th; p.th_exact = th_exact; p.wrap_unsure = wrap_unsure;
                p.ux = __dadd_rn(__ddiv_rn(v.re, r), 0.0);
                p.uy = __dadd_rn(__ddiv_rn(v.im, r), 0.0);
                insert_phase(sets, cand, p, v, prod);
            }
            tc.pre = v.re; tc.pim = v.im;
        }
        return result;
    }
};

// ---- per-CTA memo of input codes -> output codes -------------------------------------
// Within one pass the tables are fixed, so the output codes of a work item are a pure
// function of its input codes: (m0, p0, m1, p1) -> (code0, code1) for a 1Q pair,
// (m, p) -> code for a diagonal factor.  Structured states repeat a handful of code
// tuples, so most items are one shared-memory probe instead of decode + gate +
// canonicalise + table search.  An entry is key << 32 | value in one 64-bit word,
// published with a single CAS; only results without an uncertain phase are stored
// (uncertain amplitudes must reach the host per index), and candidate collection
// already happened when the tuple was first computed in this CTA.
constexpr int MEMO_SLOTS = 2048;
constexpr unsigned MEMO_NOKEY = 0xffffffffu;          // never stored (all-255 tuple)

__device__ __forceinline__ unsigned memo_hash(unsigned k) {   // Fibonacci hashing, top 11 bits
    return (k * 0x9e3779b1u) >> (32 - 11);
}
static_assert(MEMO_SLOTS == 2048, "memo_hash yields 11 bits");
// returns the slot of the entry, -1 if absent
__device__ __forceinline__ int memo_get(const unsigned long long* memo, unsigned key, unsigned* val) {
    unsigned h = memo_hash(key);
#pragma unroll
    for (int probe = 0; probe < 4; ++probe) {
        const unsigned long long e = memo[h];
        if (e == ~0ull) return -1;
        if ((unsigned)(e >> 32) == key) { *val = (unsigned)e; return (int)h; }
        h = (h + 1) & (MEMO_SLOTS - 1);
    }
    return -1;
}
__device__ __forceinline__ int memo_put(unsigned long long* memo, unsigned key, unsigned val) {
    if (key == MEMO_NOKEY) return -1;
    const unsigned long long e = ((unsigned long long)key << 32) | val;
    unsigned h = memo_hash(key);
#pragma unroll
    for (int probe = 0; probe < 4; ++probe) {
        const unsigned long long prev = atomicCAS(&memo[h], ~0ull, e);
        if (prev == ~0ull || (unsigned)(prev >> 32) == key) return (int)h;
        h = (h + 1) & (MEMO_SLOTS - 1);
    }
    return -1;
}
// tagged collection: which producer regions already recorded the candidates of a
// memo entry (a hit for a new producer still takes the slow path once)
struct MemoTags {
    unsigned* seen;         // MEMO_SLOTS bit masks, nullptr when not tagging
    __device__ __forceinline__ bool fresh(int slot, int prod) const {
        return seen && !((seen[slot] >> prod) & 1u);
    }
    __device__ __forceinline__ void mark(int slot, int prod) const {
        if (seen && slot >= 0) atomicOr(&seen[slot], 1u << prod);
    }
};

__device__ __forceinline__ void load8(const uint8_t* p, uint8_t (&b)[8]) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) { b[i] = (w.x >> (8 * i)) & 255; b[4 + i] = (w.y >> (8 * i)) & 255; }
}
__device__ __forceinline__ void store8(uint8_t* p, const uint8_t (&b)[8]) {
    uint2 w;
    w.x = b[0] | (b[1] << 8) | (b[2] << 16) | ((unsigned)b[3] << 24);
    w.y = b[4] | (b[5] << 8) | (b[6] << 16) | ((unsigned)b[7] << 24);
    *reinterpret_cast<uint2*>(p) = w;
}

__device__ void load_tables(STables& t, const ByteTables* gt) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        t.dmag[i] = gt->dmag[i]; t.dux[i] = gt->dux[i]; t.duy[i] = gt->duy[i];
        t.smag[i] = gt->smag[i]; t.sth[i] = gt->sth[i];
        t.smag_idx[i] = gt->smag_idx[i]; t.sth_idx[i] = gt->sth_idx[i];
        t.sqmid[i] = gt->sqmid[i]; t.sqmag[i] = gt->sqmag[i];
    }
    if (threadIdx.x == 0) {
        t.n_mag = gt->n_mag;
        t.n_ph = gt->n_ph;
        int top = 0;                       // smallest power of two with 2*top >= n_mag
        while (2 * top < gt->n_mag) top = top ? 2 * top : 1;
        t.search_top = top;
    }
}
}  // namespace

// memo miss of a 1Q pair: decode, gate, encode both outputs, remember the tuple
__device__ __noinline__ unsigned pair_slow(const STables& t, const Emitter& em, ThreadCache& tc,
                                           unsigned long long* memo, const MemoTags& mt, unsigned key,
                                           uint64_t i0, uint64_t i1, const double* m, bool real, int prod) {
    const cplx a0 = decode(t, key & 255u, (key >> 8) & 255u), a1 = decode(t, (key >> 16) & 255u, key >> 24);
    cplx r0, r1;
    if (real) {   // numpy's +-0 imaginary products dropped (exact up to the sign of zero)
        r0 = {__dadd_rn(__dmul_rn(m[0], a0.re), __dmul_rn(m[2], a1.re)),
              __dadd_rn(__dmul_rn(m[0], a0.im), __dmul_rn(m[2], a1.im))};
        r1 = {__dadd_rn(__dmul_rn(m[4], a0.re), __dmul_rn(m[6], a1.re)),
              __dadd_rn(__dmul_rn(m[4], a0.im), __dmul_rn(m[6], a1.im))};
    } else {
        r0 = row2({m[0], m[1]}, {m[2], m[3]}, a0, a1);
        r1 = row2({m[4], m[5]}, {m[6], m[7]}, a0, a1);
    }
    bool s0, s1;
    const unsigned c0 = em.code(i0, r0, tc, &s0, prod), c1 = em.code(i1, r1, tc, &s1, prod);
    const unsigned cc = c0 | (c1 << 16);
    if (s0 && s1) mt.mark(memo_put(memo, key, cc), prod);
    return cc;
}

// phase plane access: a null plane is known all zero (svb_gate: a one-entry phase table
// throughout the state's history) -- reads return zeros, writes are skipped
__device__ __forceinline__ uint4 ld16z(const uint8_t* p, uint64_t off) {
    return p ? *reinterpret_cast<const uint4*>(p + off) : make_uint4(0u, 0u, 0u, 0u);
}
// L2 prefetch of a work item several grid strides ahead: the passes hold one item per
// thread in registers (one ahead), too few bytes in flight to cover the HBM latency on
// their own (scan passes read 32 bytes per item); the prefetched lines turn the
// register loads into L2 hits.  No registers, no shared memory.
constexpr int kL2Ahead = 4;
// x with a bit inserted at every position of `holes` (ascending), valued by `vals`: maps a
// compact work-item index to its index when the bits under `holes` are fixed (a support)
__device__ __forceinline__ uint64_t expand_bits(uint64_t x, uint64_t holes, uint64_t vals) {
    for (uint64_t h = holes; h; h &= h - 1) {
        const int b = __ffsll((long long)h) - 1;
        x = ((x >> b) << (b + 1)) | (x & ((1ull << b) - 1ull)) | (((vals >> b) & 1ull) << b);
    }
    return x;
}
// warp-cooperative per-pair path (k_byte_gate, 1Q on qubits >= 4) when at most this many
// lanes of a warp hold mixed items; more, and every lane walks its own item
constexpr int kCoopMaxItems = 12;
// dominant-tuple path of the 1Q passes (items that are not one tuple): at most this many
// exception pairs per 16-pair item
constexpr int kMaxExceptions = 4;
__device__ __forceinline__ void l2_prefetch(const uint8_t* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// 1Q gate on a low qubit (qa < 4): both amplitudes of every pair lie in the same
// 32-byte block of each plane, so a work item is one block (16 pairs) read and
// written with 16-byte accesses -- the per-pair byte path issued 8 one-byte
// accesses per pair (H on qubits 0-3: 22.6 ms per pass at N=32, 2.8 ms for qa >= 4).
template <int QA>
__device__ __forceinline__ void byte_low_pairs(const uint8_t* __restrict__ mi_in, const uint8_t* __restrict__ pi_in,
                                               uint8_t* __restrict__ mi_out, uint8_t* __restrict__ pi_out,
                                               const ByteGate& g, const STables& t, const Emitter& em,
                                               ThreadCache& tc, unsigned long long* memo, const MemoTags& mt,
                                               bool real, bool tagged, bool write, uint64_t first, uint64_t step) {
    // support: only the blocks whose fixed bits (>= 5) read sup_val
    const uint64_t fixb = g.sup_fixed & ~31ull, valb = g.sup_val & fixb;
    const uint64_t n_blocks = (g.n_elems >> 5) >> __popcll(fixb);
    auto block_at = [&](uint64_t w) { return fixb ? expand_bits(w << 5, fixb, valb) : (w << 5); };
    // the next block's bytes are loaded before the current one is computed (latency)
    uint4 nm0 = {0, 0, 0, 0}, nm1 = nm0, np0 = nm0, np1 = nm0;
    if (first < n_blocks) {
        const uint64_t b = block_at(first);
        nm0 = *reinterpret_cast<const uint4*>(mi_in + b);
        nm1 = *reinterpret_cast<const uint4*>(mi_in + b + 16);
        np0 = ld16z(pi_in, b);
        np1 = ld16z(pi_in, b + 16);
    }
    for (uint64_t w = first; w < n_blocks; w += step) {
        const uint64_t b = block_at(w);
        const uint4 m0 = nm0, m1 = nm1, p0 = np0, p1 = np1;
        if (w + kL2Ahead * step < n_blocks) {
            const uint64_t bp = block_at(w + kL2Ahead * step);
            l2_prefetch(mi_in + bp);
            if (pi_in) l2_prefetch(pi_in + bp);
        }
        if (w + step < n_blocks) {
            const uint64_t bn = block_at(w + step);
            nm0 = *reinterpret_cast<const uint4*>(mi_in + bn);
            nm1 = *reinterpret_cast<const uint4*>(mi_in + bn + 16);
            np0 = ld16z(pi_in, bn);
            np1 = ld16z(pi_in, bn + 16);
        }
        // all 32 amplitudes of a block share their producer (the caller checked the bits)
        if (g.producer >= 0 && producer_of(g, b) != g.producer) continue;
        const int prod = tagged ? producer_of(g, b) : 0;
        unsigned m[8], p[8], om[8], op[8];
        m[0] = m0.x; m[1] = m0.y; m[2] = m0.z; m[3] = m0.w; m[4] = m1.x; m[5] = m1.y; m[6] = m1.z; m[7] = m1.w;
        p[0] = p0.x; p[1] = p0.y; p[2] = p0.z; p[3] = p0.w; p[4] = p1.x; p[5] = p1.y; p[6] = p1.z; p[7] = p1.w;
        bool uni = m[0] == (m[0] & 255u) * 0x01010101u && p[0] == (p[0] & 255u) * 0x01010101u;
#pragma unroll
        for (int k = 1; k < 8; ++k) uni = uni && m[k] == m[0] && p[k] == p[0];
        bool done = false;
        if (uni) {   // one code tuple for all 16 pairs (structured states)
            const unsigned bm = m[0] & 255u, bp = p[0] & 255u;
            const unsigned key = bm | (bp << 8) | (bm << 16) | (bp << 24);
            unsigned cc;
            const int slot = memo_get(memo, key, &cc);
            done = true;
            if (slot < 0 || mt.fresh(slot, prod)) {
                cc = pair_slow(t, em, tc, memo, mt, key, b, b + (1u << QA), g.m, real, prod);
                done = memo_get(memo, key, &cc) >= 0;   // uncertain outputs: per pair (indices reported)
            }
            if (done) {
#pragma unroll
                for (int k = 0; k < 8; ++k) { om[k] = 0u; op[k] = 0u; }
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const bool hi = (k >> QA) & 1;
                    om[k >> 2] |= (hi ? (cc >> 16) & 255u : cc & 255u) << (8 * (k & 3));
                    op[k >> 2] |= (hi ? cc >> 24 : (cc >> 8) & 255u) << (8 * (k & 3));
                }
            }
        }
        if (!done) {
#pragma unroll
            for (int k = 0; k < 8; ++k) { om[k] = 0u; op[k] = 0u; }
            bool hit_prev = false;   // runs of equal tuples: as in k_byte_gate's per-pair loop
            unsigned key_prev = 0u, cc_prev = 0u;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int k0 = ((j >> QA) << (QA + 1)) | (j & ((1 << QA) - 1)), k1 = k0 | (1 << QA);
                const unsigned key = ((m[k0 >> 2] >> (8 * (k0 & 3))) & 255u) |
                                     (((p[k0 >> 2] >> (8 * (k0 & 3))) & 255u) << 8) |
                                     (((m[k1 >> 2] >> (8 * (k1 & 3))) & 255u) << 16) |
                                     (((p[k1 >> 2] >> (8 * (k1 & 3))) & 255u) << 24);
                unsigned cc;
                if (hit_prev && key == key_prev) {
                    cc = cc_prev;
                } else {
                    const int slot = memo_get(memo, key, &cc);
                    hit_prev = slot >= 0 && !mt.fresh(slot, prod);
                    if (!hit_prev) cc = pair_slow(t, em, tc, memo, mt, key, b + k0, b + k1, g.m, real, prod);
                    key_prev = key;
                    cc_prev = cc;
                }
                om[k0 >> 2] |= (cc & 255u) << (8 * (k0 & 3));
                op[k0 >> 2] |= ((cc >> 8) & 255u) << (8 * (k0 & 3));
                om[k1 >> 2] |= ((cc >> 16) & 255u) << (8 * (k1 & 3));
                op[k1 >> 2] |= (cc >> 24) << (8 * (k1 & 3));
            }
        }
        if (write) {
            *reinterpret_cast<uint4*>(mi_out + b) = make_uint4(om[0], om[1], om[2], om[3]);
            *reinterpret_cast<uint4*>(mi_out + b + 16) = make_uint4(om[4], om[5], om[6], om[7]);
            if (pi_out) {
                *reinterpret_cast<uint4*>(pi_out + b) = make_uint4(op[0], op[1], op[2], op[3]);
                *reinterpret_cast<uint4*>(pi_out + b + 16) = make_uint4(op[4], op[5], op[6], op[7]);
            }
        }
    }
}

// One BYTE gate pass.  Work items: pairs (1Q), quadruples (2Q) or single
// amplitudes (DIAG, and COPY for untouched amplitudes of a diagonal gate).
template <int LOWQA>   // >= 0: a 1Q gate on low qubit LOWQA, 32-byte blocks (byte_low_pairs)
__global__ void __launch_bounds__(NT, 2) k_byte_gate(const uint8_t* __restrict__ mi_in, const uint8_t* __restrict__ pi_in,
                                                  uint8_t* __restrict__ mi_out, uint8_t* __restrict__ pi_out,
                                                  const ByteTables* __restrict__ gtab, const __grid_constant__ ByteGate g,
                                                  ByteCand* cand) {
    __shared__ STables t;
    __shared__ CtaSets sets;
    extern __shared__ unsigned long long memo[];          // MEMO_SLOTS entries + MEMO_SLOTS tag masks
    unsigned* memo_seen = reinterpret_cast<unsigned*>(memo + MEMO_SLOTS);
    load_tables(t, gtab);
    const bool collect = g.collect != 0;
    // producer == -2: every work item, candidates tagged with the item's reference producer
    // rank (one set region per rank) -- one pass instead of one pass per rank
    const bool tagged = g.producer == -2;
    if (collect) sets_clear(sets, tagged ? (1 << g.rank_bits) : 1);
    for (int i = threadIdx.x; i < MEMO_SLOTS; i += blockDim.x) { memo[i] = ~0ull; memo_seen[i] = 0u; }
    __syncthreads();
    const bool write = g.scan_only == 0;
    const Emitter em{t, g, sets, cand, mi_out, pi_out, collect, write};
    const MemoTags mt{(tagged && collect) ? memo_seen : nullptr};
    ThreadCache tc{NAN, NAN, NAN, NAN, NAN, NAN, 0u, 0};
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t first = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // lowest physical bit the producer rule reads: a vector work item (a run of
    // consecutive amplitudes) has one producer only if its index bits stay below it
    int lmin = 64;
    if (g.producer >= 0 || tagged)
        for (int j = 0; j < 2 + g.rank_bits && j < 12; ++j) lmin = min(lmin, (int)g.lbit[j]);
    if constexpr (LOWQA >= 0) {
        const bool real = g.m[1] == 0.0 && g.m[3] == 0.0 && g.m[5] == 0.0 && g.m[7] == 0.0;
        byte_low_pairs<LOWQA>(mi_in, pi_in, mi_out, pi_out, g, t, em, tc, memo, mt, real, tagged, write, first, step);
    } else if (g.kind == SV_OP_1Q) {
        const cplx m0 = {g.m[0], g.m[1]}, m1 = {g.m[2], g.m[3]}, m2 = {g.m[4], g.m[5]}, m3 = {g.m[6], g.m[7]};
        const bool real = g.m[1] == 0.0 && g.m[3] == 0.0 && g.m[5] == 0.0 && g.m[7] == 0.0;
        const uint64_t n_items = g.n_elems >> 1;
        if (g.qa >= 4 && g.n_elems >= 32 && lmin >= 4) {
            // 16 consecutive pairs per work item (16-byte loads/stores of every plane); the next
            // item's bytes are loaded before the current one is computed (latency hiding).
            // The loop is warp-uniform: items whose 16 pairs are not one code tuple (or whose
            // tuple is new to the CTA) take the per-pair path, and when a few lanes of a warp
            // have such items the whole warp works on them together, one pair per lane
            // (16 lanes per item).  Otherwise one mixed item kept 31 idle lanes waiting for
            // 16 sequential pairs (Hadamard benchmark, H on qubit 9 at N=32: 1 item in 32
            // mixed, 64 % of the warps diverged, ~470 instructions per warp-iteration).
            // support: only the items whose fixed bits (>= 4, not qa) read sup_val
            const uint64_t fixi = g.sup_fixed & ~15ull & ~(1ull << g.qa), vali = g.sup_val & fixi;
            const uint64_t n_chunks = (n_items >> 4) >> __popcll(fixi);
            auto item_i0 = [&](uint64_t w) {
                return fixi ? expand_bits(w << 4, fixi | (1ull << g.qa), vali) : insert0(w << 4, g.qa);
            };
            const uint64_t off = 1ull << g.qa;
            const int lane = threadIdx.x & 31;
            uint4 nxt[4];
            auto fetch = [&](uint64_t w, uint4 (&b)[4]) {
                const uint64_t i0 = item_i0(w);
                b[0] = *reinterpret_cast<const uint4*>(mi_in + i0);
                b[1] = ld16z(pi_in, i0);
                b[2] = *reinterpret_cast<const uint4*>(mi_in + i0 + off);
                b[3] = ld16z(pi_in, i0 + off);
            };
            auto byte_of = [](const uint4& v, int j) -> unsigned {
                const unsigned w = j < 4 ? v.x : (j < 8 ? v.y : (j < 12 ? v.z : v.w));
                return (w >> (8 * (j & 3))) & 255u;
            };
            auto put_byte = [](uint4& v, int j, unsigned b) {
                const unsigned sh = 8 * (j & 3);
                if (j < 4) v.x |= b << sh; else if (j < 8) v.y |= b << sh;
                else if (j < 12) v.z |= b << sh; else v.w |= b << sh;
            };
            // uniform run: all 16 pairs carry the same code tuple (structured states, e.g. the
            // Hadamard benchmark) -> one lookup, replicated output bytes
            auto uniform = [](const uint4& v) {
                return v.x == v.y && v.x == v.z && v.x == v.w && v.x == (v.x & 255u) * 0x01010101u;
            };
            // one dominant code tuple (pair 15's) and at most kMaxExceptions pairs with other
            // tuples: the dominant outputs are replicated and the exceptions patched in (the
            // Hadamard benchmark's late stages: one nonzero pair per item).  false: the item
            // takes the per-pair path (too many exceptions, or an uncertain dominant result)
            auto dominant_item = [&](const uint4 (&c)[4], uint64_t a0, uint64_t a1, int pr) -> bool {
                const unsigned key = byte_of(c[0], 15) | (byte_of(c[1], 15) << 8) | (byte_of(c[2], 15) << 16) |
                                     (byte_of(c[3], 15) << 24);
                const unsigned r0 = (key & 255u) * 0x01010101u, r1 = ((key >> 8) & 255u) * 0x01010101u;
                const unsigned r2 = ((key >> 16) & 255u) * 0x01010101u, r3 = (key >> 24) * 0x01010101u;
                auto pack4 = [](unsigned x) {   // top bit of each byte -> 4 bits
                    return ((x >> 7) & 1u) | ((x >> 14) & 2u) | ((x >> 21) & 4u) | ((x >> 28) & 8u);
                };
                const unsigned ex =
                    pack4(__vcmpne4(c[0].x, r0) | __vcmpne4(c[1].x, r1) | __vcmpne4(c[2].x, r2) | __vcmpne4(c[3].x, r3)) |
                    (pack4(__vcmpne4(c[0].y, r0) | __vcmpne4(c[1].y, r1) | __vcmpne4(c[2].y, r2) | __vcmpne4(c[3].y, r3)) << 4) |
                    (pack4(__vcmpne4(c[0].z, r0) | __vcmpne4(c[1].z, r1) | __vcmpne4(c[2].z, r2) | __vcmpne4(c[3].z, r3)) << 8) |
                    (pack4(__vcmpne4(c[0].w, r0) | __vcmpne4(c[1].w, r1) | __vcmpne4(c[2].w, r2) | __vcmpne4(c[3].w, r3)) << 12);
                if (__popc(ex) > kMaxExceptions) return false;
                unsigned cc;
                const int slot = memo_get(memo, key, &cc);
                if (slot < 0 || mt.fresh(slot, pr)) {
                    cc = pair_slow(t, em, tc, memo, mt, key, a0 + 15, a1 + 15, g.m, real, pr);
                    if (memo_get(memo, key, &cc) < 0) return false;   // uncertain: per pair, per index
                }
                const unsigned b0 = (cc & 255u) * 0x01010101u, b1 = ((cc >> 8) & 255u) * 0x01010101u;
                const unsigned b2 = ((cc >> 16) & 255u) * 0x01010101u, b3 = (cc >> 24) * 0x01010101u;
                uint4 o0 = make_uint4(b0, b0, b0, b0), o1 = make_uint4(b1, b1, b1, b1);
                uint4 o2 = make_uint4(b2, b2, b2, b2), o3 = make_uint4(b3, b3, b3, b3);
                for (unsigned e = ex; e; e &= e - 1) {
                    const int j = __ffs(e) - 1;
                    const unsigned sh = 8 * (j & 3);
                    auto wsel = [&](const uint4& v) { return j < 4 ? v.x : (j < 8 ? v.y : (j < 12 ? v.z : v.w)); };
                    const unsigned kj = ((wsel(c[0]) >> sh) & 255u) | (((wsel(c[1]) >> sh) & 255u) << 8) |
                                        (((wsel(c[2]) >> sh) & 255u) << 16) | (((wsel(c[3]) >> sh) & 255u) << 24);
                    unsigned cj;
                    const int sj = memo_get(memo, kj, &cj);
                    if (sj < 0 || mt.fresh(sj, pr)) cj = pair_slow(t, em, tc, memo, mt, kj, a0 + j, a1 + j, g.m, real, pr);
                    auto patch = [&](uint4& v, unsigned b) {
                        const unsigned msk = ~(255u << sh), val = b << sh;
                        if (j < 4) v.x = (v.x & msk) | val;
                        else if (j < 8) v.y = (v.y & msk) | val;
                        else if (j < 12) v.z = (v.z & msk) | val;
                        else v.w = (v.w & msk) | val;
                    };
                    patch(o0, cj & 255u);
                    patch(o1, (cj >> 8) & 255u);
                    patch(o2, (cj >> 16) & 255u);
                    patch(o3, cj >> 24);
                }
                if (write) {
                    *reinterpret_cast<uint4*>(mi_out + a0) = o0;
                    if (pi_out) *reinterpret_cast<uint4*>(pi_out + a0) = o1;
                    *reinterpret_cast<uint4*>(mi_out + a1) = o2;
                    if (pi_out) *reinterpret_cast<uint4*>(pi_out + a1) = o3;
                }
                return true;
            };
            uint64_t w = first;
            if (w < n_chunks) fetch(w, nxt);
            for (; __any_sync(0xffffffffu, w < n_chunks); w += step) {
                const bool inb = w < n_chunks;
                uint4 cur[4] = {nxt[0], nxt[1], nxt[2], nxt[3]};
                if (w + step < n_chunks) fetch(w + step, nxt);
                if (w + kL2Ahead * step < n_chunks) {
                    const uint64_t ip = item_i0(w + kL2Ahead * step);
                    l2_prefetch(mi_in + ip);
                    l2_prefetch(mi_in + ip + off);
                    if (pi_in) { l2_prefetch(pi_in + ip); l2_prefetch(pi_in + ip + off); }
                }
                const uint64_t i0 = inb ? item_i0(w) : 0ull, i1 = i0 + off;
                const bool valid = inb && !(g.producer >= 0 && producer_of(g, i0) != g.producer);
                const int prod = (tagged && valid) ? producer_of(g, i0) : 0;
                bool slow = false;
                if (valid) {
                    if (uniform(cur[0]) && uniform(cur[1]) && uniform(cur[2]) && uniform(cur[3])) {
                        const unsigned key = (cur[0].x & 255u) | ((cur[1].x & 255u) << 8) |
                                             ((cur[2].x & 255u) << 16) | ((cur[3].x & 255u) << 24);
                        unsigned cc;
                        const int slot = memo_get(memo, key, &cc);
                        bool have = slot >= 0 && !mt.fresh(slot, prod);
                        if (!have) {
                            cc = pair_slow(t, em, tc, memo, mt, key, i0, i1, g.m, real, prod);
                            // uncertain amplitudes are reported per index: take the per-pair path
                            have = memo_get(memo, key, &cc) >= 0;
                        }
                        if (have && write) {
                            const unsigned b0 = (cc & 255u) * 0x01010101u, b1 = ((cc >> 8) & 255u) * 0x01010101u;
                            const unsigned b2 = ((cc >> 16) & 255u) * 0x01010101u, b3 = (cc >> 24) * 0x01010101u;
                            *reinterpret_cast<uint4*>(mi_out + i0) = make_uint4(b0, b0, b0, b0);
                            if (pi_out) *reinterpret_cast<uint4*>(pi_out + i0) = make_uint4(b1, b1, b1, b1);
                            *reinterpret_cast<uint4*>(mi_out + i1) = make_uint4(b2, b2, b2, b2);
                            if (pi_out) *reinterpret_cast<uint4*>(pi_out + i1) = make_uint4(b3, b3, b3, b3);
                        }
                        slow = !have;
                    } else {
                        slow = !dominant_item(cur, i0, i1, prod);
                    }
                }
                unsigned mm = __ballot_sync(0xffffffffu, slow);
                if (!mm) continue;
                if (__popc(mm) <= kCoopMaxItems) {
                    // cooperative: two mixed items per round, pair j of item a on lane j, of item b
                    // on lane 16 + j; outputs as byte stores (16 lanes fill one 16-byte run)
                    const int j = lane & 15;
                    while (mm) {
                        const int la = __ffs(mm) - 1;
                        mm &= mm - 1;
                        int lb = -1;
                        if (mm) {
                            lb = __ffs(mm) - 1;
                            mm &= mm - 1;
                        }
                        const int src = lane < 16 ? la : (lb >= 0 ? lb : la);
                        const bool act = lane < 16 || lb >= 0;
                        const uint64_t s_i0 = __shfl_sync(0xffffffffu, i0, src);
                        const int s_prod = __shfl_sync(0xffffffffu, prod, src);
                        unsigned wv[4];
#pragma unroll
                        for (int pl = 0; pl < 4; ++pl) {
                            const unsigned x = __shfl_sync(0xffffffffu, cur[pl].x, src);
                            const unsigned y = __shfl_sync(0xffffffffu, cur[pl].y, src);
                            const unsigned z = __shfl_sync(0xffffffffu, cur[pl].z, src);
                            const unsigned v = __shfl_sync(0xffffffffu, cur[pl].w, src);
                            wv[pl] = j < 4 ? x : (j < 8 ? y : (j < 12 ? z : v));
                        }
                        if (act) {
                            const unsigned sh = 8 * (j & 3);
                            const unsigned key = ((wv[0] >> sh) & 255u) | (((wv[1] >> sh) & 255u) << 8) |
                                                 (((wv[2] >> sh) & 255u) << 16) | (((wv[3] >> sh) & 255u) << 24);
                            unsigned cc;
                            const int slot = memo_get(memo, key, &cc);
                            if (slot < 0 || mt.fresh(slot, s_prod))
                                cc = pair_slow(t, em, tc, memo, mt, key, s_i0 + j, s_i0 + off + j, g.m, real, s_prod);
                            if (write) {
                                mi_out[s_i0 + j] = (uint8_t)(cc & 255u);
                                mi_out[s_i0 + off + j] = (uint8_t)((cc >> 16) & 255u);
                                if (pi_out) {
                                    pi_out[s_i0 + j] = (uint8_t)((cc >> 8) & 255u);
                                    pi_out[s_i0 + off + j] = (uint8_t)(cc >> 24);
                                }
                            }
                        }
                    }
                    continue;
                }
                if (!slow) continue;
                // many mixed items in the warp: every lane walks its own 16 pairs; runs of equal
                // tuples (sparse / structured states) reuse the previous memo hit; a pair
                // computed by pair_slow is looked up again (its outputs may be uncertain,
                // reported per index)
                uint4 out[4] = {{0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}};
                bool hit_prev = false;
                unsigned key_prev = 0u, cc_prev = 0u;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    // key = (m0, p0, m1, p1) bytes of pair jj; jj is a literal after unrolling
                    const unsigned key = byte_of(cur[0], jj) | (byte_of(cur[1], jj) << 8) |
                                         (byte_of(cur[2], jj) << 16) | (byte_of(cur[3], jj) << 24);
                    unsigned cc;
                    if (hit_prev && key == key_prev) {
                        cc = cc_prev;   // what the memo returns for it (entries are never evicted)
                    } else {
                        const int slot = memo_get(memo, key, &cc);
                        hit_prev = slot >= 0 && !mt.fresh(slot, prod);
                        if (!hit_prev) cc = pair_slow(t, em, tc, memo, mt, key, i0 + jj, i1 + jj, g.m, real, prod);
                        key_prev = key;
                        cc_prev = cc;
                    }
                    put_byte(out[0], jj, cc & 255u); put_byte(out[1], jj, (cc >> 8) & 255u);
                    put_byte(out[2], jj, (cc >> 16) & 255u); put_byte(out[3], jj, cc >> 24);
                }
                if (write) {
                    *reinterpret_cast<uint4*>(mi_out + i0) = out[0];
                    if (pi_out) *reinterpret_cast<uint4*>(pi_out + i0) = out[1];
                    *reinterpret_cast<uint4*>(mi_out + i1) = out[2];
                    if (pi_out) *reinterpret_cast<uint4*>(pi_out + i1) = out[3];
                }
            }
        } else
        for (uint64_t w = first; w < n_items; w += step) {
            const uint64_t i0 = insert0(w, g.qa), i1 = i0 | (1ull << g.qa);
            if (g.producer >= 0 && producer_of(g, i0) != g.producer) continue;
            const int prod = tagged ? producer_of(g, i0) : 0;
            const unsigned bm0 = mi_in[i0], bp0 = pi_in ? pi_in[i0] : 0u, bm1 = mi_in[i1], bp1 = pi_in ? pi_in[i1] : 0u;
            const unsigned key = bm0 | (bp0 << 8) | (bm1 << 16) | (bp1 << 24);
            unsigned cc;
            const int slot = memo_get(memo, key, &cc);
            if (slot < 0 || mt.fresh(slot, prod)) {
                const cplx a0 = decode(t, bm0, bp0), a1 = decode(t, bm1, bp1);
                cplx r0, r1;
                if (real) {   // numpy's +-0 imaginary products dropped (exact up to the sign of zero)
                    r0 = {__dadd_rn(__dmul_rn(m0.re, a0.re), __dmul_rn(m1.re, a1.re)),
                          __dadd_rn(__dmul_rn(m0.re, a0.im), __dmul_rn(m1.re, a1.im))};
                    r1 = {__dadd_rn(__dmul_rn(m2.re, a0.re), __dmul_rn(m3.re, a1.re)),
                          __dadd_rn(__dmul_rn(m2.re, a0.im), __dmul_rn(m3.re, a1.im))};
                } else {
                    r0 = row2(m0, m1, a0, a1);
                    r1 = row2(m2, m3, a0, a1);
                }
                bool s0, s1;
                const unsigned c0 = em.code(i0, r0, tc, &s0, prod), c1 = em.code(i1, r1, tc, &s1, prod);
                cc = c0 | (c1 << 16);
                if (s0 && s1) mt.mark(memo_put(memo, key, cc), prod);
            }
            if (write) {
                mi_out[i0] = (uint8_t)(cc & 255u);
                mi_out[i1] = (uint8_t)((cc >> 16) & 255u);
                if (pi_out) { pi_out[i0] = (uint8_t)((cc >> 8) & 255u); pi_out[i1] = (uint8_t)(cc >> 24); }
            }
        }
    } else if (g.kind == SV_OP_2Q) {
        cplx m[16];
        for (int i = 0; i < 16; ++i) m[i] = {g.m[2 * i], g.m[2 * i + 1]};
        const int lo = min(g.qa, g.qb), hi = max(g.qa, g.qb);
        const uint64_t n_items = g.n_elems >> 2;
        for (uint64_t w = first; w < n_items; w += step) {
            const uint64_t e = insert0(insert0(w, lo), hi);
            if (g.producer >= 0 && producer_of(g, e) != g.producer) continue;
            const int prod = tagged ? producer_of(g, e) : 0;
            const uint64_t idx[4] = {e, e | (1ull << g.qa), e | (1ull << g.qb), e | (1ull << g.qa) | (1ull << g.qb)};
            cplx a[4];
            for (int c = 0; c < 4; ++c) a[c] = decode(t, mi_in[idx[c]], pi_in ? pi_in[idx[c]] : 0u);
            cplx o[4];
            for (int r = 0; r < 4; ++r) o[r] = row4(&m[4 * r], a[0], a[1], a[2], a[3]);
            for (int r = 0; r < 4; ++r) em.emit(idx[r], o[r], tc, prod);
        }
    } else if (g.n_elems >= 16 && lmin >= 3) {   // DIAG, 8 amplitudes per work item
        const cplx f = {g.m[0], g.m[1]};
        // in place: visit only the chunks whose index bits >= 3 match the mask
        const uint64_t hmask = g.in_place ? ((g.mask & ~7ull) >> 3) : 0ull;
        const uint64_t n_chunks = (g.in_place && (g.mask & ~(g.n_elems - 1ull))) ? 0ull   // selects nothing
                                  : ((g.n_elems >> 3) >> __popcll(hmask));
        for (uint64_t w = first; w < n_chunks; w += step) {
            uint64_t c = w;
            for (uint64_t m = hmask; m; m &= m - 1) {   // insert a 1 at every mask position
                const int b = __ffsll((long long)m) - 1;
                c = ((c >> b) << (b + 1)) | (1ull << b) | (c & ((1ull << b) - 1ull));
            }
            const uint64_t i = c << 3;
            // the 8 amplitudes of a chunk share their producer (bits >= 3 decide it)
            const int pr = (g.producer >= 0 || tagged) ? producer_of(g, i) : 0;
            if (g.producer >= 0 && pr != g.producer) continue;
            const int prod = tagged ? pr : 0;
            if (((i | 7ull) & g.mask) != g.mask) {           // no amplitude of the chunk is active
                if (write) {
                    *reinterpret_cast<uint2*>(mi_out + i) = *reinterpret_cast<const uint2*>(mi_in + i);
                    if (pi_out) *reinterpret_cast<uint2*>(pi_out + i) = pi_in ? *reinterpret_cast<const uint2*>(pi_in + i)
                                                                             : make_uint2(0u, 0u);
                }
                continue;
            }
            uint8_t bm[8], bp[8];
            load8(mi_in + i, bm);
            if (pi_in) load8(pi_in + i, bp);
            else
#pragma unroll
                for (int j = 0; j < 8; ++j) bp[j] = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (((i + j) & g.mask) != g.mask) continue;
                const unsigned key = bm[j] | ((unsigned)bp[j] << 8);
                unsigned c;
                const int slot = memo_get(memo, key, &c);
                if (slot < 0 || mt.fresh(slot, prod)) {
                    bool sure;
                    c = em.code(i + j, cmul(decode(t, bm[j], bp[j]), f), tc, &sure, prod);
                    if (sure) mt.mark(memo_put(memo, key, c), prod);
                }
                bm[j] = c & 255;
                bp[j] = c >> 8;
            }
            if (write) {
                store8(mi_out + i, bm);
                if (pi_out) store8(pi_out + i, bp);
            }
        }
    } else {   // DIAG: masked amplitudes re-encoded, the rest copied
        const cplx f = {g.m[0], g.m[1]};
        for (uint64_t i = first; i < g.n_elems; i += step) {
            const int pr = (g.producer >= 0 || tagged) ? producer_of(g, i) : 0;
            if ((i & g.mask) == g.mask) {
                if (g.producer >= 0 && pr != g.producer) continue;
                em.emit(i, cmul(decode(t, mi_in[i], pi_in ? pi_in[i] : 0u), f), tc, tagged ? pr : 0);
            } else if (write && !g.in_place && (g.producer < 0 || pr == g.producer)) {
                mi_out[i] = mi_in[i];
                if (pi_out) pi_out[i] = pi_in ? pi_in[i] : 0u;
            }
        }
    }
    if (collect) {
        __syncthreads();
        sets_flush(sets, cand);
    }
}

// ---- diagonal write passes with fixed tables: a 65536-entry code table ---------------
// A diagonal gate maps every amplitude by its own code alone: (m, p) -> code of
// decode(m, p) * f.  When the pass collects no candidates (tables saturated, or
// scanned and merged first) the whole map is evaluated once, with the same encoder
// as the per-amplitude path, and the pass becomes a table lookup per selected
// amplitude.  Entries whose phase decision is uncertain are flagged (bit 16): those
// amplitudes are recomputed per index so they reach the host as before.
__device__ CtaSets g_no_sets;   // never touched: the table passes collect nothing

constexpr unsigned kDiagUnsure = 0xff00u;   // table entry: recompute per index (a code with
                                            // magnitude index 0 always has phase index 0)
__global__ void __launch_bounds__(NT) k_byte_diag_table(const ByteTables* __restrict__ gtab,
                                                        const __grid_constant__ ByteGate g, uint16_t* lut) {
    __shared__ STables t;
    load_tables(t, gtab);
    __syncthreads();
    const Emitter em{t, g, g_no_sets, nullptr, nullptr, nullptr, false, false};
    ThreadCache tc{NAN, NAN, NAN, NAN, NAN, NAN, 0u, 0};
    const unsigned key = blockIdx.x * NT + threadIdx.x;   // m | p << 8
    if (key >= 65536u) return;
    const cplx f = {g.m[0], g.m[1]};
    bool sure = true;
    const unsigned c = em.code(0, cmul(decode(t, key & 255u, key >> 8), f), tc, &sure, 0);
    lut[key] = (uint16_t)(sure ? c : kDiagUnsure);
}

// The pass itself: a table lookup per selected amplitude.  Collecting passes
// (speculative encode, or scan) also record which (code, producer) pairs occur, in
// a per-CTA bitmap merged into `seen`; k_byte_diag_collect then proposes the
// candidates of exactly those codes (candidate sets are sets: the order in which
// values are offered does not matter).
// SCAN: record the occurring (code, producer) pairs only.  Otherwise: rewrite the
// selected amplitudes through the table, staged in shared memory (128 KB, one
// 1024-thread CTA per SM); a collecting write pass does both.
constexpr int NTD = 1024;
template <bool SCAN>
__global__ void __launch_bounds__(NTD) k_byte_diag_apply(
    const uint8_t* mi_in, const uint8_t* pi_in, uint8_t* mi_out, uint8_t* pi_out, const ByteTables* __restrict__ gtab,
    const __grid_constant__ ByteGate g, ByteCand* cand, const uint16_t* __restrict__ lut, uint32_t* seen, int nprod) {
    constexpr int NTK = NTD;   // one CTA per SM: one bitmap flush per SM (atomics on 2048 shared words)
    __shared__ STables t;
    extern __shared__ __align__(16) unsigned char dsm[];
    uint16_t* slut = reinterpret_cast<uint16_t*>(dsm);                            // !SCAN: 65536 codes
    uint32_t* bits = reinterpret_cast<uint32_t*>(dsm + (SCAN ? 0 : 65536 * 2));   // collect: nprod x 2048
    const bool collect = seen != nullptr, tagged = g.producer == -2;
    constexpr bool write = !SCAN;
    if (collect)
        for (int k = threadIdx.x; k < nprod * 2048; k += NTK) bits[k] = 0u;
    if constexpr (!SCAN)
        for (int k = threadIdx.x; k < 65536 / 8; k += NTK)
            reinterpret_cast<uint4*>(slut)[k] = reinterpret_cast<const uint4*>(lut)[k];
    load_tables(t, gtab);
    __syncthreads();
    const Emitter em{t, g, g_no_sets, cand, mi_out, pi_out, false, write};
    ThreadCache tc{NAN, NAN, NAN, NAN, NAN, NAN, 0u, 0};
    const cplx f = {g.m[0], g.m[1]};
    const uint64_t step = (uint64_t)gridDim.x * NTK;
    const uint64_t first = (uint64_t)blockIdx.x * NTK + threadIdx.x;
    // chunks of 16 amplitudes (16-byte loads of each plane, the next chunk's loads issued
    // before the current one is processed); in place or scanning, only the chunks whose
    // index bits >= 4 match the mask are visited
    const bool sparse = g.in_place || !write;
    // chunk index bits (>= 4) that are fixed: the mask's (sparse passes: value 1) and the
    // support's (value sup_val); a mask bit the support fixes to 0 selects nothing
    const uint64_t hmask_i = sparse ? (g.mask & ~15ull) : 0ull;
    const uint64_t fix_i = g.sup_fixed & ~15ull, holes = hmask_i | fix_i;
    const uint64_t hvals = hmask_i | (g.sup_val & fix_i & ~hmask_i);
    const bool empty = sparse && (hmask_i & fix_i & ~g.sup_val);
    const uint64_t n_chunks = ((g.mask & ~(g.n_elems - 1ull)) && sparse) || empty
                                  ? 0ull
                                  : ((g.n_elems >> 4) >> __popcll(holes));
    auto chunk_at = [&](uint64_t w) { return expand_bits(w << 4, holes, hvals); };
    uint64_t w = first, inx = 0;
    uint4 nm = {0, 0, 0, 0}, np = {0, 0, 0, 0};
    const unsigned lowm = (unsigned)(g.mask & 15ull);   // selected chunk positions: j & lowm == lowm
    unsigned last_tag = 0xffffffffu;                       // scan: last (key, producer) marked
    unsigned last_key = 0xffffffffu, last_code = 0u;       // write: last key and its table code
    if (w < n_chunks) {
        inx = chunk_at(w);
        nm = *reinterpret_cast<const uint4*>(mi_in + inx);
        np = ld16z(pi_in, inx);
    }
    for (; w < n_chunks; w += step) {
        const uint64_t i = inx;
        const uint4 cm = nm, cpv = np;
        if (w + step < n_chunks) {
            inx = chunk_at(w + step);
            nm = *reinterpret_cast<const uint4*>(mi_in + inx);
            np = ld16z(pi_in, inx);
        }

        if (((i | 15ull) & g.mask) != g.mask) {   // out of place: untouched chunk copied
            if (write) {
                *reinterpret_cast<uint4*>(mi_out + i) = cm;
                if (pi_out) *reinterpret_cast<uint4*>(pi_out + i) = cpv;
            }
            continue;
        }
        // the 16 amplitudes of a chunk share their producer (the caller checked the bits)
        const int prod = tagged ? producer_of(g, i) : 0;
        unsigned mw[4] = {cm.x, cm.y, cm.z, cm.w}, pw[4] = {cpv.x, cpv.y, cpv.z, cpv.w};
        // The passes are issue-bound (ncu: 84 % issue active, 28 / 41 instructions per
        // selected amplitude for scan / write): the selection test uses the mask's low
        // bits only (the chunk's bits >= 4 match it), a key is one byte permute of the two
        // plane words, a code goes back with one permute, and the scan skips the bitmap
        // for a (key, producer) it has just marked.
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if ((j & lowm) != lowm) continue;
            const int wj = j >> 2, bj = j & 3;
            const unsigned key = __byte_perm(mw[wj], pw[wj], (unsigned)(bj | ((4 + bj) << 4))) & 0xffffu;
            if (collect) {
                const unsigned tag = key | ((unsigned)prod << 16);
                if (tag != last_tag) {
                    last_tag = tag;
                    uint32_t* wd = bits + prod * 2048 + (key >> 5);
                    if (!((*wd >> (key & 31)) & 1u)) atomicOr(wd, 1u << (key & 31));
                }
            }
            if constexpr (!SCAN) {
                unsigned code;
                if (key == last_key) {
                    code = last_code;   // never an uncertain entry (those are not cached)
                } else {
                    code = slut[key];
                    if (code == kDiagUnsure) {   // reports i + j
                        code = em.code(i + j, cmul(decode(t, key & 255u, key >> 8), f), tc);
                    } else {
                        last_key = key;
                        last_code = code;
                    }
                }
                // byte bj of the word <- byte 0 of the code part (selector nibble 4 = y.byte0)
                constexpr unsigned kIns[4] = {0x3214u, 0x3240u, 0x3410u, 0x4210u};
                mw[wj] = __byte_perm(mw[wj], code & 255u, kIns[bj]);
                pw[wj] = __byte_perm(pw[wj], code >> 8, kIns[bj]);
            }
        }
        if (write) {
            *reinterpret_cast<uint4*>(mi_out + i) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
            if (pi_out) *reinterpret_cast<uint4*>(pi_out + i) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
        }
    }
    if (collect) {
        __syncthreads();
        for (int k = threadIdx.x; k < nprod * 2048; k += NTK)
            if (bits[k]) atomicOr(seen + k, bits[k]);
    }
}

// candidates of the codes a collecting table pass saw, per producer region
__global__ void __launch_bounds__(NT) k_byte_diag_collect(const ByteTables* __restrict__ gtab,
                                                          const __grid_constant__ ByteGate g, ByteCand* cand,
                                                          const uint32_t* __restrict__ seen, int nprod) {
    __shared__ STables t;
    __shared__ CtaSets sets;
    load_tables(t, gtab);
    sets_clear(sets, g.producer == -2 ? nprod : 1);
    __syncthreads();
    const Emitter em{t, g, sets, cand, nullptr, nullptr, true, false};
    ThreadCache tc{NAN, NAN, NAN, NAN, NAN, NAN, 0u, 0};
    const cplx f = {g.m[0], g.m[1]};
    for (unsigned key = blockIdx.x * NT + threadIdx.x; key < 65536u; key += gridDim.x * NT)
        for (int pr = 0; pr < nprod; ++pr)
            if ((seen[pr * 2048 + (key >> 5)] >> (key & 31)) & 1u)
                em.code(0, cmul(decode(t, key & 255u, key >> 8), f), tc, nullptr, pr);
    __syncthreads();
    sets_flush(sets, cand);
}

// Decode into complex128 (export, host mirrors, measurement of small states).
__global__ void k_byte_decode(const uint8_t* __restrict__ mi, const uint8_t* __restrict__ pi, const ByteTables* gtab,
                              double* __restrict__ out, uint64_t n) {
    __shared__ STables t;
    load_tables(t, gtab);
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const cplx v = decode(t, mi[i], pi[i]);
        out[2 * i] = v.re;
        out[2 * i + 1] = v.im;
    }
}

// Encode complex128 values (Codebook.encode on device) with the same uncertain-
// theta reporting as the gate pass; optionally collect proposals (Codebook.propose).
__global__ void __launch_bounds__(NT) k_byte_encode(const double* __restrict__ vals, uint64_t n, const ByteTables* gtab,
                                                    uint8_t* __restrict__ mi, uint8_t* __restrict__ pi,
                                                    const __grid_constant__ ByteGate g, ByteCand* cand) {
    __shared__ STables t;
    __shared__ CtaSets sets;
    load_tables(t, gtab);
    const bool collect = g.collect != 0;
    if (collect) sets_clear(sets, 1);
    __syncthreads();
    const Emitter em{t, g, sets, cand, mi, pi, collect, true};
    ThreadCache tc{NAN, NAN, NAN, NAN, NAN, NAN, 0u, 0};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        em.emit(i, {vals[2 * i], vals[2 * i + 1]}, tc);
    if (collect) {
        __syncthreads();
        sets_flush(sets, cand);
    }
}

__global__ void k_byte_patch(uint8_t* mi, uint8_t* pi, const uint64_t* idx, const uint8_t* nm, const uint8_t* np_,
                             uint64_t n) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        mi[idx[k]] = nm[k];
        pi[idx[k]] = np_[k];
    }
}

// global<->local qubit swap of BYTE planes with the partner rank (see sv_dist.cu)
__global__ void k_byte_swap_peer(uint8_t* omi, uint8_t* opi, uint8_t* pmi, uint8_t* ppi, uint64_t t0, uint64_t n,
                                 int l, int c) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n; w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = t0 + w;
        const uint64_t low = t & ((1ull << l) - 1ull);
        const uint64_t x = ((t >> l) << (l + 1)) | ((uint64_t)(1 - c) << l) | low;
        const uint64_t y = ((t >> l) << (l + 1)) | ((uint64_t)c << l) | low;
        const uint8_t a = omi[x], b = opi[x];
        omi[x] = pmi[y];
        opi[x] = ppi[y];
        pmi[y] = a;
        ppi[y] = b;
    }
}

// vectorised: 16 consecutive rest indices per item (l >= 4)
__global__ void k_byte_swap_peer16(uint8_t* omi, uint8_t* opi, uint8_t* pmi, uint8_t* ppi, uint64_t t0, uint64_t n16,
                                   int l, int c) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n16;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = t0 + (w << 4);
        const uint64_t low = t & ((1ull << l) - 1ull);
        const uint64_t x = ((t >> l) << (l + 1)) | ((uint64_t)(1 - c) << l) | low;
        const uint64_t y = ((t >> l) << (l + 1)) | ((uint64_t)c << l) | low;
        const uint4 a = *reinterpret_cast<const uint4*>(omi + x), b = *reinterpret_cast<const uint4*>(opi + x);
        const uint4 pa = *reinterpret_cast<const uint4*>(pmi + y), pb = *reinterpret_cast<const uint4*>(ppi + y);
        *reinterpret_cast<uint4*>(omi + x) = pa;
        *reinterpret_cast<uint4*>(opi + x) = pb;
        *reinterpret_cast<uint4*>(pmi + y) = a;
        *reinterpret_cast<uint4*>(ppi + y) = b;
    }
}

// batched remap of k global qubits (see k_swap_group in sv_dist.cu): 16 rest
// indices per item when the lowest victim bit is >= 4
template <int W>
__global__ void k_byte_swap_group(uint8_t* omi, uint8_t* opi, uint8_t* pmi, uint8_t* ppi, uint64_t t0, uint64_t n,
                                  uint64_t vmask, uint64_t own_pat, uint64_t peer_pat) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n; w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t base = insert_zeros(t0 + w * W, vmask);
        const uint64_t x = base | own_pat, y = base | peer_pat;
        if constexpr (W == 16) {
            const uint4 a = *reinterpret_cast<const uint4*>(omi + x), b = *reinterpret_cast<const uint4*>(opi + x);
            const uint4 pa = *reinterpret_cast<const uint4*>(pmi + y), pb = *reinterpret_cast<const uint4*>(ppi + y);
            *reinterpret_cast<uint4*>(omi + x) = pa;
            *reinterpret_cast<uint4*>(opi + x) = pb;
            *reinterpret_cast<uint4*>(pmi + y) = a;
            *reinterpret_cast<uint4*>(ppi + y) = b;
        } else {
            const uint8_t a = omi[x], b = opi[x];
            omi[x] = pmi[y];
            opi[x] = ppi[y];
            pmi[y] = a;
            ppi[y] = b;
        }
    }
}

// sum conj(decode(a)) * decode(b) over count elements (a / b may be peer planes)
__global__ void k_byte_pair_dot(const uint8_t* ami, const uint8_t* api, const uint8_t* bmi, const uint8_t* bpi,
                                const ByteTables* gtab, uint64_t n, double* partials) {
    __shared__ STables t;
    load_tables(t, gtab);
    __syncthreads();
    double re = 0.0, im = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const cplx x = decode(t, ami[i], api[i]), y = decode(t, bmi[i], bpi[i]);
        re += x.re * y.re + x.im * y.im;
        im += x.re * y.im - x.im * y.re;
    }
    __shared__ double sr[8], si[8];
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

// scratch of the diagonal table passes, one per stream (a stream-ordered allocation per
// pass released its pool memory at every synchronisation: ~2 ms of host time per pass)
static cudaError_t diag_scratch(cudaStream_t st, unsigned char** out) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, unsigned char*>& cache =
        *new std::map<std::pair<int, cudaStream_t>, unsigned char*>;   // leaked: freed with the context
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, st});
    if (it != cache.end()) {
        *out = it->second;
        return cudaSuccess;
    }
    unsigned char* p = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p), 65536 * 2 + 2048 * 8 * 4);
    if (e != cudaSuccess) return e;
    cache[{dev, st}] = p;
    *out = p;
    return cudaSuccess;
}

static bool diag_table_enabled() {   // SVB200_BYTE_DIAG_TABLE=0: per-amplitude memo path
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("SVB200_BYTE_DIAG_TABLE");
        v = (e && std::atoi(e) == 0) ? 0 : 1;
    }
    return v == 1;
}

static unsigned byte_grid(uint64_t items) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t cap = (uint64_t)sm_count(dev) * 4;
    const uint64_t want = (items + NT - 1) / NT;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, cap));
}

// Kernel attributes of the gate passes, once per device.  The attribute call also loads the
// kernels' module (CUDA lazy loading), so svb_create calls this: a state's first gate then
// pays no module load (first BYTE pass of a process 7.7 -> 1.5 ms at N=32).
cudaError_t byte_kernels_prepare() {
    static bool configured[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64 || configured[dev]) return cudaSuccess;
    const int memo_bytes = MEMO_SLOTS * (int)(sizeof(unsigned long long) + sizeof(unsigned));
    void (*low[4])(const uint8_t*, const uint8_t*, uint8_t*, uint8_t*, const ByteTables*, const ByteGate, ByteCand*) = {
        k_byte_gate<0>, k_byte_gate<1>, k_byte_gate<2>, k_byte_gate<3>};
    cudaError_t e = cudaFuncSetAttribute(k_byte_gate<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, memo_bytes);
    for (int q = 0; q < 4 && e == cudaSuccess; ++q)
        e = cudaFuncSetAttribute(low[q], cudaFuncAttributeMaxDynamicSharedMemorySize, memo_bytes);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_byte_diag_apply<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * 8 * 4);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_byte_diag_apply<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 65536 * 2 + 2048 * 8 * 4);
    if (e == cudaSuccess) configured[dev] = true;
    return e;
}

cudaError_t launch_byte_gate(const uint8_t* mi_in, const uint8_t* pi_in, uint8_t* mi_out, uint8_t* pi_out,
                             const ByteTables* tab, const ByteGate& g, ByteCand* cand, cudaStream_t st) {
    const uint64_t items = g.kind == SV_OP_1Q ? g.n_elems / 2 : (g.kind == SV_OP_2Q ? g.n_elems / 4 : g.n_elems);
    int dev = 0;
    cudaGetDevice(&dev);
    const int memo_bytes = MEMO_SLOTS * (int)(sizeof(unsigned long long) + sizeof(unsigned));
    void (*low[4])(const uint8_t*, const uint8_t*, uint8_t*, uint8_t*, const ByteTables*, const ByteGate, ByteCand*) = {
        k_byte_gate<0>, k_byte_gate<1>, k_byte_gate<2>, k_byte_gate<3>};
    if (cudaError_t e = byte_kernels_prepare()) return e;
    // low-qubit 1Q gates: 32-byte blocks, if a block has one producer (the bits the
    // producer rule reads are all >= 5; k_byte_gate computes the same bound)
    int lmin = 64;
    if (g.producer >= 0 || g.producer == -2)
        for (int j = 0; j < 2 + g.rank_bits && j < 12; ++j) lmin = std::min(lmin, (int)g.lbit[j]);
    // diagonal gates through the 65536-entry code table (write passes, and collecting
    // passes of the whole buffer or tagged by producer when a chunk has one producer)
    const bool tagged = g.producer == -2;
    if (g.kind == SV_OP_DIAG && g.n_elems >= 4096 && diag_table_enabled() &&
        (g.producer == -1 || (tagged && lmin >= 4 && g.rank_bits <= 3)) && (g.collect || !g.scan_only)) {
        const int nprod = tagged ? (1 << g.rank_bits) : 1;
        unsigned char* scratch = nullptr;   // 65536 uint16 codes, then nprod x 2048 seen words
        cudaError_t e = diag_scratch(st, &scratch);
        if (e != cudaSuccess) return e;
        uint16_t* lut = reinterpret_cast<uint16_t*>(scratch);
        uint32_t* seen = g.collect ? reinterpret_cast<uint32_t*>(scratch + 65536 * 2) : nullptr;
        if (seen) cudaMemsetAsync(seen, 0, 2048 * nprod * sizeof(uint32_t), st);
        const uint64_t chunks = g.n_elems >> 4;
        const size_t bm_bytes = seen ? 2048 * nprod * sizeof(uint32_t) : 0;
        const unsigned grid1 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((chunks + NTD - 1) / NTD,
                                                                                  (uint64_t)sm_count(dev)));
        if (g.scan_only) {
            k_byte_diag_apply<true><<<grid1, NTD, bm_bytes, st>>>(mi_in, pi_in, mi_out, pi_out, tab, g, cand, lut,
                                                                   seen, nprod);
        } else {
            k_byte_diag_table<<<65536 / NT, NT, 0, st>>>(tab, g, lut);
            count_launch();
            const size_t smem = 65536 * 2 + bm_bytes;
            const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((chunks + NTD - 1) / NTD,
                                                                                     (uint64_t)sm_count(dev)));
            k_byte_diag_apply<false><<<grid, NTD, smem, st>>>(mi_in, pi_in, mi_out, pi_out, tab, g, cand, lut, seen,
                                                              nprod);
        }
        count_launch();
        if (seen) {
            k_byte_diag_collect<<<64, NT, 0, st>>>(tab, g, cand, seen, nprod);
            count_launch();
        }
        return cudaGetLastError();
    }
    if (g.kind == SV_OP_1Q && g.qa < 4 && g.n_elems >= 1024 && lmin >= 5)
        low[g.qa]<<<byte_grid(g.n_elems / 32), NT, memo_bytes, st>>>(mi_in, pi_in, mi_out, pi_out, tab, g, cand);
    else
        k_byte_gate<-1><<<byte_grid(items), NT, memo_bytes, st>>>(mi_in, pi_in, mi_out, pi_out, tab, g, cand);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_byte_decode(const uint8_t* mi, const uint8_t* pi, const ByteTables* tab, double* out, uint64_t n,
                               cudaStream_t st) {
    k_byte_decode<<<byte_grid(n), NT, 0, st>>>(mi, pi, tab, out, n);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_byte_encode(const double* vals, uint64_t n, const ByteTables* tab, uint8_t* mi, uint8_t* pi,
                               const ByteGate& g, ByteCand* cand, cudaStream_t st) {
    k_byte_encode<<<byte_grid(n), NT, 0, st>>>(vals, n, tab, mi, pi, g, cand);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_byte_swap_peer(uint8_t* omi, uint8_t* opi, uint8_t* pmi, uint8_t* ppi, uint64_t n_local_elems,
                                  int l, int c, cudaStream_t st) {
    const uint64_t quarter = n_local_elems / 4;
    const uint64_t t0 = (uint64_t)c * quarter;
    if (l >= 4 && quarter % 16 == 0) {
        k_byte_swap_peer16<<<byte_grid(quarter / 16), NT, 0, st>>>(omi, opi, pmi, ppi, t0, quarter / 16, l, c);
    } else {
        k_byte_swap_peer<<<byte_grid(quarter), NT, 0, st>>>(omi, opi, pmi, ppi, t0, quarter, l, c);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_byte_swap_group(uint8_t* omi, uint8_t* opi, uint8_t* pmi, uint8_t* ppi, uint64_t t0, uint64_t n,
                                   uint64_t vmask, uint64_t own_pat, uint64_t peer_pat, cudaStream_t st) {
    if ((vmask & 15ull) == 0 && t0 % 16 == 0 && n % 16 == 0)
        k_byte_swap_group<16><<<byte_grid(n / 16), NT, 0, st>>>(omi, opi, pmi, ppi, t0, n / 16, vmask, own_pat,
                                                                peer_pat);
    else
        k_byte_swap_group<1><<<byte_grid(n), NT, 0, st>>>(omi, opi, pmi, ppi, t0, n, vmask, own_pat, peer_pat);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_byte_pair_dot(const uint8_t* ami, const uint8_t* api, const uint8_t* bmi, const uint8_t* bpi,
                                 const ByteTables* tab, uint64_t n, double* partials, int grid, cudaStream_t st) {
    k_byte_pair_dot<<<grid, NT, 0, st>>>(ami, api, bmi, bpi, tab, n, partials);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_byte_patch(uint8_t* mi, uint8_t* pi, const uint64_t* idx, const uint8_t* nm, const uint8_t* np_,
                              uint64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_byte_patch<<<byte_grid(n), NT, 0, st>>>(mi, pi, idx, nm, np_, n);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sv
