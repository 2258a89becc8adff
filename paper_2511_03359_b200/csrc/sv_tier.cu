// Two-tier state (HBM + pinned host memory) executor: svsim/tier.py made physical.
//
// The reference models the paper's strategy 5 (explicit copies steered by a
// look-ahead over the gates) as a staging plan plus counters
// (tier.py:98-208).  Here the plan runs: the 2^n amplitudes are cut into chunks
// of 2^c; chunk g lives in HBM when fast[g] != 0 (TierAccount.fast_resident),
// otherwise in pinned host memory, and is staged through `slots` HBM chunk
// slots by the copy engines:
//   * run group (gates on qubits < c, or diagonal): every chunk gets the
//     group's fused passes once -- fast chunks in place, slow chunks through a
//     slot ring: H2D (copy stream 1) -> passes (compute stream) -> D2H (copy
//     stream 2), three stages in flight, so both PCIe directions and the
//     compute overlap (the reference charges 2 x slow bytes; that is exactly
//     what crosses the link);
//   * pairing gate (a non-diagonal gate with a qubit >= c: tier.py "mid" and
//     "exchange" groups): chunk groups (j, j|m0[, j|m1, j|m0|m1]) are co-staged
//     and updated by the two/four-buffer kernels (k_pair, k_quad, k_pair2q);
//   * measure-all: each slow chunk is staged in once for its own sums; the
//     cross terms of the chunk-index qubits pair it with its partners -- an HBM
//     chunk, or a slow partner read in place over the link (zero-copy, the
//     pinned host memory is device-mapped).
// Arithmetic is the same kernels' on the same amplitudes, so results equal the
// untiered run bit for bit.  Physical link bytes and copies are counted.
#include <sys/mman.h>

#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "sv_common.cuh"
#include "sv_kernels.cuh"
#include "svb200.h"

namespace sv {
int capi_fail(int code, const char* msg);
int capi_cuda_fail(cudaError_t e, const char* what);
}  // namespace sv

using sv::capi_cuda_fail;
using sv::capi_fail;
using sv::launch_pair;
using sv::launch_pair2q;
using sv::launch_quad;

struct sv_tier {
    int device = 0, n = 0, c = 0, mode = SV_FP64, n_slots = 0;
    size_t ebytes = 16;
    uint64_t chunk_elems = 0, n_chunks = 0;
    std::vector<uint8_t> fast;      // per chunk
    std::vector<void*> ptr;         // HBM pointer (fast) or pinned host pointer (slow)
    std::vector<uint8_t> zero;      // slow chunk known to be all zeros (never staged out yet)
    std::vector<uint8_t> registered;   // slow chunk: mmap'd + cudaHostRegister'ed (else cudaHostAlloc)
    void* fast_arena = nullptr;     // fast chunks, contiguous
    size_t fast_bytes = 0;
    void* slot_arena = nullptr;     // staging slots, contiguous
    std::vector<cudaEvent_t> ev_in, ev_done, ev_free;
    std::vector<cudaEvent_t> ev_host;   // per chunk: its last copy back to host memory has landed
    int next_slot = 0;
    cudaStream_t comp = nullptr, h2d = nullptr, d2h = nullptr;
    uint64_t h2d_bytes = 0, d2h_bytes = 0, h2d_copies = 0, d2h_copies = 0, zc_bytes = 0, memsets = 0, passes = 0;
};

namespace {

struct Guard {
    int prev = 0;
    explicit Guard(int d) {
        cudaGetDevice(&prev);
        cudaSetDevice(d);
    }
    ~Guard() { cudaSetDevice(prev); }
};

#define TTRY(expr, what)                                     \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return capi_cuda_fail(_e, what); \
    } while (0)

size_t chunk_bytes(const sv_tier* h) { return h->chunk_elems * h->ebytes; }
void* slot_ptr(const sv_tier* h, int s) { return static_cast<char*>(h->slot_arena) + (size_t)s * chunk_bytes(h); }

// take the next slot of the ring; the H2D stream waits until its previous occupant
// has been copied back
int acquire_slot(sv_tier* h) {
    const int s = h->next_slot;
    h->next_slot = (h->next_slot + 1) % h->n_slots;
    cudaStreamWaitEvent(h->h2d, h->ev_free[s], 0);
    return s;
}

// stage chunk g into slot s on the H2D stream (a never-written slow chunk is a memset);
// the copy waits for the chunk's previous copy back to host memory
cudaError_t stage_in(sv_tier* h, uint64_t g, int s) {
    cudaError_t e = cudaStreamWaitEvent(h->h2d, h->ev_host[g], 0);
    if (e != cudaSuccess) return e;
    if (h->zero[g]) {
        e = cudaMemsetAsync(slot_ptr(h, s), 0, chunk_bytes(h), h->h2d);
        h->memsets++;
    } else {
        e = cudaMemcpyAsync(slot_ptr(h, s), h->ptr[g], chunk_bytes(h), cudaMemcpyHostToDevice, h->h2d);
        h->h2d_bytes += chunk_bytes(h);
        h->h2d_copies++;
    }
    return e;
}

cudaError_t stage_out(sv_tier* h, uint64_t g, int s) {
    cudaError_t e = cudaMemcpyAsync(h->ptr[g], slot_ptr(h, s), chunk_bytes(h), cudaMemcpyDeviceToHost, h->d2h);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_host[g], h->d2h);
    h->zero[g] = 0;
    h->d2h_bytes += chunk_bytes(h);
    h->d2h_copies++;
    return e;
}

// the op list of a run group as seen by chunk g: diagonal ops keep their in-chunk bits
// and are dropped when a chunk-index bit of their mask reads 0 (engine.py:172-176 for
// ranks, applied to chunks)
void chunk_ops(const sv_tier* h, uint64_t g, const sv_op* ops, int n_ops, std::vector<sv_op>& out) {
    out.clear();
    const uint64_t low = h->chunk_elems - 1;
    for (int i = 0; i < n_ops; ++i) {
        sv_op o = ops[i];
        if (o.kind == SV_OP_DIAG) {
            const uint64_t hi = o.diag_mask >> h->c;
            if ((g & hi) != hi) continue;
            o.diag_mask &= low;
        }
        out.push_back(o);
    }
}

int run_on(sv_tier* h, void* p, const std::vector<sv_op>& ops, int tile_bits) {
    if (ops.empty()) return SV_OK;
    h->passes++;
    return svk_apply_fused(p, h->chunk_elems, h->mode, ops.data(), (int)ops.size(), tile_bits, h->comp);
}

}  // namespace

extern "C" {

int svt_create(int device, int n_qubits, int mode, int chunk_qubits, const uint8_t* fast, int slots,
               sv_thandle* out) {
    *out = nullptr;
    if (mode != SV_FP64 && mode != SV_FP32) return capi_fail(SV_EVALUE, "tiered states hold FP64 or FP32 storage");
    if (n_qubits < 1 || n_qubits > 40) return capi_fail(SV_EVALUE, "tiered state qubit count out of range");
    if (chunk_qubits < 5 || chunk_qubits > n_qubits)
        return capi_fail(SV_EVALUE, "tier chunks must hold 2^5 .. 2^n amplitudes");
    if (slots < 2 || slots > 64) return capi_fail(SV_EVALUE, "tier staging needs 2..64 slots");
    Guard gd(device);
    auto* h = new sv_tier;
    h->device = device;
    h->n = n_qubits;
    h->c = chunk_qubits;
    h->mode = mode;
    h->ebytes = mode == SV_FP32 ? 8 : 16;
    h->chunk_elems = 1ull << chunk_qubits;
    h->n_chunks = 1ull << (n_qubits - chunk_qubits);
    h->n_slots = slots;
    h->fast.assign(fast, fast + h->n_chunks);
    h->ptr.assign(h->n_chunks, nullptr);
    h->zero.assign(h->n_chunks, 0);
    const size_t cb = chunk_bytes(h);
    uint64_t nf = 0;
    for (uint64_t g = 0; g < h->n_chunks; ++g) nf += h->fast[g] ? 1 : 0;
    auto bail = [&](cudaError_t e, const char* what) {
        svt_destroy(h);
        return capi_cuda_fail(e, what);
    };
    cudaError_t e;
    if (nf) {
        h->fast_bytes = nf * cb;
        if ((e = cudaMalloc(&h->fast_arena, h->fast_bytes)) != cudaSuccess) return bail(e, "fast tier (HBM)");
    }
    if ((e = cudaMalloc(&h->slot_arena, cb * (size_t)slots)) != cudaSuccess) return bail(e, "staging slots (HBM)");
    uint64_t fi = 0;
    std::vector<uint64_t> slow;
    for (uint64_t g = 0; g < h->n_chunks; ++g) {
        if (h->fast[g]) h->ptr[g] = static_cast<char*>(h->fast_arena) + (fi++) * cb;
        else slow.push_back(g);
    }
    // Slow chunks: anonymous mappings on transparent huge pages, first-touched and pinned
    // (cudaHostRegister, device-mapped) by 8 threads -- measured 1.3 s for 16 GiB on the
    // B200 box against 7.0 s for cudaHostAlloc, serial or threaded (tools/pin_probe.cu).
    // Chunks below 2 MiB take cudaHostAlloc.
    h->registered.assign(h->n_chunks, 0);
    std::atomic<size_t> next{0};
    std::atomic<int> err{0};
    auto pin_worker = [&]() {
        cudaSetDevice(device);
        for (size_t i = next++; i < slow.size() && !err.load(); i = next++) {
            const uint64_t g = slow[i];
            void* p = nullptr;
            if (cb >= (2u << 20)) {
                p = mmap(nullptr, cb, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
                if (p == MAP_FAILED) { err = 1; return; }
                madvise(p, cb, MADV_HUGEPAGE);
                std::memset(p, 0, cb);
                if (cudaHostRegister(p, cb, cudaHostRegisterPortable | cudaHostRegisterMapped) != cudaSuccess) {
                    munmap(p, cb);
                    err = 2;
                    return;
                }
                h->registered[g] = 1;
            } else if (cudaHostAlloc(&p, cb, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
                err = 3;
                return;
            }
            h->ptr[g] = p;
        }
    };
    {
        const size_t nt = std::min<size_t>(8, std::max<size_t>(1, slow.size()));
        std::vector<std::thread> th;
        for (size_t t = 0; t < nt; ++t) th.emplace_back(pin_worker);
        for (auto& t : th) t.join();
    }
    if (err.load()) {
        cudaGetLastError();
        svt_destroy(h);
        return capi_fail(SV_ENOMEM, "slow tier: pinned host memory allocation failed");
    }
    if ((e = cudaStreamCreateWithFlags(&h->comp, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(e, "tier streams");
    h->ev_in.assign(slots, nullptr);
    h->ev_done.assign(slots, nullptr);
    h->ev_free.assign(slots, nullptr);
    for (int s = 0; s < slots; ++s)
        if ((e = cudaEventCreateWithFlags(&h->ev_in[s], cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&h->ev_done[s], cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&h->ev_free[s], cudaEventDisableTiming)) != cudaSuccess)
            return bail(e, "tier events");
    h->ev_host.assign(h->n_chunks, nullptr);
    for (uint64_t g = 0; g < h->n_chunks; ++g)
        if (!h->fast[g] && (e = cudaEventCreateWithFlags(&h->ev_host[g], cudaEventDisableTiming)) != cudaSuccess)
            return bail(e, "tier events");
    sv::keep_scratch_pool(device);
    *out = h;
    return SV_OK;
}

int svt_destroy(sv_thandle h) {
    if (!h) return SV_OK;
    Guard gd(h->device);
    if (h->comp) cudaStreamSynchronize(h->comp);
    if (h->h2d) cudaStreamSynchronize(h->h2d);
    if (h->d2h) cudaStreamSynchronize(h->d2h);
    const size_t cb = chunk_bytes(h);
    for (uint64_t g = 0; g < h->n_chunks; ++g) {
        if (h->fast[g] || !h->ptr[g]) continue;
        if (!h->registered.empty() && h->registered[g]) {
            cudaHostUnregister(h->ptr[g]);
            munmap(h->ptr[g], cb);
        } else {
            cudaFreeHost(h->ptr[g]);
        }
    }
    if (h->fast_arena) cudaFree(h->fast_arena);
    if (h->slot_arena) cudaFree(h->slot_arena);
    for (auto* v : {&h->ev_in, &h->ev_done, &h->ev_free, &h->ev_host})
        for (cudaEvent_t ev : *v)
            if (ev) cudaEventDestroy(ev);
    for (cudaStream_t st : {h->comp, h->h2d, h->d2h})
        if (st) cudaStreamDestroy(st);
    delete h;
    return SV_OK;
}

int svt_synchronize(sv_thandle h) {
    Guard gd(h->device);
    TTRY(cudaStreamSynchronize(h->h2d), "tier sync (h2d)");
    TTRY(cudaStreamSynchronize(h->comp), "tier sync (compute)");
    TTRY(cudaStreamSynchronize(h->d2h), "tier sync (d2h)");
    return SV_OK;
}

int svt_zero_state(sv_thandle h, int64_t unit) {
    Guard gd(h->device);
    if (int rc = svt_synchronize(h)) return rc;
    if (h->fast_arena) TTRY(cudaMemsetAsync(h->fast_arena, 0, h->fast_bytes, h->comp), "tier zero (HBM)");
    for (uint64_t g = 0; g < h->n_chunks; ++g) h->zero[g] = h->fast[g] ? 0 : 1;
    if (unit >= 0) {
        if ((uint64_t)unit >= (h->n_chunks << h->c)) return capi_fail(SV_EINDEX, "unit amplitude outside the state");
        const uint64_t g = (uint64_t)unit >> h->c, off = (uint64_t)unit & (h->chunk_elems - 1);
        const size_t cb = chunk_bytes(h);
        if (h->fast[g]) {
            const double one[2] = {1.0, 0.0};
            const float onef[2] = {1.0f, 0.0f};
            TTRY(cudaMemcpyAsync(static_cast<char*>(h->ptr[g]) + off * h->ebytes,
                                 h->mode == SV_FP32 ? (const void*)onef : (const void*)one, h->ebytes,
                                 cudaMemcpyHostToDevice, h->comp), "tier unit amplitude");
        } else {
            std::memset(h->ptr[g], 0, cb);
            if (h->mode == SV_FP32) static_cast<float*>(h->ptr[g])[2 * off] = 1.0f;
            else static_cast<double*>(h->ptr[g])[2 * off] = 1.0;
            h->zero[g] = 0;
        }
    }
    TTRY(cudaStreamSynchronize(h->comp), "tier zero sync");
    return SV_OK;
}

int svt_apply_run(sv_thandle h, const sv_op* ops, int n_ops, int tile_bits) {
    Guard gd(h->device);
    if (n_ops <= 0) return SV_OK;
    for (int i = 0; i < n_ops; ++i) {
        const sv_op& o = ops[i];
        if (o.kind == SV_OP_1Q && (o.qa < 0 || o.qa >= h->c))
            return capi_fail(SV_EVALUE, "run group op outside the chunk");
        if (o.kind == SV_OP_2Q && (o.qa < 0 || o.qb < 0 || o.qa >= h->c || o.qb >= h->c))
            return capi_fail(SV_EVALUE, "run group op outside the chunk");
        if (o.kind == SV_OP_DIAG && h->n < 64 && (o.diag_mask >> h->n))
            return capi_fail(SV_EINDEX, "diagonal mask outside the state");
    }
    std::vector<uint64_t> slow, fastc;
    for (uint64_t g = 0; g < h->n_chunks; ++g) (h->fast[g] ? fastc : slow).push_back(g);
    std::vector<sv_op> local;
    // fast chunks' passes are spread between the slow chunks' so the compute stream
    // always has HBM work while the copy engines move the next slot
    size_t fi = 0;
    for (size_t k = 0; k < slow.size(); ++k) {
        const uint64_t g = slow[k];
        chunk_ops(h, g, ops, n_ops, local);
        if (!local.empty()) {
            const int s = acquire_slot(h);
            TTRY(stage_in(h, g, s), "tier stage in");
            TTRY(cudaEventRecord(h->ev_in[s], h->h2d), "tier event");
            TTRY(cudaStreamWaitEvent(h->comp, h->ev_in[s], 0), "tier event");
            if (int rc = run_on(h, slot_ptr(h, s), local, tile_bits)) return rc;
            TTRY(cudaEventRecord(h->ev_done[s], h->comp), "tier event");
            TTRY(cudaStreamWaitEvent(h->d2h, h->ev_done[s], 0), "tier event");
            TTRY(stage_out(h, g, s), "tier stage out");
            TTRY(cudaEventRecord(h->ev_free[s], h->d2h), "tier event");
        }
        const size_t upto = slow.empty() ? fastc.size() : (fastc.size() * (k + 1)) / slow.size();
        for (; fi < upto; ++fi) {
            chunk_ops(h, fastc[fi], ops, n_ops, local);
            if (int rc = run_on(h, h->ptr[fastc[fi]], local, tile_bits)) return rc;
        }
    }
    for (; fi < fastc.size(); ++fi) {
        chunk_ops(h, fastc[fi], ops, n_ops, local);
        if (int rc = run_on(h, h->ptr[fastc[fi]], local, tile_bits)) return rc;
    }
    return SV_OK;
}

int svt_apply_pairing(sv_thandle h, const sv_op* op) {
    Guard gd(h->device);
    const sv_op& o = *op;
    if (o.kind != SV_OP_1Q && o.kind != SV_OP_2Q) return capi_fail(SV_EVALUE, "pairing gates are 1Q / 2Q ops");
    const int qs[2] = {o.qa, o.kind == SV_OP_2Q ? o.qb : -1};
    for (int q : qs)
        if (q >= h->n || (q < 0 && q != qs[1])) return capi_fail(SV_EINDEX, "qubit %d outside the state");
    if (o.kind == SV_OP_2Q && o.qa == o.qb) return capi_fail(SV_EVALUE, "two-qubit gate requires distinct qubits");
    std::vector<uint64_t> masks;
    for (int q : qs)
        if (q >= h->c) masks.push_back(1ull << (q - h->c));
    if (masks.empty()) return capi_fail(SV_EVALUE, "pairing gate has no qubit above the chunk");
    if ((1 << masks.size()) > h->n_slots) return capi_fail(SV_EVALUE, "not enough staging slots");
    uint64_t any = 0;
    for (uint64_t m : masks) any |= m;
    for (uint64_t j = 0; j < h->n_chunks; ++j) {
        if (j & any) continue;
        std::vector<uint64_t> members{j};
        for (uint64_t m : masks) {
            const size_t k = members.size();
            for (size_t i = 0; i < k; ++i) members.push_back(members[i] | m);
        }
        std::vector<void*> p(members.size());
        std::vector<int> slot_of(members.size(), -1);
        bool staged = false;
        for (size_t i = 0; i < members.size(); ++i) {
            const uint64_t g = members[i];
            if (h->fast[g]) {
                p[i] = h->ptr[g];
                continue;
            }
            const int s = acquire_slot(h);
            TTRY(stage_in(h, g, s), "tier stage in");
            slot_of[i] = s;
            p[i] = slot_ptr(h, s);
            staged = true;
        }
        if (staged) {
            // one event for the group: recorded after every member's copy on the H2D stream
            const int s0 = slot_of[0] >= 0 ? slot_of[0] : slot_of[1] >= 0 ? slot_of[1] : slot_of[2] >= 0 ? slot_of[2] : slot_of[3];
            TTRY(cudaEventRecord(h->ev_in[s0], h->h2d), "tier event");
            TTRY(cudaStreamWaitEvent(h->comp, h->ev_in[s0], 0), "tier event");
        }
        cudaError_t e;
        if (masks.size() == 2) {
            e = launch_quad(p.data(), h->chunk_elems, h->mode, o.m, h->comp);
        } else if (o.kind == SV_OP_1Q) {
            e = launch_pair(p[0], p[1], h->chunk_elems, h->mode, o.m, h->comp);
        } else {
            const bool b_hi = o.qb >= h->c;
            e = launch_pair2q(p[0], p[1], h->chunk_elems, h->mode, b_hi ? o.qa : o.qb, b_hi ? 1 : 0, o.m, h->comp);
        }
        if (e != cudaSuccess) return capi_cuda_fail(e, "tier pairing kernel");
        h->passes++;
        if (staged) {
            int s_any = -1;
            for (int s : slot_of) if (s >= 0) s_any = s;
            TTRY(cudaEventRecord(h->ev_done[s_any], h->comp), "tier event");
            TTRY(cudaStreamWaitEvent(h->d2h, h->ev_done[s_any], 0), "tier event");
            for (size_t i = 0; i < members.size(); ++i)
                if (slot_of[i] >= 0) {
                    TTRY(stage_out(h, members[i], slot_of[i]), "tier stage out");
                    TTRY(cudaEventRecord(h->ev_free[slot_of[i]], h->d2h), "tier event");
                }
        }
    }
    return SV_OK;
}

int svt_measure(sv_thandle h, double* norm, double* ones, double* cross) {
    Guard gd(h->device);
    const int n = h->n, c = h->c;
    *norm = 0.0;
    for (int q = 0; q < n; ++q) ones[q] = cross[2 * q] = cross[2 * q + 1] = 0.0;
    std::vector<double> cn(h->n_chunks), o1(c), c1(2 * c);
    for (uint64_t g = 0; g < h->n_chunks; ++g) {
        void* p = h->ptr[g];
        int s = -1;
        if (!h->fast[g]) {
            s = acquire_slot(h);
            TTRY(stage_in(h, g, s), "tier stage in");
            TTRY(cudaEventRecord(h->ev_in[s], h->h2d), "tier event");
            TTRY(cudaStreamWaitEvent(h->comp, h->ev_in[s], 0), "tier event");
            p = slot_ptr(h, s);
        }
        double nj = 0.0;
        if (int rc = svk_measure(p, h->chunk_elems, h->mode, &nj, o1.data(), c1.data(), h->comp)) return rc;
        h->passes++;
        cn[g] = nj;
        *norm += nj;
        for (int q = 0; q < c; ++q) {
            ones[q] += o1[q];
            cross[2 * q] += c1[2 * q];
            cross[2 * q + 1] += c1[2 * q + 1];
        }
        for (int b = 0; b < n - c; ++b) {       // cross terms of chunk-index qubits: pair (g, g | 2^b)
            if ((g >> b) & 1) continue;
            const uint64_t partner = g | (1ull << b);
            const void* pp = h->ptr[partner];
            if (!h->fast[partner]) {
                if (h->zero[partner]) continue;  // an all-zero partner adds nothing
                TTRY(cudaStreamWaitEvent(h->comp, h->ev_host[partner], 0), "tier event");
                void* dp = nullptr;
                TTRY(cudaHostGetDevicePointer(&dp, h->ptr[partner], 0), "tier zero-copy pointer");
                pp = dp;
                h->zc_bytes += chunk_bytes(h);
            }
            double d[2];
            if (int rc = svk_pair_dot(p, pp, h->chunk_elems, h->mode, 0, d, h->comp)) return rc;
            cross[2 * (c + b)] += d[0];
            cross[2 * (c + b) + 1] += d[1];
        }
        if (s >= 0) TTRY(cudaEventRecord(h->ev_free[s], h->comp), "tier event");
    }
    for (int b = 0; b < n - c; ++b)
        for (uint64_t g = 0; g < h->n_chunks; ++g)
            if ((g >> b) & 1) ones[c + b] += cn[g];
    return SV_OK;
}

int svt_export(sv_thandle h, void* host, uint64_t first, uint64_t count) {
    Guard gd(h->device);
    if (first + count > (h->n_chunks << h->c)) return capi_fail(SV_EINDEX, "export range outside the state");
    if (int rc = svt_synchronize(h)) return rc;
    char* dst = static_cast<char*>(host);
    while (count) {
        const uint64_t g = first >> h->c, off = first & (h->chunk_elems - 1);
        const uint64_t k = std::min<uint64_t>(count, h->chunk_elems - off);
        const size_t nb = k * h->ebytes;
        const char* src = static_cast<const char*>(h->ptr[g]) + off * h->ebytes;
        if (h->fast[g]) TTRY(cudaMemcpy(dst, src, nb, cudaMemcpyDeviceToHost), "tier export");
        else if (h->zero[g]) std::memset(dst, 0, nb);
        else std::memcpy(dst, src, nb);
        dst += nb;
        first += k;
        count -= k;
    }
    return SV_OK;
}

int svt_import(sv_thandle h, const void* host, uint64_t first, uint64_t count) {
    Guard gd(h->device);
    if (first + count > (h->n_chunks << h->c)) return capi_fail(SV_EINDEX, "import range outside the state");
    if (int rc = svt_synchronize(h)) return rc;
    const char* src = static_cast<const char*>(host);
    while (count) {
        const uint64_t g = first >> h->c, off = first & (h->chunk_elems - 1);
        const uint64_t k = std::min<uint64_t>(count, h->chunk_elems - off);
        const size_t nb = k * h->ebytes;
        char* dst = static_cast<char*>(h->ptr[g]) + off * h->ebytes;
        if (h->fast[g]) {
            TTRY(cudaMemcpy(dst, src, nb, cudaMemcpyHostToDevice), "tier import");
        } else {
            if (h->zero[g] && nb != chunk_bytes(h)) std::memset(h->ptr[g], 0, chunk_bytes(h));
            std::memcpy(dst, src, nb);
            h->zero[g] = 0;
        }
        src += nb;
        first += k;
        count -= k;
    }
    return SV_OK;
}

int svt_stats(sv_thandle h, uint64_t* out8) {
    out8[0] = h->h2d_bytes;
    out8[1] = h->d2h_bytes;
    out8[2] = h->h2d_copies;
    out8[3] = h->d2h_copies;
    out8[4] = h->zc_bytes;
    out8[5] = h->memsets;
    out8[6] = h->passes;
    out8[7] = h->fast_bytes;
    return SV_OK;
}

}  // extern "C"
