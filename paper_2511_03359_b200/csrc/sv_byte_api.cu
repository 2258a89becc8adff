// extern "C" entry points of the BYTE mode (include/svb200.h, "BYTE mode").
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "sv_byte.cuh"
#include "sv_common.cuh"
#include "sv_kernels.cuh"

using namespace sv;

namespace sv {
int capi_fail(int code, const char* msg);                 // sv_capi.cu
int capi_cuda_fail(cudaError_t e, const char* what);      // sv_capi.cu
int capi_measure(const void* psi, uint64_t n, int mode, double* norm, double* ones, double* cross,
                 cudaStream_t st);                        // sv_capi.cu
int capi_measure_byte(const void* src, uint64_t n, double* norm, double* ones, double* cross, cudaStream_t st);
int capi_measure_byte_sup(const void* src, uint64_t n, uint64_t sup_fixed, uint64_t sup_val, double* norm,
                          double* ones, double* cross, cudaStream_t st);
}

#define BTRY(expr, what)                                        \
    do {                                                        \
        cudaError_t _e = (expr);                                \
        if (_e != cudaSuccess) return capi_cuda_fail(_e, what); \
    } while (0)

struct sv_bstate {
    int device, n;
    uint8_t* plane[2][2];      // [buffer][0 = magnitude index, 1 = phase index]
    int cur;
    cudaStream_t stream;
    ByteTables* tab;
    ByteCand* cand;            // device struct
    ByteCand hcand;            // host copy of the pointers / capacities
};

namespace {
struct Guard {
    int prev = -1;
    explicit Guard(int d) { cudaGetDevice(&prev); if (prev != d) cudaSetDevice(d); }
    ~Guard() { int c = -1; cudaGetDevice(&c); if (prev >= 0 && c != prev) cudaSetDevice(prev); }
};
constexpr uint64_t CAP_MAG = 1ull << 20, CAP_PH = 1ull << 20, CAP_UNSURE = 1ull << 22;

ByteGate to_gate(const svb_gate_desc& d, uint64_t n_elems) {
    ByteGate g;
    std::memset(&g, 0, sizeof(g));
    g.kind = d.kind; g.qa = d.qa; g.qb = d.qb; g.mask = d.diag_mask;
    std::memcpy(g.m, d.m, sizeof(g.m));
    g.n_elems = n_elems;
    g.n_local = d.n_local;
    g.xkind = d.xkind; g.xmask_a = d.xmask_a; g.xmask_b = d.xmask_b; g.qlow_top = d.qlow_top;
    g.producer = d.producer;
    g.collect = d.collect;
    g.want_mag = d.want_mag; g.want_ph = d.want_ph;
    g.mag_cut = d.mag_cut; g.ph_cut = d.ph_cut;
    g.scan_only = d.scan_only;
    g.phys_base = d.phys_base;
    g.rank_bits = d.rank_bits;
    for (int j = 0; j < 12; ++j) g.lbit[j] = d.lbit[j];
    g.sup_fixed = d.sup_fixed & (n_elems - 1ull);
    g.sup_val = d.sup_val & g.sup_fixed;
    return g;
}
}  // namespace

extern "C" {

int svb_create(int device, int n_qubits, sv_bhandle* out) {
    *out = nullptr;
    if (n_qubits < 0 || n_qubits > 40) return capi_fail(SV_EVALUE, "n_qubits out of range");
    Guard gd(device);
    keep_scratch_pool(device);
    if (cudaError_t e0 = sv::byte_kernels_prepare()) return capi_cuda_fail(e0, "BYTE kernel attributes");
    sv_bstate* h = new sv_bstate();
    std::memset(h, 0, sizeof(*h));
    h->device = device;
    h->n = n_qubits;
    const size_t bytes = (size_t)1 << n_qubits;
    const size_t pbytes = bytes < 256 ? 256 : bytes;
    auto fail_free = [&](cudaError_t e, const char* what) {
        for (int b = 0; b < 2; ++b) for (int p = 0; p < 2; ++p) if (h->plane[b][p]) sv::slab_free(h->plane[b][p], pbytes);
        if (h->tab) cudaFree(h->tab);
        delete h;
        return capi_cuda_fail(e, what);
    };
    for (int b = 0; b < 2; ++b)
        for (int p = 0; p < 2; ++p) {
            cudaError_t e = sv::slab_alloc(reinterpret_cast<void**>(&h->plane[b][p]), pbytes);
            if (e != cudaSuccess) return fail_free(e, "BYTE plane allocation");
        }
    cudaError_t e = cudaMalloc(&h->tab, sizeof(ByteTables));
    if (e != cudaSuccess) return fail_free(e, "codebook tables");
    e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail_free(e, "stream");
    ByteCand& c = h->hcand;
    c.cap_mag = CAP_MAG; c.cap_ph = CAP_PH; c.cap_unsure = CAP_UNSURE;
    if ((e = cudaMalloc(&c.mag, CAP_MAG * 8)) != cudaSuccess ||
        (e = cudaMalloc(&c.ph, CAP_PH * 32)) != cudaSuccess ||
        (e = cudaMalloc(&c.mag_tag, CAP_MAG * 4)) != cudaSuccess ||
        (e = cudaMalloc(&c.ph_tag, CAP_PH * 4)) != cudaSuccess ||
        (e = cudaMalloc(&c.unsure_idx, CAP_UNSURE * 8)) != cudaSuccess ||
        (e = cudaMalloc(&c.unsure_val, CAP_UNSURE * 16)) != cudaSuccess ||
        (e = cudaMalloc(&h->cand, sizeof(ByteCand))) != cudaSuccess)
        return fail_free(e, "candidate buffers");
    BTRY(cudaMemcpy(h->cand, &c, sizeof(ByteCand), cudaMemcpyHostToDevice), "candidate header");
    // initial tables: magnitudes [0, 1], phases [0] (codec.py:102-105)
    const double m0[2] = {0.0, 1.0}, t0[1] = {0.0}, ux0[1] = {1.0}, uy0[1] = {0.0};
    *out = h;
    return svb_set_tables(h, m0, 2, t0, ux0, uy0, 1);
}

int svb_destroy(sv_bhandle h) {
    if (!h) return SV_OK;
    Guard gd(h->device);
    cudaStreamSynchronize(h->stream);
    const size_t pbytes = ((size_t)1 << h->n) < 256 ? 256 : ((size_t)1 << h->n);
    for (int b = 0; b < 2; ++b) for (int p = 0; p < 2; ++p) sv::slab_free(h->plane[b][p], pbytes);
    cudaFree(h->tab);
    cudaFree(h->hcand.mag); cudaFree(h->hcand.ph); cudaFree(h->hcand.unsure_idx); cudaFree(h->hcand.unsure_val);
    cudaFree(h->hcand.mag_tag); cudaFree(h->hcand.ph_tag);
    cudaFree(h->cand);
    cudaStreamDestroy(h->stream);
    delete h;
    return SV_OK;
}

int svb_info(sv_bhandle h, int* device, int* n_qubits, void** stream) {
    if (device) *device = h->device;
    if (n_qubits) *n_qubits = h->n;
    if (stream) *stream = reinterpret_cast<void*>(h->stream);
    return SV_OK;
}

int svb_zero_state(sv_bhandle h, int64_t unit) {
    Guard gd(h->device);
    const uint64_t n = 1ull << h->n;
    // both buffers: a support-restricted pass (sup_fixed) writes only the items inside the support
    for (int b = 0; b < 2; ++b)
        for (int p = 0; p < 2; ++p) BTRY(cudaMemsetAsync(h->plane[b][p], 0, n, h->stream), "zero planes");
    if (unit >= 0) {
        if ((uint64_t)unit >= n) return capi_fail(SV_EINDEX, "unit index outside the state");
        static const uint8_t one = 1;
        BTRY(cudaMemcpyAsync(h->plane[h->cur][0] + unit, &one, 1, cudaMemcpyHostToDevice, h->stream), "unit");
    }
    BTRY(cudaStreamSynchronize(h->stream), "zero sync");
    return SV_OK;
}

// zeros into the pending (not current) planes: after a remap swap moved the current planes
// under a tracked support, the next support-restricted write pass relies on zeros outside it
int svb_clear_pending(sv_bhandle h) {
    Guard gd(h->device);
    const uint64_t n = 1ull << h->n;
    for (int p = 0; p < 2; ++p) BTRY(cudaMemsetAsync(h->plane[1 - h->cur][p], 0, n, h->stream), "zero pending planes");
    return SV_OK;
}

int svb_set_tables(sv_bhandle h, const double* mags, int n_mag, const double* thetas, const double* ux,
                   const double* uy, int n_ph) {
    if (n_mag < 1 || n_mag > 256 || n_ph < 1 || n_ph > 256) return capi_fail(SV_EVALUE, "table size out of range");
    Guard gd(h->device);
    ByteTables t;
    std::memset(&t, 0, sizeof(t));
    for (int i = 0; i < n_mag; ++i) t.dmag[i] = mags[i];
    for (int i = 0; i < n_ph; ++i) { t.dux[i] = ux[i]; t.duy[i] = uy[i]; }
    std::vector<int> o(n_mag);
    std::iota(o.begin(), o.end(), 0);
    std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return mags[a] < mags[b]; });
    for (int i = 0; i < n_mag; ++i) { t.smag[i] = mags[o[i]]; t.smag_idx[i] = (uint8_t)o[i]; }
    std::vector<int> q(n_ph);
    std::iota(q.begin(), q.end(), 0);
    std::stable_sort(q.begin(), q.end(), [&](int a, int b) { return thetas[a] < thetas[b]; });
    for (int i = 0; i < n_ph; ++i) { t.sth[i] = thetas[q[i]]; t.sth_idx[i] = (uint8_t)q[i]; }
    t.n_mag = n_mag;
    t.n_ph = n_ph;
    for (int i = 0; i < 256; ++i) {
        if (i + 1 < n_mag) {
            const double mid = 0.5 * (t.smag[i] + t.smag[i + 1]);
            t.sqmid[i] = mid * mid;
        } else {
            t.sqmid[i] = 1.0 / 0.0;
        }
        t.sqmag[i] = i < n_mag ? t.smag[i] * t.smag[i] : 0.0;
    }
    BTRY(cudaMemcpyAsync(h->tab, &t, sizeof(t), cudaMemcpyHostToDevice, h->stream), "table upload");
    BTRY(cudaStreamSynchronize(h->stream), "table sync");
    return SV_OK;
}

int svb_gate(sv_bhandle h, const svb_gate_desc* d) {
    Guard gd(h->device);
    const uint64_t n = 1ull << h->n;
    if (d->kind == SV_OP_1Q && (d->qa < 0 || d->qa >= h->n)) return capi_fail(SV_EINDEX, "qubit outside the state");
    if (d->kind == SV_OP_2Q && (d->qa < 0 || d->qa >= h->n || d->qb < 0 || d->qb >= h->n || d->qa == d->qb))
        return capi_fail(SV_EVALUE, "bad two-qubit operands");
    const ByteGate g = to_gate(*d, n);
    const int c = h->cur, nx = 1 - h->cur;
    cudaError_t e = launch_byte_gate(h->plane[c][0], d->ph_zero_in ? nullptr : h->plane[c][1], h->plane[nx][0],
                                     d->ph_zero_out ? nullptr : h->plane[nx][1], h->tab, g, h->cand, h->stream);
    return e == cudaSuccess ? SV_OK : capi_cuda_fail(e, "BYTE gate launch");
}

int svb_gate_in_place(sv_bhandle h, const svb_gate_desc* d) {
    Guard gd(h->device);
    if (d->kind != SV_OP_DIAG) return capi_fail(SV_EVALUE, "in-place BYTE passes are for diagonal gates");
    if (d->scan_only || d->collect) return capi_fail(SV_EVALUE, "in-place BYTE pass: write pass only");
    // a mask bit outside the buffer (a rank whose global qubit reads 0) selects nothing:
    // in place, nothing is written
    if (d->diag_mask >> h->n) return SV_OK;
    ByteGate g = to_gate(*d, 1ull << h->n);
    g.in_place = 1;
    const int c = h->cur;
    cudaError_t e = launch_byte_gate(h->plane[c][0], d->ph_zero_in ? nullptr : h->plane[c][1], h->plane[c][0],
                                     d->ph_zero_out ? nullptr : h->plane[c][1], h->tab, g, h->cand, h->stream);
    return e == cudaSuccess ? SV_OK : capi_cuda_fail(e, "BYTE gate launch");
}

int svb_candidates(sv_bhandle h, double* mags, uint64_t cap_m, uint64_t* n_m, double* ph4, uint64_t cap_p,
                   uint64_t* n_p, int* flags) {
    Guard gd(h->device);
    ByteCand c;
    BTRY(cudaMemcpyAsync(&c, h->cand, sizeof(c), cudaMemcpyDeviceToHost, h->stream), "candidate header");
    BTRY(cudaStreamSynchronize(h->stream), "candidate sync");
    const uint64_t nm = std::min<uint64_t>(c.n_mag, c.cap_mag), np = std::min<uint64_t>(c.n_ph, c.cap_ph);
    *n_m = nm;
    *n_p = np;
    *flags = (c.overflow ? 1 : 0) | (c.any_mag ? 2 : 0) | (c.any_ph ? 4 : 0) | (nm > cap_m || np > cap_p ? 1 : 0);
    if (nm && mags) BTRY(cudaMemcpyAsync(mags, h->hcand.mag, 8 * std::min(nm, cap_m), cudaMemcpyDeviceToHost, h->stream), "mags");
    if (np && ph4) BTRY(cudaMemcpyAsync(ph4, h->hcand.ph, 32 * std::min(np, cap_p), cudaMemcpyDeviceToHost, h->stream), "phases");
    BTRY(cudaStreamSynchronize(h->stream), "candidate copy");
    return SV_OK;
}

int svb_candidate_tags(sv_bhandle h, int32_t* mag_tags, uint64_t cap_m, int32_t* ph_tags, uint64_t cap_p) {
    Guard gd(h->device);
    ByteCand c;
    BTRY(cudaMemcpyAsync(&c, h->cand, sizeof(c), cudaMemcpyDeviceToHost, h->stream), "candidate header");
    BTRY(cudaStreamSynchronize(h->stream), "candidate sync");
    const uint64_t nm = std::min<uint64_t>(std::min<uint64_t>(c.n_mag, c.cap_mag), cap_m);
    const uint64_t np = std::min<uint64_t>(std::min<uint64_t>(c.n_ph, c.cap_ph), cap_p);
    if (nm && mag_tags) BTRY(cudaMemcpyAsync(mag_tags, h->hcand.mag_tag, 4 * nm, cudaMemcpyDeviceToHost, h->stream), "mag tags");
    if (np && ph_tags) BTRY(cudaMemcpyAsync(ph_tags, h->hcand.ph_tag, 4 * np, cudaMemcpyDeviceToHost, h->stream), "phase tags");
    BTRY(cudaStreamSynchronize(h->stream), "tag copy");
    return SV_OK;
}

int svb_unsure(sv_bhandle h, uint64_t* idx, double* vals, uint64_t cap, uint64_t* n) {
    Guard gd(h->device);
    ByteCand c;
    BTRY(cudaMemcpyAsync(&c, h->cand, sizeof(c), cudaMemcpyDeviceToHost, h->stream), "unsure header");
    BTRY(cudaStreamSynchronize(h->stream), "unsure sync");
    if (c.n_unsure > c.cap_unsure)   // never silently drop an amplitude the host must re-encode
        return capi_fail(SV_ENOMEM, "uncertain-phase list overflow: more amplitudes than the 4M-entry buffer");
    const uint64_t k = c.n_unsure;
    *n = k;
    if (k > cap) return capi_fail(SV_EVALUE, "unsure buffer too small");
    if (k) {
        BTRY(cudaMemcpyAsync(idx, h->hcand.unsure_idx, 8 * k, cudaMemcpyDeviceToHost, h->stream), "unsure idx");
        BTRY(cudaMemcpyAsync(vals, h->hcand.unsure_val, 16 * k, cudaMemcpyDeviceToHost, h->stream), "unsure vals");
        BTRY(cudaStreamSynchronize(h->stream), "unsure copy");
    }
    return SV_OK;
}

int svb_reset(sv_bhandle h) {
    // stream-ordered: the next pass on this stream sees the cleared header; no host wait
    // (hcand lives as long as the handle and is never written after svb_create)
    Guard gd(h->device);
    BTRY(cudaMemcpyAsync(h->cand, &h->hcand, sizeof(ByteCand), cudaMemcpyHostToDevice, h->stream), "reset");
    return SV_OK;
}

static int patch_planes(sv_bhandle h, int which, const uint64_t* idx, const uint8_t* mi, const uint8_t* pi,
                        uint64_t n);
int svb_patch(sv_bhandle h, const uint64_t* idx, const uint8_t* mi, const uint8_t* pi, uint64_t n) {
    return patch_planes(h, 1 - h->cur, idx, mi, pi, n);
}
int svb_patch_in_place(sv_bhandle h, const uint64_t* idx, const uint8_t* mi, const uint8_t* pi, uint64_t n) {
    return patch_planes(h, h->cur, idx, mi, pi, n);
}
static int patch_planes(sv_bhandle h, int which, const uint64_t* idx, const uint8_t* mi, const uint8_t* pi,
                        uint64_t n) {
    if (n == 0) return SV_OK;
    Guard gd(h->device);
    uint64_t* d_idx = nullptr;
    uint8_t* d_b = nullptr;
    BTRY(cudaMallocAsync(reinterpret_cast<void**>(&d_idx), 8 * n, h->stream), "patch alloc");
    BTRY(cudaMallocAsync(reinterpret_cast<void**>(&d_b), 2 * n, h->stream), "patch alloc");
    BTRY(cudaMemcpyAsync(d_idx, idx, 8 * n, cudaMemcpyHostToDevice, h->stream), "patch idx");
    BTRY(cudaMemcpyAsync(d_b, mi, n, cudaMemcpyHostToDevice, h->stream), "patch mi");
    BTRY(cudaMemcpyAsync(d_b + n, pi, n, cudaMemcpyHostToDevice, h->stream), "patch pi");
    cudaError_t e = launch_byte_patch(h->plane[which][0], h->plane[which][1], d_idx, d_b, d_b + n, n, h->stream);
    cudaFreeAsync(d_idx, h->stream);
    cudaFreeAsync(d_b, h->stream);
    if (e != cudaSuccess) return capi_cuda_fail(e, "patch");
    BTRY(cudaStreamSynchronize(h->stream), "patch sync");
    return SV_OK;
}

int svb_commit(sv_bhandle h) {
    h->cur = 1 - h->cur;
    return SV_OK;
}

int svb_export(sv_bhandle h, uint8_t* mi, uint8_t* pi, uint64_t first, uint64_t count) {
    Guard gd(h->device);
    if (first + count > (1ull << h->n)) return capi_fail(SV_EINDEX, "export range outside the state");
    BTRY(cudaMemcpyAsync(mi, h->plane[h->cur][0] + first, count, cudaMemcpyDeviceToHost, h->stream), "export mi");
    BTRY(cudaMemcpyAsync(pi, h->plane[h->cur][1] + first, count, cudaMemcpyDeviceToHost, h->stream), "export pi");
    BTRY(cudaStreamSynchronize(h->stream), "export sync");
    return SV_OK;
}

int svb_import(sv_bhandle h, const uint8_t* mi, const uint8_t* pi, uint64_t first, uint64_t count) {
    Guard gd(h->device);
    if (first + count > (1ull << h->n)) return capi_fail(SV_EINDEX, "import range outside the state");
    BTRY(cudaMemcpyAsync(h->plane[h->cur][0] + first, mi, count, cudaMemcpyHostToDevice, h->stream), "import mi");
    BTRY(cudaMemcpyAsync(h->plane[h->cur][1] + first, pi, count, cudaMemcpyHostToDevice, h->stream), "import pi");
    BTRY(cudaStreamSynchronize(h->stream), "import sync");
    return SV_OK;
}

int svb_decode(sv_bhandle h, double* out, uint64_t first, uint64_t count) {
    Guard gd(h->device);
    if (first + count > (1ull << h->n)) return capi_fail(SV_EINDEX, "decode range outside the state");
    double* d = nullptr;
    BTRY(cudaMallocAsync(reinterpret_cast<void**>(&d), 16 * (count ? count : 1), h->stream), "decode buffer");
    cudaError_t e = launch_byte_decode(h->plane[h->cur][0] + first, h->plane[h->cur][1] + first, h->tab, d, count,
                                       h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, 16 * count, cudaMemcpyDeviceToHost, h->stream);
    cudaFreeAsync(d, h->stream);
    if (e != cudaSuccess) return capi_cuda_fail(e, "decode");
    BTRY(cudaStreamSynchronize(h->stream), "decode sync");
    return SV_OK;
}

int svb_measure_support(sv_bhandle h, uint64_t sup_fixed, uint64_t sup_val, double* norm, double* ones,
                        double* cross) {
    Guard gd(h->device);
    const uint64_t n = 1ull << h->n;
    if (h->n < 16 || !sup_fixed) return svb_measure(h, norm, ones, cross);
    struct { const uint8_t* mi; const uint8_t* pi; const double* tab; } src = {
        h->plane[h->cur][0], h->plane[h->cur][1], reinterpret_cast<const double*>(h->tab)};
    return capi_measure_byte_sup(&src, n, sup_fixed, sup_val, norm, ones, cross, h->stream);
}

int svb_measure(sv_bhandle h, double* norm, double* ones, double* cross) {
    Guard gd(h->device);
    const uint64_t n = 1ull << h->n;
    if (h->n == 0) {   // one amplitude: decode it on the host side of the copy
        double v[2];
        if (int rc = svb_decode(h, v, 0, 1)) return rc;
        *norm = v[0] * v[0] + v[1] * v[1];
        return SV_OK;
    }
    // decoded on the fly inside the tiled measurement passes (no FP64 copy of the state)
    struct { const uint8_t* mi; const uint8_t* pi; const double* tab; } src = {
        h->plane[h->cur][0], h->plane[h->cur][1], reinterpret_cast<const double*>(h->tab)};
    return capi_measure_byte(&src, n, norm, ones, cross, h->stream);
}

int svb_encode_values(sv_bhandle h, const double* vals, uint64_t n, uint8_t* mi, uint8_t* pi, int collect) {
    Guard gd(h->device);
    double* d = nullptr;
    uint8_t* b = nullptr;
    BTRY(cudaMallocAsync(reinterpret_cast<void**>(&d), 16 * (n ? n : 1), h->stream), "encode buffer");
    BTRY(cudaMallocAsync(reinterpret_cast<void**>(&b), 2 * (n ? n : 1), h->stream), "encode bytes");
    BTRY(cudaMemcpyAsync(d, vals, 16 * n, cudaMemcpyHostToDevice, h->stream), "encode upload");
    svb_gate_desc desc;
    std::memset(&desc, 0, sizeof(desc));
    desc.producer = -1;
    desc.collect = collect;
    for (int j = 0; j < 16; ++j) desc.lbit[j] = 0;
    desc.want_mag = 1;
    desc.want_ph = 1;
    desc.mag_cut = 1e308;
    desc.ph_cut = 1e308;
    const ByteGate g = to_gate(desc, n);
    cudaError_t e = launch_byte_encode(d, n, h->tab, b, b + n, g, h->cand, h->stream);
    if (e == cudaSuccess && n) e = cudaMemcpyAsync(mi, b, n, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess && n) e = cudaMemcpyAsync(pi, b + n, n, cudaMemcpyDeviceToHost, h->stream);
    cudaFreeAsync(d, h->stream);
    cudaFreeAsync(b, h->stream);
    if (e != cudaSuccess) return capi_cuda_fail(e, "encode");
    BTRY(cudaStreamSynchronize(h->stream), "encode sync");
    return SV_OK;
}

int svb_ipc_handles(sv_bhandle h, void* out256) {
    Guard gd(h->device);
    for (int b = 0; b < 2; ++b)
        for (int p = 0; p < 2; ++p) {
            cudaIpcMemHandle_t ih;
            BTRY(cudaIpcGetMemHandle(&ih, h->plane[b][p]), "cudaIpcGetMemHandle");
            sv::slab_mark_exported(h->plane[b][p]);
            std::memcpy(static_cast<char*>(out256) + 64 * (2 * b + p), &ih, 64);
        }
    return SV_OK;
}

int svb_cur(sv_bhandle h) { return h->cur; }

int svb_planes(sv_bhandle h, void** cur_mi, void** cur_pi) {
    *cur_mi = h->plane[h->cur][0];
    *cur_pi = h->plane[h->cur][1];
    return SV_OK;
}

int svb_swap_peer(sv_bhandle h, void* peer_mi, void* peer_pi, int l, int side) {
    Guard gd(h->device);
    const uint64_t n = 1ull << h->n;
    if (l < 0 || l >= h->n || h->n < 2) return capi_fail(SV_EINDEX, "swap qubit outside the slice");
    cudaError_t e = launch_byte_swap_peer(h->plane[h->cur][0], h->plane[h->cur][1], static_cast<uint8_t*>(peer_mi),
                                          static_cast<uint8_t*>(peer_pi), n, l, side, h->stream);
    return e == cudaSuccess ? SV_OK : capi_cuda_fail(e, "byte swap launch");
}

int svb_swap_group(sv_bhandle h, void* peer_mi, void* peer_pi, uint64_t victim_mask, uint64_t own_pattern,
                   uint64_t peer_pattern, uint64_t t_begin, uint64_t t_count) {
    Guard gd(h->device);
    const uint64_t n = 1ull << h->n;
    if ((victim_mask & ~(n - 1)) || ((own_pattern | peer_pattern) & ~victim_mask))
        return capi_fail(SV_EINDEX, "victim mask / patterns outside the slice");
    const uint64_t rest = n >> __builtin_popcountll(victim_mask);
    if (t_begin > rest || t_count > rest - t_begin) return capi_fail(SV_EINDEX, "rest range outside the slice");
    if (t_count == 0) return SV_OK;
    cudaError_t e = launch_byte_swap_group(h->plane[h->cur][0], h->plane[h->cur][1], static_cast<uint8_t*>(peer_mi),
                                           static_cast<uint8_t*>(peer_pi), t_begin, t_count, victim_mask, own_pattern,
                                           peer_pattern, h->stream);
    return e == cudaSuccess ? SV_OK : capi_cuda_fail(e, "byte group swap launch");
}

int svb_pair_dot(sv_bhandle h, const void* a_mi, const void* a_pi, const void* b_mi, const void* b_pi,
                 uint64_t count, double* out2) {
    Guard gd(h->device);
    out2[0] = out2[1] = 0.0;
    if (count == 0) return SV_OK;
    const int grid = (int)std::min<uint64_t>((count + 255) / 256, (uint64_t)sm_count(h->device) * 4);
    double* part = nullptr;
    BTRY(cudaMallocAsync(reinterpret_cast<void**>(&part), 16 * grid, h->stream), "pair dot scratch");
    cudaError_t e = launch_byte_pair_dot(static_cast<const uint8_t*>(a_mi), static_cast<const uint8_t*>(a_pi),
                                         static_cast<const uint8_t*>(b_mi), static_cast<const uint8_t*>(b_pi), h->tab,
                                         count, part, grid, h->stream);
    std::vector<double> hp(2 * grid);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hp.data(), part, 16 * grid, cudaMemcpyDeviceToHost, h->stream);
    cudaFreeAsync(part, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return capi_cuda_fail(e, "byte pair dot");
    for (int b = 0; b < grid; ++b) { out2[0] += hp[2 * b]; out2[1] += hp[2 * b + 1]; }
    return SV_OK;
}

}  // extern "C"
