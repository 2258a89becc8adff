// Launch-side declarations shared by the .cu translation units.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/svb200.h"

namespace sv {

// Fused-pass parameters travel as one kernel-parameter block (constant bank:
// broadcast reads, no per-CTA global loads).  Kept well under the 32 KB
// kernel-parameter limit of sm_70+ with CUDA >= 12.1.
constexpr int kMaxOps = 256;           // ops per pass (128 unless diagonal runs are combined)
constexpr int kMaxMData = 1536;         // doubles
constexpr int kMaxTileBits = 12;

struct FusedParams {
    uint64_t n_tiles;
    uint64_t out_mask;                  // local-index bits NOT in the tile
    uint64_t tile_mask;                 // local-index bits in the tile
    int n;                              // local qubits of the buffer
    int k;                              // tile bits
    int b;                              // contiguous low tile bits (T[i] == i for i < b)
    int n_ops;
    int8_t tq[kMaxTileBits];            // tile position -> qubit
    uint8_t kind[kMaxOps];              // SV_OP_*
    uint8_t pa[kMaxOps];                // tile positions (1Q: pa; 2Q: pa = pos(qa), pb = pos(qb))
    uint8_t pb[kMaxOps];
    uint16_t moff[kMaxOps];             // offset into mdata
    uint32_t dmask_t[kMaxOps];          // DIAG: required tile-position bits
    uint64_t dmask_o[kMaxOps];          // DIAG: required out-of-tile local-index bits
    double mdata[kMaxMData];
};

// v2 fused passes: register-resident 2^12-amplitude tiles (sv_fused2.cu)
enum {
    F2_1Q = 1, F2_1Q_REAL = 2, F2_1Q_MONO = 3,
    F2_2Q = 4, F2_2Q_REAL = 5, F2_2Q_MONO = 6,
    F2_DIAG = 7, F2_DIAG_NEG = 8
};
constexpr int kMaxSegs = 48;
struct Fused2Params {
    uint64_t n_tiles;
    uint64_t tile_mask;
    int n, b, n_ops, n_segs;
    int direct_in, direct_out;
    int cfg, kbits, rbits;              // kernel configuration (tile bits, register bits)
    int storage;                        // SV_FP64 / SV_FP32 (FP32 only through the specialised kernel)
    int combine_diag;                   // 1: runs of diagonal ops multiply each amplitude by their combined
                                        // factor (within 1e-12, not bit-exact; FP64 specialised passes only)
    uint64_t cmask_t, cpat_t;           // chunked pass: tile-index bits fixed to cpat_t (n_tiles counts
                                        // the remaining tiles); 0, 0 = every tile
    int64_t vinit;                      // -2: read the tiles; -1 / u: generate them (all zeros / |u>),
                                        // specialised kernel only (lazy zero state, first pass)
    uint64_t pfix, pval;                // pfix != 0: amplitudes with (i & pfix) != pval load as zeros
                                        // (a tracked support over memory not yet written; cp.async zfill)
    int8_t tq[13];                      // tile position -> qubit (2^13 tiles: config 10)
    uint8_t seg_reg[kMaxSegs][4];       // register bit j -> tile position
    uint8_t seg_thr[kMaxSegs][9];       // thread-id bit j -> tile position
    uint16_t seg_end[kMaxSegs];         // one past the segment's last op
    uint16_t seg_rsw[kMaxSegs][16];     // swizzled shared-memory offset of register slot i
    uint64_t last_rgo[16];              // HBM offset of register slot i in the last segment
    uint64_t pf_go[16];                 // HBM offset of tile element 256*j (prefetch chunks)
    uint64_t base_tab[4][256];          // tile index byte k -> local-index bits (deposit tables)
    uint8_t kind[kMaxOps];
    uint8_t ra[kMaxOps], rb[kMaxOps];   // register bits of qa / qb
    uint8_t dreg[kMaxOps];              // DIAG: register-bit mask
    uint16_t dthr[kMaxOps];             // DIAG: tile-position mask covered by thread bits
    uint16_t moff[kMaxOps];
    uint16_t mono[kMaxOps];             // monomial rows: per row src (2 bits) | unit (2 bits) << 2
    uint64_t dout[kMaxOps];             // DIAG: out-of-tile local-index mask
    double mdata[kMaxMData];
};
cudaError_t launch_fused2(void* psi, int mode, const Fused2Params& p, cudaStream_t st);
// run-time specialised form of the same pass (sv_jit.cu): 0 launched, 1 not ready, < 0 error
int jit_launch_fused(void* psi, const Fused2Params& p, cudaStream_t st);
bool jit_predicable(const Fused2Params& p);     // the pass's tile loads honour pfix / pval
int jit_prepare_fused(const Fused2Params& p);   // queue the compile; 1 if a new kernel was queued
bool jit_enabled();                             // JIT mode != 0 and NVRTC present
}  // namespace sv
#include <string>
namespace sv {
int jit_probe(const Fused2Params& P, std::string* src, bool compile, double* ms, std::string* log);
// FP64 warp instructions per amplitude the specialised pass issues (a warp instruction
// occupies the FP64 pipe for all 32 lanes, whichever lanes a diagonal mask selects)
double jit_fp64_per_amp(const Fused2Params& P);

// mode: SV_FP64 / SV_FP32 storage
cudaError_t launch_gate1(void* psi, uint64_t n_elems, int mode, int q, const double* m8,
                         cudaStream_t st);
cudaError_t launch_gate2(void* psi, uint64_t n_elems, int mode, int qa, int qb, const double* m32,
                         cudaStream_t st);
cudaError_t launch_diag(void* psi, uint64_t n_elems, int mode, uint64_t mask, const double* f2,
                        cudaStream_t st);
cudaError_t launch_pair(void* a0, void* a1, uint64_t count, int mode, const double* m8,
                        cudaStream_t st);
// two buffers of `count` elements, a 4x4 over (in-buffer bit lo, buffer choice): the tier's chunk pairs
cudaError_t launch_pair2q(void* b0, void* b1, uint64_t count, int mode, int lo, int hi_is_b, const double* m32,
                          cudaStream_t st);
cudaError_t launch_quad(void* const* parts, uint64_t count, int mode, const double* m32,
                        cudaStream_t st);
cudaError_t launch_fused(void* psi, int mode, const FusedParams& p, cudaStream_t st);

// measurement: partial sums per CTA; see sv_measure.cu
struct MeasureParams {
    uint64_t n_tiles;
    uint64_t out_mask;
    uint64_t tile_mask;
    int n, k, b;
    int want_ones;                      // first pass: norm + ones for every local qubit
    int8_t tq[kMaxTileBits];
    uint32_t cross_pos;                 // tile positions whose cross terms are wanted
    int8_t oq[64];                      // out-of-tile qubits (ascending), count n - k
};
int measure_slots(int k, int n);        // doubles per CTA partial row

// register-resident FP64 measurement pass (sv_measure3.cu); same partial-row layout
struct Measure3Params {
    uint64_t n_tiles;
    int n, kbits, b, want_ones, n_segs, n_out, rbits;   // rbits: register bits per segment (3 or 4)
    int8_t tq[12];
    int8_t oq[64];
    uint8_t seg_reg[4][4];              // register bit j -> tile position
    uint8_t seg_thr[4][9];              // thread-id bit j -> tile position
    uint16_t seg_rsw[4][16];            // swizzled shared-memory offset of register slot i
    uint32_t cross_reg[4];              // register bits whose cross term the segment produces
    uint8_t swz_cols[4];                // shared-memory swizzle: columns XORed in by tile bits 3..6
    uint64_t pf_go[16];                 // HBM offset of tile element j * threads (prefetch chunks)
    uint64_t base_tab[4][256];          // tile index byte -> local-index bits outside the tile
    uint64_t base_const;                // index bits every tile carries (fixed bits of a tracked support)
    uint64_t pfix, pval;                // pfix != 0: amplitudes with (i & pfix) != pval load as zeros
    int direct;                         // segment 0 loads its registers from HBM (lanes = qubits 0..4)
    uint64_t seg0_go[16];               // direct: HBM offset of segment-0 register slot i
};
struct MeasureBytes {                   // BYTE planes + decode tables (dmag, dux, duy)
    const uint8_t* mi;
    const uint8_t* pi;
    const double* tab;
};
cudaError_t launch_measure3(const void* psi, const Measure3Params& p, double* partials, int grid, cudaStream_t st);
cudaError_t launch_measure3_byte(const MeasureBytes& b, const Measure3Params& p, double* partials, int grid,
                                 cudaStream_t st);
int measure3_grid(int device, int kb, bool byte);                       // partial rows to allocate
int measure3_ctas_per_sm(int kb, bool byte, const Measure3Params& p);   // the variant a pass runs
cudaError_t launch_measure(const void* psi, int mode, const MeasureParams& p, double* partials,
                           int grid, cudaStream_t st);
int measure_grid(int device);

int sm_count(int device);
extern int g_swap_blocks;               // grid cap of the group-swap kernels (sv_dist.cu), 0 = default
// caching state-slab allocator (sv_slab.cu): same-size reuse per device
cudaError_t slab_alloc(void** p, size_t bytes);
void keep_scratch_pool(int device);     // default pool keeps freed scratch (release threshold)
void slab_free(void* p, size_t bytes);
// CUDA IPC export: the slab is never returned to the driver until sv_ipc_unexport_all
void slab_mark_exported(void* p);
cudaError_t launch_swap_peer(void* own, void* peer, uint64_t n_local_elems, int mode, int l, int c, cudaStream_t st);
cudaError_t launch_swap_group(void* own, void* peer, uint64_t t0, uint64_t n, int mode, uint64_t vmask,
                              uint64_t own_pat, uint64_t peer_pat, uint64_t cmask, uint64_t cpat, cudaStream_t st);
cudaError_t launch_pair_dot(const void* a0, const void* a1, uint64_t n, int mode, double* partials, int grid,
                            cudaStream_t st);
cudaError_t launch_pair_dot_chunk(const void* a0, const void* a1, uint64_t t0, uint64_t n, uint64_t cmask,
                                  uint64_t cpat, int mode, double* partials, int grid, cudaStream_t st);
void count_launch(uint64_t n = 1);

}  // namespace sv
