/*
 * svb200.h — C ABI of the B200-native gate-application hot path.
 *
 * Drop-in boundary for the reference package `svsim`
 * (/root/reference/pkg/src/svsim).  The reference is pure Python + numpy and
 * has no FFI of its own; the entry points below are what its hot-path
 * operators bind to when they are re-pointed at this library (the ctypes
 * binding lives in paper_2511_03359_b200/_native.py; INTEGRATION.md shows
 * the stub a reference maintainer would add).  Each entry point names the
 * reference interface it replaces.
 *
 * Conventions
 *   - plain C types only: pointers, sizes, int status codes;
 *   - every function returns SV_OK (0) or a negative SV_E* code, and the
 *     message of the last failure on the calling thread is available from
 *     sv_last_error();
 *   - SV_EINDEX maps to Python IndexError, SV_EVALUE to ValueError,
 *     SV_ECUDA / SV_ENOMEM to RuntimeError / MemoryError, matching the
 *     reference's exception types (kernels.py:23-24, 34-35, 49-52);
 *   - amplitude storage: SV_FP64 = interleaved complex128 (16 B),
 *     SV_FP32 = interleaved complex64 (8 B) (state.py:20-27);
 *   - a matrix is row-major complex entries as (re, im) doubles:
 *     2x2 -> 8 doubles, 4x4 -> 32 doubles, basis index bit(qa) + 2*bit(qb)
 *     (gates.py:24, kernels.py:46).
 *   - "svk_*" functions take raw device pointers and a cudaStream_t (passed
 *     as void*), "sv_*" functions take a state handle that owns its device
 *     memory and stream.
 */
#ifndef SVB200_H
#define SVB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SV_ABI_VERSION 3

enum { SV_OK = 0, SV_EINDEX = -1, SV_EVALUE = -2, SV_ECUDA = -3, SV_ENOMEM = -4 };
enum { SV_FP64 = 0, SV_FP32 = 1, SV_BYTE = 2 };              /* state.py:20-27 PrecisionMode */
enum { SV_OP_1Q = 1, SV_OP_2Q = 2, SV_OP_DIAG = 3 };

typedef struct sv_state* sv_handle;

/* One gate of a fused pass (see sv_apply_fused). */
typedef struct {
    int32_t kind;          /* SV_OP_1Q / SV_OP_2Q / SV_OP_DIAG */
    int32_t qa, qb;        /* local qubits (qb unused for 1Q; unused for DIAG) */
    int32_t reserved;
    uint64_t diag_mask;    /* DIAG: local-index bits that must all read 1 */
    double m[32];          /* 1Q: 8 doubles, 2Q: 32 doubles, DIAG: factor (re, im) */
} sv_op;

/* ---- library -------------------------------------------------------- */
int sv_abi_version(void);
const char* sv_last_error(void);
int sv_device_count(int* count);
int sv_sm_count(int device, int* count);
/* free / total device memory in bytes (cudaMemGetInfo) */
int sv_mem_info(int device, uint64_t* free_bytes, uint64_t* total_bytes);
/* make `device` current on the calling thread (svk_* launch on the current device) */
int sv_set_device(int device);

/* ---- raw device-pointer kernels (one call = one kernel launch) ------ */
/* kernels.py:30-40 apply_single: in-place 2x2 on pairs (i, i + 2^q) of a
 * buffer of n_elems amplitudes (n_elems a multiple of 2^(q+1)). */
int svk_apply_1q(void* psi, uint64_t n_elems, int mode, int q, const double* m8, void* stream);
/* kernels.py:43-64 apply_two: in-place 4x4 on the quadruples of (qa, qb). */
int svk_apply_2q(void* psi, uint64_t n_elems, int mode, int qa, int qb, const double* m32,
                 void* stream);
/* kernels.py:67-81 apply_diagonal: multiply (array first) where all bits of
 * mask are 1; mask == 0 scales the whole buffer. */
int svk_apply_diag(void* psi, uint64_t n_elems, int mode, uint64_t mask, const double* f2,
                   void* stream);
/* kernels.py:84-88 apply_pair_arrays, in place over two aligned buffers
 * (a1 may be a peer-GPU pointer: the exchange-fused update). */
int svk_pair_update(void* a0, void* a1, uint64_t count, int mode, const double* m8, void* stream);
/* kernels.py:91-98 apply_quad_arrays, in place over four aligned buffers. */
int svk_quad_update(void* const* parts, uint64_t count, int mode, const double* m32,
                    void* stream);
/* engine.py:166-180 run of local gates as ONE pass over HBM: ops applied in
 * order, each with the reference arithmetic, on tiles of 2^tile_bits
 * amplitudes staged in shared memory. n_elems must be a power of two. */
int svk_apply_fused(void* psi, uint64_t n_elems, int mode, const sv_op* ops, int n_ops,
                    int tile_bits, void* stream);
/* measure.py:51-56 + 59-109: norm, per-qubit one-weights and cross sums of
 * a buffer of 2^n amplitudes.  ones[n], cross[2n] (re, im). */
int svk_measure(const void* psi, uint64_t n_elems, int mode, double* norm, double* ones,
                double* cross, void* stream);

/* ---- state handles (state.py:34-103 LocalState) --------------------- */
int sv_create(int device, int n_qubits, int mode, sv_handle* out);
int sv_destroy(sv_handle h);
/* state.py:49-63 zero_state: all zeros, amplitude 1 at index `unit` (-1: none) */
int sv_zero_state(sv_handle h, int64_t unit);
/* the same state, recorded only: the first fused pass generates its tiles instead of reading
 * them (no memset, one HBM read fewer); every other entry point writes the state first */
int sv_zero_state_lazy(sv_handle h, int64_t unit);
int sv_info(sv_handle h, int* device, int* n_qubits, int* mode, void** dev_ptr, void** stream);
int sv_apply_1q(sv_handle h, int q, const double* m8);
int sv_apply_2q(sv_handle h, int qa, int qb, const double* m32);
int sv_apply_diag(sv_handle h, uint64_t mask, const double* f2);
int sv_apply_fused(sv_handle h, const sv_op* ops, int n_ops, int tile_bits);
/* fused passes of ops restricted to the local indices whose bits under chunk_mask equal
 * chunk_pattern (chunk bits must lie outside every pass's tile) */
int sv_apply_fused_chunk(sv_handle h, const sv_op* ops, int n_ops, int tile_bits, uint64_t chunk_mask,
                         uint64_t chunk_pattern);
int sv_measure(sv_handle h, double* norm, double* ones, double* cross);
/* raw storage elements [first, first+count) <-> host memory */
int sv_export(sv_handle h, void* host, uint64_t first, uint64_t count);
int sv_import(sv_handle h, const void* host, uint64_t first, uint64_t count);
int sv_synchronize(sv_handle h);

/* ---- BYTE mode: adaptive two-byte polar encoding (codec.py) ---------- */
typedef struct sv_bstate* sv_bhandle;

/* One gate pass over a BYTE state (engine.py:186-215, 229-377). */
typedef struct {
    int32_t kind;          /* SV_OP_1Q / SV_OP_2Q / SV_OP_DIAG */
    int32_t qa, qb;
    int32_t n_local;       /* reference rank layout: local qubits per rank */
    uint64_t diag_mask;
    double m[32];          /* matrix (1Q/2Q) or diagonal factor (re, im) */
    int32_t xkind;         /* 0 none, 1 pairwise 1q, 2 pairwise 2q, 3 quad (engine.py choreography) */
    int32_t qlow_top;      /* pairwise 2q: the local qubit is the top local bit */
    uint64_t xmask_a, xmask_b;
    int32_t producer;      /* -1 all work items; r: only those reference rank r computes;
                            * -2 all work items, candidates tagged with their reference rank */
    int32_t collect;       /* collect codebook proposals (codec.py:137-152) */
    int32_t want_mag, want_ph;   /* which tables can still change */
    double mag_cut, ph_cut;      /* collect only values below the cut (overflow retry) */
    int32_t scan_only;           /* 1: only collect candidates, write nothing */
    int32_t rank_bits;           /* log2(reference rank count) */
    uint64_t phys_base;          /* physical global index of this buffer's element 0 */
    int8_t lbit[16];             /* physical bit of logical bit n_local - 2 + j (j = 0, 1: offset
                                  * top bits; j >= 2: rank bits); identity when not remapped */
    int32_t ph_zero_in;          /* 1: every phase index of the input planes is 0 (the phase table
                                  * held one entry whenever a plane was written): not read */
    int32_t ph_zero_out;         /* 1: this pass's phase table has one entry, every output phase
                                  * index is 0 and the output phase plane already holds zeros:
                                  * not written */
    uint64_t sup_fixed;          /* support: bits every nonzero amplitude shares with sup_val (0 =
                                  * dense); both plane buffers must hold zeros outside it and it
                                  * may only grow (byte_state.py tracks it) */
    uint64_t sup_val;
} svb_gate_desc;

int svb_create(int device, int n_qubits, sv_bhandle* out);
int svb_destroy(sv_bhandle h);
int svb_info(sv_bhandle h, int* device, int* n_qubits, void** stream);
/* state.py:49-63: all zero bytes, magnitude index 1 (= 1.0) at `unit`; both buffers'
 * phase planes are zeroed (ph_zero_out passes rely on it) */
int svb_zero_state(sv_bhandle h, int64_t unit);
/* upload the codebook (append order, codec.py:100-106); sorted copies are
 * built here with a stable argsort (codec.py:112-120) */
int svb_set_tables(sv_bhandle h, const double* mags, int n_mag, const double* thetas, const double* ux,
                   const double* uy, int n_ph);
/* one pass: reads the current planes, writes the pending planes */
int svb_gate(sv_bhandle h, const svb_gate_desc* g);
/* svb_measure over a tracked support (sup_fixed / sup_val as in svb_gate_desc) */
int svb_measure_support(sv_bhandle h, uint64_t sup_fixed, uint64_t sup_val, double* norm, double* ones,
                        double* cross);
/* diagonal gate, final write pass (tables fixed: saturated, or scanned and
 * merged first): rewrites only the selected amplitudes of the CURRENT planes
 * (engine.py:186-225 encode step of a diagonal gate; no commit follows) */
int svb_gate_in_place(sv_bhandle h, const svb_gate_desc* g);
/* candidates of the passes since the last reset: distinct magnitudes and,
 * per distinct theta, (re, im, ux, uy) of its smallest-(ux, uy) value
 * (duplicates possible).  flags: 1 = a buffer overflowed (retry with a cut),
 * 2 = at least one magnitude candidate was seen */
int svb_candidates(sv_bhandle h, double* mags, uint64_t cap_m, uint64_t* n_m, double* ph4, uint64_t cap_p,
                   uint64_t* n_p, int* flags);
/* producer rank of every candidate returned by svb_candidates after a pass with
 * producer == -2 (tagged collection: one pass for all reference ranks) */
int svb_candidate_tags(sv_bhandle h, int32_t* mag_tags, uint64_t cap_m, int32_t* ph_tags, uint64_t cap_p);
/* amplitudes whose phase decision was inside the atan2 margin */
int svb_unsure(sv_bhandle h, uint64_t* idx, double* vals, uint64_t cap, uint64_t* n);
int svb_reset(sv_bhandle h);
/* overwrite bytes of the pending planes (host-resolved uncertain amplitudes) */
int svb_patch(sv_bhandle h, const uint64_t* idx, const uint8_t* mi, const uint8_t* pi, uint64_t n);
/* the same on the current planes (after svb_gate_in_place) */
int svb_patch_in_place(sv_bhandle h, const uint64_t* idx, const uint8_t* mi, const uint8_t* pi, uint64_t n);
/* pending planes become current */
int svb_commit(sv_bhandle h);
int svb_export(sv_bhandle h, uint8_t* mi, uint8_t* pi, uint64_t first, uint64_t count);
int svb_import(sv_bhandle h, const uint8_t* mi, const uint8_t* pi, uint64_t first, uint64_t count);
/* decoded complex128 amplitudes [first, first+count) to host */
int svb_decode(sv_bhandle h, double* out, uint64_t first, uint64_t count);
/* measure.py on the decoded state (FP64 sums) */
int svb_measure(sv_bhandle h, double* norm, double* ones, double* cross);
/* array-level codec: encode n complex128 host values with the handle's tables
 * (codec.py:193-201); with collect != 0 also gather proposals into the
 * handle's candidate buffers (codec.py:137-152) */
int svb_encode_values(sv_bhandle h, const double* vals, uint64_t n, uint8_t* mi, uint8_t* pi, int collect);

/* ---- multi-GPU: CUDA IPC + NVLink peer kernels ------------------------ */
/* 64-byte IPC handle of the handle's state buffer */
int sv_ipc_handle(sv_handle h, void* out64);
/* map a peer's state buffer into this process (device = this rank's GPU) */
int sv_ipc_open(int device, const void* handle64, void** peer_ptr);
int sv_ipc_close(int device, void* peer_ptr);
/* every state buffer exported by sv_ipc_handle / svb_ipc_handles stays allocated
 * (never returned to the driver by the slab cache) until this is called -- only
 * after every peer process has closed its mappings (a collective barrier).
 * was_exported (optional) = how many buffers were marked. */
int sv_ipc_unexport_all(uint64_t* was_exported);
/* global<->local qubit swap with the partner rank (the remap planner's move):
 * this rank has global bit `side`; its amplitudes with local bit l = 1-side
 * trade places with the partner's amplitudes with bit l = side.  Both ranks
 * call it; each moves half of the pairs.  n_local_elems = 2^n'. */
int svk_swap_peer(void* own, void* peer, uint64_t n_local_elems, int mode, int l, int side, void* stream);
/* batched remap (k global qubits at once, one member pair of the 2^k group):
 * this rank's amplitudes whose bits under victim_mask equal own_pattern trade
 * places with the peer's amplitudes whose victim bits equal peer_pattern, for
 * the remaining-bit indices [t_begin, t_begin + t_count). */
int svk_swap_group(void* own, void* peer, uint64_t n_local_elems, int mode, uint64_t victim_mask,
                   uint64_t own_pattern, uint64_t peer_pattern, uint64_t t_begin, uint64_t t_count, void* stream);
/* the same restricted to the amplitudes whose bits under chunk_mask equal chunk_pattern
 * (t runs over the bits outside victim_mask and chunk_mask): one chunk of a swap that
 * overlaps the following fused pass (sv_apply_fused_chunk) */
/* grid cap (blocks) of the group-swap kernel, 0 = one full wave; returns the
 * previous value (a negative argument only queries) */
int sv_swap_blocks(int blocks);
/* measurement-pass CTA slots to leave free (at most one wave of 2 per SM is launched) so
 * a concurrent pair dot (svk_pair_dot on another stream, grid capped by its max_blocks)
 * is resident at the same time; returns the previous value (negative: query) */
int sv_measure_reserve(int ctas);
int svk_swap_group_chunk(void* own, void* peer, uint64_t n_local_elems, int mode, uint64_t victim_mask,
                         uint64_t own_pattern, uint64_t peer_pattern, uint64_t chunk_mask, uint64_t chunk_pattern,
                         uint64_t t_begin, uint64_t t_count, void* stream);
/* sum conj(a0[i]) * a1[i] over count elements (a1 may be a peer pointer):
 * measure.py:83-101 cross term of a global qubit; out2 = (re, im).
 * max_blocks caps the grid (0 = two CTAs per SM). */
int svk_pair_dot(const void* a0, const void* a1, uint64_t count, int mode, int max_blocks, double* out2,
                 void* stream);
/* the same over the elements of [0, n_elems) whose bits under chunk_mask equal chunk_pattern,
 * rest indices [t_begin, t_begin + t_count) (t runs over the bits outside chunk_mask): the
 * cross term of a global qubit of a state whose tracked support fixes those bits */
int svk_pair_dot_chunk(const void* a0, const void* a1, uint64_t n_elems, int mode, uint64_t chunk_mask,
                       uint64_t chunk_pattern, uint64_t t_begin, uint64_t t_count, int max_blocks, double* out2,
                       void* stream);

/* BYTE multi-GPU: IPC handles of the 4 planes ([buffer][magnitude, phase]),
 * mapped peer planes, byte-plane swap and decoded cross term */
int svb_ipc_handles(sv_bhandle h, void* out256);
int svb_cur(sv_bhandle h);
int svb_swap_peer(sv_bhandle h, void* peer_mi, void* peer_pi, int l, int side);
/* zeros into the pending planes (a tracked support after a remap swap of the current planes) */
int svb_clear_pending(sv_bhandle h);
/* BYTE planes form of svk_swap_group (current planes of this rank and the peer) */
int svb_swap_group(sv_bhandle h, void* peer_mi, void* peer_pi, uint64_t victim_mask, uint64_t own_pattern,
                   uint64_t peer_pattern, uint64_t t_begin, uint64_t t_count);
int svb_pair_dot(sv_bhandle h, const void* a_mi, const void* a_pi, const void* b_mi, const void* b_pi,
                 uint64_t count, double* out2);
/* device pointers of the current planes (for offsets into own / peer planes) */
int svb_planes(sv_bhandle h, void** cur_mi, void** cur_pi);

/* ---- two-tier state: HBM + pinned host memory (svsim/tier.py executed) ----
 * 2^n amplitudes in chunks of 2^chunk_qubits; chunk g stays in HBM when fast[g] != 0
 * (TierAccount.fast_resident, tier.py:156-178), else lives in pinned host memory and is
 * staged through `slots` HBM chunk slots (tier.py STAGING_SLOTS = 4). */
typedef struct sv_tier* sv_thandle;
int svt_create(int device, int n_qubits, int mode, int chunk_qubits, const uint8_t* fast, int slots,
               sv_thandle* out);
int svt_destroy(sv_thandle h);
int svt_zero_state(sv_thandle h, int64_t unit);
/* a "run" staging group (tier.py:121-129): ops on qubits < chunk_qubits or diagonal */
int svt_apply_run(sv_thandle h, const sv_op* ops, int n_ops, int tile_bits);
/* one non-diagonal gate with a qubit >= chunk_qubits ("mid" / "exchange" groups,
 * tier.py:130-143): chunk groups co-staged and updated in place */
int svt_apply_pairing(sv_thandle h, const sv_op* op);
/* measure.py sums over the whole state (slow chunks staged in once) */
int svt_measure(sv_thandle h, double* norm, double* ones, double* cross);
int svt_export(sv_thandle h, void* host, uint64_t first, uint64_t count);
int svt_import(sv_thandle h, const void* host, uint64_t first, uint64_t count);
int svt_synchronize(sv_thandle h);
/* physical counters: h2d bytes, d2h bytes, h2d copies, d2h copies, zero-copy bytes,
 * slot memsets (never-written chunks), kernel passes, HBM bytes of the fast tier */
int svt_stats(sv_thandle h, uint64_t* out8);

/* FP32-storage rounding check: host values rounded on the device to float precision by
 * the specialised passes' methods -- F2F (mode 0), Veltkamp split on the FP64 pipe (1),
 * integer add-and-mask of the double's bits (2) -- returned as doubles */
int svk_f32_round(const double* host_in, double* host_out, uint64_t n, int mode);

/* ---- raw device buffers (for the array-level operator API) --------- */
int sv_buffer_alloc(int device, uint64_t bytes, void** ptr);
int sv_buffer_free(int device, void* ptr);
int sv_copy_h2d(void* dst, const void* src, uint64_t bytes, void* stream);
int sv_copy_d2h(void* dst, const void* src, uint64_t bytes, void* stream);
int sv_stream_create(int device, void** stream);
int sv_stream_destroy(void* stream);

/* ---- instrumentation ------------------------------------------------ */
/* number of kernels this library has launched in the process */
int sv_launch_count(uint64_t* count);
/* host<->device bytes this library has moved (copies plus the kernel-
 * parameter blocks of fused passes, which the driver ships per launch) */
int sv_transfer_bytes(uint64_t* h2d, uint64_t* d2h);
/* select the fused-pass kernel (FP64): 0 = shared-memory-per-gate v1;
 * register-resident cp.async-pipelined v3 with 1 = 2^12 tiles x 16 amplitudes
 * per thread, 2 = 2^11 tiles x 8 per thread (2 CTAs/SM), 3 = 2^12 tiles x 8
 * per thread (512 threads).  FP32 storage always uses v1. */
/* state slabs freed by sv_destroy / svb_destroy are cached per device and reused
 * for the next allocation of the same size; release them to the driver: */
int sv_release_cached(void);
int sv_cached_bytes(uint64_t* out);
/* run-time specialised fused passes (NVRTC, one kernel per pass structure; see
 * paper_2511_03359_b200/csrc/sv_jit.cu): mode 0 off, 1 compile-and-wait,
 * 2 compile in the background and run the generic kernel meanwhile (default).
 * Returns the previous mode.  Both kernels are bit-identical. */
int sv_jit_mode(int mode);
int sv_jit_wait(void);                        /* block until queued compiles finish */
int sv_jit_shutdown(void);                    /* drop queued compiles, wait for running ones (call
                                               * before process teardown; registered with atexit) */
/* plan the fused passes sv_apply_fused would run for ops on 2^n_qubits FP64
 * amplitudes and queue their specialised kernels (no launch, no device needed);
 * returns the number of new kernels queued */
int sv_jit_prepare(int n_qubits, const sv_op* ops, int n_ops, int tile_bits);
int sv_jit_prepare_mode(int n_qubits, int mode, const sv_op* ops, int n_ops, int tile_bits);  /* FP64 / FP32 */
/* flags bit 0: the kernels of combined diagonal runs (sv_set_diag_combine) */
int sv_jit_prepare_opts(int n_qubits, int mode, const sv_op* ops, int n_ops, int tile_bits, int flags);
/* FP64 handles: runs of consecutive diagonal ops inside a fused pass multiply each
 * amplitude by the product of their factors (one multiply per distinct register mask)
 * instead of one rounding per gate -- amplitudes within 1e-12 relative of the
 * reference (the north star's FP64 tolerance), NOT bit-identical.  Default off. */
int sv_set_diag_combine(sv_handle h, int on);
/* Support tracking (default off; run_circuit turns it on for its state): after
 * sv_zero_state[_lazy](h, unit) the handle records which index bits may differ from
 * unit's -- freed by non-monomial gates, moved by monomials, untouched by diagonal
 * gates -- and fused passes run only the tiles that can hold nonzero amplitudes.
 * Results are identical (the skipped amplitudes are zeros that stay zero); writes
 * through the raw device pointer require turning tracking off first.  sv_import,
 * sv_apply_fused_chunk and all-zero states turn it off. */
int sv_set_support_tracking(sv_handle h, int on);
int sv_support_info(sv_handle h, int* on, uint64_t* free_mask, uint64_t* val, uint64_t* tiles_skipped);
/* set the tracked support explicitly ({i : (i & ~free_mask) == val}; tracking on) -- the
 * distributed layer's rank slice of the global support after a remap swap */
int sv_set_support(sv_handle h, uint64_t free_mask, uint64_t val);
/* host only: move a support through ops by the rule the passes apply (non-monomial 1Q/2Q
 * ops free their qubits, monomials on fixed qubits move val, diagonal ops keep it) */
int sv_support_advance(const sv_op* ops, int n_ops, uint64_t* free_mask, uint64_t* val);
/* the pass split sv_apply_fused uses for ops: ends[p] = one past the last op of pass p;
 * returns the number of passes (also queues their specialised kernels) */
int sv_plan_passes(int n_qubits, int mode, const sv_op* ops, int n_ops, int tile_bits, int* ends, int cap);
/* the same split without queueing kernels, plus each pass's FP64 warp instructions per
 * amplitude in its specialised kernel (fp64_per_amp[p] = -1: generic kernel); the
 * FP64 floor of a pass is that x 2^n / (64 lanes x SMs x SM clock) -- bench.py roofline */
int sv_plan_pass_costs(int n_qubits, int mode, const sv_op* ops, int n_ops, int tile_bits, int* ends,
                       double* fp64_per_amp, int cap, int flags);   /* flags bit 0: combined diagonal runs */
int sv_jit_stats(double* out8);               /* compiled, failed, jit launches, fallbacks, compile ms, cached,
                                                 disk-cache hits, disk-cache writes ($SVB200_JIT_CACHE) */
int sv_jit_available(void);                   /* 1 when NVRTC and the driver entry points resolved */
/* CPU-side check: plan the first fused pass of ops on 2^n_qubits amplitudes, write
 * its specialised source to src_out and, when compile_ms is non-NULL, compile it
 * with NVRTC.  Returns the number of ops in the pass (>= 1) or an error code. */
int sv_jit_probe(const sv_op* ops, int n_ops, int n_qubits, char* src_out, size_t cap, double* compile_ms);
int sv_fused_variant(int v2);
/* passes whose v3 plan needs more than `limit` register segments use v1
 * instead (0 = no limit) */
int sv_fused_segment_limit(int limit);
/* per-launch CUDA-event timing of fused passes (off by default): when on,
 * every fused-pass kernel is bracketed by events on its own stream */
int sv_pass_timing(int enable);
/* passes timed since the last call, their summed device time (ms) and the
 * summed algorithmic bytes (one read + one write of the buffer per pass);
 * synchronises on the recorded events and resets the record */
int sv_pass_timing_read(uint64_t* passes, double* ms, double* bytes);

/* ---- device timing (CUDA events on the handle's / given stream) ------ */
int sv_event_create(void** ev);
int sv_event_destroy(void* ev);
/* inter-process events (cross-GPU ordering of chunked swaps and passes) */
int sv_event_create_ipc(void** ev, void* handle_out64);
int sv_event_open_ipc(const void* handle64, void** ev);
int sv_stream_wait_event(void* stream, void* ev);
int sv_event_record(void* ev, void* stream);
int sv_event_elapsed_ms(void* start, void* stop, float* ms);
int sv_stream_synchronize(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SVB200_H */
