// BYTE-mode device structures shared by sv_byte.cu and the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/svb200.h"

namespace sv {

// Codebook tables as the kernels read them: decode tables by original index
// (codec.py:203-206) and the ascending copies + original indices used by the
// nearest-entry search (codec.py:110-120, 193-201).
struct ByteTables {
    double dmag[256], dux[256], duy[256];    // must stay first (decode-fused measurement reads them)
    double smag[256], sth[256];
    uint8_t smag_idx[256], sth_idx[256];
    int n_mag, n_ph;
    double sqmid[256];                         // ((s[i] + s[i+1]) / 2)^2, +inf after the last
    double sqmag[256];                         // s[i]^2
};

// One gate pass (fields mirror svb_gate_desc in include/svb200.h).
struct ByteGate {
    int kind, qa, qb;
    uint64_t mask;
    double m[32];
    uint64_t n_elems;
    int n_local;
    int xkind;                  // 0 none, 1 pairwise-1q, 2 pairwise-2q, 3 quad (reference choreography)
    uint64_t xmask_a, xmask_b;  // partner rank masks
    int qlow_top;               // pairwise-2q: the local qubit is the top local bit
    int producer;               // -1: every work item; r: only items the reference's rank r computes;
                                // -2: every work item, candidates tagged with their producer rank
    uint64_t phys_base;         // this buffer's first physical global index
    int rank_bits;              // log2 of the reference rank count
    int8_t lbit[12];            // physical bit of logical bit (n_local - 2 + j)
    int collect, want_mag, want_ph;
    int mag_room, ph_room;      // free table entries (informational)
    double mag_cut, ph_cut;     // only values below the cut are collected (overflow retry)
    int scan_only;              // 1: collect candidates, write nothing
    int in_place;               // DIAG write pass into the input planes: untouched amplitudes
                                // are neither read nor written
    uint64_t sup_fixed;         // support: index bits every nonzero amplitude has equal to sup_val
    uint64_t sup_val;           // (0 = dense); the vector paths visit only those work items
};

// Candidate / uncertain-amplitude output of a pass (device memory).
struct ByteCand {
    unsigned long long n_mag, n_ph, n_unsure;
    unsigned long long cap_mag, cap_ph, cap_unsure;
    double* mag;                // distinct unrepresentable magnitudes
    double* ph;                 // per distinct theta: (re, im, ux, uy) of the min-(ux, uy) value
    int* mag_tag;               // producer rank of each candidate (tagged collection, producer == -2)
    int* ph_tag;
    unsigned long long* unsure_idx;
    double* unsure_val;         // (re, im)
    int overflow, any_mag, any_ph, pad;
};

cudaError_t byte_kernels_prepare();   // attributes + module load of the gate kernels (svb_create)
cudaError_t launch_byte_gate(const uint8_t* mi_in, const uint8_t* pi_in, uint8_t* mi_out, uint8_t* pi_out,
                             const ByteTables* tab, const ByteGate& g, ByteCand* cand, cudaStream_t st);
cudaError_t launch_byte_decode(const uint8_t* mi, const uint8_t* pi, const ByteTables* tab, double* out, uint64_t n,
                               cudaStream_t st);
cudaError_t launch_byte_encode(const double* vals, uint64_t n, const ByteTables* tab, uint8_t* mi, uint8_t* pi,
                               const ByteGate& g, ByteCand* cand, cudaStream_t st);
cudaError_t launch_byte_swap_group(uint8_t* omi, uint8_t* opi, uint8_t* pmi, uint8_t* ppi, uint64_t t0, uint64_t n,
                                   uint64_t vmask, uint64_t own_pat, uint64_t peer_pat, cudaStream_t st);
cudaError_t launch_byte_swap_peer(uint8_t* omi, uint8_t* opi, uint8_t* pmi, uint8_t* ppi, uint64_t n_local_elems,
                                  int l, int c, cudaStream_t st);
cudaError_t launch_byte_pair_dot(const uint8_t* ami, const uint8_t* api, const uint8_t* bmi, const uint8_t* bpi,
                                 const ByteTables* tab, uint64_t n, double* partials, int grid, cudaStream_t st);
cudaError_t launch_byte_patch(uint8_t* mi, uint8_t* pi, const uint64_t* idx, const uint8_t* nm, const uint8_t* np_,
                              uint64_t n, cudaStream_t st);

}  // namespace sv
