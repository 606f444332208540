// cbp_internal.h -- host/device shared definitions of libcbp (not part of the ABI).
#pragma once
#include <cstdint>

namespace cbp {

// Per nonzero base entry b (row-major over nonzero entries), packed in an int4:
//   x = var_base (j*Z)            | s_prev_base (row(prev(b))*Z) << 16
//   y = shift s | ds << 11 | first << 22 | self << 23
//       ds = (s - s_prev) mod Z: lifted row of the previous check of the same
//       variable is (r + ds) mod Z; first: b is the first nonzero row of its
//       column (no latest check in sweep 1, reading R1); self: prev(b) == b
//       (degree-1 column, reading R3)
//   z = R slot base of b      (b*Z; edge (check i*Z+r, its variable) = z + r)
//   w = R slot base of prev(b)
struct DevCode {
    int32_t N, K, M, Z, mb, nb, kb, core;
    int32_t nent, E, nwords, kwords;
    int32_t max_dc;
    int32_t can_encode;
    int32_t mid;           // floor(core/2)
    const int4* ent;       // [nent]
    const int32_t* row_ptr;// [mb+1]
    const int16_t* pshift; // [mb]: shift of column kb in row i (-1 if none)
    const float4* phi_tab; // [929] phi contract v2 coefficients
};

enum Mode : int32_t { MODE_DECODE_F32 = 0, MODE_DECODE_I8 = 1, MODE_BER_SIM = 2, MODE_CHANNEL = 3 };

struct KernelArgs {
    DevCode code;
    int32_t mode;
    int32_t max_iter, stop_rule;
    int32_t algorithm;     // 0 log-tanh, 1 normalized min-sum
    float alpha;           // min-sum normalisation
    int32_t llr_mode;
    // inputs
    const float* llr;
    const int8_t* q;
    int64_t ld;
    float qscale;
    int64_t frames;
    int64_t frame_begin;
    uint64_t seed;
    float sigma, scale;
    // outputs
    uint32_t* bits;
    int64_t ld_words;
    int32_t* iters;
    uint8_t* flags;
    float* omega;
    int64_t* ev;
    float* llr_out;        // MODE_CHANNEL
    uint32_t* cw_out;      // MODE_CHANNEL
    unsigned long long* counts;   // MODE_BER_SIM: 8 x int64
    unsigned long long* queue;    // frame work counter (zeroed)
    // geometry
    int32_t Zp, F, slot_words, table_words, team_threads;
    uint32_t phi_m19, phi_one;     // 0x7ffff, 0x3f800000 (phi local variable, runtime operands)
    float* gstate;         // per-CTA global state (state_in_smem == 0)
};

constexpr int kCtlTeamWords = 72;   // shared control words per team: 2 x 32 ballot words + broadcast

struct Geometry {
    int32_t threads, F, Zp, slot_words, table_words, smem_bytes, state_in_smem, multi;
    int32_t team_threads, teams;   // threads per team, teams per CTA
    int32_t alg;                   // cbp_algorithm of this geometry
};

// launch (cbp_kernels.cu); returns cudaError_t as int
int launch_cbp(const KernelArgs& a, const Geometry& g, int grid, void* stream);
int occupancy_ctas_per_sm(const Geometry& g, int* out);
int launch_contract_eval(int fn, const float* x, float* y, int64_t n, const float4* tab, void* stream);
int launch_phi_table(float4* out, void* stream);
constexpr int kPhiTableSegs = 929;

}  // namespace cbp
