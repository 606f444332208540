// cbp_internal.h -- host/device shared definitions of libcbp (not part of the ABI).
#pragma once
#include <cstdint>

namespace cbp {

// Schedule tables: two int4 per nonzero base entry, byte offsets scaled for the
// launch geometry's frames per lane P (layout documented in cbp_kernels.cu).
struct DevCode {
    int32_t N, K, M, Z, mb, nb, kb, core;
    int32_t nent, E, nwords, kwords;
    int32_t max_dc;
    int32_t can_encode;
    int32_t mid;           // floor(core/2)
    const float4* phi_tab; // [kPhiTableSegs] phi contract v3 coefficients
    unsigned long long phi_tex;   // cudaTextureObject_t over phi_tab (float4 elements)
};

// MODE_BER_LLR: the decode half of a split cbp_ber_sim -- fp32 LLRs and the transmitted codewords from
// HBM (written by a MODE_CHANNEL launch of the same kernel), error counting as in MODE_BER_SIM
enum Mode : int32_t { MODE_DECODE_F32 = 0, MODE_DECODE_I8 = 1, MODE_BER_SIM = 2, MODE_CHANNEL = 3, MODE_BER_LLR = 4 };

// Limits of the schedule tables carried in the kernel parameters (constant bank):
// read through the constant cache, they take no shared-memory bandwidth.
constexpr int kMaxEnt = 512;    // nonzero base entries
constexpr int kMaxRows = 128;   // base rows

struct KernelArgs {
    DevCode code;
    int4 ent[2 * kMaxEnt];          // schedule entries of this geometry (cbp_kernels.cu)
    int32_t row_ptr[kMaxRows + 1];  // entry range of base row i
    int16_t pshift[kMaxRows];       // shift of column kb in row i (-1 if none)
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
    int32_t ctl_words;     // shared control words per team (multi-warp teams; warp teams: syndrome scratch)
    int32_t fast_syn;      // warp teams with Z <= 32 and mb <= Zp: ballot-packed syndromes
    uint32_t phi_m19, phi_one;     // 0x7ffff, 0x3f800000 (phi local variable, runtime operands)
    const int4* ent_dev;   // device copy of `ent` (bulk-copied into shared memory by cbp_warp_kernel)
    int32_t lanes;         // cbp_warp_kernel: lanes with check slots, L = ceil(Z / K)
    float* gstate;         // per-CTA global state (state_in_smem == 0)
    float* rstate;         // per-group R sections of the split layout (r_global), r_words each
    int32_t r_words;
    const uint32_t* cw_in; // MODE_BER_LLR: transmitted codewords [frames][ld_words]
};

// phi lookups through the texture pipe (C2B default on, B2V default off)
#ifndef CBP_TEX_C2B
#define CBP_TEX_C2B 1
#endif
#ifndef CBP_TEX_B2V
#define CBP_TEX_B2V 0
#endif

// thread limits (launch bounds) of cbp_warp_kernel: K = 1 (Z <= 32) and K >= 2 check slots per lane
#ifndef CBP_WARPK1_MAXT
#define CBP_WARPK1_MAXT 512
#endif
#ifndef CBP_WARPK_MAXT
#define CBP_WARPK_MAXT 640
#endif

// thread limit of cbp_warp_kernel's team instantiations (one frame per CTA)
#ifndef CBP_WARPT_MAXT
#define CBP_WARPT_MAXT 384
#endif

// rows with at most CBP_DC_REG edges are updated from registers, longer rows by the park path
#ifndef CBP_DC_REG
#define CBP_DC_REG 8
#endif
#ifdef __CUDACC__
#define CBP_HD __host__ __device__
#else
#define CBP_HD
#endif
// cbp_warp_kernel per-warp state, in 32-bit words (cbp_warp.cuh):
//   counters [16] | Lambda [N floats] | H [N bytes] | cw [nwords] | park buffer | R (if in shared) | S [M] (Omega)
CBP_HD inline int warp_hb_words(int N) { return (N + 15) / 16 * 4; }          // N bytes, 16-byte padded
CBP_HD inline int warp_cw_words(int nwords) { return (nwords + 3) / 4 * 4; }
CBP_HD inline int warp_pb_words(int max_dc) { return max_dc > CBP_DC_REG ? max_dc * 32 : 0; }   // park rows' Phi

// thread limit (launch bound) of the one-frame-per-lane warp-team instantiation
#ifndef CBP_WARP_MAXT
#define CBP_WARP_MAXT 512
#endif

// shared control words per multi-warp team: row reduction [2 buffers][P <= 2][first 32 | last 32 per warp]
// + the queue-index broadcast (2 x int64)
constexpr int kCtlTeamWords = 264;

struct Geometry {
    int32_t threads, F, Zp, slot_words, table_words, smem_bytes, state_in_smem, multi;
    int32_t team_threads, teams;   // threads per team, teams per CTA
    int32_t alg;                   // cbp_algorithm of this geometry
    int32_t P;                     // frames per lane (1 or 2), interleaved in a group
    int32_t ctl_words, fast_syn;   // see KernelArgs
    int32_t r_global, r_words;     // split layout: R in the global workspace, r_words per group
    int32_t wk;                    // 1: cbp_warp_kernel (one frame per warp, K check slots per lane)
    int32_t kslots, lanes;         // cbp_warp_kernel: K and L = ceil(Z / K)
    int32_t tex2;                  // cbp_warp_kernel phi rows: 0 C2B through TEX, 1 both (no smem table), 2 none
};

// launch (cbp_kernels.cu); returns cudaError_t as int
int launch_cbp(const KernelArgs& a, const Geometry& g, int grid, void* stream);
int occupancy_ctas_per_sm(const Geometry& g, int* out);
int launch_contract_eval(int fn, const float* x, float* y, int64_t n, const float4* tab, void* stream);
constexpr int kPhiTableSegs = 1153;   // phi contract v3 (contract.cuh kPhiSegs)

}  // namespace cbp
