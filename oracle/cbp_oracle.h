/*
 * cbp_oracle.h -- plain, slow, single-threaded CPU ORACLE of check-belief
 * propagation (CBP) decoding, §IV-C Steps 1-3 (l.400-487) and hidden
 * Algorithm 1 (l.493-523), with the readings listed in DESIGN.md §2.
 *
 * THIS IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load liboracle.so.
 * It shares no code with the CUDA path (paper_2305_05286_b200/); the only
 * common source is the seeded input generator inputs/qc_construct.c, which
 * holds none of the method's arithmetic.
 *
 * All pointers are host pointers owned by the caller.  Functions return 0 on
 * success and a nonzero code on invalid arguments.
 */
#ifndef CBP_ORACLE_H
#define CBP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_code or_code;

/* Expand a QC base matrix (int16 mb x nb, -1 = zero block, s = shift; check row
 * r of block (i,j) <-> variable j*Z + (r+s)%Z) into the code graph
 * G = (V, C, E) of PAPER.md l.92.  Edge ids are row-major: checks ascending,
 * variables ascending within a check. */
or_code* oracle_code_create(const int16_t* base, int32_t mb, int32_t nb, int32_t Z);
void     oracle_code_destroy(or_code* c);
void     oracle_code_dims(const or_code* c, int32_t* N, int32_t* K, int32_t* M, int64_t* E);
/* edges in id order: chk[e], var[e] (each array E entries) */
void     oracle_code_edges(const or_code* c, int32_t* chk, int32_t* var);

/* stop rules (readings R4-R6) */
enum { OR_STOP_BELIEF_M = 0, OR_STOP_BELIEF_N = 1, OR_STOP_SYNDROME = 2, OR_STOP_NONE = 3 };
/* arithmetic */
enum { OR_FP32_CONTRACT = 0,   /* fp32, phi from the arithmetic contract (parity reference) */
       OR_FP64 = 1,            /* fp64, phi = log1p(2/expm1(x)) (= -log tanh(x/2)), phi-domain C2B */
       OR_FP64_LITERAL = 2,    /* fp64, literal psi+ recursion of equ_s4e5/equ_s4e6 (test variant) */
       OR_MINSUM = 3,          /* fp32 normalized min-sum CBP (equ_s4e18xx / equ_s4e21xx, reading R20) */
       OR_LBP = 4,             /* fp32 layered BP, the paper's comparison schedule (l.171-197, equ_s2e10/e12; R22) */
       OR_FBP = 5 };           /* fp32 flooding BP, the paper's comparison schedule (l.102-169, equ_s2e3-e7; R22) */

typedef struct {
    int32_t max_iter;
    int32_t stop_rule;
    int32_t arith;
    float alpha;               /* normalisation of the min-sum variant (OR_MINSUM only) */
} or_opts;

/* Decode `frames` LLR vectors (row f at llr + f*ld, N floats).
 * OR_LBP / OR_FBP take only the stop rules OR_STOP_SYNDROME and OR_STOP_NONE
 * (the belief window is CBP's); their omega output is all zeros (no check-beliefs).
 * bits: packed hard decisions, bit v%32 of word v/32 (LSB first), ld_words per frame.
 * iters: 1-based sweep in which the stop fired, max_iter if it never did.
 * flags: bit0 converged (stop rule fired and, for belief rules, syndrome verified),
 *        bit1 syndrome of the output bits is zero, bit2 belief criterion fired
 *        with nonzero syndrome at least once.
 * edge_visits, fires (failed verifications), omega (final check-beliefs
 * Omega_c = +-phi(S_c), [frames][M]) are optional (NULL to skip). */
int oracle_decode(const or_code* c, const float* llr, int64_t ld, int64_t frames, const or_opts* o,
                  uint32_t* bits, int64_t ld_words, int32_t* iters, uint8_t* flags,
                  int64_t* edge_visits, int32_t* fires, float* omega);

/* Encoder: info bits (K bits, packed LSB first) -> codeword (N bits, packed),
 * systematic c = [s | p] with H c = 0 solved by GF(2) elimination.
 * Returns nonzero if the base has no dual-diagonal core + degree-1 extension. */
int oracle_encode(const or_code* c, const uint32_t* info, uint32_t* cw);
/* number of unsatisfied checks of a packed N-bit word */
int oracle_syndrome_weight(const or_code* c, const uint32_t* cw);

/* Philox4x32-10 (Salmon et al. 2011), one block */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* the channel's normals n_v, v < n, of frame `frame` */
void oracle_normals(uint64_t seed, uint64_t frame, int32_t n, float* out);

/* BPSK/AWGN channel of DESIGN.md §4 for global frames [frame_begin, frame_begin+frames):
 * llr[f*ld + v] (llr_mode bit0: int8-quantised q = sat(rint(4L), +-127), L' = q/4;
 * bit1: the all-zero codeword is sent, no info bits or encoder -- reading R23),
 * cw[f*ld_words + w] the transmitted codeword (either may be NULL). */
int oracle_channel(const or_code* c, double ebn0_db, uint64_t seed, int64_t frame_begin, int64_t frames,
                   int32_t llr_mode, float* llr, int64_t ld, uint32_t* cw, int64_t ld_words);

/* counts[8] = frames, bit_errors, frame_errors, cw_frame_errors, iter_sum,
 *             edge_visits, not_converged, undetected_fires (accumulated +=) */
int oracle_ber_sim(const or_code* c, double ebn0_db, uint64_t seed, int64_t frame_begin, int64_t frames,
                   const or_opts* o, int32_t llr_mode, int64_t* counts);

/* fp64 traces for the CBP == layered-BP pin (pin P5).  Both run
 * `sweeps` full sweeps without stopping and record, for every edge e = (c, v)
 * in visit order, lam[s*E + e] = the posterior of v used when c is processed in
 * sweep s (CBP: Lambda^new of equ_s4e20; LBP: Lambda_v before processing c). */
int oracle_cbp_trace_f64(const or_code* c, const float* llr, int32_t sweeps, double* lam);
int oracle_lbp_trace_f64(const or_code* c, const float* llr, int32_t sweeps, double* lam);
/* fp32 traces of normalized min-sum CBP and of textbook layered normalized min-sum
 * BP (leave-one-out minimum by brute force), same layout as above. */
int oracle_minsum_cbp_trace(const or_code* c, const float* llr, int32_t sweeps, float alpha, float* lam);
int oracle_minsum_lbp_trace(const or_code* c, const float* llr, int32_t sweeps, float alpha, float* lam);

/* Test-only hooks of the stop-rule pin (tests/test_oracle_stop.py).
 * oracle_decode_window: oracle_decode of the CBP arithmetics (log-tanh fp32/fp64/literal, min-sum)
 * with the belief window W of reading R4 replaced by `window` (> 0); no omega output.
 * oracle_cbp_visit_trace: `sweeps` full sweeps without stopping (arith OR_FP32_CONTRACT, OR_FP64
 * or OR_MINSUM); lam[s*E + e] = Lambda^new (equ_s4e20) and qn[s*E + e] = Q^new (equ_s4e19) of the
 * visit of edge e = (c, v) in sweep s -- the raw trajectory, none of the stop logic. */
int oracle_decode_window(const or_code* c, const float* llr, int64_t ld, int64_t frames, const or_opts* o,
                         int64_t window, uint32_t* bits, int64_t ld_words, int32_t* iters, uint8_t* flags,
                         int64_t* edge_visits, int32_t* fires);
int oracle_cbp_visit_trace(const or_code* c, const float* llr, int32_t sweeps, int32_t arith, float alpha,
                           double* lam, double* qn);

/* brute-force maximum-likelihood codeword (K <= 20): argmax sum_v L_v (1 - 2 c_v) */
int oracle_ml_decode(const or_code* c, const float* llr, uint32_t* cw);

/* contract functions re-exported for the pin tests */
float oracle_phi32(float x);
void  oracle_phi32_table(float* out);    /* 1153 x 4 floats */
/* every binary32 x in [PHI_LO, PHI_HI]: unclamped cubic below / above the bounds, max ulp error */
void  oracle_phi32_exhaustive(int64_t* below, int64_t* above, double* max_ulp, float* at);
float oracle_ln32(float x);
void  oracle_sincos_quarter32(uint32_t m24, float* s, float* c);
/* element-wise over arrays (pin tests) */
void  oracle_phi32_n(const float* x, float* y, int64_t n);
void  oracle_ln32_n(const float* x, float* y, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
