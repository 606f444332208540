/*
 * cbp.h -- C ABI of the B200-native check-belief propagation (CBP) decoder.
 *
 * Method: Guan & Liang, "Check-Belief Propagation Decoding of LDPC Codes"
 * (arXiv 2305.05286), §IV-C Steps 1-3 (l.400-487), with the readings
 * R1-R21 of DESIGN.md §2 and the fp32 arithmetic contract of DESIGN.md §3.
 * Implemented by paper_2305_05286_b200/libcbp.so (sm_100a kernels + host code).
 *
 * Conventions
 *  - Every function returns a cbp_status; nothing else crosses the ABI (no
 *    exceptions).  On a non-OK status cbp_last_error() returns a thread-local
 *    message.  Decoding failure is a RESULT (flags bit0 = 0), not an error.
 *  - "device pointer" = memory on the code's device, allocated and owned by
 *    the caller; "host pointer" = caller-owned host memory.  The library never
 *    frees caller memory.  All work is enqueued on the caller's CUDA stream
 *    (a cudaStream_t passed as void*, NULL = legacy default stream) and is
 *    asynchronous: asynchronous device faults surface at the caller's next
 *    synchronisation (reported then by the CUDA runtime, not by this ABI).
 *  - A cbp_code is immutable after creation and may be used concurrently from
 *    several host threads and streams.
 *  - Launch workspace (the frame work-queue counter; for codes whose per-frame
 *    state does not fit in shared memory, the global frame state: ~0.7 MB per SM
 *    for N = 26112) is allocated stream-ordered from a library-private memory
 *    pool per device that keeps its memory for reuse (it is never trimmed).
 *  - Bits are packed LSB first: bit v of a frame is bit (v % 32) of word v / 32.
 *  - Results depend only on (code, inputs, options) -- never on grid size,
 *    stream or GPU count.  cbp_ber_sim / cbp_channel depend only on
 *    (seed, global frame index): frames shard across GPUs by frame range.
 */
#ifndef CBP_H
#define CBP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CBP_OK = 0,
    CBP_E_INVALID = 1,      /* bad argument (null pointer, size, range)        */
    CBP_E_UNSUPPORTED = 2,  /* valid but not supported (e.g. no encoder structure) */
    CBP_E_NOMEM = 3,        /* host or device allocation failed                */
    CBP_E_CUDA = 4,         /* CUDA runtime error at enqueue time              */
    CBP_E_INTERNAL = 5
} cbp_status;

/* Thread-local text of the last non-OK status of this thread ("" if none). */
const char* cbp_last_error(void);
/* Library version string. */
const char* cbp_version(void);

/* ------------------------------------------------------------------ codes */

/* Seeded QC base-matrix constructor (BASELINE.json
 * configs).  Host only.  base_out: host int16[mb*nb], row-major; -1 = zero
 * block, s in [0,Z) = identity cyclically shifted by s (check row r of block
 * (i,j) connects to variable j*Z + (r+s)%Z).  Identical to the shared input
 * generator inputs/qc_construct.c (same source). */
typedef struct {
    int32_t mb, nb, Z;      /* base rows, base columns, lifting size            */
    int32_t mb_core;        /* rows of the dual-diagonal core (mb if no extension) */
    int32_t wmode;          /* info column weight rule: 0 const, 1 uniform, 2 heavy-tailed */
    int32_t w_lo, w_hi;
} cbp_construct_spec;
cbp_status cbp_construct_base(const cbp_construct_spec* spec, uint64_t seed, int16_t* base_out);

/* Opaque code handle: the expanded code graph G = (V, C, E) of PAPER.md l.92
 * (N = nb*Z variables, M = mb*Z checks, K = N - M info bits) as per-base-entry
 * schedule tables resident on `device`.
 *   base  : host int16[mb*nb] (copied; caller keeps ownership)
 *   Z     : 1 <= Z <= 1024; shifts must lie in [-1, Z)
 *   every base row and column must be non-empty.
 * Encoding (cbp_channel, cbp_ber_sim) additionally needs the dual-diagonal
 * parity structure of SURVEY Appendix B; otherwise those return
 * CBP_E_UNSUPPORTED (unless CBP_TX_ZERO is set) while decoding still works. */
typedef struct cbp_code cbp_code;
cbp_status cbp_code_create(const int16_t* base, int32_t mb, int32_t nb, int32_t Z, int32_t device, cbp_code** out);
void       cbp_code_destroy(cbp_code* code);
/* Optional build settings of a code handle (cbp_code_create_ex).
 *   frames_per_lane: 0 = automatic (default), 1 or 2.  With 2, every lane of a frame
 *   group decodes its lifted check for two frames at once (interleaved state,
 *   DESIGN.md §5); results are identical for every setting -- it is a performance
 *   choice only.  2 needs the per-frame state in shared memory and teams of at most
 *   256 threads (Z <= 256), else CBP_E_UNSUPPORTED.  With 0 the environment variable
 *   CBP_FRAMES_PER_LANE=1|2 (A/B measurements) overrides the automatic choice. */
typedef struct {
    int32_t frames_per_lane;
} cbp_code_config;
/* cbp_code_create with settings; cfg == NULL is cbp_code_create. */
cbp_status cbp_code_create_ex(const int16_t* base, int32_t mb, int32_t nb, int32_t Z, int32_t device,
                              const cbp_code_config* cfg, cbp_code** out);
/* any output pointer may be NULL */
cbp_status cbp_code_dims(const cbp_code* code, int32_t* N, int32_t* K, int32_t* M, int64_t* E);

/* ----------------------------------------------------------------- decode */

/* Stop rules (readings R4-R6). */
typedef enum {
    CBP_STOP_BELIEF_M = 0,  /* M consecutive clean check updates (Omega>0, no flips), then syndrome verify (default) */
    CBP_STOP_BELIEF_N = 1,  /* the literal "N consecutive" window, then syndrome verify */
    CBP_STOP_SYNDROME = 2,  /* syndrome of the hard bits after every full sweep        */
    CBP_STOP_NONE = 3       /* always run max_iter sweeps                              */
} cbp_stop_rule;

/* Decoding algorithms: the two CBP check-belief update rules, and the paper's two
 * comparison schedules (reading R22) on the same
 * code graph, channel and counters -- for the CBP vs LBP vs FBP convergence and
 * error-rate comparisons of the paper (Fig. 6-9, l.613-724).  All four run in fp32
 * under the arithmetic contract.  LBP / FBP take only CBP_STOP_SYNDROME or
 * CBP_STOP_NONE (the belief window is CBP's), always run one frame per lane, and
 * leave d_omega zero (no check-beliefs). */
typedef enum {
    CBP_ALG_LOG_TANH = 0,   /* CBP, phi-domain psi+/psi- (equ_s4e18, equ_s4e21), fp32 arithmetic contract */
    CBP_ALG_MIN_SUM = 1,    /* CBP, normalized min-sum (equ_s4e18xx, equ_s4e21xx, reading R20); row degree >= 2 */
    CBP_ALG_LBP = 2,        /* layered BP (equ_s2e10, equ_s2e4, equ_s2e12), checks in ascending order */
    CBP_ALG_FBP = 3         /* flooding BP (equ_s2e3, equ_s2e4, equ_s2e6) */
} cbp_algorithm;

typedef struct {
    int32_t max_iter;       /* sweeps over all M checks, 1..65535                    */
    int32_t stop_rule;      /* cbp_stop_rule                                         */
    int32_t algorithm;      /* cbp_algorithm                                         */
    float alpha;            /* min-sum normalisation in (0, 1] (ignored for log-tanh) */
} cbp_opts;

/* Decode `frames` channel-LLR vectors (PAPER.md equ_s4e15: L_v = ln Pr(y|0)/Pr(y|1)).
 *   d_llr    : device float[frames][ld], ld >= N, (ld*4) % 16 == 0, 16-byte aligned
 *   d_bits   : device uint32[frames][ld_words], ld_words >= ceil(N/32): hard decisions
 *              of the V2C phase (reading R14)
 *   d_iters  : device int32[frames]: 1-based sweep in which the stop fired, max_iter if none
 *   d_flags  : device uint8[frames]: bit0 converged, bit1 output syndrome zero,
 *              bit2 belief criterion fired with a nonzero syndrome at least once
 *   d_omega  : optional device float[frames][M]: final check-beliefs Omega_c = +-phi(S_c)
 *              (equ_s4e1/equ_s4e3), NULL to skip
 *   d_ev     : optional device int64[frames]: edge visits (= B2V = V2C = C2B updates)
 * frames == 0 is a no-op.  Non-finite LLRs give unspecified bits but stay memory-safe. */
cbp_status cbp_decode(const cbp_code* code, const float* d_llr, int64_t ld, int64_t frames, const cbp_opts* opts,
                      uint32_t* d_bits, int64_t ld_words, int32_t* d_iters, uint8_t* d_flags, float* d_omega,
                      int64_t* d_ev, void* stream);

/* Same with int8-quantised LLRs: L_v = scale * q_v (BASELINE config 5: q = sat(rint(4L), +-127),
 * scale = 0.25).  d_q: device int8[frames][ld], ld >= N, ld % 16 == 0, 16-byte aligned. */
cbp_status cbp_decode_i8(const cbp_code* code, const int8_t* d_q, int64_t ld, float scale, int64_t frames,
                         const cbp_opts* opts, uint32_t* d_bits, int64_t ld_words, int32_t* d_iters,
                         uint8_t* d_flags, float* d_omega, int64_t* d_ev, void* stream);

/* Host-buffer decoding (SPEC.md decode_cbp: LLRs in, hard bits, iteration counts
 * and flags out): the same results as cbp_decode / cbp_decode_i8 for caller-owned HOST buffers.
 * The library splits the batch into chunks of `chunk_frames` frames (0 = 16384) and pipelines
 * host->device copy, decode and device->host copy of each chunk round-robin over `nstreams`
 * (0 = 4, at most 16) CUDA streams of its own, with device buffers from its memory pool, so the
 * PCIe transfers overlap the kernels.  The call BLOCKS until every output is in host memory.
 * Pinned (page-locked) host memory is strongly recommended: with pageable memory the copies
 * are staged by the driver and do not overlap.
 *   h_llr / h_q : host float[frames][ld] (ld >= N) / int8[frames][ld] (ld >= N, ld % 16 == 0)
 *   h_bits      : host uint32[frames][ld_words] (ld_words >= ceil(N/32))
 *   h_iters     : host int32[frames];   h_flags : host uint8[frames]
 * Errors: CBP_E_INVALID as for cbp_decode (null buffers, sizes, options); CBP_E_NOMEM if a
 * device buffer cannot be allocated; CBP_E_CUDA for copy / launch / synchronisation failures
 * (the contents of the outputs are then unspecified). */
cbp_status cbp_decode_host(const cbp_code* code, const float* h_llr, int64_t ld, int64_t frames, const cbp_opts* opts,
                           uint32_t* h_bits, int64_t ld_words, int32_t* h_iters, uint8_t* h_flags,
                           int64_t chunk_frames, int32_t nstreams);
cbp_status cbp_decode_host_i8(const cbp_code* code, const int8_t* h_q, int64_t ld, float scale, int64_t frames,
                              const cbp_opts* opts, uint32_t* h_bits, int64_t ld_words, int32_t* h_iters,
                              uint8_t* h_flags, int64_t chunk_frames, int32_t nstreams);

/* ---------------------------------------------------------------- channel */

/* llr_mode flags of cbp_channel / cbp_ber_sim (OR-ed; 0..3 valid). */
enum {
    CBP_LLR_INT8 = 1,   /* int8 stream: q = sat(rint(4L), +-127), L = q/4 (BASELINE config 5) */
    CBP_TX_ZERO = 2     /* transmit the all-zero codeword instead of encoded random info bits
                           (reading R23).  Needs no encoder, so it works for every
                           code (e.g. the PEG codes of PAPER.md l.608); the noise is the same
                           Philox stream, so L equals the encoded run's L wherever c_v = 0. */
};

/* BPSK/AWGN channel of DESIGN.md §4 on device for global frames
 * [frame_begin, frame_begin + frames): uniform info bits (Philox4x32-10 keyed by
 * seed), systematic encoding, y = (1-2c) + sigma n, L = 2y/sigma^2 with
 * sigma^2 = 1/(2 (K/N) 10^(ebn0_db/10)); llr_mode: OR of the flags above (0 = fp32,
 * encoded random info bits).  Without CBP_TX_ZERO the code needs the dual-diagonal
 * encoder structure, else CBP_E_UNSUPPORTED.
 *   d_llr : device float[frames][ld] (ld >= N) or NULL
 *   d_cw  : device uint32[frames][ld_words] transmitted codewords or NULL */
cbp_status cbp_channel(const cbp_code* code, double ebn0_db, uint64_t seed, int64_t frame_begin, int64_t frames,
                       int32_t llr_mode, float* d_llr, int64_t ld, uint32_t* d_cw, int64_t ld_words, void* stream);

/* ------------------------------------------------------------------ BER sim */

/* Counters accumulated (+=) by cbp_ber_sim; device memory, caller zeroes it. */
typedef struct {
    int64_t frames;
    int64_t bit_errors;       /* over the K systematic info bits       */
    int64_t frame_errors;     /* frames with >= 1 info bit error        */
    int64_t cw_frame_errors;  /* frames with >= 1 codeword bit error    */
    int64_t iter_sum;         /* sum of per-frame iteration counts      */
    int64_t edge_visits;      /* sum of per-frame edge visits           */
    int64_t not_converged;    /* frames with flags bit0 = 0             */
    int64_t undetected_fires; /* failed syndrome verifications          */
} cbp_counts;

/* Channel + CBP decode + error counting for one Eb/N0 point: counts the
 * frames of cbp_channel -> cbp_decode -> compare (llr_mode as for cbp_channel;
 * bit errors count over variables 0..K-1, the systematic part for encoded
 * codes).  Codes on the one-frame-per-warp kernel run it as
 * cbp_channel + cbp_ber_count per chunk of 2^20 frames through a stream-ordered
 * HBM workspace (N floats + ceil(N/32) words per frame of the chunk); the
 * others in one fused kernel.  The counters are the same either way. */
cbp_status cbp_ber_sim(const cbp_code* code, double ebn0_db, uint64_t seed, int64_t frame_begin, int64_t frames,
                       const cbp_opts* opts, int32_t llr_mode, cbp_counts* d_counts, void* stream);

/* Decode + error counting on given frames (the decode half of cbp_ber_sim, for
 * LLRs from any source).  PAPER.md §IV (Steps 1-3, Algorithm 1) per frame as in
 * cbp_decode; the decision bits are compared with the transmitted codeword and
 * accumulated (+=) into d_counts as cbp_ber_sim does.
 *   d_llr    : device float[frames][ld], ld >= N, ld % 4 == 0, 16-byte aligned
 *   d_cw     : device uint32[frames][ld_words] transmitted codewords (bit v%32 of
 *              word v/32), ld_words >= ceil(N/32)
 *   d_counts : device cbp_counts, accumulated (caller zeroes it)
 * Needs a code on the one-frame-per-warp kernel (17 <= Z <= 384) and the
 * log-tanh CBP or layered-BP algorithm, else CBP_E_UNSUPPORTED.  Buffers are the
 * caller's; nothing is retained after the call. */
cbp_status cbp_ber_count(const cbp_code* code, const float* d_llr, int64_t ld, const uint32_t* d_cw, int64_t ld_words,
                         int64_t frames, const cbp_opts* opts, cbp_counts* d_counts, void* stream);

/* ----------------------------------------------------------- introspection */

/* Launch geometry the library picks for this code's log-tanh decoder (for reports):
 * threads per CTA, CTAs per SM, frames per CTA, dynamic smem bytes, state in smem (1)
 * or global (0), SMs, frames per lane (1 or 2), and r_in_global = 1 for the split layout
 * (state in smem except the R messages, which live in a global workspace). */
typedef struct {
    int32_t threads, ctas_per_sm, frames_per_cta, smem_bytes, state_in_smem, num_sms, frames_per_lane;
    int32_t r_in_global;
} cbp_launch_info;
cbp_status cbp_get_launch_info(const cbp_code* code, cbp_launch_info* out);

/* Element-wise evaluation of the fp32 arithmetic contract on the device
 * for the bit-equality pins: fn 0 phi32(x), 1 ln32(x),
 * 2 / 3 sin / cos(2 pi m 2^-24) with m = the low 24 bits of x's bit pattern.
 * d_x, d_y: device float[n] on `device`. */
cbp_status cbp_eval_contract(int32_t fn, const float* d_x, float* d_y, int64_t n, int32_t device, void* stream);

/* Copy the phi contract v3 table of `device` (1153 segments x {c0, c1, c2, c3} in the
 * kernel's storage form; built on the host and uploaded at first use) into
 * d_out (device float[4612]). */
cbp_status cbp_phi_table(int32_t device, float* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
