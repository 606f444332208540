/*
 * cbp_inputs.h -- seeded input generators shared by the product and the oracle.
 *
 * This module holds NONE of the method's arithmetic (no phi, no message
 * passing, no channel, no encoder).  It only draws the QC base matrix of an
 * LDPC code from a seed, i.e. the "code graph
 * G = (V, C, E)" input of PAPER.md l.92 written as a quasi-cyclic base
 * matrix plus lifting size Z.  Both libcbp.so (exported as
 * cbp_construct_base) and the test oracle consume the base matrix it writes.
 *
 * Base-matrix convention (row-major, mb x nb, int16):
 *   -1      : zero Z x Z block
 *   s>=0    : identity cyclically shifted by s; check row r of block (i, j)
 *             connects to variable j*Z + (r + s) % Z.
 */
#ifndef CBP_INPUTS_H
#define CBP_INPUTS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Info-column weight rule. */
enum {
    CBP_W_CONST = 0,      /* w = w_lo                                           */
    CBP_W_UNIFORM = 1,    /* w uniform in {w_lo, ..., w_hi}                     */
    CBP_W_HEAVY = 2       /* w = clamp(floor(3/u), w_lo, w_hi), u in (0,1]      */
};

typedef struct {
    int32_t mb;        /* base rows                                            */
    int32_t nb;        /* base columns; kb = nb - mb info columns              */
    int32_t Z;         /* lifting size, 2 <= Z <= 1024                         */
    int32_t mb_core;   /* rows of the dual-diagonal core (mb unless extended)  */
    int32_t wmode;     /* CBP_W_*                                              */
    int32_t w_lo;
    int32_t w_hi;
} cbp_inputs_spec;

/*
 * Draw a base matrix.  base_out must hold mb*nb int16.  Returns 0 on success,
 * nonzero on an invalid spec (message in *err if err != NULL).
 * Deterministic in (spec, seed) on every platform (SplitMix64, rejection
 * sampling, integer arithmetic only; the heavy-tailed rule uses one IEEE
 * double division).
 */
int cbp_inputs_construct_base(const cbp_inputs_spec* spec, uint64_t seed,
                              int16_t* base_out, const char** err);

/* Named specs of BASELINE.json configs: "C1", "C2", "C3a", "C3b", "C4",
 * plus "T24" (N=24 code for the brute-force ML pin).  Returns 0 if found. */
int cbp_inputs_named_spec(const char* name, cbp_inputs_spec* out);

#ifdef __cplusplus
}
#endif
#endif
