/*
 * contract32.h -- the ORACLE's implementation of the fp32 arithmetic contract
 * (DESIGN.md §3).  TEST INFRASTRUCTURE ONLY: see oracle/cbp_oracle.h.
 *
 * The contract fixes phi(x) = -log(tanh(x/2)) (eq.
 * equ_s2e5) and the Box-Muller helpers to a sequence of IEEE-754 binary32
 * operations (+ - * / sqrt, explicit fmaf, compares, integer bit ops) so the
 * CUDA path (own implementation in paper_2305_05286_b200/csrc/contract.cuh)
 * and this oracle produce identical bits.  Build with -ffp-contract=off.
 */
#ifndef ORACLE_CONTRACT32_H
#define ORACLE_CONTRACT32_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* clamp bounds of phi: PHI_HI = 30, PHI_LO = fl32(phi(30)) (reading R9) */
#define OR_PHI_HI 30.0f
#define OR_PHI_LO 0x1.a56e0cp-43f

float oracle_ln32(float x);              /* natural log, x normal and > 0          */
float oracle_phi32(float x);             /* phi contract v3 (table-driven cubic)   */
void  oracle_phi32_table(float* out);    /* the 1153 x 4 v3 coefficients           */
void  oracle_phi32_exhaustive(int64_t* below, int64_t* above, double* max_ulp, float* at);
void  oracle_sincos_quarter32(uint32_t m24, float* s, float* c); /* sin/cos(2*pi*m24*2^-24) */

#ifdef __cplusplus
}
#endif
#endif
