/*
 * contract32.c -- ORACLE implementation of the fp32 arithmetic contract
 * (DESIGN.md §3 "Arithmetic contract").  TEST INFRASTRUCTURE ONLY.
 *
 * Written from the contract table in DESIGN.md, not from the CUDA source.
 * Compile with -O2 -ffp-contract=off (no implicit FMA contraction); every
 * fused multiply-add below is an explicit fmaf() and therefore correctly
 * rounded on any conforming platform.
 *
 * Pinned by tests/test_oracle_contract.py against double-precision libm
 * (-log(tanh(x/2)), log, sin, cos) on dense grids and the closed forms
 * phi(ln 3) = ln 2, phi(ln 2) = ln 3, phi(ln(1+sqrt 2)) = ln(1+sqrt 2).
 */
#include "contract32.h"
#include <math.h>
#include <string.h>

static float f_from_bits(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t bits_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* constants of DESIGN.md §3 table "K" */
#define LN2_HI   0x1.62e400p-1f
#define LN2_LO   0x1.7f7d1cp-20f
#define INV_LN2  0x1.715476p+0f
#define PHI_XA   1.0f

/* natural log: x = 2^k m, m in [sqrt(2)/2, sqrt(2)), ln = k ln2 + f + f^2 P(f), f = m - 1 */
float oracle_ln32(float x)
{
    const int32_t ix = (int32_t)(bits_of(x) - 0x3f3504f3u);
    const int32_t k = ix >> 23;                       /* arithmetic shift */
    const float m = f_from_bits(((uint32_t)ix & 0x007fffffu) + 0x3f3504f3u);
    const float f = m - 1.0f;                         /* exact (Sterbenz) */
    float p = -0x1.36cf20p-4f;                        /* P_ln c8 .. c0 */
    p = fmaf(p, f, 0x1.03a7f6p-3f);
    p = fmaf(p, f, -0x1.0d15eap-3f);
    p = fmaf(p, f, 0x1.230f94p-3f);
    p = fmaf(p, f, -0x1.54816ep-3f);
    p = fmaf(p, f, 0x1.999e58p-3f);
    p = fmaf(p, f, -0x1.00020ep-2f);
    p = fmaf(p, f, 0x1.555556p-2f);
    p = fmaf(p, f, -0x1.fffffep-2f);
    const float f2 = f * f;
    const float lnm = fmaf(f2, p, f);
    const float kf = (float)k;
    const float t = fmaf(kf, LN2_LO, lnm);
    return fmaf(kf, LN2_HI, t);
}

/*
 * phi(x) = -log(tanh(x/2))  (equ_s2e5), clamped in and out to
 * [PHI_LO, PHI_HI] (reading R9).
 *   regime A, x < 1 :  phi = x^2 G(x^2) - ln(x/2)
 *                      (G(y) = ln((sqrt(y)/2) coth(sqrt(y)/2)) / y)
 *   regime B, x >= 1:  t = e^{-x} = 2^{-n} e^{-r};  phi = 2 t H(t^2)
 *                      (H(w) = atanh(sqrt(w)) / sqrt(w))
 */
float oracle_phi32(float x)
{
    x = fmaxf(x, OR_PHI_LO);
    x = fminf(x, OR_PHI_HI);
    float r;
    if (x < PHI_XA) {
        const float h = 0.5f * x;
        const float l = oracle_ln32(h);
        const float y = x * x;
        float g = -0x1.78439ep-16f;                   /* G_A c3 .. c0 */
        g = fmaf(g, y, 0x1.63e3a2p-12f);
        g = fmaf(g, y, -0x1.3e8c42p-8f);
        g = fmaf(g, y, 0x1.555552p-4f);
        g = g * y;
        r = g - l;
    } else {
        const float a = x * INV_LN2;
        const float n = rintf(a);
        float rr = fmaf(-n, LN2_HI, x);
        rr = fmaf(-n, LN2_LO, rr);
        float e = 0x1.6b4e62p-10f;                    /* E_exp c6 .. c1, c0 = 1 */
        e = fmaf(e, rr, -0x1.126f76p-7f);
        e = fmaf(e, rr, 0x1.555796p-5f);
        e = fmaf(e, rr, -0x1.555406p-3f);
        e = fmaf(e, rr, 0x1.fffffcp-2f);
        e = fmaf(e, rr, -1.0f);
        e = fmaf(e, rr, 1.0f);
        const int32_t ni = (int32_t)n;
        const float s = f_from_bits((uint32_t)(127 - ni) << 23);   /* 2^-n, exact */
        const float t = e * s;
        const float w = t * t;
        float hh = 0x1.2e8fe8p-3f;                    /* H_B c4 .. c1, c0 = 1 */
        hh = fmaf(hh, w, 0x1.1b78f8p-3f);
        hh = fmaf(hh, w, 0x1.9a05a6p-3f);
        hh = fmaf(hh, w, 0x1.555490p-2f);
        hh = fmaf(hh, w, 1.0f);
        const float u = t * hh;
        r = u + u;
    }
    r = fmaxf(r, OR_PHI_LO);
    r = fminf(r, OR_PHI_HI);
    return r;
}

/*
 * sin and cos of theta = 2 pi m 2^-24, m in [0, 2^24) (Box-Muller angle,
 * DESIGN.md §4).  Exact quadrant reduction in integers:
 *   q = (m + 2^21) >> 22,  f = (m - q 2^22) 2^-22 in [-1/2, 1/2),  theta = (pi/2)(q + f)
 */
void oracle_sincos_quarter32(uint32_t m, float* s_out, float* c_out)
{
    const uint32_t q = (m + 0x200000u) >> 22;
    const int32_t fi = (int32_t)m - (int32_t)(q << 22);
    const float f = (float)fi * 0x1p-22f;
    const float z = f * f;
    float sp = -0x1.2d92c6p-8f;                       /* S_sin c3 .. c0 */
    sp = fmaf(sp, z, 0x1.465e90p-4f);
    sp = fmaf(sp, z, -0x1.4abbb8p-1f);
    sp = fmaf(sp, z, 0x1.921fb6p+0f);
    const float sn = sp * f;
    float cp = 0x1.d9cf32p-11f;                       /* C_cos c4 .. c1, c0 = 1 */
    cp = fmaf(cp, z, -0x1.55c5c6p-6f);
    cp = fmaf(cp, z, 0x1.03c1dep-2f);
    cp = fmaf(cp, z, -0x1.3bd3ccp+0f);
    cp = fmaf(cp, z, 1.0f);
    switch (q & 3u) {
    case 0: *s_out = sn;  *c_out = cp;  break;
    case 1: *s_out = cp;  *c_out = -sn; break;
    case 2: *s_out = -sn; *c_out = -cp; break;
    default: *s_out = -cp; *c_out = sn; break;
    }
}
