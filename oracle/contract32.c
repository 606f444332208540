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
 * Reference formula phi_v1(x) = -log(tanh(x/2))  (equ_s2e5),
 * unclamped, for x in [2^-43, 31] ("v1"):
 *   regime A, x < 1 :  phi = x^2 G(x^2) - ln(x/2)
 *                      (G(y) = ln((sqrt(y)/2) coth(sqrt(y)/2)) / y)
 *   regime B, x >= 1:  t = e^{-x} = 2^{-n} e^{-r};  phi = 2 t H(t^2)
 *                      (H(w) = atanh(sqrt(w)) / sqrt(w))
 */
static float phi_v1_unclamped(float x)
{
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
    return r;
}

/* v1 with the input/output clamp of reading R9 (kept for the pins) */
float oracle_phi32_v1(float x)
{
    x = fmaxf(x, OR_PHI_LO);
    x = fminf(x, OR_PHI_HI);
    float r = phi_v1_unclamped(x);
    r = fmaxf(r, OR_PHI_LO);
    r = fminf(r, OR_PHI_HI);
    return r;
}

/*
 * phi contract v2: piecewise cubic in a local variable u in [0,1)
 * over 929 segments --
 *   seg 0..703   x < 2:  16 segments per binade 2^e, e = -43..0:
 *                        seg = (bits(x) >> 19) - 1344,  u = 19 low mantissa bits / 2^19,
 *                        x(u) = 2^e (1 + (j + u)/16), j = seg % 16
 *   seg 704..928 x >= 2: t = fmaf(x, 8, -16), i = (int)t, u = t - i, seg = 704 + i,
 *                        x(u) = 2 + (i + u)/8
 * Coefficients: cubic interpolation of phi_v1 at u = 0, 1/4, 3/4, 1 (exact floats
 * x(u)), Newton divided differences in IEEE double in the order written below,
 * each coefficient rounded to binary32.
 */
#define OR_PHI_SEGS 929
static float phi_tab[OR_PHI_SEGS][4];
static int phi_tab_ready;

static void phi_segment(float f0, float f1, float f2, float f3, float* c)
{
    const double F0 = f0, F1 = f1, F2 = f2, F3 = f3;
    const double d01 = (F1 - F0) * 4.0;
    const double d12 = (F2 - F1) * 2.0;
    const double d23 = (F3 - F2) * 4.0;
    const double d012 = ((d12 - d01) * 4.0) / 3.0;
    const double d123 = ((d23 - d12) * 4.0) / 3.0;
    const double d0123 = d123 - d012;
    const double t1 = d012 * 0.25;
    const double t2 = d01 - t1;
    const double t3 = d0123 * 0.1875;
    c[0] = (float)F0;
    c[1] = (float)(t2 + t3);
    c[2] = (float)(d012 - d0123);
    c[3] = (float)d0123;
}

static void phi_build_table(void)
{
    static const int Q4[4] = {0, 1, 3, 4};                 /* u = Q4/4 */
    for (int seg = 0; seg < OR_PHI_SEGS; ++seg) {
        float f[4];
        for (int k = 0; k < 4; ++k) {
            float x;
            if (seg < 704) {
                const int e = -43 + seg / 16, j = seg % 16;
                x = ldexpf((float)(64 + 4 * j + Q4[k]), e - 6);     /* 2^e (1 + (j + u)/16), exact */
            } else {
                const int i = seg - 704;
                x = (float)(64 + 4 * i + Q4[k]) * 0.03125f;         /* 2 + (i + u)/8, exact */
            }
            f[k] = phi_v1_unclamped(x);
        }
        phi_segment(f[0], f[1], f[2], f[3], phi_tab[seg]);
    }
    phi_tab_ready = 1;
}

/* Exhaustive check over every binary32 x in [PHI_LO, PHI_HI] of the v2 cubic
 * WITHOUT the output clamp: counts results below PHI_LO / above PHI_HI and the
 * maximum (pin: the output clamp of the contract never binds). */
void oracle_phi32_clamp_check(int64_t* below, int64_t* above, float* maxp)
{
    if (!phi_tab_ready) phi_build_table();
    const uint32_t a = bits_of(OR_PHI_LO), z = bits_of(OR_PHI_HI);
    int64_t nb = 0, na = 0;
    float mx = 0.0f;
    for (uint32_t w = a; w <= z; ++w) {
        const float x = f_from_bits(w);
        int seg;
        float u;
        if (x < 2.0f) {
            seg = (int)(w >> 19) - 1344;
            u = f_from_bits(((w & 0x7ffffu) << 4) | 0x3f800000u) - 1.0f;
        } else {
            const float t = fmaf(x, 8.0f, -16.0f);
            const int i = (int)t;
            u = t - (float)i;
            seg = 704 + i;
        }
        const float* c = phi_tab[seg];
        float p = fmaf(c[3], u, c[2]);
        p = fmaf(p, u, c[1]);
        p = fmaf(p, u, c[0]);
        nb += p < OR_PHI_LO;
        na += p > OR_PHI_HI;
        if (p > mx) mx = p;
    }
    *below = nb;
    *above = na;
    *maxp = mx;
}

void oracle_phi32_table(float* out)
{
    if (!phi_tab_ready) phi_build_table();
    memcpy(out, phi_tab, sizeof(phi_tab));
}

float oracle_phi32(float x)
{
    if (!phi_tab_ready) phi_build_table();
    x = fmaxf(x, OR_PHI_LO);
    x = fminf(x, OR_PHI_HI);
    int seg;
    float u;
    if (x < 2.0f) {
        const uint32_t b = bits_of(x);
        seg = (int)(b >> 19) - 1344;
        u = f_from_bits(((b & 0x7ffffu) << 4) | 0x3f800000u) - 1.0f;   /* exact */
    } else {
        const float t = fmaf(x, 8.0f, -16.0f);                     /* exact */
        const int i = (int)t;
        u = t - (float)i;                                          /* exact */
        seg = 704 + i;
    }
    const float* c = phi_tab[seg];
    float p = fmaf(c[3], u, c[2]);
    p = fmaf(p, u, c[1]);
    p = fmaf(p, u, c[0]);
    p = fmaxf(p, OR_PHI_LO);
    p = fminf(p, OR_PHI_HI);
    return p;
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
