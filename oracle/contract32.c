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
 * (-log(tanh(x/2)), log, sin, cos) on dense grids and exhaustively (phi), and the
 * closed forms phi(ln 3) = ln 2, phi(ln 2) = ln 3, phi(ln(1+sqrt 2)) = ln(1+sqrt 2).
 */
#include "contract32.h"
#include <math.h>
#include <string.h>

static float f_from_bits(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t bits_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* constants of DESIGN.md §3 table "K" */
#define LN2_HI   0x1.62e400p-1f
#define LN2_LO   0x1.7f7d1cp-20f

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
 * phi(x) = -log(tanh(x/2))  (equ_s2e5) in IEEE double, written as
 * log1p(2 / expm1(x)) -- algebraically equal ((1 + t)/(1 - t) with t = tanh(x/2) =
 * (e^x - 1)/(e^x + 1) gives 1 + 2/(e^x - 1)), without the cancellation of tanh -> 1
 * for large x.  libm double (<= 1 ulp of double, ~2^-29 of a binary32 ulp).
 */
static double phi_double(double x) { return log1p(2.0 / expm1(x)); }

/*
 * phi contract v3: piecewise cubic in a local variable u in [0,1)
 * over 1153 segments --
 *   seg 0..703    x < 2:  16 segments per binade 2^e, e = -43..0:
 *                         seg = (bits(x) >> 19) - 1344,  u = 19 low mantissa bits / 2^19,
 *                         x(u) = 2^e (1 + (j + u)/16), j = seg % 16
 *   seg 704..1152 x >= 2: t = fmaf(x, 16, -32), i = (int)t, u = t - i, seg = 704 + i,
 *                         x(u) = 2 + (i + u)/16
 * Coefficients: the cubic through phi_double at u = 0, 1/4, 3/4, 1 (x(u) exact binary32),
 * Newton divided differences in IEEE double in the order written below, each coefficient
 * rounded to binary32.  Max error over every binary32 x in [PHI_LO, PHI_HI]: 1.66 ulp of
 * the double phi (exhaustive, oracle_phi32_exhaustive).
 */
#define OR_PHI_SEGS 1153
static float phi_tab[OR_PHI_SEGS][4];
static int phi_tab_ready;

static void phi_segment(double F0, double F1, double F2, double F3, float* c)
{
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
        double f[4];
        for (int k = 0; k < 4; ++k) {
            float x;
            if (seg < 704) {
                const int e = -43 + seg / 16, j = seg % 16;
                x = ldexpf((float)(64 + 4 * j + Q4[k]), e - 6);     /* 2^e (1 + (j + u)/16), exact */
            } else {
                const int i = seg - 704;
                x = (float)(128 + 4 * i + Q4[k]) * 0.015625f;       /* 2 + (i + u)/16, exact */
            }
            f[k] = phi_double((double)x);
        }
        phi_segment(f[0], f[1], f[2], f[3], phi_tab[seg]);
    }
    phi_tab_ready = 1;
}

/* the unclamped cubic of x in [PHI_LO, PHI_HI] */
static float phi_cubic(float x)
{
    int seg;
    float u;
    if (x < 2.0f) {
        const uint32_t b = bits_of(x);
        seg = (int)(b >> 19) - 1344;
        u = f_from_bits(((b & 0x7ffffu) << 4) | 0x3f800000u) - 1.0f;   /* exact */
    } else {
        const float t = fmaf(x, 16.0f, -32.0f);                    /* exact */
        const int i = (int)t;
        u = t - (float)i;                                          /* exact */
        seg = 704 + i;
    }
    const float* c = phi_tab[seg];
    float p = fmaf(c[3], u, c[2]);
    p = fmaf(p, u, c[1]);
    return fmaf(p, u, c[0]);
}

/* Exhaustive check over every binary32 x in [PHI_LO, PHI_HI]: counts unclamped results
 * below PHI_LO / above PHI_HI (pin: the contract's output clamp never binds) and the
 * maximum error in binary32 ulps of the double phi (clamped to the same bounds). */
void oracle_phi32_exhaustive(int64_t* below, int64_t* above, double* max_ulp, float* at)
{
    if (!phi_tab_ready) phi_build_table();
    const uint32_t a = bits_of(OR_PHI_LO), z = bits_of(OR_PHI_HI);
    int64_t nb = 0, na = 0;
    double mx = 0.0;
    float mx_at = 0.0f;
    for (uint32_t w = a; w <= z; ++w) {
        const float x = f_from_bits(w);
        const float p = phi_cubic(x);
        nb += p < OR_PHI_LO;
        na += p > OR_PHI_HI;
        double ref = phi_double((double)x);
        ref = fmin(fmax(ref, (double)OR_PHI_LO), (double)OR_PHI_HI);
        const float rf = (float)ref;
        const double ulp = (double)nextafterf(rf, INFINITY) - (double)rf;
        const double e = fabs((double)p - ref) / ulp;
        if (e > mx) { mx = e; mx_at = x; }
    }
    *below = nb;
    *above = na;
    *max_ulp = mx;
    *at = mx_at;
}

void oracle_phi32_table(float* out)
{
    if (!phi_tab_ready) phi_build_table();
    memcpy(out, phi_tab, sizeof(phi_tab));
}

/* phi contract v3 with the input / output clamp of reading R9 */
float oracle_phi32(float x)
{
    if (!phi_tab_ready) phi_build_table();
    x = fmaxf(x, OR_PHI_LO);
    x = fminf(x, OR_PHI_HI);
    float p = phi_cubic(x);
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
