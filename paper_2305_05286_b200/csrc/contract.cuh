// contract.cuh -- device implementation of the fp32 arithmetic contract
// (DESIGN.md §3).  Written from the DESIGN.md table, independently of the
// oracle (oracle/contract32.c); both must produce identical bits.
//
// Build requirement: nvcc --fmad=false (no implicit contraction) with
// IEEE div/sqrt and denormals kept.  Every FMA below is an explicit
// __fmaf_rn (one correctly rounded FFMA), never formed by the compiler.
#pragma once
#include <cuda_runtime.h>

#include <cassert>
#include <cstdint>

// CBP_DEBUG_BOUNDS: device asserts on every table / shared-state index (debug builds
// only; compute-sanitizer is not available on the GPU pool)
#ifdef CBP_DEBUG_BOUNDS
#define CBP_CHECK(c) assert(c)
#else
#define CBP_CHECK(c) ((void)0)
#endif

namespace cbp {

// phi clamp bounds (reading R9): PHI_HI = 30, PHI_LO = fl32(phi(30))
constexpr float kPhiHi = 30.0f;
constexpr float kPhiLo = 0x1.a56e0cp-43f;

constexpr float kLn2Hi = 0x1.62e400p-1f;
constexpr float kLn2Lo = 0x1.7f7d1cp-20f;
constexpr float kInvLn2 = 0x1.715476p+0f;

__device__ __forceinline__ float ln32(float x)
{
    const int32_t ix = static_cast<int32_t>(__float_as_uint(x) - 0x3f3504f3u);
    const int32_t k = ix >> 23;
    const float m = __uint_as_float((static_cast<uint32_t>(ix) & 0x007fffffu) + 0x3f3504f3u);
    const float f = __fsub_rn(m, 1.0f);
    float p = -0x1.36cf20p-4f;
    p = __fmaf_rn(p, f, 0x1.03a7f6p-3f);
    p = __fmaf_rn(p, f, -0x1.0d15eap-3f);
    p = __fmaf_rn(p, f, 0x1.230f94p-3f);
    p = __fmaf_rn(p, f, -0x1.54816ep-3f);
    p = __fmaf_rn(p, f, 0x1.999e58p-3f);
    p = __fmaf_rn(p, f, -0x1.00020ep-2f);
    p = __fmaf_rn(p, f, 0x1.555556p-2f);
    p = __fmaf_rn(p, f, -0x1.fffffep-2f);
    const float f2 = __fmul_rn(f, f);
    const float lnm = __fmaf_rn(f2, p, f);
    const float kf = static_cast<float>(k);
    const float t = __fmaf_rn(kf, kLn2Lo, lnm);
    return __fmaf_rn(kf, kLn2Hi, t);
}

// regime A (x < 1): phi = x^2 G(x^2) - ln(x/2)
__device__ __forceinline__ float phi_small(float x)
{
    const float l = ln32(__fmul_rn(0.5f, x));
    const float y = __fmul_rn(x, x);
    float g = -0x1.78439ep-16f;
    g = __fmaf_rn(g, y, 0x1.63e3a2p-12f);
    g = __fmaf_rn(g, y, -0x1.3e8c42p-8f);
    g = __fmaf_rn(g, y, 0x1.555552p-4f);
    g = __fmul_rn(g, y);
    return __fsub_rn(g, l);
}

// regime B (x >= 1): t = e^-x = 2^-n e^-r, phi = 2 t H(t^2)
__device__ __forceinline__ float phi_large(float x)
{
    const float a = __fmul_rn(x, kInvLn2);
    const float n = rintf(a);
    float rr = __fmaf_rn(-n, kLn2Hi, x);
    rr = __fmaf_rn(-n, kLn2Lo, rr);
    float e = 0x1.6b4e62p-10f;
    e = __fmaf_rn(e, rr, -0x1.126f76p-7f);
    e = __fmaf_rn(e, rr, 0x1.555796p-5f);
    e = __fmaf_rn(e, rr, -0x1.555406p-3f);
    e = __fmaf_rn(e, rr, 0x1.fffffcp-2f);
    e = __fmaf_rn(e, rr, -1.0f);
    e = __fmaf_rn(e, rr, 1.0f);
    const int32_t ni = static_cast<int32_t>(n);
    const float s = __uint_as_float(static_cast<uint32_t>(127 - ni) << 23);
    const float t = __fmul_rn(e, s);
    const float w = __fmul_rn(t, t);
    float h = 0x1.2e8fe8p-3f;
    h = __fmaf_rn(h, w, 0x1.1b78f8p-3f);
    h = __fmaf_rn(h, w, 0x1.9a05a6p-3f);
    h = __fmaf_rn(h, w, 0x1.555490p-2f);
    h = __fmaf_rn(h, w, 1.0f);
    const float u = __fmul_rn(t, h);
    return __fadd_rn(u, u);
}

// phi v1 reference formula (unclamped): only used to build the v2 table
__device__ __forceinline__ float phi_v1_unclamped(float x)
{
    return (x < 1.0f) ? phi_small(x) : phi_large(x);
}

// ---- phi contract v2: 929-segment cubic in u in [0, 1)
constexpr int kPhiSegs = 929;

// Coefficients of one segment: cubic through v1 at u = 0, 1/4, 3/4, 1 by
// Newton divided differences in IEEE double, in the DESIGN.md order.
__device__ __forceinline__ float4 phi_segment_coeffs(int seg)
{
    const int q4[4] = {0, 1, 3, 4};
    double f[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float x;
        if (seg < 704) {
            const int e = -43 + seg / 16, j = seg % 16;
            x = __fmul_rn(static_cast<float>(64 + 4 * j + q4[k]), __uint_as_float(static_cast<uint32_t>(127 + e - 6) << 23));
        } else {
            x = __fmul_rn(static_cast<float>(64 + 4 * (seg - 704) + q4[k]), 0.03125f);
        }
        f[k] = static_cast<double>(phi_v1_unclamped(x));
    }
    const double d01 = __dmul_rn(__dsub_rn(f[1], f[0]), 4.0);
    const double d12 = __dmul_rn(__dsub_rn(f[2], f[1]), 2.0);
    const double d23 = __dmul_rn(__dsub_rn(f[3], f[2]), 4.0);
    const double d012 = __ddiv_rn(__dmul_rn(__dsub_rn(d12, d01), 4.0), 3.0);
    const double d123 = __ddiv_rn(__dmul_rn(__dsub_rn(d23, d12), 4.0), 3.0);
    const double d0123 = __dsub_rn(d123, d012);
    const double t2 = __dsub_rn(d01, __dmul_rn(d012, 0.25));
    const double t3 = __dmul_rn(d0123, 0.1875);
    float4 c = make_float4(__double2float_rn(f[0]), __double2float_rn(__dadd_rn(t2, t3)),
                           __double2float_rn(__dsub_rn(d012, d0123)), __double2float_rn(d0123));
    if (seg < 704) {
        // device storage form: the local variable of x < 2 is taken as u' = u/16 (no shift),
        // so c1, c2, c3 are stored times 16, 256, 4096 -- exact, and every product of the
        // Horner evaluation is scaled by the same power of two: identical results.
        c.y = __fmul_rn(c.y, 16.0f);
        c.z = __fmul_rn(c.z, 256.0f);
        c.w = __fmul_rn(c.w, 4096.0f);
    }
    return c;
}

// phi(x) = -log(tanh(x/2)) (equ_s2e5) with the R9 input clamp:
// segment index and local u from the float's bits (x < 2) or from 8(x - 2)
// (x >= 2), one 16-byte table load, three FMA.  The contract's output clamp is
// omitted: on every float of [PHI_LO, 30] the cubic already lies in [PHI_LO, 30]
// (exhaustive check, tests/test_oracle_contract.py), so results are identical.
// m19 = 0x7ffff and one = 0x3f800000 are passed in registers so that
// (b & m19) | one is a single LOP3 (immediates would take two).
// x >= 2 without the XU pipe: m = fma_rz(x, 8, 2^23 - 16) = 2^23 + floor(8x - 16)
// exactly (the fma is exact before its one rounding toward zero, ulp 1 in
// [2^23, 2^24)), so seg = bits(m) - bits(2^23) + 704 and u = fma(x, 8, -(16 + i))
// = t - i exactly: the contract's i = (int)t and u = t - (float)i, bit for bit.
// segment index and local variable of x (clamped to [PHI_LO, PHI_HI])
__device__ __forceinline__ void phi32_index(float x, uint32_t m19, uint32_t one, int& seg, float& u)
{
    x = fminf(fmaxf(x, kPhiLo), kPhiHi);
    const uint32_t b = __float_as_uint(x);
    const int seg_lo = static_cast<int>(b >> 19) - 1344;
    uint32_t ub;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(ub) : "r"(b), "r"(m19), "r"(one));   // (b & m19) | one
    const float u_lo = __fsub_rn(__uint_as_float(ub), 1.0f);   // u/16, see phi_segment_coeffs
    const float m = __fmaf_rz(x, 8.0f, 8388592.0f);
    const float u_hi = __fmaf_rn(x, 8.0f, __fsub_rn(8388592.0f, m));
    const int seg_hi = static_cast<int>(__float_as_uint(m)) - (0x4b000000 - 704);
    const bool hi = x >= 2.0f;
    seg = hi ? seg_hi : seg_lo;
    u = hi ? u_hi : u_lo;
    CBP_CHECK(seg >= 0 && seg < kPhiSegs);
}

__device__ __forceinline__ float phi32_cubic(float4 c, float u)
{
    float p = __fmaf_rn(c.w, u, c.z);
    p = __fmaf_rn(p, u, c.y);
    return __fmaf_rn(p, u, c.x);
}

__device__ __forceinline__ float phi32(float x, const float4* __restrict__ tab, uint32_t m19, uint32_t one)
{
    int seg;
    float u;
    phi32_index(x, m19, one, seg, u);
    return phi32_cubic(tab[seg], u);
}

__device__ __forceinline__ float phi32(float x, const float4* __restrict__ tab)
{
    return phi32(x, tab, 0x7ffffu, 0x3f800000u);
}

// The same function with the segment row fetched through the texture path (TEX data
// pipe) from the device copy of the table: identical bits, and its bandwidth adds to the
// shared-memory pipe's (tools/ubench_lookup.cu: 2 LDS.128 + 1 TEX lookups per step take
// the time of the 2 LDS.128 alone).
__device__ __forceinline__ float phi32_tex(float x, cudaTextureObject_t tex, uint32_t m19, uint32_t one)
{
    int seg;
    float u;
    phi32_index(x, m19, one, seg, u);
    return phi32_cubic(tex1Dfetch<float4>(tex, seg), u);
}

// sin / cos of 2 pi m 2^-24 with exact integer quadrant reduction (Box-Muller)
__device__ __forceinline__ void sincos_quarter32(uint32_t m, float& s_out, float& c_out)
{
    const uint32_t q = (m + 0x200000u) >> 22;
    const int32_t fi = static_cast<int32_t>(m) - static_cast<int32_t>(q << 22);
    const float f = __fmul_rn(static_cast<float>(fi), 0x1p-22f);
    const float z = __fmul_rn(f, f);
    float sp = -0x1.2d92c6p-8f;
    sp = __fmaf_rn(sp, z, 0x1.465e90p-4f);
    sp = __fmaf_rn(sp, z, -0x1.4abbb8p-1f);
    sp = __fmaf_rn(sp, z, 0x1.921fb6p+0f);
    const float sn = __fmul_rn(sp, f);
    float cp = 0x1.d9cf32p-11f;
    cp = __fmaf_rn(cp, z, -0x1.55c5c6p-6f);
    cp = __fmaf_rn(cp, z, 0x1.03c1dep-2f);
    cp = __fmaf_rn(cp, z, -0x1.3bd3ccp+0f);
    cp = __fmaf_rn(cp, z, 1.0f);
    switch (q & 3u) {
    case 0: s_out = sn;  c_out = cp;  break;
    case 1: s_out = cp;  c_out = -sn; break;
    case 2: s_out = -sn; c_out = -cp; break;
    default: s_out = -cp; c_out = sn; break;
    }
}

// Philox4x32-10 (Salmon et al., SC'11)
struct u32x4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    }
    return c;
}

// Box-Muller pair from two Philox words
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& n_even, float& n_odd)
{
    const float u1 = __fmul_rn(static_cast<float>((a >> 8) + 1u), 0x1p-24f);
    const float l = ln32(u1);
    const float t = __fmul_rn(-2.0f, l);
    const float rad = __fsqrt_rn(t);
    float s, c;
    sincos_quarter32(b >> 8, s, c);
    n_even = __fmul_rn(rad, c);
    n_odd = __fmul_rn(rad, s);
}

}  // namespace cbp
