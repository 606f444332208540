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

// ---- phi contract v3: 1153-segment cubic in u in [0, 1)
constexpr int kPhiSegs = 1153;

// phi(x) = -log(tanh(x/2)) (equ_s2e5) with the R9 input clamp:
// segment index and local u from the float's bits (x < 2) or from 16(x - 2)
// (x >= 2), one 16-byte table row (built on the host, cbp_api.cpp), three FMA.  The
// contract's output clamp is omitted: on every float of [PHI_LO, 30] the cubic already lies
// in [PHI_LO, 30] (exhaustive check, tests/test_oracle_contract.py), so results are identical.
// m19 = 0x7ffff and one = 0x3f800000 are passed in registers so that
// (b & m19) | one is a single LOP3 (immediates would take two); the x < 2 rows are stored
// for the local variable u' = u/16 (c1, c2, c3 scaled by 16, 256, 4096: exact).
// x >= 2 without the XU pipe: m = fma_rz(x, 16, 2^23 - 32) = 2^23 + floor(16x - 32)
// exactly (the fma is exact before its one rounding toward zero, ulp 1 in
// [2^23, 2^24)), so seg = bits(m) - bits(2^23) + 704 and u = fma(x, 16, -(32 + i))
// = t - i exactly: the contract's i = (int)t and u = t - (float)i, bit for bit.
// segment index and local variable of x (clamped to [PHI_LO, PHI_HI])
__device__ __forceinline__ void phi32_index(float x, uint32_t m19, uint32_t one, int& seg, float& u)
{
    x = fminf(fmaxf(x, kPhiLo), kPhiHi);
    const uint32_t b = __float_as_uint(x);
    const int seg_lo = static_cast<int>(b >> 19) - 1344;
    uint32_t ub;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(ub) : "r"(b), "r"(m19), "r"(one));   // (b & m19) | one
    const float u_lo = __fsub_rn(__uint_as_float(ub), 1.0f);   // u/16
    const float m = __fmaf_rz(x, 16.0f, 8388576.0f);
    const float u_hi = __fmaf_rn(x, 16.0f, __fsub_rn(8388576.0f, m));
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
