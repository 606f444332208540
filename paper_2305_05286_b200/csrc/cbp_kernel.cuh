// cbp_kernel.cuh -- sm_100a kernels of check-belief propagation decoding (templates).
//
// Instantiated per decoding algorithm by cbp_kernels_alg{0,1,2,3}.cu (compiled in parallel);
// the launch dispatch over algorithms lives in cbp_kernels.cu.
//
// One persistent kernel serves cbp_decode, cbp_decode_i8, cbp_channel and
// cbp_ber_sim.  A CTA holds several independent teams; a team
// owns F groups of Zp lanes, a group holds P frames (P = 1 or 2) and lane r of
// a group processes lifted check i*Z + r of the current base row i for all P
// frames at once.  The Z lifted checks of one base row touch disjoint
// variables (each block is a permutation), so processing them in parallel is
// bit-identical to the paper's sequential check order (reading R12).
// Per-group state lives in shared memory with the P frames interleaved, so one
// schedule entry, one address computation and one wide load/store serve all P
// frames (and P = 2 pairs run on the packed FADD2 pipe):
//   QP[N] {Q_v(0..P-1), Phi_v(0..P-1) | hard bit in the sign}, S[M] records, R[E] x P, cw[P][nwords]
// The phi table (contract v2) and the code's schedule tables are staged once per CTA.
//
// Paper steps (§IV-C): init = Step 1 (l.402-422, equ_s4e15-17);
// process_row = Step 2(1) B2V/V2C/C2B (equ_s4e18-22) and 2(2) (equ_s4e23);
// stop logic = Step 2(3) (l.478-485) with readings R4/R5; finish = Step 3 (l.487).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "cbp_internal.h"
#include "contract.cuh"

namespace cbp {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kSign = 0x80000000u;

// independent edges of a check processed together (ILP); remainder two / one at a time
#ifndef CBP_CHUNK
#define CBP_CHUNK 3
#endif
// R_{ci->v} loaded with the chunk's other operands instead of after the commits (DESIGN.md §5:
// C3a -7 %, P2048 -16 %, C2 neutral); 0 restores the load after the commits
#ifndef CBP_EARLY_R
#define CBP_EARLY_R 1
#endif
// A/B switches CBP_TEX_C2B / CBP_TEX_B2V: evaluate the C2B / B2V phi with the table row
// fetched through the texture pipe instead of LDS (default: C2B through TEX, DESIGN.md §5;
// B2V through TEX as well, or one B2V lookup per chunk, measured 4-10% slower).


// ---------------------------------------------------------------- byte-addressed vector access
template <int N>
__device__ __forceinline__ void ldf(const char* b, int off, float* o)
{
    if constexpr (N == 1) {
        o[0] = *reinterpret_cast<const float*>(b + off);
    } else if constexpr (N == 2) {
        const float2 t = *reinterpret_cast<const float2*>(b + off);
        o[0] = t.x; o[1] = t.y;
    } else {
        const float4 t = *reinterpret_cast<const float4*>(b + off);
        o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
    }
}

template <int N>
__device__ __forceinline__ void stf(char* b, int off, const float* v)
{
    if constexpr (N == 1) *reinterpret_cast<float*>(b + off) = v[0];
    else if constexpr (N == 2) *reinterpret_cast<float2*>(b + off) = make_float2(v[0], v[1]);
    else *reinterpret_cast<float4*>(b + off) = make_float4(v[0], v[1], v[2], v[3]);
}

// o = a + b and o = a - b over the P frames (FADD2 for a pair; IEEE rn either way)
template <int P>
__device__ __forceinline__ void vadd(const float* a, const float* b, float* o)
{
    if constexpr (P == 2) {
        const float2 t = __fadd2_rn(make_float2(a[0], a[1]), make_float2(b[0], b[1]));
        o[0] = t.x; o[1] = t.y;
    } else {
        o[0] = __fadd_rn(a[0], b[0]);
    }
}

template <int P>
__device__ __forceinline__ void vsub(const float* a, const float* b, float* o)
{
    if constexpr (P == 2) {
        const float2 t = __fadd2_rn(make_float2(a[0], a[1]), make_float2(-b[0], -b[1]));
        o[0] = t.x; o[1] = t.y;
    } else {
        o[0] = __fsub_rn(a[0], b[0]);
    }
}

// |a| - |b| over the P frames
template <int P>
__device__ __forceinline__ void vabsdiff(const float* a, const float* b, float* o)
{
    if constexpr (P == 2) {
        const float2 t = __fadd2_rn(make_float2(fabsf(a[0]), fabsf(a[1])), make_float2(-fabsf(b[0]), -fabsf(b[1])));
        o[0] = t.x; o[1] = t.y;
    } else {
        o[0] = __fsub_rn(fabsf(a[0]), fabsf(b[0]));
    }
}

// ---------------------------------------------------------------- group state
// Byte strides: QS per variable (QP), RS per edge (R), SS per check record.
template <int P, int ALG>
struct Lay {
    static constexpr int QS = 8 * P;
    static constexpr int RS = 4 * P;
    static constexpr int SU = (ALG == 1) ? 4 : 1;   // check-record stride in units of RS
    static constexpr int SS = RS * SU;
    static constexpr int SW = (ALG == 1) ? 4 : 1;   // words per frame in a check record
};

// A group of P frames.  Record word k of frame p at byte 4 (k P + p) of the record
// (log-tanh: k = 0, S_c with sign = Omega < 0; min-sum: {min, submin, owner | sign, pad}).
template <int P, int ALG>
struct Grp {
    char* qp;
    char* S;
    char* R;
    char* rb;             // base of the hot loop's R offsets: qp (R inside the group) or R (split layout)
    uint32_t* cw;
    int nwords;
    using Ly = Lay<P, ALG>;
    __device__ __forceinline__ float& Q(int v, int p) const { return reinterpret_cast<float*>(qp + v * Ly::QS)[p]; }
    __device__ __forceinline__ float& PH(int v, int p) const { return reinterpret_cast<float*>(qp + v * Ly::QS)[P + p]; }
    __device__ __forceinline__ float& Rw(int e, int p) const { return reinterpret_cast<float*>(R + e * Ly::RS)[p]; }
    __device__ __forceinline__ float& Sw(int c, int k, int p) const
    {
        return reinterpret_cast<float*>(S + c * Ly::SS)[k * P + p];
    }
    __device__ __forceinline__ uint32_t* cwp(int p) const { return cw + p * nwords; }
    // flooding BP (ALG 3): channel LLRs L_v, after the codewords
    __device__ __forceinline__ float& Lv(int v, int p) const
    {
        return reinterpret_cast<float*>(cw + P * nwords)[v * P + p];
    }
};

// Schedule table entry b (two int4, built in cbp_api.cpp for the launch's P and algorithm),
// byte offsets from the group base (QP at 0, check records at S0, R at R0):
//   E0 = {QS jZ, S0 + SU RS row(prev(b)) Z, R0 + RS prev(b) Z, QS s}: variable block (QP), check
//        block of the previous check of the same variables, R block of prev(b), rotation of the block
//   E1 = {RS ds, first ? 0 : ~0, first | kp << 8 | s << 16, R0 + RS b Z}   ds = (s - s_prev) mod Z;
//        first: no latest check in sweep 1 (R1), as a keep mask and a bit; kp = position of prev(b)
//        in its row (min-sum owner, R20); own R block
// The hot loop reads E0 and E1.xy (16 + 8 bytes, 3 shared-memory wavefronts per warp instead of
// 4) and computes the own R block as R0 + b Z RS.
// prev(b) = previous nonzero row of b's column, cyclically (the static "latest check" of
// every variable of the block after sweep 1); prev(b) == b for a degree-1
// column (R3).  Variable of lane r: j Z + (r + s) mod Z; its previous check's row (r + ds) mod Z.

// (t mod n) for t in [0, 2n): unsigned min of t and t - n (two instructions, no predicate)
__device__ __forceinline__ int wrap(int t, int n)
{
    return static_cast<int>(min(static_cast<unsigned>(t), static_cast<unsigned>(t - n)));
}

// variable of lane r in entry e: j Z + (r + s) mod Z, j Z = A.x / QS
template <int QS>
__device__ __forceinline__ int lane_var(const int4* ent, int e, int r, int Z)
{
    int t = r + (ent[2 * e + 1].z >> 16);
    t = (t >= Z) ? t - Z : t;
    return ent[2 * e].x / QS + t;
}

// ---------------------------------------------------------------- team helpers
// !MULTI: a team is one warp holding F groups of Zp lanes; MULTI: a team is TW
// warps holding one group.  Teams synchronise with their own named barrier.
__device__ __forceinline__ void named_bar_sync(int id, int n)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ bool named_bar_or(int id, int n, bool pred)
{
    unsigned out;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.u32 p, %1, 0;\n\t"
        "bar.red.or.pred q, %2, %3, p;\n\t"
        "selp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(out)
        : "r"(static_cast<unsigned>(pred)), "r"(id), "r"(n)
        : "memory");
    return out != 0u;
}

template <bool MULTI>
struct Team {
    int tidx;             // team index in the CTA
    int nthreads;         // threads per team
    int tl;               // thread index within the team
    int slot, r, lane_base;
    bool lane_on;
    unsigned slot_mask;   // lanes of this group within the warp (!MULTI)

    __device__ __forceinline__ void sync() const
    {
        if (MULTI) named_bar_sync(1 + tidx, nthreads);
        else __syncwarp();
    }
    // OR of a group-uniform predicate over the team's groups.  A MULTI team holds one
    // group and every thread derives the control state identically, so the predicate
    // is already team-uniform (no barrier); a warp team votes over its F groups.
    __device__ __forceinline__ bool team_any(bool pred) const
    {
        if (MULTI) return pred;
        return __any_sync(kFull, pred) != 0;
    }
    // OR over the lanes of this group (a synchronisation point)
    __device__ __forceinline__ bool slot_any(bool pred) const
    {
        if (MULTI) return named_bar_or(1 + tidx, nthreads, pred);
        return (__ballot_sync(kFull, pred) & slot_mask) != 0u;
    }
};

// ---------------------------------------------------------------- per-row edge chain
struct Lane {
    int r, rq, rr, ZQ, ZR;            // lane, r QS, r RS, Z QS, Z RS
    int R0;                           // byte offset of the R section in a group
    int slot_bytes;                   // group size (bounds checks of debug builds)
    int r_bytes;                      // end of the R section relative to the R base (debug builds)
    uint32_t m19, one;                // phi local-variable masks as runtime operands (one LOP3)
};

// The texture object of the phi table is passed by value from the kernel parameter at every call
// (never stored in a struct that may be spilled): only a handle the compiler can trace to the
// parameter bank stays in a uniform register; otherwise every TLD is wrapped in a
// uniformisation loop (R2UR + BRA.U.ANY) that serialises the lookups.
using TexH = cudaTextureObject_t;

template <bool TEX>
__device__ __forceinline__ float phi_sel(float x, const float4* __restrict__ ptab, const Lane& L, TexH tex)
{
    if constexpr (TEX) return phi32_tex(x, tex, L.m19, L.one);
    else return phi32(x, ptab, L.m19, L.one);
}

template <int P>
struct RowAcc {
    float Ssum[P];
    uint32_t negw[P];     // bit 31: XOR of the signs of Q^new over the check (sign of Omega)
    uint32_t flipw[P];    // bit 31: some posterior sign flipped (equ_s4e24)
    uint32_t oldbits[P];  // previous hard bits of the check's variables (rollback of a mid-row stop)
};

// check records of the row before / after (log-tanh: S in .x; min-sum: the record)
template <int P>
struct RowOut {
    float4 Snew[P], Sold[P];
    uint32_t oldbits[P];
    bool ok[P];
};

// ---------------------------------------------------------------- CBP log-tanh, producer-side B2V
// DESIGN.md §5.  The B2V message R^new_{cj->v} = sgn(Omega_cj) sgn(Q_v) phi(|S_cj - phi(|Q_v|)|)
// (equ_s4e18, R11) that check c_i applies to its variable v depends only on values that the
// previous check c_j of v left behind: S_cj and neg_cj are not touched again before c_i runs (a
// check is updated once per sweep), and Q_v, Phi_v are c_j's own Q^new_v and phi(|Q^new_v|) (no
// other check visits v in between).  So c_j's lane evaluates it at the end of its own update,
// from the S it has just accumulated, commits it to R_{cj->v} (equ_s4e22) and leaves the
// posterior Lambda_v = Q^new_v + R^new_{cj->v} (equ_s4e20 of c_i, same fp32 operations, same
// bits) in the variable's slot.  c_i then reads Lambda_v and its own R_{ci->v}:
// Q^new = Lambda_v - R_{ci->v} (equ_s4e19).  Every quantity keeps the paper's values and
// rounding; only the lane that evaluates the B2V phi changes.  Consequences:
//  * R is lane-private: lane r reads and writes only R_{iZ+r -> v}, slot b Z + r (coalesced);
//  * no S_cj read, no cached Phi, no first-visit mask: before v's first visit its slot holds
//    Lambda_v = L_v + 0 (R1: R^new = +0, so Lambda = fl(L_v + 0));
//  * a degree-1 column (prev(b) = b, R3) needs no special case: R_{ci->v} is the value this lane
//    committed at its previous update, which is exactly the R^new of the commit-before-read.
// Variable slot QP[v] = {Lambda'_v (the next visitor's posterior), H_v (sign = hard decision
// x_v of the latest visit: the Lambda that visit read; layered BP: Lambda'_v itself)}.
// Schedule entry b for this layout: E0 = {QS jZ, QS s} (cbp_api.cpp).

// the R slot of lane r for entry b, relative to g.rb
__device__ __forceinline__ int r_slot(const Lane& L, int b) { return L.R0 + b * L.ZR + L.rr; }

// Phase 1 of edge k: Lambda, flip, Q^new, C2B phi and the ordered S accumulation (R12).
template <int P, bool TEXC = CBP_TEX_C2B>
__device__ __forceinline__ void cbp_phase1(const float (&qp)[2 * P], const float (&ro)[P], float (&q)[P],
                                           float (&ph)[P], const float4* __restrict__ ptab, const Lane& L,
                                           TexH tex, RowAcc<P>& acc)
{
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const uint32_t lw = __float_as_uint(qp[p]), hw = __float_as_uint(qp[P + p]);
        acc.flipw[p] |= lw ^ hw;                                // equ_s4e24 (R7): sgn Lambda vs previous decision
        acc.oldbits[p] = __funnelshift_l(hw, acc.oldbits[p], 1);   // previous hard bit, edge k at bit dc-1-k
    }
    vsub<P>(qp, ro, q);                                         // equ_s4e19 (R15): Q^new = Lambda - R_{ci->v}
#pragma unroll
    for (int p = 0; p < P; ++p) ph[p] = phi_sel<TEXC>(fabsf(q[p]), ptab, L, tex);   // C2B (equ_s4e21, equ_ae4)
    vadd<P>(acc.Ssum, ph, acc.Ssum);                            // S in ascending variable order (R12)
#pragma unroll
    for (int p = 0; p < P; ++p) acc.negw[p] ^= __float_as_uint(q[p]);   // Q^new is never -0
}

// Phase 2 of edge k: R^new_{c->v} = sgn(Omega_c) sgn(Q^new) phi(|S - Phi|) and Lambda' = Q^new + R^new.
template <int P, bool TEXB = CBP_TEX_B2V>
__device__ __forceinline__ void cbp_phase2(const RowAcc<P>& acc, const float (&q)[P], const float (&ph)[P],
                                           float (&rn)[P], float (&lamn)[P], const float4* __restrict__ ptab,
                                           const Lane& L, TexH tex)
{
    float d[P];
    vsub<P>(acc.Ssum, ph, d);                                   // |S - Phi| (R10); S >= 0 here
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const float mag = phi_sel<TEXB>(fabsf(d[p]), ptab, L, tex);
        rn[p] = __uint_as_float(__float_as_uint(mag) | ((acc.negw[p] ^ __float_as_uint(q[p])) & kSign));
    }
    vadd<P>(q, rn, lamn);                                       // equ_s4e20 of the next visitor (never -0)
}

// One check update with DC edges held in registers (DC <= CBP_DC_REG).  ALG 2: layered BP
// (reading R22) -- the same messages, with the hard decision taken from Lambda' at once.
template <int DC, int P, int ALG>
__device__ __forceinline__ RowAcc<P> cbp_row_reg(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0,
                                                 const Lane& L, TexH tex, const Grp<P, ALG>& g)
{
    using Ly = Lay<P, ALG>;
    constexpr bool LBP = ALG == 2;
    RowAcc<P> acc;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        acc.Ssum[p] = 0.0f;
        acc.negw[p] = acc.flipw[p] = acc.oldbits[p] = 0u;
    }
    int aqp[DC];
    float vs[DC][2 * P], ro[DC][P], q[DC][P], ph[DC][P];
    const int rrow = r_slot(L, e0);
#pragma unroll
    for (int k = 0; k < DC; ++k) {                              // all loads of the row first
        const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + k));
        aqp[k] = A.x + wrap(L.rq + A.y, L.ZQ);
        CBP_CHECK(aqp[k] >= 0 && aqp[k] + Ly::QS <= L.slot_bytes && rrow + k * L.ZR + Ly::RS <= L.r_bytes);
        ldf<2 * P>(g.qp, aqp[k], vs[k]);                        // {Lambda_v, H_v}
        ldf<P>(g.rb, rrow + k * L.ZR, ro[k]);                   // R_{c->v}
        if constexpr (LBP) {
#pragma unroll
            for (int p = 0; p < P; ++p) vs[k][P + p] = vs[k][p];
        }
    }
#pragma unroll
    for (int k = 0; k < DC; ++k) cbp_phase1<P>(vs[k], ro[k], q[k], ph[k], ptab, L, tex, acc);
    // all B2V lookups before the first store (a table load may not move above a shared-memory
    // store the compiler cannot prove disjoint)
    float rn[DC][P], lamn[DC][P];
#pragma unroll
    for (int k = 0; k < DC; ++k) cbp_phase2<P>(acc, q[k], ph[k], rn[k], lamn[k], ptab, L, tex);
#pragma unroll
    for (int k = 0; k < DC; ++k) {
        float st[2 * P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            st[p] = lamn[k][p];
            st[P + p] = LBP ? lamn[k][p] : vs[k][p];            // H_v: this visit's decision (equ_s2e7)
        }
        stf<2 * P>(g.qp, aqp[k], st);
        stf<P>(g.rb, rrow + k * L.ZR, rn[k]);                   // equ_s4e22 commit of R_{c->v}
    }
    return acc;
}

// The same update for rows longer than CBP_DC_REG: two passes in chunks of U edges (all loads of
// a chunk first: U independent phi chains) and a remainder one edge at a time; between the phases
// each variable's slot parks {Q^new, Phi | sign of the decision} (only this lane touches the
// variable during the row).  Both phi rows from the shared-memory table (a function that is not
// inlined cannot keep the texture handle in a uniform register).
template <int U, int P, int ALG>
__device__ __forceinline__ void park_p1(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0, int k0,
                                        int rrow, const Lane& L, const Grp<P, ALG>& g, RowAcc<P>& acc)
{
    constexpr bool LBP = ALG == 2;
    int a[U];
    float qp[U][2 * P], ro[U][P], q[U][P], ph[U][P];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + k0 + u));
        a[u] = A.x + wrap(L.rq + A.y, L.ZQ);
        ldf<2 * P>(g.qp, a[u], qp[u]);
        ldf<P>(g.rb, rrow + (k0 + u) * L.ZR, ro[u]);
        if (LBP) {
#pragma unroll
            for (int p = 0; p < P; ++p) qp[u][P + p] = qp[u][p];
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cbp_phase1<P, false>(qp[u], ro[u], q[u], ph[u], ptab, L, 0, acc);
#pragma unroll
    for (int u = 0; u < U; ++u) {
        float st[2 * P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            st[p] = q[u][p];
            st[P + p] = __uint_as_float(__float_as_uint(ph[u][p]) | (__float_as_uint(qp[u][p]) & kSign));
        }
        stf<2 * P>(g.qp, a[u], st);
    }
}

template <int U, int P, int ALG>
__device__ __forceinline__ void park_p2(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0, int k0,
                                        int rrow, const Lane& L, const Grp<P, ALG>& g, const RowAcc<P>& acc)
{
    constexpr bool LBP = ALG == 2;
    int a[U];
    float qp[U][2 * P];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + k0 + u));
        a[u] = A.x + wrap(L.rq + A.y, L.ZQ);
        ldf<2 * P>(g.qp, a[u], qp[u]);
    }
    float rn[U][P], lamn[U][P];
#pragma unroll
    for (int u = 0; u < U; ++u) {                               // lookups first (see cbp_row_reg)
        float q[P], ph[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            q[p] = qp[u][p];
            ph[p] = fabsf(qp[u][P + p]);
        }
        cbp_phase2<P, false>(acc, q, ph, rn[u], lamn[u], ptab, L, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        float st[2 * P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            st[p] = lamn[u][p];
            st[P + p] = LBP ? lamn[u][p] : qp[u][P + p];       // sign = the decision of this visit
        }
        stf<2 * P>(g.qp, a[u], st);
        stf<P>(g.rb, rrow + (k0 + u) * L.ZR, rn[u]);
    }
}

template <int P, int ALG>
__device__ __noinline__ RowAcc<P> cbp_row_park(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0,
                                               int dc, const Lane& L, const Grp<P, ALG>& g)
{
    constexpr int U = 4;
    RowAcc<P> acc;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        acc.Ssum[p] = 0.0f;
        acc.negw[p] = acc.flipw[p] = acc.oldbits[p] = 0u;
    }
    const int rrow = r_slot(L, e0);
    int k = 0;
#pragma unroll 1
    for (; k + U <= dc; k += U) park_p1<U, P, ALG>(ent, ptab, e0, k, rrow, L, g, acc);
#pragma unroll 1
    for (; k < dc; ++k) park_p1<1, P, ALG>(ent, ptab, e0, k, rrow, L, g, acc);
    k = 0;
#pragma unroll 1
    for (; k + U <= dc; k += U) park_p2<U, P, ALG>(ent, ptab, e0, k, rrow, L, g, acc);
#pragma unroll 1
    for (; k < dc; ++k) park_p2<1, P, ALG>(ent, ptab, e0, k, rrow, L, g, acc);
    return acc;
}

template <int P, int ALG>
__device__ __forceinline__ RowAcc<P> cbp_row_dispatch(const int4* __restrict__ ent, const float4* __restrict__ ptab,
                                                      int e0, int dc, const Lane& L, TexH tex, const Grp<P, ALG>& g)
{
    switch (dc) {
#if CBP_DC_REG >= 1
    case 1: return cbp_row_reg<1, P, ALG>(ent, ptab, e0, L, tex, g);
    case 2: return cbp_row_reg<2, P, ALG>(ent, ptab, e0, L, tex, g);
    case 3: return cbp_row_reg<3, P, ALG>(ent, ptab, e0, L, tex, g);
    case 4: return cbp_row_reg<4, P, ALG>(ent, ptab, e0, L, tex, g);
    case 5: return cbp_row_reg<5, P, ALG>(ent, ptab, e0, L, tex, g);
    case 6: return cbp_row_reg<6, P, ALG>(ent, ptab, e0, L, tex, g);
#endif
#if CBP_DC_REG >= 8
    case 7: return cbp_row_reg<7, P, ALG>(ent, ptab, e0, L, tex, g);
    case 8: return cbp_row_reg<8, P, ALG>(ent, ptab, e0, L, tex, g);
#endif
    default: return cbp_row_park<P, ALG>(ent, ptab, e0, dc, L, g);
    }
}

// Step 2(1)-(2) of one check per lane (log-tanh CBP or layered BP): the row update, the stored
// S_c (with sign = Omega < 0; the Omega output and the rollback of a mid-row stop), the stop
// flags.  `keep_old`: the stop window may fill in this row, keep the previous record.
template <int P, int ALG>
__device__ __forceinline__ RowOut<P> process_row(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0,
                                                 int dc, int sidx, const Lane& L, TexH tex, const Grp<P, ALG>& g,
                                                 bool keep_old)
{
    constexpr bool LBP = ALG == 2;
    RowOut<P> o;
    float Sold[P];
#pragma unroll
    for (int p = 0; p < P; ++p) Sold[p] = 0.0f;
    if (keep_old) ldf<P>(g.S, sidx, Sold);
    const RowAcc<P> acc = cbp_row_dispatch<P, ALG>(ent, ptab, e0, dc, L, tex, g);
    float Snew[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        Snew[p] = __uint_as_float(__float_as_uint(acc.Ssum[p]) | (acc.negw[p] & kSign));
        o.Snew[p] = make_float4(Snew[p], 0.0f, 0.0f, 0.0f);
        o.Sold[p] = make_float4(Sold[p], 0.0f, 0.0f, 0.0f);
        o.oldbits[p] = acc.oldbits[p];
        o.ok[p] = ((acc.negw[p] | acc.flipw[p]) & kSign) == 0u;   // equ_s4e2 and equ_s4e24 for this check
    }
    if (!LBP) stf<P>(g.S, sidx, Snew);                            // equ_s4e23
    return o;
}

// ---------------------------------------------------------------- normalized min-sum CBP
// PAPER.md l.577-603 (equ_s4e18xx, equ_s4e21xx) with reading R20: per check and frame a
// record {min, submin, owner | sign << 31, -} of m = fl(alpha |Q^new|); B2V magnitude =
// submin if v owns the minimum (owner = v's edge index in the check) else min; signs as
// psi- (equ_s4e13).  Schedule, V2C, commit and stop rule are those of the log-tanh path.
template <int P>
struct MsAcc {
    float m1[P], m2[P];
    uint32_t own[P], negw[P], flipw[P], oldbits[P];
};

// words {m1, m2, ow} of the P frames of a record: P = 1 one 16-byte load, P = 2 16 + 8 bytes
template <int P>
__device__ __forceinline__ void ld_rec(const char* S, int off, float (&m1)[P], float (&m2)[P], uint32_t (&ow)[P])
{
    if constexpr (P == 1) {
        const float4 t = *reinterpret_cast<const float4*>(S + off);
        m1[0] = t.x; m2[0] = t.y; ow[0] = __float_as_uint(t.z);
    } else {
        const float4 t = *reinterpret_cast<const float4*>(S + off);
        const uint2 w = *reinterpret_cast<const uint2*>(S + off + 16);
        m1[0] = t.x; m1[1] = t.y; m2[0] = t.z; m2[1] = t.w; ow[0] = w.x; ow[1] = w.y;
    }
}

template <int P>
__device__ __forceinline__ void st_rec(char* S, int off, const float (&m1)[P], const float (&m2)[P], const uint32_t (&ow)[P])
{
    if constexpr (P == 1) {
        *reinterpret_cast<float4*>(S + off) = make_float4(m1[0], m2[0], __uint_as_float(ow[0]), 0.0f);
    } else {
        *reinterpret_cast<float4*>(S + off) = make_float4(m1[0], m1[1], m2[0], m2[1]);
        *reinterpret_cast<uint2*>(S + off + 16) = make_uint2(ow[0], ow[1]);
    }
}

template <int U, int P>
__device__ __forceinline__ void edge_chunk_ms(const int4* __restrict__ ent, int e0, int k0, const Lane& L,
                                              const Grp<P, 1>& g, const uint32_t (&s1m)[P], float alpha, MsAcc<P>& acc)
{
    using Ly = Lay<P, 1>;
    int aqp[U], aw[U], ar[U], kp[U];
    float q[U][P], p0[U][P], Rn[U][P];
    float cm1[U][P], cm2[U][P];
    uint32_t cow[U][P], fkeep[U];
#if CBP_EARLY_R
    float roe[U][P];
#endif
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int b = e0 + k0 + u;
        const int4 A = ent[2 * b];
        const int4 B = ent[2 * b + 1];
        const int tq = wrap(L.rq + A.w, L.ZQ);
        const int tr = wrap(L.rr + B.x, L.ZR);
        CBP_CHECK(A.y + Ly::SU * tr + Ly::SS <= L.slot_bytes);
        aqp[u] = A.x + tq;
        aw[u] = A.z + tr;
        ar[u] = L.R0 + b * L.ZR + L.rr;
        fkeep[u] = static_cast<uint32_t>(B.y);
        kp[u] = (B.z >> 8) & 0xff;
        float qp[2 * P];
        ldf<2 * P>(g.qp, aqp[u], qp);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            q[u][p] = qp[p];
            p0[u][p] = qp[P + p];
        }
        ld_rec<P>(g.qp, A.y + Ly::SU * tr, cm1[u], cm2[u], cow[u]);   // record of the previous check c_j
#if CBP_EARLY_R
        ldf<P>(g.rb, ar[u], roe[u]);                        // R_{ci->v} early (edge_chunk)
#endif
    }
    // B2V (equ_s4e18xx)
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const uint32_t ow = cow[u][p];
            const float mag = (static_cast<int>(ow & 0xffu) == kp[u]) ? cm2[u][p] : cm1[u][p];
            Rn[u][p] = __uint_as_float((__float_as_uint(mag) | ((ow ^ __float_as_uint(q[u][p])) & kSign)) &
                                       (fkeep[u] | s1m[p]));
        }
#pragma unroll
    for (int u = 0; u < U; ++u) stf<P>(g.rb, aw[u], Rn[u]);   // commit of R_{cj->v} (R2, R3)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        float ro[P], lam[P], qn[P], st[2 * P];
#if CBP_EARLY_R
#pragma unroll
        for (int p = 0; p < P; ++p) ro[p] = (aw[u] == ar[u]) ? Rn[u][p] : roe[u][p];   // degree-1 column: R3
#else
        ldf<P>(g.rb, ar[u], ro);
#endif
        vadd<P>(q[u], Rn[u], lam);                           // equ_s4e20
        vsub<P>(lam, ro, qn);                                // equ_s4e19
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const uint32_t lb = __float_as_uint(lam[p]) & kSign;
            acc.flipw[p] |= __float_as_uint(lam[p]) ^ __float_as_uint(p0[u][p]);
            // previous hard bit, edge k at bit dc-1-k (one funnel shift)
            acc.oldbits[p] = __funnelshift_l(__float_as_uint(p0[u][p]), acc.oldbits[p], 1);
            // C2B (equ_s4e21xx), in ascending edge order, branch-free:
            // m < m1: (m1, m2, own) <- (m, m1, k); else m2 <- min(m2, m).  m1 <= m2 always.
            const float m = __fmul_rn(alpha, fabsf(qn[p]));
            const bool lt = m < acc.m1[p];
            acc.m2[p] = fminf(acc.m2[p], fmaxf(acc.m1[p], m));
            acc.own[p] = lt ? static_cast<uint32_t>(k0 + u) : acc.own[p];
            acc.m1[p] = fminf(acc.m1[p], m);
            acc.negw[p] ^= __float_as_uint(qn[p]);
            st[p] = qn[p];
            st[P + p] = __uint_as_float(lb);
        }
        stf<2 * P>(g.qp, aqp[u], st);
    }
}

template <int P>
__device__ __forceinline__ RowOut<P> process_row_ms(const int4* __restrict__ ent, int e0, int dc, int sidx,
                                                    const Lane& L, const Grp<P, 1>& g, const uint32_t (&s1)[P],
                                                    float alpha)
{
    using Ly = Lay<P, 1>;
    const float inf = __uint_as_float(0x7f800000u);
    MsAcc<P> acc;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        acc.m1[p] = acc.m2[p] = inf;                         // Omega^(-1) = (inf, inf)
        acc.own[p] = acc.negw[p] = acc.flipw[p] = acc.oldbits[p] = 0u;
    }
    float om1[P], om2[P];
    uint32_t oow[P];
    ld_rec<P>(g.S, Ly::SU * sidx, om1, om2, oow);
    int k0 = 0;
    for (; k0 + CBP_CHUNK <= dc; k0 += CBP_CHUNK) edge_chunk_ms<CBP_CHUNK, P>(ent, e0, k0, L, g, s1, alpha, acc);
    if (CBP_CHUNK > 2)
        for (; k0 + 2 <= dc; k0 += 2) edge_chunk_ms<2, P>(ent, e0, k0, L, g, s1, alpha, acc);
    if (k0 < dc) edge_chunk_ms<1, P>(ent, e0, k0, L, g, s1, alpha, acc);
    uint32_t nw[P];
    RowOut<P> o;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        nw[p] = acc.own[p] | (acc.negw[p] & kSign);
        o.Snew[p] = make_float4(acc.m1[p], acc.m2[p], __uint_as_float(nw[p]), 0.0f);
        o.Sold[p] = make_float4(om1[p], om2[p], __uint_as_float(oow[p]), 0.0f);
        o.oldbits[p] = acc.oldbits[p];
        o.ok[p] = ((acc.negw[p] | acc.flipw[p]) & kSign) == 0u;
    }
    st_rec<P>(g.S, Ly::SU * sidx, acc.m1, acc.m2, nw);
    return o;
}

// ---------------------------------------------------------------- comparison schedules (NEXT-3)
// Layered BP (ALG 2, reading R22): process_row<P, true> above -- the same
// messages as CBP's producer-side form, Q = Lambda - R_{c->v} (equ_s2e10), R^new by the
// phi-domain leave-one-out rule (equ_s2e4), Lambda = Q + R^new (equ_s2e12), with the hard
// decision taken from the new Lambda at once.

// Flooding BP (ALG 3, reading R22).  QP = {Lambda_acc, Lambda_old}: all
// checks read Lambda_old (the previous iteration's posterior, .y, whose sign is the hard bit)
// and add their new messages into Lambda_acc (.x, started at L_v) in ascending row order
// (equ_s2e6); after the last row the variable pass makes Lambda_acc the new Lambda_old.
// Pass 1: Q = Lambda_old - R (equ_s2e3), Phi = phi(|Q|), S += Phi; the R slot (own edge) parks
// Phi with the sign of Q.  Pass 2: R^new = sgn phi(|S - Phi|) (equ_s2e4), Lambda_acc += R^new.
template <int U, int P>
__device__ __forceinline__ void fbp_pass1(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0,
                                          int k0, const Lane& L, TexH tex, const Grp<P, 3>& g, float (&S)[P],
                                          uint32_t (&negw)[P])
{
    int ar[U];
    float q[U][P], ph[U][P];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int b = e0 + k0 + u;
        const int4 A = ent[2 * b];
        const int aqp = A.x + wrap(L.rq + A.w, L.ZQ);
        ar[u] = L.R0 + b * L.ZR + L.rr;
        CBP_CHECK(aqp >= 0 && aqp + 8 * P <= L.slot_bytes && ar[u] + 4 * P <= L.r_bytes);
        float qp[2 * P], ro[P], lo[P];
        ldf<2 * P>(g.qp, aqp, qp);
        ldf<P>(g.rb, ar[u], ro);
#pragma unroll
        for (int p = 0; p < P; ++p) lo[p] = qp[P + p];
        vsub<P>(lo, ro, q[u]);                                   // equ_s2e3 (Lambda_old - R)
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int p = 0; p < P; ++p) ph[u][p] = phi_sel<CBP_TEX_C2B>(fabsf(q[u][p]), ptab, L, tex);
#pragma unroll
    for (int u = 0; u < U; ++u) {
        vadd<P>(S, ph[u], S);
        float st[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            negw[p] ^= __float_as_uint(q[u][p]);
            st[p] = __uint_as_float(__float_as_uint(ph[u][p]) | (__float_as_uint(q[u][p]) & kSign));
        }
        stf<P>(g.rb, ar[u], st);
    }
}

template <int U, int P>
__device__ __forceinline__ void fbp_pass2(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0,
                                          int k0, const Lane& L, TexH tex, const Grp<P, 3>& g, const float (&S)[P],
                                          const uint32_t (&negw)[P])
{
    int aqp[U], ar[U];
    float w[U][P], acc[U][P], Rn[U][P];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int b = e0 + k0 + u;
        const int4 A = ent[2 * b];
        aqp[u] = A.x + wrap(L.rq + A.w, L.ZQ);
        ar[u] = L.R0 + b * L.ZR + L.rr;
        ldf<P>(g.rb, ar[u], w[u]);
        float qp[2 * P];
        ldf<2 * P>(g.qp, aqp[u], qp);
#pragma unroll
        for (int p = 0; p < P; ++p) acc[u][p] = qp[p];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        float ph[P], d[P];
#pragma unroll
        for (int p = 0; p < P; ++p) ph[p] = fabsf(w[u][p]);
        vsub<P>(S, ph, d);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const float mag = phi_sel<CBP_TEX_B2V>(fabsf(d[p]), ptab, L, tex);   // equ_s2e4
            Rn[u][p] = __uint_as_float(__float_as_uint(mag) | ((negw[p] ^ __float_as_uint(w[u][p])) & kSign));
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        float na[P];
        vadd<P>(acc[u], Rn[u], na);                              // equ_s2e6, ascending checks
        stf<P>(g.rb, ar[u], Rn[u]);
#pragma unroll
        for (int p = 0; p < P; ++p) reinterpret_cast<float*>(g.qp + aqp[u])[p] = na[p];
    }
}

template <int P>
__device__ __forceinline__ void process_row_fbp(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0,
                                                int dc, const Lane& L, TexH tex, const Grp<P, 3>& g)
{
    float S[P];
    uint32_t negw[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        S[p] = 0.0f;
        negw[p] = 0u;
    }
    int k0 = 0;
    for (; k0 + CBP_CHUNK <= dc; k0 += CBP_CHUNK) fbp_pass1<CBP_CHUNK, P>(ent, ptab, e0, k0, L, tex, g, S, negw);
    for (; k0 < dc; ++k0) fbp_pass1<1, P>(ent, ptab, e0, k0, L, tex, g, S, negw);
    k0 = 0;
    for (; k0 + CBP_CHUNK <= dc; k0 += CBP_CHUNK) fbp_pass2<CBP_CHUNK, P>(ent, ptab, e0, k0, L, tex, g, S, negw);
    for (; k0 < dc; ++k0) fbp_pass2<1, P>(ent, ptab, e0, k0, L, tex, g, S, negw);
}

// write hard bits (sign of Phi) of lane r's variables of frame p in row (e0, dc); returns the previous ones
template <int P, int ALG>
__device__ __forceinline__ uint32_t swap_row_bits(const int4* __restrict__ ent, int e0, int dc, int r, int Z, int p,
                                                  uint32_t bits, const Grp<P, ALG>& g)
{
    // bit of edge k at position dc-1-k (the order edge_chunk accumulates them in)
    uint32_t prev = 0;
    for (int k = 0; k < dc; ++k) {
        const int v = lane_var<8 * P>(ent, e0 + k, r, Z);
        const uint32_t w = __float_as_uint(g.PH(v, p));
        prev = (prev << 1) | (w >> 31);
        g.PH(v, p) = __uint_as_float((w & ~kSign) | (((bits >> (dc - 1 - k)) & 1u) << 31));
    }
    return prev;
}

// parity of lane r's checks over all rows, from the hard bits (sign of Phi) of frame p
template <int P, int ALG>
__device__ __forceinline__ bool lane_syndrome(const int4* __restrict__ ent, const int32_t* row_ptr, int mb, int r,
                                              int Z, int p, const Grp<P, ALG>& g)
{
    uint32_t nz = 0;
    for (int i = 0; i < mb; ++i) {
        uint32_t par = 0;
        for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) par ^= __float_as_uint(g.PH(lane_var<8 * P>(ent, k, r, Z), p)) >> 31;
        nz |= par;
    }
    return nz != 0u;
}

// lambda_i[r] = XOR of the info bits of lifted check i*Z + r (encoder)
template <int QS>
__device__ __forceinline__ uint32_t info_parity(const int4* __restrict__ ent, const int32_t* row_ptr, int i, int r,
                                                int Z, int K, const uint32_t* cw)
{
    uint32_t par = 0;
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        if (ent[2 * k].x / QS >= K) continue;                   // parity column
        const int v = lane_var<QS>(ent, k, r, Z);
        par ^= (cw[v >> 5] >> (v & 31)) & 1u;
    }
    return par;
}

// Step 1 (equ_s4e15) for variable v of frame p with channel LLR L_v.
// CBP log-tanh / layered BP (producer-side layout): {Lambda_v, H_v} = fl(L_v + 0) twice -- the
// first visit's posterior Q_v + R^new with R^new = +0 (R1), and the initial decision L_v < 0 (R7,
// the +0 turns an input -0 into +0).  Min-sum CBP: Q_v = L_v and the decision bit as +-0.
// Flooding BP: Lambda (old) = L_v, the accumulator and L_v itself.
// (`raw`: cbp_channel, which outputs L_v itself)
template <int P, int ALG>
__device__ __forceinline__ void init_var(const Grp<P, ALG>& g, int v, int p, float Lv, bool raw = false)
{
    if constexpr (ALG == 0 || ALG == 2) {
        const float l0 = raw ? Lv : __fadd_rn(Lv, 0.0f);
        g.Q(v, p) = l0;
        g.PH(v, p) = l0;
    } else if constexpr (ALG == 1) {
        g.Q(v, p) = Lv;
        g.PH(v, p) = Lv < 0.0f ? -0.0f : 0.0f;
    } else {
        g.Q(v, p) = Lv;
        g.PH(v, p) = Lv;
        g.Lv(v, p) = Lv;
    }
}

// ---------------------------------------------------------------- channel (a2-a4)
// Frames p with fresh[p] of the group: info bits, encoding, BPSK/AWGN LLRs written into
// the group state (Q_v = L_v, hard bit of L_v), R and the check records zeroed.
template <bool MULTI, int P, int ALG>
__device__ void channel_frames(const KernelArgs& a, const Team<MULTI>& tm, const bool (&fresh)[P],
                               const int64_t (&fidx)[P], const int4* ent, const int32_t* row_ptr,
                               const int16_t* pshift, const Grp<P, ALG>& g)
{
    using Ly = Lay<P, ALG>;
    const DevCode& C = a.code;
    const int Z = C.Z, r = tm.r;
    const uint32_t k0 = static_cast<uint32_t>(a.seed), k1 = static_cast<uint32_t>(a.seed >> 32);
    if (a.llr_mode & 2) {
        // all-zero codeword (CBP_TX_ZERO, reading R23): symbols +1, no info bits, no encoder
#pragma unroll
        for (int p = 0; p < P; ++p) {
            if (!(fresh[p] && tm.lane_on)) continue;
            for (int v = r; v < C.N; v += Z) g.Q(v, p) = 1.0f;
            for (int w = r; w < C.nwords; w += Z) g.cwp(p)[w] = 0u;
        }
        tm.sync();
    } else {
    // (a2) info words: word w = Philox(w/4, f_lo, f_hi, 0)[w%4]
#pragma unroll
    for (int p = 0; p < P; ++p) {
        if (!(fresh[p] && tm.lane_on)) continue;
        const int64_t gframe = a.frame_begin + fidx[p];
        const uint32_t flo = static_cast<uint32_t>(gframe), fhi = static_cast<uint32_t>(static_cast<uint64_t>(gframe) >> 32);
        uint32_t* cw = g.cwp(p);
        const int nblk = (C.kwords + 3) / 4;
        for (int b = r; b < nblk; b += Z) {
            const u32x4 x = philox4x32_10(u32x4{static_cast<uint32_t>(b), flo, fhi, 0u}, k0, k1);
            const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int w = 4 * b + m;
                if (w < C.kwords) {
                    uint32_t word = xs[m];
                    if (w == C.kwords - 1 && (C.K & 31)) word &= (1u << (C.K & 31)) - 1u;
                    cw[w] = word;
                }
            }
        }
    }
    tm.sync();
    // (a3) systematic part and p0 = XOR of the core rows' lambda (Q holds the symbol 1 - 2c)
#pragma unroll
    for (int p = 0; p < P; ++p) {
        if (!(fresh[p] && tm.lane_on)) continue;
        const uint32_t* cw = g.cwp(p);
        for (int v = r; v < C.K; v += Z) g.Q(v, p) = ((cw[v >> 5] >> (v & 31)) & 1u) ? -1.0f : 1.0f;
        uint32_t p0 = 0;
        for (int i = 0; i < C.core; ++i) {
            const uint32_t lam = info_parity<8 * P>(ent, row_ptr, i, r, Z, C.K, cw);
            g.Sw(i * Z + r, 0, p) = __uint_as_float(lam);   // lambda_i[r] kept for the next pass (S is free here)
            p0 ^= lam;
        }
        g.Q(C.kb * Z + r, p) = p0 ? -1.0f : 1.0f;
    }
    tm.sync();
    // p_t = lambda_{t-1} ^ p_{t-1} ^ P^{s0} p0 (row t-1), extension p = lambda
#pragma unroll
    for (int p = 0; p < P; ++p) {
        if (!(fresh[p] && tm.lane_on)) continue;
        uint32_t pprev = 0;
        for (int t = 1; t < C.core; ++t) {
            uint32_t pt = __float_as_uint(g.Sw((t - 1) * Z + r, 0, p));   // lambda_{t-1}[r]
            if (t >= 2) pt ^= pprev;
            const int s0 = pshift[t - 1];
            if (s0 >= 0) {
                int rr = r + s0;
                rr = (rr >= Z) ? rr - Z : rr;
                pt ^= g.Q(C.kb * Z + rr, p) < 0.0f ? 1u : 0u;
            }
            g.Q((C.kb + t) * Z + r, p) = pt ? -1.0f : 1.0f;
            pprev = pt;
        }
        for (int k = 0; k < C.mb - C.core; ++k) {
            const uint32_t pe = info_parity<8 * P>(ent, row_ptr, C.core + k, r, Z, C.K, g.cwp(p));
            g.Q((C.kb + C.core + k) * Z + r, p) = pe ? -1.0f : 1.0f;
        }
    }
    tm.sync();
    // transmitted codeword words
#pragma unroll
    for (int p = 0; p < P; ++p) {
        if (!(fresh[p] && tm.lane_on)) continue;
        for (int w = r; w < C.nwords; w += Z) {
            uint32_t word = 0;
            for (int b = 0; b < 32; ++b) {
                const int v = 32 * w + b;
                if (v < C.N && g.Q(v, p) < 0.0f) word |= 1u << b;
            }
            g.cwp(p)[w] = word;
        }
    }
    tm.sync();
    }
    // (a4) BPSK + AWGN + LLR: y = (1-2c) + sigma n, L = (2/sigma^2) y  (equ_s4e15, R17)
#pragma unroll
    for (int p = 0; p < P; ++p) {
        if (!(fresh[p] && tm.lane_on)) continue;
        const int64_t gframe = a.frame_begin + fidx[p];
        const uint32_t flo = static_cast<uint32_t>(gframe), fhi = static_cast<uint32_t>(static_cast<uint64_t>(gframe) >> 32);
        const int nblk = (C.N + 3) / 4;
        for (int b = r; b < nblk; b += Z) {
            const u32x4 x = philox4x32_10(u32x4{static_cast<uint32_t>(b), flo, fhi, 1u}, k0, k1);
            float n[4];
            box_muller(x.x, x.y, n[0], n[1]);
            box_muller(x.z, x.w, n[2], n[3]);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int v = 4 * b + m;
                if (v >= C.N) break;
                const float y = __fadd_rn(g.Q(v, p), __fmul_rn(a.sigma, n[m]));
                float Lv = __fmul_rn(a.scale, y);
                if (a.llr_mode & 1) {
                    float qq = rintf(__fmul_rn(Lv, 4.0f));
                    qq = fminf(fmaxf(qq, -127.0f), 127.0f);
                    Lv = __fmul_rn(qq, 0.25f);
                }
                init_var<P, ALG>(g, v, p, Lv, a.mode == MODE_CHANNEL);
            }
        }
        for (int e = r; e < C.E; e += Z) g.Rw(e, p) = 0.0f;
        for (int c = r; c < C.M; c += Z)
#pragma unroll
            for (int k = 0; k < Ly::SW; ++k) g.Sw(c, k, p) = 0.0f;
    }
    tm.sync();
}

// ---------------------------------------------------------------- the kernel
// SMEM: 0 the group state in the global workspace, 1 in shared memory, 2 in shared memory
// except R, which lives in the global workspace (split layout)
template <bool MULTI, int SMEM, int MAXT, int ALG, int P>
__global__ void __launch_bounds__(MAXT, 1) cbp_kernel(const __grid_constant__ KernelArgs a)
{
    using Ly = Lay<P, ALG>;
    extern __shared__ __align__(16) uint32_t smem[];
    const DevCode& C = a.code;
    const int Z = C.Z, mb = C.mb;

    // ---- stage the phi table and the schedule tables (a1).  The tables travel in the
    // kernel parameters; reading them in the hot loop straight from the constant bank
    // measured 20% slower on C2 than from shared memory (constant-cache misses).
    // (with both phi lookups on the texture pipe the table is not staged at all)
    constexpr int kTabWords = (CBP_TEX_B2V && CBP_TEX_C2B) ? 0 : 4 * kPhiSegs;
    float4* ptab = reinterpret_cast<float4*>(smem);
    for (int k = threadIdx.x; k < kTabWords / 4; k += blockDim.x) ptab[k] = C.phi_tab[k];
    int4* ent = reinterpret_cast<int4*>(smem + kTabWords);
    int32_t* row_ptr = reinterpret_cast<int32_t*>(smem + kTabWords + 8 * C.nent);
    int16_t* pshift = reinterpret_cast<int16_t*>(row_ptr + mb + 1);
    for (int k = threadIdx.x; k < 2 * C.nent; k += blockDim.x) ent[k] = a.ent[k];
    for (int k = threadIdx.x; k <= mb; k += blockDim.x) row_ptr[k] = a.row_ptr[k];
    for (int k = threadIdx.x; k < mb; k += blockDim.x) pshift[k] = a.pshift[k];
    Team<MULTI> tm;
    tm.nthreads = a.team_threads;
    tm.tidx = threadIdx.x / a.team_threads;
    tm.tl = threadIdx.x - tm.tidx * a.team_threads;
    if (MULTI) {
        tm.slot = 0;
        tm.r = tm.tl;
        tm.lane_base = 0;
        tm.slot_mask = kFull;
    } else {
        tm.slot = tm.tl / a.Zp;
        tm.r = tm.tl % a.Zp;
        tm.lane_base = tm.slot * a.Zp;
        tm.slot_mask = (a.Zp == 32) ? kFull : (((1u << a.Zp) - 1u) << tm.lane_base);
    }
    tm.lane_on = tm.r < Z && tm.slot < a.F;
    const int r = tm.r;
    const int r_off = ((2 * P * C.N + 3) & ~3) + P * Ly::SW * C.M;   // word offset of R inside a group
    const Lane lane{r, r * Ly::QS, r * Ly::RS, Z * Ly::QS, Z * Ly::RS,
                    SMEM == 2 ? 0 : 4 * r_off, 4 * a.slot_words, SMEM == 2 ? 4 * a.r_words : 4 * a.slot_words,
                    a.phi_m19, a.phi_one};
    // shared control words: only multi-warp teams exchange ballots / queue indices through them
    const int kCtl = a.ctl_words;
    uint32_t* ctl = smem + a.table_words + tm.tidx * kCtl;
    long long* ctl64 = reinterpret_cast<long long*>(ctl + 256);

    const int nteams = blockDim.x / a.team_threads;
    const int gidx = tm.tidx * a.F + (tm.slot < a.F ? tm.slot : 0);   // group index in the CTA
    float* sbase = SMEM ? reinterpret_cast<float*>(smem + a.table_words + nteams * kCtl)
                        : a.gstate + static_cast<size_t>(blockIdx.x) * nteams * a.F * a.slot_words;
    float* grp0 = sbase + static_cast<size_t>(gidx) * a.slot_words;
    // group layout (word offsets; slot_words % 4 == 0): QP [2PN] | pad to 4 | S [P SW M] | R [P E] | cw [P nwords];
    // split layout (SMEM 2): R [P E] in its own global slot of r_words, the rest in shared memory
    Grp<P, ALG> g;
    const int s_off = (2 * P * C.N + 3) & ~3;              // 16-byte aligned check records
    g.qp = reinterpret_cast<char*>(grp0);
    g.S = reinterpret_cast<char*>(grp0 + s_off);
    if constexpr (SMEM == 2) {
        g.R = reinterpret_cast<char*>(a.rstate + (static_cast<size_t>(blockIdx.x) * nteams * a.F + gidx) * a.r_words);
        g.rb = g.R;
        g.cw = reinterpret_cast<uint32_t*>(grp0 + r_off);
    } else {
        g.R = reinterpret_cast<char*>(grp0 + r_off);
        g.rb = g.qp;
        g.cw = reinterpret_cast<uint32_t*>(grp0 + r_off + P * C.E);
    }
    g.nwords = C.nwords;
    if (MULTI)   // neutral first / last words of the row reduction (both buffers, both frames, all 32 warp slots)
        for (int k = tm.tl; k < 256; k += a.team_threads) ctl[k] = ((k & 63) < 32) ? 0xffffu : 0u;
    __syncthreads();
    auto put_check = [&](int p, int c, float4 v) {
        g.Sw(c, 0, p) = v.x;
        if constexpr (ALG == 1) {
            g.Sw(c, 1, p) = v.y;
            g.Sw(c, 2, p) = v.z;
        }
    };

    const bool belief = a.stop_rule <= 1;
    const int W = (a.stop_rule == 1) ? C.N : C.M;            // R4 (N, M < 65536)
    const bool decoding = a.mode != MODE_CHANNEL;

    // per-frame control (uniform over the group's lanes)
    bool active[P], exhausted[P], conv[P];
    int64_t fidx[P];
    int ev_dc[P], ev_part[P], consec[P], sweep[P], fires[P];   // edge visits = ev_dc * Z + ev_part
#pragma unroll
    for (int p = 0; p < P; ++p) {
        active[p] = conv[p] = false;
        exhausted[p] = tm.slot >= a.F;
        fidx[p] = -1;
        ev_dc[p] = ev_part[p] = consec[p] = fires[p] = 0;
        sweep[p] = 1;
    }
    // per-lane counters (ber_sim)
    unsigned long long cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};

    // ---- syndrome of frame p's current hard bits, team-uniform call; valid where `want`.
    // Warp teams (Z <= 32, mb <= Zp): the hard bits of each column block are packed by one
    // ballot (group g's lanes in bits lane_base.., bit lane_base + t = variable jZ + t); lane i
    // of a group XORs its field of the rotated words of base row i's entries (bit r of
    // rot_s(field) = bit (r+s) mod Z = the variable of check iZ+r), and a vote over the group
    // says whether any check is unsatisfied -- nb ballots + ~dc words per lane instead of E
    // per-lane bit reads.  Multi-warp teams check their own checks lane by lane.
    auto syndrome_nz = [&](int p, bool want) -> bool {
        if (!MULTI && a.fast_syn) {
            for (int j = 0; j < C.nb; ++j) {
                const bool bit = want && tm.lane_on && (__float_as_uint(g.PH(j * Z + (tm.lane_on ? r : 0), p)) >> 31);
                const unsigned w = __ballot_sync(kFull, bit);
                if (tm.tl == 0) ctl[j] = w;
            }
            __syncwarp();
            const uint32_t zmask = (Z == 32) ? kFull : ((1u << Z) - 1u);
            uint32_t x = 0;
            if (want && tm.slot < a.F && r < mb)
                for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
                    const int j = ent[2 * k].x / (8 * P * Z);          // A.x = QS j Z
                    const int sft = ent[2 * k + 1].z >> 16;
                    const uint32_t w = (ctl[j] >> tm.lane_base) & zmask;
                    x ^= sft ? (((w >> sft) | (w << (Z - sft))) & zmask) : w;
                }
            const bool nz = (__ballot_sync(kFull, x != 0u) & tm.slot_mask) != 0u;
            __syncwarp();
            return nz;
        }
        return tm.slot_any(want && tm.lane_on && lane_syndrome<P, ALG>(ent, row_ptr, mb, r, Z, p, g));
    };

    // ---- Step 3: outputs of the frames with done[p] (a8); team-uniform call
    auto finish = [&](const bool (&done)[P]) {
        bool anyd = false;
#pragma unroll
        for (int p = 0; p < P; ++p) anyd |= done[p];
        if (!tm.team_any(anyd)) return;
        tm.sync();
#pragma unroll
        for (int p = 0; p < P; ++p) {
            bool synd_zero = conv[p];
            const bool need_syn = done[p] && !conv[p] && decoding;
            if (tm.team_any(need_syn)) {
                const bool nz = syndrome_nz(p, need_syn);
                if (need_syn) synd_zero = !nz;
            }
            const int iters = conv[p] ? sweep[p] : a.max_iter;
            const uint8_t flags = static_cast<uint8_t>((conv[p] ? 1 : 0) | (synd_zero ? 2 : 0) | (fires[p] > 0 ? 4 : 0));
            const int64_t evs = static_cast<int64_t>(ev_dc[p]) * Z + ev_part[p];
            if (a.mode == MODE_DECODE_F32 || a.mode == MODE_DECODE_I8) {
                if (done[p] && tm.lane_on) {
                    uint32_t* out = a.bits + static_cast<size_t>(fidx[p]) * a.ld_words;
                    for (int w = r; w < a.ld_words; w += Z) {
                        uint32_t word = 0;
                        if (w < C.nwords)
                            for (int b = 0; b < 32; ++b) {
                                const int v = 32 * w + b;
                                if (v < C.N) word |= (__float_as_uint(g.PH(v, p)) >> 31) << b;
                            }
                        out[w] = word;
                    }
                    if (a.omega) {
                        float* om = a.omega + static_cast<size_t>(fidx[p]) * C.M;
                        for (int c = r; c < C.M; c += Z) {
                            float Sv, m;
                            if constexpr (ALG >= 2) {
                                Sv = 0.0f;                               // LBP / FBP: no check-beliefs
                                m = 0.0f;
                            } else if constexpr (ALG == 1) {
                                Sv = g.Sw(c, 2, p);                      // sign bit = sign of Omega
                                m = g.Sw(c, 0, p);                       // Omega = sgn * min (reading R20)
                            } else {
                                Sv = g.Sw(c, 0, p);
                                m = phi_sel<CBP_TEX_B2V && CBP_TEX_C2B>(fabsf(Sv), ptab, lane, static_cast<TexH>(a.code.phi_tex));   // Omega = sgn phi(S)
                            }
                            om[c] = (__float_as_uint(Sv) >> 31) ? -m : m;
                        }
                    }
                    if (r == 0) {
                        a.iters[fidx[p]] = iters;
                        a.flags[fidx[p]] = flags;
                        if (a.ev) a.ev[fidx[p]] = evs;
                    }
                }
            } else if (a.mode == MODE_BER_SIM) {
                bool info_err = false, cw_err = false;
                if (done[p] && tm.lane_on) {
                    const uint32_t* cw = g.cwp(p);
                    for (int w = r; w < C.nwords; w += Z) {
                        uint32_t word = 0;
                        for (int b = 0; b < 32; ++b) {
                            const int v = 32 * w + b;
                            if (v < C.N) word |= (__float_as_uint(g.PH(v, p)) >> 31) << b;
                        }
                        const uint32_t d = word ^ cw[w];
                        uint32_t im = 0;
                        if (32 * w + 32 <= C.K) im = kFull;
                        else if (32 * w < C.K) im = (1u << (C.K - 32 * w)) - 1u;
                        cnt[1] += __popc(d & im);
                        info_err |= (d & im) != 0u;
                        cw_err |= d != 0u;
                    }
                }
                const bool fe = tm.slot_any(info_err);
                const bool ce = tm.slot_any(cw_err);
                if (done[p] && r == 0) {
                    cnt[0] += 1;
                    cnt[2] += fe;
                    cnt[3] += ce;
                    cnt[4] += iters;
                    cnt[5] += evs;
                    cnt[6] += conv[p] ? 0 : 1;
                    cnt[7] += fires[p];
                }
            } else {  // MODE_CHANNEL
                if (done[p] && tm.lane_on) {
                    if (a.llr_out) {
                        float* out = a.llr_out + static_cast<size_t>(fidx[p]) * a.ld;
                        for (int v = r; v < C.N; v += Z) out[v] = g.Q(v, p);
                    }
                    if (a.cw_out) {
                        uint32_t* out = a.cw_out + static_cast<size_t>(fidx[p]) * a.ld_words;
                        for (int w = r; w < a.ld_words; w += Z) out[w] = (w < C.nwords) ? g.cwp(p)[w] : 0u;
                    }
                }
            }
        }
#pragma unroll
        for (int p = 0; p < P; ++p)
            if (done[p]) active[p] = false;
        tm.sync();
    };

    for (;;) {
        // ---- refill free frame slots from the queue
        bool fresh[P], any_fresh = false;
        long long f[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const bool need = !active[p] && !exhausted[p];
            f[p] = -1;
            if (need && r == 0) f[p] = static_cast<long long>(atomicAdd(a.queue, 1ull));
        }
        if (MULTI) {
            if (tm.tl == 0)
#pragma unroll
                for (int p = 0; p < P; ++p) ctl64[p] = f[p];
            tm.sync();
#pragma unroll
            for (int p = 0; p < P; ++p) f[p] = ctl64[p];
            tm.sync();
        } else {
#pragma unroll
            for (int p = 0; p < P; ++p) f[p] = __shfl_sync(kFull, f[p], tm.lane_base);
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const bool need = !active[p] && !exhausted[p];
            fresh[p] = false;
            if (need) {
                if (f[p] < a.frames) {
                    active[p] = fresh[p] = true;
                    fidx[p] = f[p];
                    conv[p] = false;
                    ev_dc[p] = ev_part[p] = 0;
                    consec[p] = 0;
                    sweep[p] = 1;
                    fires[p] = 0;
                } else {
                    exhausted[p] = true;
                }
            }
            any_fresh |= fresh[p];
        }
        // ---- Step 1: initialisation (a4/a5)
        if (a.mode == MODE_BER_SIM || a.mode == MODE_CHANNEL) {
            if (tm.team_any(any_fresh)) channel_frames<MULTI, P, ALG>(a, tm, fresh, fidx, ent, row_ptr, pshift, g);
        } else {
#pragma unroll
            for (int p = 0; p < P; ++p) {
                if (!(fresh[p] && tm.lane_on)) continue;
                const size_t base = static_cast<size_t>(fidx[p]) * a.ld;
                // channel LLRs read once, 16 bytes per lane and load (rows are 16-byte aligned and
                // padded: ld * elem % 16 == 0, so the last vector stays inside the row); streaming
                // loads (evict-first), the frame's lanes cover one contiguous segment per step
                if (a.mode == MODE_DECODE_I8) {
                    const int4* src = reinterpret_cast<const int4*>(a.q + base);
                    for (int v16 = r; 16 * v16 < C.N; v16 += Z) {
                        const int4 w = __ldcs(src + v16);
                        const uint32_t ws[4] = {static_cast<uint32_t>(w.x), static_cast<uint32_t>(w.y),
                                                static_cast<uint32_t>(w.z), static_cast<uint32_t>(w.w)};
#pragma unroll
                        for (int t = 0; t < 16; ++t) {
                            const int v = 16 * v16 + t;
                            const int8_t qv = static_cast<int8_t>(ws[t >> 2] >> (8 * (t & 3)));
                            if (v < C.N) init_var<P, ALG>(g, v, p, __fmul_rn(static_cast<float>(qv), a.qscale));
                        }
                    }
                } else {
                    const float4* src = reinterpret_cast<const float4*>(a.llr + base);
                    for (int v4 = r; 4 * v4 < C.N; v4 += Z) {
                        const float4 x = __ldcs(src + v4);
                        const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                        for (int t = 0; t < 4; ++t)
                            if (4 * v4 + t < C.N) init_var<P, ALG>(g, 4 * v4 + t, p, xs[t]);
                    }
                }
                for (int e = r; e < C.E; e += Z) g.Rw(e, p) = 0.0f;   // equ_s4e17
                for (int c = r; c < C.M; c += Z)                      // equ_s4e16: Omega = inf <=> S = 0
#pragma unroll
                    for (int k = 0; k < Ly::SW; ++k) g.Sw(c, k, p) = 0.0f;
            }
            tm.sync();
        }
        bool any_active = false;
#pragma unroll
        for (int p = 0; p < P; ++p) any_active |= active[p];
        if (!tm.team_any(any_active)) break;

        if (decoding) {
            // ---- Step 2: one sweep over the base rows (checks in ascending order).  A frame
            // that converges mid-sweep is finished at once; its lanes then idle on garbage
            // state (never read again) while the other frame of the group continues.
            for (int i = 0; i < mb; ++i) {
                bool live = false;
#pragma unroll
                for (int p = 0; p < P; ++p) live |= active[p];
                if (!tm.team_any(live)) break;
                const int e0 = row_ptr[i], dc = row_ptr[i + 1] - e0;
                RowOut<P> ro;
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    ro.ok[p] = true;
                    ro.oldbits[p] = 0;
                    ro.Snew[p] = ro.Sold[p] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                }
                if (live && tm.lane_on) {
                    const int sidx = (i * Z + r) * Ly::RS;
                    if constexpr (ALG == 1) {
                        uint32_t s1[P];   // zero for a frame in sweep 1, else all ones (first-visit keep mask, R1)
#pragma unroll
                        for (int p = 0; p < P; ++p) s1[p] = (active[p] && sweep[p] == 1) ? 0u : kFull;
                        ro = process_row_ms<P>(ent, e0, dc, sidx, lane, g, s1, a.alpha);
                    } else if constexpr (ALG == 3) {
                        process_row_fbp<P>(ent, ptab, e0, dc, lane, static_cast<TexH>(a.code.phi_tex), g);
                    } else {
                        // the previous check record is kept only when the window can fill in this row
                        bool keep = false;
#pragma unroll
                        for (int p = 0; p < P; ++p) keep |= belief && active[p] && W - consec[p] - 1 < Z;
                        ro = process_row<P, ALG>(ent, ptab, e0, dc, sidx, lane, static_cast<TexH>(a.code.phi_tex), g,
                                                 keep);
                    }
                }
                // ---- Step 2(3): stopping criterion, counted per check update (R4, R5).  The
                // ballots double as the team's row barrier; without a belief rule a plain
                // barrier orders the rows.
                int first_bad[P], last_bad[P];   // first / last unclean check of the row
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    first_bad[p] = Z;
                    last_bad[p] = -1;
                }
                if (!belief) {
                    tm.sync();
                } else if (MULTI) {
                    // each warp publishes the first / last unclean check among its lanes; after the
                    // barrier every thread reduces the team's words (4 per 16-byte load; the words of
                    // warps beyond the team stay at their neutral values)
                    uint32_t* cb = ctl + (i & 1) * 128;
                    const int w = tm.tl >> 5;
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const unsigned m = __ballot_sync(kFull, tm.lane_on && !ro.ok[p]);
                        if ((tm.tl & 31) == 0) {
                            cb[64 * p + w] = m ? 32 * w + __ffs(m) - 1 : 0xffffu;
                            cb[64 * p + 32 + w] = m ? 32 * w + 32 - __clz(m) : 0u;      // last + 1
                        }
                    }
                    tm.sync();
                    const int nw4 = (tm.nthreads + 127) >> 7;
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        uint32_t f = 0xffffu, l = 0u;
                        for (int w4 = 0; w4 < nw4; ++w4) {
                            const uint4 F = *reinterpret_cast<const uint4*>(cb + 64 * p + 4 * w4);
                            const uint4 Lw = *reinterpret_cast<const uint4*>(cb + 64 * p + 32 + 4 * w4);
                            f = min(min(f, F.x), min(F.y, min(F.z, F.w)));
                            l = max(max(l, Lw.x), max(Lw.y, max(Lw.z, Lw.w)));
                        }
                        first_bad[p] = static_cast<int>(min(f, static_cast<uint32_t>(Z)));
                        last_bad[p] = static_cast<int>(l) - 1;
                    }
                } else {
                    __syncwarp();
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const unsigned m = (__ballot_sync(kFull, tm.lane_on && !ro.ok[p]) & tm.slot_mask) >> tm.lane_base;
                        if (m) {
                            first_bad[p] = __ffs(m) - 1;
                            last_bad[p] = 31 - __clz(m);
                        }
                    }
                }
                bool fire[P], any_fire = false;
                int rstar[P];
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    fire[p] = false;
                    rstar[p] = 0;
                    if (active[p] && belief) {
                        rstar[p] = W - consec[p] - 1;   // the window fills at check i*Z + rstar
                        fire[p] = rstar[p] < Z && first_bad[p] > rstar[p];
                        if (!fire[p]) consec[p] = (last_bad[p] < 0) ? consec[p] + Z : (Z - 1 - last_bad[p]);
                    }
                    if (active[p] && !fire[p]) ev_dc[p] += dc;
                    any_fire |= fire[p];
                }
                if (tm.team_any(any_fire)) {
                    // the sequential decoder stops right after check i*Z + rstar: lanes r > rstar
                    // show their pre-row hard bits and S while the syndrome is verified (R5)
                    bool back[P], conv_now[P];
                    uint32_t newbits[P];
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        back[p] = fire[p] && tm.lane_on && r > rstar[p];
                        newbits[p] = 0;
                        if (back[p]) {
                            newbits[p] = swap_row_bits<P, ALG>(ent, e0, dc, r, Z, p, ro.oldbits[p], g);
                            put_check(p, i * Z + r, ro.Sold[p]);
                        }
                    }
                    tm.sync();
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const bool nz = syndrome_nz(p, fire[p]);
                        conv_now[p] = false;
                        if (fire[p]) {
                            if (!nz) {
                                conv[p] = conv_now[p] = true;   // converged: output = state after check i*Z + rstar
                                ev_part[p] += dc * (rstar[p] + 1);
                            } else {
                                fires[p] += 1;                  // undetected fire: resume (R5)
                                ev_dc[p] += dc;
                                consec[p] = Z - 1 - max(last_bad[p], rstar[p]);
                                if (back[p]) {
                                    swap_row_bits<P, ALG>(ent, e0, dc, r, Z, p, newbits[p], g);
                                    put_check(p, i * Z + r, ro.Snew[p]);
                                }
                            }
                        }
                    }
                    tm.sync();
                    finish(conv_now);
                }
            }
            // ---- end of sweep
            if constexpr (ALG == 3) {
                // flooding BP variable pass (equ_s2e6): the accumulated posterior becomes
                // Lambda_old (sign = hard bit, equ_s2e7); the accumulator restarts at L_v
                tm.sync();
#pragma unroll
                for (int p = 0; p < P; ++p)
                    if (active[p] && tm.lane_on)
                        for (int v = r; v < C.N; v += Z) {
                            g.PH(v, p) = g.Q(v, p);
                            g.Q(v, p) = g.Lv(v, p);
                        }
                tm.sync();
            }
            bool done[P];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const bool want_syn = active[p] && a.stop_rule == 2;
                if (tm.team_any(want_syn)) {
                    tm.sync();
                    const bool nz = syndrome_nz(p, want_syn);
                    if (want_syn && !nz) conv[p] = true;
                }
                done[p] = active[p] && (conv[p] || sweep[p] >= a.max_iter);
            }
            finish(done);
#pragma unroll
            for (int p = 0; p < P; ++p)
                if (active[p]) sweep[p] += 1;
        } else {
            bool done[P];
#pragma unroll
            for (int p = 0; p < P; ++p) done[p] = active[p];
            finish(done);
        }
    }

    if (a.mode == MODE_BER_SIM) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            unsigned long long x = cnt[k];
            for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(kFull, x, o);
            if ((threadIdx.x & 31) == 0 && x) atomicAdd(a.counts + k, x);
        }
    }
}

// ---------------------------------------------------------------- host-side launch of one algorithm
// Instantiations: P = 1 for every geometry (state in smem or global, warp or multi-warp
// teams up to 1024 threads); P = 2 only with state in smem and at most 256 threads, and
// only for the CBP rules (ALG 0, 1).
template <bool MULTI, int SMEM, int MAXT, int ALG, int P>
static int launch_t(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st)
{
    auto k = cbp_kernel<MULTI, SMEM, MAXT, ALG, P>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
    k<<<grid, g.threads, g.smem_bytes, st>>>(a);
    return static_cast<int>(cudaGetLastError());
}

template <bool MULTI, int SMEM, int MAXT, int ALG, int P>
static int occ_t(const Geometry& g, int* out)
{
    auto k = cbp_kernel<MULTI, SMEM, MAXT, ALG, P>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
    return static_cast<int>(cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, g.threads, g.smem_bytes));
}

template <int ALG, template <bool, int, int, int, int> class Fn, typename... Args>
static int dispatch_alg(const Geometry& g, Args... args)
{
    if (g.P == 2) {
        if constexpr (ALG <= 1) {
            if (!g.state_in_smem || g.threads > 256 || g.r_global) return static_cast<int>(cudaErrorInvalidConfiguration);
            return g.multi ? Fn<true, 1, 256, ALG, 2>::run(g, args...) : Fn<false, 1, 256, ALG, 2>::run(g, args...);
        } else {
            return static_cast<int>(cudaErrorInvalidConfiguration);
        }
    }
    const int sm = g.state_in_smem ? (g.r_global ? 2 : 1) : 0;
    if (!g.multi)
        return sm == 2 ? Fn<false, 2, CBP_WARP_MAXT, ALG, 1>::run(g, args...)
             : sm == 1 ? Fn<false, 1, CBP_WARP_MAXT, ALG, 1>::run(g, args...)
                       : Fn<false, 0, CBP_WARP_MAXT, ALG, 1>::run(g, args...);
    if (g.threads <= 512)
        return sm == 2 ? Fn<true, 2, 512, ALG, 1>::run(g, args...)
             : sm == 1 ? Fn<true, 1, 512, ALG, 1>::run(g, args...) : Fn<true, 0, 512, ALG, 1>::run(g, args...);
    if (g.threads <= 768 && sm == 2) return Fn<true, 2, 768, ALG, 1>::run(g, args...);   // split layout
    if (g.threads <= 768 && sm == 0) return Fn<true, 0, 768, ALG, 1>::run(g, args...);   // 2 C4 teams, 85 registers
    return sm == 2 ? Fn<true, 2, 1024, ALG, 1>::run(g, args...)
         : sm == 1 ? Fn<true, 1, 1024, ALG, 1>::run(g, args...) : Fn<true, 0, 1024, ALG, 1>::run(g, args...);
}

template <bool MULTI, int SMEM, int MAXT, int ALG, int P>
struct LaunchFn {
    static int run(const Geometry& g, const KernelArgs* a, int grid, cudaStream_t st)
    {
        return launch_t<MULTI, SMEM, MAXT, ALG, P>(*a, g, grid, st);
    }
};

template <bool MULTI, int SMEM, int MAXT, int ALG, int P>
struct OccFn {
    static int run(const Geometry& g, int* out) { return occ_t<MULTI, SMEM, MAXT, ALG, P>(g, out); }
};

// defined in cbp_kernels_alg<k>.cu
#define CBP_DECLARE_ALG(k)                                                              \
    int launch_alg##k(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st); \
    int occupancy_alg##k(const Geometry& g, int* out);
CBP_DECLARE_ALG(0)
CBP_DECLARE_ALG(1)
CBP_DECLARE_ALG(2)
CBP_DECLARE_ALG(3)
#undef CBP_DECLARE_ALG

}  // namespace cbp
