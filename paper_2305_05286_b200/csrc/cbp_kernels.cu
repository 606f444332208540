// cbp_kernels.cu -- sm_100a kernels of check-belief propagation decoding.
//
// One persistent kernel serves cbp_decode, cbp_decode_i8, cbp_channel and
// cbp_ber_sim.  A CTA holds several independent teams; a team
// owns F frame slots of Zp lanes, and lane r of a slot processes lifted check
// i*Z + r of the current base row i.  The Z lifted checks of one base row touch
// disjoint variables (each block is a permutation), so processing them in
// parallel is bit-identical to the paper's sequential check order (reading
// R12).  Per-frame state lives in shared memory:
//   QP[N] float2 (Q_v, Phi_v | hard bit in the sign), R[E], S[M] (sign = Omega<0)
// The phi table (contract v2) and the code's schedule tables are staged once per CTA.
//
// Paper steps (§IV-C): init = Step 1 (l.402-422, equ_s4e15-17);
// process_row = Step 2(1) B2V/V2C/C2B (equ_s4e18-22) and 2(2) (equ_s4e23);
// stop logic = Step 2(3) (l.478-485) with readings R4/R5; finish = Step 3 (l.487).
#include <cuda_runtime.h>

#include <algorithm>

#include "cbp_internal.h"
#include "contract.cuh"

namespace cbp {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kSign = 0x80000000u;

// independent edges of a check processed together (ILP); remainder one at a time
#ifndef CBP_CHUNK
#define CBP_CHUNK 3
#endif

// Per-slot state.  Byte-addressed bases plus typed views for the cold paths.
struct SlotPtrs {
    char* qp;       // float2 [N]: (Q_{v->c*}, Phi_v = phi(|Q_v|) with sign bit = hard decision x_v)
    char* R;        // float [E]: C2V message of edge (check i*Z+r, entry b) at byte 4*(b*Z + r)
    char* S;        // float [M]: phi-domain check-belief sum S_c, sign bit = (Omega_c < 0)
    uint32_t* cw;   // [nwords] transmitted codeword (ber_sim) / scratch
    __device__ __forceinline__ float2* QP() const { return reinterpret_cast<float2*>(qp); }
    __device__ __forceinline__ float* Rf() const { return reinterpret_cast<float*>(R); }
    __device__ __forceinline__ float* Sf() const { return reinterpret_cast<float*>(S); }
};

__device__ __forceinline__ float2 ld2(const char* b, int off) { return *reinterpret_cast<const float2*>(b + off); }
__device__ __forceinline__ float ld1(const char* b, int off) { return *reinterpret_cast<const float*>(b + off); }
__device__ __forceinline__ void st2(char* b, int off, float2 v) { *reinterpret_cast<float2*>(b + off) = v; }
__device__ __forceinline__ void st1(char* b, int off, float v) { *reinterpret_cast<float*>(b + off) = v; }

// Schedule table entry b (two int4, built in cbp_api.cpp):
//   A = {8 j Z, 4 row(prev(b)) Z, 4 b Z, 4 prev(b) Z}    byte bases: variable block (QP),
//        S block of the previous check of the same variables, own R block, R block of prev(b)
//   B = {8 s, 4 ds, first, j Z}   ds = (s - s_prev) mod Z; first: no latest check in sweep 1 (R1)
// prev(b) = previous nonzero row of b's column, cyclically (the static "latest check" of
// every variable of the block after sweep 1); prev(b) == b for a degree-1
// column (R3).  Variable of lane r: j Z + (r + s) mod Z; its previous check's row (r + ds) mod Z.

__device__ __forceinline__ int lane_var(const int4* ent, int e, int r, int Z)
{
    const int4 B = ent[2 * e + 1];
    int t = r + (B.x >> 3);
    t = (t >= Z) ? t - Z : t;
    return B.w + t;
}

// ---------------------------------------------------------------- team helpers
// !MULTI: a team is one warp holding F frame slots of Zp lanes; MULTI: a team is
// TW warps holding one frame.  Teams synchronise with their own named barrier.
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
    unsigned slot_mask;   // lanes of this slot within the warp (!MULTI)

    __device__ __forceinline__ void sync() const
    {
        if (MULTI) named_bar_sync(1 + tidx, nthreads);
        else __syncwarp();
    }
    // OR of a slot-uniform predicate over the team's slots.  A MULTI team holds one
    // frame and every thread derives the control state identically, so the predicate
    // is already team-uniform (no barrier); a warp team votes over its F slots.
    __device__ __forceinline__ bool team_any(bool pred) const
    {
        if (MULTI) return pred;
        return __any_sync(kFull, pred) != 0;
    }
    // OR over the lanes of this slot (a synchronisation point)
    __device__ __forceinline__ bool slot_any(bool pred) const
    {
        if (MULTI) return named_bar_or(1 + tidx, nthreads, pred);
        return (__ballot_sync(kFull, pred) & slot_mask) != 0u;
    }
};

// ---------------------------------------------------------------- per-row edge chain
struct Lane {
    int r, r4, r8, Z, Z4, Z8;
    int qp_bytes, R_bytes, S_bytes;   // slot array sizes (bounds checks of debug builds)
    uint32_t m19, one;                // phi local-variable masks as runtime operands (one LOP3)
};

struct RowAcc {
    float Ssum;
    uint32_t negw;     // bit 31: XOR of the signs of Q^new over the check (sign of Omega)
    uint32_t flipw;    // bit 31: some posterior sign flipped (equ_s4e24)
    uint32_t oldbits;  // previous hard bits of the check's variables (rollback of a mid-row stop)
};

// U consecutive edges of lane r's check.  Loads first, then U independent B2V
// phi chains, commits / V2C, U independent C2B phi chains and the ordered S
// accumulation (reading R12).  SWEEP1 handles first visits (reading R1); TRACK
// records the previous hard bits (only rows where the belief window can fire).
// R_{ci->v} is read after the commit of R_{cj->v}: for a degree-1 column both are
// the same slot, which realises "commit before read" (R3) through memory order.
template <int U, bool SWEEP1, bool TRACK>
__device__ __forceinline__ void edge_chunk(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0, int k0,
                                           const Lane& L, const SlotPtrs& s, RowAcc& acc)
{
    int aqp[U], aw[U], ar[U];
    float q[U], p[U], scj[U], Rn[U];
    bool fst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int4 A = ent[2 * (e0 + k0 + u)];
        const int4 B = ent[2 * (e0 + k0 + u) + 1];
        int t8 = L.r8 + B.x;
        t8 = (t8 >= L.Z8) ? t8 - L.Z8 : t8;
        int rp4 = L.r4 + B.y;
        rp4 = (rp4 >= L.Z4) ? rp4 - L.Z4 : rp4;
        CBP_CHECK(t8 >= 0 && t8 < L.Z8 && rp4 >= 0 && rp4 < L.Z4);
        CBP_CHECK(A.x + t8 + 8 <= L.qp_bytes && A.y + rp4 + 4 <= L.S_bytes && A.z + L.r4 + 4 <= L.R_bytes &&
                  A.w + rp4 + 4 <= L.R_bytes);
        aqp[u] = A.x + t8;
        aw[u] = A.w + rp4;
        ar[u] = A.z + L.r4;
        fst[u] = SWEEP1 && (B.z & 1) != 0;
        const float2 qp = ld2(s.qp, aqp[u]);
        q[u] = qp.x;
        p[u] = qp.y;
        scj[u] = ld1(s.S, A.y + rp4);
    }
    // B2V (equ_s4e18): R^new_{cj->v} = sgn(Omega_cj) sgn(Q) phi(|phi(|Omega_cj|) - phi(|Q|)|), phi(|Omega|) = S (R11)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const float mag = phi32(fabsf(__fsub_rn(fabsf(scj[u]), fabsf(p[u]))), ptab, L.m19, L.one);
        const uint32_t sg = (__float_as_uint(scj[u]) ^ __float_as_uint(q[u])) & kSign;
        Rn[u] = __uint_as_float(__float_as_uint(mag) | sg);
        if (SWEEP1 && fst[u]) Rn[u] = 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (!(SWEEP1 && fst[u])) st1(s.R, aw[u], Rn[u]);   // equ_s4e22 commit of R_{cj->v} (R2), before the read (R3)
    float qn[U];
    uint32_t lb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const float ro = ld1(s.R, ar[u]);                    // R_{ci->v}
        const float lam = __fadd_rn(q[u], Rn[u]);            // equ_s4e20 (Lambda is never -0)
        qn[u] = __fsub_rn(lam, ro);                          // equ_s4e19 (R15)
        lb[u] = __float_as_uint(lam) & kSign;                // hard decision, equ_s2e7
        acc.flipw |= __float_as_uint(lam) ^ __float_as_uint(p[u]);   // equ_s4e24 (R7), bit 31
        if (TRACK) acc.oldbits |= (__float_as_uint(p[u]) >> 31) << (k0 + u);
    }
    float ph[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ph[u] = phi32(fabsf(qn[u]), ptab, L.m19, L.one);   // C2B (equ_s4e21, App. equ_ae4)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        acc.Ssum = __fadd_rn(acc.Ssum, ph[u]);
        acc.negw ^= __float_as_uint(qn[u]);                  // Q^new is never -0
        st2(s.qp, aqp[u], make_float2(qn[u], __uint_as_float(__float_as_uint(ph[u]) | lb[u])));
    }
}

// check record of the row (log-tanh: S in .x; min-sum: the 16-byte record) before / after
struct RowOut {
    float4 Snew, Sold;
    uint32_t oldbits;
    bool ok;
};

template <bool SWEEP1, bool TRACK>
__device__ __forceinline__ RowOut process_row(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0,
                                              int dc, int sidx4, const Lane& L, const SlotPtrs& s)
{
    RowAcc acc{0.0f, 0u, 0u, 0u};
    const float Sold = ld1(s.S, sidx4);
    int k0 = 0;
    for (; k0 + CBP_CHUNK <= dc; k0 += CBP_CHUNK) edge_chunk<CBP_CHUNK, SWEEP1, TRACK>(ent, ptab, e0, k0, L, s, acc);
    for (; k0 < dc; ++k0) edge_chunk<1, SWEEP1, TRACK>(ent, ptab, e0, k0, L, s, acc);
    const float Snew = __uint_as_float(__float_as_uint(acc.Ssum) | (acc.negw & kSign));
    st1(s.S, sidx4, Snew);                                   // equ_s4e23
    RowOut o;
    o.Snew.x = Snew;
    o.Sold.x = Sold;
    o.oldbits = acc.oldbits;
    o.ok = ((acc.negw | acc.flipw) & kSign) == 0u;           // equ_s4e2 and equ_s4e24 for this check
    return o;
}

// ---------------------------------------------------------------- normalized min-sum CBP
// PAPER.md l.577-603 (equ_s4e18xx, equ_s4e21xx) with reading R20: per check a 16-byte
// record {min, submin, owner | sign << 31, -} of m = fl(alpha |Q^new|); B2V magnitude =
// submin if v owns the minimum (owner = v's edge index in the check) else min; signs as
// psi- (equ_s4e13).  Schedule, V2C, commit and stop rule are those of the log-tanh path.
struct MsAcc {
    float m1, m2;
    uint32_t own, negw, flipw, oldbits;
};

__device__ __forceinline__ float4 ld4(const char* b, int off) { return *reinterpret_cast<const float4*>(b + off); }
__device__ __forceinline__ void st4(char* b, int off, float4 v) { *reinterpret_cast<float4*>(b + off) = v; }

template <int U, bool SWEEP1, bool TRACK>
__device__ __forceinline__ void edge_chunk_ms(const int4* __restrict__ ent, int e0, int k0, const Lane& L,
                                              const SlotPtrs& s, float alpha, MsAcc& acc)
{
    int aqp[U], aw[U], ar[U], kp[U];
    float q[U], p[U], Rn[U];
    float4 cs[U];
    bool fst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int4 A = ent[2 * (e0 + k0 + u)];
        const int4 B = ent[2 * (e0 + k0 + u) + 1];
        int t8 = L.r8 + B.x;
        t8 = (t8 >= L.Z8) ? t8 - L.Z8 : t8;
        int rp4 = L.r4 + B.y;
        rp4 = (rp4 >= L.Z4) ? rp4 - L.Z4 : rp4;
        CBP_CHECK(4 * (A.y + rp4) + 16 <= 4 * L.S_bytes);
        aqp[u] = A.x + t8;
        aw[u] = A.w + rp4;
        ar[u] = A.z + L.r4;
        fst[u] = SWEEP1 && (B.z & 1) != 0;
        kp[u] = B.z >> 8;
        const float2 qp = ld2(s.qp, aqp[u]);
        q[u] = qp.x;
        p[u] = qp.y;
        cs[u] = ld4(s.S, 4 * (A.y + rp4));                   // record of the previous check c_j
    }
    // B2V (equ_s4e18xx)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint32_t ow = __float_as_uint(cs[u].z);
        const float mag = (static_cast<int>(ow & 0xffu) == kp[u]) ? cs[u].y : cs[u].x;
        Rn[u] = __uint_as_float(__float_as_uint(mag) | ((ow ^ __float_as_uint(q[u])) & kSign));
        if (SWEEP1 && fst[u]) Rn[u] = 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (!(SWEEP1 && fst[u])) st1(s.R, aw[u], Rn[u]);   // commit of R_{cj->v} (R2, R3)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const float ro = ld1(s.R, ar[u]);
        const float lam = __fadd_rn(q[u], Rn[u]);            // equ_s4e20
        const float qn = __fsub_rn(lam, ro);                 // equ_s4e19
        const uint32_t lb = __float_as_uint(lam) & kSign;
        acc.flipw |= __float_as_uint(lam) ^ __float_as_uint(p[u]);
        if (TRACK) acc.oldbits |= (__float_as_uint(p[u]) >> 31) << (k0 + u);
        // C2B (equ_s4e21xx), in ascending edge order
        const float m = __fmul_rn(alpha, fabsf(qn));
        if (m < acc.m1) {
            acc.m2 = acc.m1;
            acc.m1 = m;
            acc.own = static_cast<uint32_t>(k0 + u);
        } else if (m < acc.m2) {
            acc.m2 = m;
        }
        acc.negw ^= __float_as_uint(qn);
        st2(s.qp, aqp[u], make_float2(qn, __uint_as_float(lb)));
    }
}

template <bool SWEEP1, bool TRACK>
__device__ __forceinline__ RowOut process_row_ms(const int4* __restrict__ ent, int e0, int dc, int sidx4, const Lane& L,
                                                 const SlotPtrs& s, float alpha)
{
    const float inf = __uint_as_float(0x7f800000u);
    MsAcc acc{inf, inf, 0u, 0u, 0u, 0u};                    // Omega^(-1) = (inf, inf)
    const float4 Sold = ld4(s.S, 4 * sidx4);
    int k0 = 0;
    for (; k0 + CBP_CHUNK <= dc; k0 += CBP_CHUNK) edge_chunk_ms<CBP_CHUNK, SWEEP1, TRACK>(ent, e0, k0, L, s, alpha, acc);
    for (; k0 < dc; ++k0) edge_chunk_ms<1, SWEEP1, TRACK>(ent, e0, k0, L, s, alpha, acc);
    const float4 Snew = make_float4(acc.m1, acc.m2, __uint_as_float(acc.own | (acc.negw & kSign)), 0.0f);
    st4(s.S, 4 * sidx4, Snew);
    RowOut o;
    o.Snew = Snew;
    o.Sold = Sold;
    o.oldbits = acc.oldbits;
    o.ok = ((acc.negw | acc.flipw) & kSign) == 0u;
    return o;
}

// write hard bits (sign of Phi) of lane r's variables in row (e0, dc); returns the previous ones
__device__ __forceinline__ uint32_t swap_row_bits(const int4* __restrict__ ent, int e0, int dc, int r, int Z,
                                                  uint32_t bits, const SlotPtrs& s)
{
    uint32_t prev = 0;
    for (int k = 0; k < dc; ++k) {
        const int v = lane_var(ent, e0 + k, r, Z);
        const uint32_t w = __float_as_uint(s.QP()[v].y);
        prev |= (w >> 31) << k;
        s.QP()[v].y = __uint_as_float((w & ~kSign) | (((bits >> k) & 1u) << 31));
    }
    return prev;
}

// parity of lane r's checks over all rows, from the hard bits (sign of Phi)
__device__ __forceinline__ bool lane_syndrome(const int4* __restrict__ ent, const int32_t* row_ptr, int mb, int r,
                                              int Z, const SlotPtrs& s)
{
    uint32_t nz = 0;
    for (int i = 0; i < mb; ++i) {
        uint32_t par = 0;
        for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
            par ^= __float_as_uint(s.QP()[lane_var(ent, k, r, Z)].y) >> 31;
        nz |= par;
    }
    return nz != 0u;
}

// lambda_i[r] = XOR of the info bits of lifted check i*Z + r (encoder)
__device__ __forceinline__ uint32_t info_parity(const int4* __restrict__ ent, const int32_t* row_ptr, int i, int r,
                                                int Z, int K, const uint32_t* cw)
{
    uint32_t par = 0;
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        if (ent[2 * k + 1].w >= K) continue;
        const int v = lane_var(ent, k, r, Z);
        par ^= (cw[v >> 5] >> (v & 31)) & 1u;
    }
    return par;
}

// ---------------------------------------------------------------- channel (a2-a4)
template <bool MULTI>
__device__ void channel_frame(const KernelArgs& a, const Team<MULTI>& tm, bool fresh, int64_t gframe,
                              const int4* ent, const int32_t* row_ptr, const int16_t* pshift, const SlotPtrs& s,
                              int s_words)
{
    const DevCode& C = a.code;
    const int Z = C.Z, r = tm.r;
    const bool on = fresh && tm.lane_on;
    float2* QP = s.QP();
    const uint32_t flo = static_cast<uint32_t>(gframe), fhi = static_cast<uint32_t>(static_cast<uint64_t>(gframe) >> 32);
    const uint32_t k0 = static_cast<uint32_t>(a.seed), k1 = static_cast<uint32_t>(a.seed >> 32);
    // (a2) info words: word w = Philox(w/4, f_lo, f_hi, 0)[w%4]
    if (on) {
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
                    s.cw[w] = word;
                }
            }
        }
    }
    tm.sync();
    // (a3) systematic part and p0 = XOR of the core rows' lambda (QP.x holds the symbol 1 - 2c)
    if (on) {
        for (int v = r; v < C.K; v += Z) QP[v].x = ((s.cw[v >> 5] >> (v & 31)) & 1u) ? -1.0f : 1.0f;
        uint32_t p0 = 0;
        for (int i = 0; i < C.core; ++i) {
            const uint32_t lam = info_parity(ent, row_ptr, i, r, Z, C.K, s.cw);
            s.Sf()[i * Z + r] = __uint_as_float(lam);      // lambda_i[r] kept for the next pass (S is free here)
            p0 ^= lam;
        }
        QP[C.kb * Z + r].x = p0 ? -1.0f : 1.0f;
    }
    tm.sync();
    // p_t = lambda_{t-1} ^ p_{t-1} ^ P^{s0} p0 (row t-1), extension p = lambda
    if (on) {
        uint32_t pprev = 0;
        for (int t = 1; t < C.core; ++t) {
            uint32_t pt = __float_as_uint(s.Sf()[(t - 1) * Z + r]);   // lambda_{t-1}[r]
            if (t >= 2) pt ^= pprev;
            const int s0 = pshift[t - 1];
            if (s0 >= 0) {
                int rr = r + s0;
                rr = (rr >= Z) ? rr - Z : rr;
                pt ^= QP[C.kb * Z + rr].x < 0.0f ? 1u : 0u;
            }
            QP[(C.kb + t) * Z + r].x = pt ? -1.0f : 1.0f;
            pprev = pt;
        }
        for (int k = 0; k < C.mb - C.core; ++k) {
            const uint32_t pe = info_parity(ent, row_ptr, C.core + k, r, Z, C.K, s.cw);
            QP[(C.kb + C.core + k) * Z + r].x = pe ? -1.0f : 1.0f;
        }
    }
    tm.sync();
    // transmitted codeword words
    if (on) {
        for (int w = r; w < C.nwords; w += Z) {
            uint32_t word = 0;
            for (int b = 0; b < 32; ++b) {
                const int v = 32 * w + b;
                if (v < C.N && QP[v].x < 0.0f) word |= 1u << b;
            }
            s.cw[w] = word;
        }
    }
    tm.sync();
    // (a4) BPSK + AWGN + LLR: y = (1-2c) + sigma n, L = (2/sigma^2) y  (equ_s4e15, R17)
    if (on) {
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
                const float y = __fadd_rn(QP[v].x, __fmul_rn(a.sigma, n[m]));
                float Lv = __fmul_rn(a.scale, y);
                if (a.llr_mode == 1) {
                    float qq = rintf(__fmul_rn(Lv, 4.0f));
                    qq = fminf(fmaxf(qq, -127.0f), 127.0f);
                    Lv = __fmul_rn(qq, 0.25f);
                }
                QP[v] = make_float2(Lv, Lv < 0.0f ? -0.0f : 0.0f);
            }
        }
        for (int e = r; e < C.E; e += Z) s.Rf()[e] = 0.0f;
        for (int c = r; c < s_words; c += Z) s.Sf()[c] = 0.0f;
    }
    tm.sync();
}

// ---------------------------------------------------------------- the kernel
template <bool MULTI, bool SMEM, int MAXT, int ALG>
__global__ void __launch_bounds__(MAXT, 1) cbp_kernel(const KernelArgs a)
{
    extern __shared__ __align__(16) uint32_t smem[];
    const DevCode& C = a.code;
    const int Z = C.Z, mb = C.mb;

    // ---- stage the phi table and the schedule tables (a1)
    float4* ptab = reinterpret_cast<float4*>(smem);
    int4* ent = reinterpret_cast<int4*>(smem + 4 * kPhiSegs);
    int32_t* row_ptr = reinterpret_cast<int32_t*>(smem + 4 * kPhiSegs + 8 * C.nent);
    int16_t* pshift = reinterpret_cast<int16_t*>(row_ptr + mb + 1);
    for (int k = threadIdx.x; k < kPhiSegs; k += blockDim.x) ptab[k] = C.phi_tab[k];
    for (int k = threadIdx.x; k < 2 * C.nent; k += blockDim.x) ent[k] = C.ent[k];
    for (int k = threadIdx.x; k <= mb; k += blockDim.x) row_ptr[k] = C.row_ptr[k];
    for (int k = threadIdx.x; k < mb; k += blockDim.x) pshift[k] = C.pshift[k];
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
    const int s_words = ALG ? 4 * C.M : C.M;               // words of the per-check records
    const Lane lane{r, 4 * r, 8 * r, Z, 4 * Z, 8 * Z, 8 * C.N, 4 * C.E, 4 * s_words, a.phi_m19, a.phi_one};
    uint32_t* ctl = smem + a.table_words + tm.tidx * kCtlTeamWords;
    long long* ctl64 = reinterpret_cast<long long*>(ctl + 64);

    const int nteams = blockDim.x / a.team_threads;
    float* sbase = SMEM ? reinterpret_cast<float*>(smem + a.table_words + nteams * kCtlTeamWords)
                        : a.gstate + static_cast<size_t>(blockIdx.x) * nteams * a.F * a.slot_words;
    SlotPtrs s;
    float* slot0 = sbase + static_cast<size_t>(tm.tidx * a.F + (tm.slot < a.F ? tm.slot : 0)) * a.slot_words;
    // slot layout (word offsets; slot_words % 4 == 0): QP [2N] | pad to 4 | S [s_words] | R [E] | cw
    const int s_off = (2 * C.N + 3) & ~3;                  // 16-byte aligned check records
    s.qp = reinterpret_cast<char*>(slot0);
    s.S = reinterpret_cast<char*>(slot0 + s_off);
    s.R = reinterpret_cast<char*>(slot0 + s_off + s_words);
    s.cw = reinterpret_cast<uint32_t*>(slot0 + s_off + s_words + C.E);
    __syncthreads();
    auto put_check = [&](const SlotPtrs& sp, int c, float4 v) {
        if constexpr (ALG == 1) st4(sp.S, 16 * c, v);
        else st1(sp.S, 4 * c, v.x);
    };

    const bool belief = a.stop_rule <= 1;
    const int W = (a.stop_rule == 1) ? C.N : C.M;            // R4 (N, M < 65536)
    const bool decoding = a.mode != MODE_CHANNEL;

    // per-slot control (uniform over the slot's lanes)
    bool active = false, exhausted = (tm.slot >= a.F), conv = false;
    int64_t fidx = -1;
    int ev_dc = 0, ev_part = 0, consec = 0;   // edge visits = ev_dc * Z + ev_part
    int sweep = 1, fires = 0;
    // per-lane counters (ber_sim)
    unsigned long long cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};

    for (;;) {
        // ---- refill free slots from the frame queue
        const bool need = !active && !exhausted;
        long long f = -1;
        if (need && r == 0) f = static_cast<long long>(atomicAdd(a.queue, 1ull));
        if (MULTI) {
            if (tm.tl == 0) ctl64[0] = f;
            tm.sync();
            f = ctl64[0];
            tm.sync();
        } else {
            f = __shfl_sync(kFull, f, tm.lane_base);
        }
        bool fresh = false;
        if (need) {
            if (f < a.frames) {
                active = fresh = true;
                fidx = f;
                conv = false;
                ev_dc = ev_part = 0;
                consec = 0;
                sweep = 1;
                fires = 0;
            } else {
                exhausted = true;
            }
        }
        // ---- Step 1: initialisation (a4/a5)
        if (a.mode == MODE_BER_SIM || a.mode == MODE_CHANNEL) {
            if (tm.team_any(fresh))
                channel_frame<MULTI>(a, tm, fresh, a.frame_begin + fidx, ent, row_ptr, pshift, s, s_words);
        } else {
            if (fresh && tm.lane_on) {
                const size_t base = static_cast<size_t>(fidx) * a.ld;
                for (int v = r; v < C.N; v += Z) {
                    const float Lv = (a.mode == MODE_DECODE_I8) ? __fmul_rn(static_cast<float>(a.q[base + v]), a.qscale)
                                                                : a.llr[base + v];
                    s.QP()[v] = make_float2(Lv, Lv < 0.0f ? -0.0f : 0.0f);   // equ_s4e15, hard bit from L (R7)
                }
                for (int e = r; e < C.E; e += Z) s.Rf()[e] = 0.0f;   // equ_s4e17
                for (int c = r; c < s_words; c += Z) s.Sf()[c] = 0.0f;   // equ_s4e16: Omega = inf <=> S = 0
            }
            tm.sync();
        }
        if (!tm.team_any(active)) break;

        bool done = false;
        if (decoding) {
            // ---- Step 2: one sweep over the base rows (checks in ascending order)
            for (int i = 0; i < mb; ++i) {
                const bool live = active && !conv;
                if (!tm.team_any(live)) break;
                const int e0 = row_ptr[i], dc = row_ptr[i + 1] - e0;
                RowOut ro;
                ro.ok = true;
                ro.oldbits = 0;
                ro.Snew = ro.Sold = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                if (live && tm.lane_on) {
                    // the window can only fill in this row if consec + Z >= W (R4); otherwise
                    // no rollback information is needed
                    const bool track = belief && consec + Z >= W;
                    const int sidx4 = 4 * (i * Z + r);
                    if (sweep == 1) {
                        if constexpr (ALG == 1)
                            ro = track ? process_row_ms<true, true>(ent, e0, dc, sidx4, lane, s, a.alpha)
                                       : process_row_ms<true, false>(ent, e0, dc, sidx4, lane, s, a.alpha);
                        else
                            ro = track ? process_row<true, true>(ent, ptab, e0, dc, sidx4, lane, s)
                                       : process_row<true, false>(ent, ptab, e0, dc, sidx4, lane, s);
                    } else {
                        if constexpr (ALG == 1)
                            ro = track ? process_row_ms<false, true>(ent, e0, dc, sidx4, lane, s, a.alpha)
                                       : process_row_ms<false, false>(ent, e0, dc, sidx4, lane, s, a.alpha);
                        else
                            ro = track ? process_row<false, true>(ent, ptab, e0, dc, sidx4, lane, s)
                                       : process_row<false, false>(ent, ptab, e0, dc, sidx4, lane, s);
                    }
                }
                // ---- Step 2(3): stopping criterion, counted per check update (R4, R5)
                int first_bad = Z, last_bad = -1;   // first / last unclean check of the row
                if (MULTI) {
                    const int buf = (i & 1) * 32;
                    const unsigned m = __ballot_sync(kFull, tm.lane_on && !ro.ok);
                    if ((tm.tl & 31) == 0) ctl[buf + (tm.tl >> 5)] = m;
                    tm.sync();
                    if (belief) {
                        const int nw = tm.nthreads >> 5;
                        for (int w = 0; w < nw; ++w) {
                            const unsigned mw = ctl[buf + w];
                            if (mw) {
                                first_bad = min(first_bad, 32 * w + __ffs(mw) - 1);
                                last_bad = max(last_bad, 32 * w + 31 - __clz(mw));
                            }
                        }
                    }
                } else {
                    __syncwarp();
                    const unsigned m = (__ballot_sync(kFull, tm.lane_on && !ro.ok) & tm.slot_mask) >> tm.lane_base;
                    if (m) {
                        first_bad = __ffs(m) - 1;
                        last_bad = 31 - __clz(m);
                    }
                }
                bool fire = false;
                int rstar = 0;
                if (live && belief) {
                    rstar = W - consec - 1;           // the window fills at check i*Z + rstar
                    fire = rstar < Z && first_bad > rstar;
                    if (!fire) consec = (last_bad < 0) ? consec + Z : (Z - 1 - last_bad);
                }
                if (live && !fire) ev_dc += dc;
                if (tm.team_any(fire)) {
                    // the sequential decoder stops right after check i*Z + rstar: lanes r > rstar
                    // show their pre-row hard bits and S while the syndrome is verified (R5)
                    const bool back = fire && tm.lane_on && r > rstar;
                    uint32_t newbits = 0;
                    if (back) {
                        newbits = swap_row_bits(ent, e0, dc, r, Z, ro.oldbits, s);
                        put_check(s, i * Z + r, ro.Sold);
                    }
                    tm.sync();
                    const bool nz = tm.slot_any(fire && tm.lane_on && lane_syndrome(ent, row_ptr, mb, r, Z, s));
                    if (fire) {
                        if (!nz) {
                            conv = true;             // converged: output = state after check i*Z + rstar
                            ev_part += dc * (rstar + 1);
                        } else {
                            fires += 1;              // undetected fire: resume (R5)
                            ev_dc += dc;
                            consec = Z - 1 - max(last_bad, rstar);
                            if (back) {
                                swap_row_bits(ent, e0, dc, r, Z, newbits, s);
                                put_check(s, i * Z + r, ro.Snew);
                            }
                        }
                    }
                    tm.sync();
                }
            }
            // ---- end of sweep
            const bool want_syn = active && !conv && a.stop_rule == 2;
            if (tm.team_any(want_syn)) {
                tm.sync();
                const bool nz = tm.slot_any(want_syn && tm.lane_on && lane_syndrome(ent, row_ptr, mb, r, Z, s));
                if (want_syn && !nz) conv = true;
            }
            done = active && (conv || sweep >= a.max_iter);
            if (active && !done) sweep += 1;
        } else {
            done = active;
        }

        // ---- Step 3: outputs of finished frames (a8)
        if (tm.team_any(done)) {
            tm.sync();
            bool synd_zero = conv;
            const bool need_syn = done && !conv && decoding;
            if (tm.team_any(need_syn)) {
                const bool nz = tm.slot_any(need_syn && tm.lane_on && lane_syndrome(ent, row_ptr, mb, r, Z, s));
                if (need_syn) synd_zero = !nz;
            }
            const int iters = conv ? sweep : a.max_iter;
            const uint8_t flags = static_cast<uint8_t>((conv ? 1 : 0) | (synd_zero ? 2 : 0) | (fires > 0 ? 4 : 0));
            const float2* QP = s.QP();
            if (a.mode == MODE_DECODE_F32 || a.mode == MODE_DECODE_I8) {
                if (done && tm.lane_on) {
                    uint32_t* out = a.bits + static_cast<size_t>(fidx) * a.ld_words;
                    for (int w = r; w < a.ld_words; w += Z) {
                        uint32_t word = 0;
                        if (w < C.nwords)
                            for (int b = 0; b < 32; ++b) {
                                const int v = 32 * w + b;
                                if (v < C.N) word |= (__float_as_uint(QP[v].y) >> 31) << b;
                            }
                        out[w] = word;
                    }
                    if (a.omega) {
                        float* om = a.omega + static_cast<size_t>(fidx) * C.M;
                        for (int c = r; c < C.M; c += Z) {
                            float Sv, m;
                            if constexpr (ALG == 1) {
                                const float4 cs = reinterpret_cast<const float4*>(s.S)[c];
                                Sv = cs.z;                               // sign bit = sign of Omega
                                m = cs.x;                                // Omega = sgn * min (reading R20)
                            } else {
                                Sv = s.Sf()[c];
                                m = phi32(fabsf(Sv), ptab);               // Omega = sgn * phi(S)
                            }
                            om[c] = (__float_as_uint(Sv) >> 31) ? -m : m;
                        }
                    }
                    if (r == 0) {
                        a.iters[fidx] = iters;
                        a.flags[fidx] = flags;
                        if (a.ev) a.ev[fidx] = static_cast<int64_t>(ev_dc) * Z + ev_part;
                    }
                }
            } else if (a.mode == MODE_BER_SIM) {
                bool info_err = false, cw_err = false;
                if (done && tm.lane_on) {
                    for (int w = r; w < C.nwords; w += Z) {
                        uint32_t word = 0;
                        for (int b = 0; b < 32; ++b) {
                            const int v = 32 * w + b;
                            if (v < C.N) word |= (__float_as_uint(QP[v].y) >> 31) << b;
                        }
                        const uint32_t d = word ^ s.cw[w];
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
                if (done && r == 0) {
                    cnt[0] += 1;
                    cnt[2] += fe;
                    cnt[3] += ce;
                    cnt[4] += iters;
                    cnt[5] += static_cast<int64_t>(ev_dc) * Z + ev_part;
                    cnt[6] += conv ? 0 : 1;
                    cnt[7] += fires;
                }
            } else {  // MODE_CHANNEL
                if (done && tm.lane_on) {
                    if (a.llr_out) {
                        float* out = a.llr_out + static_cast<size_t>(fidx) * a.ld;
                        for (int v = r; v < C.N; v += Z) out[v] = QP[v].x;
                    }
                    if (a.cw_out) {
                        uint32_t* out = a.cw_out + static_cast<size_t>(fidx) * a.ld_words;
                        for (int w = r; w < a.ld_words; w += Z) out[w] = (w < C.nwords) ? s.cw[w] : 0u;
                    }
                }
            }
            if (done) active = false;
            tm.sync();
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

// element-wise evaluation of the contract functions (pin of device vs oracle bits)
__global__ void contract_eval_kernel(int fn, const float* __restrict__ x, float* __restrict__ y, int64_t n,
                                     const float4* __restrict__ tab)
{
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float v = x[k];
        float out;
        if (fn == 0) {
            out = phi32(v, tab);
        } else if (fn == 4) {
            out = phi_v1_unclamped(fminf(fmaxf(v, kPhiLo), kPhiHi));
            out = fminf(fmaxf(out, kPhiLo), kPhiHi);
        } else if (fn == 1) {
            out = ln32(v);
        } else {
            float sn, cs;
            sincos_quarter32(__float_as_uint(v) & 0xffffffu, sn, cs);
            out = (fn == 2) ? sn : cs;
        }
        y[k] = out;
    }
}

int launch_contract_eval(int fn, const float* x, float* y, int64_t n, const float4* tab, void* stream)
{
    if (n <= 0) return 0;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    contract_eval_kernel<<<static_cast<int>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(fn, x, y, n, tab);
    return static_cast<int>(cudaGetLastError());
}

// phi contract v2 table, one thread per segment (fp32 v1 values, fp64 Newton differences)
__global__ void phi_table_kernel(float4* __restrict__ out)
{
    const int seg = blockIdx.x * blockDim.x + threadIdx.x;
    if (seg < kPhiSegs) out[seg] = phi_segment_coeffs(seg);
}

int launch_phi_table(float4* out, void* stream)
{
    phi_table_kernel<<<(kPhiSegs + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(out);
    return static_cast<int>(cudaGetLastError());
}

// ---------------------------------------------------------------- host-side launch
template <bool MULTI, bool SMEM, int MAXT>
static int launch_t(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st)
{
    auto k = (g.alg == 1) ? cbp_kernel<MULTI, SMEM, MAXT, 1> : cbp_kernel<MULTI, SMEM, MAXT, 0>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
    k<<<grid, g.threads, g.smem_bytes, st>>>(a);
    return static_cast<int>(cudaGetLastError());
}

template <bool MULTI, bool SMEM, int MAXT>
static int occ_t(const Geometry& g, int* out)
{
    auto k = (g.alg == 1) ? cbp_kernel<MULTI, SMEM, MAXT, 1> : cbp_kernel<MULTI, SMEM, MAXT, 0>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
    return static_cast<int>(cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, g.threads, g.smem_bytes));
}

int launch_cbp(const KernelArgs& a, const Geometry& g, int grid, void* stream)
{
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!g.multi) return g.state_in_smem ? launch_t<false, true, 512>(a, g, grid, st) : launch_t<false, false, 512>(a, g, grid, st);
    if (g.threads <= 512)
        return g.state_in_smem ? launch_t<true, true, 512>(a, g, grid, st) : launch_t<true, false, 512>(a, g, grid, st);
    return g.state_in_smem ? launch_t<true, true, 1024>(a, g, grid, st) : launch_t<true, false, 1024>(a, g, grid, st);
}

int occupancy_ctas_per_sm(const Geometry& g, int* out)
{
    if (!g.multi) return g.state_in_smem ? occ_t<false, true, 512>(g, out) : occ_t<false, false, 512>(g, out);
    if (g.threads <= 512) return g.state_in_smem ? occ_t<true, true, 512>(g, out) : occ_t<true, false, 512>(g, out);
    return g.state_in_smem ? occ_t<true, true, 1024>(g, out) : occ_t<true, false, 1024>(g, out);
}

}  // namespace cbp
