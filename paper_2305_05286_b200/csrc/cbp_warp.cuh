// cbp_warp.cuh -- one frame per warp, K check slots per lane: the sm_100a kernel of the
// producer-side log-tanh CBP rows (and of layered BP, the same messages) for 17 <= Z <= 128
// (DESIGN.md §5).
//
// Lane l of the warp updates the lifted checks r_k = l + k L (k < K, L = ceil(Z/K) <= 32) of
// every base row.  The Z checks of a base row touch disjoint variables, so any assignment of
// them to lanes and slots gives the paper's sequential result bit for bit (reading R12); the K
// updates of a lane are independent and are interleaved by the compiler.  A warp is a whole
// team: rows are ordered by __syncwarp and the stop window's ballots, there are no named
// barriers, a finished frame is replaced at once (no sweep-boundary wait), and the per-row
// control is paid once per K dc edges of a lane.
//
// Per-warp state in shared memory: Lambda'[N] (the producer-side posterior, cbp_kernel.cuh) and
// H[N] -- the decision of v's latest visit as one byte whose sign bit is the sign of the Lambda
// that visit read (layered BP: of Lambda'), so a warp's frame takes 5 N bytes instead of 8 N and
// more frames fit on an SM --, S[M] (check records with sign = Omega < 0: Omega output and
// rollback only), the transmitted codeword (ber_sim), a park buffer for rows longer than
// CBP_DC_REG, and R (here, or in a global slot per warp: RG) laid out as
// R[(b K + k) 32 + l] -- coalesced, and the R words of a row's edges sit at compile-time
// offsets from one row pointer.  The phi table and the schedule entries are staged once per
// CTA by the bulk-copy (TMA) engine.
#pragma once
#include "cbp_kernel.cuh"

namespace cbp {

// ---------------------------------------------------------------- bulk copy global -> shared (TMA engine)
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// bytes % 16 == 0, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}

// ---------------------------------------------------------------- the rows
// Pipe balance of the phi-row fetches (rows with K >= 2 slots per lane: C3a / C5, C3b): edge 0's
// C2B row from shared memory instead of TEX, edge 6's B2V row through TEX instead of shared memory.
// C5 -1.5..2 % (A/B over several boxes; K = 1 codes measured slower with it and keep 0).
#ifndef CBP_B2V_TEX_MASK
#define CBP_B2V_TEX_MASK 0x40  // bit e: edge e (mod 8) of a row fetches its B2V phi row through TEX
#endif
#ifndef CBP_C2B_LDS_MASK
#define CBP_C2B_LDS_MASK 0x01  // bit e: edge e (mod 8) of a row fetches its C2B phi row from shared memory
#endif
#ifndef CBP_UNIFORM_WARP
#define CBP_UNIFORM_WARP 1
#endif
#ifndef CBP_WARP_LEAN
#define CBP_WARP_LEAN 0     // 1: entries and R re-read per slot (fewer registers, A/B runs)
#endif
#ifndef CBP_PARK_U
#define CBP_PARK_U 4        // edges per chunk of a long (parked) row
#endif
#ifndef CBP_PARK_C2B_TEX
#define CBP_PARK_C2B_TEX 0xF  // bit u: edge u of a 4-edge chunk of a long (parked) row fetches its C2B phi row through TEX
                              // (all four: C3b -3.3 %; two of four -1.6 %; B2V rows through TEX as well: no better)
#endif
#ifndef CBP_PARK_B2V_TEX
#define CBP_PARK_B2V_TEX 0x0  // the same for the B2V phi row
#endif
#ifndef CBP_RPRE
#define CBP_RPRE 0          // 1: a row's last slot requests the next row's slot-0 R words (A/B switch)
#endif
#ifndef CBP_LLR_BATCH
#define CBP_LLR_BATCH 8     // 128-bit LLR loads in flight per lane at a frame's start (decode modes)
#endif
#ifndef CBP_R_CG
#define CBP_R_CG 2          // R words in global memory: 1 = loads / stores cached in L2 only (keep L1 for the TEX phi
                            // rows), 2 = the same with an L2 evict_last policy (C5 -1.1 %, C3a at 1.5 dB -1.6 %, DRAM writes -43 %)
#endif
// R word access: RG = R in the global workspace (L2-only when CBP_R_CG), else in shared memory.
// CBP_R_CG == 2: L2-only with an L2 evict_last policy descriptor (createpolicy folds into a constant
// descriptor in uniform registers: no extra instruction or register in the row body).
// The asm statements are volatile (ordered among themselves: R is touched only through them) without a
// memory clobber, so shared-memory accesses still move across them.
template <bool RG>
__device__ __forceinline__ float rld(const float* p)
{
#if CBP_R_CG == 2
    if constexpr (RG) {
        float v; unsigned long long pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.cg.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
        return v;
    } else return *p;
#else
    if constexpr (RG && CBP_R_CG) return __ldcg(p);
    else return *p;
#endif
}
template <bool RG>
__device__ __forceinline__ void rst(float* p, float v)
{
#if CBP_R_CG == 2
    if constexpr (RG) {
        unsigned long long pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("st.global.cg.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(p), "f"(v), "l"(pol));
    } else *p = v;
#else
    if constexpr (RG && CBP_R_CG) __stcg(p, v);
    else *p = v;
#endif
}

// ---------------------------------------------------------------- two edges on the packed FP32x2 pipe
// CBP_PAIR: the fp32 steps of two independent edges of a row issue as one FADD2 / FFMA2 (sm_100
// packed FP32: each element is the same IEEE operation with the same rounding, so every bit is
// the contract's): Q^new = Lambda - R, the phi index's 16x magic (fma.rz), C - m, u_hi and u_lo,
// S - Phi and Lambda' = Q^new + R^new.  The cubic stays scalar (its coefficients come from two
// different table rows).  A/B switch, off: measured slower twice (C5 +1.3 % with the round-2 body,
// +4 % after the instruction-cache work; C2 +2..4 %) although it issues ~4.5 fewer instructions per
// edge visit -- the packed forms cost latency / register-pair moves on this dependent chain.
#ifndef CBP_PAIR
#define CBP_PAIR 0
#endif

// phi32 of |x.x| and |x.y| (contract.cuh phi32_index + phi32_cubic, the FP steps paired); TA / TB:
// the row of element a / b through the texture pipe
// (ta / tb are compile-time constants after the callers' unrolling)
__device__ __forceinline__ float2 phi2_sel(float2 x, bool ta, bool tb, const float4* __restrict__ ptab, const Lane& L,
                                           TexH tex)
{
    x.x = fminf(fmaxf(fabsf(x.x), kPhiLo), kPhiHi);
    x.y = fminf(fmaxf(fabsf(x.y), kPhiLo), kPhiHi);
    const uint32_t b0 = __float_as_uint(x.x), b1 = __float_as_uint(x.y);
    uint32_t ub0, ub1;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(ub0) : "r"(b0), "r"(L.m19), "r"(L.one));   // (b & m19) | one
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(ub1) : "r"(b1), "r"(L.m19), "r"(L.one));
    const float2 u_lo = __fadd2_rn(make_float2(__uint_as_float(ub0), __uint_as_float(ub1)), make_float2(-1.0f, -1.0f));
    const float2 m = __ffma2_rz(x, make_float2(16.0f, 16.0f), make_float2(8388576.0f, 8388576.0f));
    const float2 cm = __fadd2_rn(make_float2(8388576.0f, 8388576.0f), make_float2(-m.x, -m.y));
    const float2 u_hi = __ffma2_rn(x, make_float2(16.0f, 16.0f), cm);
    const bool h0 = x.x >= 2.0f, h1 = x.y >= 2.0f;
    const int s0 = h0 ? static_cast<int>(__float_as_uint(m.x)) - (0x4b000000 - 704) : static_cast<int>(b0 >> 19) - 1344;
    const int s1 = h1 ? static_cast<int>(__float_as_uint(m.y)) - (0x4b000000 - 704) : static_cast<int>(b1 >> 19) - 1344;
    CBP_CHECK(s0 >= 0 && s0 < kPhiSegs && s1 >= 0 && s1 < kPhiSegs);
    const float u0 = h0 ? u_hi.x : u_lo.x, u1 = h1 ? u_hi.y : u_lo.y;
    const float4 c0 = ta ? tex1Dfetch<float4>(tex, s0) : ptab[s0];
    const float4 c1 = tb ? tex1Dfetch<float4>(tex, s1) : ptab[s1];
    return make_float2(phi32_cubic(c0, u0), phi32_cubic(c1, u1));
}

// cbp_phase1 (cbp_kernel.cuh) for edges a, b in this order: flip test, rollback bits, Q^new, C2B phi,
// S in ascending order, sign
__device__ __forceinline__ void wphase1_pair(const float (&va)[2], const float (&vb)[2], float ra, float rb, float2& q,
                                             float2& ph, bool ta, bool tb, const float4* __restrict__ ptab,
                                             const Lane& L, TexH tex, RowAcc<1>& acc)
{
    const uint32_t la = __float_as_uint(va[0]), ha = __float_as_uint(va[1]);
    const uint32_t lb = __float_as_uint(vb[0]), hb = __float_as_uint(vb[1]);
    acc.flipw[0] |= (la ^ ha) | (lb ^ hb);                      // equ_s4e24 (R7)
    acc.oldbits[0] = __funnelshift_l(hb, __funnelshift_l(ha, acc.oldbits[0], 1), 1);
    q = __fadd2_rn(make_float2(va[0], vb[0]), make_float2(-ra, -rb));   // equ_s4e19: Lambda - R (exact negation)
    ph = phi2_sel(q, ta, tb, ptab, L, tex);                     // C2B (equ_s4e21)
    acc.Ssum[0] = __fadd_rn(__fadd_rn(acc.Ssum[0], ph.x), ph.y);   // R12
    acc.negw[0] ^= __float_as_uint(q.x) ^ __float_as_uint(q.y);
}

// cbp_phase2 for edges a, b: R^new = sgn(Omega) sgn(Q^new) phi(|S - Phi|), Lambda' = Q^new + R^new
__device__ __forceinline__ void wphase2_pair(const RowAcc<1>& acc, float2 q, float2 ph, float2& rn, float2& lamn,
                                             bool ta, bool tb, const float4* __restrict__ ptab, const Lane& L,
                                             TexH tex)
{
    const float2 d = __fadd2_rn(make_float2(acc.Ssum[0], acc.Ssum[0]), make_float2(-ph.x, -ph.y));   // S - Phi (R10)
    const float2 mag = phi2_sel(d, ta, tb, ptab, L, tex);
    rn.x = __uint_as_float(__float_as_uint(mag.x) | ((acc.negw[0] ^ __float_as_uint(q.x)) & kSign));
    rn.y = __uint_as_float(__float_as_uint(mag.y) | ((acc.negw[0] ^ __float_as_uint(q.y)) & kSign));
    lamn = __fadd2_rn(q, rn);                                   // equ_s4e20 of the next visitor
}

// K per-slot values in registers, written / read at a runtime slot index by predicated moves
// (a dynamically indexed array would live in local memory)
template <int K, typename T>
struct SlotVals {
    T v[K];
    __device__ __forceinline__ void set(int k, T x)
    {
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (j == k) v[j] = x;
    }
    __device__ __forceinline__ T get(int k) const
    {
        T x = v[0];
#pragma unroll
        for (int j = 1; j < K; ++j)
            if (j == k) x = v[j];
        return x;
    }
};

// ---------------------------------------------------------------- per-frame (cold) code
// The per-frame code (channel, encoder, stop-window verification, final syndrome, outputs) runs
// once per frame between long stretches of the row loop.  Its instructions share the SM's 32 KB
// L1.5 instruction cache with the hot row body, so it is kept compact: loops over the K slots are
// not unrolled, and the syndrome is one out-of-line function instead of three inlined copies
// (C5 at 2.5 dB switches frames every ~7 sweeps; measured: one shared max-dc body -9 %).

// Philox4x32-10 (contract.cuh) out of line: one copy for the info words and the noise
static __device__ __noinline__ u32x4 w_philox(u32x4 c, uint32_t k0, uint32_t k1) { return philox4x32_10(c, k0, k1); }

// parity of the team's valid checks over all rows from the hard decisions (sign of H): true if
// some check is unsatisfied (early exit every 4 rows)
template <int K, bool TEAM>
__device__ __noinline__ bool w_syndrome_nz(const int4* __restrict__ ent, const int32_t* __restrict__ row_ptr,
                                           const int8_t* __restrict__ hb, int mb, int Z, int tl, int Lk)
{
    auto tany = [&](bool p) -> bool {
        if constexpr (TEAM) return __syncthreads_or(p) != 0;
        else return __any_sync(0xffffffffu, p);
    };
    uint32_t nz = 0;
    for (int i = 0; i < mb; ++i) {
        if ((i & 3) == 0 && i && tany(nz != 0u)) return true;   // an unsatisfied check: done
        uint32_t par = 0;                                     // bit k: parity of check i Z + r_k
        for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            const int2 A = *reinterpret_cast<const int2*>(ent + 2 * e);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int r = tl + k * Lk;
                const bool v = tl < Lk && r < Z;
                const int vv = A.x + wrap((v ? r : Z - 1) + A.y, Z);
                par ^= v ? static_cast<uint32_t>(hb[vv] < 0) << k : 0u;
            }
        }
        nz |= par;
    }
    return tany(nz != 0u);
}

// What a row reports to the stop logic: first / last unclean check, and for a possible mid-row
// stop the slots' previous decision bits and check records (old / new).
template <int K>
struct WRow {
    int first_bad, last_bad;
    SlotVals<K, uint32_t> oldb;
    SlotVals<K, float> sold, snew;
};

// The per-row context of a lane.
struct WCtx {
    int l, Lk, Z;                // l: the lane's index in the frame's team (warp mode: lane)
    int l0;                      // index of the warp's lane 0 in the team (warp mode: 0)
    bool fire_possible, keepS;   // the window may fill in this row; S records are kept (Omega output)
    bool r0;                     // sweep 1: every R_{c->v} still holds its initial 0 (equ_s4e17) -- not read
    float* lam;                  // Lambda'[N]
    int8_t* hb;                  // H[N]: sign = hard decision of v's latest visit
    float* pb;                   // park buffer: Phi of edge e at pb[e 32 + l]
    float* rrow;                 // this lane's R word of (row entry 0, slot 0); (edge e, slot k) at rrow[(e K + k) 32]
    float* Srow;                 // S records of this row (keepS)
    const float* nrow = nullptr; // CBP_RPRE: this lane's slot-0 R word of the next row's entry 0 (nullptr: no request)
    int npre = 0;                // CBP_RPRE: words of rpre[] the previous row requested for this row
};

// Slot k's check update done: its record, the rollback values and its stop flags (equ_s4e2, equ_s4e24).
template <int K, bool LBP>
__device__ __forceinline__ void wslot_done(const WCtx& c, int k, int rr, bool v, const RowAcc<1>& acc, WRow<K>& o)
{
    const float sn = __uint_as_float(__float_as_uint(acc.Ssum[0]) | (acc.negw[0] & kSign));
    if (c.keepS && !LBP && v) c.Srow[rr] = sn;                  // equ_s4e23
    if (c.fire_possible) {
        o.oldb.set(k, acc.oldbits[0]);
        o.snew.set(k, sn);
    }
    const unsigned m = __ballot_sync(kFull, v && (((acc.negw[0] | acc.flipw[0]) & kSign) != 0u));
    if (m) {
        o.first_bad = min(o.first_bad, k * c.Lk + c.l0 + __ffs(m) - 1);
        o.last_bad = max(o.last_bad, k * c.Lk + c.l0 + 31 - __clz(m));
    }
}

// One base row with DC edges for the K slots of the lane (producer-side update, cbp_kernel.cuh):
// the row's schedule entries once, then per slot all loads, phase 1, phase 2.  The slots run in
// a loop that is not unrolled: the unrolled K x DC bodies overflowed the 32 KB L1.5 instruction
// cache (ncu: no_instruction stalls 2.3 per issue, issue active 37 %).  A slot beyond Z (v false)
// computes on check Z - 1 and stores nothing but its private R words.
// lastoff: the row has DC - 1 edges and runs this body with its last edge masked (CBP_DCMERGE:
// rows of the code's max dc and of max dc - 1 share one body, halving the hot code that the
// warps of an SMSP stream through the instruction caches).  The masked edge reads the previous
// edge's variable (valid addresses), loads no R, adds nothing to S / the sign / flip / rollback
// words and stores nothing.
template <int DC, int K, int ALG, int TM, bool RG>
__device__ __forceinline__ void wrow(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0,
                                     const Lane& L, TexH tex, const WCtx& c, WRow<K>& o, float (&rpre)[CBP_DC_REG],
                                     bool lastoff = false)
{
    constexpr bool LBP = ALG == 2;
    constexpr bool TEXC = TM != 2, TEXB = TM == 1;             // phi rows: C2B / B2V through the texture pipe
#if !CBP_WARP_LEAN
    int2 A[DC];
#pragma unroll
    for (int e = 0; e < DC; ++e) A[e] = *reinterpret_cast<const int2*>(ent + 2 * (e0 + e));
    if constexpr (DC >= 2)
        if (lastoff) A[DC - 1] = A[DC - 2];
    // R words of the next slot are requested before the current slot's update (their global /
    // L2 latency then overlaps it); slot 0's are loaded here
    float rnext[DC];
#pragma unroll
    for (int e = 0; e < DC; ++e)
        rnext[e] = (c.r0 || (e == DC - 1 && lastoff)) ? 0.0f
                   : (CBP_RPRE && RG && e < c.npre)   ? rpre[e]      // requested by the previous row's last slot
                                                      : rld<RG>(c.rrow + e * K * 32);
#endif
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const int r = c.l + k * c.Lk;
        const bool v = c.l < c.Lk && r < c.Z;
        const int rr = v ? r : c.Z - 1;
        if (c.keepS && c.fire_possible) o.sold.set(k, c.Srow[rr]);
        float* rk = c.rrow + k * 32;
        float ro[DC][1];
#if CBP_WARP_LEAN
        int2 A[DC];
#pragma unroll
        for (int e = 0; e < DC; ++e) {
            A[e] = *reinterpret_cast<const int2*>(ent + 2 * (e0 + e));
            ro[e][0] = c.r0 ? 0.0f : rld<RG>(rk + e * K * 32);
        }
#else
#pragma unroll
        for (int e = 0; e < DC; ++e) ro[e][0] = rnext[e];          // R_{c->v}
        if (k + 1 < K) {
#pragma unroll
            for (int e = 0; e < DC; ++e)
                rnext[e] = (c.r0 || (e == DC - 1 && lastoff)) ? 0.0f : rld<RG>(rk + 32 + e * K * 32);
        }
#if CBP_RPRE
        else if (RG && c.nrow) {                                  // last slot: the next row's slot-0 words
#pragma unroll
            for (int e = 0; e < DC; ++e) rnext[e] = rld<RG>(c.nrow + e * K * 32);
        }
#endif
#endif
        RowAcc<1> acc;
        acc.Ssum[0] = 0.0f;
        acc.negw[0] = acc.flipw[0] = acc.oldbits[0] = 0u;
        int vi[DC];
        float vs[DC][2], q[DC][1], ph[DC][1];
#pragma unroll
        for (int e = 0; e < DC; ++e) {
            vi[e] = A[e].x + wrap(rr + A[e].y, c.Z);                // variable j Z + (r + s) mod Z
            CBP_CHECK(vi[e] >= 0 && vi[e] < L.slot_bytes);
            vs[e][0] = c.lam[vi[e]];                                // Lambda_v
            // H_v: the sign-extended byte carries the decision in bit 31 (layered BP: Lambda_v itself)
            vs[e][1] = LBP ? vs[e][0] : __int_as_float(static_cast<int>(c.hb[vi[e]]));
        }
        // C2B rows through TEX except for the edges CBP_C2B_LDS_MASK selects, B2V rows from shared memory
        // except for the edges CBP_B2V_TEX_MASK selects (folded after unrolling)
        constexpr int kC2BLds = (K >= 2 && TM == 0) ? CBP_C2B_LDS_MASK : 0;   // TM 1: no table in shared memory
        constexpr int kB2VTex = (K >= 2 && TM == 0) ? CBP_B2V_TEX_MASK : 0;
        float rn[DC][1], lamn[DC][1];
        // edges (0,1), (2,3), ... below the last on the packed pipe (CBP_PAIR); the last edge (maskable,
        // lastoff) and an odd one alone
        constexpr int NP = CBP_PAIR ? (DC - 1) / 2 : 0;
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int e = 2 * j;
            float2 q2, ph2;
            wphase1_pair(vs[e], vs[e + 1], ro[e][0], ro[e + 1][0], q2, ph2, TEXC && ((kC2BLds >> (e & 7)) & 1) == 0,
                         TEXC && ((kC2BLds >> ((e + 1) & 7)) & 1) == 0, ptab, L, tex, acc);
            q[e][0] = q2.x; q[e + 1][0] = q2.y;
            ph[e][0] = ph2.x; ph[e + 1][0] = ph2.y;
        }
#pragma unroll
        for (int e = 2 * NP; e < DC; ++e) {
            if (e == DC - 1 && DC >= 2) {                       // possibly masked (lastoff)
                RowAcc<1> t = acc;
                if (TEXC && ((kC2BLds >> (e & 7)) & 1) == 0)
                    cbp_phase1<1, true>(vs[e], ro[e], q[e], ph[e], ptab, L, tex, t);
                else
                    cbp_phase1<1, false>(vs[e], ro[e], q[e], ph[e], ptab, L, tex, t);
                if (!lastoff) acc = t;
            } else if (TEXC && ((kC2BLds >> (e & 7)) & 1) == 0) {
                cbp_phase1<1, true>(vs[e], ro[e], q[e], ph[e], ptab, L, tex, acc);
            } else {
                cbp_phase1<1, false>(vs[e], ro[e], q[e], ph[e], ptab, L, tex, acc);
            }
        }
        // all B2V lookups of the row before its first store: a table load may not move above a
        // shared-memory store the compiler cannot prove disjoint (one dependent chain per edge otherwise)
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int e = 2 * j;
            float2 rn2, lamn2;
            wphase2_pair(acc, make_float2(q[e][0], q[e + 1][0]), make_float2(ph[e][0], ph[e + 1][0]), rn2, lamn2,
                         TEXB || ((kB2VTex >> (e & 7)) & 1) != 0, TEXB || ((kB2VTex >> ((e + 1) & 7)) & 1) != 0, ptab,
                         L, tex);
            rn[e][0] = rn2.x; rn[e + 1][0] = rn2.y;
            lamn[e][0] = lamn2.x; lamn[e + 1][0] = lamn2.y;
        }
#pragma unroll
        for (int e = 2 * NP; e < DC; ++e) {
            if (TEXB || ((kB2VTex >> (e & 7)) & 1) != 0)
                cbp_phase2<1, true>(acc, q[e], ph[e], rn[e], lamn[e], ptab, L, tex);
            else
                cbp_phase2<1, false>(acc, q[e], ph[e], rn[e], lamn[e], ptab, L, tex);
        }
#pragma unroll
        for (int e = 0; e < DC; ++e) {
            const bool on = !(e == DC - 1 && lastoff);
            if (v && on) {
                c.lam[vi[e]] = lamn[e][0];
                c.hb[vi[e]] = static_cast<int8_t>(__float_as_uint(LBP ? lamn[e][0] : vs[e][0]) >> 24);   // H_v
            }
            if (on) rst<RG>(rk + e * K * 32, rn[e][0]);            // equ_s4e22 commit of R_{c->v}
        }
        wslot_done<K, LBP>(c, k, rr, v, acc, o);
    }
#if CBP_RPRE && !CBP_WARP_LEAN
#pragma unroll
    for (int e = 0; e < DC; ++e) rpre[e] = rnext[e];
#endif
}

// Rows longer than CBP_DC_REG: per slot two passes over the edges in chunks of U (all loads of a
// chunk first, U independent phi chains), a remainder one edge at a time, parking {Q^new,
// Phi | sign of the decision} in the variable's slot between the phases (only this lane touches
// the variable during the row).  Both phi rows from the shared-memory table.
template <int U, int K, int ALG, bool RG, int TM>
__device__ __forceinline__ void wpark_p1(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0, int e,
                                         int rr, bool v, const Lane& L, const WCtx& c, float* rk, RowAcc<1>& acc, TexH tex)
{
    constexpr bool LBP = ALG == 2;
    int a[U];
    float vv[U][2], ro[U][1], q[U][1], ph[U][1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + e + u));
        a[u] = A.x + wrap(rr + A.y, c.Z);
        vv[u][0] = c.lam[a[u]];
        vv[u][1] = LBP ? vv[u][0] : __int_as_float(static_cast<int>(c.hb[a[u]]));
        ro[u][0] = c.r0 ? 0.0f : rld<RG>(rk + (e + u) * K * 32);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        // chunk edges CBP_PARK_C2B_TEX selects fetch their C2B phi row through TEX (pipe balance, as in wrow)
        if (TM == 0 && U > 1 && ((CBP_PARK_C2B_TEX >> u) & 1))
            cbp_phase1<1, true>(vv[u], ro[u], q[u], ph[u], ptab, L, tex, acc);
        else
            cbp_phase1<1, false>(vv[u], ro[u], q[u], ph[u], ptab, L, tex, acc);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) c.pb[(e + u) * 32] = ph[u][0];    // Phi, lane-private
    if (v) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            c.lam[a[u]] = q[u][0];                                // Q^new parked in the Lambda word
            if (!LBP) c.hb[a[u]] = static_cast<int8_t>(__float_as_uint(vv[u][0]) >> 24);   // H_v (decided here)
        }
    }
}

template <int U, int K, int ALG, bool RG, int TM>
__device__ __forceinline__ void wpark_p2(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0, int e,
                                         int rr, bool v, const Lane& L, const WCtx& c, float* rk, const RowAcc<1>& acc,
                                         TexH tex)
{
    constexpr bool LBP = ALG == 2;
    int a[U];
    float vv[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + e + u));
        a[u] = A.x + wrap(rr + A.y, c.Z);
        vv[u][0] = c.lam[a[u]];                                   // Q^new
        vv[u][1] = c.pb[(e + u) * 32];                            // Phi
    }
    float rn[U][1], lamn[U][1];
#pragma unroll
    for (int u = 0; u < U; ++u) {                               // lookups first (see wrow)
        const float q[1] = {vv[u][0]}, ph[1] = {vv[u][1]};
        if (TM == 0 && U > 1 && ((CBP_PARK_B2V_TEX >> u) & 1))
            cbp_phase2<1, true>(acc, q, ph, rn[u], lamn[u], ptab, L, tex);
        else
            cbp_phase2<1, false>(acc, q, ph, rn[u], lamn[u], ptab, L, tex);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (v) {
            c.lam[a[u]] = lamn[u][0];
            if (LBP) c.hb[a[u]] = static_cast<int8_t>(__float_as_uint(lamn[u][0]) >> 24);
        }
        rst<RG>(rk + (e + u) * K * 32, rn[u][0]);
    }
}

template <int K, int ALG, int TM, bool RG>
__device__ __forceinline__ void wrow_park(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0, int dc,
                                          const Lane& L, TexH tex, const WCtx& c, WRow<K>& o)
{
    constexpr int U = CBP_PARK_U;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const int r = c.l + k * c.Lk;
        const bool v = c.l < c.Lk && r < c.Z;
        const int rr = v ? r : c.Z - 1;
        if (c.keepS && c.fire_possible) o.sold.set(k, c.Srow[rr]);
        float* rk = c.rrow + k * 32;
        RowAcc<1> acc;
        acc.Ssum[0] = 0.0f;
        acc.negw[0] = acc.flipw[0] = acc.oldbits[0] = 0u;
        int e = 0;
#pragma unroll 1
        for (; e + U <= dc; e += U) wpark_p1<U, K, ALG, RG, TM>(ent, ptab, e0, e, rr, v, L, c, rk, acc, tex);
#pragma unroll 1
        for (; e < dc; ++e) wpark_p1<1, K, ALG, RG, TM>(ent, ptab, e0, e, rr, v, L, c, rk, acc, tex);
        e = 0;
#pragma unroll 1
        for (; e + U <= dc; e += U) wpark_p2<U, K, ALG, RG, TM>(ent, ptab, e0, e, rr, v, L, c, rk, acc, tex);
#pragma unroll 1
        for (; e < dc; ++e) wpark_p2<1, K, ALG, RG, TM>(ent, ptab, e0, e, rr, v, L, c, rk, acc, tex);
        wslot_done<K, ALG == 2>(c, k, rr, v, acc, o);
    }
}

#ifndef CBP_DCMERGE
#define CBP_DCMERGE 1
#endif
#ifndef CBP_DCMERGE_MINK
#define CBP_DCMERGE_MINK 2   // smallest K (slots per lane) that merges
#endif
template <int K, int ALG, int TM, bool RG>
__device__ __forceinline__ void wrow_dispatch(int dc, int max_dc, bool merge, const int4* __restrict__ ent,
                                              const float4* __restrict__ ptab, int e0, const Lane& L, TexH tex,
                                              const WCtx& c, WRow<K>& o, float (&rpre)[CBP_DC_REG])
{
    // rows of max dc - 1 edges run the max-dc body with the last edge masked: one call site per body
    // (wrow is inlined, so a second call site would be a second copy).  Only for K >= 2 slots per lane
    // (C3a / C5); with K = 1 (C2, P2048) the merged body measured slower (+26 %, +2 %).  `merge`: only in
    // the fused ber_sim, whose per-frame channel code competes for the instruction cache (C5 -4.5 %); plain
    // decoding keeps one body per dc (the masked edge's work costs it 4 %).
    const bool lastoff = CBP_DCMERGE && K >= CBP_DCMERGE_MINK && merge && dc + 1 == max_dc && max_dc <= CBP_DC_REG && dc >= 2;
    if (lastoff) dc += 1;
    switch (dc) {
#if CBP_DC_REG >= 1
    case 1: wrow<1, K, ALG, TM, RG>(ent, ptab, e0, L, tex, c, o, rpre, lastoff); break;
    case 2: wrow<2, K, ALG, TM, RG>(ent, ptab, e0, L, tex, c, o, rpre, lastoff); break;
    case 3: wrow<3, K, ALG, TM, RG>(ent, ptab, e0, L, tex, c, o, rpre, lastoff); break;
    case 4: wrow<4, K, ALG, TM, RG>(ent, ptab, e0, L, tex, c, o, rpre, lastoff); break;
    case 5: wrow<5, K, ALG, TM, RG>(ent, ptab, e0, L, tex, c, o, rpre, lastoff); break;
    case 6: wrow<6, K, ALG, TM, RG>(ent, ptab, e0, L, tex, c, o, rpre, lastoff); break;
#endif
#if CBP_DC_REG >= 8
    case 7: wrow<7, K, ALG, TM, RG>(ent, ptab, e0, L, tex, c, o, rpre, lastoff); break;
    case 8: wrow<8, K, ALG, TM, RG>(ent, ptab, e0, L, tex, c, o, rpre, lastoff); break;
#endif
    default: wrow_park<K, ALG, TM, RG>(ent, ptab, e0, dc, L, tex, c, o); break;
    }
}

// ---------------------------------------------------------------- the kernel
// RG: R in a global slot per warp (else in the warp's shared state).  Modes: decode (fp32 /
// int8 LLRs from HBM), the fused ber_sim, and the two halves of a split one -- channel only
// (MODE_CHANNEL: L and the codewords to HBM) and decode + error count (MODE_BER_LLR).
// TM: phi table rows for C2B / B2V through the texture pipe (0: C2B only, 1: both -- the table
// is then not staged in shared memory, 2: neither).
// TEAM: one frame per CTA instead of one per warp (large frames, C4: N = 26112, Z = 384): the CTA's
// warps are the team, lane t of the team updates checks t + k L, rows are ordered by a CTA barrier
// that also reduces the stop window's first / last unclean check; R stays lane-private in a global
// slot per warp.
template <int K, bool RG, int MAXT, int ALG, int TM, bool TEAM = false>
__global__ void __launch_bounds__(MAXT, 1) cbp_warp_kernel(const __grid_constant__ KernelArgs a)
{
    static_assert(!TEAM || RG, "team frames keep R in the global workspace");
    constexpr bool TEXB = TM == 1;
    constexpr bool LBP = ALG == 2;
    extern __shared__ __align__(16) uint32_t smem[];
    const DevCode& C = a.code;
    const int Z = C.Z, mb = C.mb, N = C.N;

    // ---- a1: stage the phi table and the schedule entries with the bulk-copy engine (one
    // elected thread arms an mbarrier with the byte count, every thread waits on its phase)
    constexpr int kTabWords = TEXB ? 0 : 4 * kPhiSegs;
    float4* ptab = reinterpret_cast<float4*>(smem);
    int4* ent = reinterpret_cast<int4*>(smem + kTabWords);
    int32_t* row_ptr = reinterpret_cast<int32_t*>(smem + kTabWords + 8 * C.nent);
    int16_t* pshift = reinterpret_cast<int16_t*>(row_ptr + mb + 1);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.table_words - 4);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        const uint32_t tb = 4u * kTabWords, eb = 32u * static_cast<uint32_t>(C.nent);
        mbar_expect_tx(bar, tb + eb);
        if (tb) bulk_g2s(ptab, C.phi_tab, tb, bar);
        bulk_g2s(ent, a.ent_dev, eb, bar);
    }
    for (int k = threadIdx.x; k <= mb; k += blockDim.x) row_ptr[k] = a.row_ptr[k];
    for (int k = threadIdx.x; k < mb; k += blockDim.x) pshift[k] = a.pshift[k];

    // the warp index through a warp reduction: REDUX writes a uniform register, so the per-warp state
    // bases derived from it stay in the uniform datapath instead of being rematerialised per slot
    // (K >= 2: C5 -0.7 %, C3b -1.3 %; K = 1 codes measured +1.7 % and keep threadIdx >> 5)
    const int warp = (CBP_UNIFORM_WARP && K >= 2) ? static_cast<int>(__reduce_min_sync(kFull, threadIdx.x >> 5))
                                                  : static_cast<int>(threadIdx.x >> 5);
    const int l = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    const int tl = TEAM ? static_cast<int>(threadIdx.x) : l;  // lane index in the frame's team
    const int TL = TEAM ? static_cast<int>(blockDim.x) : 32;  // team size
    const int w0 = TEAM ? warp : 0, wstep = TEAM ? nwarps : 1;   // this warp's share of word-wise loops
    const int Lk = a.lanes;                                   // L: lanes with check slots
    int rk[K];
    bool vk[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int r = tl + k * Lk;
        vk[k] = tl < Lk && r < Z;
        rk[k] = vk[k] ? r : Z - 1;                            // invalid slots compute on check Z - 1, store nothing
    }
    // team barrier (warp mode: the warp's) and team-wide any
    auto tsync = [&]() {
        if constexpr (TEAM) __syncthreads();
        else __syncwarp();
    };
    auto tany = [&](bool p) -> bool {
        if constexpr (TEAM) return __syncthreads_or(p) != 0;
        else return __any_sync(kFull, p);
    };
    // per-warp state (cbp_internal.h): counters (8 x u64) | Lambda [N] | H [N bytes] | cw [nwords] |
    // park buffer | R (if !RG) | S [M] (if the launch outputs Omega: the geometry then has room for it)
    // (team: one state per CTA, its park buffer per warp, and 2 x 2 x nwarps control words after it)
    unsigned long long* wcnt =
        reinterpret_cast<unsigned long long*>(smem + a.table_words + static_cast<size_t>(TEAM ? 0 : warp) * a.slot_words);
    float* const lam = reinterpret_cast<float*>(wcnt + 8);
    int8_t* const hb = reinterpret_cast<int8_t*>(lam + N);
    uint32_t* cw = reinterpret_cast<uint32_t*>(lam + N + warp_hb_words(N));
    float* const pb = reinterpret_cast<float*>(cw + warp_cw_words(C.nwords)) + (TEAM ? warp * warp_pb_words(C.max_dc) : 0) + l;
    const int rwords = C.nent * K * 32;                       // R words of one warp
    float* const Rs = reinterpret_cast<float*>(cw + warp_cw_words(C.nwords) + (TEAM ? nwarps : 1) * warp_pb_words(C.max_dc));
    float* Rw = !RG ? Rs
                    : a.rstate + (TEAM ? static_cast<size_t>(blockIdx.x) * a.r_words + static_cast<size_t>(warp) * rwords
                                       : (static_cast<size_t>(blockIdx.x) * nwarps + warp) * a.r_words);
    float* S = RG ? Rs : Rs + rwords;
    // team: [2 buffers][first | last][nwarps] (after S, which only the log-tanh Omega output keeps)
    int* const tctl = reinterpret_cast<int*>(S + ((a.omega != nullptr && !LBP) ? C.M : 0));
    long long* const tfrm = reinterpret_cast<long long*>((reinterpret_cast<uintptr_t>(tctl + 4 * nwarps) + 7) &
                                                         ~static_cast<uintptr_t>(7));   // team: frame index
    const Lane lane{0, 0, 0, 0, 0, 0, N, 0, a.phi_m19, a.phi_one};   // slot_bytes: variable bound (debug builds)
    if (TEAM ? threadIdx.x < 8 : l < 8) wcnt[TEAM ? threadIdx.x : l] = 0ull;
    __syncwarp();
    __syncthreads();
    mbar_wait(bar, 0);

    const bool belief = a.stop_rule <= 1;
    const int W = (a.stop_rule == 1) ? N : C.M;               // R4
    // gen: channel generated in the warp (fused ber_sim, channel-only); ber: error counting against the
    // transmitted codeword (fused ber_sim, and the decode half of a split one: LLRs and codewords from HBM)
    const bool gen = a.mode == MODE_BER_SIM || a.mode == MODE_CHANNEL;
    const bool ber = a.mode == MODE_BER_SIM || a.mode == MODE_BER_LLR;
    const bool keep_S = a.omega != nullptr && !LBP;           // S only feeds the Omega output (none for LBP)
    const uint32_t key0 = static_cast<uint32_t>(a.seed), key1 = static_cast<uint32_t>(a.seed >> 32);
    unsigned long long bit_err = 0;                           // this lane's share (ber_sim)

    auto syndrome_nz = [&]() -> bool { return w_syndrome_nz<K, TEAM>(ent, row_ptr, hb, mb, Z, tl, Lk); };
    // hard decisions of slot k's variables in row (e0, dc) <- bits (edge e at bit dc-1-e); returns the previous
    auto swap_bits = [&](int r, int e0, int dc, uint32_t bits) -> uint32_t {
        uint32_t prev = 0;
        for (int e = 0; e < dc; ++e) {
            const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + e));
            int8_t* h = hb + A.x + wrap(r + A.y, Z);
            prev = (prev << 1) | static_cast<uint32_t>(*h < 0);
            *h = ((bits >> (dc - 1 - e)) & 1u) ? static_cast<int8_t>(-128) : static_cast<int8_t>(0);
        }
        return prev;
    };

    int rowpar = 0;                                           // team: control-word buffer of the row
    for (;;) {
        long long f = 0;
        if constexpr (TEAM) {
            if (threadIdx.x == 0) *tfrm = static_cast<long long>(atomicAdd(a.queue, 1ull));
            __syncthreads();
            f = *tfrm;
            __syncthreads();                                  // every thread has the index before it is rewritten
        } else {
            if (l == 0) f = static_cast<long long>(atomicAdd(a.queue, 1ull));
            f = __shfl_sync(kFull, f, 0);
        }
        if (f >= a.frames) break;
        // ---- Step 1 (a2-a5): channel LLRs (decode: from HBM, 16 bytes per lane and load;
        // ber_sim: Philox info bits, encoder, BPSK/AWGN in the warp), {Lambda, H} = L + 0, R = 0
        if (!gen) {
            const size_t base = static_cast<size_t>(f) * a.ld;
            if (a.mode == MODE_BER_LLR) {                     // the frame's transmitted codeword (counting)
                const uint32_t* src = a.cw_in + static_cast<size_t>(f) * a.ld_words;
                for (int w = tl; w < C.nwords; w += TL) cw[w] = __ldcs(src + w);
            }
            if (a.mode == MODE_DECODE_I8) {
                const int4* src = reinterpret_cast<const int4*>(a.q + base);
                for (int v16 = tl; 16 * v16 < N; v16 += TL) {
                    const int4 w = __ldcs(src + v16);
                    const uint32_t ws[4] = {static_cast<uint32_t>(w.x), static_cast<uint32_t>(w.y),
                                            static_cast<uint32_t>(w.z), static_cast<uint32_t>(w.w)};
#pragma unroll
                    for (int t = 0; t < 16; ++t) {
                        const int v = 16 * v16 + t;
                        const float x = __fadd_rn(__fmul_rn(static_cast<float>(static_cast<int8_t>(ws[t >> 2] >> (8 * (t & 3)))),
                                                            a.qscale), 0.0f);
                        if (v < N) {
                            lam[v] = x;
                            hb[v] = static_cast<int8_t>(__float_as_uint(x) >> 24);
                        }
                    }
                }
            } else {
                // CBP_LLR_BATCH 128-bit loads in flight per lane before the first use: the frame's LLRs come from
                // HBM (~1 us), and a loop of load -> use exposed that latency once per 512 bytes of the frame
                const float4* src = reinterpret_cast<const float4*>(a.llr + base);
                for (int v0 = tl; 4 * v0 < N; v0 += CBP_LLR_BATCH * TL) {
                    float4 xb[CBP_LLR_BATCH];
#pragma unroll
                    for (int u = 0; u < CBP_LLR_BATCH; ++u)
                        xb[u] = (4 * (v0 + u * TL) < N) ? __ldcs(src + v0 + u * TL) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
                    for (int u = 0; u < CBP_LLR_BATCH; ++u) {
                        const int v4 = v0 + u * TL;
                        const float4 x = xb[u];
                        const float4 x0 = make_float4(__fadd_rn(x.x, 0.0f), __fadd_rn(x.y, 0.0f), __fadd_rn(x.z, 0.0f),
                                                      __fadd_rn(x.w, 0.0f));
                        // H bytes = the sign bytes of the four posteriors, one 32-bit store
                        const uint32_t hw4 = __byte_perm(__byte_perm(__float_as_uint(x0.x), __float_as_uint(x0.y), 0x0073),
                                                         __byte_perm(__float_as_uint(x0.z), __float_as_uint(x0.w), 0x0073), 0x5410);
                        if (4 * v4 + 3 < N) {
                            *reinterpret_cast<float4*>(lam + 4 * v4) = x0;
                            *reinterpret_cast<uint32_t*>(hb + 4 * v4) = hw4;
                        } else if (4 * v4 < N) {
                            const float xs[4] = {x0.x, x0.y, x0.z, x0.w};
#pragma unroll
                            for (int t = 0; t < 4; ++t)
                                if (4 * v4 + t < N) {
                                    lam[4 * v4 + t] = xs[t];
                                    hb[4 * v4 + t] = static_cast<int8_t>(__float_as_uint(xs[t]) >> 24);
                                }
                        }
                    }
                }
            }
        } else {
            const uint64_t gframe = static_cast<uint64_t>(a.frame_begin + f);
            const uint32_t flo = static_cast<uint32_t>(gframe), fhi = static_cast<uint32_t>(gframe >> 32);
            float* Qs = lam;                                  // symbols 1 - 2c in the Lambda words during encoding
            if (a.llr_mode & 2) {                             // all-zero codeword (R23)
                for (int v = tl; v < N; v += TL) Qs[v] = 1.0f;
                for (int w = tl; w < C.nwords; w += TL) cw[w] = 0u;
                tsync();
            } else {
                // (a2) info word w = Philox(w/4, f_lo, f_hi, 0)[w % 4]
                const int nblk = (C.kwords + 3) / 4;
                for (int b = tl; b < nblk; b += TL) {
                    const u32x4 x = w_philox(u32x4{static_cast<uint32_t>(b), flo, fhi, 0u}, key0, key1);
                    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int w = 4 * b + m;
                        if (w < C.kwords) cw[w] = (w == C.kwords - 1 && (C.K & 31)) ? xs[m] & ((1u << (C.K & 31)) - 1u) : xs[m];
                    }
                }
                tsync();
                // (a3) dual-diagonal encoder: systematic symbols, lambda_i[r] of the
                // core rows, p0 = XOR_i lambda_i, the parity chain, the extension
                for (int v = tl; v < C.K; v += TL) Qs[v] = ((cw[v >> 5] >> (v & 31)) & 1u) ? -1.0f : 1.0f;
                tsync();
                // lambda_i[r] = XOR of the info bits of check i Z + r (the sign bits of their symbols: one load
                // and one XOR per bit): each entry read once per row for the K slots (kept in the H bytes, free
                // until the channel step); p0 = XOR over the core rows
                uint32_t p0[K];
#pragma unroll
                for (int k = 0; k < K; ++k) p0[k] = 0u;
                for (int i = 0; i < C.core; ++i) {
                    uint32_t lamb[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) lamb[k] = 0u;
                    for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
                        const int jz = ent[2 * e].x;                  // j Z
                        if (jz >= C.K) continue;                      // a parity column (warp-uniform)
                        const int sft = ent[2 * e + 1].z >> 16;
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            int t = rk[k] + sft;
                            t = (t >= Z) ? t - Z : t;
                            lamb[k] ^= __float_as_uint(Qs[jz + t]);
                        }
                    }
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        if (vk[k]) {
                            hb[i * Z + rk[k]] = static_cast<int8_t>(lamb[k] >> 31);
                            p0[k] ^= lamb[k] >> 31;
                        }
                }
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (vk[k]) Qs[C.kb * Z + rk[k]] = p0[k] ? -1.0f : 1.0f;
                tsync();
#pragma unroll 1
                for (int k = 0; k < K; ++k) {                 // not unrolled: per-frame code
                    const int r = tl + k * Lk;
                    if (!(tl < Lk && r < Z)) continue;
                    uint32_t pprev = 0;
                    for (int t = 1; t < C.core; ++t) {
                        uint32_t pt = static_cast<uint32_t>(hb[(t - 1) * Z + r]);
                        if (t >= 2) pt ^= pprev;
                        const int s0 = pshift[t - 1];
                        if (s0 >= 0) {
                            int rr = r + s0;
                            rr = (rr >= Z) ? rr - Z : rr;
                            pt ^= Qs[C.kb * Z + rr] < 0.0f ? 1u : 0u;
                        }
                        Qs[(C.kb + t) * Z + r] = pt ? -1.0f : 1.0f;
                        pprev = pt;
                    }
                    for (int x = 0; x < mb - C.core; ++x) {
                        const uint32_t pe = info_parity<1>(ent, row_ptr, C.core + x, r, Z, C.K, cw);
                        Qs[(C.kb + C.core + x) * Z + r] = pe ? -1.0f : 1.0f;
                    }
                }
                tsync();
                for (int w = w0; w < C.nwords; w += wstep) {  // transmitted codeword words: one ballot each
                    const int v = 32 * w + l;
                    const unsigned word = __ballot_sync(kFull, v < N && Qs[v] < 0.0f);
                    if (l == 0) cw[w] = word;
                }
                tsync();
            }
            // (a4) y = (1 - 2c) + sigma n, L = (2/sigma^2) y (equ_s4e15, R17); int8 stream
            const int nblk = (N + 3) / 4;
            if (a.mode == MODE_CHANNEL) {
                // channel-only launch (cbp_channel, the first half of a split cbp_ber_sim): no row body shares
                // the instruction cache, so this is the throughput form of the loop below -- two Philox blocks
                // per step, Philox and the four Box-Muller bodies inline (independent chains), and the four
                // LLRs of a block stored from registers with one 128-bit streaming store (rows of ld % 4 == 0
                // floats on a 16-byte aligned buffer; else one by one).  Same counters, same operations per value.
                if (a.llr_out) {
                    float* out = a.llr_out + static_cast<size_t>(f) * a.ld;
                    const bool vec = (a.ld & 3) == 0 && (reinterpret_cast<uintptr_t>(a.llr_out) & 15) == 0;
                    auto emit = [&](int b, const float (&n)[4]) {
                        float Lv[4];
#pragma unroll
                        for (int m = 0; m < 4; ++m) {
                            const int v = min(4 * b + m, N - 1);
                            const float y = __fadd_rn(Qs[v], __fmul_rn(a.sigma, n[m]));
                            Lv[m] = __fmul_rn(a.scale, y);
                            if (a.llr_mode & 1) {
                                float qq = rintf(__fmul_rn(Lv[m], 4.0f));
                                qq = fminf(fmaxf(qq, -127.0f), 127.0f);
                                Lv[m] = __fmul_rn(qq, 0.25f);
                            }
                        }
                        if (vec && 4 * b + 3 < N) {
                            __stcs(reinterpret_cast<float4*>(out + 4 * b), make_float4(Lv[0], Lv[1], Lv[2], Lv[3]));
                        } else {
#pragma unroll
                            for (int m = 0; m < 4; ++m)
                                if (4 * b + m < N) __stcs(out + 4 * b + m, Lv[m]);
                        }
                    };
                    for (int b = tl; b < nblk; b += 2 * TL) {
                        const u32x4 x0 = philox4x32_10(u32x4{static_cast<uint32_t>(b), flo, fhi, 1u}, key0, key1);
                        const u32x4 x1 = philox4x32_10(u32x4{static_cast<uint32_t>(b + TL), flo, fhi, 1u}, key0, key1);
                        float n0[4], n1[4];
                        box_muller(x0.x, x0.y, n0[0], n0[1]);
                        box_muller(x0.z, x0.w, n0[2], n0[3]);
                        box_muller(x1.x, x1.y, n1[0], n1[1]);
                        box_muller(x1.z, x1.w, n1[2], n1[3]);
                        emit(b, n0);
                        if (b + TL < nblk) emit(b + TL, n1);
                    }
                }
            } else
            for (int b = tl; b < nblk; b += TL) {
                const u32x4 x = w_philox(u32x4{static_cast<uint32_t>(b), flo, fhi, 1u}, key0, key1);
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {                 // one Box-Muller body for both pairs (per-frame code)
                  float n[2];
                  box_muller(h ? x.z : x.x, h ? x.w : x.y, n[0], n[1]);
#pragma unroll
                  for (int m = 0; m < 2; ++m) {
                    const int v = 4 * b + 2 * h + m;
                    if (v >= N) break;
                    const float y = __fadd_rn(Qs[v], __fmul_rn(a.sigma, n[m]));
                    float Lv = __fmul_rn(a.scale, y);
                    if (a.llr_mode & 1) {
                        float qq = rintf(__fmul_rn(Lv, 4.0f));
                        qq = fminf(fmaxf(qq, -127.0f), 127.0f);
                        Lv = __fmul_rn(qq, 0.25f);
                    }
                    const float x0 = __fadd_rn(Lv, 0.0f);
                    lam[v] = (a.mode == MODE_CHANNEL) ? Lv : x0;   // channel only: L itself (decoders add the + 0)
                    hb[v] = static_cast<int8_t>(__float_as_uint(x0) >> 24);
                  }
                }
            }
        }
        if (a.mode == MODE_CHANNEL) {                         // channel only: L and the codeword to HBM
            tsync();
            if (a.cw_out) {
                uint32_t* out = a.cw_out + static_cast<size_t>(f) * a.ld_words;
                for (int w = tl; w < a.ld_words; w += TL) __stcs(out + w, w < C.nwords ? cw[w] : 0u);
            }
            tsync();
            continue;
        }
        // R = 0 (equ_s4e17) needs no stores: sweep 1 reads no R word (WCtx::r0), and every word is
        // written in sweep 1 before sweep 2 reads it (a frame that stops in sweep 1 reads none)
        if (keep_S)
            for (int c = tl; c < C.M; c += TL) S[c] = 0.0f;   // equ_s4e16: Omega = inf <=> S = 0
        tsync();

        // ---- Step 2: sweeps over the base rows (checks ascending, R12)
        int consec = 0, fires = 0, sweep = 1;
        float rpre[CBP_DC_REG];                               // CBP_RPRE: R words requested for the next row
        int npre = 0;
        (void)rpre; (void)npre;
        long long ev = 0;
        bool conv = false;
        for (;; ++sweep) {
            bool stop = false;
            for (int i = 0; i < mb; ++i) {
                const int e0 = row_ptr[i], dc = row_ptr[i + 1] - e0;
                // the window can fill in this row: keep what a mid-row stop has to roll back
                WCtx cx{tl, Lk, Z, TEAM ? 32 * warp : 0, belief && W - consec - 1 < Z, keep_S, sweep == 1, lam, hb, pb,
                        Rw + static_cast<size_t>(e0) * K * 32 + l, S + i * Z};
#if CBP_RPRE
                // the row's last slot requests the next row's slot-0 R words (their L2 latency then overlaps the
                // slot's update): from sweep 2 on, register rows only, dc words that lie inside the R array, and
                // not in the fused launch's merged body (whose row may run with a masked edge)
                const int e0n = row_ptr[i + 1 < mb ? i + 1 : 0], dcn = row_ptr[(i + 1 < mb ? i + 1 : 0) + 1] - e0n;
                const bool pf = RG && sweep > 1 && a.mode != MODE_BER_SIM && dc <= CBP_DC_REG && dcn <= CBP_DC_REG &&
                                e0n + dc <= C.nent;
                cx.nrow = pf ? Rw + static_cast<size_t>(e0n) * K * 32 + l : nullptr;
                cx.npre = npre;
                npre = pf ? min(dc, dcn) : 0;
#endif
                WRow<K> ro;
                ro.first_bad = Z;
                ro.last_bad = -1;
                wrow_dispatch<K, ALG, TM, RG>(dc, C.max_dc, a.mode == MODE_BER_SIM, ent, ptab, e0, lane, static_cast<TexH>(C.phi_tex), cx, ro, rpre);
                int first_bad = ro.first_bad, last_bad = ro.last_bad;
                if constexpr (TEAM) {
                    // the team's first / last unclean check of the row (two buffers: a fast warp may write
                    // the next row's values while a slow one still reads these)
                    int* cb = tctl + rowpar * 2 * nwarps;
                    if (l == 0) {
                        cb[warp] = first_bad;
                        cb[nwarps + warp] = last_bad;
                    }
                    __syncthreads();                          // also orders the row's stores before the next row
                    if (belief) {                             // lane w reads warp w's pair, one reduction each
                        first_bad = __reduce_min_sync(kFull, l < nwarps ? cb[l] : first_bad);
                        last_bad = __reduce_max_sync(kFull, l < nwarps ? cb[nwarps + l] : last_bad);
                    }
                    rowpar ^= 1;
                } else {
                    __syncwarp();
                }
                if (!belief) {
                    ev += static_cast<long long>(dc) * Z;
                    continue;
                }
                // ---- Step 2(3): window of clean check updates (R4, R5, R7)
                const int rstar = W - consec - 1;             // the window fills at check i Z + rstar
                if (!(rstar < Z && first_bad > rstar)) {
                    consec = (last_bad < 0) ? consec + Z : Z - 1 - last_bad;
                    ev += static_cast<long long>(dc) * Z;
                    continue;
                }
                // the sequential decoder stops right after check i Z + rstar: slots of later
                // checks show their pre-row decisions and S while the syndrome is verified (R5)
                SlotVals<K, uint32_t> newbits;
#pragma unroll
                for (int k = 0; k < K; ++k) newbits.v[k] = 0;
#pragma unroll 1
                for (int k = 0; k < K; ++k) {                 // not unrolled: per-frame code (see above)
                    const int r = tl + k * Lk;
                    if (tl < Lk && r < Z && r > rstar) {
                        newbits.set(k, swap_bits(r, e0, dc, ro.oldb.get(k)));
                        if (keep_S && !LBP) S[i * Z + r] = ro.sold.get(k);
                    }
                }
                tsync();
                if (!syndrome_nz()) {
                    conv = stop = true;                       // output = state after check i Z + rstar
                    ev += static_cast<long long>(dc) * (rstar + 1);
                    break;
                }
                fires += 1;                                   // failed verification: resume (R5)
                ev += static_cast<long long>(dc) * Z;
                consec = Z - 1 - max(last_bad, rstar);
#pragma unroll 1
                for (int k = 0; k < K; ++k) {
                    const int r = tl + k * Lk;
                    if (tl < Lk && r < Z && r > rstar) {
                        swap_bits(r, e0, dc, newbits.get(k));
                        if (keep_S && !LBP) S[i * Z + r] = ro.snew.get(k);
                    }
                }
                tsync();
            }
            if (stop) break;
            if (a.stop_rule == 2 && !syndrome_nz()) {         // R6: syndrome after every full sweep
                conv = true;
                break;
            }
            if (sweep >= a.max_iter) break;
        }
        // ---- Step 3 (a8): outputs
        const int iters = conv ? sweep : a.max_iter;
        bool synd_zero = conv;
        if (!conv) synd_zero = !syndrome_nz();
        const uint8_t flags = static_cast<uint8_t>((conv ? 1 : 0) | (synd_zero ? 2 : 0) | (fires > 0 ? 4 : 0));
        if (!ber) {
            // packed hard decisions (sign of the H bytes), one ballot per word: lane l reads variable 32 w + l
            uint32_t* out = a.bits + static_cast<size_t>(f) * a.ld_words;
            for (int w = w0; w < a.ld_words; w += wstep) {
                const int v = 32 * w + l;
                const unsigned word = __ballot_sync(kFull, v < N && hb[v] < 0);
                if (l == (w & 31)) out[w] = word;
            }
            if (a.omega) {
                float* om = a.omega + static_cast<size_t>(f) * C.M;
                for (int c = tl; c < C.M; c += TL) {
                    if (LBP) {
                        om[c] = 0.0f;                         // layered BP: no check-beliefs
                        continue;
                    }
                    const float Sv = S[c];
                    const float m = TEXB ? phi32_tex(fabsf(Sv), static_cast<TexH>(C.phi_tex), a.phi_m19, a.phi_one)
                                         : phi32(fabsf(Sv), ptab, a.phi_m19, a.phi_one);   // Omega = sgn phi(S)
                    om[c] = (__float_as_uint(Sv) >> 31) ? -m : m;
                }
            }
            if (tl == 0) {
                a.iters[f] = iters;
                a.flags[f] = flags;
                if (a.ev) a.ev[f] = ev;
            }
        } else {
            // decided vs sent: lane l compares variable 32 w + l, a ballot counts the word's errors
            bool info_err = false, cw_err = false;
            for (int w = w0; w < C.nwords; w += wstep) {
                const int v = 32 * w + l;
                const bool dv = v < N && (static_cast<uint32_t>(hb[v] < 0) != ((cw[w] >> l) & 1u));
                const unsigned d = __ballot_sync(kFull, dv);
                const unsigned ie = __ballot_sync(kFull, dv && v < C.K);
                bit_err += (l == 0) ? __popc(ie) : 0;
                info_err |= ie != 0u;
                cw_err |= d != 0u;
            }
            const bool fe = tany(info_err), ce = tany(cw_err);
            if (tl == 0) {
                wcnt[0] += 1;
                wcnt[2] += fe;
                wcnt[3] += ce;
                wcnt[4] += iters;
                wcnt[5] += ev;
                wcnt[6] += conv ? 0 : 1;
                wcnt[7] += fires;
            }
        }
        tsync();
    }
    if (ber) {
        for (int o = 16; o > 0; o >>= 1) bit_err += __shfl_down_sync(kFull, bit_err, o);
        __syncwarp();
        if (TEAM) {                                           // every warp adds its bit errors, lane 0 of the team the rest
            if (l == 0 && bit_err) atomicAdd(a.counts + 1, bit_err);
            if (tl == 0)
                for (int k = 0; k < 8; ++k)
                    if (k != 1 && wcnt[k]) atomicAdd(a.counts + k, wcnt[k]);
        } else if (l == 0) {
            wcnt[1] = bit_err;
            for (int k = 0; k < 8; ++k)
                if (wcnt[k]) atomicAdd(a.counts + k, wcnt[k]);
        }
    }
}

// ---------------------------------------------------------------- launch of one instantiation
template <int K, bool RG, int MAXT, int ALG, int TM, bool TEAM = false>
static int wlaunch_t(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st)
{
    auto k = cbp_warp_kernel<K, RG, MAXT, ALG, TM, TEAM>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
    k<<<grid, g.threads, g.smem_bytes, st>>>(a);
    return static_cast<int>(cudaGetLastError());
}

template <int K, bool RG, int MAXT, int ALG, int TM, bool TEAM = false>
static int wocc_t(const Geometry& g, int* out)
{
    auto k = cbp_warp_kernel<K, RG, MAXT, ALG, TM, TEAM>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
    return static_cast<int>(cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, g.threads, g.smem_bytes));
}

// K = 1: up to CBP_WARPK1_MAXT threads (512: 128 registers); K = 2..4: CBP_WARPK_MAXT (384: 170 registers)
template <int ALG>
static int wdispatch(const Geometry& g, const KernelArgs* a, int grid, cudaStream_t st, int* occ)
{
    const bool rg = g.r_global != 0;
    const int tm = g.tex2;                    // 0 C2B through TEX, 1 both, 2 none
    if (g.multi) {                            // team frames (one per CTA), K = 1 or 2
#define CBP_WG(KK)                                                                                            \
        if (g.kslots == KK)                                                                                   \
            return occ ? wocc_t<KK, true, CBP_WARPT_MAXT, ALG, 0, true>(g, occ)                                 \
                       : wlaunch_t<KK, true, CBP_WARPT_MAXT, ALG, 0, true>(*a, g, grid, st);
        CBP_WG(1)
        CBP_WG(2)
#undef CBP_WG
        return static_cast<int>(cudaErrorInvalidConfiguration);
    }
#define CBP_WT(KK, RGV, MT)                                                                                   \
    if (tm == 1) return occ ? wocc_t<KK, RGV, MT, ALG, 1>(g, occ) : wlaunch_t<KK, RGV, MT, ALG, 1>(*a, g, grid, st); \
    if (tm == 2) return occ ? wocc_t<KK, RGV, MT, ALG, 2>(g, occ) : wlaunch_t<KK, RGV, MT, ALG, 2>(*a, g, grid, st); \
    return occ ? wocc_t<KK, RGV, MT, ALG, 0>(g, occ) : wlaunch_t<KK, RGV, MT, ALG, 0>(*a, g, grid, st);
#define CBP_W(KK, MT)                 \
    if (g.kslots == KK) {             \
        if (rg) { CBP_WT(KK, true, MT) } \
        CBP_WT(KK, false, MT)         \
    }
    CBP_W(1, CBP_WARPK1_MAXT)
    CBP_W(2, CBP_WARPK_MAXT)
    CBP_W(3, CBP_WARPK_MAXT)
    CBP_W(4, CBP_WARPK_MAXT)
#undef CBP_WT
#undef CBP_W
    return static_cast<int>(cudaErrorInvalidConfiguration);
}

}  // namespace cbp
