// cbp_kernels.cu -- sm_100a kernels of check-belief propagation decoding.
//
// One persistent kernel serves cbp_decode, cbp_decode_i8, cbp_channel and
// cbp_ber_sim.  Mapping: a CTA is a "team" of F frame slots;
// each slot owns Z lanes, lane r processes lifted check i*Z + r of the current
// base row i.  The Z lifted checks of one base row touch disjoint variables
// (each block is a permutation), so processing them in parallel is bit-identical
// to the paper's sequential check order (reading R12).  Per-frame state
// (Q, Phi|hard bit, R, S|sign of Omega) lives in shared memory; the code's
// schedule tables are staged once per CTA.
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

struct SlotPtrs {
    float* Q;       // [N] latest V2C message Q_{v->c*}
    float* P;       // [N] Phi_v = phi(|Q_v|) with the sign bit = hard decision x_v
    float* R;       // [E] C2V messages, slot b*Z + r = edge of (check i*Z+r, entry b)
    float* S;       // [M] phi-domain check-belief sum, sign bit = (Omega_c < 0)
    uint32_t* cw;   // [nwords] transmitted codeword (ber_sim) / scratch
};

// ---------------------------------------------------------------- team helpers
// A CTA holds several independent teams.  !MULTI: a team is one warp holding F
// frame slots of Zp lanes; MULTI: a team is TW warps holding one frame.  Teams
// synchronise with their own named barrier (id 1 + team index).
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
    // OR over the team (a synchronisation point)
    __device__ __forceinline__ bool team_any(bool pred) const
    {
        if (MULTI) return named_bar_or(1 + tidx, nthreads, pred);
        return __any_sync(kFull, pred) != 0;
    }
    // OR over the lanes of this slot (a synchronisation point)
    __device__ __forceinline__ bool slot_any(bool pred) const
    {
        if (MULTI) return team_any(pred);
        return (__ballot_sync(kFull, pred) & slot_mask) != 0u;
    }
    // kept for readability at call sites that mean "any slot of this team"
    __device__ __forceinline__ bool cta_any(bool pred) const { return team_any(pred); }
};

// ---------------------------------------------------------------- per-row edge chain
struct RowOut {
    float Snew, Sold;
    uint32_t oldbits, newbits;
    bool ok;
};

// U consecutive edges of lane r's check (entries e0+k0 .. e0+k0+U-1, U <= remaining).
// Loads first, then U independent B2V phi chains, commits/V2C, U independent C2B
// phi chains, and the ordered S accumulation (reading R12).
template <int U>
__device__ __forceinline__ void edge_chunk(const int4* __restrict__ ent, int e0, int k0, int r, int Z, bool sweep1,
                                           const SlotPtrs& s, float& Ssum, uint32_t& negf, uint32_t& flip,
                                           uint32_t& oldbits, uint32_t& newbits)
{
    int v[U], wsl[U];
    float q[U], p[U], scj[U], rold[U], Rn[U];
    bool fst[U], slf[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int4 e = ent[e0 + k0 + u];
        const int vb = e.x & 0xffff, psb = static_cast<int>(static_cast<uint32_t>(e.x) >> 16);
        const int sh = e.y & 0x7ff, ds = (e.y >> 11) & 0x7ff;
        fst[u] = sweep1 && ((e.y >> 22) & 1);
        slf[u] = (e.y >> 23) & 1;
        int t = r + sh;
        t = (t >= Z) ? t - Z : t;
        int rp = r + ds;
        rp = (rp >= Z) ? rp - Z : rp;
        v[u] = vb + t;
        wsl[u] = e.w + rp;
        q[u] = s.Q[v[u]];
        p[u] = s.P[v[u]];
        scj[u] = s.S[psb + rp];
        rold[u] = s.R[e.z + r];
    }
    // B2V (equ_s4e18): R^new_{cj->v} = sgn(Omega_cj) sgn(Q) phi(|phi(|Omega_cj|) - phi(|Q|)|), phi(|Omega|) = S (R11)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const float D = fabsf(__fsub_rn(fabsf(scj[u]), fabsf(p[u])));
        const float mag = phi32(D);
        const bool sg = ((__float_as_uint(scj[u]) >> 31) != 0u) != (q[u] < 0.0f);
        Rn[u] = fst[u] ? 0.0f : (sg ? -mag : mag);
    }
    float qn[U];
    uint32_t bit[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (!fst[u]) s.R[wsl[u]] = Rn[u];                 // equ_s4e22 commit of R_{cj->v} (R2), before the read (R3)
        const float ro = slf[u] ? Rn[u] : rold[u];
        const float lam = __fadd_rn(q[u], Rn[u]);         // equ_s4e20
        qn[u] = __fsub_rn(lam, ro);                       // equ_s4e19 (R15)
        bit[u] = lam < 0.0f ? 1u : 0u;                    // equ_s2e7
        const uint32_t ob = __float_as_uint(p[u]) >> 31;
        flip |= bit[u] ^ ob;                              // equ_s4e24 (R7)
        oldbits |= ob << (k0 + u);
        newbits |= bit[u] << (k0 + u);
    }
    float ph[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ph[u] = phi32(fabsf(qn[u]));   // C2B (equ_s4e21, App. equ_ae4)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        Ssum = __fadd_rn(Ssum, ph[u]);
        negf ^= qn[u] < 0.0f ? 1u : 0u;
        s.Q[v[u]] = qn[u];
        s.P[v[u]] = bit[u] ? -ph[u] : ph[u];
    }
}

__device__ __forceinline__ RowOut process_row(const int4* __restrict__ ent, int e0, int dc, int r, int Z, int sidx,
                                              bool sweep1, const SlotPtrs& s)
{
    float Ssum = 0.0f;
    uint32_t negf = 0, flip = 0, oldbits = 0, newbits = 0;
    const float Sold = s.S[sidx];
    int k0 = 0;
    for (; k0 + 4 <= dc; k0 += 4) edge_chunk<4>(ent, e0, k0, r, Z, sweep1, s, Ssum, negf, flip, oldbits, newbits);
    for (; k0 < dc; ++k0) edge_chunk<1>(ent, e0, k0, r, Z, sweep1, s, Ssum, negf, flip, oldbits, newbits);
    const float Snew = negf ? -Ssum : Ssum;
    s.S[sidx] = Snew;                                     // equ_s4e23
    RowOut o;
    o.Snew = Snew;
    o.Sold = Sold;
    o.oldbits = oldbits;
    o.newbits = newbits;
    o.ok = (negf == 0u) && (flip == 0u);                  // equ_s4e2 and equ_s4e24 for this check
    return o;
}

// rewrite the hard-decision bits (sign of P) of lane r's variables in row (e0, dc)
__device__ __forceinline__ void put_row_bits(const int4* __restrict__ ent, int e0, int dc, int r, int Z, uint32_t bits,
                                             const SlotPtrs& s)
{
    for (int k = 0; k < dc; ++k) {
        const int4 e = ent[e0 + k];
        int t = r + (e.y & 0x7ff);
        t = (t >= Z) ? t - Z : t;
        const int v = (e.x & 0xffff) + t;
        const float a = fabsf(s.P[v]);
        s.P[v] = ((bits >> k) & 1u) ? -a : a;
    }
}

// parity of lane r's checks over all rows, from the hard bits (sign of P)
__device__ __forceinline__ bool lane_syndrome(const int4* __restrict__ ent, const int32_t* row_ptr, int mb, int r,
                                              int Z, const SlotPtrs& s)
{
    uint32_t nz = 0;
    for (int i = 0; i < mb; ++i) {
        uint32_t par = 0;
        for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            const int4 e = ent[k];
            int t = r + (e.y & 0x7ff);
            t = (t >= Z) ? t - Z : t;
            par ^= __float_as_uint(s.P[(e.x & 0xffff) + t]) >> 31;
        }
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
        const int4 e = ent[k];
        const int vb = e.x & 0xffff;
        if (vb >= K) continue;
        int t = r + (e.y & 0x7ff);
        t = (t >= Z) ? t - Z : t;
        const int v = vb + t;
        par ^= (cw[v >> 5] >> (v & 31)) & 1u;
    }
    return par;
}

// ---------------------------------------------------------------- channel (a2-a4)
template <bool MULTI>
__device__ void channel_frame(const KernelArgs& a, const Team<MULTI>& tm, bool fresh, int64_t gframe,
                              const int4* ent, const int32_t* row_ptr, const int16_t* pshift, const SlotPtrs& s)
{
    const DevCode& C = a.code;
    const int Z = C.Z, r = tm.r;
    const bool on = fresh && tm.lane_on;
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
    // (a3) systematic part and p0 = XOR of the core rows' lambda
    if (on) {
        for (int v = r; v < C.K; v += Z) s.Q[v] = ((s.cw[v >> 5] >> (v & 31)) & 1u) ? -1.0f : 1.0f;
        uint32_t p0 = 0;
        for (int i = 0; i < C.core; ++i) p0 ^= info_parity(ent, row_ptr, i, r, Z, C.K, s.cw);
        s.Q[C.kb * Z + r] = p0 ? -1.0f : 1.0f;
    }
    tm.sync();
    // p_t = lambda_{t-1} ^ p_{t-1} ^ P^{s0} p0 (row t-1), extension p = lambda
    if (on) {
        uint32_t pprev = 0;
        for (int t = 1; t < C.core; ++t) {
            uint32_t pt = info_parity(ent, row_ptr, t - 1, r, Z, C.K, s.cw);
            if (t >= 2) pt ^= pprev;
            const int s0 = pshift[t - 1];
            if (s0 >= 0) {
                int rr = r + s0;
                rr = (rr >= Z) ? rr - Z : rr;
                pt ^= s.Q[C.kb * Z + rr] < 0.0f ? 1u : 0u;
            }
            s.Q[(C.kb + t) * Z + r] = pt ? -1.0f : 1.0f;
            pprev = pt;
        }
        for (int k = 0; k < C.mb - C.core; ++k) {
            const uint32_t pe = info_parity(ent, row_ptr, C.core + k, r, Z, C.K, s.cw);
            s.Q[(C.kb + C.core + k) * Z + r] = pe ? -1.0f : 1.0f;
        }
    }
    tm.sync();
    // transmitted codeword words
    if (on) {
        for (int w = r; w < C.nwords; w += Z) {
            uint32_t word = 0;
            for (int b = 0; b < 32; ++b) {
                const int v = 32 * w + b;
                if (v < C.N && s.Q[v] < 0.0f) word |= 1u << b;
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
                const float y = __fadd_rn(s.Q[v], __fmul_rn(a.sigma, n[m]));
                float L = __fmul_rn(a.scale, y);
                if (a.llr_mode == 1) {
                    float qq = rintf(__fmul_rn(L, 4.0f));
                    qq = fminf(fmaxf(qq, -127.0f), 127.0f);
                    L = __fmul_rn(qq, 0.25f);
                }
                s.Q[v] = L;
                s.P[v] = L < 0.0f ? -0.0f : 0.0f;
            }
        }
        for (int e = r; e < C.E; e += Z) s.R[e] = 0.0f;
        for (int c = r; c < C.M; c += Z) s.S[c] = 0.0f;
    }
    tm.sync();
}

// ---------------------------------------------------------------- the kernel
template <bool MULTI, bool SMEM, int MAXT>
__global__ void __launch_bounds__(MAXT) cbp_kernel(const KernelArgs a)
{
    extern __shared__ __align__(16) uint32_t smem[];
    const DevCode& C = a.code;
    const int Z = C.Z, mb = C.mb;

    // ---- stage the schedule tables (a1)
    int4* ent = reinterpret_cast<int4*>(smem);
    int32_t* row_ptr = reinterpret_cast<int32_t*>(smem + 4 * C.nent);
    int16_t* pshift = reinterpret_cast<int16_t*>(row_ptr + mb + 1);
    for (int k = threadIdx.x; k < C.nent; k += blockDim.x) ent[k] = C.ent[k];
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
    uint32_t* ctl = smem + a.table_words + tm.tidx * kCtlTeamWords;
    long long* ctl64 = reinterpret_cast<long long*>(ctl + 64);

    const int nteams = blockDim.x / a.team_threads;
    float* sbase = SMEM ? reinterpret_cast<float*>(smem + a.table_words + nteams * kCtlTeamWords)
                        : a.gstate + static_cast<size_t>(blockIdx.x) * nteams * a.F * a.slot_words;
    SlotPtrs s;
    s.Q = sbase + static_cast<size_t>(tm.tidx * a.F + (tm.slot < a.F ? tm.slot : 0)) * a.slot_words;
    s.P = s.Q + C.N;
    s.R = s.P + C.N;
    s.S = s.R + C.E;
    s.cw = reinterpret_cast<uint32_t*>(s.S + C.M);
    __syncthreads();

    const bool belief = a.stop_rule <= 1;
    const int64_t W = (a.stop_rule == 1) ? C.N : C.M;        // R4
    const bool decoding = a.mode != MODE_CHANNEL;

    // per-slot control (uniform over the slot's lanes)
    bool active = false, exhausted = (tm.slot >= a.F), conv = false;
    int64_t fidx = -1, ev = 0, consec = 0;
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
                ev = 0;
                consec = 0;
                sweep = 1;
                fires = 0;
            } else {
                exhausted = true;
            }
        }
        // ---- Step 1: initialisation (a4/a5)
        if (a.mode == MODE_BER_SIM || a.mode == MODE_CHANNEL) {
            if (tm.cta_any(fresh))
                channel_frame<MULTI>(a, tm, fresh, a.frame_begin + fidx, ent, row_ptr, pshift, s);
        } else {
            if (fresh && tm.lane_on) {
                const size_t base = static_cast<size_t>(fidx) * a.ld;
                for (int v = r; v < C.N; v += Z) {
                    const float L = (a.mode == MODE_DECODE_I8) ? __fmul_rn(static_cast<float>(a.q[base + v]), a.qscale)
                                                               : a.llr[base + v];
                    s.Q[v] = L;                                   // equ_s4e15
                    s.P[v] = L < 0.0f ? -0.0f : 0.0f;             // hard bit from L (R7)
                }
                for (int e = r; e < C.E; e += Z) s.R[e] = 0.0f;   // equ_s4e17
                for (int c = r; c < C.M; c += Z) s.S[c] = 0.0f;   // equ_s4e16: Omega = inf <=> S = 0
            }
            tm.sync();
        }
        if (!tm.cta_any(active)) break;

        bool done = false;
        if (decoding) {
            // ---- Step 2: one sweep over the base rows (checks in ascending order)
            for (int i = 0; i < mb; ++i) {
                const bool live = active && !conv;
                if (!tm.cta_any(live)) break;
                const int e0 = row_ptr[i], dc = row_ptr[i + 1] - e0;
                RowOut ro;
                ro.ok = true;
                ro.oldbits = ro.newbits = 0;
                ro.Snew = ro.Sold = 0.0f;
                if (live && tm.lane_on) ro = process_row(ent, e0, dc, r, Z, i * Z + r, sweep == 1, s);
                // ---- Step 2(3): stopping criterion, counted per check update (R4, R5)
                int first_bad = Z, last_bad = -1;
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
                int64_t rstar = 0;
                if (live && belief) {
                    rstar = W - consec - 1;           // the window fills at check i*Z + rstar
                    fire = rstar < Z && first_bad > rstar;
                    if (!fire) consec = (last_bad < 0) ? consec + Z : (Z - 1 - last_bad);
                }
                if (live && !fire) ev += static_cast<int64_t>(dc) * Z;
                if (tm.cta_any(fire)) {
                    // the sequential decoder stops right after check i*Z + rstar: lanes r > rstar
                    // show their pre-row hard bits and S while the syndrome is verified (R5)
                    const bool back = fire && tm.lane_on && r > rstar;
                    if (back) {
                        put_row_bits(ent, e0, dc, r, Z, ro.oldbits, s);
                        s.S[i * Z + r] = ro.Sold;
                    }
                    tm.sync();
                    const bool nz = tm.slot_any(fire && tm.lane_on && lane_syndrome(ent, row_ptr, mb, r, Z, s));
                    if (fire) {
                        if (!nz) {
                            conv = true;             // converged: output = state after check i*Z + rstar
                            ev += static_cast<int64_t>(dc) * (rstar + 1);
                        } else {
                            fires += 1;              // undetected fire: resume (R5)
                            ev += static_cast<int64_t>(dc) * Z;
                            consec = Z - 1 - max(static_cast<int64_t>(last_bad), rstar);
                            if (back) {
                                put_row_bits(ent, e0, dc, r, Z, ro.newbits, s);
                                s.S[i * Z + r] = ro.Snew;
                            }
                        }
                    }
                    tm.sync();
                }
            }
            // ---- end of sweep
            const bool want_syn = active && !conv && a.stop_rule == 2;
            if (tm.cta_any(want_syn)) {
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
        if (tm.cta_any(done)) {
            tm.sync();
            bool synd_zero = conv;
            const bool need_syn = done && !conv && decoding;
            if (tm.cta_any(need_syn)) {
                const bool nz = tm.slot_any(need_syn && tm.lane_on && lane_syndrome(ent, row_ptr, mb, r, Z, s));
                if (need_syn) synd_zero = !nz;
            }
            const int iters = conv ? sweep : a.max_iter;
            const uint8_t flags = static_cast<uint8_t>((conv ? 1 : 0) | (synd_zero ? 2 : 0) | (fires > 0 ? 4 : 0));
            if (a.mode == MODE_DECODE_F32 || a.mode == MODE_DECODE_I8) {
                if (done && tm.lane_on) {
                    uint32_t* out = a.bits + static_cast<size_t>(fidx) * a.ld_words;
                    for (int w = r; w < a.ld_words; w += Z) {
                        uint32_t word = 0;
                        if (w < C.nwords)
                            for (int b = 0; b < 32; ++b) {
                                const int v = 32 * w + b;
                                if (v < C.N) word |= (__float_as_uint(s.P[v]) >> 31) << b;
                            }
                        out[w] = word;
                    }
                    if (a.omega) {
                        float* om = a.omega + static_cast<size_t>(fidx) * C.M;
                        for (int c = r; c < C.M; c += Z) {
                            const float Sv = s.S[c];
                            const float m = phi32(fabsf(Sv));
                            om[c] = (__float_as_uint(Sv) >> 31) ? -m : m;
                        }
                    }
                    if (r == 0) {
                        a.iters[fidx] = iters;
                        a.flags[fidx] = flags;
                        if (a.ev) a.ev[fidx] = ev;
                    }
                }
            } else if (a.mode == MODE_BER_SIM) {
                bool info_err = false, cw_err = false;
                if (done && tm.lane_on) {
                    for (int w = r; w < C.nwords; w += Z) {
                        uint32_t word = 0;
                        for (int b = 0; b < 32; ++b) {
                            const int v = 32 * w + b;
                            if (v < C.N) word |= (__float_as_uint(s.P[v]) >> 31) << b;
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
                    cnt[5] += ev;
                    cnt[6] += conv ? 0 : 1;
                    cnt[7] += fires;
                }
            } else {  // MODE_CHANNEL
                if (done && tm.lane_on) {
                    if (a.llr_out) {
                        float* out = a.llr_out + static_cast<size_t>(fidx) * a.ld;
                        for (int v = r; v < C.N; v += Z) out[v] = s.Q[v];
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
__global__ void contract_eval_kernel(int fn, const float* __restrict__ x, float* __restrict__ y, int64_t n)
{
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float v = x[k];
        float out;
        if (fn == 0) {
            out = phi32(v);
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

int launch_contract_eval(int fn, const float* x, float* y, int64_t n, void* stream)
{
    if (n <= 0) return 0;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    contract_eval_kernel<<<static_cast<int>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(fn, x, y, n);
    return static_cast<int>(cudaGetLastError());
}

// ---------------------------------------------------------------- host-side launch
template <bool MULTI, bool SMEM, int MAXT>
static int launch_t(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st)
{
    auto k = cbp_kernel<MULTI, SMEM, MAXT>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
    k<<<grid, g.threads, g.smem_bytes, st>>>(a);
    return static_cast<int>(cudaGetLastError());
}

template <bool MULTI, bool SMEM, int MAXT>
static int occ_t(const Geometry& g, int* out)
{
    auto k = cbp_kernel<MULTI, SMEM, MAXT>;
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
