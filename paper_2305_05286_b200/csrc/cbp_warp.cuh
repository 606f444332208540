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
// Per-warp state in shared memory: QP[N] = {Lambda'_v, H_v} (cbp_kernel.cuh, producer-side
// layout), S[M] (check records with sign = Omega < 0: Omega output and rollback only), the
// transmitted codeword (ber_sim), and R (here, or in a global slot per warp: RG) laid out as
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
// One slot's check of a base row with DC edges (producer-side update, cbp_kernel.cuh): the
// row's schedule entries, all loads, phase 1, phase 2.  rrow: this lane's R word of (row entry 0,
// this slot); the word of edge e is rrow[e K 32].  A slot beyond Z (vk false) computes on a
// valid address and stores nothing but its private R words.  The slots of a row run in a loop
// (not unrolled): the unrolled K x DC bodies overflowed the 32 KB L1.5 instruction cache
// (ncu: no_instruction stalls 2.3 per issue, issue active 37 %).
template <int DC, int K, int ALG>
__device__ __forceinline__ void wrow(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0, int rq,
                                     bool vk, const Lane& L, TexH tex, char* qp, float* rrow, RowAcc<1>& acc)
{
    constexpr bool LBP = ALG == 2;
    int aqp[DC];
    float vs[DC][2], ro[DC][1], q[DC][1], ph[DC][1];
    acc.Ssum[0] = 0.0f;
    acc.negw[0] = acc.flipw[0] = acc.oldbits[0] = 0u;
#pragma unroll
    for (int e = 0; e < DC; ++e) {
        const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + e));
        aqp[e] = A.x + wrap(rq + A.y, L.ZQ);
        CBP_CHECK(aqp[e] >= 0 && aqp[e] + 8 <= L.slot_bytes);
        ldf<2>(qp, aqp[e], vs[e]);                                 // {Lambda_v, H_v}
        ro[e][0] = rrow[e * K * 32];                               // R_{c->v}
        if constexpr (LBP) vs[e][1] = vs[e][0];
    }
#pragma unroll
    for (int e = 0; e < DC; ++e) cbp_phase1<1>(vs[e], ro[e], q[e], ph[e], ptab, L, tex, acc);
#pragma unroll
    for (int e = 0; e < DC; ++e) {
        float rn[1], lamn[1];
        cbp_phase2<1>(acc, q[e], ph[e], rn, lamn, ptab, L, tex);
        if (vk) {
            const float st[2] = {lamn[0], LBP ? lamn[0] : vs[e][0]};
            stf<2>(qp, aqp[e], st);
        }
        rrow[e * K * 32] = rn[0];                                  // equ_s4e22 commit of R_{c->v}
    }
}

// rows longer than CBP_DC_REG: two passes over the edges, parking {Q^new, Phi | sign of the
// decision} in the variable's slot between the phases (as cbp_row_park)
template <int K, int ALG>
__device__ __forceinline__ void wrow_park(const int4* __restrict__ ent, const float4* __restrict__ ptab, int e0, int dc,
                                          int rq, bool vk, const Lane& L, char* qp, float* rrow, RowAcc<1>& acc)
{
    constexpr bool LBP = ALG == 2;
    acc.Ssum[0] = 0.0f;
    acc.negw[0] = acc.flipw[0] = acc.oldbits[0] = 0u;
    for (int e = 0; e < dc; ++e) {
        const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + e));
        const int a = A.x + wrap(rq + A.y, L.ZQ);
        float v[2], ro[1] = {rrow[e * K * 32]}, q[1], ph[1];
        ldf<2>(qp, a, v);
        if (LBP) v[1] = v[0];
        cbp_phase1<1, false>(v, ro, q, ph, ptab, L, 0, acc);
        if (vk) {
            const float st[2] = {q[0], __uint_as_float(__float_as_uint(ph[0]) | (__float_as_uint(v[0]) & kSign))};
            stf<2>(qp, a, st);
        }
    }
    for (int e = 0; e < dc; ++e) {
        const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + e));
        const int a = A.x + wrap(rq + A.y, L.ZQ);
        float v[2], rn[1], lamn[1];
        ldf<2>(qp, a, v);
        const float q[1] = {v[0]}, ph[1] = {fabsf(v[1])};
        cbp_phase2<1, false>(acc, q, ph, rn, lamn, ptab, L, 0);
        if (vk) {
            const float st[2] = {lamn[0], LBP ? lamn[0] : v[1]};
            stf<2>(qp, a, st);
        }
        rrow[e * K * 32] = rn[0];
    }
}

template <int K, int ALG>
__device__ __forceinline__ void wrow_dispatch(int dc, const int4* __restrict__ ent, const float4* __restrict__ ptab,
                                              int e0, int rq, bool vk, const Lane& L, TexH tex, char* qp, float* rrow,
                                              RowAcc<1>& acc)
{
    switch (dc) {
#if CBP_DC_REG >= 1
    case 1: wrow<1, K, ALG>(ent, ptab, e0, rq, vk, L, tex, qp, rrow, acc); break;
    case 2: wrow<2, K, ALG>(ent, ptab, e0, rq, vk, L, tex, qp, rrow, acc); break;
    case 3: wrow<3, K, ALG>(ent, ptab, e0, rq, vk, L, tex, qp, rrow, acc); break;
    case 4: wrow<4, K, ALG>(ent, ptab, e0, rq, vk, L, tex, qp, rrow, acc); break;
    case 5: wrow<5, K, ALG>(ent, ptab, e0, rq, vk, L, tex, qp, rrow, acc); break;
    case 6: wrow<6, K, ALG>(ent, ptab, e0, rq, vk, L, tex, qp, rrow, acc); break;
#endif
#if CBP_DC_REG >= 8
    case 7: wrow<7, K, ALG>(ent, ptab, e0, rq, vk, L, tex, qp, rrow, acc); break;
    case 8: wrow<8, K, ALG>(ent, ptab, e0, rq, vk, L, tex, qp, rrow, acc); break;
#endif
    default: wrow_park<K, ALG>(ent, ptab, e0, dc, rq, vk, L, qp, rrow, acc); break;
    }
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

// ---------------------------------------------------------------- the kernel
// RG: R in a global slot per warp (else in the warp's shared state).  Modes: decode (fp32 /
// int8 LLRs from HBM) and the fused ber_sim; cbp_channel runs on cbp_kernel.
template <int K, bool RG, int MAXT, int ALG>
__global__ void __launch_bounds__(MAXT, 1) cbp_warp_kernel(const __grid_constant__ KernelArgs a)
{
    constexpr bool LBP = ALG == 2;
    extern __shared__ __align__(16) uint32_t smem[];
    const DevCode& C = a.code;
    const int Z = C.Z, mb = C.mb, N = C.N;

    // ---- a1: stage the phi table and the schedule entries with the bulk-copy engine (one
    // elected thread arms an mbarrier with the byte count, every thread waits on its phase)
    float4* ptab = reinterpret_cast<float4*>(smem);
    int4* ent = reinterpret_cast<int4*>(smem + 4 * kPhiSegs);
    int32_t* row_ptr = reinterpret_cast<int32_t*>(smem + 4 * kPhiSegs + 8 * C.nent);
    int16_t* pshift = reinterpret_cast<int16_t*>(row_ptr + mb + 1);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.table_words - 4);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        const uint32_t tb = 16u * kPhiSegs, eb = 32u * static_cast<uint32_t>(C.nent);
        mbar_expect_tx(bar, tb + eb);
        bulk_g2s(ptab, C.phi_tab, tb, bar);
        bulk_g2s(ent, a.ent_dev, eb, bar);
    }
    for (int k = threadIdx.x; k <= mb; k += blockDim.x) row_ptr[k] = a.row_ptr[k];
    for (int k = threadIdx.x; k < mb; k += blockDim.x) pshift[k] = a.pshift[k];

    const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int Lk = a.lanes;                                   // L: lanes with check slots
    int rk[K], rq[K];
    bool vk[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int r = l + k * Lk;
        vk[k] = l < Lk && r < Z;
        rk[k] = vk[k] ? r : Z - 1;                            // invalid slots compute on check Z - 1, store nothing
        rq[k] = rk[k] * 8;
    }
    // per-warp shared state: counters (8 x u64) | QP [2N] | S [M] | cw [nwords] | R (if !RG)
    unsigned long long* wcnt =
        reinterpret_cast<unsigned long long*>(smem + a.table_words + static_cast<size_t>(warp) * a.slot_words);
    float* st0 = reinterpret_cast<float*>(wcnt + 8);
    char* qp = reinterpret_cast<char*>(st0);
    float* S = st0 + 2 * N;
    uint32_t* cw = reinterpret_cast<uint32_t*>(S + C.M);
    const int rwords = C.nent * K * 32;
    float* Rw = RG ? a.rstate + (static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + warp) * a.r_words
                   : reinterpret_cast<float*>(cw + ((C.nwords + 3) & ~3));
    const Lane lane{0, 0, 0, Z * 8, 0, 0, 4 * a.slot_words, 0, a.phi_m19, a.phi_one};
    if (l < 8) wcnt[l] = 0ull;
    __syncthreads();
    mbar_wait(bar, 0);

    const bool belief = a.stop_rule <= 1;
    const int W = (a.stop_rule == 1) ? N : C.M;               // R4
    const bool ber = a.mode == MODE_BER_SIM;
    const bool keep_S = a.omega != nullptr;                   // S only feeds the Omega output
    const uint32_t key0 = static_cast<uint32_t>(a.seed), key1 = static_cast<uint32_t>(a.seed >> 32);
    unsigned long long bit_err = 0;                           // this lane's share (ber_sim)

    // parity of this lane's valid checks over all rows from the hard decisions (sign of H)
    auto syndrome_nz = [&]() -> bool {
        uint32_t nz = 0;
        for (int i = 0; i < mb; ++i) {
            uint32_t par = 0;                                 // bit k: parity of check i Z + r_k
            for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
                const int2 A = *reinterpret_cast<const int2*>(ent + 2 * e);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int at = A.x + wrap(rq[k] + A.y, Z * 8) + 4;
                    par ^= vk[k] ? (__float_as_uint(*reinterpret_cast<const float*>(qp + at)) >> 31) << k : 0u;
                }
            }
            nz |= par;
        }
        return __any_sync(kFull, nz != 0u);
    };
    // hard decisions of slot k's variables in row (e0, dc) <- bits (edge e at bit dc-1-e); returns the previous
    auto swap_bits = [&](int rqk, int e0, int dc, uint32_t bits) -> uint32_t {
        uint32_t prev = 0;
        for (int e = 0; e < dc; ++e) {
            const int2 A = *reinterpret_cast<const int2*>(ent + 2 * (e0 + e));
            float* h = reinterpret_cast<float*>(qp + A.x + wrap(rqk + A.y, Z * 8) + 4);
            const uint32_t w = __float_as_uint(*h);
            prev = (prev << 1) | (w >> 31);
            *h = __uint_as_float((w & ~kSign) | (((bits >> (dc - 1 - e)) & 1u) << 31));
        }
        return prev;
    };

    for (;;) {
        long long f = 0;
        if (l == 0) f = static_cast<long long>(atomicAdd(a.queue, 1ull));
        f = __shfl_sync(kFull, f, 0);
        if (f >= a.frames) break;
        // ---- Step 1 (a2-a5): channel LLRs (decode: from HBM, 16 bytes per lane and load;
        // ber_sim: Philox info bits, encoder, BPSK/AWGN in the warp), {Lambda, H} = L + 0, R = 0
        if (!ber) {
            const size_t base = static_cast<size_t>(f) * a.ld;
            if (a.mode == MODE_DECODE_I8) {
                const int4* src = reinterpret_cast<const int4*>(a.q + base);
                for (int v16 = l; 16 * v16 < N; v16 += 32) {
                    const int4 w = __ldcs(src + v16);
                    const uint32_t ws[4] = {static_cast<uint32_t>(w.x), static_cast<uint32_t>(w.y),
                                            static_cast<uint32_t>(w.z), static_cast<uint32_t>(w.w)};
#pragma unroll
                    for (int t = 0; t < 16; ++t) {
                        const int v = 16 * v16 + t;
                        const float x = __fadd_rn(__fmul_rn(static_cast<float>(static_cast<int8_t>(ws[t >> 2] >> (8 * (t & 3)))),
                                                            a.qscale), 0.0f);
                        if (v < N) *reinterpret_cast<float2*>(qp + 8 * v) = make_float2(x, x);
                    }
                }
            } else {
                const float4* src = reinterpret_cast<const float4*>(a.llr + base);
                for (int v4 = l; 4 * v4 < N; v4 += 32) {
                    const float4 x = __ldcs(src + v4);
                    const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float x0 = __fadd_rn(xs[t], 0.0f);
                        if (4 * v4 + t < N) *reinterpret_cast<float2*>(qp + 8 * (4 * v4 + t)) = make_float2(x0, x0);
                    }
                }
            }
        } else {
            const uint64_t gframe = static_cast<uint64_t>(a.frame_begin + f);
            const uint32_t flo = static_cast<uint32_t>(gframe), fhi = static_cast<uint32_t>(gframe >> 32);
            float* Qs = st0;                                  // symbols 1 - 2c in the Lambda words during encoding
            if (a.llr_mode & 2) {                             // all-zero codeword (R23)
                for (int v = l; v < N; v += 32) Qs[2 * v] = 1.0f;
                for (int w = l; w < C.nwords; w += 32) cw[w] = 0u;
                __syncwarp();
            } else {
                // (a2) info word w = Philox(w/4, f_lo, f_hi, 0)[w % 4]
                const int nblk = (C.kwords + 3) / 4;
                for (int b = l; b < nblk; b += 32) {
                    const u32x4 x = philox4x32_10(u32x4{static_cast<uint32_t>(b), flo, fhi, 0u}, key0, key1);
                    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int w = 4 * b + m;
                        if (w < C.kwords) cw[w] = (w == C.kwords - 1 && (C.K & 31)) ? xs[m] & ((1u << (C.K & 31)) - 1u) : xs[m];
                    }
                }
                __syncwarp();
                // (a3) dual-diagonal encoder: systematic symbols, lambda_i[r] of the
                // core rows (kept in S), p0 = XOR_i lambda_i, the parity chain, the extension
                for (int v = l; v < C.K; v += 32) Qs[2 * v] = ((cw[v >> 5] >> (v & 31)) & 1u) ? -1.0f : 1.0f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (!vk[k]) continue;
                    uint32_t p0 = 0;
                    for (int i = 0; i < C.core; ++i) {
                        const uint32_t lam = info_parity<8>(ent, row_ptr, i, rk[k], Z, C.K, cw);
                        S[i * Z + rk[k]] = __uint_as_float(lam);
                        p0 ^= lam;
                    }
                    Qs[2 * (C.kb * Z + rk[k])] = p0 ? -1.0f : 1.0f;
                }
                __syncwarp();
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (!vk[k]) continue;
                    const int r = rk[k];
                    uint32_t pprev = 0;
                    for (int t = 1; t < C.core; ++t) {
                        uint32_t pt = __float_as_uint(S[(t - 1) * Z + r]);
                        if (t >= 2) pt ^= pprev;
                        const int s0 = pshift[t - 1];
                        if (s0 >= 0) {
                            int rr = r + s0;
                            rr = (rr >= Z) ? rr - Z : rr;
                            pt ^= Qs[2 * (C.kb * Z + rr)] < 0.0f ? 1u : 0u;
                        }
                        Qs[2 * ((C.kb + t) * Z + r)] = pt ? -1.0f : 1.0f;
                        pprev = pt;
                    }
                    for (int x = 0; x < mb - C.core; ++x) {
                        const uint32_t pe = info_parity<8>(ent, row_ptr, C.core + x, r, Z, C.K, cw);
                        Qs[2 * ((C.kb + C.core + x) * Z + r)] = pe ? -1.0f : 1.0f;
                    }
                }
                __syncwarp();
                for (int w = l; w < C.nwords; w += 32) {      // transmitted codeword words
                    uint32_t word = 0;
                    for (int b = 0; b < 32; ++b) {
                        const int v = 32 * w + b;
                        if (v < N && Qs[2 * v] < 0.0f) word |= 1u << b;
                    }
                    cw[w] = word;
                }
                __syncwarp();
            }
            // (a4) y = (1 - 2c) + sigma n, L = (2/sigma^2) y (equ_s4e15, R17); int8 stream
            const int nblk = (N + 3) / 4;
            for (int b = l; b < nblk; b += 32) {
                const u32x4 x = philox4x32_10(u32x4{static_cast<uint32_t>(b), flo, fhi, 1u}, key0, key1);
                float n[4];
                box_muller(x.x, x.y, n[0], n[1]);
                box_muller(x.z, x.w, n[2], n[3]);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int v = 4 * b + m;
                    if (v >= N) break;
                    const float y = __fadd_rn(Qs[2 * v], __fmul_rn(a.sigma, n[m]));
                    float Lv = __fmul_rn(a.scale, y);
                    if (a.llr_mode & 1) {
                        float qq = rintf(__fmul_rn(Lv, 4.0f));
                        qq = fminf(fmaxf(qq, -127.0f), 127.0f);
                        Lv = __fmul_rn(qq, 0.25f);
                    }
                    const float x0 = __fadd_rn(Lv, 0.0f);
                    *reinterpret_cast<float2*>(qp + 8 * v) = make_float2(x0, x0);
                }
            }
        }
        for (int w = l; w < rwords; w += 32) Rw[w] = 0.0f;    // equ_s4e17
        if (keep_S)
            for (int c = l; c < C.M; c += 32) S[c] = 0.0f;    // equ_s4e16: Omega = inf <=> S = 0
        __syncwarp();

        // ---- Step 2: sweeps over the base rows (checks ascending, R12)
        int consec = 0, fires = 0, sweep = 1;
        long long ev = 0;
        bool conv = false;
        for (;; ++sweep) {
            bool stop = false;
            for (int i = 0; i < mb; ++i) {
                const int e0 = row_ptr[i], dc = row_ptr[i + 1] - e0;
                // the window can fill in this row: keep what a mid-row stop has to roll back
                const bool fire_possible = belief && W - consec - 1 < Z;
                const bool keep = keep_S && fire_possible;
                SlotVals<K, uint32_t> oldb;
                SlotVals<K, float> sold, snew;
                int first_bad = Z, last_bad = -1;
#pragma unroll 1
                for (int k = 0; k < K; ++k) {
                    const int r = l + k * Lk;
                    const bool v = l < Lk && r < Z;
                    const int rr = v ? r : Z - 1;
                    if (keep) sold.set(k, S[i * Z + rr]);
                    RowAcc<1> acc;
                    wrow_dispatch<K, ALG>(dc, ent, ptab, e0, rr * 8, v, lane, static_cast<TexH>(C.phi_tex), qp,
                                          Rw + static_cast<size_t>(e0) * K * 32 + k * 32 + l, acc);
                    const float sn = __uint_as_float(__float_as_uint(acc.Ssum[0]) | (acc.negw[0] & kSign));
                    if (keep_S && !LBP && v) S[i * Z + rr] = sn;                     // equ_s4e23
                    if (fire_possible) {
                        oldb.set(k, acc.oldbits[0]);
                        snew.set(k, sn);
                    }
                    // Step 2(3) flags of this slot's check (equ_s4e2, equ_s4e24)
                    const unsigned m = __ballot_sync(kFull, v && (((acc.negw[0] | acc.flipw[0]) & kSign) != 0u));
                    if (m) {
                        first_bad = min(first_bad, k * Lk + __ffs(m) - 1);
                        last_bad = max(last_bad, k * Lk + 31 - __clz(m));
                    }
                }
                __syncwarp();
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
                for (int k = 0; k < K; ++k) {
                    newbits.v[k] = 0;
                    if (vk[k] && rk[k] > rstar) {
                        newbits.v[k] = swap_bits(rq[k], e0, dc, oldb.v[k]);
                        if (keep_S && !LBP) S[i * Z + rk[k]] = sold.v[k];
                    }
                }
                __syncwarp();
                if (!syndrome_nz()) {
                    conv = stop = true;                       // output = state after check i Z + rstar
                    ev += static_cast<long long>(dc) * (rstar + 1);
                    break;
                }
                fires += 1;                                   // failed verification: resume (R5)
                ev += static_cast<long long>(dc) * Z;
                consec = Z - 1 - max(last_bad, rstar);
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (vk[k] && rk[k] > rstar) {
                        swap_bits(rq[k], e0, dc, newbits.v[k]);
                        if (keep_S && !LBP) S[i * Z + rk[k]] = snew.v[k];
                    }
                __syncwarp();
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
            uint32_t* out = a.bits + static_cast<size_t>(f) * a.ld_words;
            for (int w = l; w < a.ld_words; w += 32) {
                uint32_t word = 0;
                if (w < C.nwords)
                    for (int b = 0; b < 32; ++b) {
                        const int v = 32 * w + b;
                        if (v < N) word |= (__float_as_uint(st0[2 * v + 1]) >> 31) << b;
                    }
                out[w] = word;
            }
            if (a.omega) {
                float* om = a.omega + static_cast<size_t>(f) * C.M;
                for (int c = l; c < C.M; c += 32) {
                    const float Sv = S[c];
                    const float m = LBP ? 0.0f : phi32(fabsf(Sv), ptab, a.phi_m19, a.phi_one);   // Omega = sgn phi(S)
                    om[c] = LBP ? 0.0f : ((__float_as_uint(Sv) >> 31) ? -m : m);
                }
            }
            if (l == 0) {
                a.iters[f] = iters;
                a.flags[f] = flags;
                if (a.ev) a.ev[f] = ev;
            }
        } else {
            bool info_err = false, cw_err = false;
            for (int w = l; w < C.nwords; w += 32) {
                uint32_t word = 0;
                for (int b = 0; b < 32; ++b) {
                    const int v = 32 * w + b;
                    if (v < N) word |= (__float_as_uint(st0[2 * v + 1]) >> 31) << b;
                }
                const uint32_t d = word ^ cw[w];
                uint32_t im = 0;
                if (32 * w + 32 <= C.K) im = kFull;
                else if (32 * w < C.K) im = (1u << (C.K - 32 * w)) - 1u;
                bit_err += __popc(d & im);
                info_err |= (d & im) != 0u;
                cw_err |= d != 0u;
            }
            const bool fe = __any_sync(kFull, info_err), ce = __any_sync(kFull, cw_err);
            if (l == 0) {
                wcnt[0] += 1;
                wcnt[2] += fe;
                wcnt[3] += ce;
                wcnt[4] += iters;
                wcnt[5] += ev;
                wcnt[6] += conv ? 0 : 1;
                wcnt[7] += fires;
            }
        }
        __syncwarp();
    }
    if (ber) {
        for (int o = 16; o > 0; o >>= 1) bit_err += __shfl_down_sync(kFull, bit_err, o);
        __syncwarp();
        if (l == 0) {
            wcnt[1] = bit_err;
            for (int k = 0; k < 8; ++k)
                if (wcnt[k]) atomicAdd(a.counts + k, wcnt[k]);
        }
    }
}

// ---------------------------------------------------------------- launch of one instantiation
template <int K, bool RG, int MAXT, int ALG>
static int wlaunch_t(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st)
{
    auto k = cbp_warp_kernel<K, RG, MAXT, ALG>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
    k<<<grid, g.threads, g.smem_bytes, st>>>(a);
    return static_cast<int>(cudaGetLastError());
}

template <int K, bool RG, int MAXT, int ALG>
static int wocc_t(const Geometry& g, int* out)
{
    auto k = cbp_warp_kernel<K, RG, MAXT, ALG>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
    return static_cast<int>(cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, g.threads, g.smem_bytes));
}

// K = 1: up to 512 threads (128 registers); K = 2..4: up to 384 threads (170 registers)
template <int ALG>
static int wdispatch(const Geometry& g, const KernelArgs* a, int grid, cudaStream_t st, int* occ)
{
    const bool rg = g.r_global != 0;
#define CBP_W(KK, MT)                                                                                     \
    if (g.kslots == KK)                                                                                   \
        return occ ? (rg ? wocc_t<KK, true, MT, ALG>(g, occ) : wocc_t<KK, false, MT, ALG>(g, occ))        \
                   : (rg ? wlaunch_t<KK, true, MT, ALG>(*a, g, grid, st) : wlaunch_t<KK, false, MT, ALG>(*a, g, grid, st));
    CBP_W(1, 512)
    CBP_W(2, 384)
    CBP_W(3, 384)
    CBP_W(4, 384)
#undef CBP_W
    return static_cast<int>(cudaErrorInvalidConfiguration);
}

}  // namespace cbp
