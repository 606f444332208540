// cbp_oracle.cpp -- plain single-threaded CPU ORACLE of CBP decoding.
//
// TEST INFRASTRUCTURE ONLY (see cbp_oracle.h).  Written from PAPER.md and the
// readings R1-R21 of DESIGN.md §2; no code is shared with the CUDA path.
// Build: g++ -std=c++17 -O2 -ffp-contract=off (no -ffast-math).
//
// "Parity unpinned" functions: none -- every function below is pinned by a
// -m "not gpu" test (tests/test_oracle_*.py), see DESIGN.md §6.
#include "cbp_oracle.h"
#include "contract32.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

struct or_code {
    int32_t mb = 0, nb = 0, Z = 0, N = 0, M = 0, K = 0, kb = 0;
    int64_t E = 0;
    std::vector<int16_t> base;
    std::vector<int32_t> chk_ptr;   // M+1, edges of check c are [chk_ptr[c], chk_ptr[c+1])
    std::vector<int32_t> e_var;     // E
    std::vector<int32_t> e_chk;     // E
    // encoder: dense GF(2) inverse of the core block (encoder)
    bool can_encode = false;
    int32_t core = 0, n_core = 0, core_words = 0;
    std::vector<uint64_t> core_inv; // n_core rows x core_words
};

// ---------------------------------------------------------------- code graph
// G = (V, C, E), N(v), N(c).  QC expansion of the base matrix.
or_code* oracle_code_create(const int16_t* base, int32_t mb, int32_t nb, int32_t Z)
{
    if (!base || mb < 1 || nb <= mb || Z < 1) return nullptr;
    or_code* c = new or_code();
    c->mb = mb; c->nb = nb; c->Z = Z; c->kb = nb - mb;
    c->N = nb * Z; c->M = mb * Z; c->K = c->N - c->M;
    c->base.assign(base, base + (size_t)mb * nb);
    c->chk_ptr.assign(c->M + 1, 0);
    for (int32_t i = 0; i < mb; ++i)
        for (int32_t r = 0; r < Z; ++r) {
            const int32_t ck = i * Z + r;
            for (int32_t j = 0; j < nb; ++j) {
                const int32_t s = base[i * nb + j];
                if (s < 0) continue;
                if (s >= Z) { delete c; return nullptr; }
                c->e_var.push_back(j * Z + (r + s) % Z);
                c->e_chk.push_back(ck);
            }
            c->chk_ptr[ck + 1] = (int32_t)c->e_var.size();
        }
    c->E = (int64_t)c->e_var.size();

    // --- encoder set-up.  Parity columns kb..nb-1 must be a core of columns with
    // weight >= 2 living in rows < core, followed by degree-1 extension columns.
    std::vector<int32_t> colw(nb, 0);
    for (int32_t i = 0; i < mb; ++i)
        for (int32_t j = 0; j < nb; ++j) colw[j] += base[i * nb + j] >= 0;
    int32_t core = 0;
    while (c->kb + core < nb && colw[c->kb + core] >= 2) ++core;
    bool ok = core >= 1;
    for (int32_t t = 0; ok && t < core; ++t)
        for (int32_t i = core; i < mb; ++i) ok = ok && base[i * nb + c->kb + t] < 0;
    for (int32_t k = 0; ok && c->kb + core + k < nb; ++k) {
        const int32_t j = c->kb + core + k;
        ok = colw[j] == 1 && core + k < mb && base[(core + k) * nb + j] >= 0;
    }
    ok = ok && (nb - c->kb - core) == (mb - core);
    if (ok) {
        // Gauss-Jordan over GF(2) on A (core checks x core unknowns) | I
        const int32_t n = core * Z, w = (n + 63) / 64;
        std::vector<uint64_t> A((size_t)n * w, 0), I((size_t)n * w, 0);
        const int32_t v0 = c->kb * Z;
        for (int32_t ck = 0; ck < n; ++ck) {
            for (int32_t e = c->chk_ptr[ck]; e < c->chk_ptr[ck + 1]; ++e) {
                const int32_t v = c->e_var[e];
                if (v >= v0 && v < v0 + n) A[(size_t)ck * w + (v - v0) / 64] ^= 1ull << ((v - v0) % 64);
            }
            I[(size_t)ck * w + ck / 64] |= 1ull << (ck % 64);
        }
        for (int32_t col = 0; ok && col < n; ++col) {
            int32_t piv = -1;
            for (int32_t r = col; r < n; ++r)
                if (A[(size_t)r * w + col / 64] >> (col % 64) & 1) { piv = r; break; }
            if (piv < 0) { ok = false; break; }
            if (piv != col)
                for (int32_t k = 0; k < w; ++k) {
                    std::swap(A[(size_t)piv * w + k], A[(size_t)col * w + k]);
                    std::swap(I[(size_t)piv * w + k], I[(size_t)col * w + k]);
                }
            for (int32_t r = 0; r < n; ++r) {
                if (r == col || !(A[(size_t)r * w + col / 64] >> (col % 64) & 1)) continue;
                for (int32_t k = 0; k < w; ++k) {
                    A[(size_t)r * w + k] ^= A[(size_t)col * w + k];
                    I[(size_t)r * w + k] ^= I[(size_t)col * w + k];
                }
            }
        }
        if (ok) {
            c->core = core; c->n_core = n; c->core_words = w;
            c->core_inv.swap(I);   // row u of A^{-1}: unknown u = <row u, rhs>
        }
    }
    c->can_encode = ok;
    return c;
}

void oracle_code_destroy(or_code* c) { delete c; }

void oracle_code_dims(const or_code* c, int32_t* N, int32_t* K, int32_t* M, int64_t* E)
{
    if (N) *N = c->N;
    if (K) *K = c->K;
    if (M) *M = c->M;
    if (E) *E = c->E;
}

void oracle_code_edges(const or_code* c, int32_t* chk, int32_t* var)
{
    for (int64_t e = 0; e < c->E; ++e) { chk[e] = c->e_chk[e]; var[e] = c->e_var[e]; }
}

static inline int get_bit(const uint32_t* w, int64_t v) { return (int)(w[v >> 5] >> (v & 31) & 1u); }
static inline void put_bit(uint32_t* w, int64_t v, int b)
{
    if (b) w[v >> 5] |= 1u << (v & 31);
    else w[v >> 5] &= ~(1u << (v & 31));
}

int oracle_syndrome_weight(const or_code* c, const uint32_t* cw)
{
    int wgt = 0;
    for (int32_t ck = 0; ck < c->M; ++ck) {
        int p = 0;
        for (int32_t e = c->chk_ptr[ck]; e < c->chk_ptr[ck + 1]; ++e) p ^= get_bit(cw, c->e_var[e]);
        wgt += p;
    }
    return wgt;
}

// ---------------------------------------------------------------- encoder
// Systematic c = [s | p], H c = 0: core parity by the precomputed GF(2)
// inverse, each degree-1 extension bit = parity of the rest of its check.
int oracle_encode(const or_code* c, const uint32_t* info, uint32_t* cw)
{
    if (!c->can_encode) return 1;
    const int32_t nw = (c->N + 31) / 32;
    std::fill(cw, cw + nw, 0u);
    for (int32_t v = 0; v < c->K; ++v) put_bit(cw, v, get_bit(info, v));
    const int32_t n = c->n_core, w = c->core_words, Z = c->Z;
    std::vector<uint64_t> rhs(w, 0);
    for (int32_t ck = 0; ck < n; ++ck) {
        int p = 0;
        for (int32_t e = c->chk_ptr[ck]; e < c->chk_ptr[ck + 1]; ++e)
            if (c->e_var[e] < c->K) p ^= get_bit(cw, c->e_var[e]);
        if (p) rhs[ck / 64] |= 1ull << (ck % 64);
    }
    for (int32_t u = 0; u < n; ++u) {
        uint64_t acc = 0;
        for (int32_t k = 0; k < w; ++k) acc ^= c->core_inv[(size_t)u * w + k] & rhs[k];
        put_bit(cw, (int64_t)c->kb * Z + u, __builtin_popcountll(acc) & 1);
    }
    const int32_t v_ext0 = (c->kb + c->core) * Z;
    for (int32_t ck = c->core * Z; ck < c->M; ++ck) {
        int p = 0, ext = -1;
        for (int32_t e = c->chk_ptr[ck]; e < c->chk_ptr[ck + 1]; ++e) {
            const int32_t v = c->e_var[e];
            if (v >= v_ext0) ext = v;
            else p ^= get_bit(cw, v);
        }
        if (ext < 0) return 2;
        put_bit(cw, ext, p);
    }
    return 0;
}

// ---------------------------------------------------------------- Philox + channel
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): 10 rounds of
// (hi0^c1^k0, lo1, hi1^c3^k1, lo0) with multipliers D2511F53 / CD9E8D57 and
// Weyl key increments 9E3779B9 / BB67AE85.
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// normal n_v of a frame: block k4 = v/4 of purpose 1; pair (x0,x1) -> n_{4k4}, n_{4k4+1},
// pair (x2,x3) -> n_{4k4+2}, n_{4k4+3}; Box-Muller with u1 = ((a>>8)+1) 2^-24,
// theta = 2 pi (b>>8) 2^-24, radius sqrt(-2 ln u1).
static float normal_of(uint64_t seed, uint64_t frame, int32_t v)
{
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const uint32_t ctr[4] = {(uint32_t)(v / 4), (uint32_t)frame, (uint32_t)(frame >> 32), 1u};
    uint32_t x[4];
    oracle_philox4x32_10(ctr, key, x);
    const int pair = (v % 4) / 2;
    const uint32_t a = x[2 * pair], b = x[2 * pair + 1];
    const float u1 = (float)((a >> 8) + 1u) * 0x1p-24f;
    const float l = oracle_ln32(u1);
    const float t = -2.0f * l;
    const float rad = std::sqrt(t);
    float s, co;
    oracle_sincos_quarter32(b >> 8, &s, &co);
    return (v % 2 == 0) ? rad * co : rad * s;
}

void oracle_normals(uint64_t seed, uint64_t frame, int32_t n, float* out)
{
    for (int32_t v = 0; v < n; ++v) out[v] = normal_of(seed, frame, v);
}

int oracle_channel(const or_code* c, double ebn0_db, uint64_t seed, int64_t frame_begin, int64_t frames,
                   int32_t llr_mode, float* llr, int64_t ld, uint32_t* cw_out, int64_t ld_words)
{
    if (frames < 0 || (llr && ld < c->N) || (cw_out && ld_words < (c->N + 31) / 32)) return 1;
    if (llr_mode < 0 || llr_mode > 3) return 1;                      // bit0 int8, bit1 all-zero codeword
    const bool tx_zero = (llr_mode & 2) != 0;                        // reading R23
    if (!tx_zero && !c->can_encode) return 1;
    // sigma^2 = 1 / (2 R 10^(Eb/N0 / 10)), R = K/N, L = 2 y / sigma^2 (reading R17)
    const double R = (double)c->K / (double)c->N;
    const double sigma2 = 1.0 / (2.0 * R * std::pow(10.0, ebn0_db / 10.0));
    const float sigf = (float)std::sqrt(sigma2);
    const float scalef = (float)(2.0 / sigma2);
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const int32_t nw = (c->N + 31) / 32, kw = (c->K + 31) / 32;
    std::vector<uint32_t> info(kw), cw(nw);
    for (int64_t f = 0; f < frames; ++f) {
        const uint64_t g = (uint64_t)(frame_begin + f);
        if (tx_zero) {
            std::fill(cw.begin(), cw.end(), 0u);                     // the all-zero codeword, no info bits drawn
        } else {
        for (int32_t w = 0; w < kw; ++w) {
            const uint32_t ctr[4] = {(uint32_t)(w / 4), (uint32_t)g, (uint32_t)(g >> 32), 0u};
            uint32_t x[4];
            oracle_philox4x32_10(ctr, key, x);
            info[w] = x[w % 4];
        }
        if (c->K % 32) info[kw - 1] &= (1u << (c->K % 32)) - 1u;
        oracle_encode(c, info.data(), cw.data());
        }
        if (cw_out) std::copy(cw.begin(), cw.end(), cw_out + f * ld_words);
        if (!llr) continue;
        for (int32_t v = 0; v < c->N; ++v) {
            const float sym = get_bit(cw.data(), v) ? -1.0f : 1.0f;     // BPSK 0 -> +1
            const float n = normal_of(seed, g, v);
            const float y = sym + sigf * n;
            float L = scalef * y;
            if (llr_mode & 1) {                                          // int8 stream (BJ config 5)
                float q = std::rint(L * 4.0f);
                q = std::fmin(std::fmax(q, -127.0f), 127.0f);
                L = q * 0.25f;
            }
            llr[f * ld + v] = L;
        }
    }
    return 0;
}

// ---------------------------------------------------------------- CBP
// phi of PAPER.md l.142 (equ_s2e5): fp32 = arithmetic contract; fp64 =
// log1p(2/expm1(x)), algebraically -log(tanh(x/2)) but without the
// cancellation of tanh -> 1; both clamped to [PHI_LO, PHI_HI] (reading R9).
template <class T> static inline T phi_t(T x);
template <> inline float phi_t<float>(float x) { return oracle_phi32(x); }
template <> inline double phi_t<double>(double x)
{
    x = std::fmin(std::fmax(x, (double)OR_PHI_LO), (double)OR_PHI_HI);
    const double r = std::log1p(2.0 / std::expm1(x));
    return std::fmin(std::fmax(r, (double)OR_PHI_LO), (double)OR_PHI_HI);
}

static int syndrome_weight_bits(const or_code* c, const std::vector<uint8_t>& xhat)
{
    int wgt = 0;
    for (int32_t ck = 0; ck < c->M; ++ck) {
        int p = 0;
        for (int32_t e = c->chk_ptr[ck]; e < c->chk_ptr[ck + 1]; ++e) p ^= xhat[c->e_var[e]];
        wgt += p;
    }
    return wgt;
}

struct FrameResult {
    int32_t iters = 0;
    uint8_t flags = 0;
    int64_t edge_visits = 0;
    int32_t fires = 0;
};

// Test-only instrumentation of cbp_frame (no effect on the arithmetic): `window` > 0 replaces
// the stop window W of reading R4 (a small W forces mid-row fires and failed verifications
// for the stop-rule pin); `lam` / `qn` receive Lambda^new / Q^new of every edge visit, at
// [(sweep-1) E + e] when `per_sweep`, else at [e] (overwritten every sweep).
struct Instr {
    int64_t window = 0;
    double* lam = nullptr;
    double* qn = nullptr;
    bool per_sweep = false;
};

// One frame of CBP, §IV-C.  `literal` selects the literal psi+
// recursion (equ_s4e5/equ_s4e6) instead of the phi-domain accumulator (R11).
template <class T>
static FrameResult cbp_frame(const or_code* c, const float* L, const or_opts* o, bool literal,
                             std::vector<uint8_t>& xhat, std::vector<T>* S_out, std::vector<uint8_t>* neg_out,
                             const Instr& ins = Instr())
{
    const int32_t N = c->N, M = c->M;
    const int32_t NONE = -1;
    // ---- Step 1: initialization (l.402-422)
    std::vector<T> Q(N);                         // Q_{v->c*} = L_v            (equ_s4e15)
    std::vector<T> R(c->E, (T)0);                // R_{c->v} = 0               (equ_s4e17)
    std::vector<T> S(M, (T)0);                   // Omega_c = inf  <=>  S_c = 0 (equ_s4e16, R9)
    std::vector<uint8_t> neg(M, 0);              // sign of Omega_c
    std::vector<T> Om(M, std::numeric_limits<T>::infinity());   // literal variant only
    std::vector<int32_t> latest(N, NONE);        // edge id of (latest check, v); none yet (R1)
    xhat.assign(N, 0);
    for (int32_t v = 0; v < N; ++v) {
        Q[v] = (T)L[v];
        xhat[v] = Q[v] < (T)0;                   // decision rule equ_s2e7
    }
    int64_t W = (o->stop_rule == OR_STOP_BELIEF_N) ? (int64_t)N : (int64_t)M;   // R4
    if (ins.window > 0) W = ins.window;
    const bool belief = o->stop_rule == OR_STOP_BELIEF_M || o->stop_rule == OR_STOP_BELIEF_N;
    int64_t consec = 0;
    FrameResult res;
    bool converged = false;
    // ---- Step 2 (Alg. 1 lines 5-21)
    for (int32_t sweep = 1; sweep <= o->max_iter && !converged; ++sweep) {
        for (int32_t ci = 0; ci < M && !converged; ++ci) {
            T Ssum = (T)0;                       // phi-domain C2B accumulator, Omega^(-1) = inf
            T om = std::numeric_limits<T>::infinity();
            uint8_t ng = 0;
            bool flip = false;
            for (int32_t e = c->chk_ptr[ci]; e < c->chk_ptr[ci + 1]; ++e) {
                const int32_t v = c->e_var[e];
                // (1a) latest updated neighbouring check c_j of v_a (l.430)
                const int32_t ej = latest[v];
                // (1b) B2V, equ_s4e18: R^new_{cj->v} = psi-(Omega_cj, Q_{v->c*}),
                //      psi-(x,y) = sgn x sgn y phi(|phi(|x|) - phi(|y|)|)  (equ_s4e13, App. equ_ae8)
                T Rn = (T)0;
                if (ej != NONE) {
                    const int32_t cj = c->e_chk[ej];
                    T mag;
                    bool sg;
                    if (!literal) {
                        mag = phi_t<T>(std::fabs(S[cj] - phi_t<T>(std::fabs(Q[v]))));   // phi(|Omega|) = S (R11)
                        sg = (neg[cj] != 0) != (Q[v] < (T)0);
                    } else {
                        mag = phi_t<T>(std::fabs(phi_t<T>(std::fabs(Om[cj])) - phi_t<T>(std::fabs(Q[v]))));
                        sg = (Om[cj] < (T)0) != (Q[v] < (T)0);
                    }
                    Rn = sg ? -mag : mag;
                    R[ej] = Rn;                  // (1e) equ_s4e22 commit of R_{cj->v}, before the read (R2, R3)
                }
                // (1c) V2C, equ_s4e20 / equ_s4e19 (rounding order R15)
                const T lam = Q[v] + Rn;
                const T qn = lam - R[e];
                if (ins.lam) {
                    const int64_t at = (ins.per_sweep ? (int64_t)(sweep - 1) * c->E : 0) + e;
                    ins.lam[at] = (double)lam;
                    if (ins.qn) ins.qn[at] = (double)qn;
                }
                const uint8_t bit = lam < (T)0;  // hard decision, equ_s2e7 (l.450)
                if (bit != xhat[v]) flip = true; // equ_s4e24 (R7)
                xhat[v] = bit;
                // (1d) C2B, equ_s4e21
                if (!literal) {
                    Ssum += phi_t<T>(std::fabs(qn));   // App. equ_ae4: phi^-1(Y_{n+1}) = phi^-1(Y_n) + phi(x_n)
                    ng ^= (uint8_t)(qn < (T)0);
                } else {
                    // psi+(x, y) = sgn x sgn y phi(phi(|x|) + phi(|y|)) (equ_s4e6), phi(inf) = 0
                    const T px = std::isinf(om) ? (T)0 : phi_t<T>(std::fabs(om));
                    const T m = phi_t<T>(px + phi_t<T>(std::fabs(qn)));
                    const bool s = ((om < (T)0) != (qn < (T)0));
                    om = s ? -m : m;
                }
                // (1e) equ_s4e22: Q_{v->c*} <- Q^new
                Q[v] = qn;
                latest[v] = e;
            }
            // (2) equ_s4e23: Omega_ci <- Omega^new
            if (!literal) { S[ci] = Ssum; neg[ci] = ng; }
            else { Om[ci] = om; ng = om < (T)0; }
            res.edge_visits += c->chk_ptr[ci + 1] - c->chk_ptr[ci];
            // (3) stopping criterion (l.478-485, equ_s4e2 + equ_s4e24; readings R4, R5)
            if (belief) {
                const bool ok = (ng == 0) && !flip;
                consec = ok ? consec + 1 : 0;
                if (consec >= W) {
                    if (syndrome_weight_bits(c, xhat) == 0) {
                        converged = true;
                        res.iters = sweep;
                    } else {
                        res.fires += 1;
                        consec = 0;
                    }
                }
            }
        }
        if (!converged && o->stop_rule == OR_STOP_SYNDROME && syndrome_weight_bits(c, xhat) == 0) {
            converged = true;
            res.iters = sweep;
        }
    }
    if (!converged) res.iters = o->max_iter;
    // ---- Step 3: output the hard decisions of the V2C phase (l.487, R14)
    res.flags = (uint8_t)((converged ? 1 : 0) | (syndrome_weight_bits(c, xhat) == 0 ? 2 : 0) |
                          (res.fires > 0 ? 4 : 0));
    if (S_out) {
        S_out->resize(M);
        for (int32_t ck = 0; ck < M; ++ck) (*S_out)[ck] = literal ? Om[ck] : S[ck];
    }
    if (neg_out) *neg_out = neg;
    return res;
}

// ---------------------------------------------------------------- normalized min-sum CBP
// B2V equ_s4e18xx  R^new = (Omega^min_cj == Q) ? Omega^submin_cj : Omega^min_cj,
// C2B equ_s4e21xx  (Omega^min, Omega^submin) updated with alpha * Q^new.  Completion (reading
// R20): magnitudes compared after scaling, m = fl(alpha |Q^new|) < min (strict); the minimum's
// owner is tracked by edge instead of comparing values; signs as in psi- (equ_s4e13):
// sgn(R^new) = sgn(Omega_cj) sgn(Q), sgn(Omega_c) = prod sgn(Q^new).  Omega^(-1) = (inf, inf).
// Everything else (Step 1, V2C, commit, stop rule) is the CBP schedule of cbp_frame.
static FrameResult minsum_frame(const or_code* c, const float* L, const or_opts* o, std::vector<uint8_t>& xhat,
                                std::vector<float>* om_out, const Instr& ins = Instr())
{
    const int32_t N = c->N, M = c->M;
    const int32_t NONE = -1;
    const float INF = std::numeric_limits<float>::infinity();
    const float alpha = o->alpha;
    std::vector<float> Q(N), R(c->E, 0.0f);
    std::vector<float> mn(M, INF), smn(M, INF);
    std::vector<int32_t> own(M, NONE), latest(N, NONE);
    std::vector<uint8_t> neg(M, 0);
    xhat.assign(N, 0);
    for (int32_t v = 0; v < N; ++v) {
        Q[v] = L[v];
        xhat[v] = Q[v] < 0.0f;
    }
    int64_t W = (o->stop_rule == OR_STOP_BELIEF_N) ? (int64_t)N : (int64_t)M;
    if (ins.window > 0) W = ins.window;
    const bool belief = o->stop_rule == OR_STOP_BELIEF_M || o->stop_rule == OR_STOP_BELIEF_N;
    int64_t consec = 0;
    FrameResult res;
    bool converged = false;
    for (int32_t sweep = 1; sweep <= o->max_iter && !converged; ++sweep) {
        for (int32_t ci = 0; ci < M && !converged; ++ci) {
            float m1 = INF, m2 = INF;
            int32_t ow = NONE;
            uint8_t ng = 0;
            bool flip = false;
            for (int32_t e = c->chk_ptr[ci]; e < c->chk_ptr[ci + 1]; ++e) {
                const int32_t v = c->e_var[e];
                const int32_t ej = latest[v];
                float Rn = 0.0f;
                if (ej != NONE) {                                 // B2V, equ_s4e18xx
                    const int32_t cj = c->e_chk[ej];
                    const float mag = (own[cj] == ej) ? smn[cj] : mn[cj];
                    const bool sg = (neg[cj] != 0) != (Q[v] < 0.0f);
                    Rn = sg ? -mag : mag;
                    R[ej] = Rn;                                   // commit before the read (R2, R3)
                }
                const float lam = Q[v] + Rn;                      // V2C, equ_s4e20 / equ_s4e19
                const float qn = lam - R[e];
                if (ins.lam) {
                    const int64_t at = (ins.per_sweep ? (int64_t)(sweep - 1) * c->E : 0) + e;
                    ins.lam[at] = (double)lam;
                    if (ins.qn) ins.qn[at] = (double)qn;
                }
                const uint8_t bit = lam < 0.0f;
                if (bit != xhat[v]) flip = true;
                xhat[v] = bit;
                const float m = alpha * std::fabs(qn);            // C2B, equ_s4e21xx
                if (m < m1) {
                    m2 = m1;
                    m1 = m;
                    ow = e;
                } else if (m < m2) {
                    m2 = m;
                }
                ng ^= (uint8_t)(qn < 0.0f);
                Q[v] = qn;
                latest[v] = e;
            }
            mn[ci] = m1;
            smn[ci] = m2;
            own[ci] = ow;
            neg[ci] = ng;
            res.edge_visits += c->chk_ptr[ci + 1] - c->chk_ptr[ci];
            if (belief) {                                         // stop rule, as cbp_frame
                const bool ok = (ng == 0) && !flip;
                consec = ok ? consec + 1 : 0;
                if (consec >= W) {
                    if (syndrome_weight_bits(c, xhat) == 0) {
                        converged = true;
                        res.iters = sweep;
                    } else {
                        res.fires += 1;
                        consec = 0;
                    }
                }
            }
        }
        if (!converged && o->stop_rule == OR_STOP_SYNDROME && syndrome_weight_bits(c, xhat) == 0) {
            converged = true;
            res.iters = sweep;
        }
    }
    if (!converged) res.iters = o->max_iter;
    res.flags = (uint8_t)((converged ? 1 : 0) | (syndrome_weight_bits(c, xhat) == 0 ? 2 : 0) |
                          (res.fires > 0 ? 4 : 0));
    if (om_out) {
        om_out->resize(M);
        for (int32_t ck = 0; ck < M; ++ck) (*om_out)[ck] = neg[ck] ? -mn[ck] : mn[ck];   // signed minimum
    }
    return res;
}

// ---------------------------------------------------------------- comparison schedules (NEXT-3)
// Layered BP, in fp32 under the arithmetic contract (reading R22):
// checks ascending; for c and every v in N(c) (ascending): Q_{v->c} = Lambda_v - R_{c->v}
// (equ_s2e10); the C2V rule equ_s2e4 in the phi domain with the leave-one-out sum as
// S - phi(|Q_v|), S = sum of phi(|Q|) over N(c) in ascending order (as CBP's R11) and the
// sign product as the XOR of all signs with v's own; Lambda^new_v = Q + R^new (equ_s2e12).
// Decision equ_s2e7; stop: syndrome after every sweep (the hidden stop rule, l.157-160) or none.
static FrameResult lbp_frame(const or_code* c, const float* L, const or_opts* o, std::vector<uint8_t>& xhat)
{
    const int32_t N = c->N, M = c->M;
    std::vector<float> Lam(N), R(c->E, 0.0f);    // equ_s2e2: R = 0
    xhat.assign(N, 0);
    for (int32_t v = 0; v < N; ++v) {
        Lam[v] = L[v];
        xhat[v] = Lam[v] < 0.0f;
    }
    FrameResult res;
    bool converged = false;
    for (int32_t sweep = 1; sweep <= o->max_iter && !converged; ++sweep) {
        for (int32_t ci = 0; ci < M; ++ci) {
            const int32_t b = c->chk_ptr[ci], d = c->chk_ptr[ci + 1] - b;
            std::vector<float> Qe(d), Ph(d);
            float S = 0.0f;
            bool ng = false;
            for (int32_t k = 0; k < d; ++k) {
                Qe[k] = Lam[c->e_var[b + k]] - R[b + k];          // equ_s2e10
                Ph[k] = oracle_phi32(std::fabs(Qe[k]));
                S += Ph[k];
                ng = ng != (Qe[k] < 0.0f);
            }
            for (int32_t k = 0; k < d; ++k) {
                const float mag = oracle_phi32(std::fabs(S - Ph[k]));   // equ_s2e4, leave-one-out
                const bool sg = ng != (Qe[k] < 0.0f);
                const float Rn = sg ? -mag : mag;
                const int32_t v = c->e_var[b + k];
                Lam[v] = Qe[k] + Rn;                              // equ_s2e12
                R[b + k] = Rn;
                xhat[v] = Lam[v] < 0.0f;                          // equ_s2e7
            }
            res.edge_visits += d;
        }
        if (o->stop_rule == OR_STOP_SYNDROME && syndrome_weight_bits(c, xhat) == 0) {
            converged = true;
            res.iters = sweep;
        }
    }
    if (!converged) res.iters = o->max_iter;
    res.flags = (uint8_t)((converged ? 1 : 0) | (syndrome_weight_bits(c, xhat) == 0 ? 2 : 0));
    return res;
}

// Flooding BP, fp32 under the contract (reading R22): every iteration
// computes all V2C messages from the previous posterior, Q_{v->c} = Lambda_v - R_{c->v}
// (equ_s2e3 written as Lambda minus the own message), then all C2V messages by the phi-domain
// leave-one-out rule (equ_s2e4, as lbp_frame), then Lambda_v = L_v + sum_c R_{c->v}
// (equ_s2e6) summed from L_v in ascending check order; decision equ_s2e7; stop as lbp_frame.
static FrameResult fbp_frame(const or_code* c, const float* L, const or_opts* o, std::vector<uint8_t>& xhat)
{
    const int32_t N = c->N, M = c->M;
    std::vector<float> Lam(N), Rn(c->E, 0.0f);
    xhat.assign(N, 0);
    for (int32_t v = 0; v < N; ++v) {
        Lam[v] = L[v];
        xhat[v] = Lam[v] < 0.0f;
    }
    FrameResult res;
    bool converged = false;
    for (int32_t it = 1; it <= o->max_iter && !converged; ++it) {
        std::vector<float> Rold = Rn;
        for (int32_t ci = 0; ci < M; ++ci) {
            const int32_t b = c->chk_ptr[ci], d = c->chk_ptr[ci + 1] - b;
            std::vector<float> Qe(d), Ph(d);
            float S = 0.0f;
            bool ng = false;
            for (int32_t k = 0; k < d; ++k) {
                Qe[k] = Lam[c->e_var[b + k]] - Rold[b + k];       // equ_s2e3
                Ph[k] = oracle_phi32(std::fabs(Qe[k]));
                S += Ph[k];
                ng = ng != (Qe[k] < 0.0f);
            }
            for (int32_t k = 0; k < d; ++k) {
                const float mag = oracle_phi32(std::fabs(S - Ph[k]));   // equ_s2e4
                Rn[b + k] = (ng != (Qe[k] < 0.0f)) ? -mag : mag;
            }
            res.edge_visits += d;
        }
        for (int32_t v = 0; v < N; ++v) Lam[v] = L[v];
        for (int32_t ci = 0; ci < M; ++ci)                          // equ_s2e6, ascending checks
            for (int32_t e = c->chk_ptr[ci]; e < c->chk_ptr[ci + 1]; ++e) Lam[c->e_var[e]] += Rn[e];
        for (int32_t v = 0; v < N; ++v) xhat[v] = Lam[v] < 0.0f;    // equ_s2e7
        if (o->stop_rule == OR_STOP_SYNDROME && syndrome_weight_bits(c, xhat) == 0) {
            converged = true;
            res.iters = it;
        }
    }
    if (!converged) res.iters = o->max_iter;
    res.flags = (uint8_t)((converged ? 1 : 0) | (syndrome_weight_bits(c, xhat) == 0 ? 2 : 0));
    return res;
}

static bool opts_ok(const or_opts* o)
{
    if (!o || o->max_iter < 1 || o->max_iter > 65535 || o->stop_rule < 0 || o->stop_rule > 3 || o->arith < 0 ||
        o->arith > 5)
        return false;
    if (o->arith == OR_MINSUM && !(o->alpha > 0.0f && o->alpha <= 1.0f)) return false;
    if ((o->arith == OR_LBP || o->arith == OR_FBP) && o->stop_rule != OR_STOP_SYNDROME && o->stop_rule != OR_STOP_NONE)
        return false;
    return true;
}

static int decode_impl(const or_code* c, const float* llr, int64_t ld, int64_t frames, const or_opts* o,
                       uint32_t* bits, int64_t ld_words, int32_t* iters, uint8_t* flags,
                       int64_t* edge_visits, int32_t* fires, float* omega, const Instr& ins)
{
    if (!c || !opts_ok(o) || frames < 0 || ld < c->N || (bits && ld_words < (c->N + 31) / 32)) return 1;
    std::vector<uint8_t> xhat;
    for (int64_t f = 0; f < frames; ++f) {
        const float* L = llr + f * ld;
        FrameResult r;
        if (o->arith == OR_LBP || o->arith == OR_FBP) {
            r = (o->arith == OR_LBP) ? lbp_frame(c, L, o, xhat) : fbp_frame(c, L, o, xhat);
            if (omega) std::fill(omega + f * c->M, omega + (f + 1) * c->M, 0.0f);
        } else if (o->arith == OR_MINSUM) {
            std::vector<float> om;
            r = minsum_frame(c, L, o, xhat, omega ? &om : nullptr, ins);
            if (omega) std::copy(om.begin(), om.end(), omega + f * c->M);
        } else if (o->arith == OR_FP32_CONTRACT) {
            std::vector<float> S;
            std::vector<uint8_t> neg;
            r = cbp_frame<float>(c, L, o, false, xhat, omega ? &S : nullptr, &neg, ins);
            // Omega_c = sgn * phi(S_c)  (equ_s4e3 in the phi domain)
            if (omega)
                for (int32_t ck = 0; ck < c->M; ++ck) {
                    const float m = oracle_phi32(S[ck]);
                    omega[f * c->M + ck] = neg[ck] ? -m : m;
                }
        } else {
            std::vector<double> S;
            std::vector<uint8_t> neg;
            const bool lit = o->arith == OR_FP64_LITERAL;
            r = cbp_frame<double>(c, L, o, lit, xhat, omega ? &S : nullptr, &neg, ins);
            if (omega)
                for (int32_t ck = 0; ck < c->M; ++ck) {
                    double m;
                    if (lit) m = std::isinf(S[ck]) ? (double)OR_PHI_HI : S[ck];
                    else m = neg[ck] ? -phi_t<double>(S[ck]) : phi_t<double>(S[ck]);
                    omega[f * c->M + ck] = (float)m;
                }
        }
        if (bits) {
            uint32_t* w = bits + f * ld_words;
            std::fill(w, w + ld_words, 0u);
            for (int32_t v = 0; v < c->N; ++v) put_bit(w, v, xhat[v]);
        }
        if (iters) iters[f] = r.iters;
        if (flags) flags[f] = r.flags;
        if (edge_visits) edge_visits[f] = r.edge_visits;
        if (fires) fires[f] = r.fires;
    }
    return 0;
}

int oracle_decode(const or_code* c, const float* llr, int64_t ld, int64_t frames, const or_opts* o,
                  uint32_t* bits, int64_t ld_words, int32_t* iters, uint8_t* flags,
                  int64_t* edge_visits, int32_t* fires, float* omega)
{
    return decode_impl(c, llr, ld, frames, o, bits, ld_words, iters, flags, edge_visits, fires, omega, Instr());
}

int oracle_decode_window(const or_code* c, const float* llr, int64_t ld, int64_t frames, const or_opts* o,
                         int64_t window, uint32_t* bits, int64_t ld_words, int32_t* iters, uint8_t* flags,
                         int64_t* edge_visits, int32_t* fires)
{
    if (window < 1 || !o || o->arith == OR_LBP || o->arith == OR_FBP) return 1;
    Instr ins;
    ins.window = window;
    return decode_impl(c, llr, ld, frames, o, bits, ld_words, iters, flags, edge_visits, fires, nullptr, ins);
}

int oracle_ber_sim(const or_code* c, double ebn0_db, uint64_t seed, int64_t frame_begin, int64_t frames,
                   const or_opts* o, int32_t llr_mode, int64_t* counts)
{
    if (!c || !opts_ok(o) || frames < 0 || !counts) return 1;
    const int32_t N = c->N, K = c->K, nw = (N + 31) / 32;
    std::vector<float> L(N);
    std::vector<uint32_t> cw(nw), dec(nw);
    for (int64_t f = 0; f < frames; ++f) {
        if (oracle_channel(c, ebn0_db, seed, frame_begin + f, 1, llr_mode, L.data(), N, cw.data(), nw)) return 1;
        int32_t it = 0, fi = 0;
        uint8_t fl = 0;
        int64_t ev = 0;
        oracle_decode(c, L.data(), N, 1, o, dec.data(), nw, &it, &fl, &ev, &fi, nullptr);
        int64_t be = 0, ce = 0;
        for (int32_t v = 0; v < N; ++v) {
            const int d = get_bit(dec.data(), v) != get_bit(cw.data(), v);
            if (v < K) be += d;
            ce += d;
        }
        counts[0] += 1;
        counts[1] += be;
        counts[2] += be > 0;
        counts[3] += ce > 0;
        counts[4] += it;
        counts[5] += ev;
        counts[6] += (fl & 1) ? 0 : 1;
        counts[7] += fi;
    }
    return 0;
}

// ---------------------------------------------------------------- test-only references
int oracle_cbp_trace_f64(const or_code* c, const float* llr, int32_t sweeps, double* lam)
{
    if (!c || sweeps < 1) return 1;
    or_opts o = {sweeps, OR_STOP_NONE, OR_FP64, 0};
    Instr ins;
    ins.lam = lam;
    ins.per_sweep = true;
    std::vector<uint8_t> xhat;
    cbp_frame<double>(c, llr, &o, false, xhat, nullptr, nullptr, ins);
    return 0;
}

int oracle_cbp_visit_trace(const or_code* c, const float* llr, int32_t sweeps, int32_t arith, float alpha,
                           double* lam, double* qn)
{
    if (!c || sweeps < 1 || !lam || !qn || (arith != OR_FP32_CONTRACT && arith != OR_FP64 && arith != OR_MINSUM))
        return 1;
    or_opts o = {sweeps, OR_STOP_NONE, arith, alpha};
    Instr ins;
    ins.lam = lam;
    ins.qn = qn;
    ins.per_sweep = true;
    std::vector<uint8_t> xhat;
    if (arith == OR_FP64) cbp_frame<double>(c, llr, &o, false, xhat, nullptr, nullptr, ins);
    else if (arith == OR_MINSUM) minsum_frame(c, llr, &o, xhat, nullptr, ins);
    else cbp_frame<float>(c, llr, &o, false, xhat, nullptr, nullptr, ins);
    return 0;
}

int oracle_lbp_trace_f64(const or_code* c, const float* llr, int32_t sweeps, double* lam)
{
    // Layered BP: Q = Lambda - R (equ_s2e10), R^new by the
    // leave-one-out rule equ_s2e4 evaluated by brute force, Lambda = Q + R^new (equ_s2e12).
    if (!c || sweeps < 1) return 1;
    std::vector<double> Lam(c->N), R(c->E, 0.0);
    for (int32_t v = 0; v < c->N; ++v) Lam[v] = llr[v];
    for (int32_t s = 0; s < sweeps; ++s)
        for (int32_t ck = 0; ck < c->M; ++ck) {
            const int32_t b = c->chk_ptr[ck], d = c->chk_ptr[ck + 1] - b;
            std::vector<double> Qe(d), Rn(d);
            for (int32_t k = 0; k < d; ++k) {
                const int32_t v = c->e_var[b + k];
                lam[(int64_t)s * c->E + b + k] = Lam[v];
                Qe[k] = Lam[v] - R[b + k];
            }
            for (int32_t k = 0; k < d; ++k) {
                double sum = 0.0;
                bool sg = false;
                for (int32_t k2 = 0; k2 < d; ++k2) {
                    if (k2 == k) continue;
                    sum += phi_t<double>(std::fabs(Qe[k2]));
                    sg = sg != (Qe[k2] < 0.0);
                }
                const double m = phi_t<double>(sum);
                Rn[k] = sg ? -m : m;
            }
            for (int32_t k = 0; k < d; ++k) {
                Lam[c->e_var[b + k]] = Qe[k] + Rn[k];
                R[b + k] = Rn[k];
            }
        }
    return 0;
}

int oracle_ml_decode(const or_code* c, const float* llr, uint32_t* cw_out)
{
    if (!c || !c->can_encode || c->K > 20) return 1;
    const int32_t nw = (c->N + 31) / 32;
    std::vector<uint32_t> info((c->K + 31) / 32), cw(nw);
    double best = -std::numeric_limits<double>::infinity();
    for (uint32_t m = 0; m < (1u << c->K); ++m) {
        info[0] = m;
        oracle_encode(c, info.data(), cw.data());
        double corr = 0.0;
        for (int32_t v = 0; v < c->N; ++v) corr += get_bit(cw.data(), v) ? -(double)llr[v] : (double)llr[v];
        if (corr > best) {
            best = corr;
            std::copy(cw.begin(), cw.end(), cw_out);
        }
    }
    return 0;
}

void oracle_phi32_n(const float* x, float* y, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) y[i] = oracle_phi32(x[i]);
}

void oracle_ln32_n(const float* x, float* y, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) y[i] = oracle_ln32(x[i]);
}

int oracle_minsum_cbp_trace(const or_code* c, const float* llr, int32_t sweeps, float alpha, float* lam)
{
    if (!c || sweeps < 1) return 1;
    or_opts o = {sweeps, OR_STOP_NONE, OR_MINSUM, alpha};
    std::vector<double> tmp((size_t)sweeps * c->E);
    Instr ins;
    ins.lam = tmp.data();
    ins.per_sweep = true;
    std::vector<uint8_t> xhat;
    minsum_frame(c, llr, &o, xhat, nullptr, ins);
    for (size_t k = 0; k < tmp.size(); ++k) lam[k] = (float)tmp[k];
    return 0;
}

int oracle_minsum_lbp_trace(const or_code* c, const float* llr, int32_t sweeps, float alpha, float* lam)
{
    // Layered normalized min-sum BP: Q = Lambda - R (equ_s2e10); R^new_{c->v} = prod_{others} sgn(Q)
    // * min_{others} fl(alpha |Q|) (the min-sum form of equ_s2e4, by brute force); Lambda = Q + R^new.
    if (!c || sweeps < 1) return 1;
    std::vector<float> Lam(c->N), R(c->E, 0.0f);
    for (int32_t v = 0; v < c->N; ++v) Lam[v] = llr[v];
    for (int32_t s = 0; s < sweeps; ++s)
        for (int32_t ck = 0; ck < c->M; ++ck) {
            const int32_t b = c->chk_ptr[ck], d = c->chk_ptr[ck + 1] - b;
            std::vector<float> Qe(d), Rn(d);
            for (int32_t k = 0; k < d; ++k) {
                const int32_t v = c->e_var[b + k];
                lam[(int64_t)s * c->E + b + k] = Lam[v];
                Qe[k] = Lam[v] - R[b + k];
            }
            for (int32_t k = 0; k < d; ++k) {
                float m = std::numeric_limits<float>::infinity();
                bool sg = false;
                for (int32_t k2 = 0; k2 < d; ++k2) {
                    if (k2 == k) continue;
                    m = std::fmin(m, alpha * std::fabs(Qe[k2]));
                    sg = sg != (Qe[k2] < 0.0f);
                }
                Rn[k] = sg ? -m : m;
            }
            for (int32_t k = 0; k < d; ++k) {
                Lam[c->e_var[b + k]] = Qe[k] + Rn[k];
                R[b + k] = Rn[k];
            }
        }
    return 0;
}
