// cbp_api.cpp -- host side of the C ABI (include/cbp.h): validation, schedule
// tables of the expanded code graph, launch geometry, launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "cbp.h"
#include "cbp_inputs.h"
#include "cbp_internal.h"


namespace {

thread_local std::string g_err;

cbp_status fail(cbp_status s, const std::string& msg)
{
    g_err = msg;
    return s;
}

cbp_status cuda_fail(cudaError_t e, const char* what)
{
    return fail(CBP_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII switch of the current device
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) return;
        ok = (prev == dev) || cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard()
    {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// phi contract v3 table, device storage form: segment seg holds the cubic
// through phi at u = 0, 1/4, 3/4, 1 of its interval, phi(x) = -log(tanh(x/2))
// evaluated in IEEE double as log1p(2 / expm1(x)) (no cancellation of tanh -> 1); Newton divided
// differences in double in the contract's order, coefficients rounded to binary32; the x < 2
// rows scaled for the kernel's local variable u/16 (c1 x 16, c2 x 256, c3 x 4096, exact).
//   seg < 704:  x(u) = 2^e (1 + (j + u)/16), e = -43 + seg/16, j = seg % 16
//   seg >= 704: x(u) = 2 + (seg - 704 + u)/16
void build_phi_rows(float4* rows)
{
    static const int kQ4[4] = {0, 1, 3, 4};
    for (int seg = 0; seg < cbp::kPhiTableSegs; ++seg) {
        double f[4];
        for (int k = 0; k < 4; ++k) {
            const float x = (seg < 704) ? std::ldexp(static_cast<float>(64 + 4 * (seg % 16) + kQ4[k]), -43 + seg / 16 - 6)
                                        : static_cast<float>(128 + 4 * (seg - 704) + kQ4[k]) * 0.015625f;
            f[k] = std::log1p(2.0 / std::expm1(static_cast<double>(x)));
        }
        const double d01 = (f[1] - f[0]) * 4.0, d12 = (f[2] - f[1]) * 2.0, d23 = (f[3] - f[2]) * 4.0;
        const double d012 = ((d12 - d01) * 4.0) / 3.0, d123 = ((d23 - d12) * 4.0) / 3.0;
        const double d0123 = d123 - d012;
        float4 c = make_float4(static_cast<float>(f[0]), static_cast<float>((d01 - d012 * 0.25) + d0123 * 0.1875),
                               static_cast<float>(d012 - d0123), static_cast<float>(d0123));
        if (seg < 704) {
            c.y *= 16.0f;
            c.z *= 256.0f;
            c.w *= 4096.0f;
        }
        rows[seg] = c;
    }
}

std::mutex g_tab_mu;
float4* g_tab[128] = {};
cudaTextureObject_t g_tex[128] = {};   // texture objects over g_tab (TEX-pipe lookups)

const float4* phi_table(int device, std::string* err, cudaTextureObject_t* tex = nullptr)
{
    std::lock_guard<std::mutex> lk(g_tab_mu);
    if (device < 0 || device >= 128) { *err = "device index out of range"; return nullptr; }
    if (g_tab[device]) {
        if (tex) *tex = g_tex[device];
        return g_tab[device];
    }
    DeviceGuard g(device);
    float4* p = nullptr;
    std::vector<float4> rows(cbp::kPhiTableSegs);
    build_phi_rows(rows.data());
    cudaError_t e = cudaMalloc(&p, sizeof(float4) * cbp::kPhiTableSegs);
    if (e == cudaSuccess) e = cudaMemcpy(p, rows.data(), sizeof(float4) * cbp::kPhiTableSegs, cudaMemcpyHostToDevice);
    cudaTextureObject_t t = 0;
    if (e == cudaSuccess) {
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = p;
        rd.res.linear.desc = cudaCreateChannelDesc<float4>();
        rd.res.linear.sizeInBytes = sizeof(float4) * cbp::kPhiTableSegs;
        cudaTextureDesc td{};
        td.readMode = cudaReadModeElementType;   // point fetch of the stored words, no filtering
        e = cudaCreateTextureObject(&t, &rd, &td, nullptr);
    }
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        *err = std::string("phi table: ") + cudaGetErrorString(e);
        return nullptr;
    }
    g_tab[device] = p;
    g_tex[device] = t;
    if (tex) *tex = t;
    return p;
}

// Per-device memory pool for the launch workspace (work-queue counter, global frame state):
// stream-ordered allocations that stay cached across launches.  The default pool of the
// device returns freed memory at every synchronisation (release threshold 0), which made
// each launch re-map memory -- measured as intermittent 2-20x slower launches.
std::mutex g_pool_mu;
cudaMemPool_t g_pool[128] = {};

cudaMemPool_t work_pool(int device)
{
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (device < 0 || device >= 128) return nullptr;
    if (g_pool[device]) return g_pool[device];
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    uint64_t keep = UINT64_MAX;   // never trim: the workspace is reused launch after launch
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    g_pool[device] = p;
    return p;
}

}  // namespace

struct cbp_code {
    int device = 0;
    int32_t mb = 0, nb = 0, Z = 0, N = 0, K = 0, M = 0, kb = 0, core = 0, mid = 0, nent = 0, max_dc = 0, min_dc = 0;
    int64_t E = 0;
    bool can_encode = false;
    std::vector<int4> ent[4];             // schedule tables scaled for geo[alg] (kernel parameters)
    std::vector<int32_t> row_ptr;
    std::vector<int16_t> pshift;
    const float4* phi_tab = nullptr;   // per-device table, not owned
    cudaTextureObject_t phi_tex = 0;   // per-device texture object over phi_tab, not owned
    cbp::Geometry geo[4]{};           // per cbp_algorithm
    int ctas_per_sm[4] = {1, 1, 1, 1}, num_sms = 1;
    cbp::Geometry geo_chan{};          // cbp_channel: cbp_kernel (the warp kernel has no channel-only mode)
    int ctas_chan = 1;
    cbp::Geometry geo_omega{};         // log-tanh decode with Omega output (geo[0] is cbp_warp_kernel's): room for S
    int ctas_omega = 1;
    int4* ent_dev[4] = {};             // device copies of ent[] (bulk-copied by cbp_warp_kernel)
    ~cbp_code()
    {
        for (int4* p : ent_dev)
            if (p) cudaFree(p);
    }
};

extern "C" {

const char* cbp_last_error(void) { return g_err.c_str(); }

const char* cbp_version(void) { return "cbp-b200 0.1 (sm_100a)"; }

cbp_status cbp_construct_base(const cbp_construct_spec* spec, uint64_t seed, int16_t* base_out)
{
    if (!spec || !base_out) return fail(CBP_E_INVALID, "cbp_construct_base: null argument");
    cbp_inputs_spec s{spec->mb, spec->nb, spec->Z, spec->mb_core, spec->wmode, spec->w_lo, spec->w_hi};
    const char* err = nullptr;
    if (cbp_inputs_construct_base(&s, seed, base_out, &err) != 0)
        return fail(CBP_E_INVALID, std::string("cbp_construct_base: ") + (err ? err : "invalid spec"));
    return CBP_OK;
}

void cbp_code_destroy(cbp_code* c)
{
    if (!c) return;
    DeviceGuard g(c->device);
    delete c;
}

cbp_status cbp_code_create(const int16_t* base, int32_t mb, int32_t nb, int32_t Z, int32_t device, cbp_code** out)
{
    return cbp_code_create_ex(base, mb, nb, Z, device, nullptr, out);
}

cbp_status cbp_code_create_ex(const int16_t* base, int32_t mb, int32_t nb, int32_t Z, int32_t device,
                              const cbp_code_config* cfg, cbp_code** out)
{
    if (!base || !out) return fail(CBP_E_INVALID, "cbp_code_create: null argument");
    int want_P = cfg ? cfg->frames_per_lane : 0;
    if (want_P < 0 || want_P > 2) return fail(CBP_E_INVALID, "cbp_code_create: frames_per_lane must be 0, 1 or 2");
    if (want_P == 0) {
        // debugging override of the automatic choice (A/B measurements)
        const char* ev = std::getenv("CBP_FRAMES_PER_LANE");
        if (ev && (ev[0] == '1' || ev[0] == '2') && ev[1] == 0) want_P = ev[0] - '0';
    }
    *out = nullptr;
    if (mb < 1 || nb <= mb) return fail(CBP_E_INVALID, "cbp_code_create: need 1 <= mb < nb");
    if (Z < 1 || Z > 1024) return fail(CBP_E_INVALID, "cbp_code_create: need 1 <= Z <= 1024");
    if (static_cast<int64_t>(nb) * Z > 65535 || static_cast<int64_t>(mb) * Z > 65535)
        return fail(CBP_E_UNSUPPORTED, "cbp_code_create: N and M must be < 65536");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(CBP_E_INVALID, "cbp_code_create: no such CUDA device");

    std::vector<int32_t> colw(nb, 0), roww(mb, 0);
    for (int i = 0; i < mb; ++i)
        for (int j = 0; j < nb; ++j) {
            const int s = base[i * nb + j];
            if (s < -1 || s >= Z) return fail(CBP_E_INVALID, "cbp_code_create: shift out of [-1, Z)");
            if (s >= 0) { ++colw[j]; ++roww[i]; }
        }
    for (int j = 0; j < nb; ++j)
        if (!colw[j]) return fail(CBP_E_INVALID, "cbp_code_create: empty base column");
    for (int i = 0; i < mb; ++i)
        if (!roww[i]) return fail(CBP_E_INVALID, "cbp_code_create: empty base row");
    const int max_dc = *std::max_element(roww.begin(), roww.end());
    if (max_dc > 32) return fail(CBP_E_UNSUPPORTED, "cbp_code_create: base row degree > 32");

    // entries row-major; per column the list of its nonzero rows (ascending)
    std::vector<int> ent_row, ent_col, ent_s, row_ptr(mb + 1, 0);
    std::vector<std::vector<int>> col_ent(nb);
    for (int i = 0; i < mb; ++i) {
        for (int j = 0; j < nb; ++j) {
            const int s = base[i * nb + j];
            if (s < 0) continue;
            col_ent[j].push_back(static_cast<int>(ent_row.size()));
            ent_row.push_back(i);
            ent_col.push_back(j);
            ent_s.push_back(s);
        }
        row_ptr[i + 1] = static_cast<int>(ent_row.size());
    }
    const int nent = static_cast<int>(ent_row.size());
    if (nent > cbp::kMaxEnt || mb > cbp::kMaxRows)
        return fail(CBP_E_UNSUPPORTED, "cbp_code_create: more than 512 nonzero base entries or 128 base rows");
    // two int4 per entry b for a geometry with P frames per lane (layout documented in
    // cbp_kernels.cu; QS = 8P bytes per variable, RS = 4P bytes per edge, SU = 4 for the
    // 16-byte min-sum check records, else 1):
    //   E0 = {QS jZ, S0 + SU RS row(p) Z, R0 + RS pZ, QS s},
    //   E1 = {RS ds, first ? ~0 : 0, first | kp << 8 | s << 16, R0 + RS bZ}
    // Byte offsets are relative to the group base: QP at 0, the check records at S0, R at R0.
    auto make_ent = [&](int P, int alg, bool r_global) {
        const int QS = 8 * P, RS = 4 * P, SU = (alg == 1) ? 4 : 1, SW = (alg == 1) ? 4 : 1;
        const int S0 = 4 * ((2 * P * nb * Z + 3) & ~3), R0 = r_global ? 0 : S0 + 4 * P * SW * mb * Z;
        std::vector<int4> ent(2 * static_cast<size_t>(nent));
        for (int j = 0; j < nb; ++j) {
            const auto& L = col_ent[j];
            for (size_t k = 0; k < L.size(); ++k) {
                const int b = L[k];
                const int p = L[(k + L.size() - 1) % L.size()];       // previous nonzero row of column j, cyclic
                const int ds = ((ent_s[b] - ent_s[p]) % Z + Z) % Z;
                const int first = (k == 0) ? 1 : 0;                   // R1: no latest check before this visit
                // kp: position of prev(b) among its row's entries = the variable's edge index inside
                // the previous check (min-sum minimum owner, reading R20)
                const int kp = p - row_ptr[ent_row[p]];
                if (alg == 0 || alg == 2) {
                    // producer-side layout (CBP log-tanh, layered BP): variable block and rotation only
                    ent[2 * b] = make_int4(QS * j * Z, QS * ent_s[b], 0, 0);
                    ent[2 * b + 1] = make_int4(0, 0, ent_s[b] << 16, 0);
                    continue;
                }
                ent[2 * b] = make_int4(QS * j * Z, S0 + SU * RS * ent_row[p] * Z, R0 + RS * p * Z, QS * ent_s[b]);
                ent[2 * b + 1] = make_int4(RS * ds, first ? 0 : -1, first | (kp << 8) | (ent_s[b] << 16), R0 + RS * b * Z);
            }
        }
        return ent;
    };

    cbp_code* c = new cbp_code();
    c->device = device;
    c->mb = mb; c->nb = nb; c->Z = Z;
    c->N = nb * Z; c->M = mb * Z; c->K = c->N - c->M; c->kb = nb - mb;
    c->E = static_cast<int64_t>(nent) * Z;
    c->nent = nent;
    c->max_dc = max_dc;

    // encoder structure: dual-diagonal core + degree-1 extension
    {
        const int kb = c->kb;
        int core = 0;
        while (kb + core < nb && colw[kb + core] >= 2) ++core;
        bool ok = core >= 3;
        const int mid = core / 2;
        auto at = [&](int i, int j) { return static_cast<int>(base[i * nb + j]); };
        if (ok) {
            for (int i = 0; i < mb && ok; ++i) {
                const bool want = (i == 0 || i == mid || i == core - 1);
                ok = want == (at(i, kb) >= 0);
            }
            ok = ok && at(mid, kb) == 0 && at(0, kb) == at(core - 1, kb);
            for (int t = 1; t < core && ok; ++t)
                for (int i = 0; i < mb && ok; ++i) {
                    const bool want = (i == t - 1 || i == t);
                    ok = want ? at(i, kb + t) == 0 : at(i, kb + t) < 0;
                }
            ok = ok && (nb - kb - core) == (mb - core);
            for (int k = 0; kb + core + k < nb && ok; ++k)
                for (int i = 0; i < mb && ok; ++i) {
                    const bool want = (i == core + k);
                    ok = want ? at(i, kb + core + k) == 0 : at(i, kb + core + k) < 0;
                }
        }
        c->can_encode = ok;
        c->core = ok ? core : 0;
        c->mid = ok ? mid : 0;
    }
    std::vector<int16_t> pshift(mb, -1);
    for (int i = 0; i < mb; ++i) pshift[i] = base[i * nb + c->kb];

    DeviceGuard g(device);
    if (!g.ok) { delete c; return fail(CBP_E_CUDA, "cbp_code_create: cudaSetDevice failed"); }
    {
        std::string terr;
        c->phi_tab = phi_table(device, &terr, &c->phi_tex);
        if (!c->phi_tab) { delete c; return fail(CBP_E_CUDA, "cbp_code_create: " + terr); }
    }
    c->row_ptr = row_ptr;
    c->pshift = pshift;

    // ---- launch geometry per algorithm
    int smem_optin = 0, nsm = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    c->num_sms = nsm > 0 ? nsm : 1;
    c->min_dc = *std::min_element(roww.begin(), roww.end());
    const int nwords = (c->N + 31) / 32;
    // split layout (R in global memory): automatic (below), or forced on / off with CBP_SPLIT_R=1 / 0 (A/B runs)
    const char* sr = std::getenv("CBP_SPLIT_R");
    const int split_env = (sr && (sr[0] == '0' || sr[0] == '1') && sr[1] == 0) ? sr[0] - '0' : -1;
    // geometry with P frames per lane; G.teams == 0 if it does not apply
    static const int multi_maxt_env = [] { const char* e = std::getenv("CBP_MULTI_MAXT"); return e ? std::atoi(e) : 0; }();
    const char* wv = std::getenv("CBP_WARP_KERNEL");     // 0: cbp_kernel only (A/B runs)
    // (CBP_GLOBAL_TEAMS forces cbp_kernel's global-state path and so disables the warp kernel too)
    const bool use_warp = !(wv && wv[0] == '0' && wv[1] == 0) && !std::getenv("CBP_GLOBAL_TEAMS");
    const int split_r_env = split_env;
    // cbp_warp_kernel phi-row path (A/B runs): CBP_WARP_TEX=0 C2B rows through TEX (default), 1 both, 2 none
    const char* t2 = std::getenv("CBP_WARP_TEX");
    const int tex2_env = (t2 && t2[0] >= '0' && t2[0] <= '2' && t2[1] == 0) ? t2[0] - '0' : -1;
    // cbp_warp_kernel per-warp state in words (cbp_internal.h): counters | Lambda | H bytes | cw |
    // park buffer | R (r_words, if in the slot) | S [M] (Omega output only)
    auto warp_state_words = [&](int64_t r_words, bool with_S) -> int64_t {
        return (16 + static_cast<int64_t>(c->N) + cbp::warp_hb_words(c->N) + cbp::warp_cw_words(nwords) +
                cbp::warp_pb_words(max_dc) + r_words + (with_S ? c->M : 0) + 3) / 4 * 4;
    };
    auto make_geo = [&](int alg, int P, bool split_r, int multi_maxt = 512, bool allow_warp = true,
                        bool with_S = false) {
        cbp::Geometry G{};
        G.alg = alg;
        G.P = P;
        // cbp_warp_kernel team frames: one frame per CTA, its warps share the state in
        // shared memory (5 N bytes), rows ordered by a CTA barrier.  For codes whose frames do not fit 6 per
        // SM in warp mode (Z > 128: C4; P8192).  CBP_WARP_TEAM=0 keeps cbp_kernel's teams (A/B runs).
        const char* tv = std::getenv("CBP_WARP_TEAM");
        const bool team_on = !(tv && tv[0] == '0' && tv[1] == 0);
        auto warp_team = [&]() -> bool {
            if (!(use_warp && allow_warp && team_on && (alg == 0 || alg == 2) && P == 1 && Z >= 17 && tex2_env < 0))
                return false;
            const int K = Z <= CBP_WARPT_MAXT ? 1 : (Z <= 2 * CBP_WARPT_MAXT ? 2 : 0);
            if (K == 0) return false;
            const int lanes = (Z + K - 1) / K, W = (lanes + 31) / 32;
            const int64_t tw = 4 * cbp::kPhiTableSegs + (8 * nent + (mb + 1) + (mb + 1) / 2 + 3) / 4 * 4 + 4;
            // counters | Lambda | H | cw | park buffer per warp | S (Omega) | row control [2][2][W] | frame index
            const int64_t sw = (16 + static_cast<int64_t>(c->N) + cbp::warp_hb_words(c->N) + cbp::warp_cw_words(nwords) +
                                static_cast<int64_t>(W) * cbp::warp_pb_words(max_dc) + (with_S ? c->M : 0) + 4 * W + 4 + 3) /
                               4 * 4;
            if (4 * (tw + sw) > smem_optin) return false;
            G = cbp::Geometry{};
            G.alg = alg; G.P = P; G.wk = 1; G.multi = 1; G.kslots = K; G.lanes = lanes; G.F = 1; G.Zp = 32;
            G.team_threads = 32 * W; G.threads = 32 * W; G.teams = 1; G.state_in_smem = 1; G.r_global = 1;
            G.r_words = static_cast<int32_t>(static_cast<int64_t>(W) * nent * K * 32);
            G.slot_words = static_cast<int32_t>(sw); G.table_words = static_cast<int32_t>(tw); G.tex2 = 0;
            G.smem_bytes = static_cast<int32_t>(4 * (tw + sw));
            return true;
        };
        if (Z > 128) {
            if (warp_team()) return G;
            goto team_geometry;
        }
        if (use_warp && allow_warp && (alg == 0 || alg == 2) && P == 1 && Z >= 17 && Z <= 128) {
            // cbp_warp_kernel: one frame per warp, K = ceil(Z/32) check slots per lane
            G.wk = 1;
            G.kslots = (Z + 31) / 32;
            G.lanes = (Z + G.kslots - 1) / G.kslots;
            G.multi = 0; G.F = 1; G.Zp = 32; G.team_threads = 32; G.state_in_smem = 1;
            const int maxt = G.kslots == 1 ? CBP_WARPK1_MAXT : CBP_WARPK_MAXT;
            const int64_t rw = static_cast<int64_t>(nent) * G.kslots * 32;
            G.tex2 = tex2_env >= 0 ? tex2_env : 0;
            G.table_words = (G.tex2 == 1 ? 0 : 4 * cbp::kPhiTableSegs) + (8 * nent + (mb + 1) + (mb + 1) / 2 + 3) / 4 * 4 + 4;
            auto per_warp = [&](bool rg) { return warp_state_words(rg ? 0 : rw, with_S); };
            auto warps_of = [&](bool rg) {
                const int64_t w = (smem_optin - 4LL * G.table_words) / (4 * per_warp(rg));
                return static_cast<int>(std::min<int64_t>(w, maxt / 32));
            };
            const int ws = warps_of(false), wg = warps_of(true);
            if (std::max(ws, wg) < 6) {
                // frames too large for 6 per SM even with R in global memory (P8192: 5 warps): team frames,
                // else cbp_kernel's teams
                if (warp_team()) return G;
                G = cbp::Geometry{};
                G.alg = alg;
                G.P = P;
                goto team_geometry;
            }
            // R in global memory (coalesced, L1/L2-served) when shared memory holds fewer than 8 frames
            bool rg = ws < 8 && wg > ws;
            if (split_r_env == 0) rg = false;
            if (split_r_env == 1) rg = true;
            G.r_global = rg ? 1 : 0;
            G.r_words = rg ? static_cast<int32_t>(rw) : 0;
            G.slot_words = static_cast<int32_t>(per_warp(rg));
            G.teams = rg ? wg : ws;
            static const int warps_env = [] { const char* e = std::getenv("CBP_WARPS"); return e ? std::atoi(e) : 0; }();
            if (warps_env > 0) G.teams = std::min(G.teams, warps_env);   // A/B runs: fewer warps, more L1
            if (G.teams < 1) { G.wk = 0; G.teams = 0; }
            else {
                G.threads = 32 * G.teams;
                G.smem_bytes = static_cast<int32_t>(4LL * G.table_words + 4LL * G.teams * G.slot_words);
                return G;
            }
        }
    team_geometry:
        if (Z <= 16) {
            int zp = 1;
            while (zp < Z) zp <<= 1;
            G.Zp = zp; G.F = 32 / zp; G.threads = 32; G.multi = 0;
        } else if (Z <= 32) {
            G.Zp = 32; G.F = 1; G.threads = 32; G.multi = 0;
        } else {
            G.Zp = (Z + 31) / 32 * 32; G.F = 1; G.threads = G.Zp; G.multi = 1;
        }
        // group of P frames: QP (2P words per variable), pad to 4 words, check records
        // (P words, or 4P for min-sum's 16-byte records), R (P words per edge), P codewords;
        // groups 16-byte aligned, F > 1 groups staggered by max(Zp, 4) words across banks
        // (flooding BP adds its channel LLRs, P words per variable, after the codewords)
        // split layout (r_global): R [P E] moves to a global slot of its own, the rest stays in shared memory
        G.r_global = (split_r && P == 1) ? 1 : 0;
        G.r_words = G.r_global ? static_cast<int32_t>((P * c->E + 3) / 4 * 4) : 0;
        const int64_t raw = (2LL * P * c->N + 3) / 4 * 4 +
                            P * ((alg == 1 ? 4LL : 1LL) * c->M + (G.r_global ? 0 : c->E) + nwords + (alg == 3 ? c->N : 0));
        G.slot_words = static_cast<int32_t>(G.F > 1 ? (raw + 31) / 32 * 32 + std::max(G.Zp, 4) : (raw + 3) / 4 * 4);
        G.table_words = ((CBP_TEX_B2V && CBP_TEX_C2B) ? 0 : 4 * cbp::kPhiTableSegs) +
                        (8 * nent + (mb + 1) + (mb + 1) / 2 + 3) / 4 * 4;
        G.team_threads = G.threads;
        // teams per CTA: as many independent teams as shared memory, the thread limit of the
        // instantiation (512 for P = 1, 256 for P = 2) and 15 named barriers allow
        // thread limit of the instantiation: 512 for multi-warp teams, 768 (80 registers) for the split
        // layout's multi-warp teams; CBP_MULTI_MAXT overrides it for A/B runs
        if (multi_maxt_env == 512 || multi_maxt_env == 768 || multi_maxt_env == 1024) multi_maxt = multi_maxt_env;
        const int maxt = (P == 2) ? 256 : (G.multi ? multi_maxt : CBP_WARP_MAXT);
        if (G.team_threads > maxt && P == 2) return G;
        // shared control words: multi-warp teams exchange ballots and queue indices; warp teams keep
        // nb ballot words for the packed syndrome (kernel syndrome_nz)
        G.fast_syn = (!G.multi && Z <= 32 && mb <= G.Zp) ? 1 : 0;
        G.ctl_words = G.multi ? cbp::kCtlTeamWords : (G.fast_syn ? (nb + 3) / 4 * 4 : 0);
        const int64_t ctl = G.ctl_words;
        const int64_t per_team = 4LL * (ctl + static_cast<int64_t>(G.F) * G.slot_words);
        const int64_t fixed = 4LL * G.table_words;
        int nt = static_cast<int>((smem_optin - fixed) / per_team);
        nt = std::min(nt, std::max(1, maxt / G.team_threads));
        if (G.multi) nt = std::min(nt, 15);
        // Large frames with small teams: when shared memory holds a single team of < 8 warps
        // and no second CTA fits beside it, the SM runs nearly idle (P8192: one 64-thread team
        // per SM).  The global-state path runs maxt / team_threads teams per CTA with the
        // state served from L2/L1 instead: 2.0-2.3x faster on P8192.
        if (G.multi && P == 1 && nt >= 1 && nt * G.team_threads < 256 && 2 * (fixed + nt * per_team) > smem_optin)
            nt = 0;
        G.state_in_smem = nt >= 1 ? 1 : 0;
        if (!G.state_in_smem && G.r_global) {            // no split without shared memory: all-global path
            G.r_global = 0;
            G.r_words = 0;
            G.slot_words += static_cast<int32_t>((P * c->E + 3) / 4 * 4);
        }
        if (P == 2 && !G.state_in_smem) return G;
        G.teams = G.state_in_smem ? nt : std::max(1, maxt / G.team_threads);
        // a single large team (C4: 384 threads) leaves the global-state path latency-bound; two
        // teams run in the 1024-thread instantiation (64 registers): C4 455 vs 580 ms per 2e4 frames
        if (!G.state_in_smem && G.multi && P == 1 && G.teams == 1 && 2 * G.team_threads <= 1024) G.teams = 2;
        if (const char* gt = std::getenv("CBP_GLOBAL_TEAMS"); gt && P == 1) {
            // A/B measurements only: force the global-state path with k teams per CTA
            const int k = std::atoi(gt);
            if (k >= 1 && (G.multi ? k <= 15 && k * G.team_threads <= 1024 : k * G.team_threads <= maxt)) {
                G.state_in_smem = 0;
                G.teams = k;
                if (G.r_global) {
                    G.r_global = 0;
                    G.r_words = 0;
                    G.slot_words += static_cast<int32_t>((P * c->E + 3) / 4 * 4);
                }
            }
        }
        G.threads = G.teams * G.team_threads;
        G.smem_bytes = static_cast<int32_t>(G.state_in_smem ? fixed + G.teams * per_team
                                                            : fixed + 4LL * ctl * G.teams);
        return G;
    };
    for (int alg = 0; alg < 4; ++alg) {
        cbp::Geometry g1 = make_geo(alg, 1, split_env == 1);
        const cbp::Geometry g2 = alg <= 1 ? make_geo(alg, 2, false) : cbp::Geometry{};
        // Warp teams whose frames are too large for more than a few per SM (P2048: 45 KB, 4 warps per
        // SM) are latency-bound; moving R to global memory (L1/L2-served) fits 2x+ the frames in
        // shared memory: P2048 28.5 vs 34.8 ms per 1e5 frames.  Codes that already hold >= 8 warps
        // per SM lose by it (C2 +8 %, C1 +4 %, C3a/C3b +5 %), so they keep R in shared memory.
        if (split_env < 0 && !g1.multi && g1.state_in_smem && g1.teams * g1.team_threads < 256) {
            const cbp::Geometry gs = make_geo(alg, 1, true);
            if (gs.state_in_smem && gs.r_global && gs.teams >= 2 * g1.teams) g1 = gs;
        }
        // Multi-warp teams (Z > 32): the split layout with up to 768 threads doubles C3a's teams per SM
        // (4 -> 8): C3a 11.1 vs 12.4 ms per 5e4 frames at 2.5 dB, 7.9 vs 8.5 at 1.5 dB, C3b 11.7 vs 12.7.
        // Taken when it at least doubles the threads of the shared-memory geometry (P8192's global
        // workspace with 8 teams keeps more frames in flight than 2 split teams and stays).
        if (split_env < 0 && g1.multi && !g1.r_global) {
            const cbp::Geometry gs = make_geo(alg, 1, true, 768);
            if (gs.state_in_smem && gs.r_global && gs.teams * gs.team_threads >= 2 * g1.teams * g1.team_threads) g1 = gs;
        }
        // automatic: one frame per lane.  Two interleaved frames per lane halve the warps
        // per SM at the same shared memory and measured slower on every config (C2
        // ber_sim 12.0 vs 7.65 ms); they remain a selectable geometry.
        // (the comparison schedules LBP / FBP always run one frame per lane)
        const int P = (alg >= 2) ? 1 : (want_P ? want_P : 1);
        if (P == 2 && g2.teams == 0) {
            cbp_code_destroy(c);
            return fail(CBP_E_UNSUPPORTED, "cbp_code_create: two frames per lane need the state in shared memory "
                                           "and at most 256 threads per team");
        }
        cbp::Geometry& G = c->geo[alg];
        G = (P == 2) ? g2 : g1;
        int occ = 0;
        if (cbp::occupancy_ctas_per_sm(G, &occ) != 0 || occ < 1) {
            cudaGetLastError();
            cbp_code_destroy(c);
            return fail(CBP_E_UNSUPPORTED, "cbp_code_create: kernel does not fit on this device");
        }
        c->ctas_per_sm[alg] = G.state_in_smem ? occ : 1;
        c->ent[alg] = make_ent(G.P, alg, G.r_global != 0);
        // cbp_warp_kernel (alg 0 / 2) reads its own entries, bulk-copied: {j Z, s, 0, 0}, {0, 0, s << 16, 0}
        // (variable indices; the kernel parameters keep cbp_kernel's byte offsets for cbp_channel)
        std::vector<int4> went = c->ent[alg];
        if (alg == 0 || alg == 2)
            for (int b = 0; b < nent; ++b) {
                went[2 * b] = make_int4(ent_col[b] * Z, ent_s[b], 0, 0);
                went[2 * b + 1] = make_int4(0, 0, ent_s[b] << 16, 0);
            }
        const size_t eb = sizeof(int4) * went.size();
        if (cudaMalloc(&c->ent_dev[alg], eb) != cudaSuccess ||
            cudaMemcpy(c->ent_dev[alg], went.data(), eb, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            cbp_code_destroy(c);
            return fail(CBP_E_NOMEM, "cbp_code_create: schedule table upload failed");
        }
    }
    // cbp_channel (no decoding) runs on cbp_kernel with the log-tanh entries
    c->geo_chan = c->geo[0];
    c->ctas_chan = c->ctas_per_sm[0];
    c->geo_omega = c->geo[0];
    c->ctas_omega = c->ctas_per_sm[0];
    if (c->geo[0].wk) {
        // (a frame plus S that no longer fits on chip -- C4's team frames -- runs on cbp_kernel's teams)
        c->geo_omega = make_geo(0, 1, false, 512, true, true);
        int occ = 0;
        if (cbp::occupancy_ctas_per_sm(c->geo_omega, &occ) != 0 || occ < 1) {
            cudaGetLastError();
            cbp_code_destroy(c);
            return fail(CBP_E_UNSUPPORTED, "cbp_code_create: Omega-output kernel does not fit on this device");
        }
        c->ctas_omega = occ;
    }
    if (c->geo[0].wk) {
        c->geo_chan = make_geo(0, 1, false, 512, false);
        int occ = 0;
        if (cbp::occupancy_ctas_per_sm(c->geo_chan, &occ) != 0 || occ < 1) {
            cudaGetLastError();
            cbp_code_destroy(c);
            return fail(CBP_E_UNSUPPORTED, "cbp_code_create: channel kernel does not fit on this device");
        }
        c->ctas_chan = c->geo_chan.state_in_smem ? occ : 1;
    }
    *out = c;
    return CBP_OK;
}

cbp_status cbp_code_dims(const cbp_code* c, int32_t* N, int32_t* K, int32_t* M, int64_t* E)
{
    if (!c) return fail(CBP_E_INVALID, "cbp_code_dims: null code");
    if (N) *N = c->N;
    if (K) *K = c->K;
    if (M) *M = c->M;
    if (E) *E = c->E;
    return CBP_OK;
}

cbp_status cbp_get_launch_info(const cbp_code* c, cbp_launch_info* o)
{
    if (!c || !o) return fail(CBP_E_INVALID, "cbp_get_launch_info: null argument");
    const cbp::Geometry& G = c->geo[0];     // log-tanh geometry (min-sum: same teams, larger slots)
    o->threads = G.threads;
    o->ctas_per_sm = c->ctas_per_sm[0];
    o->frames_per_cta = G.F * G.teams * G.P;
    o->smem_bytes = G.smem_bytes;
    o->state_in_smem = G.state_in_smem;
    o->num_sms = c->num_sms;
    o->frames_per_lane = G.P;
    o->r_in_global = G.r_global;
    return CBP_OK;
}

}  // extern "C"

namespace {

// the geometry a launch runs with: cbp_channel on the warp kernel of the code (else on cbp_kernel); a
// log-tanh decode with Omega output on the warp kernel's geometry that has room for the check records
const cbp::Geometry& geo_for(const cbp_code* c, int alg, bool chan, bool omega, int* ctas)
{
    if (chan && !c->geo[alg].wk) {
        *ctas = c->ctas_chan;
        return c->geo_chan;
    }
    if (omega && alg == 0 && c->geo[0].wk) {
        *ctas = c->ctas_omega;
        return c->geo_omega;
    }
    *ctas = c->ctas_per_sm[alg];
    return c->geo[alg];
}

cbp::KernelArgs base_args(const cbp_code* c, int alg = 0, bool chan = false, bool omega = false)
{
    cbp::KernelArgs a{};
    cbp::DevCode& d = a.code;
    int ctas = 0;
    const cbp::Geometry& G = geo_for(c, alg, chan, omega, &ctas);
    d.N = c->N; d.K = c->K; d.M = c->M; d.Z = c->Z; d.mb = c->mb; d.nb = c->nb; d.kb = c->kb; d.core = c->core;
    d.nent = c->nent; d.E = static_cast<int32_t>(c->E); d.nwords = (c->N + 31) / 32; d.kwords = (c->K + 31) / 32;
    d.max_dc = c->max_dc; d.can_encode = c->can_encode; d.mid = c->mid;
    d.phi_tab = c->phi_tab;
    d.phi_tex = static_cast<unsigned long long>(c->phi_tex);
    std::memcpy(a.ent, c->ent[alg].data(), sizeof(int4) * c->ent[alg].size());
    a.ent_dev = c->ent_dev[alg];
    a.lanes = G.lanes;
    std::memcpy(a.row_ptr, c->row_ptr.data(), sizeof(int32_t) * c->row_ptr.size());
    std::memcpy(a.pshift, c->pshift.data(), sizeof(int16_t) * c->pshift.size());
    a.Zp = G.Zp; a.F = G.F; a.slot_words = G.slot_words; a.table_words = G.table_words;
    a.ctl_words = G.ctl_words; a.fast_syn = G.fast_syn;
    a.r_words = G.r_words;
    a.team_threads = G.team_threads;
    a.phi_m19 = 0x7ffffu;
    a.phi_one = 0x3f800000u;
    a.max_iter = 1; a.stop_rule = 0;
    a.alpha = 1.0f;
    return a;
}

cbp_status check_opts(const cbp_code* c, const cbp_opts* o)
{
    if (!o) return fail(CBP_E_INVALID, "null opts");
    if (o->max_iter < 1 || o->max_iter > 65535) return fail(CBP_E_INVALID, "opts.max_iter must be in [1, 65535]");
    if (o->stop_rule < 0 || o->stop_rule > 3) return fail(CBP_E_INVALID, "opts.stop_rule must be in [0, 3]");
    if (o->algorithm < CBP_ALG_LOG_TANH || o->algorithm > CBP_ALG_FBP)
        return fail(CBP_E_INVALID, "opts.algorithm must be a cbp_algorithm (0..3)");
    if ((o->algorithm == CBP_ALG_LBP || o->algorithm == CBP_ALG_FBP) && o->stop_rule != CBP_STOP_SYNDROME &&
        o->stop_rule != CBP_STOP_NONE)
        return fail(CBP_E_INVALID, "layered / flooding BP take the stop rules CBP_STOP_SYNDROME or CBP_STOP_NONE");
    if (o->algorithm == CBP_ALG_MIN_SUM) {
        if (!(o->alpha > 0.0f && o->alpha <= 1.0f)) return fail(CBP_E_INVALID, "opts.alpha must be in (0, 1]");
        if (c->min_dc < 2) return fail(CBP_E_UNSUPPORTED, "min-sum needs every base row degree >= 2");
    }
    return CBP_OK;
}

// allocate the work queue (+ global state), launch, release -- all stream-ordered
cbp_status run(const cbp_code* c, cbp::KernelArgs& a, int64_t frames, void* stream, const char* who)
{
    DeviceGuard g(c->device);
    if (!g.ok) return fail(CBP_E_CUDA, std::string(who) + ": cudaSetDevice failed");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int ctas = 1;
    const cbp::Geometry& G = geo_for(c, a.algorithm, a.mode == cbp::MODE_CHANNEL, a.omega != nullptr, &ctas);
    const int64_t per_cta = static_cast<int64_t>(G.F) * G.teams * G.P;
    const int64_t ctas_needed = (frames + per_cta - 1) / per_cta;
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(static_cast<int64_t>(c->num_sms) * ctas, ctas_needed)));
    cudaError_t e;
    unsigned long long* q = nullptr;
    cudaMemPool_t pool = work_pool(c->device);
    auto alloc = [&](void** p, size_t bytes) {
        return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
    };
    if ((e = alloc(reinterpret_cast<void**>(&q), sizeof(unsigned long long))) != cudaSuccess)
        return fail(CBP_E_NOMEM, std::string(who) + ": " + cudaGetErrorString(e));
    float* gs = nullptr;
    if (!G.state_in_smem || G.r_global) {
        // all-global layout: whole groups; split layout: the R sections only
        const size_t words = G.state_in_smem && G.r_global ? G.r_words : G.slot_words;
        const size_t bytes = sizeof(float) * static_cast<size_t>(grid) * G.F * G.teams * words;
        if ((e = alloc(reinterpret_cast<void**>(&gs), bytes)) != cudaSuccess) {
            cudaFreeAsync(q, st);
            return fail(CBP_E_NOMEM, std::string(who) + ": " + cudaGetErrorString(e));
        }
    }
    a.queue = q;
    a.gstate = G.state_in_smem ? nullptr : gs;
    a.rstate = G.state_in_smem ? gs : nullptr;
    e = cudaMemsetAsync(q, 0, sizeof(unsigned long long), st);
    int le = (e == cudaSuccess) ? cbp::launch_cbp(a, G, grid, stream) : static_cast<int>(e);
    cudaFreeAsync(q, st);
    if (gs) cudaFreeAsync(gs, st);
    if (le != 0) return cuda_fail(static_cast<cudaError_t>(le), who);
    return CBP_OK;
}

// decode of fp32 LLRs + error counting against the transmitted codewords (MODE_BER_LLR; arguments checked)
cbp_status ber_count_launch(const cbp_code* c, const float* llr, int64_t ld, const uint32_t* cw, int64_t ld_words,
                            int64_t frames, const cbp_opts* opts, cbp_counts* counts, void* stream, const char* who)
{
    cbp::KernelArgs a = base_args(c, opts->algorithm);
    a.mode = cbp::MODE_BER_LLR;
    a.max_iter = opts->max_iter;
    a.stop_rule = opts->stop_rule;
    a.algorithm = opts->algorithm;
    a.alpha = opts->alpha;
    a.frames = frames;
    a.llr = llr;
    a.ld = ld;
    a.cw_in = cw;
    a.ld_words = ld_words;
    a.counts = reinterpret_cast<unsigned long long*>(counts);
    return run(c, a, frames, stream, who);
}

// cbp_ber_sim as channel + decode launches through an HBM chunk (codes on cbp_warp_kernel with one
// frame per warp); CBP_BER_SPLIT=0|1 overrides (A/B runs), CBP_BER_CHUNK sets the frames per chunk
bool ber_split(const cbp_code* c, int alg)
{
    const cbp::Geometry& G = c->geo[alg];
    if (!G.wk) return false;
    static const int env = [] { const char* e = std::getenv("CBP_BER_SPLIT"); return e && *e ? std::atoi(e) : -1; }();
    if (env >= 0) return env != 0;
    return !G.multi;
}

int64_t ber_chunk_frames()
{
    static const int64_t env = [] { const char* e = std::getenv("CBP_BER_CHUNK"); return e ? std::atoll(e) : 0LL; }();
    return env > 0 ? env : (int64_t{1} << 20);
}

void channel_params(const cbp_code* c, double ebn0_db, float* sigma, float* scale)
{
    // sigma^2 = 1 / (2 R 10^(Eb/N0 / 10)), R = K/N; L = 2 y / sigma^2 (reading R17)
    const double R = static_cast<double>(c->K) / static_cast<double>(c->N);
    const double sigma2 = 1.0 / (2.0 * R * std::pow(10.0, ebn0_db / 10.0));
    *sigma = static_cast<float>(std::sqrt(sigma2));
    *scale = static_cast<float>(2.0 / sigma2);
}

cbp_status decode_common(const cbp_code* c, const void* in, int32_t mode, int64_t ld, float scale, int64_t frames,
                         const cbp_opts* opts, uint32_t* d_bits, int64_t ld_words, int32_t* d_iters, uint8_t* d_flags,
                         float* d_omega, int64_t* d_ev, void* stream, const char* who)
{
    if (!c) return fail(CBP_E_INVALID, std::string(who) + ": null code");
    cbp_status s = check_opts(c, opts);
    if (s != CBP_OK) return s;
    if (frames < 0) return fail(CBP_E_INVALID, std::string(who) + ": frames < 0");
    if (frames == 0) return CBP_OK;
    if (!in || !d_bits || !d_iters || !d_flags) return fail(CBP_E_INVALID, std::string(who) + ": null buffer");
    const int64_t esz = (mode == cbp::MODE_DECODE_I8) ? 1 : 4;
    if (ld < c->N || (ld * esz) % 16 != 0) return fail(CBP_E_INVALID, std::string(who) + ": need ld >= N and ld*elem % 16 == 0");
    if (reinterpret_cast<uintptr_t>(in) % 16 != 0) return fail(CBP_E_INVALID, std::string(who) + ": input not 16-byte aligned");
    if (ld_words < (c->N + 31) / 32) return fail(CBP_E_INVALID, std::string(who) + ": ld_words < ceil(N/32)");
    if (mode == cbp::MODE_DECODE_I8 && !(std::isfinite(scale) && scale > 0.0f))
        return fail(CBP_E_INVALID, std::string(who) + ": scale must be finite and > 0");
    cbp::KernelArgs a = base_args(c, opts->algorithm, false, d_omega != nullptr);
    a.mode = mode;
    a.max_iter = opts->max_iter;
    a.stop_rule = opts->stop_rule;
    a.algorithm = opts->algorithm;
    a.alpha = opts->alpha;
    a.llr = static_cast<const float*>(in);
    a.q = static_cast<const int8_t*>(in);
    a.ld = ld;
    a.qscale = scale;
    a.frames = frames;
    a.bits = d_bits;
    a.ld_words = ld_words;
    a.iters = d_iters;
    a.flags = d_flags;
    a.omega = d_omega;
    a.ev = d_ev;
    return run(c, a, frames, stream, who);
}

// Host-buffer decode (include/cbp.h cbp_decode_host): chunks of `chunk` frames round-robin over
// `ns` streams, each chunk H2D -> decode kernel -> D2H on its stream (stream order makes the reuse
// of a stream's device buffers safe); blocks until all streams are done.
cbp_status decode_host_common(const cbp_code* c, const void* h_in, int32_t mode, int64_t ld, float scale,
                              int64_t frames, const cbp_opts* opts, uint32_t* h_bits, int64_t ld_words,
                              int32_t* h_iters, uint8_t* h_flags, int64_t chunk, int32_t ns, const char* who)
{
    if (!c) return fail(CBP_E_INVALID, std::string(who) + ": null code");
    cbp_status s = check_opts(c, opts);
    if (s != CBP_OK) return s;
    if (frames < 0) return fail(CBP_E_INVALID, std::string(who) + ": frames < 0");
    if (chunk < 0 || ns < 0 || ns > 16) return fail(CBP_E_INVALID, std::string(who) + ": need chunk_frames >= 0, 0 <= nstreams <= 16");
    if (frames == 0) return CBP_OK;
    if (!h_in || !h_bits || !h_iters || !h_flags) return fail(CBP_E_INVALID, std::string(who) + ": null buffer");
    const int64_t esz = (mode == cbp::MODE_DECODE_I8) ? 1 : 4;
    if (ld < c->N || (ld * esz) % 16 != 0) return fail(CBP_E_INVALID, std::string(who) + ": need ld >= N and ld*elem % 16 == 0");
    if (ld_words < (c->N + 31) / 32) return fail(CBP_E_INVALID, std::string(who) + ": ld_words < ceil(N/32)");
    if (mode == cbp::MODE_DECODE_I8 && !(std::isfinite(scale) && scale > 0.0f))
        return fail(CBP_E_INVALID, std::string(who) + ": scale must be finite and > 0");
    if (chunk == 0) chunk = 1 << 14;
    if (ns == 0) ns = 4;
    chunk = std::min(chunk, frames);
    const int64_t nchunks = (frames + chunk - 1) / chunk;
    ns = static_cast<int32_t>(std::min<int64_t>(ns, nchunks));
    DeviceGuard g(c->device);
    if (!g.ok) return fail(CBP_E_CUDA, std::string(who) + ": cudaSetDevice failed");
    cudaMemPool_t pool = work_pool(c->device);
    struct Slot {
        cudaStream_t st = nullptr;
        void* in = nullptr;
        uint32_t* bits = nullptr;
        int32_t* iters = nullptr;
        uint8_t* flags = nullptr;
    };
    std::vector<Slot> slots(ns);
    cudaError_t e = cudaSuccess;
    auto alloc = [&](void** p, size_t bytes, cudaStream_t st) {
        return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
    };
    for (auto& sl : slots) {
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = alloc(&sl.in, static_cast<size_t>(chunk * ld * esz), sl.st);
        if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&sl.bits), static_cast<size_t>(chunk * ld_words * 4), sl.st);
        if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&sl.iters), static_cast<size_t>(chunk * 4), sl.st);
        if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&sl.flags), static_cast<size_t>((chunk + 15) / 16 * 16), sl.st);
    }
    cbp_status rs = (e == cudaSuccess) ? CBP_OK : fail(CBP_E_NOMEM, std::string(who) + ": " + cudaGetErrorString(e));
    const char* src = static_cast<const char*>(h_in);
    for (int64_t k = 0; k < nchunks && rs == CBP_OK; ++k) {
        Slot& sl = slots[k % ns];
        const int64_t b = k * chunk, n = std::min(chunk, frames - b);
        e = cudaMemcpyAsync(sl.in, src + b * ld * esz, static_cast<size_t>(n * ld * esz), cudaMemcpyHostToDevice, sl.st);
        if (e != cudaSuccess) { rs = cuda_fail(e, who); break; }
        rs = decode_common(c, sl.in, mode, ld, scale, n, opts, sl.bits, ld_words, sl.iters, sl.flags, nullptr, nullptr,
                           sl.st, who);
        if (rs != CBP_OK) break;
        e = cudaMemcpyAsync(h_bits + b * ld_words, sl.bits, static_cast<size_t>(n * ld_words * 4), cudaMemcpyDeviceToHost, sl.st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h_iters + b, sl.iters, static_cast<size_t>(n * 4), cudaMemcpyDeviceToHost, sl.st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h_flags + b, sl.flags, static_cast<size_t>(n), cudaMemcpyDeviceToHost, sl.st);
        if (e != cudaSuccess) rs = cuda_fail(e, who);
    }
    for (auto& sl : slots) {
        if (!sl.st) continue;
        for (void* p : {sl.in, static_cast<void*>(sl.bits), static_cast<void*>(sl.iters), static_cast<void*>(sl.flags)})
            if (p) cudaFreeAsync(p, sl.st);
        const cudaError_t se = cudaStreamSynchronize(sl.st);
        if (se != cudaSuccess && rs == CBP_OK) rs = cuda_fail(se, who);
        cudaStreamDestroy(sl.st);
    }
    return rs;
}

}  // namespace

extern "C" {

cbp_status cbp_decode_host(const cbp_code* c, const float* h_llr, int64_t ld, int64_t frames, const cbp_opts* opts,
                           uint32_t* h_bits, int64_t ld_words, int32_t* h_iters, uint8_t* h_flags,
                           int64_t chunk_frames, int32_t nstreams)
{
    return decode_host_common(c, h_llr, cbp::MODE_DECODE_F32, ld, 1.0f, frames, opts, h_bits, ld_words, h_iters,
                              h_flags, chunk_frames, nstreams, "cbp_decode_host");
}

cbp_status cbp_decode_host_i8(const cbp_code* c, const int8_t* h_q, int64_t ld, float scale, int64_t frames,
                              const cbp_opts* opts, uint32_t* h_bits, int64_t ld_words, int32_t* h_iters,
                              uint8_t* h_flags, int64_t chunk_frames, int32_t nstreams)
{
    return decode_host_common(c, h_q, cbp::MODE_DECODE_I8, ld, scale, frames, opts, h_bits, ld_words, h_iters,
                              h_flags, chunk_frames, nstreams, "cbp_decode_host_i8");
}

cbp_status cbp_decode(const cbp_code* c, const float* d_llr, int64_t ld, int64_t frames, const cbp_opts* opts,
                      uint32_t* d_bits, int64_t ld_words, int32_t* d_iters, uint8_t* d_flags, float* d_omega,
                      int64_t* d_ev, void* stream)
{
    return decode_common(c, d_llr, cbp::MODE_DECODE_F32, ld, 1.0f, frames, opts, d_bits, ld_words, d_iters, d_flags,
                         d_omega, d_ev, stream, "cbp_decode");
}

cbp_status cbp_decode_i8(const cbp_code* c, const int8_t* d_q, int64_t ld, float scale, int64_t frames,
                         const cbp_opts* opts, uint32_t* d_bits, int64_t ld_words, int32_t* d_iters, uint8_t* d_flags,
                         float* d_omega, int64_t* d_ev, void* stream)
{
    return decode_common(c, d_q, cbp::MODE_DECODE_I8, ld, scale, frames, opts, d_bits, ld_words, d_iters, d_flags,
                         d_omega, d_ev, stream, "cbp_decode_i8");
}

cbp_status cbp_channel(const cbp_code* c, double ebn0_db, uint64_t seed, int64_t frame_begin, int64_t frames,
                       int32_t llr_mode, float* d_llr, int64_t ld, uint32_t* d_cw, int64_t ld_words, void* stream)
{
    if (!c) return fail(CBP_E_INVALID, "cbp_channel: null code");
    if (frames < 0 || frame_begin < 0) return fail(CBP_E_INVALID, "cbp_channel: negative frame range");
    if (llr_mode < 0 || llr_mode > 3) return fail(CBP_E_INVALID, "cbp_channel: llr_mode must be 0..3");
    if (!(llr_mode & CBP_TX_ZERO) && !c->can_encode)
        return fail(CBP_E_UNSUPPORTED, "cbp_channel: base has no dual-diagonal encoder structure (use CBP_TX_ZERO)");
    if (!std::isfinite(ebn0_db)) return fail(CBP_E_INVALID, "cbp_channel: ebn0_db not finite");
    if (frames == 0) return CBP_OK;
    if (!d_llr && !d_cw) return fail(CBP_E_INVALID, "cbp_channel: both outputs NULL");
    if (d_llr && ld < c->N) return fail(CBP_E_INVALID, "cbp_channel: ld < N");
    if (d_cw && ld_words < (c->N + 31) / 32) return fail(CBP_E_INVALID, "cbp_channel: ld_words < ceil(N/32)");
    cbp::KernelArgs a = base_args(c, 0, true);
    a.mode = cbp::MODE_CHANNEL;
    a.frames = frames;
    a.frame_begin = frame_begin;
    a.seed = seed;
    a.llr_mode = llr_mode;
    channel_params(c, ebn0_db, &a.sigma, &a.scale);
    a.llr_out = d_llr;
    a.ld = ld;
    a.cw_out = d_cw;
    a.ld_words = ld_words;
    return run(c, a, frames, stream, "cbp_channel");
}

cbp_status cbp_ber_count(const cbp_code* c, const float* d_llr, int64_t ld, const uint32_t* d_cw, int64_t ld_words,
                         int64_t frames, const cbp_opts* opts, cbp_counts* d_counts, void* stream)
{
    if (!c) return fail(CBP_E_INVALID, "cbp_ber_count: null code");
    cbp_status s = check_opts(c, opts);
    if (s != CBP_OK) return s;
    if (!c->geo[opts->algorithm].wk)
        return fail(CBP_E_UNSUPPORTED, "cbp_ber_count: needs a code on cbp_warp_kernel (17 <= Z <= 384; log-tanh CBP or layered BP)");
    if (frames < 0) return fail(CBP_E_INVALID, "cbp_ber_count: frames < 0");
    if (frames == 0) return CBP_OK;
    if (!d_llr || !d_cw || !d_counts) return fail(CBP_E_INVALID, "cbp_ber_count: null buffer");
    if (ld < c->N || ld % 4 != 0) return fail(CBP_E_INVALID, "cbp_ber_count: need ld >= N and ld % 4 == 0");
    if (reinterpret_cast<uintptr_t>(d_llr) % 16 != 0) return fail(CBP_E_INVALID, "cbp_ber_count: llr not 16-byte aligned");
    if (ld_words < (c->N + 31) / 32) return fail(CBP_E_INVALID, "cbp_ber_count: ld_words < ceil(N/32)");
    return ber_count_launch(c, d_llr, ld, d_cw, ld_words, frames, opts, d_counts, stream, "cbp_ber_count");
}

cbp_status cbp_ber_sim(const cbp_code* c, double ebn0_db, uint64_t seed, int64_t frame_begin, int64_t frames,
                       const cbp_opts* opts, int32_t llr_mode, cbp_counts* d_counts, void* stream)
{
    if (!c) return fail(CBP_E_INVALID, "cbp_ber_sim: null code");
    cbp_status s = check_opts(c, opts);
    if (s != CBP_OK) return s;
    if (frames < 0 || frame_begin < 0) return fail(CBP_E_INVALID, "cbp_ber_sim: negative frame range");
    if (llr_mode < 0 || llr_mode > 3) return fail(CBP_E_INVALID, "cbp_ber_sim: llr_mode must be 0..3");
    if (!(llr_mode & CBP_TX_ZERO) && !c->can_encode)
        return fail(CBP_E_UNSUPPORTED, "cbp_ber_sim: base has no dual-diagonal encoder structure (use CBP_TX_ZERO)");
    if (!std::isfinite(ebn0_db)) return fail(CBP_E_INVALID, "cbp_ber_sim: ebn0_db not finite");
    if (!d_counts) return fail(CBP_E_INVALID, "cbp_ber_sim: null counts");
    if (frames == 0) return CBP_OK;
    cbp::KernelArgs a = base_args(c, opts->algorithm);
    a.mode = cbp::MODE_BER_SIM;
    a.max_iter = opts->max_iter;
    a.stop_rule = opts->stop_rule;
    a.algorithm = opts->algorithm;
    a.alpha = opts->alpha;
    a.frames = frames;
    a.frame_begin = frame_begin;
    a.seed = seed;
    a.llr_mode = llr_mode;
    channel_params(c, ebn0_db, &a.sigma, &a.scale);
    a.counts = reinterpret_cast<unsigned long long*>(d_counts);
    if (!ber_split(c, opts->algorithm)) return run(c, a, frames, stream, "cbp_ber_sim");
    // split: per chunk of frames, a channel-only launch writes L and the codewords to a workspace in HBM
    // and a MODE_BER_LLR launch decodes and counts them.  Same kernel, same frames and arithmetic as the
    // fused launch (bit-identical counters); the per-frame channel code then no longer shares the SM's
    // instruction cache with the hot row bodies.
    DeviceGuard g(c->device);
    if (!g.ok) return fail(CBP_E_CUDA, "cbp_ber_sim: cudaSetDevice failed");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t chunk = std::min<int64_t>(frames, ber_chunk_frames());
    const int64_t ld = (c->N + 3) / 4 * 4, ldw = (c->N + 31) / 32;   // 16-byte rows: 128-bit LLR loads
    float* llr = nullptr;
    uint32_t* cw = nullptr;
    cudaMemPool_t pool = work_pool(c->device);
    auto alloc = [&](void** p, size_t bytes) {
        return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
    };
    cudaError_t e = alloc(reinterpret_cast<void**>(&llr), sizeof(float) * static_cast<size_t>(chunk * ld));
    if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&cw), sizeof(uint32_t) * static_cast<size_t>(chunk * ldw));
    if (e != cudaSuccess) {
        if (llr) cudaFreeAsync(llr, st);
        return fail(CBP_E_NOMEM, std::string("cbp_ber_sim: ") + cudaGetErrorString(e));
    }
    cbp_status s2 = CBP_OK;
    for (int64_t f0 = 0; f0 < frames && s2 == CBP_OK; f0 += chunk) {
        const int64_t n = std::min(chunk, frames - f0);
        cbp::KernelArgs ch = a;
        ch.mode = cbp::MODE_CHANNEL;
        ch.frames = n;
        ch.frame_begin = frame_begin + f0;
        ch.llr_out = llr;
        ch.ld = ld;
        ch.cw_out = cw;
        ch.ld_words = ldw;
        ch.counts = nullptr;
        s2 = run(c, ch, n, stream, "cbp_ber_sim (channel)");
        if (s2 != CBP_OK) break;
        s2 = ber_count_launch(c, llr, ld, cw, ldw, n, opts, d_counts, stream, "cbp_ber_sim");
    }
    cudaFreeAsync(llr, st);
    cudaFreeAsync(cw, st);
    return s2;
}

cbp_status cbp_eval_contract(int32_t fn, const float* d_x, float* d_y, int64_t n, int32_t device, void* stream)
{
    if (fn < 0 || fn > 3) return fail(CBP_E_INVALID, "cbp_eval_contract: fn must be 0..3");
    if (n < 0 || (n > 0 && (!d_x || !d_y))) return fail(CBP_E_INVALID, "cbp_eval_contract: bad buffers");
    DeviceGuard g(device);
    if (!g.ok) return fail(CBP_E_CUDA, "cbp_eval_contract: cudaSetDevice failed");
    std::string terr;
    const float4* tab = phi_table(device, &terr);
    if (!tab) return fail(CBP_E_CUDA, "cbp_eval_contract: " + terr);
    const int e = cbp::launch_contract_eval(fn, d_x, d_y, n, tab, stream);
    if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cbp_eval_contract");
    return CBP_OK;
}

cbp_status cbp_phi_table(int32_t device, float* d_out, void* stream)
{
    if (!d_out) return fail(CBP_E_INVALID, "cbp_phi_table: null output");
    std::string terr;
    const float4* tab = phi_table(device, &terr);
    if (!tab) return fail(CBP_E_CUDA, "cbp_phi_table: " + terr);
    DeviceGuard g(device);
    const cudaError_t e = cudaMemcpyAsync(d_out, tab, sizeof(float4) * cbp::kPhiTableSegs, cudaMemcpyDeviceToDevice,
                                          static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cbp_phi_table");
    return CBP_OK;
}

}  // extern "C"
