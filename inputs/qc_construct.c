/*
 * qc_construct.c -- seeded QC-LDPC base-matrix constructor (SURVEY.md
 * Appendix B; BASELINE.json configs).  Input generator only: no decoding,
 * channel or encoding arithmetic lives here.
 *
 * Procedure (frozen; golden hashes in tests/golden/base_hashes.txt):
 *   rng = SplitMix64(seed)
 *   for info column j = 0 .. kb-1 (ascending):
 *     w   = weight rule (CBP_W_*)
 *     key = one fresh 64-bit draw per base row (rows 0..mb-1, ascending)
 *     pick the w rows with the smallest (row_degree, key), ascending order
 *     for the picked rows in ascending row index: shift = uniform(rng, Z)
 *   parity part (columns kb .. nb-1), 802.11n-style dual diagonal:
 *     column kb:      rows 0, floor(mb_core/2), mb_core-1 with shifts 1, 0, 1
 *     column kb+t:    rows t-1 and t, shift 0            (t = 1 .. mb_core-1)
 *     column kb+mb_core+k: row mb_core+k, shift 0 (degree-1 extension)
 */
#include "cbp_inputs.h"
#include <string.h>

static uint64_t splitmix64(uint64_t* s)
{
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* uniform integer in [0, n) by rejection (no modulo bias) */
static uint32_t uniform_below(uint64_t* s, uint32_t n)
{
    const uint64_t bound = (UINT64_MAX / n) * n;
    uint64_t x;
    do {
        x = splitmix64(s);
    } while (x >= bound);
    return (uint32_t)(x % n);
}

int cbp_inputs_construct_base(const cbp_inputs_spec* sp, uint64_t seed,
                              int16_t* base, const char** err)
{
    const char* dummy;
    if (!err) err = &dummy;
    *err = "";
    if (!sp || !base) { *err = "null argument"; return 1; }
    const int mb = sp->mb, nb = sp->nb, Z = sp->Z, core = sp->mb_core;
    const int kb = nb - mb;
    if (mb < 3 || nb <= mb || mb > 256 || nb > 512) { *err = "need 3 <= mb < nb, mb <= 256, nb <= 512"; return 1; }
    if (Z < 2 || Z > 1024) { *err = "need 2 <= Z <= 1024"; return 1; }
    if (core < 3 || core > mb) { *err = "need 3 <= mb_core <= mb"; return 1; }
    if (sp->w_lo < 1 || sp->w_hi < sp->w_lo || sp->w_hi > mb) { *err = "need 1 <= w_lo <= w_hi <= mb"; return 1; }
    if (sp->wmode < CBP_W_CONST || sp->wmode > CBP_W_HEAVY) { *err = "unknown weight rule"; return 1; }

    for (int i = 0; i < mb * nb; ++i) base[i] = -1;

    uint64_t st = seed;
    int row_deg[256];
    uint64_t key[256];
    int picked[256];
    memset(row_deg, 0, sizeof(row_deg));

    for (int j = 0; j < kb; ++j) {
        int w;
        if (sp->wmode == CBP_W_CONST) {
            w = sp->w_lo;
        } else if (sp->wmode == CBP_W_UNIFORM) {
            w = sp->w_lo + (int)uniform_below(&st, (uint32_t)(sp->w_hi - sp->w_lo + 1));
        } else {
            const double u = (double)((splitmix64(&st) >> 40) + 1) * (1.0 / 16777216.0);
            double f = 3.0 / u;
            if (f > (double)sp->w_hi) f = (double)sp->w_hi;
            w = (int)f;
            if (w < sp->w_lo) w = sp->w_lo;
        }
        for (int i = 0; i < mb; ++i) { key[i] = splitmix64(&st); picked[i] = 0; }
        /* w selections of the minimum (row_deg, key) among unpicked rows.  With a
         * degree-1 extension (core < mb) the first two go to core rows and the rest
         * to extension rows, so every info bit is protected by the core (otherwise
         * an info column lying only on extension rows is a weight-4 codeword). */
        const int ncore_pick = (core < mb) ? (w < 2 ? w : 2) : w;
        for (int n = 0; n < w; ++n) {
            const int lo = (core < mb && n >= ncore_pick) ? core : 0;
            const int hi = (core < mb && n < ncore_pick) ? core : mb;
            int best = -1;
            for (int i = lo; i < hi; ++i) {
                if (picked[i]) continue;
                if (best < 0 || row_deg[i] < row_deg[best] ||
                    (row_deg[i] == row_deg[best] && key[i] < key[best]))
                    best = i;
            }
            if (best >= 0) picked[best] = 1;
        }
        for (int i = 0; i < mb; ++i) {
            if (!picked[i]) continue;
            base[i * nb + j] = (int16_t)uniform_below(&st, (uint32_t)Z);
            row_deg[i] += 1;
        }
    }
    /* dual-diagonal core */
    const int mid = core / 2;
    base[0 * nb + kb] = (int16_t)(1 % Z);
    base[mid * nb + kb] = 0;
    base[(core - 1) * nb + kb] = (int16_t)(1 % Z);
    for (int t = 1; t < core; ++t) {
        base[(t - 1) * nb + kb + t] = 0;
        base[t * nb + kb + t] = 0;
    }
    /* degree-1 extension columns */
    for (int k = 0; k < mb - core; ++k) base[(core + k) * nb + kb + core + k] = 0;
    return 0;
}

int cbp_inputs_named_spec(const char* name, cbp_inputs_spec* o)
{
    /* BASELINE.json configs */
    static const struct { const char* n; cbp_inputs_spec s; } T[] = {
        {"C1",  {6, 12, 8, 6, CBP_W_CONST, 3, 3}},
        {"C2",  {12, 24, 27, 12, CBP_W_UNIFORM, 3, 4}},
        {"C3a", {12, 24, 81, 12, CBP_W_UNIFORM, 3, 6}},
        {"C3b", {4, 24, 81, 4, CBP_W_UNIFORM, 3, 4}},
        {"C4",  {46, 68, 384, 4, CBP_W_HEAVY, 3, 30}},
        {"T24", {3, 6, 4, 3, CBP_W_CONST, 2, 2}},
    };
    for (unsigned i = 0; i < sizeof(T) / sizeof(T[0]); ++i) {
        if (strcmp(T[i].n, name) == 0) { *o = T[i].s; return 0; }
    }
    return 1;
}
