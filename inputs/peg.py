"""Seeded quasi-cyclic progressive-edge-growth (QC-PEG) constructor for the paper's own
code families (§V: "regular (3,6) LDPC codes and irregular LDPC codes
under degree distributions lambda(x) = 0.45x + 0.3708x^2 + 0.0307x^3 + 0.1485x^11,
rho(x) = 0.5467x^4 + 0.4533x^5 ... constructed using the progress edge growth (PEG)
algorithm [24] ... rate-1/2"; Fig. 6/7: lengths 2048 and 8192).

Input generator only (no decoder arithmetic): it returns a QC base matrix in the
same format as inputs.construct_base, which the GPU path and the oracle consume alike.

The paper's matrices are not available, so this regenerates the ENSEMBLE, not the
codes: PEG (Hu, Eleftheriou, Arnold) run on the base graph of a QC lifting, the
common "QC-PEG" variant.  Edges are placed column by column in nondecreasing degree
order; the first edge of a column goes to a lowest-degree base row with a seeded
random shift, every further edge to a lifted check that is unreachable from the
column's offset-0 variable, else reached at the deepest BFS level (maximising the
local girth), among those in a lowest-degree row.  By the QC symmetry, BFS from the
offset-0 variable of a column describes every variable of it.  The BFS runs on
Z-bit offset masks per base node (one rotation per base edge per level).

Degree distributions are edge-perspective (lambda_i = fraction of edges on degree-i
variables); node counts are lambda_i / i normalised and rounded by largest
remainder.  The check degrees follow from the edge count: E - 5 mb rows of degree 6,
the rest degree 5, assigned by a seeded shuffle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M64 = (1 << 64) - 1


class _SplitMix64:
    """SplitMix64 with rejection sampling, as in inputs/qc_construct.c."""

    def __init__(self, seed: int):
        self.s = seed & _M64

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & _M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def below(self, n: int) -> int:
        bound = (_M64 // n) * n
        while True:
            x = self.next()
            if x < bound:
                return x % n


def node_counts(n: int, lam: dict) -> dict:
    """Edge-perspective {degree: lambda_d} -> {degree: node count} summing to n."""
    w = {d: lam[d] / d for d in lam}
    tot = sum(w.values())
    exact = {d: n * w[d] / tot for d in lam}
    cnt = {d: int(np.floor(exact[d])) for d in lam}
    rest = n - sum(cnt.values())
    for d in sorted(lam, key=lambda d: (-(exact[d] - cnt[d]), d))[:rest]:
        cnt[d] += 1
    return cnt


def _rotl(m: int, k: int, Z: int, full: int) -> int:
    k %= Z
    return ((m << k) | (m >> (Z - k))) & full if k else m


def qc_peg(mb: int, nb: int, Z: int, col_deg, row_deg, seed: int) -> np.ndarray:
    """QC-PEG base matrix int16[mb, nb] (-1 = zero block, s = shift; check row r of
    block (i, j) <-> variable j*Z + (r + s) % Z, as inputs.construct_base)."""
    col_deg, row_deg = list(col_deg), list(row_deg)
    if len(col_deg) != nb or len(row_deg) != mb or sum(col_deg) != sum(row_deg):
        raise ValueError("qc_peg: degree sequences do not match the base size / edge count")
    if max(col_deg) > mb or max(row_deg) > nb or min(col_deg) < 1 or min(row_deg) < 1:
        raise ValueError("qc_peg: degree out of range")
    rng = _SplitMix64(seed)
    full = (1 << Z) - 1
    base = -np.ones((mb, nb), np.int64)
    col_ent = [[] for _ in range(nb)]     # (row, shift)
    row_ent = [[] for _ in range(mb)]     # (col, shift)
    rdeg = [0] * mb
    for j in sorted(range(nb), key=lambda j: (col_deg[j], j)):
        for k in range(col_deg[j]):
            open_rows = [i for i in range(mb) if rdeg[i] < row_deg[i] and base[i, j] < 0]
            if not open_rows:
                raise ValueError("qc_peg: no open row (degree sequences infeasible)")
            if k == 0:
                cand = {i: full for i in open_rows}
            else:
                cand = _deepest(j, col_ent, row_ent, mb, nb, Z, full, open_rows)
            dmin = min(rdeg[i] for i in cand)
            rows = [i for i in sorted(cand) if rdeg[i] == dmin]
            i = rows[rng.below(len(rows))]
            offs = [r for r in range(Z) if (cand[i] >> r) & 1]
            r = offs[rng.below(len(offs))]
            s = (Z - r) % Z                     # connects variable j*Z + 0 to check i*Z + r
            base[i, j] = s
            col_ent[j].append((i, s))
            row_ent[i].append((j, s))
            rdeg[i] += 1
    return base.astype(np.int16)


def _deepest(j, col_ent, row_ent, mb, nb, Z, full, open_rows) -> dict:
    """{row: offset mask} of the PEG candidates for the next edge of column j: lifted
    checks of open rows not reachable from variable j*Z, else those first reached at
    the deepest BFS level."""
    vreach = [0] * nb
    creach = [0] * mb
    vreach[j] = 1
    vfront = {j: 1}
    levels = []                                   # per level: {row: newly reached mask}
    while vfront:
        cnew = {}
        for jj, m in vfront.items():
            for i, s in col_ent[jj]:
                cm = _rotl(m, -s, Z, full) & ~creach[i] & full   # variable offset t -> check offset t - s
                if cm:
                    cnew[i] = cnew.get(i, 0) | cm
        if not cnew:
            break
        for i, cm in cnew.items():
            creach[i] |= cm
        levels.append(cnew)
        vnext = {}
        for i, cm in cnew.items():
            for jj, s in row_ent[i]:
                vm = _rotl(cm, s, Z, full) & ~vreach[jj] & full
                if vm:
                    vnext[jj] = vnext.get(jj, 0) | vm
        for jj, vm in vnext.items():
            vreach[jj] |= vm
        vfront = vnext
    unreached = {i: full & ~creach[i] for i in open_rows if full & ~creach[i]}
    if unreached:
        return unreached
    for lev in reversed(levels):
        cand = {i: lev[i] for i in open_rows if lev.get(i, 0)}
        if cand:
            return cand
    raise ValueError("qc_peg: no candidate check")   # unreachable: open rows are reached at some level


@dataclass(frozen=True)
class PegConfig:
    """One of the paper's own code families as a QC-PEG ensemble member."""
    name: str
    mb: int
    nb: int
    Z: int
    lam: tuple             # edge-perspective ((degree, lambda_d), ...)
    code_seed: int
    ebn0_db: tuple
    frames: int
    max_iter: int          # "The maximum number of iterations is 200."


# PAPER.md l.608 and Fig. 6/7: N = 2048 regular (3,6) and N = 8192 irregular, rate 1/2.
PEG_CONFIGS = {
    "P2048": PegConfig("P2048", 32, 64, 32, ((3, 1.0),), 1, (1.0, 1.5, 2.0, 2.5), 100_000, 200),
    "P8192": PegConfig("P8192", 64, 128, 64, ((2, 0.45), (3, 0.3708), (4, 0.0307), (12, 0.1485)), 1,
                       (0.75, 1.0, 1.25, 1.5), 100_000, 200),
}


def peg_degrees(cfg: PegConfig, seed: int):
    """(column degrees, row degrees): columns in DEScending degree order (the heavy
    columns first, so variables 0..K-1 hold the best-protected positions, as an IRA
    information set would), row degrees 5/6 placed by a seeded shuffle."""
    cnt = node_counts(cfg.nb, dict(cfg.lam))
    col = [d for d in sorted(cnt, reverse=True) for _ in range(cnt[d])]
    E = sum(col)
    if E % cfg.mb == 0:
        row = [E // cfg.mb] * cfg.mb
    else:
        hi = E - 5 * cfg.mb                       # rho(x) = 0.5467x^4 + 0.4533x^5: degrees 5 and 6
        if not 0 <= hi <= cfg.mb:
            raise ValueError("peg_degrees: edge count does not fit check degrees 5/6")
        row = [6] * hi + [5] * (cfg.mb - hi)
        rng = _SplitMix64(seed ^ 0x5EED)
        for a in range(cfg.mb - 1, 0, -1):        # Fisher-Yates
            b = rng.below(a + 1)
            row[a], row[b] = row[b], row[a]
    return col, row


def peg_base(name: str) -> tuple[np.ndarray, int]:
    cfg = PEG_CONFIGS[name]
    col, row = peg_degrees(cfg, cfg.code_seed)
    return qc_peg(cfg.mb, cfg.nb, cfg.Z, col, row, cfg.code_seed), cfg.Z
