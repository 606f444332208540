"""Complexity and memory accounting of the paper (NEXT-4): PAPER.md §V (l.740-900), Tables I-VI.

Analytic side -- the paper's closed forms for a code with E edges and edge-perspective degree
distributions lambda(x) = sum_i lambda_i x^(d_v^i - 1), rho(x) = sum_j rho_j x^(d_c^j - 1):
  * Table I   (l.750-767)  updates per iteration by kind: V2C, C2V, B2V, C2B, residual,
                            comparison, dispatching, CI;
  * Table II  (l.775-793)  calculations per update (sums, products, comparisons, selections);
  * Table III (l.797-822)  total per iteration with the convergence speeds 1, 1/2, 1/2, 1/4,
                            1/4, 1/6 of FBP, LBP, CBP, RBP, SVNF-RBP, CI-RBP (l.797);
  * Tables IV / V (l.834-866) Table III evaluated for the (3,6) code and the irregular ensemble;
  * Table VI  (l.872-887)  memory cells, and the 5G-NR-like register example of l.898.
The RBP-family rows are the paper's formulas only (those decoders are comparison systems and
out of scope); CBP, LBP and FBP are also MEASURED on the GPU.

Measured side -- `measured_updates`: the decoders count every edge visit in the kernel (the
cbp_decode `d_ev` output / ber_sim counter 5).  One edge visit is, by construction of each
schedule, exactly one update of each of its kinds (CBP: one B2V, one V2C, one C2B; LBP / FBP:
one V2C and one C2V, plus the dispatching of a row / column), so the per-kind counts of a run
are the edge visits, and per iteration they are edge visits / sweeps.  `verify_counters`
compares them with Table I (deviation 0 for FBP / LBP / CBP).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SCHEDULES = ("FBP", "LBP", "RBP", "SVNF-RBP", "CI-RBP", "CBP")
KINDS = ("V2C", "C2V", "B2V", "C2B", "Residual", "Comparison", "Dispatching", "CI")
# convergence speed of each schedule relative to FBP
CONVERGENCE = {"FBP": 1.0, "LBP": 0.5, "CBP": 0.5, "RBP": 0.25, "SVNF-RBP": 0.25, "CI-RBP": 1.0 / 6.0}


@dataclass(frozen=True)
class Ensemble:
    """Edge-perspective degree distributions: lam[d_v] = lambda_i of variable degree d_v,
    rho[d_c] = rho_j of check degree d_c (fractions of the E edges)."""
    lam: dict
    rho: dict

    @property
    def max_dv(self) -> int:
        return max(self.lam)

    @property
    def max_dc(self) -> int:
        return max(self.rho)


# the paper's ensembles: regular (3,6) and the irregular rate-1/2 pair
REGULAR_36 = Ensemble({3: 1.0}, {6: 1.0})
IRREGULAR = Ensemble({2: 0.45, 3: 0.3708, 4: 0.0307, 12: 0.1485}, {5: 0.5467, 6: 0.4533})


def ensemble_of_code(chk: np.ndarray, var: np.ndarray) -> Ensemble:
    """Edge-perspective distributions of a concrete code graph (edge lists)."""
    dv = np.bincount(var)
    dc = np.bincount(chk)
    E = len(chk)
    lam = {int(d): float((dv == d).sum() * d / E) for d in np.unique(dv) if d > 0}
    rho = {int(d): float((dc == d).sum() * d / E) for d in np.unique(dc) if d > 0}
    return Ensemble(lam, rho)


def _sum_v(ens: Ensemble, f) -> float:
    return sum(l * f(d) for d, l in ens.lam.items())


def _sum_vc(ens: Ensemble, f) -> float:
    return sum(l * r * f(dv, dc) for dv, l in ens.lam.items() for dc, r in ens.rho.items())


def updates_per_iteration(schedule: str, E: float, ens: Ensemble) -> dict:
    """Table I: average updates of each kind in one iteration."""
    z = {k: 0.0 for k in KINDS}
    if schedule in ("FBP", "LBP"):
        z.update(V2C=E, C2V=E, Dispatching=E)
    elif schedule in ("RBP", "SVNF-RBP", "CI-RBP"):
        z.update(V2C=E * _sum_v(ens, lambda dv: dv - 1), C2V=E,
                 Residual=E * _sum_vc(ens, lambda dv, dc: (dv - 1) * (dc - 1)), Comparison=E * (E - 1))
        if schedule == "CI-RBP":
            z["CI"] = E * (E - 1)
    elif schedule == "CBP":
        z.update(V2C=E, B2V=E, C2B=E)
    else:
        raise ValueError(schedule)
    return z


def calculations_per_update(schedule: str, dv: float, dc: float, max_dv: int, max_dc: int) -> dict:
    """Table II for a variable of degree dv / check of degree dc:
    {kind: (operation, count)}; the dispatching count is the max degree of the row/column."""
    if schedule == "FBP":
        return {"V2C": ("sums", 2), "C2V": ("products", 2), "Dispatching": ("selections", max(max_dv, max_dc))}
    if schedule == "LBP":
        return {"V2C": ("sums", 2), "C2V": ("products", 2), "Dispatching": ("selections", max_dc)}
    if schedule in ("RBP", "SVNF-RBP", "CI-RBP"):
        d = {"V2C": ("sums", dv - 1), "C2V": ("products", dc - 1), "Residual": ("products", dc - 1),
             "Comparison": ("comparisons", 1)}
        if schedule == "CI-RBP":
            d["CI"] = ("products", 2)
        return d
    if schedule == "CBP":
        return {"V2C": ("sums", 2), "B2V": ("products", 1), "C2B": ("products", 1)}
    raise ValueError(schedule)


def total_complexity(schedule: str, E: float, ens: Ensemble) -> dict:
    """Table III: sums, products, comparisons, selections per iteration,
    convergence speed applied.  Returned as coefficients times E where the paper writes them
    so (values are plain numbers for a numeric E)."""
    c = CONVERGENCE[schedule]
    if schedule == "FBP":
        return {"sums": 2 * E, "products": 2 * E, "comparisons": 0.0, "selections": E * max(ens.max_dv, ens.max_dc)}
    if schedule == "LBP":
        return {"sums": E, "products": E, "comparisons": 0.0, "selections": E * ens.max_dc / 2}
    if schedule == "CBP":
        return {"sums": E, "products": E, "comparisons": 0.0, "selections": 0.0}
    sums = E * _sum_v(ens, lambda dv: (dv - 1) ** 2) * c
    prods = (E * sum(r * (dc - 1) for dc, r in ens.rho.items()) * c +
             E * _sum_vc(ens, lambda dv, dc: (dv - 1) * (dc - 1) ** 2) * c)
    if schedule == "CI-RBP":
        prods += E * (E - 1) / 3
    return {"sums": sums, "products": prods, "comparisons": E * (E - 1) * c, "selections": 0.0}


def table_iv_v_coefficients(ens: Ensemble, E: float = 1e6) -> dict:
    """Tables IV / V: Table III divided by E (the E(E-1) terms reported
    as their E-independent remainder, e.g. CI-RBP products E(E/3 + 8.83) -> 8.83)."""
    out = {}
    for s in SCHEDULES:
        t = total_complexity(s, E, ens)
        row = {k: v / E for k, v in t.items()}
        if s == "CI-RBP":
            row["products"] = (t["products"] - E * (E - 1) / 3) / E - 1.0 / 3.0   # E(E/3 + x) = E^2/3 + xE
        row["comparisons_over_E2"] = t["comparisons"] / (E * (E - 1)) if t["comparisons"] else 0.0
        out[s] = row
    return out


def memory_cells(schedule: str, N: int, M: int, E: int, P: int, max_dv: int, max_dc: int) -> dict:
    """Table VI: general memory cells and variable-depth-pool registers."""
    pool = {"FBP": P * max(max_dv, max_dc), "LBP": P * max_dc}.get(schedule, 0)
    general = {"FBP": N + 2 * E, "LBP": N + E, "RBP": N + 3 * E, "SVNF-RBP": N + 3 * E, "CI-RBP": N + 3 * E,
               "CBP": N + E + M}[schedule]
    return {"general_cells": general, "pool_registers": pool}


def register_example_5g(P: int = 384, mb: int = 46, pool_depth: int = 19, q_bits: int = 8,
                        register_area_factor: float = 10.0) -> dict:
    """pool registers removed, check-belief bits added (as register equivalents), net saving."""
    pool_bits = P * pool_depth * q_bits
    belief_bits = P * mb * q_bits
    belief_regs = int(belief_bits // register_area_factor)
    return {"pool_register_bits": pool_bits, "check_belief_bits": belief_bits,
            "check_belief_register_equivalents": belief_regs, "net_register_saving": pool_bits - belief_regs}


# ---------------------------------------------------------------- measured counters
ALG_SCHEDULE = {0: "CBP", 1: "CBP", 2: "LBP", 3: "FBP"}


def measured_updates(algorithm: int, edge_visits: int, sweeps: int) -> dict:
    """Per-iteration updates of each kind from the kernel's exact edge-visit count of `sweeps`
    full sweeps (stop rule NONE): one edge visit = one update of each kind of the schedule."""
    per = edge_visits / sweeps
    z = {k: 0.0 for k in KINDS}
    if ALG_SCHEDULE[algorithm] == "CBP":
        z.update(V2C=per, B2V=per, C2B=per)
    else:
        z.update(V2C=per, C2V=per, Dispatching=per)
    return z


def verify_counters(measured: dict, predicted: dict, tolerance: float = 0.0) -> dict:
    """Per-kind relative deviation of measured from predicted updates."""
    dev = {}
    for k in KINDS:
        p, m = predicted.get(k, 0.0), measured.get(k, 0.0)
        dev[k] = 0.0 if p == m else (abs(m - p) / p if p else float("inf"))
    return {"deviation": dev, "pass": all(d <= tolerance for d in dev.values())}
