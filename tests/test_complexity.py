"""NEXT-4: the paper's complexity and memory tables (§V, l.740-900) reproduced by
paper_2305_05286_b200/complexity.py, and the kernel's update counters checked against Table I.

CPU: every printed number of Tables I-V and the l.898 example.  GPU (marked): measured
per-iteration updates of CBP / LBP / FBP on the BASELINE codes equal Table I exactly."""
import numpy as np
import pytest

import inputs
import oracle
from paper_2305_05286_b200 import complexity as cx

E = 1.0e6


def test_table1_update_counts():
    """Table I (l.750-767): CBP V2C = B2V = C2B = E, no C2V; FBP/LBP V2C = C2V = dispatching = E;
    RBP residual = sum E lambda_i rho_j (d_v-1)(d_c-1) -- 10E for (3,6) (SPEC S:458 example)."""
    t = cx.updates_per_iteration("CBP", E, cx.REGULAR_36)
    assert (t["V2C"], t["B2V"], t["C2B"], t["C2V"]) == (E, E, E, 0.0)
    for s in ("FBP", "LBP"):
        t = cx.updates_per_iteration(s, E, cx.REGULAR_36)
        assert (t["V2C"], t["C2V"], t["Dispatching"], t["B2V"]) == (E, E, E, 0.0)
    t = cx.updates_per_iteration("RBP", E, cx.REGULAR_36)
    assert t["Residual"] == pytest.approx(10 * E) and t["V2C"] == pytest.approx(2 * E)
    assert t["Comparison"] == E * (E - 1)
    assert cx.updates_per_iteration("CI-RBP", E, cx.IRREGULAR)["CI"] == E * (E - 1)


def test_table2_calculations_per_update():
    """Table II (l.775-793): CBP 2 sums (V2C), 1 product (B2V), 1 product (C2B); LBP 2/2 and
    max(d_c) selections; FBP 2/2 and max(d_v, d_c)."""
    assert cx.calculations_per_update("CBP", 3, 6, 3, 6) == {"V2C": ("sums", 2), "B2V": ("products", 1),
                                                             "C2B": ("products", 1)}
    assert cx.calculations_per_update("LBP", 3, 6, 3, 6)["Dispatching"] == ("selections", 6)
    assert cx.calculations_per_update("FBP", 3, 6, 12, 6)["Dispatching"] == ("selections", 12)
    assert cx.calculations_per_update("RBP", 3, 6, 3, 6)["Residual"] == ("products", 5)


@pytest.mark.parametrize("ens,want", [
    # Table IV (l.834-849), (3,6) regular
    (cx.REGULAR_36, {"FBP": (2, 2, 6), "LBP": (1, 1, 3), "RBP": (1, 13.75, 0), "SVNF-RBP": (1, 13.75, 0),
                     "CI-RBP": (0.67, 8.83, 0), "CBP": (1, 1, 0)}),
    # Table V (l.852-866), the irregular (lambda, rho) ensemble of l.608
    (cx.IRREGULAR, {"FBP": (2, 2, 12), "LBP": (1, 1, 3), "RBP": (5.04, 15.76, 0), "SVNF-RBP": (5.04, 15.76, 0),
                    "CI-RBP": (3.36, 10.17, 0), "CBP": (1, 1, 0)}),
])
def test_tables_iv_v(ens, want):
    """Table III's closed forms (l.797-822, convergence speeds of l.797) evaluated for the two
    ensembles give the printed coefficients of Tables IV / V (sums, products, selections per E;
    the RBP family's comparisons are E(E-1)/4, CI-RBP's E(E-1)/6)."""
    got = cx.table_iv_v_coefficients(ens, E)
    for s, (sums, prods, sel) in want.items():
        assert got[s]["sums"] == pytest.approx(sums, abs=0.006), s
        assert got[s]["products"] == pytest.approx(prods, abs=0.006), s
        assert got[s]["selections"] == pytest.approx(sel, abs=1e-9), s
    assert got["RBP"]["comparisons_over_E2"] == pytest.approx(0.25)
    assert got["CI-RBP"]["comparisons_over_E2"] == pytest.approx(1 / 6)
    assert got["CBP"]["comparisons_over_E2"] == 0.0


def test_table6_memory_and_5g_example():
    """Table VI (l.872-887) differences quoted in the text, and the l.898 example:
    58,368 pool bits, 141,312 check-belief bits = 14,131 registers, net 44,237."""
    N, M, Ee, P = 2048, 1024, 6144, 384
    cbp = cx.memory_cells("CBP", N, M, Ee, P, 3, 6)["general_cells"]
    assert cx.memory_cells("RBP", N, M, Ee, P, 3, 6)["general_cells"] - cbp == 2 * Ee - M
    assert cx.memory_cells("FBP", N, M, Ee, P, 3, 6)["general_cells"] - cbp == Ee - M
    assert cbp - cx.memory_cells("LBP", N, M, Ee, P, 3, 6)["general_cells"] == M
    ex = cx.register_example_5g()
    assert ex == {"pool_register_bits": 58368, "check_belief_bits": 141312,
                  "check_belief_register_equivalents": 14131, "net_register_saving": 44237}


def test_ensemble_of_code_and_verify_counters():
    """The QC-PEG member of the (3,6) family has the regular ensemble; verify_counters flags a
    deviation and passes an exact match."""
    base, Z = inputs.config_base("P2048")
    o = oracle.OracleCode(base, Z)
    chk, var = o.edges()
    ens = cx.ensemble_of_code(chk, var)
    assert ens.lam == {3: 1.0} and ens.rho == {6: 1.0}
    pred = cx.updates_per_iteration("CBP", o.E, ens)
    assert cx.verify_counters(cx.measured_updates(0, 5 * o.E, 5), pred)["pass"]
    bad = cx.verify_counters(cx.measured_updates(0, 5 * o.E + 7, 5), pred)
    assert not bad["pass"] and bad["deviation"]["B2V"] > 0


def test_oracle_counts_match_table1():
    """The oracle's edge-visit count per full sweep is E for CBP, LBP and FBP (one update of each
    kind per edge visit)."""
    base, Z = inputs.config_base("C2")
    o = oracle.OracleCode(base, Z)
    llr = inputs.random_llr(o.N, 4, 2.0, seed=3)
    for arith, alg in ((oracle.FP32_CONTRACT, 0), (oracle.LBP, 2), (oracle.FBP, 3)):
        r = o.decode(llr, 3, oracle.STOP_NONE, arith)
        chk, var = o.edges()
        pred = cx.updates_per_iteration(cx.ALG_SCHEDULE[alg], o.E, cx.ensemble_of_code(chk, var))
        for ev in r["edge_visits"]:
            assert cx.verify_counters(cx.measured_updates(alg, int(ev), 3), pred)["pass"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C2", "C3a", "C3b", "P2048"])
@pytest.mark.parametrize("alg", [0, 2, 3])
def test_gpu_counters_match_table1(name, alg):
    """GPU: the kernels' per-frame update counters over 4 full sweeps equal Table I exactly."""
    import torch
    import paper_2305_05286_b200 as cbp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base, Z = inputs.config_base(name)
    g = cbp.Code(base, Z)
    o = oracle.OracleCode(base, Z)
    chk, var = o.edges()
    pred = cx.updates_per_iteration(cx.ALG_SCHEDULE[alg], g.E, cx.ensemble_of_code(chk, var))
    llr, _ = g.channel(1.0, 5, 0, 64, llr_mode=2 if inputs.is_peg(name) else 0, want_cw=False)
    out = g.decode(llr, 4, cbp.CBP_STOP_NONE, ev=True, algorithm=alg)
    evs = out["ev"].cpu().numpy()
    assert (evs == 4 * g.E).all()
    rep = cx.verify_counters(cx.measured_updates(alg, int(evs[0]), 4), pred)
    assert rep["pass"], rep
