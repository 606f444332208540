"""Pins of the oracle's normalized min-sum CBP (reading R20)."""
import numpy as np
import pytest

import inputs
import oracle


def code(name):
    base, Z = inputs.config_base(name)
    return oracle.OracleCode(base, Z)


@pytest.mark.parametrize("name,alpha", [("C1", 0.75), ("C2", 0.75), ("C2", 1.0), ("T24", 0.8)])
def test_minsum_cbp_equals_layered_minsum_bit_exact(name, alpha):
    """CBP's lagged posterior at each visit equals textbook layered normalized
    min-sum BP's posterior before the check (leave-one-out minimum by brute
    force), bit for bit in fp32: the min-sum CBP B2V/C2B rules (owner by edge,
    signs as psi-) are exactly the layered min-sum C2V rule evaluated lazily."""
    c = code(name)
    llr, _ = c.channel(2.0, seed=5, frame_begin=0, frames=3)
    for f in range(3):
        a = c.minsum_cbp_trace(llr[f], 4, alpha)
        b = c.minsum_lbp_trace(llr[f], 4, alpha)
        assert (a.view(np.uint32) == b.view(np.uint32)).all()


def test_minsum_single_check():
    # H = [1 1], L = (5, -3): Omega after one sweep = sgn * alpha * min(|Q|) = -(alpha * 3)
    c = oracle.OracleCode(np.array([[0, 0]], np.int16), 1)
    for alpha in (1.0, 0.75):
        r = c.decode(np.float32([[5, -3]]), 1, oracle.STOP_NONE, oracle.MINSUM, want_omega=True, alpha=alpha)
        assert r["omega"][0, 0] == np.float32(-alpha * 3.0)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_minsum_noiseless_and_counts(name):
    c = code(name)
    rng = np.random.default_rng(3)
    info = rng.integers(0, 2, (2, c.K)).astype(np.uint8)
    cws = np.stack([c.encode(i) for i in info])
    llr = (20.0 * (1.0 - 2.0 * cws)).astype(np.float32)
    r = c.decode(llr, 30, arith=oracle.MINSUM)
    assert (r["iters"] == 1).all() and (r["flags"] == 3).all()
    assert (np.stack([oracle.unpack_bits(b, c.N) for b in r["bits"]]) == cws).all()
    llr2, _ = c.channel(1.0, seed=2, frame_begin=0, frames=3)
    r = c.decode(llr2, 3, oracle.STOP_NONE, oracle.MINSUM)
    assert (r["edge_visits"] == 3 * c.E).all()                                  # Table I


def test_minsum_soundness_and_tie_rule():
    c = code("C2")
    llr, _ = c.channel(1.5, seed=4, frame_begin=0, frames=60)
    r = c.decode(llr, 30, arith=oracle.MINSUM)
    for b, fl in zip(r["bits"], r["flags"]):
        if fl & 1:
            assert c.syndrome_weight(oracle.unpack_bits(b, c.N)) == 0
    z = c.decode(np.zeros((1, c.N), np.float32), 5, arith=oracle.MINSUM)
    assert not z["bits"].any() and z["flags"][0] == 3


def test_minsum_paper_claims_c2():
    """normalized min-sum CBP loses little against log-tanh CBP and
    needs more iterations in the waterfall region (seeded, C2)."""
    c = code("C2")
    lt = c.ber_sim(2.0, 1, 0, 300, 30)
    ms = c.ber_sim(2.0, 1, 0, 300, 30, arith=oracle.MINSUM)
    assert ms[4] > lt[4]                                   # more iterations at 2.0 dB
    assert ms[2] <= 3 * lt[2] + 5                          # comparable frame errors
    with pytest.raises(ValueError):
        c.decode(np.zeros((1, c.N), np.float32), 5, arith=oracle.MINSUM, alpha=0.0)
