"""Pins of the oracle's CBP decoder (§IV-C) against things other than
itself: textbook layered BP, closed forms, brute-force ML, invariants."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

import inputs
import oracle
from tests.test_oracle_encoder import numpy_H


def code(name):
    base, Z = inputs.config_base(name)
    return oracle.OracleCode(base, Z)


def bits_of(out, N):
    return np.stack([oracle.unpack_bits(b, N) for b in out["bits"]])


@pytest.fixture(scope="module")
def c1():
    return code("C1")


@pytest.fixture(scope="module")
def c2():
    return code("C2")


def single_check():
    """H = [1 1]: one check, two degree-1 variables."""
    return oracle.OracleCode(np.array([[0, 0]], np.int16), 1)


def test_single_check_omega():
    # Omega after one sweep = psi+(5, 5) = 2 atanh(tanh(2.5)^2) = 4.3068982 (equ_s4e5/6)
    c = single_check()
    want = 2 * math.atanh(math.tanh(2.5) ** 2)
    for arith, tol in ((oracle.FP32_CONTRACT, 1e-6), (oracle.FP64, 1e-9)):
        r = c.decode(np.float32([[5, 5]]), 1, oracle.STOP_NONE, arith, want_omega=True)
        assert r["omega"][0, 0] == pytest.approx(want, rel=max(tol, 1e-7))
        # sweep 2: degree-1 variables pull R_new = psi-(Omega, Q) = phi(phi(5)) = 5 from
        # their own check (commit before read, R3): Q stays 5, Omega unchanged
        r2 = c.decode(np.float32([[5, 5]]), 2, oracle.STOP_NONE, arith, want_omega=True)
        assert r2["omega"][0, 0] == pytest.approx(want, rel=1e-6)
    # one negative LLR: the check-belief is negative (equ_s4e2 violated)
    r = c.decode(np.float32([[5, -3]]), 1, oracle.STOP_NONE, oracle.FP64, want_omega=True)
    assert r["omega"][0, 0] == pytest.approx(-2 * math.atanh(math.tanh(2.5) * math.tanh(1.5)), rel=1e-9)


@pytest.mark.parametrize("name,ebn0", [("C1", 2.0), ("C2", 2.0), ("C2", 1.0), ("T24", 3.0)])
def test_cbp_equals_layered_bp(name, ebn0):
    """In exact arithmetic CBP's lagged posterior Lambda^new at visit (c_i, v)
    (equ_s4e20) equals textbook layered BP's Lambda_v just before c_i is processed
    (equ_s2e10/equ_s2e12 with the leave-one-out rule equ_s2e4 by brute force).
    A wrong commit target (R2), commit order (R3), first-visit value (R1) or a
    dropped term fails this."""
    c = code(name)
    llr, _ = c.channel(ebn0, seed=5, frame_begin=0, frames=3)
    _, var = c.edges()
    first = np.unique(var, return_index=True)[1]          # first visit of every variable
    for f in range(3):
        cbp = c.cbp_trace(llr[f], 4)
        lbp = c.lbp_trace(llr[f], 4)
        assert (cbp[0, first] == llr[f][var[first]]).all()           # first visit: Lambda = L (R1)
        np.testing.assert_allclose(cbp, lbp, rtol=1e-8, atol=1e-9)


def test_literal_initialisation_would_fail(c1):
    """Reading R1: with the literal Omega=inf & 'first check as latest' the first
    B2V returns psi-(inf, Q) = Q, doubling the channel LLR -- the LBP trace rules
    it out because its first-sweep posterior is exactly L."""
    llr, _ = c1.channel(2.0, seed=1, frame_begin=0, frames=1)
    lbp = c1.lbp_trace(llr[0], 1)
    chk, var = c1.edges()
    first = np.unique(var, return_index=True)[1]
    assert (lbp[0, first] == llr[0][var[first]]).all()


@pytest.mark.parametrize("name", ["C1", "C2", "T24"])
def test_update_counts_table_I(name):
    """Table I (l.763): CBP does exactly E B2V, E V2C and E C2B per iteration."""
    c = code(name)
    llr, _ = c.channel(1.0, seed=2, frame_begin=0, frames=3)
    for k in (1, 3):
        r = c.decode(llr, k, oracle.STOP_NONE)
        assert (r["edge_visits"] == k * c.E).all() and (r["iters"] == k).all()
        assert (r["flags"] & 1 == 0).all()


@pytest.mark.parametrize("name", ["C1", "C2", "C3b"])
def test_noiseless_one_pass(name):
    """BASELINE invariant: noiseless input decodes in one pass (W = M)."""
    c = code(name)
    rng = np.random.default_rng(3)
    info = rng.integers(0, 2, (2, c.K)).astype(np.uint8)
    cws = np.stack([c.encode(i) for i in info])
    llr = (20.0 * (1.0 - 2.0 * cws)).astype(np.float32)
    r = c.decode(llr, 30)
    assert (r["iters"] == 1).all() and (r["flags"] == 3).all()
    assert (bits_of(r, c.N) == cws).all()
    assert (r["edge_visits"] == c.E).all()
    r = c.decode(llr, 30, oracle.STOP_SYNDROME)
    assert (r["iters"] == 1).all() and (r["flags"] == 3).all()
    r = c.decode(llr, 30, oracle.STOP_BELIEF_N)        # window N > M needs part of sweep 2
    assert (r["iters"] == 1 + (c.N - 1) // c.M).all() and (r["flags"] == 3).all()
    # high SNR without channel errors: one pass as well
    llr2, cw2 = c.channel(12.0, seed=1, frame_begin=0, frames=5)
    r = c.decode(llr2, 30)
    assert (r["iters"] == 1).all() and (r["bits"] == cw2).all()


def test_zero_llr_tie_rule(c1):
    """x_hat = 0 iff Lambda >= 0 (equ_s2e7): all-zero LLRs decode to the zero word."""
    r = c1.decode(np.zeros((1, c1.N), np.float32), 5)
    assert not r["bits"].any() and r["iters"][0] == 1 and r["flags"][0] == 3


def test_max_iter_one(c2):
    llr, _ = c2.channel(1.0, seed=3, frame_begin=0, frames=20)
    r = c2.decode(llr, 1)
    assert (r["iters"] == 1).all()
    assert (r["edge_visits"] <= c2.E).all()


def test_soundness_converged_implies_codeword(c2):
    H = numpy_H(c2.base, c2.Z)
    llr, _ = c2.channel(1.5, seed=4, frame_begin=0, frames=80)
    r = c2.decode(llr, 30)
    b = bits_of(r, c2.N).astype(np.int64)
    synd = (H @ b.T % 2).any(axis=0)
    assert ((r["flags"] & 1) == 1).sum() > 40
    assert not synd[(r["flags"] & 1) == 1].any()
    assert ((r["flags"] & 2 == 2) == ~synd).all()                           # flag bit1 = zero syndrome


def test_brute_force_ml_tiny_code():
    """N=24 code at high SNR: CBP returns the maximum-likelihood codeword."""
    c = code("T24")
    assert c.N == 24 and c.K == 12
    llr, _ = c.channel(6.0, seed=8, frame_begin=0, frames=400)
    r = c.decode(llr, 20)
    b = bits_of(r, c.N)
    ml = np.stack([c.ml_decode(x) for x in llr])
    assert (b == ml).all(axis=1).mean() >= 0.995
    # every ML codeword is a codeword
    assert all(c.syndrome_weight(m) == 0 for m in ml[:20])


def test_fp32_contract_tracks_fp64(c1, c2):
    """fp32 contract vs fp64 libm phi: identical decisions except on rare
    non-converged frames."""
    for c, eb in ((c1, 2.0), (c2, 2.0)):
        llr, _ = c.channel(eb, seed=6, frame_begin=0, frames=150)
        a = c.decode(llr, 30)
        b = c.decode(llr, 30, arith=oracle.FP64)
        same = (a["bits"] == b["bits"]).all(axis=1) & (a["iters"] == b["iters"])
        assert same.mean() >= 0.97
        assert ((a["flags"][~same] & 1) == 0).all() or ((b["flags"][~same] & 1) == 0).all()


def test_phi_domain_equals_literal_psi_recursion(c2):
    """Reading R11: accumulating S = sum phi(|Q|) (Appendix equ_ae4) instead of the
    literal psi+ recursion (equ_s4e5/6) changes nothing but rounding."""
    llr, _ = c2.channel(2.0, seed=7, frame_begin=0, frames=60)
    a = c2.decode(llr, 30, arith=oracle.FP64, want_omega=True)
    b = c2.decode(llr, 30, arith=oracle.FP64_LITERAL, want_omega=True)
    assert (a["iters"] == b["iters"]).mean() >= 0.98
    assert ((a["bits"] == b["bits"]).all(axis=1)).mean() >= 0.98
    ok = a["iters"] == b["iters"]
    np.testing.assert_allclose(a["omega"][ok], b["omega"][ok], rtol=1e-3, atol=1e-4)


def test_window_n_needs_more_sweeps(c2):
    llr, _ = c2.channel(2.0, seed=9, frame_begin=0, frames=60)
    m = c2.decode(llr, 30, oracle.STOP_BELIEF_M)
    n = c2.decode(llr, 30, oracle.STOP_BELIEF_N)
    s = c2.decode(llr, 30, oracle.STOP_SYNDROME)
    assert n["iters"].mean() >= m["iters"].mean() >= s["iters"].mean()


def test_batch_equals_single_frames(c2):
    llr, _ = c2.channel(1.5, seed=10, frame_begin=0, frames=6)
    a = c2.decode(llr, 30, want_omega=True)
    for f in range(6):
        b = c2.decode(llr[f:f + 1], 30, want_omega=True)
        for k in ("bits", "iters", "flags", "edge_visits", "fires", "omega"):
            assert (a[k][f] == b[k][0]).all()


def test_ber_sim_counts_consistent(c1):
    counts = c1.ber_sim(2.0, seed=11, frame_begin=100, frames=200, max_iter=20)
    llr, cw = c1.channel(2.0, seed=11, frame_begin=100, frames=200)
    r = c1.decode(llr, 20)
    d = bits_of(r, c1.N) != np.stack([oracle.unpack_bits(w, c1.N) for w in cw])
    want = [200, d[:, :c1.K].sum(), d[:, :c1.K].any(1).sum(), d.any(1).sum(), r["iters"].sum(),
            r["edge_visits"].sum(), ((r["flags"] & 1) == 0).sum(), r["fires"].sum()]
    assert list(map(int, counts)) == list(map(int, want))
    # shard invariance: counts do not depend on how the frame range is split
    a = c1.ber_sim(2.0, 11, 100, 77, 20) + c1.ber_sim(2.0, 11, 177, 123, 20)
    assert (a == counts).all()


def test_degree_one_extension_rows():
    """C4-like degree-1 columns (reading R3/R6): commit-before-read keeps
    Q = L for those bits; with the syndrome stop the decoder converges."""
    spec = (8, 14, 8, 4, 0, 3, 3)                 # 4-row core + 4 degree-1 extension rows
    base = inputs.construct_base(spec, 1)
    c = oracle.OracleCode(base, 8)
    llr, cw = c.channel(4.0, seed=1, frame_begin=0, frames=100)
    s = c.decode(llr, 30, oracle.STOP_SYNDROME)
    assert ((s["flags"] & 1) == 1).mean() > 0.8
    conv = (s["flags"] & 1) == 1
    assert (s["bits"][conv] == cw[conv]).all(axis=1).mean() > 0.95
