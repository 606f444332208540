"""Pins of the oracle's comparison schedules (NEXT-3): fp32 layered BP and
flooding BP (equ_s2e3-e7, equ_s2e10, equ_s2e12; reading R22).

The independent reference here is the textbook in numpy fp64: the leave-one-out
sums of equ_s2e3 / equ_s2e4 evaluated by brute force over the other edges (not
as a total minus the own term), phi = -log tanh(x/2) from numpy."""
import numpy as np
import pytest

import inputs
import oracle


def code(name):
    base, Z = inputs.config_base(name)
    return oracle.OracleCode(base, Z)


def phi64(x):
    x = np.clip(np.abs(x), oracle.PHI_LO, oracle.PHI_HI)
    return np.clip(-np.log(np.tanh(x / 2.0)), oracle.PHI_LO, oracle.PHI_HI)


def c2v_bruteforce(Q):
    """equ_s2e4 by brute force: for each k, sign product and phi-sum over the others."""
    d = len(Q)
    R = np.empty(d)
    for k in range(d):
        o = np.delete(Q, k)
        R[k] = np.prod(np.sign(np.where(o < 0, -1.0, 1.0))) * phi64(np.sum(phi64(o)))
    return R


def lbp64(c, L, sweeps):
    chk, var = c.edges()
    ptr = np.searchsorted(chk, np.arange(c.M + 1))
    Lam = L.astype(np.float64).copy()
    R = np.zeros(c.E)
    for _ in range(sweeps):
        for ck in range(c.M):
            e = np.arange(ptr[ck], ptr[ck + 1])
            Q = Lam[var[e]] - R[e]                     # equ_s2e10
            Rn = c2v_bruteforce(Q)
            Lam[var[e]] = Q + Rn                       # equ_s2e12
            R[e] = Rn
    return Lam


def fbp64(c, L, iters):
    chk, var = c.edges()
    ptr = np.searchsorted(chk, np.arange(c.M + 1))
    R = np.zeros(c.E)
    Lam = L.astype(np.float64).copy()
    for _ in range(iters):
        Rn = np.zeros(c.E)
        for ck in range(c.M):
            e = np.arange(ptr[ck], ptr[ck + 1])
            # equ_s2e3 by brute force: L_v + sum of the OTHER checks' messages to v
            Q = np.array([L[v] + R[(var == v)].sum() - R[ee] for ee, v in zip(e, var[e])])
            Rn[e] = c2v_bruteforce(Q)
        R = Rn
        Lam = L.astype(np.float64) + np.bincount(var, weights=R, minlength=c.N)   # equ_s2e6
    return Lam


def bits_of(out, N):
    """hard decisions of the first frame of an oracle.decode result, uint8[N]"""
    return oracle.unpack_bits(out["bits"][0], N)


@pytest.mark.parametrize("arith,ref", [(oracle.LBP, lbp64), (oracle.FBP, fbp64)])
@pytest.mark.parametrize("name,ebn0", [("C1", 2.0), ("T24", 3.0)])
def test_bp_schedules_match_textbook_fp64(arith, ref, name, ebn0):
    """After k sweeps without stopping, the fp32 oracle's hard decisions equal the
    fp64 textbook's on every bit whose fp64 posterior is not within rounding of a
    tie; a dropped term, a wrong sign or the wrong schedule flips many bits."""
    c = code(name)
    llr, _ = c.channel(ebn0, seed=11, frame_begin=0, frames=6)
    for f in range(6):
        for k in (1, 2, 4):
            got = bits_of(c.decode(llr[f], k, oracle.STOP_NONE, arith), c.N)
            lam = ref(c, llr[f], k)
            want = (lam < 0).astype(np.uint8)
            bad = got != want
            assert np.all(np.abs(lam[bad]) < 1e-3), (f, k, lam[bad])


@pytest.mark.parametrize("arith", [oracle.LBP, oracle.FBP])
def test_bp_single_check_closed_form(arith):
    # H = [1 1], L = (5, -3): one update gives R_{c->v1} = -3, R_{c->v2} = 5 (phi(phi(x)) = x),
    # so both posteriors are 2 > 0: decisions (0, 0), which is a codeword -> stop after 1 sweep.
    c = oracle.OracleCode(np.array([[0, 0]], np.int16), 1)
    r = c.decode(np.float32([[5, -3]]), 5, oracle.STOP_SYNDROME, arith)
    assert r["iters"][0] == 1 and r["flags"][0] == 3
    assert bits_of(r, 2).tolist() == [0, 0]


@pytest.mark.parametrize("arith", [oracle.LBP, oracle.FBP])
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_bp_noiseless_one_iteration_and_counts(arith, name):
    c = code(name)
    rng = np.random.default_rng(5)
    info = rng.integers(0, 2, c.K).astype(np.uint8)
    cw = c.encode(info)
    L = np.where(cw == 1, -8.0, 8.0).astype(np.float32)
    r = c.decode(L, 10, oracle.STOP_SYNDROME, arith)
    assert r["iters"][0] == 1 and r["flags"][0] == 3
    assert (bits_of(r, c.N) == cw).all()
    assert r["edge_visits"][0] == c.E                    # Table I: E updates per iteration
    r = c.decode(L, 3, oracle.STOP_NONE, arith)
    assert r["edge_visits"][0] == 3 * c.E and r["iters"][0] == 3


def test_bp_rejects_belief_stop_rules():
    c = code("C1")
    L = np.zeros(c.N, np.float32)
    for arith in (oracle.LBP, oracle.FBP):
        for rule in (oracle.STOP_BELIEF_M, oracle.STOP_BELIEF_N):
            with pytest.raises(ValueError):
                c.decode(L, 5, rule, arith)


def test_layered_converges_faster_than_flooding():
    """The paper's convergence claim for the comparison schedules (l.713: CBP
    needs about half the iterations of FBP, like LBP): on C2 at 2 dB, layered BP
    needs clearly fewer sweeps than flooding BP, and both decode the same frames."""
    c = code("C2")
    llr, _ = c.channel(2.0, seed=7, frame_begin=0, frames=150)
    lb = c.decode(llr, 60, oracle.STOP_SYNDROME, oracle.LBP)
    fb = c.decode(llr, 60, oracle.STOP_SYNDROME, oracle.FBP)
    both = ((lb["flags"] & 1) == 1) & ((fb["flags"] & 1) == 1)
    assert both.mean() > 0.9
    ratio = lb["iters"][both].mean() / fb["iters"][both].mean()
    assert 0.35 < ratio < 0.75, ratio
