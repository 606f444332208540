"""Pin of the oracle's stopping criterion (§IV-C Step 2(3), l.478-485: equ_s4e2 for
every check-belief, equ_s4e24 "no sign flips", Alg. 1 line 16 at l.513) against an independent
numpy model of the rule.

The model reads only the oracle's raw decoding trajectory -- Lambda^new (equ_s4e20) and Q^new
(equ_s4e19) of every edge visit over `max_iter` full sweeps, recorded with no stop rule at all
(`oracle_cbp_visit_trace`) -- and evaluates the rule from the paper's definitions with the
readings of DESIGN.md §2:
  * sgn(Omega_c) = product of sgn(Q^new) over the check's edges (equ_s4e2 through the psi+ sign
    rule equ_s4e5 / equ_s4e6; R8: sign tests are `x < 0`);
  * a flip = (Lambda^new < 0) differs from the variable's previous hard decision (R7), the
    decision of its previous visit, initially L_v < 0;
  * a check update is clean iff Omega_c > 0 and none of its posteriors flipped; W consecutive
    clean updates, counted cyclically over check updates (R4: W = M, or N);
  * when the window fills: the syndrome of the current hard decisions (computed here from an
    independent numpy expansion of the base matrix); zero -> stop after that check update,
    converged; nonzero -> one failed verification, the window restarts empty (R5).
It returns iterations, flags, edge visits, failed verifications and the output bits, which must
equal the oracle's decode (with the stop rule) frame by frame.  Small test-only windows
(`oracle_decode_window`) force fires in the middle of a base row and failed verifications.
The mutants "flip test ignored" and "no reset after a failed verification" each change these
outputs on the frames below (checked in test_model_detects_mutants, on the model itself).
"""
import numpy as np
import pytest

import inputs
import oracle


def numpy_edges(base: np.ndarray, Z: int):
    """Row-major edge list of the QC expansion (check r of block (i,j) <-> variable jZ + (r+s) mod Z),
    checks ascending, variables ascending within a check -- written independently of the oracle."""
    mb, nb = base.shape
    chk, var = [], []
    for i in range(mb):
        for r in range(Z):
            for j in range(nb):
                s = int(base[i, j])
                if s >= 0:
                    chk.append(i * Z + r)
                    var.append(j * Z + (r + s) % Z)
    return np.array(chk, np.int64), np.array(var, np.int64)


class StopModel:
    """The belief-window stop rule evaluated on a recorded trajectory (see the module docstring).
    `flip_test` / `reset` switch the two parts off (mutants)."""

    def __init__(self, base, Z, flip_test=True, reset=True):
        self.chk, self.var = numpy_edges(base, Z)
        self.M = int(self.chk.max()) + 1
        self.N = base.shape[1] * Z
        self.ptr = np.searchsorted(self.chk, np.arange(self.M + 1))
        self.flip_test, self.reset = flip_test, reset

    def syndrome_zero(self, hb):
        return not np.bitwise_xor.reduceat(hb[self.var].astype(np.uint8), self.ptr[:-1]).any()

    def run(self, L, lam, qn, W, max_iter):
        S, E, M, N = max_iter, len(self.chk), self.M, self.N
        lam, qn = lam[:S].reshape(-1), qn[:S].reshape(-1)
        bits = lam < 0                                        # decision of each visit (equ_s2e7, R8)
        V = np.tile(self.var, S)
        T = np.arange(S * E)
        # previous decision of the visit's variable: the previous visit's, or L_v < 0 (R7)
        order = np.lexsort((T, V))
        prev = np.empty(S * E, bool)
        first = np.ones(S * E, bool)
        first[1:] = V[order][1:] != V[order][:-1]
        prev[order] = np.where(first, (L < 0)[V[order]], np.roll(bits[order], 1))
        flip_visit = (bits != prev) if self.flip_test else np.zeros(S * E, bool)
        starts = (np.arange(S)[:, None] * E + self.ptr[:-1][None, :]).reshape(-1)    # first visit of each update
        neg = np.bitwise_xor.reduceat((qn < 0).astype(np.uint8), starts).astype(bool)  # sgn Omega_c < 0
        flip = np.logical_or.reduceat(flip_visit, starts)
        ok = ~neg & ~flip                                     # check update t = (sweep t // M, check t % M)
        t_idx = np.arange(S * M)
        last_bad = np.maximum.accumulate(np.where(ok, -1, t_idx))
        good = np.nonzero(t_idx - last_bad >= W)[0]           # W clean updates end here (no reset inside)
        key_sorted = V[order] * (S * E) + T[order]

        def hard_bits(u_end):                                 # decisions after visit u_end (inclusive)
            q = np.searchsorted(key_sorted, np.arange(N) * (S * E) + u_end, side="right") - 1
            hit = (q >= 0) & (V[order][np.maximum(q, 0)] == np.arange(N))
            return np.where(hit, bits[order][np.maximum(q, 0)], L < 0)

        fires, t_reset = 0, -1
        while True:
            # next t with W clean updates in (t_reset, t]: t - last_bad >= W and t - t_reset >= W
            k = np.searchsorted(good, t_reset + W if self.reset else 0)
            if not self.reset:
                k = np.searchsorted(good, t_reset + 1)
            if k >= len(good):
                break
            t = int(good[k])
            s, c = divmod(t, M)
            u_end = s * E + int(self.ptr[c + 1]) - 1
            hb = hard_bits(u_end)
            if self.syndrome_zero(hb):
                return {"iters": s + 1, "conv": True, "fires": fires, "ev": u_end + 1, "bits": hb}
            fires += 1
            t_reset = t
        hb = hard_bits(S * E - 1)
        return {"iters": max_iter, "conv": False, "fires": fires, "ev": S * E, "bits": hb}


def model_outputs(model, o, llr, W, max_iter, arith):
    res = {"bits": [], "iters": [], "flags": [], "edge_visits": [], "fires": []}
    for L in llr:
        lam, qn = o.visit_trace(L, max_iter, arith)
        r = model.run(L, lam, qn, W, max_iter)
        res["bits"].append(oracle.pack_bits(r["bits"].astype(np.uint8))[: o.words])
        res["iters"].append(r["iters"])
        res["flags"].append((1 if r["conv"] else 0) | (2 if model.syndrome_zero(r["bits"]) else 0) |
                            (4 if r["fires"] else 0))
        res["edge_visits"].append(r["ev"])
        res["fires"].append(r["fires"])
    return {k: np.array(v) for k, v in res.items()}


def degree_one_code():
    return inputs.construct_base((8, 14, 8, 4, 0, 3, 3), 1), 8


def code_of(name):
    if name == "deg1":
        return degree_one_code()
    return inputs.config_base(name)


# (code, Eb/N0, frames, max_iter): noisy frames around each code's waterfall
CASES = [("C1", 2.0, 300, 20), ("C2", 2.0, 300, 30), ("T24", 3.0, 300, 20), ("deg1", 3.0, 300, 25)]


def assert_equal(got, want):
    for k in ("iters", "flags", "edge_visits", "fires"):
        bad = np.nonzero(got[k] != want[k])[0]
        assert len(bad) == 0, f"{k} differs on {len(bad)} frames, first {bad[:5]}: {got[k][bad[:5]]} vs {want[k][bad[:5]]}"
    assert (got["bits"] == want["bits"][:, : got["bits"].shape[1]]).all()


@pytest.mark.parametrize("name,ebn0,frames,max_iter", CASES)
@pytest.mark.parametrize("window", ["M", "N", 4, 10, 37])
@pytest.mark.parametrize("arith", [oracle.FP64, oracle.FP32_CONTRACT])
def test_stop_rule_equals_numpy_model(name, ebn0, frames, max_iter, window, arith):
    base, Z = code_of(name)
    o = oracle.OracleCode(base, Z)
    chk, var = o.edges()
    mchk, mvar = numpy_edges(base, Z)
    assert (chk == mchk).all() and (var == mvar).all()        # the model's graph is the oracle's
    # the small window fires (and re-verifies) every few checks: fewer frames keep the CPU suite short
    llr, _ = o.channel(ebn0, seed=11, frame_begin=0, frames=frames if window != 4 else frames // 3)
    model = StopModel(base, Z)
    if window == "M":
        W, want = o.M, o.decode(llr, max_iter, oracle.STOP_BELIEF_M, arith)
    elif window == "N":
        W, want = o.N, o.decode(llr, max_iter, oracle.STOP_BELIEF_N, arith)
    else:
        W, want = window, o.decode_window(llr, max_iter, window, oracle.STOP_BELIEF_M, arith)
    got = model_outputs(model, o, llr, W, max_iter, arith)
    assert_equal(got, want)
    if window == 4:
        # the small window really exercises the verification: failed verifications and stops
        # in the middle of a base row occur
        assert want["fires"].sum() > 0
        conv = (want["flags"] & 1).astype(bool)
        rem = want["edge_visits"][conv] % o.E
        stop_chk = np.searchsorted(model.ptr, np.where(rem == 0, o.E, rem)) - 1     # last check updated
        assert (stop_chk % Z != Z - 1).any()


def test_minsum_stop_rule_equals_numpy_model():
    """The same rule on normalized min-sum CBP's trajectory (reading R20)."""
    base, Z = inputs.config_base("C2")
    o = oracle.OracleCode(base, Z)
    llr, _ = o.channel(2.0, seed=12, frame_begin=0, frames=200)
    model = StopModel(base, Z)
    for W in (o.M, 10):
        want = o.decode_window(llr, 30, W, oracle.STOP_BELIEF_M, oracle.MINSUM)
        got = model_outputs(model, o, llr, W, 30, oracle.MINSUM)
        assert_equal(got, want)


def test_model_detects_mutants():
    """The pin has teeth: the model with the flip test (equ_s4e24) dropped, or without the window
    reset after a failed verification (R5), disagrees with the oracle on these frames."""
    base, Z = inputs.config_base("C2")
    o = oracle.OracleCode(base, Z)
    llr, _ = o.channel(2.0, seed=11, frame_begin=0, frames=200)
    want_m = o.decode(llr, 30, oracle.STOP_BELIEF_M, oracle.FP64)
    no_flip = model_outputs(StopModel(base, Z, flip_test=False), o, llr, o.M, 30, oracle.FP64)
    assert (no_flip["edge_visits"] != want_m["edge_visits"]).any()
    want_w = o.decode_window(llr, 30, 10, oracle.STOP_BELIEF_M, oracle.FP64)
    no_reset = model_outputs(StopModel(base, Z, reset=False), o, llr, 10, 30, oracle.FP64)
    assert (no_reset["fires"] != want_w["fires"]).any()
