"""The paper's own code families (rate-1/2 PEG codes, regular (3,6) and
irregular lambda/rho, Fig. 6/7 lengths 2048 / 8192) as QC-PEG ensemble members
(inputs/peg.py, reading R21b), and the all-zero-codeword channel they are
simulated with (reading R23).  CPU only."""
from collections import deque

import numpy as np
import pytest

import inputs
import oracle
from inputs import peg

LAM_8192 = {2: 0.45, 3: 0.3708, 4: 0.0307, 12: 0.1485}   # PAPER.md l.608 (edge perspective)


def _lifted_adj(b, Z):
    mb, nb = b.shape
    N = nb * Z
    adj = [[] for _ in range(N + mb * Z)]
    for i in range(mb):
        for j in range(nb):
            s = int(b[i, j])
            if s < 0:
                continue
            for r in range(Z):
                v, c = j * Z + (r + s) % Z, N + i * Z + r
                adj[v].append(c)
                adj[c].append(v)
    return adj


def _girth(b, Z):
    """Shortest cycle of the lifted Tanner graph by BFS from every offset-0 variable
    (every variable is a cyclic shift of one of them)."""
    adj, best = _lifted_adj(b, Z), 10 ** 9
    for j in range(b.shape[1]):
        root = j * Z
        dist, par, q = {root: 0}, {root: -1}, deque([root])
        while q:
            u = q.popleft()
            if 2 * dist[u] + 1 >= best:
                break
            for w in adj[u]:
                if w == par[u]:
                    continue
                if w in dist:
                    best = min(best, dist[u] + dist[w] + 1)
                else:
                    dist[w], par[w] = dist[u] + 1, u
                    q.append(w)
    return best


def test_node_counts_follow_the_papers_lambda():
    cnt = peg.node_counts(128, LAM_8192)
    assert cnt == {2: 78, 3: 43, 4: 3, 12: 4} and sum(cnt.values()) == 128
    E = sum(d * n for d, n in cnt.items())
    for d, lam in LAM_8192.items():          # realised edge fractions within 1/64 of lambda
        assert abs(d * cnt[d] / E - lam) < 1 / 64
    assert peg.node_counts(64, {3: 1.0}) == {3: 64}


@pytest.mark.parametrize("name", ["P2048", "P8192"])
def test_peg_code_shape_and_degrees(name):
    cfg = inputs.PEG_CONFIGS[name]
    b, Z = inputs.config_base(name)
    assert b.shape == (cfg.mb, cfg.nb) and Z == cfg.Z
    assert cfg.nb * Z == int(name[1:]) and cfg.mb * 2 == cfg.nb          # N, rate 1/2 (l.608)
    assert ((b >= -1) & (b < Z)).all()
    cd, rd = (b >= 0).sum(0), (b >= 0).sum(1)
    if name == "P2048":
        assert (cd == 3).all() and (rd == 6).all()                          # regular (3,6)
    else:
        assert dict(zip(*np.unique(cd, return_counts=True))) == {2: 78, 3: 43, 4: 3, 12: 4}
        assert set(rd.tolist()) == {5, 6} and rd.sum() == cd.sum()         # rho: check degrees 5 and 6
        assert list(cd) == sorted(cd, reverse=True)                          # heavy columns first
    assert cfg.max_iter == 200                                               # l.608


@pytest.mark.parametrize("name,girth", [("P2048", 8), ("P8192", 8)])
def test_peg_lifted_girth(name, girth):
    """No 4-cycles (the QC condition s1 - s2 + s3 - s4 != 0 mod Z on every base
    rectangle) and the lifted girth measured by brute-force BFS."""
    b, Z = inputs.config_base(name)
    mb, nb = b.shape
    for i1 in range(mb):
        for i2 in range(i1 + 1, mb):
            js = np.nonzero((b[i1] >= 0) & (b[i2] >= 0))[0]
            for a in range(len(js)):
                for c in range(a + 1, len(js)):
                    j1, j2 = js[a], js[c]
                    assert (int(b[i1, j1]) - int(b[i1, j2]) + int(b[i2, j2]) - int(b[i2, j1])) % Z != 0
    assert _girth(b, Z) == girth


def test_peg_candidates_are_the_farthest_checks():
    """The offset-mask BFS of the constructor against a brute-force BFS on the lifted
    graph: on random partial QC graphs, the candidates are exactly the lifted checks
    of the open rows at maximum distance from variable j*Z (or unreachable)."""
    rng = np.random.default_rng(5)
    for trial in range(40):
        mb, nb, Z = int(rng.integers(3, 7)), int(rng.integers(4, 10)), int(rng.integers(2, 9))
        b = np.where(rng.random((mb, nb)) < 0.35, rng.integers(0, Z, (mb, nb)), -1)
        j = int(rng.integers(0, nb))
        b[:, j] = -1
        b[int(rng.integers(0, mb)), j] = int(rng.integers(0, Z))              # column j has one edge
        col_ent = [[(i, int(b[i, jj])) for i in range(mb) if b[i, jj] >= 0] for jj in range(nb)]
        row_ent = [[(jj, int(b[i, jj])) for jj in range(nb) if b[i, jj] >= 0] for i in range(mb)]
        open_rows = [i for i in range(mb) if b[i, j] < 0]
        if not open_rows:
            continue
        full = (1 << Z) - 1
        got = peg._deepest(j, col_ent, row_ent, mb, nb, Z, full, open_rows)
        adj, N = _lifted_adj(b, Z), nb * Z
        dist, q = {j * Z: 0}, deque([j * Z])
        while q:
            u = q.popleft()
            for w in adj[u]:
                if w not in dist:
                    dist[w] = dist[u] + 1
                    q.append(w)
        checks = [(i, r) for i in open_rows for r in range(Z)]
        far = [(i, r) for i, r in checks if N + i * Z + r not in dist]
        if not far:
            dmax = max(dist[N + i * Z + r] for i, r in checks)
            far = [(i, r) for i, r in checks if dist[N + i * Z + r] == dmax]
        want = {}
        for i, r in far:
            want[i] = want.get(i, 0) | (1 << r)
        assert got == want, (trial, got, want)


def test_peg_is_deterministic_and_seeded():
    cfg = inputs.PEG_CONFIGS["P2048"]
    col, row = peg.peg_degrees(cfg, 1)
    a = peg.qc_peg(cfg.mb, cfg.nb, cfg.Z, col, row, 1)
    assert (a == inputs.config_base("P2048")[0]).all()
    assert not (a == peg.qc_peg(cfg.mb, cfg.nb, cfg.Z, col, row, 2)).all()
    with pytest.raises(ValueError):
        peg.qc_peg(4, 8, 4, [3] * 8, [5] * 4, 1)                              # 24 != 20 edges


# ---------------------------------------------------------------- all-zero codeword (R23)
def _unpack(words, n):
    return np.stack([oracle.unpack_bits(w, n) for w in words])


def test_oracle_tx_zero_channel():
    """TX_ZERO sends c = 0 with the same Philox noise: L equals the encoded run's L
    bit for bit wherever the encoded codeword has c_v = 0, and L = fl(s (1 + sigma n))."""
    base, Z = inputs.config_base("C2")
    o = oracle.OracleCode(base, Z)
    le, ce = o.channel(2.0, 7, 100, 20)
    lz, cz = o.channel(2.0, 7, 100, 20, llr_mode=oracle.TX_ZERO)
    assert (cz == 0).all()
    c = _unpack(ce, o.N).astype(bool)
    assert c.any() and (lz[~c].view(np.uint32) == le[~c].view(np.uint32)).all()
    R = o.K / o.N
    s2 = 1.0 / (2.0 * R * 10 ** 0.2)
    sig, sc = np.float32(np.sqrt(s2)), np.float32(2.0 / s2)
    n = oracle.normals(7, 105, o.N)
    assert (lz[5].view(np.uint32) == (sc * (np.float32(1.0) + sig * n)).astype(np.float32).view(np.uint32)).all()
    lq, _ = o.channel(2.0, 7, 100, 20, llr_mode=oracle.TX_ZERO | oracle.LLR_INT8)
    assert ((lq * 4) == np.clip(np.rint(lz * 4), -127, 127)).all()


@pytest.mark.parametrize("arith", [oracle.FP32_CONTRACT, oracle.MINSUM])
def test_oracle_codeword_symmetry(arith):
    """Why the all-zero codeword is a valid stand-in (R23): the decoder commutes with
    the codeword flip, decode(L * (1 - 2c)) = decode(L) xor c with the same iteration
    count and flags, for every codeword c (the signs enter only through XORs and the
    fp32 ops are odd functions under round-to-nearest)."""
    base, Z = inputs.config_base("C2")
    o = oracle.OracleCode(base, Z)
    lz, _ = o.channel(1.5, 3, 0, 120, llr_mode=oracle.TX_ZERO)
    _, ce = o.channel(1.5, 9, 0, 120)                      # random codewords of the code
    c = _unpack(ce, o.N)
    a = o.decode(lz, 30, arith=arith)
    b = o.decode(lz * (1 - 2 * c.astype(np.float32)), 30, arith=arith)
    assert (a["iters"] == b["iters"]).all() and (a["flags"] == b["flags"]).all()
    assert (a["edge_visits"] == b["edge_visits"]).all()
    ab, bb = _unpack(a["bits"], o.N), _unpack(b["bits"], o.N)
    assert ((ab ^ c) == bb).all()
    assert (a["iters"] > 1).any() and ab.any()             # nontrivial decodes (errors corrected or left)


def test_oracle_ber_sim_peg_tx_zero():
    """P2048 through the oracle's ber_sim: needs TX_ZERO (no encoder structure);
    at 3 dB every frame converges to the all-zero codeword."""
    base, Z = inputs.config_base("P2048")
    o = oracle.OracleCode(base, Z)
    with pytest.raises(ValueError):
        o.ber_sim(3.0, 1, 0, 2, 200)
    c = o.ber_sim(3.0, 1, 0, 20, 200, llr_mode=oracle.TX_ZERO)
    assert c[0] == 20 and c[1] == 0 and c[3] == 0 and c[6] == 0


@pytest.mark.parametrize("name", ["P2048", "P8192"])
def test_peg_golden_hash(name):
    """The QC-PEG members are frozen like the BASELINE codes (tests/golden/base_hashes.txt,
    tools/write_goldens.py): a change to the constructor must regenerate them and say why."""
    from tests.test_inputs import _golden
    base, Z = inputs.config_base(name)
    assert inputs.base_sha256(base, Z) == _golden()[name]
