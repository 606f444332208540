"""Pins of the oracle's code expansion and encoder: H c = 0 checked against an
independent numpy expansion of the base matrix and a numpy GF(2) rank."""
import numpy as np
import pytest
import scipy.sparse as sp

import inputs
import oracle


def numpy_H(base, Z):
    """QC expansion: check row r of block (i,j) <-> variable j*Z + (r + s) % Z."""
    mb, nb = base.shape
    rows, cols = [], []
    for i in range(mb):
        for j in range(nb):
            s = int(base[i, j])
            if s < 0:
                continue
            r = np.arange(Z)
            rows.append(i * Z + r)
            cols.append(j * Z + (r + s) % Z)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    return sp.csr_matrix((np.ones(len(rows), np.uint8), (rows, cols)), shape=(mb * Z, nb * Z))


def gf2_rank(H):
    A = np.array(H, dtype=np.uint8) & 1
    r = 0
    for c in range(A.shape[1]):
        piv = np.nonzero(A[r:, c])[0]
        if len(piv) == 0:
            continue
        p = r + piv[0]
        A[[r, p]] = A[[p, r]]
        rows = np.nonzero(A[:, c])[0]
        rows = rows[rows != r]
        A[rows] ^= A[r]
        r += 1
        if r == A.shape[0]:
            break
    return r


@pytest.mark.parametrize("name", ["T24", "C1", "C2", "C3a", "C3b", "C4"])
def test_expansion_and_encoder(name):
    base, Z = inputs.config_base(name)
    c = oracle.OracleCode(base, Z)
    H = numpy_H(base, Z)
    chk, var = c.edges()
    Ho = sp.csr_matrix((np.ones(c.E, np.uint8), (chk, var)), shape=(c.M, c.N))
    assert (H != Ho).nnz == 0
    assert c.E == H.nnz and c.N == base.shape[1] * Z and c.K == c.N - c.M
    # edge ids row-major: checks ascending, variables ascending within a check (R12)
    order = np.lexsort((var, chk))
    assert (order == np.arange(c.E)).all()
    rng = np.random.default_rng(0)
    for _ in range(4 if name != "C4" else 2):
        info = rng.integers(0, 2, c.K).astype(np.uint8)
        cw = c.encode(info)
        assert (cw[:c.K] == info).all()                                 # systematic
        assert not (H @ cw.astype(np.int64) % 2).any()                  # H c = 0


@pytest.mark.parametrize("name", ["T24", "C1", "C2"])
def test_full_rank(name):
    base, Z = inputs.config_base(name)
    H = numpy_H(base, Z).toarray()
    assert gf2_rank(H) == H.shape[0]                                    # K = N - M


def test_encoder_linear_and_unique():
    base, Z = inputs.config_base("C1")
    c = oracle.OracleCode(base, Z)
    rng = np.random.default_rng(1)
    a = rng.integers(0, 2, c.K).astype(np.uint8)
    b = rng.integers(0, 2, c.K).astype(np.uint8)
    assert ((c.encode(a) ^ c.encode(b)) == c.encode(a ^ b)).all()
    assert not c.encode(np.zeros(c.K, np.uint8)).any()
