"""Pins of the oracle's fp32 arithmetic contract against libm
double precision and the closed forms of PAPER.md Appendix A (l.906-961)."""
import math

import numpy as np
import pytest

import oracle

ULP_MAX_PHI = 2.0   # contract v3 (table cubic through the double phi): 1.66 ulp, exhaustive


def phi_ref(x):
    """phi(x) = -log(tanh(x/2)) in float64 via libm; for x >= 1
    the equal form 2 atanh(e^-x) avoids the cancellation of tanh -> 1."""
    x = np.asarray(x, np.float64)
    return np.where(x < 1.0, -np.log(np.tanh(x / 2.0)), 2.0 * np.arctanh(np.exp(-x)))


def ulp32(v):
    v = np.abs(np.asarray(v, np.float64)).astype(np.float32)
    return (np.nextafter(v, np.float32(np.inf)) - v).astype(np.float64)


def test_phi_closed_forms():
    # tanh(ln3 / 2) = 1/2  =>  phi(ln 3) = ln 2, and by self-reciprocity phi(ln 2) = ln 3
    assert oracle.phi32(math.log(3)) == pytest.approx(math.log(2), rel=3e-7)
    assert oracle.phi32(math.log(2)) == pytest.approx(math.log(3), rel=3e-7)
    fp = math.log(1 + math.sqrt(2))      # fixed point phi(x) = x
    assert oracle.phi32(fp) == pytest.approx(fp, rel=3e-7)
    # (SPEC.md S:194's fixed point 0.7719 is phi(1), not a fixed point)
    assert oracle.phi32(1.0) == pytest.approx(0.7719368329, rel=3e-7)


def test_phi_ulp_dense_grid():
    rng = np.random.default_rng(5)
    lo, hi = np.log(oracle.PHI_LO), np.log(30.0)
    x = np.exp(rng.uniform(lo, hi, 1 << 20)).astype(np.float32)
    x = np.concatenate([x, np.float32([oracle.PHI_LO, 0.5, 0.99999994, 1.0, 1.0000001, 2.0, 29.999998, 30.0])])
    y = oracle.phi32_array(x).astype(np.float64)
    ref = np.clip(phi_ref(x), oracle.PHI_LO, oracle.PHI_HI)
    err = np.abs(y - ref) / ulp32(ref)
    assert err.max() <= ULP_MAX_PHI, f"max {err.max()} ulp at x={x[err.argmax()]}"


def test_phi_self_reciprocal_and_monotone():
    # Appendix A l.907: phi^{-1} = phi
    x = np.linspace(0.05, 12.0, 20001).astype(np.float32)
    y = oracle.phi32_array(oracle.phi32_array(x))
    assert np.max(np.abs(y - x) / x) < 2e-5
    z = oracle.phi32_array(np.sort(np.exp(np.linspace(-30, 3.4, 200001))).astype(np.float32))
    assert (np.diff(z) <= 0).all()


def test_phi_clamps():
    assert oracle.phi32(0.0) == oracle.PHI_HI            # phi(0) = inf -> PHI_HI
    assert oracle.phi32(1000.0) == np.float32(oracle.PHI_LO)
    assert oracle.phi32(float("inf")) == np.float32(oracle.PHI_LO)
    assert abs(oracle.phi32(30.0) - oracle.PHI_LO) <= 2 * float(ulp32(oracle.PHI_LO))
    assert oracle.PHI_LO == pytest.approx(2 * math.atanh(math.exp(-30)), rel=6e-8)   # fl32(phi(30))


def test_ln32_on_box_muller_grid():
    u = (np.arange(1, (1 << 24) + 1, 3, dtype=np.float64) * 2.0 ** -24).astype(np.float32)
    y = oracle.ln32_array(u).astype(np.float64)
    ref = np.log(u.astype(np.float64))
    nz = ref != 0
    assert (y[~nz] == 0).all()
    err = np.abs(y[nz] - ref[nz]) / ulp32(ref[nz])
    assert err.max() <= 1.0


def test_ln32_full_range():
    rng = np.random.default_rng(1)
    bits = rng.integers(0x00800000, 0x7F800000, 1 << 18, dtype=np.uint32)
    x = bits.view(np.float32)
    err = np.abs(oracle.ln32_array(x).astype(np.float64) - np.log(x.astype(np.float64)))
    assert (err / ulp32(np.log(x.astype(np.float64)))).max() <= 1.0


def test_sincos_quarter():
    rng = np.random.default_rng(2)
    ms = np.concatenate([rng.integers(0, 1 << 24, 40000),
                         np.array([0, 1, (1 << 21) - 1, 1 << 21, (1 << 22), 3 << 21, (1 << 24) - 1])])
    for m in ms:
        s, c = oracle.sincos_quarter32(int(m))
        th = 2.0 * math.pi * int(m) * 2.0 ** -24
        assert abs(s - math.sin(th)) < 2.5e-7 and abs(c - math.cos(th)) < 2.5e-7, m


@pytest.mark.parametrize("a,b,want", [(5.0, 5.0, 4.3068982), (2.0, 3.0, 1.6934537), (0.5, 8.0, 0.4996505)])
def test_psi_plus_textbook(a, b, want):
    """psi+(x,y) = sgn sgn phi(phi|x| + phi|y|) (equ_s4e6) equals the tanh rule
    2 atanh(tanh(a/2) tanh(b/2)); SPEC S:385's 3.69 for (5,5) is wrong."""
    got = oracle.phi32(oracle.phi32(a) + oracle.phi32(b))
    tanh_rule = 2 * math.atanh(math.tanh(a / 2) * math.tanh(b / 2))
    assert tanh_rule == pytest.approx(want, rel=1e-7)
    assert got == pytest.approx(tanh_rule, rel=2e-6)


def test_psi_minus_inverts_psi_plus():
    # Appendix A equ_ae6-ae8: psi-(psi+(a,b), b) = a
    rng = np.random.default_rng(3)
    for a, b in rng.uniform(0.5, 8.0, (500, 2)):
        om = oracle.phi32(oracle.phi32(a) + oracle.phi32(b))
        back = oracle.phi32(abs(oracle.phi32(om) - oracle.phi32(b)))
        assert back == pytest.approx(a, rel=2e-3)


def test_recursion_equals_batch():
    # equ_s4e3 (batch) vs equ_s4e5 (psi+ recursion from Omega^(-1) = inf) for degrees 3..20
    rng = np.random.default_rng(4)
    for d in range(3, 21):
        q = rng.normal(0, 4, d)
        batch = np.prod(np.sign(q)) * phi_ref(np.sum(phi_ref(np.abs(q))))
        om = math.inf
        for x in q:
            px = 0.0 if math.isinf(om) else oracle.phi32(abs(om))
            m = oracle.phi32(px + oracle.phi32(abs(x)))
            om = m if (om < 0) == (x < 0) else -m
        assert om == pytest.approx(batch, rel=5e-4, abs=1e-6)


def test_phi_v3_table_interpolates_phi_at_nodes():
    """Each v3 segment is the cubic through phi (double) at u = 0, 1/4, 3/4, 1:
    the table evaluated at the nodes reproduces numpy's phi to ~1e-7 relative."""
    t = oracle.phi32_table().astype(np.float64)
    assert t.shape == (oracle.PHI_SEGS, 4)
    for seg in list(range(0, oracle.PHI_SEGS, 37)) + [10, 703, 704, 1151, 1152]:
        for q in (0, 1, 3, 4):
            if seg < 704:
                e, j = -43 + seg // 16, seg % 16
                x = np.float32(np.ldexp(np.float64(64 + 4 * j + q), e - 6))
            else:
                x = np.float32((128 + 4 * (seg - 704) + q) * 0.015625)
            u = q / 4.0
            if seg < 704:
                p = t[seg, 0] + u * (t[seg, 1] + u * (t[seg, 2] + u * t[seg, 3]))
            else:
                p = t[seg, 0] + u * (t[seg, 1] + u * (t[seg, 2] + u * t[seg, 3]))
            f = float(phi_ref(np.float64(x)))
            assert p == pytest.approx(f, rel=3e-7), (seg, q)


def test_phi_v3_exhaustive():
    """Every binary32 x in [PHI_LO, 30]: the unclamped v3 cubic stays in [PHI_LO, 30] (so an
    implementation may omit the output clamp -- the GPU does) and is within ULP_MAX_PHI of the
    double phi (SURVEY Appendix C asks <= 4 ulp)."""
    below, above, mx, at = oracle.phi32_exhaustive()
    assert below == 0 and above == 0
    assert mx <= ULP_MAX_PHI, (mx, at)
