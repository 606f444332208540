"""Seeded QC constructor (inputs/, BASELINE.json configs)."""
from pathlib import Path

import numpy as np
import pytest

import inputs

GOLDEN = Path(__file__).parent / "golden" / "base_hashes.txt"
NAMES = ("C1", "C2", "C3a", "C3b", "C4", "T24")


def _golden():
    out = {}
    for line in GOLDEN.read_text().splitlines():
        if line and not line.startswith("#"):
            k, v = line.split()
            out[k] = v
    return out


@pytest.mark.parametrize("name", NAMES)
def test_structure(name):
    cfg = inputs.CONFIGS[name]
    mb, nb, Z, core, wmode, wlo, whi = cfg.spec
    base, Z2 = inputs.config_base(name)
    assert Z2 == Z and base.shape == (mb, nb)
    assert ((base >= -1) & (base < Z)).all()
    kb = nb - mb
    nz = base >= 0
    assert nz.any(axis=0).all() and nz.any(axis=1).all(), "empty row or column"
    w = nz[:, :kb].sum(axis=0)
    assert ((w >= wlo) & (w <= whi)).all()
    if wmode == 0:
        assert (w == wlo).all()
    # dual-diagonal core (802.11n style): column kb rows 0, core//2, core-1 with shifts 1, 0, 1
    col = base[:, kb]
    expect = np.full(mb, -1)
    expect[0], expect[core // 2], expect[core - 1] = 1 % Z, 0, 1 % Z
    assert (col == expect).all()
    for t in range(1, core):
        c = base[:, kb + t]
        e = np.full(mb, -1)
        e[t - 1] = 0
        e[t] = 0
        assert (c == e).all()
    for k in range(mb - core):          # degree-1 extension (C4)
        c = base[:, kb + core + k]
        assert (c >= 0).sum() == 1 and c[core + k] == 0
    # Appendix B row balancing: row degrees of the info part differ by at most one
    # per column drawn (lowest-degree rows are always picked first)
    rd = nz[:, :kb].sum(axis=1)
    assert rd.max() - rd.min() <= whi


@pytest.mark.parametrize("name", NAMES)
def test_golden_hash_and_determinism(name):
    base, Z = inputs.config_base(name)
    assert inputs.base_sha256(base, Z) == _golden()[name]
    base2, _ = inputs.config_base(name)
    assert (base == base2).all()
    other = inputs.construct_base(inputs.CONFIGS[name].spec, 2)
    assert not (other == base).all()


def test_heavy_tail_weights_c4():
    base, _ = inputs.config_base("C4")
    w = (base[:, :22] >= 0).sum(axis=0)
    assert w.min() == 3 and w.max() > 6          # heavy-tailed: some columns well above 3


def test_invalid_specs():
    with pytest.raises(ValueError):
        inputs.construct_base((2, 4, 8, 2, 0, 1, 1), 1)      # mb < 3
    with pytest.raises(ValueError):
        inputs.construct_base((6, 12, 1, 6, 0, 3, 3), 1)     # Z < 2
    with pytest.raises(ValueError):
        inputs.construct_base((6, 12, 8, 6, 0, 7, 7), 1)     # weight > mb
    with pytest.raises(ValueError):
        inputs.construct_base((6, 12, 8, 7, 0, 3, 3), 1)     # core > mb
