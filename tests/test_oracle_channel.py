"""Pins of the oracle's Philox / Box-Muller / BPSK-AWGN channel."""
import math
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

import inputs
import oracle

CUDA_INC = Path("/usr/local/cuda/include")

_KAT_SRC = r"""
#include <cstdio>
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main() {
    unsigned a[6];
    while (scanf("%x %x %x %x %x %x", &a[0], &a[1], &a[2], &a[3], &a[4], &a[5]) == 6) {
        uint4 c = {a[0], a[1], a[2], a[3]};
        uint2 k = {a[4], a[5]};
        uint4 o = curand_Philox4x32_10(c, k);
        printf("%08x %08x %08x %08x\n", o.x, o.y, o.z, o.w);
    }
}
"""


@pytest.mark.skipif(not (CUDA_INC / "curand_philox4x32_x.h").exists() or shutil.which("g++") is None,
                    reason="CUDA headers / g++ missing")
def test_philox_matches_curand_header(tmp_path):
    """The toolkit's Philox4x32-10 (host path of curand_philox4x32_x.h) is an
    independent implementation of the same published generator."""
    src = tmp_path / "kat.cpp"
    src.write_text(_KAT_SRC)
    exe = tmp_path / "kat"
    subprocess.run(["g++", "-O1", "-I", str(CUDA_INC), str(src), "-o", str(exe)], check=True)
    rng = np.random.default_rng(11)
    cases = rng.integers(0, 2 ** 32, (2000, 6), dtype=np.uint64)
    cases[0] = 0
    cases[1] = 0xFFFFFFFF
    stdin = "\n".join(" ".join(f"{int(x):x}" for x in row) for row in cases)
    out = subprocess.run([str(exe)], input=stdin, capture_output=True, text=True, check=True).stdout.split("\n")
    for row, line in zip(cases, out):
        want = [int(t, 16) for t in line.split()]
        got = oracle.philox4x32_10(row[:4], row[4:])
        assert list(map(int, got)) == want


def test_normals_statistics():
    n = np.concatenate([oracle.normals(seed=7, frame=f, n=4096) for f in range(256)]).astype(np.float64)
    assert abs(n.mean()) < 5e-3
    assert abs(n.var() - 1.0) < 1e-2
    assert abs(np.mean(np.abs(n) < 1.0) - 0.682689) < 3e-3
    assert abs(np.mean(np.abs(n) < 2.0) - 0.954500) < 1.5e-3
    assert np.abs(n).max() < 5.8                      # u1 >= 2^-24 truncates the tail at 5.77 sigma


def test_normals_box_muller_mapping():
    """n_{4k}, n_{4k+1} from words (x0, x1); n_{4k+2}, n_{4k+3} from (x2, x3) of
    Philox block (k, frame_lo, frame_hi, 1) keyed by the seed; float64 libm ref."""
    seed, frame = 0x1234_5678_9ABC_DEF0, 3 + (5 << 32)
    n = oracle.normals(seed, frame, 64)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for k in range(16):
        x = oracle.philox4x32_10([k, frame & 0xFFFFFFFF, frame >> 32, 1], key)
        for p in range(2):
            a, b = int(x[2 * p]), int(x[2 * p + 1])
            u1 = ((a >> 8) + 1) * 2.0 ** -24
            th = 2 * math.pi * (b >> 8) * 2.0 ** -24
            r = math.sqrt(-2 * math.log(u1))
            assert n[4 * k + 2 * p] == pytest.approx(r * math.cos(th), abs=2e-6)
            assert n[4 * k + 2 * p + 1] == pytest.approx(r * math.sin(th), abs=2e-6)


@pytest.fixture(scope="module")
def c1():
    base, Z = inputs.config_base("C1")
    return oracle.OracleCode(base, Z)


def test_channel_closed_form(c1):
    # Eb/N0 = 1 dB, R = 1/2 -> sigma^2 = 0.79432823, LLR(y=+1) = 2.51785082
    sigma2 = 1.0 / (2 * 0.5 * 10 ** 0.1)
    assert sigma2 == pytest.approx(0.79432823, rel=1e-8)
    assert 2 / sigma2 == pytest.approx(2.51785082, rel=1e-8)
    llr, cw = c1.channel(1.0, seed=3, frame_begin=10, frames=4)
    for f in range(4):
        bits = oracle.unpack_bits(cw[f], c1.N)
        n = oracle.normals(3, 10 + f, c1.N).astype(np.float64)
        y = (1.0 - 2.0 * bits) + math.sqrt(sigma2) * n
        assert np.allclose(llr[f], 2 / sigma2 * y, rtol=1e-5, atol=1e-5)
        assert c1.syndrome_weight(bits) == 0                                # codeword sent


def test_channel_int8_and_determinism(c1):
    l32, cw = c1.channel(2.0, seed=9, frame_begin=0, frames=20, llr_mode=0)
    l8, cw8 = c1.channel(2.0, seed=9, frame_begin=0, frames=20, llr_mode=1)
    assert (cw == cw8).all()
    q = np.clip(np.rint(l32 * 4.0), -127, 127)
    assert (l8 == (q * 0.25).astype(np.float32)).all()
    a, _ = c1.channel(2.0, seed=9, frame_begin=5, frames=7)
    assert (a == l32[5:12]).all()                                           # keyed by global frame index


def test_info_bits_uniform():
    base, Z = inputs.config_base("C2")
    c = oracle.OracleCode(base, Z)
    _, cw = c.channel(3.0, seed=4, frame_begin=0, frames=200)
    bits = np.stack([oracle.unpack_bits(w, c.N) for w in cw])
    assert abs(bits[:, :c.K].mean() - 0.5) < 0.01
    # paired noise: same seed/frame at another Eb/N0 -> same codewords
    _, cw2 = c.channel(1.0, seed=4, frame_begin=0, frames=200)
    assert (cw == cw2).all()
