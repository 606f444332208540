"""Seeded input generators shared by the product tests, the oracle and bench.py.

Holds none of the method's arithmetic (DESIGN.md §5 "input recipe"):
  * the QC base-matrix constructor (C, inputs/qc_construct.c) for the
    BASELINE.json configs,
  * the QC-PEG constructor (inputs/peg.py) for the paper's own code families, and
  * numpy LLR generators for decode-only tests (all-zero codeword over BPSK/AWGN,
    which is a codeword of every linear code, or raw random LLR vectors).
"""
from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .peg import PEG_CONFIGS, PegConfig, peg_base, qc_peg  # noqa: F401  (the paper's own code families)

_HERE = Path(__file__).resolve().parent
_LIB = None


class ConstructSpec(ctypes.Structure):
    _fields_ = [("mb", ctypes.c_int32), ("nb", ctypes.c_int32), ("Z", ctypes.c_int32),
                ("mb_core", ctypes.c_int32), ("wmode", ctypes.c_int32), ("w_lo", ctypes.c_int32),
                ("w_hi", ctypes.c_int32)]


def _lib():
    global _LIB
    if _LIB is None:
        so = _HERE / "libcbp_inputs.so"
        if not so.exists():
            from tools.build_native import build_inputs  # noqa: WPS433
            build_inputs()
        lib = ctypes.CDLL(str(so))
        lib.cbp_inputs_construct_base.argtypes = [ctypes.POINTER(ConstructSpec), ctypes.c_uint64,
                                                  ctypes.POINTER(ctypes.c_int16),
                                                  ctypes.POINTER(ctypes.c_char_p)]
        lib.cbp_inputs_construct_base.restype = ctypes.c_int
        lib.cbp_inputs_named_spec.argtypes = [ctypes.c_char_p, ctypes.POINTER(ConstructSpec)]
        lib.cbp_inputs_named_spec.restype = ctypes.c_int
        _LIB = lib
    return _LIB


@dataclass(frozen=True)
class CodeConfig:
    """One BASELINE.json workload: code spec + channel/decoder settings."""
    name: str
    spec: tuple            # (mb, nb, Z, mb_core, wmode, w_lo, w_hi)
    code_seed: int
    ebn0_db: tuple         # Eb/N0 points (dB)
    frames: int            # frames per point in the BASELINE config
    max_iter: int


# BASELINE.json "configs"; code seed 1 throughout.
CONFIGS = {
    "C1": CodeConfig("C1", (6, 12, 8, 6, 0, 3, 3), 1, (2.0,), 10_000, 20),
    "C2": CodeConfig("C2", (12, 24, 27, 12, 1, 3, 4), 1, (1.0, 1.5, 2.0, 2.5, 3.0), 1_000_000, 30),
    "C3a": CodeConfig("C3a", (12, 24, 81, 12, 1, 3, 6), 1, (1.5, 2.0, 2.5, 3.0, 3.5, 4.0, 4.5), 10_000_000, 30),
    "C3b": CodeConfig("C3b", (4, 24, 81, 4, 1, 3, 4), 1, (1.5, 2.0, 2.5, 3.0, 3.5, 4.0, 4.5), 10_000_000, 30),
    "C4": CodeConfig("C4", (46, 68, 384, 4, 2, 3, 30), 1, (1.0, 1.5, 2.0), 1_000_000, 25),
    "C5": CodeConfig("C5", (12, 24, 81, 12, 1, 3, 6), 1, (2.5,), 1_000_000_000, 30),
    "T24": CodeConfig("T24", (3, 6, 4, 3, 0, 2, 2), 1, (6.0,), 1000, 20),
}


def construct_base(spec, seed: int) -> np.ndarray:
    """QC base matrix (int16, mb x nb) for `spec` = (mb, nb, Z, mb_core, wmode, w_lo, w_hi)."""
    sp = ConstructSpec(*[int(x) for x in spec])
    out = np.empty((sp.mb, sp.nb), dtype=np.int16)
    err = ctypes.c_char_p()
    rc = _lib().cbp_inputs_construct_base(ctypes.byref(sp), ctypes.c_uint64(seed),
                                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_int16)), ctypes.byref(err))
    if rc != 0:
        raise ValueError(f"construct_base: {err.value.decode() if err.value else rc}")
    return out


def config_base(name: str) -> tuple[np.ndarray, int]:
    """(base, Z) of a BASELINE config (CONFIGS) or of one of the paper's PEG families (PEG_CONFIGS)."""
    if name in PEG_CONFIGS:
        return peg_base(name)
    cfg = CONFIGS[name]
    return construct_base(cfg.spec, cfg.code_seed), cfg.spec[2]


def get_config(name: str):
    """CodeConfig or PegConfig by name (both carry name, code_seed, ebn0_db, frames, max_iter)."""
    return PEG_CONFIGS[name] if name in PEG_CONFIGS else CONFIGS[name]


def is_peg(name: str) -> bool:
    """PEG codes have no encoder structure: channels send the all-zero codeword (TX_ZERO)."""
    return name in PEG_CONFIGS


def base_sha256(base: np.ndarray, Z: int) -> str:
    h = hashlib.sha256()
    h.update(np.array(base.shape + (Z,), dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(base, dtype="<i2").tobytes())
    return h.hexdigest()


def awgn_llr_zero_codeword(N: int, frames: int, ebn0_db: float, rate: float, seed: int) -> np.ndarray:
    """LLRs of the all-zero codeword (BPSK +1) over AWGN, float32 [frames, N].

    numpy PCG64 stream; decode-only test input (the product's on-device
    channel is checked separately against the oracle's channel)."""
    rng = np.random.default_rng(seed)
    sigma2 = 1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0))
    y = 1.0 + np.sqrt(sigma2) * rng.standard_normal((frames, N))
    return (2.0 / sigma2 * y).astype(np.float32)


def random_llr(N: int, frames: int, scale: float, seed: int) -> np.ndarray:
    """Arbitrary LLR vectors (no codeword structure), float32 [frames, N]."""
    rng = np.random.default_rng(seed)
    return (scale * rng.standard_normal((frames, N))).astype(np.float32)
