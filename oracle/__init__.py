"""ctypes wrapper of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package; the product
package paper_2305_05286_b200 never does (checked by tests/test_boundary.py).
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

STOP_BELIEF_M, STOP_BELIEF_N, STOP_SYNDROME, STOP_NONE = 0, 1, 2, 3
FP32_CONTRACT, FP64, FP64_LITERAL, MINSUM, LBP, FBP = 0, 1, 2, 3, 4, 5
LLR_INT8, TX_ZERO = 1, 2   # llr_mode flags (TX_ZERO: the all-zero codeword is sent, reading R23)
ALPHA_DEFAULT = 0.75   # normalized min-sum parameter (reading R20; the paper leaves alpha open)
PHI_LO = float.fromhex("0x1.a56e0cp-43")
PHI_HI = 30.0

_p = ctypes.c_void_p
_i32, _i64, _u64, _f32, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_double


class Opts(ctypes.Structure):
    _fields_ = [("max_iter", _i32), ("stop_rule", _i32), ("arith", _i32), ("alpha", _f32)]


def _lib():
    global _LIB
    if _LIB is None:
        so = _HERE / "liboracle.so"
        if not so.exists():
            from tools.build_native import build_oracle
            build_oracle()
        lib = ctypes.CDLL(str(so))
        sig = {
            "oracle_code_create": ([_p, _i32, _i32, _i32], _p),
            "oracle_code_destroy": ([_p], None),
            "oracle_code_dims": ([_p, _p, _p, _p, _p], None),
            "oracle_code_edges": ([_p, _p, _p], None),
            "oracle_decode": ([_p, _p, _i64, _i64, _p, _p, _i64, _p, _p, _p, _p, _p], ctypes.c_int),
            "oracle_encode": ([_p, _p, _p], ctypes.c_int),
            "oracle_syndrome_weight": ([_p, _p], ctypes.c_int),
            "oracle_philox4x32_10": ([_p, _p, _p], None),
            "oracle_normals": ([_u64, _u64, _i32, _p], None),
            "oracle_channel": ([_p, _f64, _u64, _i64, _i64, _i32, _p, _i64, _p, _i64], ctypes.c_int),
            "oracle_ber_sim": ([_p, _f64, _u64, _i64, _i64, _p, _i32, _p], ctypes.c_int),
            "oracle_cbp_trace_f64": ([_p, _p, _i32, _p], ctypes.c_int),
            "oracle_lbp_trace_f64": ([_p, _p, _i32, _p], ctypes.c_int),
            "oracle_minsum_cbp_trace": ([_p, _p, _i32, _f32, _p], ctypes.c_int),
            "oracle_minsum_lbp_trace": ([_p, _p, _i32, _f32, _p], ctypes.c_int),
            "oracle_ml_decode": ([_p, _p, _p], ctypes.c_int),
            "oracle_decode_window": ([_p, _p, _i64, _i64, _p, _i64, _p, _i64, _p, _p, _p, _p], ctypes.c_int),
            "oracle_cbp_visit_trace": ([_p, _p, _i32, _i32, _f32, _p, _p], ctypes.c_int),
            "oracle_phi32": ([_f32], _f32),
            "oracle_ln32": ([_f32], _f32),
            "oracle_sincos_quarter32": ([ctypes.c_uint32, _p, _p], None),
            "oracle_phi32_n": ([_p, _p, _i64], None),
            "oracle_phi32_table": ([_p], None),
            "oracle_phi32_exhaustive": ([_p, _p, _p, _p], None),
            "oracle_ln32_n": ([_p, _p, _i64], None),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = lib
    return _LIB


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


class OracleCode:
    """Expanded code graph G = (V, C, E) of a QC base matrix."""

    def __init__(self, base: np.ndarray, Z: int):
        base = np.ascontiguousarray(base, dtype=np.int16)
        self.base, self.Z = base, int(Z)
        self.mb, self.nb = base.shape
        self._h = _lib().oracle_code_create(_ptr(base), self.mb, self.nb, self.Z)
        if not self._h:
            raise ValueError("oracle_code_create failed")
        N, K, M, E = _i32(), _i32(), _i32(), _i64()
        _lib().oracle_code_dims(self._h, ctypes.byref(N), ctypes.byref(K), ctypes.byref(M), ctypes.byref(E))
        self.N, self.K, self.M, self.E = N.value, K.value, M.value, E.value
        self.words = (self.N + 31) // 32

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _LIB is not None:
            _LIB.oracle_code_destroy(h)
            self._h = None

    def edges(self):
        chk = np.empty(self.E, np.int32)
        var = np.empty(self.E, np.int32)
        _lib().oracle_code_edges(self._h, _ptr(chk), _ptr(var))
        return chk, var

    def H(self) -> np.ndarray:
        chk, var = self.edges()
        H = np.zeros((self.M, self.N), np.uint8)
        H[chk, var] = 1
        return H

    def decode(self, llr: np.ndarray, max_iter: int, stop_rule: int = STOP_BELIEF_M,
               arith: int = FP32_CONTRACT, want_omega: bool = False, alpha: float = ALPHA_DEFAULT) -> dict:
        llr = np.ascontiguousarray(llr, dtype=np.float32).reshape(-1, self.N)
        F = llr.shape[0]
        out = {"bits": np.zeros((F, self.words), np.uint32), "iters": np.zeros(F, np.int32),
               "flags": np.zeros(F, np.uint8), "edge_visits": np.zeros(F, np.int64),
               "fires": np.zeros(F, np.int32)}
        om = np.zeros((F, self.M), np.float32) if want_omega else None
        o = Opts(max_iter, stop_rule, arith, alpha)
        rc = _lib().oracle_decode(self._h, _ptr(llr), self.N, F, ctypes.byref(o), _ptr(out["bits"]), self.words,
                                  _ptr(out["iters"]), _ptr(out["flags"]), _ptr(out["edge_visits"]),
                                  _ptr(out["fires"]), _ptr(om))
        if rc:
            raise ValueError(f"oracle_decode rc={rc}")
        if want_omega:
            out["omega"] = om
        return out

    def decode_window(self, llr: np.ndarray, max_iter: int, window: int, stop_rule: int = STOP_BELIEF_M,
                      arith: int = FP32_CONTRACT, alpha: float = ALPHA_DEFAULT) -> dict:
        """decode with the belief window W (reading R4) replaced by `window` (test-only hook)."""
        llr = np.ascontiguousarray(llr, dtype=np.float32).reshape(-1, self.N)
        F = llr.shape[0]
        out = {"bits": np.zeros((F, self.words), np.uint32), "iters": np.zeros(F, np.int32),
               "flags": np.zeros(F, np.uint8), "edge_visits": np.zeros(F, np.int64),
               "fires": np.zeros(F, np.int32)}
        o = Opts(max_iter, stop_rule, arith, alpha)
        rc = _lib().oracle_decode_window(self._h, _ptr(llr), self.N, F, ctypes.byref(o), window, _ptr(out["bits"]),
                                         self.words, _ptr(out["iters"]), _ptr(out["flags"]),
                                         _ptr(out["edge_visits"]), _ptr(out["fires"]))
        if rc:
            raise ValueError(f"oracle_decode_window rc={rc}")
        return out

    def visit_trace(self, llr: np.ndarray, sweeps: int, arith: int = FP64, alpha: float = ALPHA_DEFAULT):
        """(lam, qn) float64 [sweeps, E]: Lambda^new and Q^new of every edge visit, no stop rule."""
        lam = np.zeros((sweeps, self.E), np.float64)
        qn = np.zeros((sweeps, self.E), np.float64)
        rc = _lib().oracle_cbp_visit_trace(self._h, _ptr(np.ascontiguousarray(llr, np.float32)), sweeps, arith,
                                           alpha, _ptr(lam), _ptr(qn))
        if rc:
            raise ValueError("oracle_cbp_visit_trace failed")
        return lam, qn

    def encode(self, info_bits: np.ndarray) -> np.ndarray:
        """info_bits: uint8[K] -> codeword uint8[N]."""
        info = np.packbits(np.asarray(info_bits, np.uint8), bitorder="little")
        info = np.frombuffer(np.pad(info, (0, (-len(info)) % 4)).tobytes(), np.uint32).copy()
        cw = np.zeros(self.words, np.uint32)
        rc = _lib().oracle_encode(self._h, _ptr(info), _ptr(cw))
        if rc:
            raise ValueError(f"oracle_encode rc={rc}")
        return unpack_bits(cw, self.N)

    def syndrome_weight(self, bits: np.ndarray) -> int:
        w = pack_bits(np.asarray(bits, np.uint8))
        return int(_lib().oracle_syndrome_weight(self._h, _ptr(w)))

    def channel(self, ebn0_db: float, seed: int, frame_begin: int, frames: int, llr_mode: int = 0):
        llr = np.zeros((frames, self.N), np.float32)
        cw = np.zeros((frames, self.words), np.uint32)
        rc = _lib().oracle_channel(self._h, ebn0_db, seed, frame_begin, frames, llr_mode, _ptr(llr), self.N,
                                   _ptr(cw), self.words)
        if rc:
            raise ValueError(f"oracle_channel rc={rc}")
        return llr, cw

    def ber_sim(self, ebn0_db: float, seed: int, frame_begin: int, frames: int, max_iter: int,
                stop_rule: int = STOP_BELIEF_M, llr_mode: int = 0, arith: int = FP32_CONTRACT,
                alpha: float = ALPHA_DEFAULT) -> np.ndarray:
        counts = np.zeros(8, np.int64)
        o = Opts(max_iter, stop_rule, arith, alpha)
        rc = _lib().oracle_ber_sim(self._h, ebn0_db, seed, frame_begin, frames, ctypes.byref(o), llr_mode,
                                   _ptr(counts))
        if rc:
            raise ValueError(f"oracle_ber_sim rc={rc}")
        return counts

    def cbp_trace(self, llr: np.ndarray, sweeps: int) -> np.ndarray:
        lam = np.zeros((sweeps, self.E), np.float64)
        _lib().oracle_cbp_trace_f64(self._h, _ptr(np.ascontiguousarray(llr, np.float32)), sweeps, _ptr(lam))
        return lam

    def lbp_trace(self, llr: np.ndarray, sweeps: int) -> np.ndarray:
        lam = np.zeros((sweeps, self.E), np.float64)
        _lib().oracle_lbp_trace_f64(self._h, _ptr(np.ascontiguousarray(llr, np.float32)), sweeps, _ptr(lam))
        return lam

    def minsum_cbp_trace(self, llr: np.ndarray, sweeps: int, alpha: float = ALPHA_DEFAULT) -> np.ndarray:
        lam = np.zeros((sweeps, self.E), np.float32)
        _lib().oracle_minsum_cbp_trace(self._h, _ptr(np.ascontiguousarray(llr, np.float32)), sweeps, alpha,
                                       _ptr(lam))
        return lam

    def minsum_lbp_trace(self, llr: np.ndarray, sweeps: int, alpha: float = ALPHA_DEFAULT) -> np.ndarray:
        lam = np.zeros((sweeps, self.E), np.float32)
        _lib().oracle_minsum_lbp_trace(self._h, _ptr(np.ascontiguousarray(llr, np.float32)), sweeps, alpha,
                                       _ptr(lam))
        return lam

    def ml_decode(self, llr: np.ndarray) -> np.ndarray:
        cw = np.zeros(self.words, np.uint32)
        rc = _lib().oracle_ml_decode(self._h, _ptr(np.ascontiguousarray(llr, np.float32)), _ptr(cw))
        if rc:
            raise ValueError("oracle_ml_decode failed")
        return unpack_bits(cw, self.N)


COUNT_NAMES = ("frames", "bit_errors", "frame_errors", "cw_frame_errors", "iter_sum", "edge_visits",
               "not_converged", "undetected_fires")


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """uint8[N] (0/1) -> uint32 words, bit v%32 of word v/32."""
    b = np.packbits(np.asarray(bits, np.uint8), bitorder="little")
    b = np.pad(b, (0, (-len(b)) % 4))
    return np.frombuffer(b.tobytes(), np.uint32).copy()


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    w = np.ascontiguousarray(words, np.uint32)
    return np.unpackbits(w.view(np.uint8), bitorder="little")[:n]


def phi32(x: float) -> float:
    return float(_lib().oracle_phi32(x))


def phi32_array(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    _lib().oracle_phi32_n(_ptr(x), _ptr(y), x.size)
    return y


def ln32_array(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    _lib().oracle_ln32_n(_ptr(x), _ptr(y), x.size)
    return y


PHI_SEGS = 1153


def phi32_exhaustive():
    """(#below PHI_LO, #above PHI_HI, max ulp, argmax) of the unclamped v3 cubic over every
    binary32 x in [PHI_LO, 30], error against the double phi."""
    b, a, m, at = _i64(), _i64(), _f64(), _f32()
    _lib().oracle_phi32_exhaustive(ctypes.byref(b), ctypes.byref(a), ctypes.byref(m), ctypes.byref(at))
    return b.value, a.value, m.value, at.value


def phi32_table() -> np.ndarray:
    t = np.zeros((PHI_SEGS, 4), np.float32)
    _lib().oracle_phi32_table(_ptr(t))
    return t


def ln32(x: float) -> float:
    return float(_lib().oracle_ln32(x))


def sincos_quarter32(m24: int):
    s, c = _f32(), _f32()
    _lib().oracle_sincos_quarter32(m24, ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def philox4x32_10(ctr, key):
    c = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    _lib().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def normals(seed: int, frame: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float32)
    _lib().oracle_normals(seed, frame, n, _ptr(out))
    return out
