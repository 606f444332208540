"""Thin ctypes binding of libcbp.so (include/cbp.h).

Argument marshalling only: every step of the hot path runs in the sm_100a
kernels behind the C ABI.  PyTorch is used for device memory and streams.
There is no CPU fallback: if libcbp.so is missing or no CUDA device is
present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
# CBP_LIB selects an alternate build of the same library (A/B kernel experiments)
_SO = Path(os.environ["CBP_LIB"]) if os.environ.get("CBP_LIB") else _HERE / "libcbp.so"
_LIB = None

CBP_STOP_BELIEF_M, CBP_STOP_BELIEF_N, CBP_STOP_SYNDROME, CBP_STOP_NONE = 0, 1, 2, 3
COUNT_NAMES = ("frames", "bit_errors", "frame_errors", "cw_frame_errors", "iter_sum", "edge_visits",
               "not_converged", "undetected_fires")

_p, _i32, _i64, _u64, _f32, _f64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_float, ctypes.c_double)


class CbpError(RuntimeError):
    pass


class _Spec(ctypes.Structure):
    _fields_ = [(n, _i32) for n in ("mb", "nb", "Z", "mb_core", "wmode", "w_lo", "w_hi")]


class _Opts(ctypes.Structure):
    _fields_ = [("max_iter", _i32), ("stop_rule", _i32), ("algorithm", _i32), ("alpha", _f32)]


CBP_ALG_LOG_TANH, CBP_ALG_MIN_SUM, CBP_ALG_LBP, CBP_ALG_FBP = 0, 1, 2, 3
# llr_mode flags of channel / ber_sim (include/cbp.h): int8 stream, all-zero codeword (reading R23)
CBP_LLR_INT8, CBP_TX_ZERO = 1, 2
ALPHA_DEFAULT = 0.75
PHI_SEGS = 1153        # segments of the phi contract v3 table (include/cbp.h, cbp_phi_table)


def _opts(max_iter, stop_rule, algorithm, alpha):
    return _Opts(int(max_iter), int(stop_rule), int(algorithm), float(alpha))


class LaunchInfo(ctypes.Structure):
    _fields_ = [(n, _i32) for n in ("threads", "ctas_per_sm", "frames_per_cta", "smem_bytes", "state_in_smem",
                                    "num_sms", "frames_per_lane", "r_in_global")]


class _CodeConfig(ctypes.Structure):
    _fields_ = [("frames_per_lane", _i32)]


SIGNATURES = {
    "cbp_last_error": ([], ctypes.c_char_p),
    "cbp_version": ([], ctypes.c_char_p),
    "cbp_construct_base": ([_p, _u64, _p], _i32),
    "cbp_code_create": ([_p, _i32, _i32, _i32, _i32, _p], _i32),
    "cbp_code_create_ex": ([_p, _i32, _i32, _i32, _i32, _p, _p], _i32),
    "cbp_code_destroy": ([_p], None),
    "cbp_code_dims": ([_p, _p, _p, _p, _p], _i32),
    "cbp_decode": ([_p, _p, _i64, _i64, _p, _p, _i64, _p, _p, _p, _p, _p], _i32),
    "cbp_decode_i8": ([_p, _p, _i64, _f32, _i64, _p, _p, _i64, _p, _p, _p, _p, _p], _i32),
    "cbp_decode_host": ([_p, _p, _i64, _i64, _p, _p, _i64, _p, _p, _i64, _i32], _i32),
    "cbp_decode_host_i8": ([_p, _p, _i64, _f32, _i64, _p, _p, _i64, _p, _p, _i64, _i32], _i32),
    "cbp_channel": ([_p, _f64, _u64, _i64, _i64, _i32, _p, _i64, _p, _i64, _p], _i32),
    "cbp_ber_sim": ([_p, _f64, _u64, _i64, _i64, _p, _i32, _p, _p], _i32),
    "cbp_ber_count": ([_p, _p, _i64, _p, _i64, _i64, _p, _p, _p], _i32),
    "cbp_get_launch_info": ([_p, _p], _i32),
    "cbp_eval_contract": ([_i32, _p, _p, _i64, _i32, _p], _i32),
    "cbp_phi_table": ([_i32, _p, _p], _i32),
}


def lib():
    """Load libcbp.so (fails loudly if it was not built)."""
    global _LIB
    if _LIB is None:
        if not _SO.exists():
            raise CbpError(f"{_SO} not found: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(str(_SO))
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = L
    return _LIB


def _check(rc: int, what: str):
    if rc != 0:
        raise CbpError(f"{what} failed (status {rc}): {lib().cbp_last_error().decode()}")


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _dptr(t: torch.Tensor | None, dtype, device, name):
    if t is None:
        return None
    if not t.is_cuda or t.device != device:
        raise CbpError(f"{name} must be a CUDA tensor on {device}")
    if t.dtype != dtype:
        raise CbpError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise CbpError(f"{name} must be contiguous")
    return t.data_ptr()


def construct_base(spec, seed: int):
    """cbp_construct_base: spec = (mb, nb, Z, mb_core, wmode, w_lo, w_hi) -> int16 [mb, nb] (torch, CPU)."""
    s = _Spec(*[int(x) for x in spec])
    out = torch.empty((s.mb, s.nb), dtype=torch.int16)
    _check(lib().cbp_construct_base(ctypes.byref(s), seed, out.data_ptr()), "cbp_construct_base")
    return out


class Code:
    """cbp_code_create_ex / cbp_code_destroy: a QC code resident on one CUDA device.
    frames_per_lane: 0 automatic, 1 or 2 (a performance setting; results are identical)."""

    def __init__(self, base, Z: int, device=None, frames_per_lane: int = 0):
        base_t = torch.as_tensor(base, dtype=torch.int16).contiguous().cpu()
        self.mb, self.nb = base_t.shape
        self.Z = int(Z)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        h = ctypes.c_void_p()
        cfg = _CodeConfig(int(frames_per_lane))
        _check(lib().cbp_code_create_ex(base_t.data_ptr(), self.mb, self.nb, self.Z, self.device.index,
                                        ctypes.byref(cfg), ctypes.byref(h)), "cbp_code_create_ex")
        self._h = h
        N, K, M, E = _i32(), _i32(), _i32(), _i64()
        _check(lib().cbp_code_dims(h, ctypes.byref(N), ctypes.byref(K), ctypes.byref(M), ctypes.byref(E)),
               "cbp_code_dims")
        self.N, self.K, self.M, self.E = N.value, K.value, M.value, E.value
        self.words = (self.N + 31) // 32

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _LIB is not None:
            _LIB.cbp_code_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def launch_info(self) -> dict:
        li = LaunchInfo()
        _check(lib().cbp_get_launch_info(self._h, ctypes.byref(li)), "cbp_get_launch_info")
        return {n: getattr(li, n) for n, _ in LaunchInfo._fields_}

    # -------------------------------------------------------------- decode
    def alloc_outputs(self, frames: int, omega: bool = False, ev: bool = False) -> dict:
        d = self.device
        out = {"bits": torch.empty((frames, self.words), dtype=torch.int32, device=d),
               "iters": torch.empty(frames, dtype=torch.int32, device=d),
               "flags": torch.empty(frames, dtype=torch.uint8, device=d)}
        if omega:
            out["omega"] = torch.empty((frames, self.M), dtype=torch.float32, device=d)
        if ev:
            out["ev"] = torch.empty(frames, dtype=torch.int64, device=d)
        return out

    def _check_out(self, out: dict, frames: int, who: str):
        """The C ABI cannot see buffer sizes: every output must hold `frames` rows (omega [frames, M])."""
        rows = {"bits": 2, "iters": 1, "flags": 1, "omega": 2, "ev": 1}
        for k, t in out.items():
            if k not in rows or t is None:
                continue
            if t.dim() != rows[k] or t.shape[0] < frames:
                raise CbpError(f"{who}: out[{k!r}] must be {rows[k]}-D with >= {frames} rows, got {tuple(t.shape)}")
        if out["bits"].shape[1] < self.words:
            raise CbpError(f"{who}: out['bits'] needs >= {self.words} words per frame")
        if out.get("omega") is not None and out["omega"].shape[1] != self.M:
            raise CbpError(f"{who}: out['omega'] must be [frames, M={self.M}]")

    def decode(self, llr: torch.Tensor, max_iter: int, stop_rule: int = CBP_STOP_BELIEF_M, out: dict | None = None,
               omega: bool = False, ev: bool = False, stream=None, algorithm: int = CBP_ALG_LOG_TANH,
               alpha: float = ALPHA_DEFAULT) -> dict:
        """cbp_decode: llr float32 [frames, ld] on the code's device (ld >= N, ld % 4 == 0)."""
        frames, ld = llr.shape
        out = out if out is not None else self.alloc_outputs(frames, omega, ev)
        self._check_out(out, frames, "decode")
        o = _opts(max_iter, stop_rule, algorithm, alpha)
        d = self.device
        rc = lib().cbp_decode(self._h, _dptr(llr, torch.float32, d, "llr"), ld, frames, ctypes.byref(o),
                              _dptr(out["bits"], torch.int32, d, "bits"), out["bits"].shape[1],
                              _dptr(out["iters"], torch.int32, d, "iters"), _dptr(out["flags"], torch.uint8, d, "flags"),
                              _dptr(out.get("omega"), torch.float32, d, "omega"),
                              _dptr(out.get("ev"), torch.int64, d, "ev"), _stream(stream))
        _check(rc, "cbp_decode")
        return out

    def decode_i8(self, q: torch.Tensor, scale: float, max_iter: int, stop_rule: int = CBP_STOP_BELIEF_M,
                  out: dict | None = None, omega: bool = False, ev: bool = False, stream=None,
                  algorithm: int = CBP_ALG_LOG_TANH, alpha: float = ALPHA_DEFAULT) -> dict:
        """cbp_decode_i8: q int8 [frames, ld] (ld % 16 == 0), L = scale * q."""
        frames, ld = q.shape
        out = out if out is not None else self.alloc_outputs(frames, omega, ev)
        self._check_out(out, frames, "decode_i8")
        o = _opts(max_iter, stop_rule, algorithm, alpha)
        d = self.device
        rc = lib().cbp_decode_i8(self._h, _dptr(q, torch.int8, d, "q"), ld, scale, frames, ctypes.byref(o),
                                 _dptr(out["bits"], torch.int32, d, "bits"), out["bits"].shape[1],
                                 _dptr(out["iters"], torch.int32, d, "iters"),
                                 _dptr(out["flags"], torch.uint8, d, "flags"),
                                 _dptr(out.get("omega"), torch.float32, d, "omega"),
                                 _dptr(out.get("ev"), torch.int64, d, "ev"), _stream(stream))
        _check(rc, "cbp_decode_i8")
        return out

    # -------------------------------------------------------------- host buffers
    def alloc_host_outputs(self, frames: int) -> dict:
        """pinned host outputs of decode_host"""
        return {"bits": torch.empty((frames, self.words), dtype=torch.int32, pin_memory=True),
                "iters": torch.empty(frames, dtype=torch.int32, pin_memory=True),
                "flags": torch.empty(frames, dtype=torch.uint8, pin_memory=True)}

    def decode_host(self, llr: torch.Tensor, max_iter: int, stop_rule: int = CBP_STOP_BELIEF_M,
                    out: dict | None = None, scale: float | None = None, chunk_frames: int = 0, nstreams: int = 0,
                    algorithm: int = CBP_ALG_LOG_TANH, alpha: float = ALPHA_DEFAULT) -> dict:
        """cbp_decode_host / cbp_decode_host_i8: host (pinned) float32 [frames, ld] LLRs, or int8
        [frames, ld] with `scale`, -> host outputs; blocks until the outputs are in host memory."""
        if llr.is_cuda or llr.dim() != 2 or not llr.is_contiguous():
            raise CbpError("decode_host: llr must be a contiguous 2-D host tensor")
        frames, ld = llr.shape
        out = out if out is not None else self.alloc_host_outputs(frames)
        for k, dt in (("bits", torch.int32), ("iters", torch.int32), ("flags", torch.uint8)):
            t = out[k]
            if t.is_cuda or t.dtype != dt or not t.is_contiguous() or t.shape[0] < frames:
                raise CbpError(f"decode_host: out[{k!r}] must be a contiguous host {dt} tensor with >= {frames} rows")
        if out["bits"].dim() != 2 or out["bits"].shape[1] < self.words:
            raise CbpError(f"decode_host: out['bits'] needs >= {self.words} words per frame")
        o = _opts(max_iter, stop_rule, algorithm, alpha)
        if llr.dtype == torch.int8:
            if scale is None:
                raise CbpError("decode_host: int8 LLRs need `scale`")
            rc = lib().cbp_decode_host_i8(self._h, llr.data_ptr(), ld, float(scale), frames, ctypes.byref(o),
                                          out["bits"].data_ptr(), out["bits"].shape[1], out["iters"].data_ptr(),
                                          out["flags"].data_ptr(), chunk_frames, nstreams)
            _check(rc, "cbp_decode_host_i8")
        elif llr.dtype == torch.float32:
            rc = lib().cbp_decode_host(self._h, llr.data_ptr(), ld, frames, ctypes.byref(o), out["bits"].data_ptr(),
                                       out["bits"].shape[1], out["iters"].data_ptr(), out["flags"].data_ptr(),
                                       chunk_frames, nstreams)
            _check(rc, "cbp_decode_host")
        else:
            raise CbpError("decode_host: llr must be float32 or int8")
        return out

    # -------------------------------------------------------------- channel / ber
    def channel(self, ebn0_db: float, seed: int, frame_begin: int, frames: int, llr_mode: int = 0,
                ld: int | None = None, want_llr: bool = True, want_cw: bool = True, stream=None, out=None):
        """cbp_channel: returns (llr float32 [frames, ld] or None, codewords int32 [frames, words] or None);
        `out` = (llr, cw): caller's buffers (either may be None), written instead of new ones."""
        d = self.device
        if out is not None:
            llr, cw = out
            for t, nm, cols in ((llr, "llr", self.N), (cw, "cw", self.words)):
                if t is not None and (t.dim() != 2 or t.shape[0] != frames or t.shape[1] < cols):
                    raise CbpError(f"channel: out {nm} must be [frames={frames}, >= {cols}], got {tuple(t.shape)}")
            ld = llr.shape[1] if llr is not None else (self.N + 3) // 4 * 4
            wds = cw.shape[1] if cw is not None else self.words
        else:
            ld = ld or (self.N + 3) // 4 * 4
            wds = self.words
            llr = torch.empty((frames, ld), dtype=torch.float32, device=d) if want_llr else None
            cw = torch.empty((frames, self.words), dtype=torch.int32, device=d) if want_cw else None
        rc = lib().cbp_channel(self._h, float(ebn0_db), seed, frame_begin, frames, llr_mode,
                               _dptr(llr, torch.float32, d, "llr"), ld, _dptr(cw, torch.int32, d, "cw"), wds,
                               _stream(stream))
        _check(rc, "cbp_channel")
        return llr, cw

    def ber_sim(self, ebn0_db: float, seed: int, frame_begin: int, frames: int, max_iter: int,
                stop_rule: int = CBP_STOP_BELIEF_M, llr_mode: int = 0, counts: torch.Tensor | None = None,
                stream=None, algorithm: int = CBP_ALG_LOG_TANH, alpha: float = ALPHA_DEFAULT) -> torch.Tensor:
        """cbp_ber_sim: accumulates into `counts` (int64 [8] on device; zeroed if not given)."""
        if counts is None:
            counts = torch.zeros(8, dtype=torch.int64, device=self.device)
        if counts.numel() != 8:
            raise CbpError("ber_sim: counts must hold the 8 int64 counters of cbp_counts")
        o = _opts(max_iter, stop_rule, algorithm, alpha)
        rc = lib().cbp_ber_sim(self._h, float(ebn0_db), seed, frame_begin, frames, ctypes.byref(o), llr_mode,
                               _dptr(counts, torch.int64, self.device, "counts"), _stream(stream))
        _check(rc, "cbp_ber_sim")
        return counts

    def ber_count(self, llr: torch.Tensor, cw: torch.Tensor, max_iter: int, stop_rule: int = CBP_STOP_BELIEF_M,
                  counts: torch.Tensor | None = None, stream=None, algorithm: int = CBP_ALG_LOG_TANH,
                  alpha: float = ALPHA_DEFAULT) -> torch.Tensor:
        """cbp_ber_count: decode fp32 LLRs [frames, ld] and count errors against the codewords [frames, words]
        (int32 words, as `channel` returns them); accumulates into `counts` (zeroed if not given)."""
        if counts is None:
            counts = torch.zeros(8, dtype=torch.int64, device=self.device)
        if counts.numel() != 8:
            raise CbpError("ber_count: counts must hold the 8 int64 counters of cbp_counts")
        if llr.dim() != 2 or cw.dim() != 2 or cw.shape[0] < llr.shape[0]:
            raise CbpError(f"ber_count: llr [frames, ld] and cw [>= frames, words] expected, got {tuple(llr.shape)}, "
                           f"{tuple(cw.shape)}")
        if cw.shape[1] < self.words:
            raise CbpError(f"ber_count: cw needs >= {self.words} words per frame")
        frames, ld = llr.shape
        o = _opts(max_iter, stop_rule, algorithm, alpha)
        rc = lib().cbp_ber_count(self._h, _dptr(llr, torch.float32, self.device, "llr"), ld,
                                 _dptr(cw, torch.int32, self.device, "cw"), cw.shape[1], frames, ctypes.byref(o),
                                 _dptr(counts, torch.int64, self.device, "counts"), _stream(stream))
        _check(rc, "cbp_ber_count")
        return counts


def eval_contract(fn: int, x: torch.Tensor, stream=None) -> torch.Tensor:
    """cbp_eval_contract: device evaluation of phi32 (0), ln32 (1), sin (2) / cos (3) of 2 pi m 2^-24."""
    y = torch.empty_like(x)
    _check(lib().cbp_eval_contract(fn, _dptr(x, torch.float32, x.device, "x"), y.data_ptr(), x.numel(),
                                   x.device.index, _stream(stream)), "cbp_eval_contract")
    return y


def phi_table(device: int = 0, stream=None) -> torch.Tensor:
    """cbp_phi_table: the device's phi contract v3 table, float32 [PHI_SEGS, 4] (on the device)."""
    out = torch.empty((PHI_SEGS, 4), dtype=torch.float32, device=torch.device("cuda", device))
    _check(lib().cbp_phi_table(device, out.data_ptr(), _stream(stream)), "cbp_phi_table")
    return out


def unpack_bits(words: torch.Tensor, n: int) -> torch.Tensor:
    """int32/uint32 words [.., W] (bit v%32 of word v/32) -> uint8 bits [.., n] (on the same device)."""
    w = words.to(torch.int64) & 0xFFFFFFFF
    shifts = torch.arange(32, device=words.device, dtype=torch.int64)
    b = (w.unsqueeze(-1) >> shifts) & 1
    return b.reshape(*words.shape[:-1], -1)[..., :n].to(torch.uint8)
