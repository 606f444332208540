"""Host-buffer decoding: the C ABI's cbp_decode_host (include/cbp.h) -- chunked H2D ->
cbp_decode -> D2H pipelined over library-owned CUDA streams, so PCIe transfers overlap the
decode kernels.  This module only keeps the round-1 Python entry points as thin wrappers."""
from __future__ import annotations

import torch

from .cbp import CBP_STOP_BELIEF_M, Code

API_NAME = "cbp_decode_host (C ABI: chunked H2D -> decode -> D2H on 4 library streams)"


def alloc_host_outputs(code: Code, frames: int) -> dict:
    return code.alloc_host_outputs(frames)


def decode_host(code: Code, llr_host: torch.Tensor, max_iter: int, stop_rule: int = CBP_STOP_BELIEF_M,
                out: dict | None = None, chunk: int = 1 << 14, nstreams: int = 4) -> dict:
    """Decode float32 LLRs [frames, ld] held in (pinned) host memory; returns host outputs."""
    return code.decode_host(llr_host, max_iter, stop_rule, out=out, chunk_frames=chunk, nstreams=nstreams)
