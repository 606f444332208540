"""Experiment: end-to-end decode of pinned host LLRs with the kernel reading them in
place (mapped pinned memory under UVA, one launch for the whole batch, outputs written
straight to pinned host memory) against pipeline.decode_host (chunked H2D / decode /
D2H over four streams).  C2, 200k frames, at the given Eb/N0 points."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2305_05286_b200 as cbp  # noqa: E402
from paper_2305_05286_b200 import pipeline  # noqa: E402
from paper_2305_05286_b200.cbp import _opts, lib  # noqa: E402

base, Z = inputs.config_base("C2")
code = cbp.Code(base, Z)
F = 200_000
ld = (code.N + 3) // 4 * 4
for eb in [float(x) for x in (sys.argv[1:] or ["1.0", "2.0", "3.0"])]:
    host = torch.empty((F, ld), dtype=torch.float32, pin_memory=True)
    for b in range(0, F, 1 << 17):
        n = min(1 << 17, F - b)
        llr, _ = code.channel(eb, 2, b, n, want_cw=False)
        host[b:b + n].copy_(llr)
    torch.cuda.synchronize()
    ref = pipeline.decode_host(code, host, 30)
    hout = pipeline.alloc_host_outputs(code, F)
    t0 = time.perf_counter()
    for _ in range(3):
        pipeline.decode_host(code, host, 30, out=hout)
    tp = (time.perf_counter() - t0) / 3
    zb = torch.empty((F, code.words), dtype=torch.int32, pin_memory=True)
    zi = torch.empty(F, dtype=torch.int32, pin_memory=True)
    zf = torch.empty(F, dtype=torch.uint8, pin_memory=True)
    o = _opts(30, 0, 0, 0.75)
    st = torch.cuda.current_stream().cuda_stream

    def zc():
        rc = lib().cbp_decode(code.handle, host.data_ptr(), ld, F, ctypes.byref(o), zb.data_ptr(), code.words,
                              zi.data_ptr(), zf.data_ptr(), None, None, st)
        assert rc == 0, lib().cbp_last_error()
    zc()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        zc()
        torch.cuda.synchronize()
    tz = (time.perf_counter() - t0) / 3
    same = torch.equal(zb, ref["bits"]) and torch.equal(zi, ref["iters"]) and torch.equal(zf, ref["flags"])
    print(f"{eb} dB: pipeline {F / tp:.3e} frames/s, zero-copy {F / tz:.3e} frames/s, identical {same}", flush=True)
