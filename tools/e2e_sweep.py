"""Tune pipeline.decode_host: chunk size x number of streams, plus raw pinned H2D
bandwidth, on the bench's e2e workload (C2 at 2.0 dB, 200k host-resident frames)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2305_05286_b200 as cbp  # noqa: E402
from paper_2305_05286_b200 import pipeline  # noqa: E402

EB = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
base, Z = inputs.config_base("C2")
code = cbp.Code(base, Z)
F = 200_000
ld = (code.N + 3) // 4 * 4
host = torch.empty((F, ld), dtype=torch.float32, pin_memory=True)
for b in range(0, F, 1 << 17):
    n = min(1 << 17, F - b)
    llr, _ = code.channel(EB, 2, b, n, want_cw=False)
    host[b:b + n].copy_(llr)
dev = torch.empty_like(host, device="cuda")
for _ in range(2):
    dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
bw = 5 * host.numel() * 4 / (time.perf_counter() - t0)
print(f"raw pinned H2D {bw / 1e9:.1f} GB/s")
t0 = time.perf_counter()
out = code.decode(dev, 30)
torch.cuda.synchronize()
t1 = time.perf_counter()
out = code.decode(dev, 30)
torch.cuda.synchronize()
print(f"device-resident decode {F / (time.perf_counter() - t1):.3e} frames/s at {EB} dB")
cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
code.ber_sim(EB, 2, 0, F, 30, counts=cnt)
torch.cuda.synchronize()
t1 = time.perf_counter()
code.ber_sim(EB, 2, 0, F, 30, counts=cnt)
torch.cuda.synchronize()
print(f"fused ber_sim {F / (time.perf_counter() - t1):.3e} frames/s")
hout = pipeline.alloc_host_outputs(code, F)
for chunk in (1 << 14, 1 << 15, 1 << 16):
    for ns in (4, 6):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        pipeline.decode_host(code, host, 30, out=hout, chunk=chunk, streams=streams)
        t0 = time.perf_counter()
        for _ in range(3):
            pipeline.decode_host(code, host, 30, out=hout, chunk=chunk, streams=streams)
        te = (time.perf_counter() - t0) / 3
        print(f"chunk {chunk:7d} streams {ns}: {F / te:.3e} frames/s  {F * code.K / te / 1e9:.2f} info Gbit/s")
