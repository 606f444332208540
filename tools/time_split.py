"""Split the timed region of one cbp_ber_sim call: host enqueue time, CUDA-event
time, and the kernel's own duration from the torch profiler (CUPTI).

python tools/time_split.py C2 [frames_per_lane]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2305_05286_b200 as cbp  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
fpl = int(sys.argv[2]) if len(sys.argv) > 2 else 0
frames = int(sys.argv[3]) if len(sys.argv) > 3 else 100_000
base, Z = inputs.config_base(cfgname)
g = cbp.Code(base, Z, frames_per_lane=fpl)
print(g.launch_info())
mi = inputs.CONFIGS[cfgname].max_iter
cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
for _ in range(3):
    g.ber_sim(2.0, 1, 0, frames, mi, counts=cnt)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    g.ber_sim(2.0, 1, 0, frames, mi, counts=cnt)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: host enqueue {1e3 * (t1 - t0):.3f} ms, events {e0.elapsed_time(e1):.3f} ms")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        g.ber_sim(2.0, 1, 0, frames, mi, counts=cnt)
    torch.cuda.synchronize()
for ev in prof.key_averages():
    if "cbp" in ev.key or "emset" in ev.key:
        print(ev.key[:60], ev.count, f"{ev.device_time_total / max(ev.count, 1) / 1e3:.3f} ms avg")
