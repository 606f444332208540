"""One warm-up + one measured cbp_ber_sim launch (for ncu captures).

python tools/prof_one.py --config C2 --ebn0 2.0 --frames 100000
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2305_05286_b200 as cbp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--ebn0", type=float, default=2.0)
ap.add_argument("--frames", type=int, default=100_000)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--mode", default="ber", choices=["ber", "decode"])
a = ap.parse_args()
cfg = inputs.CONFIGS[a.config]
base, Z = inputs.config_base(a.config)
g = cbp.Code(base, Z)
print(g.launch_info())
if a.mode == "decode":
    llr, _ = g.channel(a.ebn0, 1, 0, a.frames, want_cw=False)
g.ber_sim(a.ebn0, 1, 0, 4096, cfg.max_iter)
torch.cuda.synchronize()
for _ in range(a.reps):
    t0 = time.perf_counter()
    if a.mode == "ber":
        c = g.ber_sim(a.ebn0, 1, 0, a.frames, cfg.max_iter)
    else:
        out = g.decode(llr, cfg.max_iter, ev=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if a.mode == "ber":
        c = c.cpu().tolist()
        print(dict(zip(cbp.COUNT_NAMES, c)), f"{dt * 1e3:.2f} ms  {c[0] / dt:.3e} frames/s  "
              f"{c[5] / dt:.3e} EV/s")
    else:
        ev = out["ev"].sum().item()
        print(f"decode {dt * 1e3:.2f} ms {a.frames / dt:.3e} frames/s {ev / dt:.3e} EV/s")
