"""A/B of cbp_ber_sim fused vs split (channel + decode launches through an HBM chunk): counters must be
identical, times per launch (CUDA events, best of reps).
python tools/ab_split.py --config C5 --ebn0 2.5 --frames 400000"""
import argparse
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--ebn0", type=float, default=2.5)
ap.add_argument("--frames", type=int, default=400_000)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--child", default="")
a = ap.parse_args()

if not a.child:
    res = {}
    for split in ("0", "1"):
        env = dict(os.environ, CBP_BER_SPLIT=split)
        out = subprocess.run([sys.executable, __file__, "--config", a.config, "--ebn0", str(a.ebn0), "--frames",
                              str(a.frames), "--reps", str(a.reps), "--child", split], env=env, capture_output=True,
                             text=True, timeout=600)
        print(out.stdout.strip(), out.stderr.strip()[-500:])
        res[split] = out.stdout.strip().split("counts=")[-1]
    print("counters identical:", res["0"] == res["1"])
    sys.exit(0)

import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2305_05286_b200 as cbp  # noqa: E402

cfg = inputs.get_config(a.config)
base, Z = inputs.config_base(a.config)
g = cbp.Code(base, Z)
for _ in range(2):
    g.ber_sim(a.ebn0, 1, 0, a.frames, cfg.max_iter)
torch.cuda.synchronize()
best = None
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c = g.ber_sim(a.ebn0, 1, 0, a.frames, cfg.max_iter)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    best = ms if best is None else min(best, ms)
print(f"split={a.child} {a.config} {a.ebn0} dB {a.frames} frames: best {best:.3f} ms "
      f"({a.frames / best * 1e3:.3e} frames/s) counts={c.cpu().tolist()}")
