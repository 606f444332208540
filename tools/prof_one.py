"""Warm-up (~1 s) then timed cbp_ber_sim / cbp_decode launches (CUDA events).

python tools/prof_one.py --config C2 --ebn0 2.0 --frames 100000 --reps 5
Under ncu, the measured launch is the second kernel launch of the run (-s 1 -c 1).
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
ap.add_argument("--warm", type=float, default=1.0, help="seconds of warm-up (0 under ncu)")
ap.add_argument("--mode", default="ber", choices=["ber", "decode"])
ap.add_argument("--rule", type=int, default=0)
ap.add_argument("--alg", type=int, default=0, help="0 log-tanh, 1 normalized min-sum")
ap.add_argument("--alpha", type=float, default=0.75)
ap.add_argument("--fpl", type=int, default=0, help="frames per lane: 0 auto, 1, 2")
a = ap.parse_args()
ALG = dict(algorithm=a.alg, alpha=a.alpha)
cfg = inputs.get_config(a.config)
LM = cbp.CBP_TX_ZERO if inputs.is_peg(a.config) else 0   # PEG codes: all-zero codeword (R23)
base, Z = inputs.config_base(a.config)
g = cbp.Code(base, Z, frames_per_lane=a.fpl)
print(g.launch_info())
if a.mode == "decode":
    llr, _ = g.channel(a.ebn0, 1, 0, a.frames, llr_mode=LM, want_cw=False)
g.ber_sim(a.ebn0, 1, 0, 4096, cfg.max_iter, llr_mode=LM)
torch.cuda.synchronize()
t_end = time.perf_counter() + a.warm
while time.perf_counter() < t_end:
    g.ber_sim(a.ebn0, 1, 0, a.frames, cfg.max_iter, stop_rule=a.rule, llr_mode=LM, **ALG)
    torch.cuda.synchronize()
best = None
cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
for _ in range(a.reps):
    cnt.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if a.mode == "ber":
        c = g.ber_sim(a.ebn0, 1, 0, a.frames, cfg.max_iter, stop_rule=a.rule, llr_mode=LM, counts=cnt, **ALG)
    else:
        out = g.decode(llr, cfg.max_iter, a.rule, ev=True, **ALG)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ev = c[5].item() if a.mode == "ber" else out["ev"].sum().item()
    best = ms if best is None else min(best, ms)
    if a.mode == "ber":
        print(dict(zip(cbp.COUNT_NAMES, c.cpu().tolist())), f"{ms:.3f} ms  {a.frames / ms * 1e3:.3e} frames/s  "
              f"{ev / ms * 1e3:.3e} EV/s")
    else:
        print(f"decode {ms:.3f} ms {a.frames / ms * 1e3:.3e} frames/s {ev / ms * 1e3:.3e} EV/s")
print(f"best {best:.3f} ms")
