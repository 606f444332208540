"""Time split of the fused cbp_ber_sim against its parts on one workload (CUDA events):
ber_sim (channel + decode + counting in one kernel), cbp_channel alone, cbp_decode of the same
frames from HBM.  python tools/split_ber.py --config C5 --ebn0 2.5 --frames 200000"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2305_05286_b200 as cbp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--ebn0", type=float, default=2.5)
ap.add_argument("--frames", type=int, default=200_000)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
cfg = inputs.get_config(a.config)
base, Z = inputs.config_base(a.config)
g = cbp.Code(base, Z)


def timed(fn):
    best = None
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best, r


for _ in range(3):
    g.ber_sim(a.ebn0, 1, 0, a.frames, cfg.max_iter)
torch.cuda.synchronize()
t_ber, c = timed(lambda: g.ber_sim(a.ebn0, 1, 0, a.frames, cfg.max_iter))
t_ch, (llr, _) = timed(lambda: g.channel(a.ebn0, 1, 0, a.frames, want_cw=False))
t_dec, out = timed(lambda: g.decode(llr, cfg.max_iter, ev=True))
ev_b, ev_d = int(c[5].item()), int(out["ev"].sum().item())
print(f"{a.config} {a.ebn0} dB {a.frames} frames: ber_sim {t_ber:.3f} ms ({ev_b / t_ber * 1e3:.3e} EV/s); "
      f"channel {t_ch:.3f} ms; decode {t_dec:.3f} ms ({ev_d / t_dec * 1e3:.3e} EV/s); channel+decode {t_ch + t_dec:.3f} ms")
print(g.launch_info())
