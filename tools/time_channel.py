"""Time cbp_channel alone (CUDA events, best of reps) for A/B runs of the channel launch.

python tools/time_channel.py --config C5 --ebn0 2.5 --frames 1048576
"""
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
ap.add_argument("--frames", type=int, default=1 << 20)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--mode", type=int, default=0, help="llr_mode (1: int8 stream, 2: all-zero codeword)")
a = ap.parse_args()
base, Z = inputs.config_base(a.config)
lm = a.mode | (cbp.CBP_TX_ZERO if inputs.is_peg(a.config) else 0)
g = cbp.Code(base, Z)
ld = (g.N + 3) // 4 * 4
llr = torch.empty((a.frames, ld), dtype=torch.float32, device="cuda")
cw = torch.empty((a.frames, g.words), dtype=torch.int32, device="cuda")
best = None
for rep in range(a.reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.channel(a.ebn0, 1, 0, a.frames, llr_mode=lm, out=(llr, cw))
    e1.record()
    torch.cuda.synchronize()
    if rep:
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
print(f"channel {a.config} {a.frames} frames: best {best:.3f} ms  {best / a.frames * 1e6:.2f} ns/frame  "
      f"checksum {llr[:, :g.N].double().sum().item():.6f} {cw.long().sum().item()}")
