"""Normalized min-sum CBP: FER and sweeps against the normalisation alpha (PAPER.md
l.577-603 leaves alpha open, reading R20) on one code, with the log-tanh CBP beside it
on the same frames.  One JSON line per (alpha, Eb/N0).

python tools/alpha_sweep.py --config P8192 --frames 20000 --ebn0 1.25,1.5
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2305_05286_b200 as cbp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--frames", type=int, default=20_000)
ap.add_argument("--ebn0", default=None)
ap.add_argument("--alphas", default="0.7,0.75,0.8,0.85,0.9,0.95,1.0")
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
cfg = inputs.get_config(a.config)
lm = cbp.CBP_TX_ZERO if inputs.is_peg(a.config) else 0
ebs = [float(x) for x in a.ebn0.split(",")] if a.ebn0 else list(cfg.ebn0_db)
base, Z = inputs.config_base(a.config)
code = cbp.Code(base, Z)
cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
runs = [("log-tanh CBP", 0, 1.0)] + [("min-sum CBP", 1, float(x)) for x in a.alphas.split(",")]
for eb in ebs:
    for name, alg, alpha in runs:
        cnt.zero_()
        code.ber_sim(eb, a.seed, 0, a.frames, cfg.max_iter, 0, lm, counts=cnt, algorithm=alg, alpha=alpha)
        t = cnt.cpu().tolist()
        print(json.dumps({"config": a.config, "decoder": name, "alpha": alpha if alg == 1 else None, "ebn0_db": eb,
                          "frames": t[0], "fer": t[2] / t[0], "ber": t[1] / (t[0] * code.K), "avg_iters": t[4] / t[0],
                          "not_converged": t[6], "max_iter": cfg.max_iter, "llr_mode": lm}), flush=True)
