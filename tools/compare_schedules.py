"""The paper's schedule comparison (Fig. 6-9, l.613-724: error rate and
average iterations of CBP vs LBP vs FBP, and normalized min-sum CBP, Fig. 10-12)
on one BASELINE code, or one of the paper's own PEG families (P2048, P8192; all-zero
codeword, reading R23), at GPU scale: fused cbp_ber_sim, same frames (seeded
channel) for every decoder, one JSON line per (decoder, Eb/N0).

python tools/compare_schedules.py --config C2 --frames 1000000 > profiles/r01b_schedules_C2.jsonl
python tools/compare_schedules.py --config P2048 --frames 100000
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
ap.add_argument("--frames", type=int, default=1_000_000)
ap.add_argument("--ebn0", default=None)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--alphas", default="0.75", help="normalized min-sum alphas (R20), comma list")
a = ap.parse_args()
cfg = inputs.get_config(a.config)
llr_mode = cbp.CBP_TX_ZERO if inputs.is_peg(a.config) else 0
ebs = [float(x) for x in a.ebn0.split(",")] if a.ebn0 else list(cfg.ebn0_db)
base, Z = inputs.config_base(a.config)
code = cbp.Code(base, Z)
DECODERS = [("CBP belief W=M", 0, 0, 0.75), ("CBP syndrome", 0, 2, 0.75), ("LBP syndrome", 2, 2, 0.75),
            ("FBP syndrome", 3, 2, 0.75)]
DECODERS += [("min-sum CBP belief W=M" + ("" if x == "0.75" else f" alpha {x}"), 1, 0, float(x))
             for x in a.alphas.split(",")]
cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
for name, alg, rule, alpha in DECODERS:
    for eb in ebs:
        cnt.zero_()
        code.ber_sim(eb, a.seed, 0, min(a.frames, 20000), cfg.max_iter, rule, llr_mode, algorithm=alg, alpha=alpha, counts=cnt)
        cnt.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        code.ber_sim(eb, a.seed, 0, a.frames, cfg.max_iter, rule, llr_mode, algorithm=alg, alpha=alpha, counts=cnt)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        t = cnt.cpu().tolist()
        print(json.dumps({"config": a.config, "decoder": name, "algorithm": alg, "alpha": alpha if alg == 1 else None, "stop_rule": rule, "ebn0_db": eb,
                          "frames": t[0], "ber": t[1] / (t[0] * code.K), "fer": t[2] / t[0],
                          "avg_iters": t[4] / t[0], "not_converged": t[6], "edge_visits": t[5], "ms": ms,
                          "frames_per_s": t[0] / ms * 1e3, "edge_visits_per_s": t[5] / ms * 1e3,
                          "max_iter": cfg.max_iter, "seed": a.seed, "llr_mode": llr_mode}), flush=True)
