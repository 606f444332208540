"""Resumable, multi-GPU BER/FER sweeps over Eb/N0 points (SURVEY B13 / §5 checkpoint-resume).

A sweep decodes global frames [0, frames) at every Eb/N0 point in chunks.  Each chunk
is split over the ranks of the process group (frame-range shards, `dist.shard_range`),
decoded with the fused cbp_ber_sim and summed with one all-reduce of the 8 counters;
rank 0 then appends one JSON line per finished (point, chunk) to the checkpoint file.
The channel is keyed by (seed, global frame index), so the totals depend on neither
the world size, the chunk size nor on where a sweep was interrupted: a rerun with
resume=True skips the chunks already in the file and ends with the same totals.

    python -m paper_2305_05286_b200.sweep --config C2 --frames 10000000 --out c2.jsonl
    torchrun --nproc-per-node 8 -m paper_2305_05286_b200.sweep --config C5 --frames 1000000000 --out c5.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
from pathlib import Path
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from .dist import allreduce_counts, shard_range

COUNT_NAMES = ("frames", "bit_errors", "frame_errors", "cw_frame_errors", "iter_sum", "edge_visits",
               "not_converged", "undetected_fires")

# runner(ebn0_db, frame_begin, frames) -> int64[8] counts of this rank's slice
Runner = Callable[[float, int, int], np.ndarray]


def gpu_runner(code, max_iter: int, seed: int, stop_rule: int = 0, algorithm: int = 0, alpha: float = 0.75,
               llr_mode: int = 0) -> Runner:
    """The product runner: cbp_ber_sim on the code's device."""
    def run(ebn0: float, begin: int, n: int) -> np.ndarray:
        c = torch.zeros(8, dtype=torch.int64, device=code.device)
        if n > 0:
            code.ber_sim(ebn0, seed, begin, n, max_iter, stop_rule, llr_mode, counts=c, algorithm=algorithm,
                         alpha=alpha)
        return c.cpu().numpy()
    return run


def _world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def _load_done(path: Path, header: dict) -> dict:
    """(ebn0, chunk) -> counts of the checkpoint lines that match `header`."""
    done = {}
    if not path.exists():
        return done
    lines = path.read_text().splitlines()
    if not lines:
        return done
    head = json.loads(lines[0])
    if head.get("header") != header:
        raise ValueError(f"checkpoint {path} belongs to another sweep: {head.get('header')} != {header}")
    for ln in lines[1:]:
        if not ln.strip():
            continue
        d = json.loads(ln)
        done[(float(d["ebn0_db"]), int(d["chunk"]))] = np.array(d["counts"], np.int64)
    return done


def run_sweep(runner: Runner, ebn0s, frames: int, chunk: int, header: dict, out: str | os.PathLike | None = None,
              resume: bool = True, group=None, counts_device=None) -> dict:
    """Run (or resume) a sweep; returns {ebn0: summary dict} on every rank.

    header: the sweep's identity (code, seed, decoder options); stored as the first line
    of the checkpoint and checked on resume.  counts_device: where the all-reduce buffer
    lives (the process group's backend: CUDA for NCCL, CPU for gloo)."""
    if frames < 0 or chunk < 1:
        raise ValueError("frames must be >= 0 and chunk >= 1")
    rank, world = _world(group)
    header = {**header, "chunk": int(chunk)}  # chunk indices only mean something for one chunk size
    path = Path(out) if out is not None else None
    done = {}
    if path is not None and resume:
        done = _load_done(path, header)      # every rank reads the file: they skip the same chunks
    if path is not None and rank == 0 and (not resume or not path.exists() or not path.read_text().strip()):
        path.write_text(json.dumps({"header": header}) + "\n")
    if world > 1:
        dist.barrier(group)
    totals = {}
    nchunks = (frames + chunk - 1) // chunk
    for eb in ebn0s:
        tot = np.zeros(8, np.int64)
        for k in range(nchunks):
            key = (float(eb), k)
            if key in done:
                tot += done[key]
                continue
            cb, ce = k * chunk, min(frames, (k + 1) * chunk)
            b, e = shard_range(ce - cb, rank, world)
            c = torch.as_tensor(runner(float(eb), cb + b, e - b), dtype=torch.int64)
            if counts_device is not None:
                c = c.to(counts_device)
            allreduce_counts(c, group)
            c = c.cpu().numpy()
            tot += c
            if path is not None and rank == 0:
                with path.open("a") as fh:
                    fh.write(json.dumps({"ebn0_db": float(eb), "chunk": k, "frame_begin": cb, "frames": ce - cb,
                                         "counts": [int(x) for x in c]}) + "\n")
        n = max(int(tot[0]), 1)
        totals[float(eb)] = {"counts": dict(zip(COUNT_NAMES, (int(x) for x in tot))),
                             "fer": tot[2] / n, "cw_fer": tot[3] / n, "avg_iters": tot[4] / n}
    return totals


def main(argv=None):
    import inputs                                          # seeded BASELINE codes (input generator)
    from .cbp import Code

    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=float, required=True, help="frames per Eb/N0 point (all ranks)")
    ap.add_argument("--ebn0", default=None, help="comma list, default: the config's points")
    ap.add_argument("--chunk", type=float, default=1e6)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--stop-rule", type=int, default=0)
    ap.add_argument("--algorithm", type=int, default=0)
    ap.add_argument("--alpha", type=float, default=0.75)
    ap.add_argument("--llr-mode", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-resume", action="store_true")
    a = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = inputs.get_config(a.config)
    if inputs.is_peg(a.config):
        a.llr_mode |= 2                                    # PEG codes: all-zero codeword (CBP_TX_ZERO)
    base, Z = inputs.config_base(a.config)
    code = Code(base, Z, device=local)
    ebs = [float(x) for x in a.ebn0.split(",")] if a.ebn0 else list(cfg.ebn0_db)
    header = {"config": a.config, "N": code.N, "K": code.K, "seed": a.seed, "max_iter": cfg.max_iter,
              "stop_rule": a.stop_rule, "algorithm": a.algorithm, "alpha": a.alpha, "llr_mode": a.llr_mode}
    run = gpu_runner(code, cfg.max_iter, a.seed, a.stop_rule, a.algorithm, a.alpha, a.llr_mode)
    res = run_sweep(run, ebs, int(a.frames), int(a.chunk), header, a.out, not a.no_resume,
                    counts_device=torch.device("cuda", local))
    if int(os.environ.get("RANK", "0")) == 0:
        for eb, r in res.items():
            c = r["counts"]
            print(json.dumps({"ebn0_db": eb, **c, "ber": c["bit_errors"] / max(1, c["frames"] * code.K),
                              "fer": r["fer"], "avg_iters": r["avg_iters"]}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
