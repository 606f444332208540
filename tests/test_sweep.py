"""Resumable multi-process sweeps (paper_2305_05286_b200/sweep.py; SURVEY B13 and
§5 checkpoint/resume).  The per-slice work is the CPU oracle's ber_sim here (the
product runs cbp_ber_sim); totals must not depend on chunking, world size or on an
interruption followed by a resume."""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle
from paper_2305_05286_b200.sweep import run_sweep

EBS = [1.5, 3.0]
HEADER = {"config": "C1", "seed": 9, "max_iter": 20}


def oracle_runner():
    base, Z = inputs.config_base("C1")
    o = oracle.OracleCode(base, Z)
    return lambda eb, begin, n: o.ber_sim(eb, 9, begin, n, 20) if n > 0 else np.zeros(8, np.int64)


def reference(frames):
    base, Z = inputs.config_base("C1")
    o = oracle.OracleCode(base, Z)
    return {eb: o.ber_sim(eb, 9, 0, frames, 20) for eb in EBS}


def as_array(res, eb):
    c = res[eb]["counts"]
    return np.array([c[k] for k in ("frames", "bit_errors", "frame_errors", "cw_frame_errors", "iter_sum",
                                     "edge_visits", "not_converged", "undetected_fires")])


def test_sweep_totals_independent_of_chunking(tmp_path):
    ref = reference(90)
    for chunk in (7, 30, 1000):
        res = run_sweep(oracle_runner(), EBS, 90, chunk, HEADER, tmp_path / f"c{chunk}.jsonl")
        for eb in EBS:
            assert (as_array(res, eb) == ref[eb]).all()
    lines = (tmp_path / "c7.jsonl").read_text().splitlines()
    assert json.loads(lines[0])["header"]["chunk"] == 7 and len(lines) == 1 + 2 * 13


def test_sweep_resume_after_interruption(tmp_path):
    out = tmp_path / "s.jsonl"
    run = oracle_runner()
    calls = {"n": 0}

    def flaky(eb, begin, n):
        calls["n"] += 1
        if calls["n"] == 5:
            raise RuntimeError("simulated crash")
        return run(eb, begin, n)

    with pytest.raises(RuntimeError):
        run_sweep(flaky, EBS, 60, 10, HEADER, out)
    assert len(out.read_text().splitlines()) == 1 + 4          # header + the 4 chunks finished before the crash
    seen = []
    res = run_sweep(lambda eb, b, n: (seen.append((eb, b)), run(eb, b, n))[1], EBS, 60, 10, HEADER, out)
    assert len(seen) == 2 * 6 - 4                               # only the missing chunks ran
    ref = reference(60)
    for eb in EBS:
        assert (as_array(res, eb) == ref[eb]).all()
    with pytest.raises(ValueError):                             # another sweep's checkpoint is refused
        run_sweep(run, EBS, 60, 10, {**HEADER, "seed": 10}, out)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, path, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = run_sweep(oracle_runner(), EBS, 45, 10, HEADER, path)
    out[rank] = {eb: as_array(res, eb).tolist() for eb in EBS}
    dist.destroy_process_group()


def test_sweep_gloo_world2_equals_single_process(tmp_path):
    path = str(tmp_path / "w2.jsonl")
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, _free_port(), path, out), nprocs=2, join=True)
        res = dict(out)
    ref = reference(45)
    for eb in EBS:
        assert res[0][eb] == res[1][eb] == list(map(int, ref[eb]))
    lines = open(path).read().splitlines()
    assert len(lines) == 1 + 2 * 5                              # rank 0 wrote each chunk once
