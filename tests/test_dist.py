"""Multi-process (gloo, world size 2) test of the frame-range sharding and the
counter all-reduce of paper_2305_05286_b200/dist.py (row a9).  The per-shard
work is the CPU oracle here; on GPUs it is cbp_ber_sim (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_05286_b200.dist import allreduce_counts, ber_sim_sharded, shard_range


def test_shard_range_partition():
    for frames in (0, 1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_range(frames, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == frames
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, frames, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import inputs
    import oracle
    base, Z = inputs.config_base("C1")
    o = oracle.OracleCode(base, Z)

    def run_shard(begin, count, counts):
        c = o.ber_sim(2.0, 3, begin, count, 20)
        counts += torch.from_numpy(c)

    counts = torch.zeros(8, dtype=torch.int64)
    ber_sim_sharded(run_shard, frames, 100, counts)
    out[rank] = counts.numpy().tolist()
    # a second all-reduce leaves every rank with the same numbers
    t = torch.tensor([rank + 1], dtype=torch.int64)
    allreduce_counts(t)
    assert int(t.item()) == world * (world + 1) // 2
    dist.destroy_process_group()


def test_gloo_world2_sharded_counts_equal_single_process():
    frames = 300
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, _free_port(), frames, out), nprocs=2, join=True)
        res = [out[0], out[1]]
    assert res[0] == res[1]
    import inputs
    import oracle
    base, Z = inputs.config_base("C1")
    single = oracle.OracleCode(base, Z).ber_sim(2.0, 3, 100, frames, 20)
    assert res[0] == list(map(int, single))
    assert np.array(res[0])[0] == frames
