"""Write tests/golden/oracle_counts_<config>.json: the CPU ORACLE's ber_sim counters over
EVERY frame of a BASELINE workload (e.g. C2: 10^6 frames at each of 1.0..3.0 dB, seed 1,
max_iter 30, belief stop) -- the all-frames parity reference of SURVEY §8(d) for the
fused GPU path (tests/test_gpu_parity.py::test_ber_sim_all_frames_equal_oracle_counts).

Calls only oracle/ (test infrastructure), never the CUDA path.  The unmodified
single-threaded oracle runs in one process per core on disjoint frame ranges; the
counters are integer sums, so the result does not depend on the split.

python tools/write_oracle_counts.py C2 1000000 [cores] [points]
python tools/write_oracle_counts.py C3a 1e7 16 2.5          (one Eb/N0 point of BASELINE configs[2])
"""
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import inputs  # noqa: E402


def work(job):
    name, eb, seed, begin, n, mi = job
    import oracle
    base, Z = inputs.config_base(name)
    return eb, oracle.OracleCode(base, Z).ber_sim(eb, seed, begin, n, mi)


if __name__ == "__main__":
    name, frames = sys.argv[1], int(float(sys.argv[2]))
    cores = int(sys.argv[3]) if len(sys.argv) > 3 else os.cpu_count()
    cfg = inputs.CONFIGS[name]
    points = tuple(float(x) for x in sys.argv[4].split(",")) if len(sys.argv) > 4 else cfg.ebn0_db
    seed, piece = 1, 5000
    jobs = [(name, eb, seed, b, min(piece, frames - b), cfg.max_iter)
            for eb in points for b in range(0, frames, piece)]
    t0 = time.time()
    tot = {eb: np.zeros(8, np.int64) for eb in points}
    with mp.get_context("fork").Pool(cores) as pool:
        for eb, c in pool.imap_unordered(work, jobs, chunksize=1):
            tot[eb] += c
    out = {"config": name, "frames_per_point": frames, "seed": seed, "max_iter": cfg.max_iter,
           "stop_rule": "belief W=M (0)", "llr_mode": 0, "algorithm": "CBP log-tanh (0)",
           "written_by": "tools/write_oracle_counts.py (oracle only)", "cpu_seconds_wall": round(time.time() - t0, 1),
           "counts": {str(eb): [int(x) for x in tot[eb]] for eb in points}}
    path = ROOT / "tests" / "golden" / f"oracle_counts_{name}.json"
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(path, out["cpu_seconds_wall"], "s")
