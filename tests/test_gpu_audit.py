"""Parity audit at the BASELINE sizes (SURVEY.md §8(d) "Parity coverage" for C3-C5):
the whole frame range of each point is decoded on the GPU (channel -> cbp_decode, the
same kernel and launch geometry as the fused bench path), every frame the GPU reports
as an error (any codeword bit wrong), not converged or with a failed stop verification
is collected, and those frames -- up to a cap per point, in frame order -- plus a seeded
uniform sample are decoded again by the oracle on all host cores and compared frame by
frame (bits, iterations, flags, edge visits).  Coverage is written to a JSON report.

Long (minutes on a B200 plus 16 host cores), so it runs only when asked:
    CBP_AUDIT=1 CBP_AUDIT_OUT=profiles/r01e_parity_audit.json python -m pytest tests/test_gpu_audit.py -m gpu
CBP_AUDIT_SCALE (default 1.0) scales the frame ranges, samples and caps for a quick run.
"""
import json
import multiprocessing as mp
import os
import time
from pathlib import Path

import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

cbp = pytest.importorskip("paper_2305_05286_b200")

SCALE = float(os.environ.get("CBP_AUDIT_SCALE", "1.0"))
SAMPLE, CAP = int(100_000 * SCALE), int(20_000 * SCALE)
# (config, Eb/N0 points, frames per point, llr_mode): BASELINE configs[2] (C3a, C3b: 10^7 frames at
# 7 points) and configs[4] (C5: 10^9 frames at 2.5 dB, fp32 and int8 streams)
AUDITS = [("C3a", (1.5, 2.0, 2.5, 3.0, 3.5, 4.0, 4.5), 10_000_000, 0),
          ("C3b", (1.5, 2.0, 2.5, 3.0, 3.5, 4.0, 4.5), 10_000_000, 0),
          ("C5", (2.5,), 1_000_000_000, 0),
          ("C5", (2.5,), 1_000_000_000, 1)]
_REPORT = {}
_CODES = {}


def _oracle_frames(job):
    """Worker: oracle channel + decode of single frames (test infrastructure only)."""
    name, eb, seed, llr_mode, mi, frames = job
    if name not in _CODES:
        base, Z = inputs.config_base(name)
        _CODES[name] = oracle.OracleCode(base, Z)
    o = _CODES[name]
    out = []
    for f in frames:
        llr, _ = o.channel(eb, seed, int(f), 1, llr_mode=llr_mode)
        d = o.decode(llr, mi)
        out.append((int(f), d["bits"][0].copy(), int(d["iters"][0]), int(d["flags"][0]), int(d["edge_visits"][0])))
    return out


def _gpu_pass(g, eb, seed, frames, mi, llr_mode, sample_set, chunk=1 << 20, cap=None):
    """Decode every frame on the GPU; return per-frame outputs of the flagged frames (up to `cap`,
    default CAP, in frame order) and of the sample, and the total flagged count."""
    cap = CAP if cap is None else cap
    keep, n_flag, words = {}, 0, g.words
    sample = torch.as_tensor(sorted(sample_set), dtype=torch.int64)
    for b in range(0, frames, chunk):
        n = min(chunk, frames - b)
        llr, cw = g.channel(eb, seed, b, n, llr_mode=llr_mode)
        out = g.decode(llr, mi, ev=True)
        del llr
        wrong = ((out["bits"] ^ cw) != 0).any(1)
        fl = out["flags"].to(torch.int32)
        flagged = wrong | ((fl & 1) == 0) | ((fl & 4) != 0)
        idx = torch.nonzero(flagged).flatten()
        n_flag += int(idx.numel())
        room = cap - sum(1 for v in keep.values() if v[4])
        idx = idx[:max(room, 0)]
        s = sample[(sample >= b) & (sample < b + n)].to(idx.device) - b
        for sel, is_flag in ((idx, True), (s, False)):
            if sel.numel() == 0:
                continue
            bits = out["bits"][sel].cpu().numpy().view(np.uint32)[:, :words]
            it, f, ev = out["iters"][sel].cpu().numpy(), out["flags"][sel].cpu().numpy(), out["ev"][sel].cpu().numpy()
            for k, fi in enumerate(sel.cpu().numpy().tolist()):
                old = keep.get(b + fi)
                keep[b + fi] = (bits[k].copy(), int(it[k]), int(f[k]), int(ev[k]), is_flag or (old is not None and old[4]))
    return keep, n_flag


@pytest.mark.skipif(not os.environ.get("CBP_AUDIT"), reason="long audit: set CBP_AUDIT=1")
@pytest.mark.parametrize("name,ebs,frames,llr_mode", AUDITS, ids=[f"{a[0]}-llr{a[3]}" for a in AUDITS])
def test_parity_audit(name, ebs, frames, llr_mode):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    frames = int(frames * SCALE)
    base, Z = inputs.config_base(name)
    g = cbp.Code(base, Z)
    mi = inputs.get_config(name).max_iter
    seed = 1
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(2024)
    points = []
    with mp.get_context("fork").Pool(cores) as pool:
        for eb in ebs:
            t0 = time.time()
            sample = set(rng.integers(0, frames, SAMPLE).tolist())
            keep, n_flag = _gpu_pass(g, eb, seed, frames, mi, llr_mode, sample)
            t1 = time.time()
            order = sorted(keep)
            jobs = [(name, eb, seed, llr_mode, mi, order[k:k + 64]) for k in range(0, len(order), 64)]
            bad = []
            for res in pool.imap_unordered(_oracle_frames, jobs, chunksize=1):
                for f, bits, it, fl, ev in res:
                    gb, gi, gf, gev, _ = keep[f]
                    if not ((gb == bits).all() and gi == it and gf == fl and gev == ev):
                        bad.append(f)
            n_fchk = sum(1 for v in keep.values() if v[4])
            points.append({"ebn0_db": eb, "frames": frames, "flagged_by_gpu": n_flag,
                           "flagged_checked": n_fchk, "flagged_coverage": n_fchk / max(n_flag, 1),
                           "uniform_sample": len(sample), "frames_checked": len(keep), "mismatches": len(bad),
                           "first_mismatches": sorted(bad)[:10], "gpu_pass_s": round(t1 - t0, 1),
                           "oracle_s": round(time.time() - t1, 1)})
            assert not bad, points[-1]
    key = f"{name}/{'int8' if llr_mode else 'fp32'}"
    _REPORT[key] = {"N": g.N, "K": g.K, "max_iter": mi, "seed": seed, "llr_mode": llr_mode, "host_cores": cores,
                    "cap_flagged_per_point": CAP, "sample_per_point": SAMPLE, "points": points}
    out = os.environ.get("CBP_AUDIT_OUT")
    if out:
        Path(out).write_text(json.dumps({"what": __doc__.split("\n\n")[0], "audits": _REPORT}, indent=1) + "\n")


@pytest.mark.parametrize("llr_mode", [0, 1], ids=["fp32", "int8"])
def test_parity_audit_bench_slice(llr_mode):
    """Frame-by-frame parity on the bench's own workload, run by default (the full audit above
    needs CBP_AUDIT): the first bench step of C5 (BASELINE configs[4]: global frames [0, 4e6) at
    2.5 dB) is decoded on the GPU; every flagged frame (error, not converged or failed
    verification; all of them up to 5000) and 3000 uniform samples are decoded again by the
    oracle and compared bit for bit (bits, iterations, flags, edge visits)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base, Z = inputs.config_base("C5")
    g = cbp.Code(base, Z)
    mi, frames = 30, 4_000_000
    rng = np.random.default_rng(7 + llr_mode)
    sample = set(rng.integers(0, frames, 3000).tolist())
    keep, n_flag = _gpu_pass(g, 2.5, 1, frames, mi, llr_mode, sample, cap=5000)
    assert n_flag <= 5000, n_flag                              # every flagged frame is checked
    order = sorted(keep)
    jobs = [("C5", 2.5, 1, llr_mode, mi, order[k:k + 32]) for k in range(0, len(order), 32)]
    bad = []
    with mp.get_context("fork").Pool(os.cpu_count() or 1) as pool:
        for res in pool.imap_unordered(_oracle_frames, jobs, chunksize=1):
            for f, bits, it, fl, ev in res:
                gb, gi, gf, gev, _ = keep[f]
                if not ((gb == bits).all() and gi == it and gf == fl and gev == ev):
                    bad.append(f)
    assert not bad, sorted(bad)[:10]
    assert len(keep) >= 3000
