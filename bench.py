#!/usr/bin/env python
"""Benchmark of the CBP hot path (BASELINE.json metric) -- one JSON line on rank 0.

Headline workload = BASELINE configs[4] (C5, the metric's "per GPU and 8xB200" scaling
workload): the N=1944 rate-1/2 QC-LDPC code (C3a) at Eb/N0 = 2.5 dB, max_iter 30, fp32 LLR
stream; the int8 stream (q = sat(rint(4L), +-127)) is measured the same way and reported
beside it.  A step = this rank's slice of the C5 frame range through the two halves of cbp_ber_sim, per
chunk of 2^20 frames: cbp_channel (Philox info bits -> encoder -> BPSK/AWGN, L and the
codewords to an HBM buffer) -> cbp_ber_count (CBP decode -> error counting), followed by the
NCCL all-reduce of the 8 counters (codes off the one-frame-per-warp kernel, e.g. C1: one fused
cbp_ber_sim launch instead).  Step s of rank g simulates global frames
[(s W + g) F, (s W + g + 1) F) of the 10^9-frame C5 range (weak scaling, F per GPU fixed).

  python bench.py [--gpus N --steps K --warmup W]      (N>1: re-launches itself under torchrun)
  python bench.py --impl reference ...                 (CPU oracle on the host cores)
  python bench.py --config C2 ...                      (another BASELINE config as the step)
"""
from __future__ import annotations

import argparse
import json
import re
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CBP info Gbit/s and frames/s per GPU and 8×B200 at Eb/N0, % of roofline"
UNIT = "info Gbit/s"
I_EDGE = 38            # algorithmic fp32/int ops per edge visit of the arithmetic contract
BASELINE_INDEX = {"C1": 0, "C2": 1, "C3a": 2, "C3b": 2, "C4": 3, "C5": 4}
CHUNK = 1 << 20         # frames per cbp_channel -> cbp_ber_count pair (cbp_ber_sim's chunk)
DEFAULT_STEP_FRAMES = {"C5": 4_000_000, "C3a": 4_000_000, "C3b": 4_000_000, "C1": 20_000_000, "C2": 1_000_000,
                       "C4": 20_000}
CPU_FRAMES = {"C5": 1000, "C3a": 1000, "C3b": 600, "C1": 20000, "C2": 3000, "C4": 4}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cbp", choices=["cbp", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--frames", type=int, default=None, help="frames per Eb/N0 point per GPU and step")
    ap.add_argument("--ebn0", type=str, default=None, help="comma list (default: the config's points)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-int8", action="store_true", help="skip the int8-stream measurement")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-decode", action="store_true", help="skip the cbp_decode (HBM LLR input) roofline")
    ap.add_argument("--no-suite", action="store_true", help="skip the other-config measurements")
    ap.add_argument("--e2e-frames", type=int, default=400_000)
    ap.add_argument("--cpu-frames", type=int, default=None,
                    help="oracle frames per Eb/N0 point and core (cpu_baseline, reference arm)")
    ap.add_argument("--cpu-cores", type=int, default=0, help="oracle processes (default: all host cores)")
    return ap.parse_args()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args):
    """--gpus N: one process per GPU.  Without torchrun's environment the script re-executes
    itself under torch.distributed.run (127.0.0.1 rendezvous); under torchrun the world size
    must equal N."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
                   *sys.argv[1:]]
            os.execv(sys.executable, cmd)
        return
    if int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch with --nproc-per-node {args.gpus}")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        import statistics
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 4 + k and r[4 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def kernel_traffic(cfg_name: str):
    """DRAM bytes per frame of the dominant kernel from the latest committed `ncu --set full`
    capture of the same workload (profiles/r*_<config>_kernel_traffic.json, written by
    tools/profile_summary.py), or None."""
    def tag(f):   # r02s < r02ba < r02bo: round, then capture letters by length and order
        m = re.match(r"r(\d+)([a-z]*)_", f.name)
        return (int(m.group(1)), len(m.group(2)), m.group(2)) if m else (0, 0, "")

    caps = sorted((ROOT / "profiles").glob(f"r*_{cfg_name.lower()}_kernel_traffic.json"), key=tag)
    if not caps:
        return None
    d = json.loads(caps[-1].read_text())
    if not d.get("frames"):
        return None
    d["file"] = caps[-1].name
    d["bytes_per_frame"] = (d["dram_bytes_read"] + d["dram_bytes_write"]) / d["frames"]
    return d


def workload_label(cfg, ebn0s):
    mb, nb, Z = cfg.spec[0], cfg.spec[1], cfg.spec[2]
    idx = BASELINE_INDEX.get(cfg.name)
    tag = f"BASELINE configs[{idx}]" if idx is not None else "test code"
    what = {"C5": "C3a code, 10^9-frame scaling workload"}.get(cfg.name, "")
    return (f"{cfg.name} ({tag}{', ' + what if what else ''}): QC-LDPC N={nb * Z} K={(nb - mb) * Z} "
            f"rate {1 - mb / nb:.3f}, Z={Z}, cbp_ber_sim (cbp_channel + cbp_ber_count) at Eb/N0 {', '.join(f'{e:g}' for e in ebn0s)} dB")


def config_block(cfg, ebn0s, frames, args, n_gpus, llr="fp32"):
    return {"workload": workload_label(cfg, ebn0s),
            "ebn0_db": list(ebn0s), "frames_per_point_per_gpu_per_step": frames, "max_iter": cfg.max_iter,
            "stop_rule": "belief W=M + syndrome verify", "llr": llr,
            "seed": args.seed, "parallelism": f"dp{n_gpus} (frame-range shards, NCCL allreduce of counters)",
            "frame_range": "step s of rank g: global frames [(s*W+g)*F, (s*W+g+1)*F)",
            "step": "per point and per chunk of 2^20 frames: cbp_channel (L + codewords to an HBM buffer) -> "
                    "cbp_ber_count (decode + error count), the two halves cbp_ber_sim runs",
            "l2": "flushed (256 MiB write) before every step; a chunk's LLRs (8.2 GB) exceed L2"}


# ------------------------------------------------------------------ reference arm (CPU oracle)
def _oracle_slice(job):
    """worker: the unmodified single-threaded oracle on one frame range (one process per core)"""
    name, eb, seed, begin, n, max_iter, llr_mode = job
    import inputs
    import oracle
    base, Z = inputs.config_base(name)
    return oracle.OracleCode(base, Z).ber_sim(eb, seed, begin, n, max_iter, llr_mode=llr_mode)


def oracle_timed(name, ebn0s, seed, begin, frames, max_iter, llr_mode, cores):
    """Time the oracle over `frames` frames per Eb/N0 point, split into `cores` independent
    frame ranges run by `cores` processes (the oracle itself is untouched and single-threaded).
    Returns (counts int64[8], seconds)."""
    import multiprocessing as mpr
    import numpy as np
    jobs = []
    for eb in ebn0s:
        per = (frames + cores - 1) // cores
        for k in range(cores):
            b = begin + k * per
            n = max(0, min(per, begin + frames - b))
            if n:
                jobs.append((name, eb, seed, b, n, max_iter, llr_mode))
    ctx = mpr.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_oracle_slice, [(j[0], j[1], j[2], j[3], 1, j[5], j[6]) for j in jobs[:cores]])   # warm the workers
        t0 = time.perf_counter()
        res = pool.map(_oracle_slice, jobs, chunksize=1)
        dt = time.perf_counter() - t0
    return np.sum(res, axis=0), dt


def run_reference(args, cfg, ebn0s):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import inputs
    import oracle
    base, Z = inputs.config_base(cfg.name)
    o = oracle.OracleCode(base, Z)
    cores = args.cpu_cores or os.cpu_count() or 1
    frames = (args.cpu_frames or CPU_FRAMES.get(cfg.name, 100)) * cores
    for _ in range(args.warmup):
        o.ber_sim(ebn0s[0], args.seed, 0, 2, cfg.max_iter)
    times = []
    tot = np.zeros(8, np.int64)
    for s in range(args.steps):
        c, dt = oracle_timed(cfg.name, ebn0s, args.seed, s * frames, frames, cfg.max_iter, 0, cores)
        tot += c
        times.append(dt)
    T = sum(times)
    fps = tot[0] / T
    gbps = fps * o.K / 1e9
    sample = (f"{frames} frames x {len(ebn0s)} Eb/N0 point(s) per step ({cfg.name}, fp32 stream): the "
              f"single-threaded oracle in {cores} processes on disjoint frame ranges")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": gbps, "unit": UNIT, "frames_per_s": fps,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_block(cfg, ebn0s, frames, args, n_gpus=1),
        "cpu_baseline": {"value": gbps, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------------ product arm
def main():
    args = parse()
    self_launch(args)
    import inputs
    cfg = inputs.CONFIGS[args.config]
    ebn0s = [float(x) for x in args.ebn0.split(",")] if args.ebn0 else list(cfg.ebn0_db)
    if args.impl == "reference":
        return run_reference(args, cfg, ebn0s)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2305_05286_b200 as cbp
    from paper_2305_05286_b200 import pipeline
    from paper_2305_05286_b200.dist import allreduce_counts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # the NCCL process group exists at every N (a one-rank group when not under torchrun), so the
    # counter all-reduce of the multi-GPU path runs through NCCL in every bench run
    if "MASTER_ADDR" not in os.environ:
        os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(_free_port()), "RANK": "0",
                           "WORLD_SIZE": "1"})
    dist.init_process_group("nccl", device_id=dev)
    n_allreduce = [0]

    def reduce(c):
        n_allreduce[0] += 1
        return allreduce_counts(c)

    frames = args.frames or DEFAULT_STEP_FRAMES.get(cfg.name, cfg.frames)
    base, Z = inputs.config_base(cfg.name)
    code = cbp.Code(base, Z, device=local)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)   # 256 MiB > L2
    stream = torch.cuda.current_stream(dev)
    peaks = measured_peaks()

    def barrier():
        dist.barrier()

    # the split step needs the code on cbp_warp_kernel (cbp_ber_count); others run the fused cbp_ber_sim
    try:
        l_, c_ = code.channel(ebn0s[0], 1, 0, 2)
        code.ber_count(l_, c_, 1)
        split = True
    except cbp.CbpError:
        split = False
    chunk = min(frames, CHUNK) if split else frames
    llr_buf = torch.empty((chunk, (code.N + 3) // 4 * 4), dtype=torch.float32, device=dev) if split else None
    cw_buf = torch.empty((chunk, code.words), dtype=torch.int32, device=dev) if split else None
    n_chunks = (frames + chunk - 1) // chunk

    def measure(llr_mode):
        """W warm-up + K timed steps on this rank's slices; a step is, per Eb/N0 point and per chunk of
        2^20 frames, cbp_channel -> HBM -> cbp_ber_count (what cbp_ber_sim runs), each launch bracketed by
        CUDA events on the launch stream.  Returns (seconds max over ranks, summed counters [points, 8],
        decode ms per point and step, channel ms per point and step, local edge visits per point)."""
        counts = [torch.zeros(8, dtype=torch.int64, device=dev) for _ in ebn0s]
        local_ev = [torch.zeros(8, dtype=torch.int64, device=dev) for _ in ebn0s]

        def ev():
            return torch.cuda.Event(enable_timing=True)

        def step(s, launch_ms=None):
            for p, eb in enumerate(ebn0s):
                c = counts[p]
                c.zero_()
                f_begin = (s * world + rank) * frames
                for f0 in range(0, frames, chunk):
                    n = min(chunk, frames - f0)
                    marks = [ev() for _ in range(3)] if launch_ms is not None else None
                    if marks:
                        marks[0].record(stream)
                    if split:
                        code.channel(eb, args.seed, f_begin + f0, n, llr_mode, stream=stream,
                                     out=(llr_buf[:n], cw_buf[:n]))
                    if marks:
                        marks[1].record(stream)
                    if split:
                        code.ber_count(llr_buf[:n], cw_buf[:n], cfg.max_iter, counts=c, stream=stream)
                    else:
                        code.ber_sim(eb, args.seed, f_begin + f0, n, cfg.max_iter, llr_mode=llr_mode, counts=c,
                                     stream=stream)
                    if marks:
                        marks[2].record(stream)
                        launch_ms.append((p, marks))
                if launch_ms is not None:
                    local_ev[p].copy_(c)
                reduce(c)

        for w in range(args.warmup):
            step(10_000 + w)                                   # warm-up frames outside the timed range
        torch.cuda.synchronize()
        launches, step_ev = [], []
        with ClockSampler(local) as clk:
            barrier()
            torch.cuda.synchronize()
            for s in range(args.steps):
                flush.fill_(1.0)                               # L2 flush outside the step events
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record(stream)
                step(s, launches)
                s1.record(stream)
                step_ev.append((s0, s1))
            torch.cuda.synchronize()
            barrier()
        t_ms = sum(a.elapsed_time(b) for a, b in step_ev)
        t_max = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dec = np.array([m[1].elapsed_time(m[2]) for _, m in launches]).reshape(args.steps, len(ebn0s), n_chunks)
        chn = np.array([m[0].elapsed_time(m[1]) for _, m in launches]).reshape(args.steps, len(ebn0s), n_chunks)
        tot = torch.stack(counts).cpu().numpy()                # last step, all ranks summed
        ev_loc = torch.stack(local_ev).cpu().numpy()[:, 5]     # last step, this rank's edge visits per point
        return t_max.item() / 1e3, tot, dec.sum(axis=2), chn.sum(axis=2), ev_loc, clk.summary()

    T, tot, per_launch, per_chan, ev_loc, clocks = measure(0)
    frames_all = frames * len(ebn0s) * args.steps * world
    fps = frames_all / T
    gbps = fps * code.K / 1e9

    # roofline of the dominant kernel (the cbp_ber_count decode launches, cbp_warp_kernel in MODE_BER_LLR):
    # I_edge x exact edge visits / the launches' CUDA-event durations, against the derived issue peak
    # (DESIGN.md §7); the channel launches' share of the step is reported beside it
    li = code.launch_info()
    f_sm = peaks.get("sm_max_mhz", 1965.0)
    peak = li["num_sms"] * 128 * f_sm * 1e6
    dur = per_launch.mean(axis=0) / 1e3                        # decode seconds per point and step
    achieved = float((ev_loc.astype(np.float64) * I_EDGE).sum() / dur.sum())
    step_s = T / args.steps
    tr = kernel_traffic(cfg.name)
    roofline = {"bound": "alu", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Top/s",
                "frac": achieved / peak,
                "traffic": tr["bytes_per_frame"] * chunk if tr else None,
                "kernel": ("cbp_warp_kernel (cbp_ber_count: decode + error count of a 2^20-frame chunk)" if split else
                           "fused cbp_ber_sim launch"),
                "launches_per_step": n_chunks * len(ebn0s),
                "edge_visits_per_launch": int(ev_loc.sum() / (n_chunks * len(ebn0s))),
                "launch_ms": float(dur.sum() * 1e3 / (n_chunks * len(ebn0s))),
                "edge_visits_per_s": float(ev_loc.sum() / dur.sum()),
                "share_of_step": float(dur.sum() * world / step_s) if world == 1 else None,
                "channel_ms_per_step": float(per_chan.mean(axis=0).sum()),
                "step_frac": float((ev_loc.astype(np.float64) * I_EDGE).sum() / step_s / peak) if world == 1 else None,
                "note": f"I_edge={I_EDGE} contract ops/edge visit x exact edge visits / mean launch time (CUDA events "
                        f"on the launch stream); peak = {li['num_sms']} SM x 128 lanes x {f_sm:.0f} MHz (sm_max, "
                        f"MEASURED_PEAKS.json; derived issue peak); step_frac = the same ops over the whole step "
                        f"(channel launches included); traffic = DRAM bytes per launch scaled from the per-frame "
                        f"bytes of {tr['file'] if tr else 'n/a'} (ncu --set full of this workload); algorithmic HBM "
                        f"bytes of a decode launch: {code.N * 4 + code.words * 4} in per frame (LLRs + codeword), "
                        f"64 out"}
    if tr:
        roofline["ncu"] = {k: tr.get(k) for k in ("issue_active_pct", "lane_slots_per_edge_visit", "smem_pipe_pct",
                                                  "tex_pipe_pct", "alu_pipe_pct", "fma_pipe_pct", "file")}

    int8 = None
    if not args.no_int8:
        T8, tot8, pl8, _, ev8, clk8 = measure(1)
        f8 = frames * len(ebn0s) * args.steps * world / T8
        d8 = pl8.mean(axis=0) / 1e3
        int8 = {"value": f8 * code.K / 1e9, "unit": UNIT, "frames_per_s": f8, "ms_per_step": 1e3 * T8 / args.steps,
                "roofline_frac": float((ev8.astype(np.float64) * I_EDGE).sum() / d8.sum() / peak),
                "ber": float(tot8[:, 1].sum() / max(1, tot8[:, 0].sum() * code.K)),
                "fer": float(tot8[:, 2].sum() / max(1, tot8[:, 0].sum())),
                "avg_iters": float(tot8[:, 4].sum() / max(1, tot8[:, 0].sum())), "clocks": clk8,
                "what": "the same steps with the int8 LLR stream (q = sat(rint(4L), +-127), L = q/4)"}

    # cbp_decode roofline: LLRs resident in HBM (read once per frame) against the ALU term
    decode_rl = None
    if not args.no_decode:
        Fd = min(frames, 2_000_000)
        ld = (code.N + 3) // 4 * 4
        llr = torch.empty((Fd, ld), dtype=torch.float32, device=dev)
        for b in range(0, Fd, 1 << 18):
            n = min(1 << 18, Fd - b)
            l_, _ = code.channel(ebn0s[0], args.seed + 2, rank * Fd + b, n, want_cw=False)
            llr[b:b + n].copy_(l_)
        out = code.alloc_outputs(Fd, ev=True)
        code.decode(llr[:1024], cfg.max_iter, out={k: v[:1024] for k, v in out.items()}, stream=stream)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            flush.fill_(1.0)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            code.decode(llr, cfg.max_iter, out=out, stream=stream)
            a1.record(stream)
            torch.cuda.synchronize()
            ts.append(a0.elapsed_time(a1) / 1e3)
        td = float(np.median(ts))
        evd = float(out["ev"].sum().item())
        llr_bytes = Fd * ld * 4
        out_bytes = Fd * (code.words * 4 + 5)
        t_hbm = (llr_bytes + out_bytes) / (peaks.get("hbm_gbs", 6556.2) * 1e9)
        t_alu = evd * I_EDGE / peak
        decode_rl = {"bound": "alu" if t_alu >= t_hbm else "hbm", "frames": Fd, "ms": td * 1e3,
                     "frames_per_s": Fd / td, "info_gbps": Fd * code.K / td / 1e9,
                     "achieved": evd * I_EDGE / td / 1e12, "peak": peak / 1e12, "unit": "Top/s",
                     "frac": max(t_alu, t_hbm) / td, "hbm_term_ms": t_hbm * 1e3, "alu_term_ms": t_alu * 1e3,
                     "llr_bytes": llr_bytes, "achieved_hbm_gbs": (llr_bytes + out_bytes) / td / 1e9,
                     "hbm_peak_gbs": peaks.get("hbm_gbs", 6556.2),
                     "what": f"cbp_decode of {Fd} device-resident fp32 C5 frames (ld={ld}); roofline time = max(LLR + "
                             f"output bytes / HBM peak, I_edge x edge visits / issue peak); frac = roofline time / "
                             f"median measured time (3 launches, L2 flushed)"}
        del llr, out

    # end-to-end: host LLRs -> cbp_decode -> host outputs (pinned host buffers, copies timed)
    e2e = None
    if not args.no_e2e:
        Fe = args.e2e_frames
        ld = (code.N + 3) // 4 * 4
        host = torch.empty((Fe, ld), dtype=torch.float32, pin_memory=True)
        hout = pipeline.alloc_host_outputs(code, Fe)
        for b in range(0, Fe, 1 << 17):
            n = min(1 << 17, Fe - b)
            llr_, _ = code.channel(ebn0s[0], args.seed + 1, rank * Fe + b, n, want_cw=False)
            host[b:b + n].copy_(llr_)
        torch.cuda.synchronize()
        pipeline.decode_host(code, host, cfg.max_iter, out=hout)         # warm-up
        reps = max(1, min(args.steps, 3))
        barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            pipeline.decode_host(code, host, cfg.max_iter, out=hout)
        te = time.perf_counter() - t0
        tmax = torch.tensor([te], dtype=torch.float64, device=dev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        te = tmax.item()
        e2e = {"value": reps * Fe * world * code.K / te / 1e9, "unit": UNIT,
               "frames_per_s": reps * Fe * world / te,
               "h2d_bytes_per_step": Fe * ld * 4 * world, "d2h_bytes_per_step": Fe * (code.words * 4 + 5) * world,
               "what": f"{pipeline.API_NAME} on {Fe} host-resident fp32 frames/GPU of the same workload (pinned host "
                       f"LLRs; H2D + decode + D2H of bits/iters/flags inside the timed region; host wall clock, "
                       f"max over ranks; {reps} reps)"}
        # the same through cbp_decode_host_i8 with the int8 stream of the workload (a quarter of the H2D bytes:
        # the fp32 e2e is bound by the pinned host-to-device copy, 7.8 KB per frame)
        ld8 = (code.N + 15) // 16 * 16
        host8 = torch.empty((Fe, ld8), dtype=torch.int8, pin_memory=True)
        for b in range(0, Fe, 1 << 17):
            n = min(1 << 17, Fe - b)
            llr_, _ = code.channel(ebn0s[0], args.seed + 1, rank * Fe + b, n, llr_mode=1, want_cw=False)
            q = torch.zeros((n, ld8), dtype=torch.int8, device=dev)
            q[:, :code.N] = (llr_[:, :code.N] * 4.0).round().to(torch.int8)   # exact: the stream's L = q / 4
            host8[b:b + n].copy_(q)
        torch.cuda.synchronize()
        code.decode_host(host8, cfg.max_iter, out=hout, scale=0.25)
        barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            code.decode_host(host8, cfg.max_iter, out=hout, scale=0.25)
        te8 = time.perf_counter() - t0
        tmax = torch.tensor([te8], dtype=torch.float64, device=dev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        te8 = tmax.item()
        e2e["int8_stream"] = {"value": reps * Fe * world * code.K / te8 / 1e9, "unit": UNIT,
                              "frames_per_s": reps * Fe * world / te8,
                              "h2d_bytes_per_step": Fe * ld8 * world, "d2h_bytes_per_step": Fe * (code.words * 4 + 5) * world,
                              "what": "cbp_decode_host_i8 on the int8 stream of the same frames (q = sat(rint(4L), "
                                      "+-127), scale 0.25), same timing"}
        del host8

    # the other BASELINE configs and variants, one timed cbp_ber_sim call each (after a warm-up call)
    others = {}
    if not args.no_suite:
        suite = [("C2", 1.0, 500_000, 0, 0, 0), ("C2", 2.0, 500_000, 0, 0, 0), ("C2", 3.0, 500_000, 0, 0, 0),
                 ("C1", 2.0, 2_000_000, 0, 0, 0), ("C3a", 1.5, 300_000, 0, 0, 0),
                 ("C3b", 4.0, 300_000, 0, 0, 0), ("C4", 1.5, 3_000, 2, 0, 0),
                 ("C2", 2.0, 500_000, 1, 0, 0), ("C2", 2.0, 500_000, 2, 0, 0), ("C2", 2.0, 500_000, 0, 0, 1),
                 ("C2", 2.0, 500_000, 2, 0, 2), ("C2", 2.0, 500_000, 2, 0, 3),
                 ("P2048", 2.0, 300_000, 0, 2, 0), ("P8192", 1.5, 30_000, 0, 2, 0)]
        for name, eb, nf, rule, lm, alg in suite:
            ocfg = inputs.get_config(name)
            ob, oz = inputs.config_base(name)
            oc = cbp.Code(ob, oz, device=local)
            c = torch.zeros(8, dtype=torch.int64, device=dev)
            # warm-up launch of the full size: a split cbp_ber_sim takes its HBM chunk (L + codewords of nf frames)
            # from the library's retained pool, whose first growth (2.4 GB for the N = 1944 codes) is a one-time cost
            # and not the decoder's (timed inside the launch it cost C3a 28-52 ms of 71)
            oc.ber_sim(eb, args.seed, 0, nf, ocfg.max_iter, rule, lm, counts=c, stream=stream, algorithm=alg)
            c.zero_()
            barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            oc.ber_sim(eb, args.seed, rank * nf, nf, ocfg.max_iter, rule, lm, counts=c, stream=stream,
                       algorithm=alg)
            a1.record(stream)
            reduce(c)
            torch.cuda.synchronize()
            ms = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device=dev)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            t = c.cpu().numpy()
            key = f"{name}@{eb}dB" + ("/int8" if lm & 1 else "") + ("/zero-cw" if lm & 2 else "") + \
                ["", "/min-sum", "/LBP", "/FBP"][alg] + \
                ("" if rule == 0 or name == "C4" else ["", "/W=N", "/syndrome", "/none"][rule])
            others[key] = {
                "N": oc.N, "K": oc.K, "frames": int(t[0]), "ms": ms.item(),
                "frames_per_s": t[0] / ms.item() * 1e3, "info_gbps": t[0] * oc.K / ms.item() / 1e6,
                "edge_visits_per_s": t[5] / ms.item() * 1e3,
                "alu_frac": t[5] / world * I_EDGE / (ms.item() / 1e3) / peak,
                "ber": t[1] / max(1, t[0] * oc.K),
                "fer": t[2] / max(1, t[0]), "avg_iters": t[4] / max(1, t[0]),
                "stop_rule": ["belief W=M", "belief W=N", "syndrome", "none"][rule],
                "algorithm": ["CBP log-tanh", "CBP normalized min-sum (alpha 0.75)", "layered BP (comparison)",
                              "flooding BP (comparison)"][alg],
                "note": "fixed 25 sweeps: FER ~1, the weak C4 code never converges" if name == "C4" else "",
                "launch": oc.launch_info()}

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            import oracle
            o = oracle.OracleCode(base, Z)
            nfc = args.cpu_frames or CPU_FRAMES.get(cfg.name, 100)
            t0 = time.perf_counter()
            c1 = np.zeros(8, np.int64)
            for eb in ebn0s:
                c1 += o.ber_sim(eb, args.seed, 0, max(1, nfc // 4), cfg.max_iter)
            t1 = time.perf_counter() - t0
            cores = args.cpu_cores or os.cpu_count() or 1
            cN, tN = oracle_timed(cfg.name, ebn0s, args.seed, 0, nfc * cores, cfg.max_iter, 0, cores)
            cpu = {"value": cN[0] * o.K / tN / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"{nfc * cores} frames x {len(ebn0s)} Eb/N0 point(s) of the same workload (fp32 "
                             f"stream): the single-threaded C++ oracle in {cores} processes on disjoint frame "
                             f"ranges, {tN:.1f} s", "frames_per_s": cN[0] / tN,
                   "single_core": {"value": c1[0] * o.K / t1 / 1e9, "frames_per_s": c1[0] / t1,
                                   "sample": f"{max(1, nfc // 4)} frames x {len(ebn0s)} point(s), {t1:.1f} s"}}
        except Exception as ex:   # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        results = {}
        for p, eb in enumerate(ebn0s):
            t = tot[p]
            results[str(eb)] = {"frames": int(t[0]), "ber": t[1] / max(1, t[0] * code.K), "fer": t[2] / max(1, t[0]),
                                "avg_iters": t[4] / max(1, t[0]), "edge_visits": int(t[5]),
                                "not_converged": int(t[6]), "undetected_fires": int(t[7])}
        line = {
            "metric": METRIC, "value": gbps, "unit": UNIT, "frames_per_s": fps, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_block(cfg, ebn0s, frames, args, world),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "int8_stream": int8, "roofline_decode": decode_rl,
            "gpu_launches": args.steps * len(ebn0s) * n_chunks * (2 if split else 1),
            "collectives": {"backend": dist.get_backend(), "world_size": world,
                            "counter_allreduce_calls": n_allreduce[0],
                            "per_timed_step": len(ebn0s)},
            "launch": li, "results_last_step": results, "other_configs": others,
        }
        print(json.dumps(line))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
