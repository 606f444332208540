#!/usr/bin/env python
"""Benchmark of the CBP hot path (BASELINE.json metric) -- one JSON line on rank 0.

A step = one fused cbp_ber_sim launch (Philox info bits -> encoder -> BPSK/AWGN
-> CBP decode -> error counting) per Eb/N0 point of BASELINE configs[1]
(C2: N=648 rate-1/2 QC-LDPC, Eb/N0 1.0..3.0 dB, 1e6 frames per point per GPU,
max_iter 30) followed by the NCCL all-reduce of the 8 counters per point.

  python bench.py [--gpus N --steps K --warmup W]          (N>1: under torchrun)
  python bench.py --impl reference ...                     (CPU oracle on the host cores)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CBP info Gbit/s and frames/s per GPU and 8×B200 at Eb/N0, % of roofline"
UNIT = "info Gbit/s"
I_EDGE = 38            # algorithmic fp32/int ops per edge visit of the arithmetic contract v2
B_EDGE = 60            # algorithmic on-chip bytes per edge visit: QP r/w 8+8, S_cj 4, R_ci 4, R_cj 4, 2 phi rows 2x16


def kernel_traffic():
    """DRAM bytes per launch and pipe utilisation of the dominant kernel from the
    latest committed ncu capture (profiles/*_kernel_traffic.json, tools/profile_summary.py)."""
    caps = sorted((ROOT / "profiles").glob("r*_kernel_traffic.json"))
    if not caps:
        return None, None
    d = json.loads(caps[-1].read_text())
    d["file"] = caps[-1].name
    return d["dram_bytes_read"] + d["dram_bytes_write"], d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cbp", choices=["cbp", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=None, help="frames per Eb/N0 point per GPU (default: BASELINE)")
    ap.add_argument("--ebn0", type=str, default=None, help="comma list (default: the config's points)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--llr-mode", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-suite", action="store_true", help="skip the other-config measurements")
    ap.add_argument("--e2e-frames", type=int, default=200_000)
    ap.add_argument("--cpu-frames", type=int, default=400,
                    help="oracle frames per Eb/N0 point and core (cpu_baseline, reference arm)")
    ap.add_argument("--cpu-cores", type=int, default=0, help="oracle processes (default: all host cores)")
    return ap.parse_args()


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
        pool.map(_oracle_slice, jobs[:cores])              # warm the workers (library load)
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
    frames = args.cpu_frames * cores
    for _ in range(args.warmup):
        o.ber_sim(ebn0s[0], args.seed, 0, 8, cfg.max_iter)
    times = []
    tot = np.zeros(8, np.int64)
    for s in range(args.steps):
        c, dt = oracle_timed(cfg.name, ebn0s, args.seed, s * frames, frames, cfg.max_iter, args.llr_mode, cores)
        tot += c
        times.append(dt)
    T = sum(times)
    fps = tot[0] / T
    gbps = fps * o.K / 1e9
    sample = (f"{frames} frames x {len(ebn0s)} Eb/N0 points per step ({cfg.name}): the single-threaded oracle in "
              f"{cores} processes on disjoint frame ranges")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": gbps, "unit": UNIT, "frames_per_s": fps,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_block(cfg, ebn0s, frames, args, n_gpus=1),
        "cpu_baseline": {"value": gbps, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def config_block(cfg, ebn0s, frames, args, n_gpus):
    return {"workload": f"{cfg.name}: QC-LDPC N={cfg.spec[1] * cfg.spec[2]} rate {1 - cfg.spec[0] / cfg.spec[1]:.3f} "
                        f"(BASELINE configs[1]) fused cbp_ber_sim, {len(ebn0s)} Eb/N0 points",
            "ebn0_db": list(ebn0s), "frames_per_point_per_gpu": frames, "max_iter": cfg.max_iter,
            "stop_rule": "belief W=M + syndrome verify", "llr": "int8" if args.llr_mode else "fp32",
            "seed": args.seed, "parallelism": f"dp{n_gpus} (frame-range shards, NCCL allreduce of counters)",
            "l2": "flushed (256 MiB write) before every step; ber_sim reads no input from HBM"}


# ------------------------------------------------------------------ product arm
def main():
    args = parse()
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
    # under torchrun the NCCL process group is set up even for one rank, so the counter
    # all-reduce and the max-over-ranks timing run through NCCL at every N
    distributed = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    frames = args.frames or cfg.frames
    base, Z = inputs.config_base(cfg.name)
    code = cbp.Code(base, Z, device=local)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)   # 256 MiB > L2
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if distributed:
            dist.barrier()

    def step(counts_per_point, launch_ms=None):
        for p, eb in enumerate(ebn0s):
            c = counts_per_point[p]
            c.zero_()
            if launch_ms is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            # this rank's frame range of the global workload (weak scaling: frames per GPU fixed)
            code.ber_sim(eb, args.seed, rank * frames, frames, cfg.max_iter, llr_mode=args.llr_mode, counts=c,
                         stream=stream)
            if launch_ms is not None:
                e1.record(stream)
                launch_ms.append((p, e0, e1))
            allreduce_counts(c)

    counts = [torch.zeros(8, dtype=torch.int64, device=dev) for _ in ebn0s]
    for _ in range(args.warmup):
        step(counts)
    torch.cuda.synchronize()

    launches = []
    step_ms = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1.0)                                   # L2 flush outside the step events
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step(counts, launches)
            s1.record(stream)
            step_ms.append((s0, s1))
        torch.cuda.synchronize()
        barrier()
    t_ms = sum(a.elapsed_time(b) for a, b in step_ms)
    t_max = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    T = t_max.item() / 1e3
    tot = torch.stack(counts).cpu().numpy()                   # counts of the last step, all ranks summed
    frames_all = int(tot[:, 0].sum()) * args.steps
    fps = frames_all / T
    gbps = fps * code.K / 1e9

    # roofline of the dominant kernel (the fused cbp_kernel launch, one per Eb/N0 point)
    per_launch_ms = [a.elapsed_time(b) for _, a, b in launches]
    ev_local = []
    for p in range(len(ebn0s)):
        ev_local.append(int(tot[p, 5]) // max(world, 1))       # edge visits per launch (this rank's share)
    dur = np.array(per_launch_ms).reshape(args.steps, len(ebn0s)).mean(axis=0) / 1e3
    ops = np.array(ev_local, dtype=np.float64) * I_EDGE
    traffic, traffic_src = kernel_traffic()
    achieved = float(ops.sum() / dur.sum())                    # ops/s averaged over the launches of a step
    li = code.launch_info()
    clocks = clk.summary()
    f_sm = measured_peaks().get("sm_max_mhz", 1965.0)
    peak = li["num_sms"] * 128 * f_sm * 1e6
    roofline = {"bound": "alu", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Top/s",
                "frac": achieved / peak, "traffic": traffic,
                "note": f"I_edge={I_EDGE} contract ops/edge-visit x exact edge visits / mean launch time; peak = "
                        f"{li['num_sms']} SM x 128 lanes x {f_sm:.0f} MHz (sm_max, MEASURED_PEAKS.json, derived "
                        f"issue peak); traffic = DRAM bytes/launch from "
                        f"{traffic_src.get('file', 'n/a') if traffic_src else 'n/a'} (algorithmic HBM bytes of "
                        f"ber_sim: 0 in, 64 out)"}
    # the resources that actually bind: the on-chip data pipes and the issue slots,
    # measured by ncu on the same kernel (C2, 2 dB, 1e5 frames) and committed under profiles/
    on_chip = float(np.array(ev_local, dtype=np.float64).sum() * B_EDGE / dur.sum())
    onchip_peak = li["num_sms"] * 128 * f_sm * 1e6
    roofline_onchip = {"bound": "smem+tex data pipes", "achieved": on_chip / 1e12, "peak": onchip_peak / 1e12,
                       "unit": "TB/s", "frac": on_chip / onchip_peak,
                       "note": f"B_edge={B_EDGE} algorithmic on-chip bytes/edge-visit (no bank conflicts) x edge "
                               f"visits / mean launch time; peak = 128 B/clk/SM x {li['num_sms']} SM x {f_sm:.0f} MHz "
                               f"(one shared-memory wavefront per clock)"}
    if traffic_src:
        roofline_onchip["ncu_pipe_utilisation_pct"] = {k: traffic_src.get(k) for k in (
            "smem_pipe_pct", "tex_pipe_pct", "issue_active_pct", "alu_pipe_pct", "fma_pipe_pct")}
        roofline_onchip["ncu_lane_slots_per_edge_visit"] = traffic_src.get("lane_slots_per_edge_visit")
        roofline_onchip["ncu_source"] = traffic_src.get("file")

    # end-to-end over the same Eb/N0 points: host LLRs -> cbp_decode (pipelined H2D / decode / D2H)
    # -> host outputs.  Per point the pinned host buffer is filled (untimed), then decode_host is
    # timed on the host clock (copies in both directions inside); the step time is the sum.
    e2e = None
    if not args.no_e2e:
        Fe = args.e2e_frames
        ld = (code.N + 3) // 4 * 4
        host = torch.empty((Fe, ld), dtype=torch.float32, pin_memory=True)
        hout = pipeline.alloc_host_outputs(code, Fe)
        te = 0.0
        reps = max(1, min(args.steps, 3))
        for eb in ebn0s:
            for b in range(0, Fe, 1 << 17):
                n = min(1 << 17, Fe - b)
                llr, _ = code.channel(eb, args.seed + 1, rank * Fe + b, n, want_cw=False)
                host[b:b + n].copy_(llr)
            torch.cuda.synchronize()
            pipeline.decode_host(code, host, cfg.max_iter, out=hout)     # warm-up of this point
            barrier()
            t0 = time.perf_counter()
            for _ in range(reps):
                pipeline.decode_host(code, host, cfg.max_iter, out=hout)
            te += time.perf_counter() - t0
        tmax = torch.tensor([te], dtype=torch.float64, device=dev)
        if distributed:
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        te = tmax.item()
        e2e = {"value": reps * len(ebn0s) * Fe * world * code.K / te / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": len(ebn0s) * Fe * ld * 4 * world,
               "d2h_bytes_per_step": len(ebn0s) * Fe * (code.words * 4 + 5) * world,
               "what": f"cbp_decode via pipeline.decode_host on {Fe} host-resident frames/GPU at each of the "
                       f"{len(ebn0s)} Eb/N0 points (pinned host LLRs, H2D + decode + D2H of bits/iters/flags "
                       f"timed, host wall clock, max over ranks)"}

    # the other BASELINE configs, one timed fused launch each (after a warm-up launch):
    # C1 @ 2 dB; C3a / C3b (rates 1/2, 5/6); C4 (global-state path, syndrome stop);
    # C5 = C3a @ 2.5 dB with the fp32 and the int8 LLR stream
    others = {}
    if not args.no_suite:
        # (config, Eb/N0, frames, stop rule, llr mode, algorithm): the other BASELINE configs, the C2 stop-rule
        # variants (W=N, syndrome per sweep), normalized min-sum CBP (NEXT-1) and the paper's comparison
        # schedules LBP / FBP (NEXT-3) on the same frames
        suite = [("C1", 2.0, 1_000_000, 0, 0, 0), ("C3a", 2.5, 300_000, 0, 0, 0), ("C5", 2.5, 300_000, 0, 1, 0),
                 ("C3b", 4.0, 300_000, 0, 0, 0), ("C4", 1.5, 3_000, 2, 0, 0), ("C2", 2.0, 1_000_000, 1, 0, 0),
                 ("C2", 2.0, 1_000_000, 2, 0, 0), ("C2", 2.0, 1_000_000, 0, 0, 1),
                 ("C2", 2.0, 1_000_000, 2, 0, 2), ("C2", 2.0, 1_000_000, 2, 0, 3),
                 # the paper's own code families (QC-PEG; all-zero codeword, max 200 iterations)
                 ("P2048", 2.0, 300_000, 0, 2, 0), ("P8192", 1.5, 30_000, 0, 2, 0)]
        for name, eb, nf, rule, lm, alg in suite:
            ocfg = inputs.get_config(name)
            ob, oz = inputs.config_base(name)
            oc = cbp.Code(ob, oz, device=local)
            c = torch.zeros(8, dtype=torch.int64, device=dev)
            oc.ber_sim(eb, args.seed, 0, min(nf, 20_000), ocfg.max_iter, rule, lm, counts=c, stream=stream,
                       algorithm=alg)
            c.zero_()
            barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            oc.ber_sim(eb, args.seed, rank * nf, nf, ocfg.max_iter, rule, lm, counts=c, stream=stream,
                       algorithm=alg)
            a1.record(stream)
            allreduce_counts(c)
            torch.cuda.synchronize()
            ms = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device=dev)
            if distributed:
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            t = c.cpu().numpy()
            key = f"{name}@{eb}dB" + ("/int8" if lm & 1 else "") + ("/zero-cw" if lm & 2 else "") + ["", "/min-sum", "/LBP", "/FBP"][alg] + \
                ("" if rule == 0 or name == "C4" else ["", "/W=N", "/syndrome", "/none"][rule])
            others[key] = {
                "N": oc.N, "K": oc.K, "frames": int(t[0]), "ms": ms.item(),
                "frames_per_s": t[0] / ms.item() * 1e3, "info_gbps": t[0] * oc.K / ms.item() / 1e6,
                "edge_visits_per_s": t[5] / ms.item() * 1e3, "ber": t[1] / max(1, t[0] * oc.K),
                "fer": t[2] / max(1, t[0]), "avg_iters": t[4] / max(1, t[0]),
                "stop_rule": ["belief W=M", "belief W=N", "syndrome", "none"][rule],
                "algorithm": ["CBP log-tanh", "CBP normalized min-sum (alpha 0.75)", "layered BP (comparison)",
                              "flooding BP (comparison)"][alg],
                "launch": oc.launch_info()}

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            import oracle
            o = oracle.OracleCode(base, Z)
            t0 = time.perf_counter()
            c1 = np.zeros(8, np.int64)
            for p, eb in enumerate(ebn0s):
                c1 += o.ber_sim(eb, args.seed, 0, args.cpu_frames, cfg.max_iter, llr_mode=args.llr_mode)
            t1 = time.perf_counter() - t0
            cores = args.cpu_cores or os.cpu_count() or 1
            cN, tN = oracle_timed(cfg.name, ebn0s, args.seed, 0, args.cpu_frames * cores, cfg.max_iter,
                                  args.llr_mode, cores)
            cpu = {"value": cN[0] * o.K / tN / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"{args.cpu_frames * cores} frames x {len(ebn0s)} Eb/N0 points of the same workload: "
                             f"the single-threaded C++ oracle in {cores} processes on disjoint frame ranges, "
                             f"{tN:.1f} s", "frames_per_s": cN[0] / tN,
                   "single_core": {"value": c1[0] * o.K / t1 / 1e9, "frames_per_s": c1[0] / t1,
                                   "sample": f"{args.cpu_frames} frames x {len(ebn0s)} points, {t1:.1f} s"}}
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
            "roofline": roofline, "roofline_onchip": roofline_onchip, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": args.steps * len(ebn0s), "launch": li, "results": results,
            "other_configs": others,
        }
        print(json.dumps(line))
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
