"""Summarise one `ncu --set full` capture of cbp_kernel into profiles/.

python tools/profile_summary.py gpurun_out/prof_a0_p1.ncu-rep <edge_visits> <prefix> "<what was captured>" [frames]

writes profiles/<prefix>_ncu_full_summary.txt (SOL / scheduler / pipe metrics,
SASS opcode mix, stall reasons) and profiles/<prefix>_kernel_traffic.json (the
numbers bench.py reports beside its roofline: DRAM bytes per launch, shared-memory
and texture data-pipe utilisation, issue utilisation, instructions per edge visit).
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep, ev, prefix, what = sys.argv[1], float(sys.argv[2]), sys.argv[3], sys.argv[4]
frames = int(float(sys.argv[5])) if len(sys.argv) > 5 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
R = dict(zip(raw[0], raw[2]))
U = dict(zip(raw[0], raw[1]))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}   # ncu's decimal byte units


def f(k):
    try:
        x = float(R[k].replace(",", ""))
    except (KeyError, ValueError):
        return None
    return x * SCALE.get(U.get(k, ""), 1.0)


M = {
    "duration_ms": f("gpu__time_duration.sum"),
    "sm_clock_ghz": f("smsp__cycles_elapsed.avg.per_second"),
    "dram_bytes_read": f("dram__bytes_read.sum"),
    "dram_bytes_write": f("dram__bytes_write.sum"),
    "inst_executed": f("smsp__inst_executed.sum"),
    "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_per_sm": f("sm__warps_active.avg.per_cycle_active"),
    "smem_pipe_pct": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "smem_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "tex_pipe_pct": f("l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    "alu_pipe_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "fma_pipe_pct": f("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": f("launch__registers_per_thread"),
    "edge_visits": ev,
    "frames": frames,
}
M["lane_slots_per_edge_visit"] = M["inst_executed"] * 32 / ev if M["inst_executed"] else None
stalls = {}
for k, v in R.items():
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            x = float(v)
        except ValueError:
            continue
        if x >= 0.05:
            stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(x, 3)

rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = rows[1]
iS, iE = h.index("Source"), h.index("Instructions Executed")
ops = collections.Counter()
tot = 0
for r in rows[2:]:
    try:
        e = int(r[iE] or 0)
    except ValueError:
        continue
    toks = r[iS].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    ops[op.split(".")[0]] += e
    tot += e

out = ROOT / "profiles"
out.mkdir(exist_ok=True)
lines = [f"# {what}", f"# source: {rep} (ncu --set full --clock-control none --import-source on)"]
for k, v in M.items():
    lines.append(f"{k:28s} {v:.6g}" if isinstance(v, float) else f"{k:28s} {v}")
lines.append("stalls (warps per issue): " + "  ".join(f"{k}:{v}" for k, v in sorted(stalls.items(), key=lambda t: -t[1])))
lines.append("opcode mix: " + "  ".join(f"{k}:{v / tot * 100:.1f}%" for k, v in ops.most_common(20)))
(out / f"{prefix}_ncu_full_summary.txt").write_text("\n".join(lines) + "\n")
M.update({"kernel": what, "source": f"ncu --set full --clock-control none ({rep})", "stalls_per_issue": stalls})
(out / f"{prefix}_kernel_traffic.json").write_text(json.dumps(M, indent=1) + "\n")
print("\n".join(lines))
