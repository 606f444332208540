"""Summarise an ncu report: key SOL / scheduler metrics and the SASS opcode mix.

python tools/ncu_summary.py gpurun_out/prof.ncu-rep [edge_visits]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ev = float(sys.argv[2]) if len(sys.argv) > 2 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


KEYS = ("Duration", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "DRAM Throughput", "Avg. Active Threads Per Warp", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Executed Instructions", "Dynamic Shared Memory Per Block", "Block Size",
        "Grid Size", "No Eligible")
rows = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
hdr = rows[0]
iN, iU, iV = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
seen = set()
for r in rows[1:]:
    if len(r) > iV and r[iN] in KEYS and r[iN] not in seen:
        seen.add(r[iN])
        print(f"{r[iN]:32s} {r[iV]:>16s} {r[iU]}")
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
print(f"warp instructions {tot:.4e}" + (f"   per edge-visit (x32 lanes) {tot * 32 / ev:.1f}" if ev else ""))
print("  ".join(f"{k}:{v / tot * 100:.1f}%" for k, v in ops.most_common(18)))

# warp-state (stall) sampling summary
rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
if len(rows) > 2:
    h, v = rows[0], rows[2]
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
            try:
                st.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot_s = sum(x for x, _ in st) or 1.0
    print("stalls: " + "  ".join(f"{n}:{x / tot_s * 100:.1f}%" for x, n in sorted(st, reverse=True)[:9]))
