"""Markdown table (FER / average iterations per decoder and Eb/N0) from the JSON lines of
tools/compare_schedules.py.

python tools/curves_table.py profiles/r01h_curves_P2048.jsonl
"""
import json
import sys


def main(path):
    rows = [json.loads(ln) for ln in open(path) if ln.strip().startswith("{")]
    decs = []
    for r in rows:
        if r["decoder"] not in decs:
            decs.append(r["decoder"])
    ebs = sorted({r["ebn0_db"] for r in rows})
    print(f"{rows[0]['config']}, {rows[0]['frames']} frames per point, max_iter {rows[0]['max_iter']}: FER / average iterations\n")
    print("| Eb/N0 | " + " | ".join(decs) + " |")
    print("|---|" + "---|" * len(decs))
    for eb in ebs:
        cells = []
        for d in decs:
            r = next(x for x in rows if x["decoder"] == d and x["ebn0_db"] == eb)
            fer = r["fer"]
            cells.append(f"{fer:.3g} / {r['avg_iters']:.2f}" if fer else f"0 / {r['avg_iters']:.2f}")
        print(f"| {eb} dB | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
