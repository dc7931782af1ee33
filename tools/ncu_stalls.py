"""Warp-stall summary of one kernel from an ncu report (source page, SASS view).

    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_stalls.py src.csv [--top 25]

Prints the share of stall samples per SASS opcode (with its top stall reasons) and the
individual instructions with the most samples — e.g. spill reloads (LDL) feeding loop control
show up as long_sb on the instruction after the LDL.
"""
import argparse
import collections
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--top", type=int, default=25)
args = ap.parse_args()
rows = list(csv.reader(open(args.csv)))
h = rows[1]
data = [r for r in rows[2:] if len(r) >= len(h)]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
lines = []
for r in data:
    src = r[ix["Source"]].strip()
    parts = src.split()
    op = (parts[1] if parts and parts[0].startswith("@") and len(parts) > 1 else (parts[0] if parts else "")).split(".")[0]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = {k[6:]: int(r[ix[k]] or 0) for k in stalls}
    lines.append((s, r[0][-6:], src[:72], st))
    for k, v in st.items():
        byop[op][k] += v
    tot[op] += s
T = sum(tot.values())
print(f"{rows[0][1] if len(rows[0]) > 1 else ''}\ntotal stall samples {T}\n")
print("per opcode: share of samples, top reasons (% of all samples)")
for op, c in tot.most_common(12):
    top = ", ".join(f"{k}:{v / T * 100:.1f}" for k, v in byop[op].most_common(4) if v)
    print(f"  {op:10s} {c / T * 100:5.1f}%  {top}")
print(f"\ntop {args.top} instructions")
for s, a, src, st in sorted(lines, key=lambda x: -x[0])[: args.top]:
    top = ", ".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
    print(f"  {s:7d} {s / T * 100:5.1f}% {a} {src:72s} {top}")
