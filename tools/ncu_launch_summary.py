"""Per-kernel share of an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file x.csv`).

    python tools/ncu_launch_summary.py x.csv "<what was run>" > summary.txt

ncu serialises the launches and runs them cold, so the absolute times are not bench times; the
shares are what the roofline's `k3_share_of_step` is checked against.
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[h + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    unit = r[unit_i] if unit_i is not None else "ns"
    ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
    tot[r[ki]] += ms
    cnt[r[ki]] += 1
T = sum(tot.values())
print(f"ncu --metrics gpu__time_duration.sum --clock-control none of {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}")
print("kernel | launches | total ms | share")
for k, v in tot.most_common():
    print(f"{k[:160]} | {cnt[k]} | {v:.1f} | {v / T * 100:.2f} %")
