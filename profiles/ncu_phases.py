"""Group an ncu cuda,sass source export into named line ranges of one file.

usage: python profiles/ncu_phases.py export.csv file.cu name:lo-hi [name:lo-hi ...]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
target = sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    name, r = spec.split(":")
    lo, hi = (int(v) for v in r.split("-"))
    ranges.append((name, lo, hi))
cur, agg = None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    try:
        ln, smp, inst = int(r[0]), int(r[4]), int(r[7])
    except (ValueError, IndexError):
        continue
    key = "other:" + str(cur)
    if cur == target:
        key = "unassigned"
        for name, lo, hi in ranges:
            if lo <= ln <= hi:
                key = name
                break
    a = agg.setdefault(key, [0, 0])
    a[0] += smp
    a[1] += inst
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:28s} samples {100*v[0]/ts:5.1f}%  inst {100*v[1]/ti:5.1f}%  ({v[1]/1e6:.0f}M warp-inst)")
