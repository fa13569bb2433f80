"""Summarise an `ncu --page source --csv --print-source cuda,sass` export by source line.

usage: python profiles/ncu_lines.py export.csv [top_n]
Prints the lines with the most warp-stall samples and executed instructions.
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur, hdr, agg = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] not in ("", "Function Name"):
        try:
            samples = int(r[4]) if r[4] not in ("", "-") else 0
            inst = int(r[7]) if r[7] not in ("", "-") else 0
        except (ValueError, IndexError):
            continue
        agg.append((samples, inst, cur, r[0], r[1].strip()[:90]))
tot_s = sum(a[0] for a in agg) or 1
tot_i = sum(a[1] for a in agg) or 1
print(f"total samples {tot_s}, warp-instructions {tot_i}")
for s, i, f, ln, src in sorted(agg, key=lambda a: (a[0], a[1]), reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {f}:{ln}  {src}")
