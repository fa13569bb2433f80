"""Summaries of the round's ncu captures for profiles/ (run here, no GPU needed).

usage: python profiles/summarize_ncu.py <launches.csv> [<full.ncu-rep> <patches_per_launch> <config>]
Writes the per-kernel share of a step from the launch list and, for a full
capture, DRAM bytes / duration / throughput per launch plus traffic_config<N>.json.
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

HERE = Path(__file__).resolve().parent


# one-off setup kernels (slide rendering, pyramid, thumbnail, mask, polygon index, RRC tables):
# excluded so the shares are those of the timed step
SETUP = ("synth_level0", "box_downsample", "box32_warp", "mask_kernel", "morph_kernel", "rrc_table_kernel",
         "poly_index", "thumbnail", "field_kernel", "raster_mark", "raster_classify")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(float)
    n = defaultdict(int)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"].split("(")[0].replace("void ", "")
                if any(t in k for t in SETUP):
                    continue
                v = float(d["Metric Value"].replace(",", ""))
                scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1e-3)
                per[k] += v * scale
                n[k] += 1
    tot = sum(per.values())
    out = []
    for k, v in sorted(per.items(), key=lambda kv: -kv[1]):
        out.append({"kernel": k, "launches": n[k], "total_us": round(v, 1), "share": round(v / tot, 4)})
    return out


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    unit_of = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
             "second": 1e9}
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))

        def f(key):
            try:
                return float(d[key].replace(",", "")) * scale.get(unit_of.get(key, ""), 1)
            except (KeyError, ValueError):
                return None

        rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
        dur = f("gpu__time_duration.sum")
        res.append({"kernel": d.get("Kernel Name", "")[:80], "grid": d.get("Grid Size"), "block": d.get("Block Size"),
                    "duration_ns": dur, "dram_read_bytes": rd, "dram_write_bytes": wr,
                    "dram_gbs": round((rd + wr) / dur, 1) if rd is not None and dur else None,
                    "regs": f("launch__registers_per_thread"),
                    "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                    "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                    "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
                    "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active")})
    return res


if __name__ == "__main__":
    print(json.dumps({"launch_shares": launches(sys.argv[1])}, indent=1))
    if len(sys.argv) > 2:
        kern = full(sys.argv[2])
        print(json.dumps({"full": kern}, indent=1))
        n = int(sys.argv[3])
        total = sum((k["dram_read_bytes"] or 0) + (k["dram_write_bytes"] or 0) for k in kern)
        (HERE / f"traffic_config{sys.argv[4]}.json").write_text(json.dumps(
            {"dram_bytes_per_patch": round(total / n, 1), "launches": len(kern), "source": Path(sys.argv[2]).name,
             "note": "dram__bytes_read.sum + dram__bytes_write.sum over the captured launches / patches"}, indent=1))
