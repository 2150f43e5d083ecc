#!/usr/bin/env python
"""DRAM traffic per visit of the FP and BP launches from ncu captures, for the
bench's roofline `traffic` field:

    python tools/traffic_from_ncu.py <tag> <fp.ncu-rep> <bp.ncu-rep> <visits_per_launch>

writes profiles/traffic_<tag>.json = {"fp": {...}, "bp": {...}} with
dram__bytes_read.sum + dram__bytes_write.sum per launch and per visit."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, r = rows[0], rows[1], rows[2]
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        tot += float(r[i]) * SCALE[u[i]]
    i = h.index("gpu__time_duration.sum")
    return tot, r[h.index("Kernel Name")][:60], float(r[i]), u[i]


def main():
    tag, fp, bp, visits = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    res = {"tag": tag, "visits_per_launch": visits}
    for k, rep in (("fp", fp), ("bp", bp)):
        b, name, dur, unit = dram(rep)
        res[k] = {"kernel": name, "dram_bytes_per_launch": b, "dram_bytes_per_visit": b / visits,
                  "algorithmic_bytes_per_visit": 4.0 if k == "fp" else 8.0,
                  "ncu_duration": f"{dur} {unit} (cold-cache, clock-control none)"}
    p = os.path.join(ROOT, "profiles", f"traffic_{tag}.json")
    json.dump(res, open(p, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
