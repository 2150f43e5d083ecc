#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) and a launch list (.csv) into
profiles/ncu_summary_<tag>.json + a short markdown table.

    python tools/ncu_summary.py <tag> gpurun_out/prof_<tag>.ncu-rep gpurun_out/launches_<tag>.csv
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "lts__t_sectors_op_red.sum": "l2_red_sectors",
    "lts__t_sectors_op_atom.sum": "l2_atom_sectors",
    "l1tex__t_bytes.sum": "l1_bytes",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
}
STALLS = "smsp__average_warp_latency_issue_stalled_"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    unit = dict(zip(hdr, units))
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3, "s": 1.0,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    res = []
    for r in data:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "")[:80]}
        for m, name in KEYS.items():
            if m in d and d[m] not in ("", "n/a"):
                try:
                    v = float(d[m].replace(",", ""))
                except ValueError:
                    continue
                u = unit.get(m, "")
                if u in scale:   # seconds / bytes in SI base units
                    v *= scale[u]
                    name = name.replace("_ns", "_s")
                k[name] = v
        stalls = {}
        for m, v in d.items():
            if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio"):
                try:
                    stalls[m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
                except ValueError:
                    pass
        k["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        res.append(k)
    return res


def launches(path):
    per = {}
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][-60:]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        if unit in ("usecond", "us"):
            v *= 1e3
        elif unit in ("msecond", "ms"):
            v *= 1e6
        e = per.setdefault(name, [0, 0.0])
        e[0] += 1
        e[1] += v
    tot = sum(v[1] for v in per.values())
    return {k: {"launches": n, "total_ms": t / 1e6, "share": t / tot} for k, (n, t) in
            sorted(per.items(), key=lambda kv: -kv[1][1])}


def main():
    tag, rep = sys.argv[1], sys.argv[2]
    lst = sys.argv[3] if len(sys.argv) > 3 else None
    out = {"tag": tag, "kernels": raw(rep) if os.path.exists(rep) else []}
    if lst and os.path.exists(lst):
        out["launch_list"] = launches(lst)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    p = os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.json")
    json.dump(out, open(p, "w"), indent=1)
    print(json.dumps(out, indent=1)[:6000])


if __name__ == "__main__":
    main()
