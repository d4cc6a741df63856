#!/usr/bin/env python
"""Summarise an ncu --set full report of the fused step kernel into
profiles/: key metrics (JSON + markdown) and the per-launch DRAM traffic
that bench.py reports as roofline.traffic.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_fused c2
  python tools/ncu_summary.py gpurun_out/seg.ncu-rep profiles/r02_ncu_dither_seg -   (other kernels: no traffic entry)
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sass__inst_executed_local_loads",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}
    stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v[0])
              for h, v in d.items() if h.startswith("smsp__average_warps_issue_stalled_") and
              h.endswith("_per_issue_active.ratio") and v[0] not in ("", "0")}
    return d, stalls


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val) * scale


def main():
    rep, prefix, cfg = sys.argv[1], sys.argv[2], (sys.argv[3] if len(sys.argv) > 3 else "c2")
    d, stalls = raw(rep)
    kern = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    names = [r[4] for r in csv.reader(io.StringIO(kern)) if len(r) > 4 and r[0] != "ID"]
    name = next((n for n in names if "k_fused" in n), names[0] if names else "")
    summary = {k: {"value": d[k][0], "unit": d[k][1]} for k in KEYS if k in d}
    traffic = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
    summary["traffic_bytes_per_launch"] = traffic
    summary["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    summary["kernel"] = name
    with open(prefix + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu --set full: {name}\n\n| metric | value | unit |\n|---|---|---|\n")
        for k in KEYS:
            if k in d:
                f.write(f"| {k} | {d[k][0]} | {d[k][1]} |\n")
        f.write(f"| traffic (read+write) per launch | {traffic:.0f} | byte |\n\n## stall reasons (warps per issue)\n\n")
        for k, v in summary["stalls_per_issue"].items():
            f.write(f"- {k}: {v:.3f}\n")
    if cfg == "-":
        print(json.dumps({"traffic": traffic, "time": d["gpu__time_duration.sum"]}))
        return
    tpath = os.path.join(os.path.dirname(prefix) or ".", "ncu_traffic.json")
    t = {}
    if os.path.exists(tpath):
        t = json.load(open(tpath))
    t[cfg] = traffic
    json.dump(t, open(tpath, "w"), indent=1)
    print(json.dumps({"traffic": traffic, "time": d["gpu__time_duration.sum"]}))


if __name__ == "__main__":
    main()
