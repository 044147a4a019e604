#!/usr/bin/env python3
"""Summaries of ncu output for profiles/ (run here, on the pulled files).

    python tools/summarize_ncu.py full  gpurun_out/prof.ncu-rep  profiles/ncu_grid_kernel.json "<capture cmd>"
      (ALGO_BYTES=<bytes per launch>, default the C2 grid's 80 MB of f64 output)
    python tools/summarize_ncu.py launches gpurun_out/launches.csv profiles/launches_round1.csv
"""
import csv
import os
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
]


def num(v):
    return float(str(v).replace(",", ""))


def full(rep, out, capture):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))

    def get(k, scale_to=None):
        v = num(d[k])
        unit = u.get(k, "")
        if scale_to == "bytes":
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        if scale_to == "us":
            v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(unit, 1)
        return v

    stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: num(v) for h, v in d.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    rd, wr = get("dram__bytes_read.sum", "bytes"), get("dram__bytes_write.sum", "bytes")
    summary = {
        "capture": capture,
        "kernel": d.get("Kernel Name"),
        "duration_us": get("gpu__time_duration.sum", "us"),
        "dram_bytes_read": rd,
        "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": int(os.environ.get("ALGO_BYTES", 80000000)),
        "warp_instructions": num(d["smsp__inst_executed.sum"]),
        "issue_active_pct": num(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
        "warps_active_pct": num(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
        "registers_per_thread": num(d["launch__registers_per_thread"]),
    }
    for k in METRICS:
        if k.startswith("sm__inst_executed_pipe") and k in d:
            summary[k] = num(d[k])
    summary["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in
                            sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    with open(out, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1))


def launches(src, out):
    rows = [r for r in csv.reader(open(src)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[1:]:
        if len(r) != len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]]
        res.append((r[idx["ID"]], name.split("(")[0].replace("void ", "").replace("unnamed>::", ""),
                    r[idx["Grid Size"]], r[idx["Block Size"]], num(r[idx["Metric Value"]])))
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["id", "kernel", "grid", "block", "duration_ns"])
        for row in res:
            w.writerow(row)
    per = {}
    for _, k, _, _, t in res:
        per.setdefault(k, []).append(t)
    for k, v in per.items():
        print(f"{k[:60]:<60} n={len(v):3d} mean {sum(v)/len(v)/1e3:8.2f} us")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "")
    else:
        launches(sys.argv[2], sys.argv[3])
