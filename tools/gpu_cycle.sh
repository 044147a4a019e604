#!/bin/bash
# Build here, then on a B200: GPU tests, bench, one ncu --set full capture of
# the grid kernel.  Usage: tools/gpu_cycle.sh <tag> [extra remote command]
set -e
cd "$(dirname "$0")/.."
TAG=${1:-run}
python -m paper_2603_00549_b200._build
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1500 -- "timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=\$? >> gpurun_out/pytest_gpu.log; timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; timeout 600 ncu --set full --clock-control none --import-source on -k regex:grid_ -s 2 -c 1 -o gpurun_out/prof_$TAG python tools/profile_grid.py 5 > gpurun_out/ncu_full.log 2>&1; ${2:-true}" 2>&1 | tail -1
tail -2 gpurun_out/pytest_gpu.log
python - "$TAG" <<'PY'
import csv, json, subprocess, sys
tag = sys.argv[1]
try:
    d = json.load(open("gpurun_out/bench.json"))
    print("value G/s %.1f  ms/step %.4f  kernel_ms %.4f  frac %.3f  e2e G/s %.2f" % (
        d["value"] / 1e9, d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"],
        d["e2e"]["value"] / 1e9))
except Exception as exc:
    print("bench failed:", exc)
out = subprocess.run(["ncu", "-i", f"gpurun_out/prof_{tag}.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
if len(rows) > 2:
    d = dict(zip(rows[0], rows[2]))
    for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_write.sum"):
        print(k, d.get(k))
    st = [(float(v.replace(",", "")), h[33:]) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    tot = sum(f for f, _ in st)
    print("stalls:", ", ".join(f"{h} {100*f/tot:.0f}%" for f, h in sorted(st, reverse=True)[:6]))
PY
