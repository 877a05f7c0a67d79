"""Summarise the profiling of one batched search (tools/batch_prof.py under
ncu --profile-from-start off) into profiles/ (tracked).

usage: python tools/batch_report.py ROUND gpurun_out/search_metrics.csv \
           gpurun_out/bscan_full.ncu-rep

  ROUND_launches.txt  per-kernel device time and DRAM bytes of one search
                      (cold-cache, serialised: ncu's replay), with shares
  ROUND_scan_ncu.txt  key --set full metrics of the dominant kernel
  ncu_scan.json       DRAM bytes per search, launches per search and the
                      dominant kernel's time share (read by bench.py)
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rnd, mcsv, full = sys.argv[1], sys.argv[2], sys.argv[3]

rows = [r for r in csv.reader(open(mcsv)) if len(r) > 5]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[1:]:
    key = (r[ii], r[ki].split("(")[0].strip())
    per.setdefault(key, {})[r[mi]] = float(r[vi].replace(",", ""))
agg = collections.OrderedDict()
for (_, name), m in per.items():
    a = agg.setdefault(name, [0.0, 0.0, 0])
    a[0] += m.get("gpu__time_duration.sum", 0.0)
    a[1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a[2] += 1
tt = sum(a[0] for a in agg.values())
tb = sum(a[1] for a in agg.values())
dom = max(agg.items(), key=lambda kv: kv[1][0])
lines = [f"One batched search (bench workload), ncu launch list: {len(per)} launches, "
         f"{tt / 1e3:.1f} us device time (serialised, cold caches), {tb / 1e6:.1f} MB DRAM",
         f"{'time_us':>9} {'share':>6} {'dram_MB':>8} {'n':>3}  kernel"]
for name, (t, b, n) in agg.items():
    lines.append(f"{t / 1e3:9.1f} {100 * t / tt:5.1f}% {b / 1e6:8.1f} {n:3d}  {name}")
(ROOT / "profiles" / f"{rnd}_launches.txt").write_text("\n".join(lines) + "\n")
print("\n".join(lines))

raw = subprocess.run(["ncu", "-i", full, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
H, U, R = rr[0], rr[1], rr[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
out = [f"{n:60s} {R[H.index(n)]} {U[H.index(n)]}" for n in want if n in H]
st = [(H[i], R[i]) for i in range(len(H)) if H[i].startswith("smsp__pcsamp_warps_issue_stalled_")
      and not H[i].endswith("not_issued")]
tot = sum(float(v or 0) for _, v in st) or 1
out.append("stall reasons (pc sampling): " + ", ".join(
    f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(v) / tot:.0f}%"
    for n, v in sorted(st, key=lambda x: -float(x[1] or 0))[:6]))
(ROOT / "profiles" / f"{rnd}_scan_ncu.txt").write_text("\n".join(out) + "\n")
print("\n".join(out))
json.dump({"workload": "ivf-ads N=1000000 D=128 nlist=1024 nprobe=32 nq=1000 K=10 eps0=2.1",
           "pipeline": "batched pdx_search (pdx_batch.cu)",
           "dram_bytes_per_search": tb, "launches_per_search": len(per),
           "dominant_kernel": dom[0], "dominant_time_share": dom[1][0] / tt,
           "ncu_search_us": tt / 1e3,
           "source": f"profiles/{rnd}_launches.txt, profiles/{rnd}_scan_ncu.txt"},
          open(ROOT / "profiles" / "ncu_scan.json", "w"), indent=1)
