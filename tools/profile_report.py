"""Summarise a profiling run into profiles/ (tracked).

usage: python tools/profile_report.py ROUND gpurun_out/prof_scan.ncu-rep \
           gpurun_out/launches.csv gpurun_out/plain.log

Writes
  profiles/<round>_scan_ncu.txt     key ncu --set full metrics of pdx_scan_kernel
  profiles/<round>_launches.txt     per-kernel device time from the ncu launch list
  profiles/ncu_scan.json            dram bytes per scan launch + the scan kernel's
                                    share of a search step (read by bench.py)
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
STEP_KERNELS = ("pdx_scan_kernel", "build_visits_kernel", "centroid_dist_kernel",
                "select_kernel", "select_radix_kernel", "project_kernel", "bound_factors_kernel")


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def main():
    rnd, rep, launches, plain = sys.argv[1:5]
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    rows, units = raw_metrics(rep)
    r = rows[0]
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]
    lines = [f"{k:62s} {r.get(k, '')} {units.get(k, '')}" for k in keys]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = sum(float(r[k]) * scale.get(units[k], 1) for k in ("dram__bytes_read.sum",
                                                             "dram__bytes_write.sum"))
    # launch list: mean device time per kernel name
    times = collections.defaultdict(list)
    with open(launches) as f:
        text = f.read()
    body = text[text.find('"ID"'):] if '"ID"' in text else text
    for row in csv.DictReader(io.StringIO(body)):
        if row.get("Metric Name") == "gpu__time_duration.sum":
            name = row["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
            v = float(row["Metric Value"].replace(",", ""))
            unit = row.get("Metric Unit", "ns")
            times[name].append(v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1,
                                    "ms": 1, "nsecond": 1e-6}.get(unit, 1e-6))
    step = {k: sum(v) / len(v) for k, v in times.items() if k in STEP_KERNELS}
    share = step.get("pdx_scan_kernel", 0) / max(sum(step.values()), 1e-12)
    ll = [f"{k:28s} n={len(v):5d} mean={sum(v) / len(v):9.4f} ms" for k, v in
          sorted(times.items(), key=lambda kv: -sum(kv[1]))]
    ll.append(f"scan kernel share of one search step (cold-cache, serialised): {share:.3f}")
    workload = None
    try:
        for line in Path(plain).read_text().splitlines():
            if line.startswith("{"):
                workload = json.loads(line)["config"]["workload"]
    except Exception:
        pass
    (prof / f"{rnd}_scan_ncu.txt").write_text("\n".join(lines) + "\n")
    (prof / f"{rnd}_launches.txt").write_text("\n".join(ll) + "\n")
    (prof / "ncu_scan.json").write_text(json.dumps({
        "workload": workload, "kernel": r.get("Kernel Name"),
        "dram_bytes_per_launch": dram, "ncu_duration_ms": float(r["gpu__time_duration.sum"]) *
        {"usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6,
         "ns": 1e-6}.get(units["gpu__time_duration.sum"], 1e-6),
        "scan_time_share": share, "source": f"profiles/{rnd}_scan_ncu.txt"}, indent=1) + "\n")
    print("\n".join(lines + ll))


if __name__ == "__main__":
    main()
