#!/usr/bin/env python
"""ncu per-launch CSV of one search (tools/one_search.py under
`ncu --profile-from-start off --metrics ...`) -> profiles/<name>.json:
every launch's device time, share, DRAM bytes and issue activity, the
pipeline's kernels labelled by role.  Usage:
    python tools/ncu_kernels.py gpurun_out/search_kernels.csv profiles/r02_kernels.json
"""
import csv
import io
import json
import re
import sys

WORKLOAD = "ivf-ads N=1000000 D=128 nlist=1024 nprobe=32 nq=1000 K=10 eps0=2.1"


def role(name):
    m = re.search(r"bscan_kernel<(\d+), (\w+), (\d+)", name)
    if m:
        return f"bscan_mode{m.group(3)}"
    if "bscan0_kernel" in name:  # results-only MODE 0 (filtered head)
        return "bscan_mode0"
    for key in ("bdense", "bchain1", "bchain_kernel", "bverify", "bfinal", "btprime", "bprep", "bfill",
                "bitems", "bchunks", "select", "centroid_dist", "project", "DeviceScan"):
        if key in name:
            return key.replace("_kernel", "")
    return "other"


def main(src, dst):
    text = open(src).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    launches = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        e = launches.setdefault(key, {"name": r["Kernel Name"]})
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        unit = r.get("Metric Unit", "")
        m = r["Metric Name"]
        if m == "gpu__time_duration.sum":
            e["time_us"] = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                                "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        elif m.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3,
                     "MB": 1e6, "GB": 1e9}.get(unit, 1)
            e["dram_bytes"] = e.get("dram_bytes", 0.0) + v * scale
        elif m == "smsp__issue_active.avg.pct_of_peak_sustained_active":
            e["issue_active_pct"] = v
        elif m == "sm__throughput.avg.pct_of_peak_sustained_elapsed":
            e["sm_throughput_pct"] = v
        elif m == "smsp__inst_executed.sum":
            e["warp_instructions"] = v
        elif m == "launch__registers_per_thread":
            e["registers"] = v
    ks = list(launches.values())
    tot = sum(k.get("time_us", 0) for k in ks) or 1
    for k in ks:
        k["role"] = role(k["name"])
        k["share"] = k.get("time_us", 0) / tot
        if k.get("time_us"):
            k["dram_gbs"] = k.get("dram_bytes", 0) / (k["time_us"] / 1e6) / 1e9
    dom = max(ks, key=lambda k: k.get("time_us", 0))
    out = {"workload": WORKLOAD, "source": f"{dst} from ncu per-launch capture of "
                                          "tools/one_search.py",
           "launches_per_search": len(ks), "ncu_search_us": tot,
           "dram_bytes_per_search": sum(k.get("dram_bytes", 0) for k in ks),
           "dominant_kernel": dom["name"], "dominant_time_share": dom["share"],
           "kernels": ks}
    json.dump(out, open(dst, "w"), indent=1)
    for k in sorted(ks, key=lambda k: -k.get("time_us", 0)):
        print(f"{k.get('time_us', 0):9.1f} us {k['share']*100:5.1f}% "
              f"{k.get('dram_bytes', 0)/1e6:8.1f} MB issue {k.get('issue_active_pct', 0):5.1f}% "
              f"{k['role']:14s} {k['name'][:60]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
