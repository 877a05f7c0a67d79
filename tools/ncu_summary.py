"""Summarise an ncu report: key raw metrics + SASS stall/instruction hotspots."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_warps", "sm__warps_active.avg.per_cycle_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__t_bytes.sum", "launch__grid_size",
        "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    for i, n in enumerate(h):
        if n in want:
            print(f"  {n:60s} {r[i]} {u[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ie, ws, sc = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
data = []
for r in rows[2:]:
    try:
        data.append((r[0], r[sc], float(r[ie] or 0), float(r[ws] or 0)))
    except Exception:
        pass
ti = sum(d[2] for d in data) or 1
ts = sum(d[3] for d in data) or 1
op, ops = collections.Counter(), collections.Counter()
for a, s, i, w in data:
    t = s.split()
    o = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?")).split(".")[0]
    op[o] += i
    ops[o] += w
print("  opcode mix (inst%, stall%):", ", ".join(f"{o} {c/ti*100:.1f}/{ops[o]/ts*100:.1f}" for o, c in op.most_common(14)))
top = sorted(range(len(data)), key=lambda j: -data[j][3])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for j in top:
    a, s, i, w = data[j]
    print(f"  {a[-5:]} stall {w/ts*100:5.1f}% inst {i/ti*100:4.1f}%  {s[:70]}")
