"""Per-kernel time table from an ncu --csv launch list (gpu__time_duration)."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = collections.OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    name = r[ki].split("(")[0][:70]
    t, n = tot.get(name, (0.0, 0))
    tot[name] = (t + v, n + 1)
unit = "ns"
s = sum(t for t, _ in tot.values())
for name, (t, n) in tot.items():
    print(f"{t / 1e3:10.1f} us  {100 * t / s:5.1f}%  x{n:<3d} {name}")
print(f"{s / 1e3:10.1f} us total")
