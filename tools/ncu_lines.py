"""Per-CUDA-source-line instruction and stall totals from an ncu report."""
import csv, io, subprocess, sys
rep = sys.argv[1]
flt = sys.argv[3].split() if len(sys.argv) > 3 else []
txt = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur_file, out = None, []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            out.append((cur_file, int(r[0]), r[1][:80], float(r[hdr.index("Instructions Executed")] or 0),
                        float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)))
        except (ValueError, IndexError):
            pass
ti = sum(o[3] for o in out) or 1
ts = sum(o[4] for o in out) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total inst {ti:.3g}")
for f, ln, src, i, w in sorted(out, key=lambda o: -o[3])[:n]:
    print(f"{f}:{ln:<4d} inst {i/ti*100:5.1f}% stall {w/ts*100:5.1f}%  {src}")
print("--- by stall")
for f, ln, src, i, w in sorted(out, key=lambda o: -o[4])[:12]:
    print(f"{f}:{ln:<4d} inst {i/ti*100:5.1f}% stall {w/ts*100:5.1f}%  {src}")
