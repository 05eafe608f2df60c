"""Aggregate an .ncu-rep's SASS-level samples / instructions / smem wavefronts per CUDA source line.
    python tools/ncu_lines.py rep.ncu-rep [file-substring]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = defaultdict(lambda: defaultdict(float))
src = {}
fname = ""
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or want not in fname:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    src[(fname, ln)] = r[1]
    for k in ("Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared",
              "L1 Wavefronts Shared Ideal", "stall_barrier", "stall_short_sb", "stall_wait", "stall_math", "stall_long_sb"):
        if k in hdr:
            try:
                agg[(fname, ln)][k] += float(r[hdr.index(k)] or 0)
            except ValueError:
                pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values()) or 1
ti = sum(v["Instructions Executed"] for v in agg.values()) or 1
print(f"{'line':>5} {'samp%':>6} {'inst%':>6} {'smemWF':>10} {'ideal':>10} {'bar':>5} {'ssb':>5} {'wait':>5} {'math':>5}  source")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:int(sys.argv[3]) if len(sys.argv) > 3 else 50]:
    s = v["Warp Stall Sampling (All Samples)"] or 1
    print(f"{key[1]:5d} {v['Warp Stall Sampling (All Samples)'] / tot * 100:6.2f} {v['Instructions Executed'] / ti * 100:6.2f} "
          f"{v['L1 Wavefronts Shared']:10.0f} {v['L1 Wavefronts Shared Ideal']:10.0f} {v['stall_barrier'] / s * 100:5.0f} "
          f"{v['stall_short_sb'] / s * 100:5.0f} {v['stall_wait'] / s * 100:5.0f} {v['stall_math'] / s * 100:5.0f}  {src[key].strip()[:70]}")
