"""Executed warp instructions per SASS opcode (from an .ncu-rep source page).
    python tools/ncu_opmix.py rep.ncu-rep [per-unit divisor]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
agg = defaultdict(float)
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= iE:
        continue
    try:
        n = float(r[iE] or 0)
    except ValueError:
        continue
    toks = r[iS].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    agg[op.split(".")[0]] += n
tot = sum(agg.values())
print(f"total {tot:.4g} ({tot / div:.1f} per unit)")
for op, n in sorted(agg.items(), key=lambda t: -t[1])[:40]:
    print(f"{op:12s} {n / div:10.1f} {100 * n / tot:5.1f}%")
