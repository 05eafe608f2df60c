"""Dev probe: BP1 / BP3 fast CG (bench p_sweep sizes) under the z-segment
heuristic overrides HEXBP_SEG_WAVES / HEXBP_SEG_MIN (read once per process)."""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import bench
r = {"bp1": bench.p_sweep(1, 10, 0, ps=(1, 2, 8), dofs=10_000_000), "bp3": bench.p_sweep(3, 10, 0, ps=(8,))}
print(json.dumps({k: {p: round(v["roofline_frac"], 3) for p, v in d.items()} for k, d in r.items()}))
'''
for waves in ("1", "2", "3", "4"):
    for mn in ("2", "4", "8"):
        env = dict(os.environ, HEXBP_SEG_WAVES=waves, HEXBP_SEG_MIN=mn)
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print(waves, mn, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:], flush=True)
