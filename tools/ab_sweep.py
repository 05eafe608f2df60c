"""Same-box A/B of library builds on the bench's p sweeps (dev tool).
    python tools/ab_sweep.py lib1.so lib2.so ...   (each in a fresh process)
Prints, per library, the fast-CG roofline fraction of BP3 p=2..8 (~50M DOFs),
BP1 p=1..8 (~10M DOFs) and BP5 p=7 (~50M DOFs), as bench.py measures them.
"""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import bench
out = {"bp3": bench.p_sweep(3, 10, 0, ps=(2, 3, 4, 5, 6, 8)), "bp1": bench.p_sweep(1, 10, 0, ps=tuple(range(1, 9)), dofs=10_000_000),
       "bp5": bench.p_sweep(5, 10, 0, ps=(7,))}
print(json.dumps({k: {p: round(v["roofline_frac"], 3) for p, v in d.items()} for k, d in out.items()}))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, HEXBP_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
    print(f"{lib}: {line}", flush=True)
