"""Build the current csrc/ into paper_2109_05072_b200/build/variants/<name>/libhexbp_b200.so
(for same-box A/B timing with HEXBP_LIB=...; dev tool).
    python tools/build_variant.py <name> [extra nvcc flags, e.g. -DHX_SMB_MIN=4]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2109_05072_b200 import build as B  # noqa: E402

name = sys.argv[1]
out = os.path.join(B.PKG, "build", "variants", name)
os.makedirs(out, exist_ok=True)
objs, procs = [], []
for src in B.SOURCES:
    obj = os.path.join(out, src + ".o")
    procs.append(subprocess.Popen([B.NVCC, *B.NVCC_FLAGS, *sys.argv[2:], "-c", os.path.join(B.CSRC, src), "-o", obj]))
    objs.append(obj)
assert all(p.wait() == 0 for p in procs)
lib = os.path.join(out, "libhexbp_b200.so")
subprocess.check_call([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-ldl", "-o", lib])
print(lib)
