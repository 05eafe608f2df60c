"""CPU baseline: the reference's own run_bench on this host -- TEST / BENCH
INFRASTRUCTURE ONLY (bench.py's cpu_baseline leg and --impl reference arm run
it in a subprocess; the product never imports oracle/).

Follows BASELINE.md section 2:
* the reference's headers compiled in place (oracle/_ref, Makefile), the
  highest portable ISA build this CPU supports (x86-64-v4 / v3, else the
  reference's own Release flags) -- the stand-in for -march=native, because
  the library is built on another host than the one it runs on;
* run_bench (bench.hpp:214-295) with the reference's timing protocol:
  warm-up solves, then best of `repeats` timed fixed-iteration solves, setup
  excluded; RHS seeded as the reference (BENCH_SEED, bench.hpp:193-204);
* OMP_NUM_THREADS = the physical cores of this host, OMP_PROC_BIND=close,
  OMP_PLACES=cores (set by the caller before the OpenMP runtime loads: run
  this module as a subprocess, see bench.py);
* the headline sample: same (bp, p) at ~10M DOFs (CPU throughput is flat in
  size: SURVEY §6), 20 fixed iterations (the reference default, bench.hpp:49);
  optionally config 1 in full (BP3 Q_3 33^3 = 1M DOFs, 50 fixed iterations).

    OMP_PROC_BIND=close OMP_PLACES=cores OMP_NUM_THREADS=<cores> \\
        python -m oracle.cpu_baseline --bp 3 --p 7 [--iters 20] [--cfg1]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def cpu_flags() -> set:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("flags"):
                return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def physical_cores() -> int:
    """Distinct (physical id, core id) pairs among the CPUs this process may use."""
    try:
        allowed = os.sched_getaffinity(0)
    except AttributeError:
        allowed = set(range(os.cpu_count() or 1))
    cores, cur = set(), {}
    try:
        for line in open("/proc/cpuinfo"):
            if ":" not in line:
                if "processor" in cur and int(cur["processor"]) in allowed:
                    cores.add((cur.get("physical id", "0"), cur.get("core id", cur["processor"])))
                cur = {}
                continue
            k, v = line.split(":", 1)
            cur[k.strip()] = v.strip()
        if "processor" in cur and int(cur["processor"]) in allowed:
            cores.add((cur.get("physical id", "0"), cur.get("core id", cur["processor"])))
    except OSError:
        pass
    return max(1, len(cores) or len(allowed))


V4 = {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl", "avx2", "fma", "bmi2"}
V3 = {"avx2", "fma", "bmi1", "bmi2", "f16c", "movbe"}


def ref_library() -> tuple:
    """Highest ISA-level build of the reference this CPU runs."""
    f = cpu_flags()
    base = os.path.join(HERE, "_ref", "libhexbp_ref")
    for tag, need in (("x86-64-v4", V4), ("x86-64-v3", V3)):
        path = f"{base}_{tag}.so"
        if need <= f and os.path.exists(path):
            return path, tag
    return base + ".so", "reference Release flags (-O3, x86-64 baseline)"


def auto_dims(p: int, dofs: float) -> tuple:
    e = 1
    while ((e + 1) * p + 1) ** 3 <= dofs:
        e += 1
    return (e, e, e)


def run(bp: int, p: int, dims, iters: int, warmup: int, repeats: int, so: str) -> dict:
    import oracle

    cfg = {"bp": f"bp{bp}", "degrees": [p], "dims": list(dims), "backends": ["fused"], "fixed_cg_iters": iters,
           "warmup_repeats": warmup, "timed_repeats": repeats, "threads": int(os.environ.get("OMP_NUM_THREADS", "1"))}
    t0 = time.perf_counter()
    rec = oracle.ref_run_bench(json.dumps(cfg), so=so)[0]
    return {"GDOFps": rec["throughput"] / 1e9, "dofs": int(rec["dofs"]), "threads": int(rec["threads"]),
            "best_solve_s": rec["seconds"], "wall_s": time.perf_counter() - t0, "bp": bp, "p": p, "dims": list(dims),
            "fixed_cg_iters": iters, "warmup_solves": warmup, "timed_solves": repeats}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bp", type=int, default=3)
    ap.add_argument("--p", type=int, default=7)
    ap.add_argument("--dofs", type=float, default=10e6)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--cfg1", action="store_true", help="also BASELINE configs[0]: BP3 Q_3 33^3, 50 iterations")
    a = ap.parse_args()
    cores = physical_cores()  # before the OpenMP runtime binds this thread (OMP_PROC_BIND)
    model = cpu_model()
    so, isa = ref_library()
    dims = auto_dims(a.p, a.dofs)
    head = run(a.bp, a.p, dims, a.iters, a.warmup, a.repeats, so)
    out = {"value": head["GDOFps"], "unit": "GDOF/s", "cores": head["threads"], "kind": "reference",
           "sample": f"reference run_bench (bench.hpp:214-295), bp{a.bp} p={a.p} {dims[0]}^3 elements "
                     f"({head['dofs']} DOFs), {a.iters} fixed CG iterations, best of {a.repeats} after {a.warmup} "
                     f"warm-up solve(s), setup excluded",
           "cpu_model": model, "physical_cores": cores,
           "omp": {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OMP_PROC_BIND", "OMP_PLACES")},
           "build": {"library": os.path.relpath(so, os.path.dirname(HERE)), "isa": isa}, "headline_sample": head}
    if a.cfg1:
        out["cfg1_bp3_q3_33cubed_50it"] = run(3, 3, (33, 33, 33), 50, 1, a.repeats, so)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
