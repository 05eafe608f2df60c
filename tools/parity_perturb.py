"""How sensitive is a golden CG solve to operator rounding? (CPU only; oracle.)

Runs the reference's CG recurrence (solver.hpp:91-153, deterministic_dot
order, dense.hpp:52-81) on the host with the oracle operator (bitwise the
reference's) whose every output is multiplied by (1 + eps * U(-1, 1)), U
drawn per entry and per apply -- a model of the fast kernels' ~1e-16
per-entry deviation. Reports the iteration count and final relative
residual per (eps, seed) against the unperturbed solve.

    python tools/parity_perturb.py bp3_p3_12_a0.1 bp5_p7_6_a0.1 > profiles/r2_parity_perturb.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from oracle import Oracle  # noqa: E402


def host_cg(apply, b, tol, maxit):
    """solver.hpp:91-153 with x0 = 0, unpreconditioned, deterministic_dot."""
    x = np.zeros_like(b)
    r = b - apply(x)
    r0 = np.sqrt(oracle.dot(r, r))
    p = r.copy()
    rz = oracle.dot(r, r)
    k = 0
    rn = r0
    for k in range(1, maxit + 1):
        Ap = apply(p)
        al = rz / oracle.dot(p, Ap)
        x += al * p
        r -= al * Ap
        rn = np.sqrt(oracle.dot(r, r))
        if rn / r0 <= tol:
            break
        rzn = oracle.dot(r, r)
        p = r + (rzn / rz) * p
        rz = rzn
    return k, rn / r0


def main():
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "cg.json")))
    out = {"what": "reference CG with the oracle operator perturbed by (1 + eps U(-1,1)) per entry and apply",
           "cases": {}}
    for name in sys.argv[1:]:
        c = gold[name]
        o = Oracle(c["bp"], c["p"], tuple(c["dims"]), c["a"])
        b = o.bench_rhs()
        con = c["bp"] != 1
        base = host_cg(lambda v: o.apply(v, con), b, c["rel_tol"], c["max_iter"])
        rows = []
        for eps in (1e-16, 2e-16, 5e-16):
            for seed in range(4):
                rng = np.random.default_rng(seed)
                it, fin = host_cg(lambda v: o.apply(v, con) * (1.0 + eps * rng.uniform(-1, 1, v.size)), b,
                                  c["rel_tol"], c["max_iter"])
                rows.append({"eps": eps, "seed": seed, "iterations": it, "final_rel_residual": fin,
                             "d_iter": it - c["iterations"], "d_final": abs(fin - c["final_rel_residual"])})
                print(name, rows[-1], file=sys.stderr)
        out["cases"][name] = {"reference_iterations": c["iterations"],
                              "reference_final_rel_residual": c["final_rel_residual"],
                              "unperturbed_host": {"iterations": base[0], "final_rel_residual": base[1]},
                              "perturbed": rows,
                              "max_abs_d_iter": max(abs(r["d_iter"]) for r in rows),
                              "max_d_final": max(r["d_final"] for r in rows)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
