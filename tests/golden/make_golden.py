"""Generate the committed golden fixtures from the REFERENCE ITSELF.

Runs the unmodified reference headers compiled in place (oracle/_ref, built
by ``make -C oracle``) in this container, where /root/reference exists, and
writes small fixtures under tests/golden/. The GPU box never reads
/root/reference; the tests there compare against these files.

    PYTHONPATH=. python tests/golden/make_golden.py

Fixtures:
  equivalence.npz  -- the reference's 72-case sweep (verify.hpp:37-44): for
                      every (bp, p, dims, a) the seeded input u (seed rule of
                      verify.hpp:63, first trial), the fused-backend output of
                      OperatorHandle::apply and ConstrainedOperator::apply, B, D,
                      and the reference AoS geometric factors.
  rules.npz        -- gl_rule / gll_rule for n = 1..12 (quadrature.hpp:75-148).
  cg.json          -- CG to rel_tol 1e-8 (and fixed-iteration runs) on the
                      bench RHS (bench.hpp:234-243): iteration counts, r0,
                      final relative residual, full residual histories.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import oracle  # noqa: E402
from oracle import RefLib, random_vector  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def equivalence_cases():
    # verify.hpp:37-44
    for bp in (1, 3, 5):
        for p in (1, 2, 3, 4):
            for dims in ((1, 1, 1), (2, 2, 2), (3, 2, 1)):
                for a in (0.0, 0.1):
                    yield bp, p, dims, a


def make_equivalence():
    arrays = {}
    index = []
    for bp, p, dims, a in equivalence_cases():
        key = f"bp{bp}_p{p}_{dims[0]}x{dims[1]}x{dims[2]}_a{a}"
        try:
            r = RefLib(bp, p, dims, a)
        except RuntimeError as e:  # degenerate geometry (geometry.hpp:129)
            index.append(dict(key=key, bp=bp, p=p, dims=dims, a=a, error=str(e)))
            continue
        seed = (2024 ^ (p << 32) ^ r.n) & 0xFFFFFFFFFFFFFFFF  # verify.hpp:63
        u = random_vector(seed, r.n)
        arrays[key + "/u"] = u
        arrays[key + "/w"] = r.apply(u, constrained=False)
        arrays[key + "/wc"] = r.apply(u, constrained=True)
        B, D = r.basis()
        arrays[key + "/B"] = B
        arrays[key + "/D"] = D
        arrays[key + "/G"] = r.factors()
        index.append(dict(key=key, bp=bp, p=p, dims=dims, a=a, n=r.n, q=r.q, seed=seed))
    np.savez_compressed(os.path.join(OUT, "equivalence.npz"), **arrays)
    with open(os.path.join(OUT, "equivalence.json"), "w") as f:
        json.dump(index, f, indent=1)


def make_rules():
    arrays = {}
    # The GL/GLL tables used by the reference are exposed through the basis of
    # a problem: GL q points come from BP1/BP3 (q = p+2), GLL from BP5 (q = p+1)
    # and from the node rule (p+1).
    for p in range(1, 11):
        r3 = RefLib(3, p, (1, 1, 1), 0.0)
        qp, qw, npn, nw = r3.rules()
        arrays[f"gl{p + 2}/x"], arrays[f"gl{p + 2}/w"] = qp, qw
        arrays[f"gll{p + 1}/x"], arrays[f"gll{p + 1}/w"] = npn, nw
    np.savez_compressed(os.path.join(OUT, "rules.npz"), **arrays)


def make_cg():
    cases = [
        # (name, bp, p, dims, a, rel_tol, max_iter)
        ("cfg1_a0", 3, 3, (33, 33, 33), 0.0, 1e-8, 2000),
        ("cfg1_a0.1", 3, 3, (33, 33, 33), 0.1, 1e-8, 2000),
        ("cfg1_fixed50", 3, 3, (33, 33, 33), 0.0, 0.0, 50),
        ("bp3_p3_12_a0.1", 3, 3, (12, 12, 12), 0.1, 1e-8, 2000),
        ("bp3_p7_6_a0.1", 3, 7, (6, 6, 6), 0.1, 1e-8, 2000),
        ("bp5_p7_6_a0.1", 5, 7, (6, 6, 6), 0.1, 1e-8, 2000),
        ("bp1_p7_6_a0.1", 1, 7, (6, 6, 6), 0.1, 1e-8, 2000),
        ("bp3_p5_5x4x7_a0.1", 3, 5, (5, 4, 7), 0.1, 1e-8, 2000),
        ("bp1_p2_fixed20", 1, 2, (9, 7, 5), 0.05, 0.0, 20),
    ]
    out = {}
    for name, bp, p, dims, a, tol, mi in cases:
        t = time.time()
        r = RefLib(bp, p, dims, a)
        b = r.bench_rhs(20240101)
        rep = r.cg(b, rel_tol=tol, max_iter=mi, constrained=(bp != 1))
        x = rep["x"]
        out[name] = dict(bp=bp, p=p, dims=list(dims), a=a, rel_tol=tol, max_iter=mi, n=r.n,
                         iterations=rep["iterations"], converged=rep["converged"],
                         final_rel_residual=rep["final_rel_residual"],
                         residual_history=rep["residual_history"].tolist(),
                         x_norm=float(np.sqrt(oracle.dot(x, x))), b_sum=float(b.sum()), b_head=b[:8].tolist())
        print(name, rep["iterations"], rep["final_rel_residual"], f"{time.time() - t:.1f}s", flush=True)
    with open(os.path.join(OUT, "cg.json"), "w") as f:
        json.dump(out, f, indent=1)


def make_flops():
    out = {}
    for bp in (1, 3, 5):
        for p in range(1, 9):
            r = RefLib(bp, p, (2, 2, 2), 0.0)
            mul, add = r.count_flops()
            out[f"bp{bp}_p{p}"] = dict(mul=mul, add=add)
    with open(os.path.join(OUT, "flops.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    oracle.build()
    what = sys.argv[1:] or ["equivalence", "rules", "flops", "cg"]
    for w in what:
        globals()["make_" + w]()
