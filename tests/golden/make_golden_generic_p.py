"""Golden fixtures for the generic degrees p = 9, 10 (the reference accepts
any p, basis.hpp:86-111; this package serves p > 8 with its multipass
pipeline, multipass.cu), generated from the REFERENCE ITSELF (oracle/_ref, the
unmodified headers compiled in place) for tests/test_generic_degree.py.

    PYTHONPATH=. python tests/golden/make_golden_generic_p.py

generic_p.npz: for each case (bp, p, dims, a) the seeded input u, the outputs
of OperatorHandle::apply / ConstrainedOperator::apply on Backend::Multipass
and Backend::Fused, the Jacobi diagonals, and the residual histories of 12 fixed
CG and Jacobi-PCG iterations on the bench RHS (Multipass).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from oracle import RefLib, random_vector  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CASES = [(1, 9, (1, 2, 1), 0.1), (3, 9, (2, 1, 1), 0.1), (5, 9, (1, 1, 2), 0.1),
         (1, 10, (1, 1, 2), 0.0), (3, 10, (1, 1, 1), 0.05), (5, 10, (1, 2, 1), 0.1)]

data = {}
for idx, (bp, p, dims, a) in enumerate(CASES):
    mp = RefLib(bp, p, dims, a, backend=0)
    fu = RefLib(bp, p, dims, a, backend=1)
    u = random_vector(2000 + idx, mp.n)
    data[f"c{idx}_u"] = u
    data[f"c{idx}_w"] = mp.apply(u, constrained=False)
    data[f"c{idx}_wc"] = mp.apply(u, constrained=True)
    data[f"c{idx}_wf"] = fu.apply(u, constrained=False)
    con = bp != 1
    rep = mp.cg(mp.bench_rhs(), rel_tol=0.0, max_iter=12, constrained=con)
    data[f"c{idx}_hist"] = rep["residual_history"]
    data[f"c{idx}_diag"] = mp.jacobi_diagonal(False)
    data[f"c{idx}_diagc"] = mp.jacobi_diagonal(True)
    rep = mp.cg(mp.bench_rhs(), rel_tol=0.0, max_iter=12, constrained=con, diag=mp.jacobi_diagonal(con))
    data[f"c{idx}_phist"] = rep["residual_history"]
data["cases"] = np.array([[bp, p, dims[0], dims[1], dims[2], a] for bp, p, dims, a in CASES])
np.savez_compressed(os.path.join(OUT, "generic_p.npz"), **data)
print("wrote generic_p.npz", len(CASES), "cases")
