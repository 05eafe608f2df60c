"""Golden fixtures of the reference's Multipass backend (operator.hpp:318-394),
generated from the REFERENCE ITSELF (oracle/_ref, the unmodified headers
compiled in place) for tests/test_multipass.py.

    PYTHONPATH=. python tests/golden/make_golden_multipass.py

multipass.npz: for each case (bp, p, dims, a) the seeded input u, the
Multipass outputs of OperatorHandle::apply / ConstrainedOperator::apply, and
the residual history of 12 fixed CG iterations on the bench RHS.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from oracle import RefLib, random_vector  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CASES = [(1, 2, (3, 2, 2), 0.1), (3, 2, (2, 3, 2), 0.1), (5, 2, (2, 2, 3), 0.1), (3, 3, (3, 2, 3), 0.05),
         (1, 7, (2, 1, 2), 0.1), (3, 7, (2, 2, 1), 0.1), (5, 7, (1, 2, 2), 0.1), (3, 8, (1, 1, 2), 0.0)]

data = {}
for idx, (bp, p, dims, a) in enumerate(CASES):
    r = RefLib(bp, p, dims, a, backend=0)
    u = random_vector(1000 + idx, r.n)
    data[f"c{idx}_u"] = u
    data[f"c{idx}_w"] = r.apply(u, constrained=False)
    data[f"c{idx}_wc"] = r.apply(u, constrained=True)
    b = r.bench_rhs()
    rep = r.cg(b, rel_tol=0.0, max_iter=12, constrained=bp != 1)
    data[f"c{idx}_hist"] = rep["residual_history"]
data["cases"] = np.array([[bp, p, dims[0], dims[1], dims[2], a] for bp, p, dims, a in CASES])
np.savez_compressed(os.path.join(OUT, "multipass.npz"), **data)
print("wrote multipass.npz", len(CASES), "cases")
