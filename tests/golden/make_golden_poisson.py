"""Golden fixtures for the manufactured-solution Poisson check (acceptance
criterion 5, proj/tests/acceptance/acceptance_main.cpp:181-222), produced
by the reference itself (oracle/_ref, ref_poisson in oracle/ref_driver.cpp):
for p = 1, 2, 3 and 2, 4, 8 elements per direction the load vector b
(essential rows zeroed), the Jacobi-PCG solution x, the discrete L2 error
and the iteration count.
    make -C oracle && python tests/golden/make_golden_poisson.py
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "..", "..", "oracle", "_ref", "libhexbp_ref.so")


def main():
    L = C.CDLL(REF)
    f = L.ref_poisson
    f.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)]
    out = {}
    cases = []
    for p in (1, 2, 3):
        for e in (2, 4, 8):
            n = (e * p + 1) ** 3
            b, x = np.zeros(n), np.zeros(n)
            err, it = C.c_double(), C.c_int()
            rc = f(e, p, b.ctypes.data, x.ctypes.data, C.byref(err), C.byref(it))
            assert rc == 0, rc
            k = f"p{p}_e{e}"
            out[k + "_b"], out[k + "_x"] = b, x
            cases.append((p, e, err.value, it.value))
    out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "poisson.npz"), **out)
    print("wrote poisson.npz", len(cases), "cases")


if __name__ == "__main__":
    main()
