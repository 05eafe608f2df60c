"""TEST INFRASTRUCTURE ONLY -- the parity oracle for the CUDA product path.

Two CPU implementations of the reference hexbp path, loaded through ctypes:

* ``Oracle``  -- ``oracle/liboracle.so``, the plain-C restatement
  (``oracle/hexbp_oracle.c``; every function cites the reference file:line).
* ``RefLib``  -- ``oracle/_ref/libhexbp_ref.so``, the UNMODIFIED reference
  headers compiled in place by ``oracle/Makefile`` (only in containers where
  ``/root/reference`` exists; the built .so travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The
product package ``paper_2109_05072_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhexbp_ref.so")
# the drop-in test binary (tests/cpp/test_dropin_ref.cpp against the reference headers)
DROPIN_BIN = os.path.join(HERE, "_ref", "test_dropin_ref")
DROPIN_SRC = os.path.join(os.path.dirname(HERE), "tests", "cpp", "test_dropin_ref.cpp")

_dp = C.POINTER(C.c_double)


def build(force: bool = False) -> None:
    """Compile the C restatement (and oracle/_ref when the reference exists)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.isdir("/root/reference") and not (
            all(os.path.exists(REF_SO.replace(".so", v + ".so")) for v in ("", "_x86-64-v3", "_x86-64-v4"))
            and os.path.exists(DROPIN_BIN) and os.path.getmtime(DROPIN_BIN) >= os.path.getmtime(DROPIN_SRC))
    ):
        subprocess.run(["make", "-C", HERE, "all"], check=True, stdout=subprocess.DEVNULL)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class _Lib:
    _cache: dict = {}

    @classmethod
    def load(cls, path: str) -> C.CDLL:
        if path not in cls._cache:
            if not os.path.exists(path):
                raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
            cls._cache[path] = C.CDLL(path)
        return cls._cache[path]


class Oracle:
    """One BP problem on the structured box mesh, C restatement."""

    prefix = "or_"
    so = ORACLE_SO

    def __init__(self, bp: int, p: int, dims, amplitude: float = 0.0):
        lib = _Lib.load(self.so)
        self.lib = lib
        pre = self.prefix
        self._fn = lambda name: getattr(lib, pre + name)
        self._declare()
        self.bp, self.p, self.dims, self.amplitude = bp, p, tuple(dims), amplitude
        self.h = self._create(bp, p, dims, amplitude)
        if not self.h:
            raise RuntimeError(self._fn("last_error")().decode())
        self.n = int(self._fn("size")(self.h))
        self.E = int(self._fn("num_elements")(self.h))
        self.q = int(self._fn("q")(self.h))
        self.comp = int(self._fn("components")(self.h))

    def _declare(self):
        f = self._fn
        f("create").restype = C.c_void_p
        f("last_error").restype = C.c_char_p
        f("size").restype = C.c_int64
        for nm in ("size", "num_elements", "q", "components", "destroy", "basis", "factors", "coords", "apply",
                   "cg", "bench_rhs", "rules"):
            f(nm).argtypes = None
        f("size").argtypes = [C.c_void_p]
        f("num_elements").argtypes = [C.c_void_p]
        f("q").argtypes = [C.c_void_p]
        f("components").argtypes = [C.c_void_p]
        f("destroy").argtypes = [C.c_void_p]
        f("basis").argtypes = [C.c_void_p, _dp, _dp]
        f("rules").argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        f("factors").argtypes = [C.c_void_p, _dp]
        f("coords").argtypes = [C.c_void_p, _dp]
        f("apply").argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        f("cg").argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_double, C.c_int, C.POINTER(C.c_int),
                            C.POINTER(C.c_int), C.POINTER(C.c_double), _dp] + self._cg_extra()
        f("bench_rhs").argtypes = [C.c_void_p, C.c_uint64, _dp]

    def _cg_extra(self):
        return []

    def _create(self, bp, p, dims, a):
        self._fn("create").argtypes = [C.c_int] * 5 + [C.c_double]
        return self._fn("create")(bp, p, dims[0], dims[1], dims[2], a)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self._fn("destroy")(h)
            self.h = None

    # -- data ---------------------------------------------------------
    def basis(self):
        nn = self.p + 1
        B = np.zeros((self.q, nn))
        D = np.zeros((self.q, nn))
        self._fn("basis")(self.h, _ptr(B), _ptr(D))
        return B, D

    def rules(self):
        nn = self.p + 1
        qp, qw, np_, nw = np.zeros(self.q), np.zeros(self.q), np.zeros(nn), np.zeros(nn)
        self._fn("rules")(self.h, _ptr(qp), _ptr(qw), _ptr(np_), _ptr(nw))
        return qp, qw, np_, nw

    def factors(self) -> np.ndarray:
        out = np.zeros(self.E * self.q**3 * self.comp)
        self._fn("factors")(self.h, _ptr(out))
        return out

    def coords(self) -> np.ndarray:
        out = np.zeros(3 * self.n)
        self._fn("coords")(self.h, _ptr(out))
        return out.reshape(-1, 3)

    # -- operator / solver --------------------------------------------
    def apply(self, u, constrained: bool = False) -> np.ndarray:
        u = _f64(u)
        assert u.size == self.n
        w = np.zeros(self.n)
        rc = self._fn("apply")(self.h, int(constrained), _ptr(u), _ptr(w))
        if rc:
            raise RuntimeError(self._fn("last_error")().decode())
        return w

    def jacobi_diagonal(self, constrained: bool = True) -> np.ndarray:
        """jacobi_diagonal (solver.hpp:155-205)."""
        out = np.zeros(self.n)
        f = self._fn("jacobi_diagonal")
        f.argtypes = [C.c_void_p, C.c_int, _dp]
        f(self.h, int(constrained), _ptr(out))
        return out

    def bench_rhs(self, seed: int = 20240101) -> np.ndarray:
        b = np.zeros(self.n)
        self._fn("bench_rhs")(self.h, C.c_uint64(seed), _ptr(b))
        return b

    def cg(self, b, x0=None, rel_tol: float = 1e-8, max_iter: int = 2000, constrained: bool = True, diag=None):
        b = _f64(b)
        x = np.zeros(self.n) if x0 is None else _f64(x0).copy()
        it, conv, fr = C.c_int(0), C.c_int(0), C.c_double(0.0)
        hist = np.zeros(max_iter + 1)
        extra = self._cg_extra_args()
        if diag is None:
            rc = self._fn("cg")(self.h, int(constrained), _ptr(b), _ptr(x), rel_tol, max_iter, C.byref(it),
                                C.byref(conv), C.byref(fr), _ptr(hist), *extra)
        else:  # Jacobi-preconditioned (solver.hpp:105-108)
            d = _f64(diag)
            assert d.size == self.n
            f = self._fn("pcg")
            f.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_double, C.c_int, C.POINTER(C.c_int),
                          C.POINTER(C.c_int), C.POINTER(C.c_double), _dp] + self._cg_extra()
            rc = f(self.h, int(constrained), _ptr(b), _ptr(x), _ptr(d), rel_tol, max_iter, C.byref(it),
                   C.byref(conv), C.byref(fr), _ptr(hist), *extra)
        if rc == 2:
            raise ArithmeticError("divergence_error: " + self._fn("last_error")().decode())
        if rc:
            raise RuntimeError(self._fn("last_error")().decode())
        return dict(iterations=it.value, converged=bool(conv.value), final_rel_residual=fr.value,
                    residual_history=hist[: it.value + 1].copy(), x=x)

    def _cg_extra_args(self):
        return []


class OracleSlab(Oracle):
    """Element layers [z0, z1) of the (ex, ey, gez) box: the local problem of
    one rank of the multi-GPU z-slab partition (coordinates from the global
    box, essential nodes on the global box surface only)."""

    def __init__(self, bp: int, p: int, gdims, z0: int, z1: int, amplitude: float = 0.0):
        self.slab = (z0, z1)
        super().__init__(bp, p, gdims, amplitude)

    def _create(self, bp, p, dims, a):
        f = self._fn("create_slab")
        f.restype = C.c_void_p
        f.argtypes = [C.c_int] * 7 + [C.c_double]
        return f(bp, p, dims[0], dims[1], dims[2], self.slab[0], self.slab[1], a)


class RefLib(Oracle):
    """The reference itself (headers compiled in place), same interface."""

    prefix = "ref_"
    so = REF_SO

    def __init__(self, bp: int, p: int, dims, amplitude: float = 0.0, backend: int = 1):
        """backend: 1 = Backend::Fused, 0 = Backend::Multipass (operator.hpp:31)."""
        self.backend = backend
        super().__init__(bp, p, dims, amplitude)

    def _create(self, bp, p, dims, a):
        self._fn("create").argtypes = [C.c_int] * 5 + [C.c_double, C.c_int]
        return self._fn("create")(bp, p, dims[0], dims[1], dims[2], a, getattr(self, "backend", 1))

    def _cg_extra(self):
        return [_dp]

    def _cg_extra_args(self):
        self._secs = C.c_double(0.0)
        return [C.byref(self._secs)]

    def count_flops(self):
        mul, add = C.c_uint64(0), C.c_uint64(0)
        f = self._fn("count_flops")
        f.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        f(self.h, C.byref(mul), C.byref(add))
        return mul.value, add.value


def oracle_lib() -> C.CDLL:
    lib = _Lib.load(ORACLE_SO)
    lib.or_dot.restype = C.c_double
    lib.or_dot.argtypes = [_dp, _dp, C.c_int64]
    lib.or_random_vector.argtypes = [C.c_uint64, C.c_int64, _dp]
    lib.or_mix_seed.restype = C.c_uint64
    lib.or_mix_seed.argtypes = [C.c_uint64] + [C.c_int] * 5
    lib.or_gl_rule.argtypes = [C.c_int, _dp, _dp]
    lib.or_gll_rule.argtypes = [C.c_int, _dp, _dp]
    return lib


def random_vector(seed: int, n: int) -> np.ndarray:
    """tests/unit/test_support.hpp:15-21 (mt19937_64 + uniform(-1,1))."""
    out = np.zeros(n)
    oracle_lib().or_random_vector(C.c_uint64(seed), n, _ptr(out))
    return out


def dot(a, b) -> float:
    """deterministic_dot, dense.hpp:74-81."""
    a, b = _f64(a), _f64(b)
    return float(oracle_lib().or_dot(_ptr(a), _ptr(b), a.size))


def ref_run_bench(config_json: str, cap: int = 64, so: str = REF_SO):
    """Reference run_bench through its JSON parser (bench.hpp:93-153,214-295)."""
    lib = _Lib.load(so)
    f = lib.ref_run_bench_json
    f.restype = C.c_int
    f.argtypes = [C.c_char_p, _dp, _dp, C.POINTER(C.c_int64), C.POINTER(C.c_int), C.c_int]
    thr, sec = np.zeros(cap), np.zeros(cap)
    dofs = (C.c_int64 * cap)()
    threads = (C.c_int * cap)()
    n = f(config_json.encode(), _ptr(thr), _ptr(sec), dofs, threads, cap)
    if n < 0:
        lib.ref_last_error.restype = C.c_char_p
        raise RuntimeError(lib.ref_last_error().decode())
    return [dict(throughput=thr[i], seconds=sec[i], dofs=dofs[i], threads=threads[i]) for i in range(n)]


def ref_check_equivalence(bp: int, p: int, dims, a: float):
    lib = _Lib.load(REF_SO)
    f = lib.ref_check_equivalence
    f.argtypes = [C.c_int] * 5 + [C.c_double, _dp]
    out = np.zeros(7)
    if f(bp, p, dims[0], dims[1], dims[2], a, _ptr(out)):
        lib.ref_last_error.restype = C.c_char_p
        raise RuntimeError(lib.ref_last_error().decode())
    keys = ["max_rel_multipass", "max_rel_fused", "max_symmetry", "max_asymmetry_matrix", "nullspace_residual",
            "min_quadratic_form", "pass"]
    return dict(zip(keys, out.tolist()))
