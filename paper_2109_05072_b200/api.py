"""Host-side mirror of the reference ``hexbp`` operator API for the B200 path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/hexbp/{mesh,operator,solver}.hpp so a caller of
the reference finds the same surface:

=========================  =====================================================
reference (file:line)      here
=========================  =====================================================
BPKind (operator.hpp:29)   ``BPKind``
Backend (operator.hpp:31)  ``Backend.Cuda`` (the new plugin value)
build_box_mesh (mesh:86)   ``build_box_mesh`` (metadata; coordinates are
                           generated on the device by ``make_setup``)
make_setup (operator:70)   ``make_setup`` -> device ``OperatorSetup``
OperatorHandle (op:244)    ``OperatorHandle`` (.apply, .size, .make_workspace,
                           .count_flops)
ConstrainedOperator (solver:48)  ``ConstrainedOperator``
cg / CGReport (solver:76-153)    ``cg`` / ``CGReport`` (device-resident recurrence)
divergence_error (solver:17)     ``divergence_error``
degenerate_element_error (geometry:19)  ``degenerate_element_error``
=========================  =====================================================

Vectors may be numpy arrays (host; the call copies through the device and
is synchronous, like the reference's std::vector signature) or CUDA torch
tensors (device-resident; launched asynchronously on torch's current stream).
Every numeric path runs in ``libhexbp_b200.so``; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib

_dp = C.POINTER(C.c_double)


# ---------------------------------------------------------------- errors
class divergence_error(RuntimeError):
    """solver.hpp:17-20"""


class degenerate_element_error(RuntimeError):
    """geometry.hpp:19-32"""


class HexbpCudaError(RuntimeError):
    pass


DivergenceError = divergence_error
DegenerateElementError = degenerate_element_error


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.lib().hexbp_last_error().decode()
    if rc == 1:
        raise ValueError(msg)  # std::invalid_argument
    if rc == 2:
        raise divergence_error(msg)
    if rc == 4:
        raise MemoryError(msg)
    if rc == 5:
        raise degenerate_element_error(msg)
    if rc == 6:
        raise RuntimeError(msg)  # std::logic_error
    raise HexbpCudaError(msg)


# ---------------------------------------------------------------- enums
class BPKind(enum.IntEnum):
    BP1 = 1
    BP3 = 3
    BP5 = 5


class Backend(enum.Enum):
    Cuda = "cuda"  # Backend::Fused on the GPU (fast or reference arithmetic, Workspace.set_mode)
    CudaMultipass = "cuda-multipass"  # Backend::Multipass on the GPU (multipass.cu), reference arithmetic


def to_string(v) -> str:
    if isinstance(v, BPKind):
        return f"bp{int(v)}"
    if isinstance(v, Backend):
        return v.value
    raise TypeError(v)


def parse_bp(s: str) -> BPKind:  # bench.hpp:80-85
    m = {"bp1": BPKind.BP1, "bp3": BPKind.BP3, "bp5": BPKind.BP5}
    if s not in m:
        raise ValueError(f"unknown bp kind '{s}' (expected bp1, bp3 or bp5)")
    return m[s]


def parse_backend(s: str) -> Backend:  # bench.hpp:86-91, with the CUDA backends' names
    for b in Backend:
        if b.value == s:
            return b
    raise ValueError(f"unknown backend '{s}' (this package provides: cuda, cuda-multipass)")


def is_diffusion(k: BPKind) -> bool:  # operator.hpp:51
    return BPKind(k) != BPKind.BP1


def default_quad_points(k: BPKind, p: int) -> int:  # operator.hpp:55
    return p + 1 if BPKind(k) == BPKind.BP5 else p + 2


# ---------------------------------------------------------------- mesh
kMaxDeformAmplitude = 0.15  # mesh.hpp:84


@dataclass
class HexMesh:
    """Structured deformed box (mesh.hpp:29-51). Node coordinates are never
    materialised on the host: the device setup evaluates mesh.hpp:107-119."""

    dims: tuple = (1, 1, 1)
    degree: int = 1
    extent: tuple = (1.0, 1.0, 1.0)
    deform_amplitude: float = 0.0

    def num_elements(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    def nodes_per_elem(self) -> int:
        return (self.degree + 1) ** 3

    def node_grid(self) -> tuple:
        return tuple(d * self.degree + 1 for d in self.dims)

    def num_nodes(self) -> int:
        g = self.node_grid()
        return g[0] * g[1] * g[2]


def build_box_mesh(dims: Sequence[int], p: int, extent=(1.0, 1.0, 1.0), deform_amplitude: float = 0.0) -> HexMesh:
    """mesh.hpp:86-123 argument validation; std::invalid_argument -> ValueError."""
    dims = tuple(int(d) for d in dims)
    if len(dims) != 3 or any(d < 1 for d in dims):
        raise ValueError("build_box_mesh: element counts must be >= 1")
    if any(not (e > 0.0) for e in extent):
        raise ValueError("build_box_mesh: extents must be positive")
    if p < 1:
        raise ValueError("build_box_mesh: degree must be >= 1")
    if not (0.0 <= deform_amplitude <= kMaxDeformAmplitude):
        raise ValueError("build_box_mesh: deform amplitude outside [0, 0.15]")
    return HexMesh(dims, int(p), tuple(float(e) for e in extent), float(deform_amplitude))


def boundary_nodes(mesh: HexMesh) -> np.ndarray:
    """mesh.hpp:126-135: global indices of box-surface nodes, ascending."""
    gx, gy, gz = mesh.node_grid()
    kz, ky, kx = np.meshgrid(np.arange(gz), np.arange(gy), np.arange(gx), indexing="ij")
    on = (kx == 0) | (kx == gx - 1) | (ky == 0) | (ky == gy - 1) | (kz == 0) | (kz == gz - 1)
    return np.flatnonzero(on.ravel()).astype(np.int32)


@dataclass
class BCSet:
    """solver.hpp:24-35"""

    dofs: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def validate(self, l_size: int) -> None:
        if len(self.dofs) != len(self.values):
            raise ValueError("BCSet: dofs/values size mismatch")
        d = np.asarray(self.dofs)
        if d.size and (d.min() < 0 or d.max() >= l_size):
            raise ValueError("BCSet: dof index out of range")
        if d.size > 1 and np.any(np.diff(d) <= 0):
            raise ValueError("BCSet: dof indices must be strictly increasing")


def boundary_bcs(mesh: HexMesh, value: float = 0.0) -> BCSet:  # solver.hpp:38-43
    d = boundary_nodes(mesh)
    return BCSet(d, np.full(d.size, value))


# ---------------------------------------------------------------- setup
def _i3(v) -> C.Array:
    return (C.c_int * 3)(*[int(x) for x in v])


class OperatorSetup:
    """Device-resident OperatorSetup (operator.hpp:60-68): basis tables and the
    geometric factors in the kernel's streaming layout."""

    def __init__(self, handle: int, device: int):
        self._h = C.c_void_p(handle)
        self.device = device
        info = _lib.SetupInfo()
        _check(_lib.lib().hexbp_setup_get_info(self._h, C.byref(info)))
        self.kind = BPKind(info.bp)
        self.p, self.q = info.p, info.q
        self.dims = tuple(info.dims)
        self.gdims = tuple(info.gdims)
        self.z0 = info.z0
        self.components = info.components
        self._l_size = int(info.l_size)
        self._E = int(info.elements)
        self.factor_bytes = int(info.factor_bytes)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().hexbp_setup_destroy(h)
            except Exception:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    def l_size(self) -> int:
        return self._l_size

    def num_elements(self) -> int:
        return self._E

    def basis(self):
        n = self.p + 1
        B, D = np.zeros((self.q, n)), np.zeros((self.q, n))
        _check(_lib.lib().hexbp_setup_basis(self._h, B.ctypes.data_as(_dp), D.ctypes.data_as(_dp)))
        return B, D

    def factors(self) -> np.ndarray:
        """Factors in the reference AoS layout (geometry.hpp:48-56)."""
        out = np.zeros(self._E * self.q**3 * self.components)
        _check(_lib.lib().hexbp_setup_factors(self._h, out.ctypes.data_as(_dp)))
        return out

    @classmethod
    def from_reference(cls, kind, p: int, dims, B, D, factors_aos, device: int = 0,
                       elem_to_global=None) -> "OperatorSetup":
        """Adopt a host OperatorSetup's tables (drop-in path). ``elem_to_global``
        (ElementRestriction, restriction.hpp:22-53), when given, is checked to be
        the structured box numbering the kernels compute (ValueError otherwise)."""
        kind = BPKind(kind)
        q = default_quad_points(kind, p)
        B = np.ascontiguousarray(B, np.float64)
        D = np.ascontiguousarray(D, np.float64)
        F = np.ascontiguousarray(factors_aos, np.float64)
        h = C.c_void_p()
        _check(_lib.lib().hexbp_setup_create(int(kind), p, q, _i3(dims), B.ctypes.data_as(_dp),
                                             D.ctypes.data_as(_dp), F.ctypes.data_as(_dp), device, C.byref(h)))
        s = cls(h.value, device)
        if elem_to_global is not None:
            s.check_restriction(elem_to_global)
        return s

    def check_restriction(self, elem_to_global) -> None:
        """hexbp_setup_check_restriction: ValueError unless the table is the
        structured numbering of this box (mesh.hpp:74-82)."""
        t = np.ascontiguousarray(elem_to_global, np.int32)
        _check(_lib.lib().hexbp_setup_check_restriction(self._h, t.ctypes.data_as(C.c_void_p), t.size))


def make_setup(kind, mesh: HexMesh, device: int = 0) -> OperatorSetup:
    """make_setup (operator.hpp:70-77) with the geometry generated on the device."""
    h = C.c_void_p()
    ext = np.asarray(mesh.extent, np.float64)
    _check(_lib.lib().hexbp_setup_create_box(int(BPKind(kind)), mesh.degree, _i3(mesh.dims),
                                             ext.ctypes.data_as(_dp), mesh.deform_amplitude, device, C.byref(h)))
    return OperatorSetup(h.value, device)


def make_slab_setup(kind, mesh: HexMesh, z0: int, z1: int, device: int = 0) -> OperatorSetup:
    """Element layers [z0, z1) of ``mesh`` (multi-GPU partition, parallel.py)."""
    h = C.c_void_p()
    ext = np.asarray(mesh.extent, np.float64)
    _check(_lib.lib().hexbp_setup_create_box_slab(int(BPKind(kind)), mesh.degree, _i3(mesh.dims), z0, z1,
                                                  ext.ctypes.data_as(_dp), mesh.deform_amplitude, device,
                                                  C.byref(h)))
    return OperatorSetup(h.value, device)


class Workspace:
    """Device Workspace (operator.hpp:148-211): allocated once, never inside apply/cg."""

    def __init__(self, setup: OperatorSetup):
        self.setup = setup
        h = C.c_void_p()
        _check(_lib.lib().hexbp_workspace_create(setup._h, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().hexbp_workspace_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def dot(self, a, b) -> float:
        """deterministic_dot (dense.hpp:74-81) of two device tensors."""
        n = a.numel()
        _check_device_vec(a, n, "dot")
        _check_device_vec(b, n, "dot")
        out = C.c_double(0.0)
        _check(_lib.lib().hexbp_dot(self._h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), n,
                                    C.byref(out), _stream_ptr(a)))
        return out.value

    def set_mode(self, mode: str) -> None:
        """'reference' (default): bit-exact reference arithmetic; 'fast': FMA / DMMA kernels, fused p.Ap;
        'fast_operator': the fast operator kernel under the reference's CG recurrence and
        deterministic_dot order (only the operator's rounding differs from the reference)."""
        _check(_lib.lib().hexbp_workspace_set_mode(self._h, {"reference": 0, "fast": 1, "fast_operator": 2}[mode]))

    def qpoint_fields(self) -> int:
        """Workspace::qpoint_fields (operator.hpp:193-194)."""
        q, b = C.c_int(0), C.c_uint64(0)
        _check(_lib.lib().hexbp_workspace_info(self._h, C.byref(q), C.byref(b)))
        return q.value

    def global_bytes(self) -> int:
        """Workspace::global_bytes (operator.hpp:196-201): element-level global scratch."""
        q, b = C.c_int(0), C.c_uint64(0)
        _check(_lib.lib().hexbp_workspace_info(self._h, C.byref(q), C.byref(b)))
        return b.value

    def kernel_info(self) -> dict:
        vals = [C.c_int(0) for _ in range(4)]
        _check(_lib.lib().hexbp_kernel_info(self.setup._h, *[C.byref(v) for v in vals]))
        return dict(zip(["registers", "smem_bytes", "threads", "ctas_per_sm"], [v.value for v in vals]))


@dataclass
class FlopCount:
    """tensor.hpp:19-29"""

    mul: int = 0
    add: int = 0

    def total(self) -> int:
        return self.mul + self.add


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _stream_ptr(t) -> C.c_void_p:
    import torch

    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _check_device_vec(t, n: int, name: str):
    import torch

    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError(f"{name}: expected a contiguous float64 CUDA tensor")
    if t.numel() != n:
        raise ValueError(f"{name}: L-vector length mismatch")


FUSED_MAX_DEGREE = 8  # the fused kernels' degrees; 9..10 run the multipass pipeline (reference arithmetic)


class OperatorHandle:
    """OperatorHandle (operator.hpp:244-420) bound to the CUDA backend."""

    def __init__(self, backend: Backend, setup: OperatorSetup):
        if backend not in (Backend.Cuda, Backend.CudaMultipass):
            raise ValueError("OperatorHandle: this package implements the CUDA backends only")
        self._backend = backend
        self._setup = setup
        self._ws = self.make_workspace()

    def kind(self) -> BPKind:
        return self._setup.kind

    def backend(self) -> Backend:
        return self._backend

    def setup(self) -> OperatorSetup:
        return self._setup

    def size(self) -> int:
        return self._setup.l_size()

    def make_workspace(self) -> Workspace:
        ws = Workspace(self._setup)
        if self._backend == Backend.CudaMultipass:
            _check(_lib.lib().hexbp_workspace_set_backend(ws._h, 1))
        return ws

    def workspace(self) -> Workspace:
        return self._ws

    def oracle_matrix(self):
        raise RuntimeError("oracle_matrix: not an oracle backend")  # operator.hpp:258 (std::logic_error)

    def _apply(self, u, w, ws: Optional[Workspace], constrained: int):
        ws = ws or self._ws
        n = self.size()
        if _is_torch(u):
            import torch

            _check_device_vec(u, n, "apply")
            if w is None:
                w = torch.empty_like(u)
            _check_device_vec(w, n, "apply")
            _check(_lib.lib().hexbp_apply(self._setup._h, ws._h, C.c_void_p(u.data_ptr()), C.c_void_p(w.data_ptr()),
                                          constrained, _stream_ptr(u)))
            return w
        u = np.ascontiguousarray(u, np.float64)
        if u.size != n:
            raise ValueError("apply: L-vector length mismatch")  # operator.hpp:268
        # write through the caller's w only when it is a contiguous float64 array of
        # length n; otherwise apply into a fresh array (the reference resizes w,
        # operator.hpp:273) and copy into w where its shape allows
        direct = isinstance(w, np.ndarray) and w.dtype == np.float64 and w.size == n and w.flags.c_contiguous
        out = w if direct else np.empty(n)
        _check(_lib.lib().hexbp_apply_host(self._setup._h, ws._h, u.ctypes.data_as(_dp), out.ctypes.data_as(_dp), n,
                                           constrained))
        if isinstance(w, list):
            w[:] = out.tolist()
        elif isinstance(w, np.ndarray) and not direct and w.size == n:
            w[...] = out.reshape(w.shape)
        return out

    def apply(self, u, w=None, ws: Optional[Workspace] = None, flops: Optional[FlopCount] = None):
        """w = A u. Returns w (allocated when not given or of the wrong size, as
        the reference resizes, operator.hpp:273)."""
        w = self._apply(u, w, ws, 0)
        if flops is not None:
            f = self.count_flops()
            flops.mul += f.mul * self._setup.num_elements()
            flops.add += f.add * self._setup.num_elements()
        return w

    def count_flops(self) -> FlopCount:
        m, a = C.c_uint64(0), C.c_uint64(0)
        _check(_lib.lib().hexbp_count_flops(self._setup._h, C.byref(m), C.byref(a)))
        return FlopCount(m.value, a.value)


def make_operator(kind, backend: Backend, mesh: HexMesh, device: int = 0) -> OperatorHandle:
    return OperatorHandle(backend, make_setup(kind, mesh, device))


class ConstrainedOperator:
    """w = P A P u + (I - P) u (solver.hpp:48-74). The device kernel applies the
    mask by a grid-boundary test, i.e. the box-surface constraint set of
    boundary_bcs(mesh); other dof sets are rejected. The constraint values are
    accepted and ignored, as the reference's apply ignores them (w = u on the
    essential dofs, solver.hpp:60-65)."""

    def __init__(self, op: OperatorHandle, bcs: Optional[BCSet] = None):
        self._op = op
        s = op.setup()
        if bcs is not None:
            bcs.validate(op.size())
            mesh = HexMesh(s.dims, s.p)
            if s.dims != s.gdims or not np.array_equal(np.asarray(bcs.dofs), boundary_nodes(mesh)):
                raise ValueError("ConstrainedOperator: the CUDA backend supports the box-surface BCSet only")
        self._bcs = bcs

    def size(self) -> int:
        return self._op.size()

    def raw(self) -> OperatorHandle:
        return self._op

    def apply(self, u, w=None, ws: Optional[Workspace] = None):
        return self._op._apply(u, w, ws, 1)


@dataclass
class CGReport:
    """solver.hpp:76-82"""

    iterations: int = 0
    converged: bool = False
    final_rel_residual: float = 0.0
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    seconds: float = 0.0


def cg(apply_op, b, x, rel_tol: float = 1e-8, max_iter: int = 2000, diag=None,
       ws: Optional[Workspace] = None, mode: str = "reference") -> CGReport:
    """cg (solver.hpp:91-153) for a device operator (OperatorHandle or
    ConstrainedOperator): the whole recurrence runs on the device. ``x`` holds
    x0 on entry and the solution on exit (numpy arrays are updated in place).
    ``reduction='reference'`` reproduces deterministic_dot and the reference's
    vector arithmetic bit for bit; ``'fused'`` fuses p.Ap into the operator."""
    if isinstance(apply_op, ConstrainedOperator):
        op, constrained = apply_op.raw(), 1
    elif isinstance(apply_op, OperatorHandle):
        op, constrained = apply_op, 0
    else:
        raise TypeError("cg: expected an OperatorHandle or ConstrainedOperator of the CUDA backend")
    ws = ws or op.workspace()
    if op.backend() == Backend.CudaMultipass or op.setup().p > FUSED_MAX_DEGREE:
        mode = "reference"  # the multipass pipeline (and every degree > 8) runs in reference arithmetic
    ws.set_mode(mode)
    n = op.size()
    rep = _lib.CGReportC()
    hist = np.zeros(max_iter + 1)
    t0 = time.perf_counter()
    if _is_torch(b):
        _check_device_vec(b, n, "cg")
        if not _is_torch(x) or x.numel() != n:
            raise ValueError("cg: x0 length mismatch")
        _check_device_vec(x, n, "cg")
        if x.device != b.device:
            raise ValueError("cg: x and b on different devices")
        dptr = None
        if diag is not None:  # Jacobi preconditioner (solver.hpp:105-108)
            import torch

            if not _is_torch(diag):
                diag = torch.as_tensor(np.ascontiguousarray(diag, np.float64), device=b.device)
            if diag.numel() != n:
                raise ValueError("cg: diagonal length mismatch")  # solver.hpp:97
            _check_device_vec(diag, n, "cg")
            dptr = C.c_void_p(diag.data_ptr())
        if dptr is None:
            rc = _lib.lib().hexbp_cg(op.setup()._h, ws._h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()),
                                     rel_tol, max_iter, constrained, C.byref(rep), hist.ctypes.data_as(_dp),
                                     _stream_ptr(b))
        else:
            rc = _lib.lib().hexbp_pcg(op.setup()._h, ws._h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()),
                                      dptr, rel_tol, max_iter, constrained, C.byref(rep), hist.ctypes.data_as(_dp),
                                      _stream_ptr(b))
    else:
        b = np.ascontiguousarray(b, np.float64)
        if not isinstance(x, np.ndarray) or x.dtype != np.float64 or x.size != n or not x.flags.c_contiguous:
            raise ValueError("cg: x0 length mismatch")
        if b.size != n:
            raise ValueError("cg: b length mismatch")
        dh = None
        if diag is not None:
            d = diag.detach().cpu().numpy() if _is_torch(diag) else diag
            dh = np.ascontiguousarray(d, np.float64)
            if dh.size != n:
                raise ValueError("cg: diagonal length mismatch")  # solver.hpp:97
        rc = _lib.lib().hexbp_pcg_host(op.setup()._h, ws._h, b.ctypes.data_as(_dp), x.ctypes.data_as(_dp),
                                       dh.ctypes.data_as(_dp) if dh is not None else None, n, rel_tol, max_iter,
                                       constrained, C.byref(rep), hist.ctypes.data_as(_dp))
    _check(rc)
    return CGReport(rep.iterations, bool(rep.converged), rep.final_rel_residual, hist[: rep.iterations + 1].copy(),
                    time.perf_counter() - t0)


def jacobi_diagonal(op, device: bool = True):
    """jacobi_diagonal (solver.hpp:155-205) of an OperatorHandle, or of a
    ConstrainedOperator (1 on the essential dofs), computed on the GPU in the
    reference's arithmetic (bit for bit). Returns a device tensor, or a numpy
    array with device=False."""
    import torch

    if isinstance(op, ConstrainedOperator):
        raw, constrained = op.raw(), 1
    elif isinstance(op, OperatorHandle):
        raw, constrained = op, 0
    else:
        raise TypeError("jacobi_diagonal: expected an OperatorHandle or ConstrainedOperator")
    setup = raw.setup()
    d = torch.empty(raw.size(), dtype=torch.float64, device=torch.device("cuda", setup.device))
    _check(_lib.lib().hexbp_jacobi_diagonal(setup._h, constrained, C.c_void_p(d.data_ptr()), _stream_ptr(d)))
    return d if device else d.cpu().numpy()


def bench_rhs(kind, p: int, dims, seed: int = 20240101, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
    """run_bench's right-hand side (bench.hpp:234-243) for the (kind, p, dims) box."""
    g = [d * p + 1 for d in dims]
    n = g[0] * g[1] * g[2]
    count = n - offset if count is None else count
    out = np.empty(count)
    _check(_lib.lib().hexbp_bench_rhs(int(BPKind(kind)), p, _i3(dims), C.c_uint64(seed), offset, count,
                                      out.ctypes.data_as(_dp)))
    return out


def device_count() -> int:
    return int(_lib.lib().hexbp_device_count())
