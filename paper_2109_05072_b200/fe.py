"""Finite-element helpers around the hot path (solver.hpp:207-300), on the
device: the pieces of the manufactured-solution Poisson check (acceptance
criterion 5, proj/tests/acceptance/acceptance_main.cpp:181-222).

User functions are evaluated by torch on device tensors of the mapped
quadrature points, the way the reference's templates take a callable
``f(x, y, z)``; everything else (node coordinates, interpolation to the
quadrature points, the transposed interpolation with scatter_add) runs in
the reference's arithmetic through the C ABI (fe_tools.cu).
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from .api import HexMesh, OperatorSetup, _check, _stream_ptr, boundary_nodes


def _torch():
    import torch

    return torch


def _dev(setup: OperatorSetup):
    return _torch().device("cuda", setup.device)


def node_coords(setup: OperatorSetup):
    """mesh.coords of a box setup (mesh.hpp:107-119) as a (3, l_size) device
    tensor, bitwise the reference's values."""
    torch = _torch()
    out = torch.empty(3 * setup.l_size(), dtype=torch.float64, device=_dev(setup))
    _check(_lib.lib().hexbp_setup_node_coords(setup._h, C.c_void_p(out.data_ptr()), _stream_ptr(out)))
    return out.view(3, setup.l_size())


def interp_to_qpts(setup: OperatorSetup, v):
    """gather + elem_interp of an L-vector: (E, q^3) values at the quadrature points."""
    torch = _torch()
    v = v.contiguous()
    q3 = setup.q ** 3
    out = torch.empty(setup.num_elements() * q3, dtype=torch.float64, device=_dev(setup))
    _check(_lib.lib().hexbp_interp_to_qpts(setup._h, C.c_void_p(v.data_ptr()), C.c_void_p(out.data_ptr()),
                                           _stream_ptr(out)))
    return out.view(setup.num_elements(), q3)


def interp_transpose(setup: OperatorSetup, vq):
    """elem_interp_transpose + scatter_add of (E, q^3) quadrature values -> L-vector."""
    torch = _torch()
    vq = vq.contiguous()
    out = torch.empty(setup.l_size(), dtype=torch.float64, device=_dev(setup))
    _check(_lib.lib().hexbp_interp_transpose(setup._h, C.c_void_p(vq.data_ptr()), C.c_void_p(out.data_ptr()),
                                             _stream_ptr(out)))
    return out


def factors_device(setup: OperatorSetup):
    """The setup's factors in the reference AoS layout (E, q^3[, comp]) on the device."""
    torch = _torch()
    n = setup.num_elements() * setup.q ** 3 * setup.components
    out = torch.empty(n, dtype=torch.float64, device=_dev(setup))
    _check(_lib.lib().hexbp_setup_factors_device(setup._h, C.c_void_p(out.data_ptr()), _stream_ptr(out)))
    return out.view(setup.num_elements(), setup.q ** 3, setup.components).squeeze(-1)


def quadrature_points(setup: OperatorSetup):
    """Mapped quadrature points x_q (3 tensors of shape (E, q^3)): elem_interp
    of gather_coords (solver.hpp:229-233)."""
    X = node_coords(setup)
    return tuple(interp_to_qpts(setup, X[c]) for c in range(3))


def _mass_check(mass: OperatorSetup, setup: OperatorSetup, who: str):
    if mass.components != 1:
        raise ValueError(f"{who}: mass factors required")  # solver.hpp:213, 265
    if (mass.p, mass.q, mass.dims) != (setup.p, setup.q, setup.dims):
        raise ValueError(f"{who}: mass factors must use the operator's basis and mesh")


def assemble_load(mesh: HexMesh, setup: OperatorSetup, mass: OperatorSetup, f):
    """assemble_load (solver.hpp:207-239): b_i = sum_q wdetJ_q f(x_q) phi_i(x_q)
    with the basis of `setup`; `mass` = a BP1 setup on the same mesh (mass
    factors on that rule). `f(x, y, z)` acts on device tensors."""
    _mass_check(mass, setup, "assemble_load")
    xq = quadrature_points(setup)
    fq = factors_device(mass) * f(*xq)
    return interp_transpose(setup, fq)


def nodal_interpolant(setup: OperatorSetup, g):
    """nodal_interpolant (solver.hpp:241-247): g at the mesh nodes."""
    X = node_coords(setup)
    return g(X[0], X[1], X[2])


def discrete_l2_error(mesh: HexMesh, setup: OperatorSetup, mass: OperatorSetup, u_h, g) -> float:
    """discrete_l2_error (solver.hpp:256-300): sqrt(sum_e sum_q wdetJ (u_h(x_q) - g(x_q))^2),
    per-element sums in point order, elements summed in index order."""
    torch = _torch()
    _mass_check(mass, setup, "discrete_l2_error")
    if not torch.is_tensor(u_h):
        u_h = torch.as_tensor(u_h, dtype=torch.float64, device=_dev(setup))
    xq = quadrature_points(setup)
    d = interp_to_qpts(setup, u_h) - g(*xq)
    per_elem = (factors_device(mass) * d * d).sum(dim=1)
    return float(torch.sqrt(per_elem.sum()).item())


def boundary_mask(mesh: HexMesh, setup: OperatorSetup):
    """Boolean device L-vector of the box-surface nodes (mesh.hpp:126-135)."""
    torch = _torch()
    m = torch.zeros(setup.l_size(), dtype=torch.bool, device=_dev(setup))
    m[torch.as_tensor(boundary_nodes(mesh), dtype=torch.long, device=_dev(setup))] = True
    return m
