"""Multi-GPU z-slab partition of the BP operator and CG.

The reference is single-address-space; this is the B200
scale-out of its hot path: one process per GPU, the box's element layers split
into contiguous z-slabs, NCCL over NVLink for the two exchange steps the
operator and CG actually have:

* **halo sum** -- after the local (slab) apply, the node plane shared by two
  neighbouring slabs holds each rank's partial sum. Ranks swap those planes
  (one send + one recv per neighbour) and add them; IEEE addition commutes,
  so both copies are bitwise identical (no ownership fix-up needed).
* **CG scalars** -- every inner product is reduced by each rank over the
  nodes it owns (a shared plane is owned by the lower rank) in
  deterministic_dot order, the per-rank partials are all-gathered and summed
  in rank order on every rank, so all ranks run the identical scalar
  recurrence (same alpha, beta, stopping decision) on the device.

The orchestration below is backend-agnostic: ``Comm`` runs on
torch.distributed (NCCL for CUDA tensors; gloo with host staging), and the
compute primitives are an ``ops`` object -- ``CudaSlabOps`` (the C ABI,
product path) or a CPU double used by the world_size-2 gloo tests.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .api import CGReport, _check, _i3, BPKind, build_box_mesh, make_slab_setup, Workspace

HEXBP_CGD_INIT, HEXBP_CGD_PAP, HEXBP_CGD_UPDATE_R = 0, 1, 2
ST_RUNNING, ST_CONVERGED, ST_DIVERGED, ST_MAXITER = 0, 1, 2, 3


@dataclass
class SlabPartition:
    """Element layers [z0, z1) of a global (ex, ey, ez) box on rank `rank`."""

    gdims: tuple
    p: int
    world: int
    rank: int

    def __post_init__(self):
        ez = self.gdims[2]
        if ez < self.world:
            raise ValueError(f"cannot split {ez} element layers over {self.world} ranks")
        base, rem = divmod(ez, self.world)
        self.z0 = self.rank * base + min(self.rank, rem)
        self.nzl = base + (1 if self.rank < rem else 0)
        self.z1 = self.z0 + self.nzl
        self.Nx = self.gdims[0] * self.p + 1
        self.Ny = self.gdims[1] * self.p + 1
        self.plane = self.Nx * self.Ny
        self.n_local = self.plane * (self.nzl * self.p + 1)
        self.n_global = self.plane * (ez * self.p + 1)
        self.global_offset = self.plane * self.z0 * self.p  # global index of local node 0
        self.owned_offset = self.plane if self.rank > 0 else 0  # bottom plane belongs to the rank below
        self.has_up = self.rank + 1 < self.world
        self.has_down = self.rank > 0

    def owned_global_range(self):
        return self.global_offset + self.owned_offset, self.global_offset + self.n_local


class Comm:
    """Neighbour plane exchange and scalar all-gather on torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)
        self.host_staging = self.backend != "nccl"

    def _stage(self, t):
        return t.cpu() if (self.host_staging and t.is_cuda) else t

    def exchange_planes(self, send_up, send_down, recv_up, recv_down):
        """send_up -> rank+1, recv_up <- rank+1; send_down -> rank-1, recv_down <- rank-1."""
        dist = self.dist
        ops, post = [], []
        if send_up is not None:
            su, ru = self._stage(send_up), self._stage(recv_up)
            ops += [dist.P2POp(dist.isend, su, self.rank + 1, self.group), dist.P2POp(dist.irecv, ru, self.rank + 1,
                                                                                      self.group)]
            if ru is not recv_up:
                post.append((recv_up, ru))
        if send_down is not None:
            sd, rd = self._stage(send_down), self._stage(recv_down)
            ops += [dist.P2POp(dist.isend, sd, self.rank - 1, self.group), dist.P2POp(dist.irecv, rd, self.rank - 1,
                                                                                      self.group)]
            if rd is not recv_down:
                post.append((recv_down, rd))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for dst, src in post:
            dst.copy_(src)

    def allgather_scalar(self, t):
        """[world] tensor of every rank's 1-element `t`, in rank order."""
        import torch

        src = self._stage(t)
        if src.is_cuda:  # NCCL: one collective straight into the gathered vector
            out = torch.empty(self.world * src.numel(), dtype=src.dtype, device=src.device)
            self.dist.all_gather_into_tensor(out, src, group=self.group)
            return out
        outs = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(outs, src, group=self.group)
        out = torch.cat(outs)
        return out.to(t.device) if out.device != t.device else out

    def max_scalar(self, v: float) -> float:
        import torch

        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


class CudaSlabOps:
    """Product compute primitives of one rank (C ABI, device tensors)."""

    def __init__(self, kind, mesh, part: SlabPartition, device: int, mode: str = "fast"):
        import torch

        self.torch = torch
        self.part = part
        self.device = torch.device("cuda", device)
        self.setup = make_slab_setup(kind, mesh, part.z0, part.z1, device=device)
        if self.setup.l_size() != part.n_local:
            raise RuntimeError("slab setup size mismatch")
        self.ws = Workspace(self.setup)
        self.ws.set_mode(mode)
        r, p, ap = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(_lib.lib().hexbp_workspace_vectors(self.ws._h, C.byref(r), C.byref(p), C.byref(ap)))
        self._ptr = {"r": r.value, "p": p.value, "Ap": ap.value}
        self.partial = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.partial2 = torch.zeros(1, dtype=torch.float64, device=self.device)
        # fast mode: the fused iteration (operator with p.Ap, ring-summing r-update)
        self.fused = mode == "fast"

    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def view(self, name):
        """Zero-copy torch view of a workspace CG vector ('r', 'p' or 'Ap')."""
        return self.torch.as_tensor(_CudaArray(self._ptr[name], self.part.n_local), device=self.device)

    def apply_partial(self, u, w, constrained):
        _check(_lib.lib().hexbp_apply(self.setup._h, self.ws._h, C.c_void_p(_addr(u)), C.c_void_p(_addr(w)),
                                      int(constrained), self._stream()))

    def plane_combine(self, dst, src, u, constrained):
        _check(_lib.lib().hexbp_plane_combine(C.c_void_p(_addr(dst)), C.c_void_p(_addr(src)),
                                              C.c_void_p(_addr(u)), self.part.Nx, self.part.Ny, int(constrained),
                                              self._stream()))

    def reduce(self, op, b=None):
        _check(_lib.lib().hexbp_cgd_reduce(self.ws._h, op, C.c_void_p(_addr(b) if b is not None else None),
                                           self.part.owned_offset, C.c_void_p(self.partial.data_ptr()),
                                           self._stream()))
        return self.partial

    def finish(self, op, gathered, world, rel_tol, max_iter):
        _check(_lib.lib().hexbp_cgd_finish(self.ws._h, op, C.c_void_p(gathered.data_ptr()), world, rel_tol, max_iter,
                                           self._stream()))

    def apply_fused(self, constrained):
        """Ap = A p (workspace p) with this rank's p.Ap share -> self.partial;
        shared planes locally assembled in Ap for the halo."""
        _check(_lib.lib().hexbp_cgd_apply_fused(self.setup._h, self.ws._h, int(constrained),
                                                C.c_void_p(self.partial.data_ptr()), self._stream()))
        return self.partial

    def update_r_fused(self, constrained):
        _check(_lib.lib().hexbp_cgd_update_r_fused(self.ws._h, int(constrained),
                                                   C.c_void_p(self.partial2.data_ptr()), self._stream()))
        return self.partial2

    def update_xp(self, x):
        _check(_lib.lib().hexbp_cgd_update_xp(self.ws._h, C.c_void_p(_addr(x)), self._stream()))

    def status(self):
        st = C.c_int(0)
        _lib.lib().hexbp_cgd_report(self.ws._h, C.byref(st), None, None, 0)
        return st.value

    def report(self, max_iter):
        st = C.c_int(0)
        rep = _lib.CGReportC()
        hist = np.zeros(max_iter + 1)
        rc = _lib.lib().hexbp_cgd_report(self.ws._h, C.byref(st), C.byref(rep), hist.ctypes.data_as(
            C.POINTER(C.c_double)), max_iter + 1)
        _check(rc)
        return CGReport(rep.iterations, bool(rep.converged), rep.final_rel_residual, hist[: rep.iterations + 1], 0.0)


class _CudaArray:
    """__cuda_array_interface__ wrapper of a library-owned device vector."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def _addr(t):
    return t.data_ptr()


class NcclSlabOperator:
    """The product multi-GPU path: this rank's z-slab operator and CG in the
    library (hexbp_dist_*, include/hexbp_b200.h), which owns the NCCL
    communicator and overlaps the shared-plane exchange with the interior
    element layers (dist.cu, overlap.cu). Rank 0 makes the NCCL id; it is
    broadcast over torch.distributed (any backend) when world > 1.
    Mirrors hexbp::b200::DistributedOperator (include/hexbp_b200.hpp)."""

    def __init__(self, kind, p: int, gdims, world: int = 1, rank: int = 0, device: int = 0,
                 amplitude: float = 0.0, extent=(1.0, 1.0, 1.0), overlap: bool = True, mode: str = "fast"):
        if gdims[2] < world:
            raise ValueError(f"cannot split {gdims[2]} element layers over {world} ranks")
        idb = C.create_string_buffer(128)
        if rank == 0:
            _check(_lib.lib().hexbp_dist_unique_id(idb, 128))
        if world > 1:
            import torch.distributed as dist

            obj = [idb.raw if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            idb = C.create_string_buffer(obj[0], 128)
        h = C.c_void_p()
        ext = np.asarray(extent, np.float64)
        _check(_lib.lib().hexbp_dist_create_box(int(BPKind(kind)), p, _i3(gdims), ext.ctypes.data_as(
            C.POINTER(C.c_double)), amplitude, world, rank, device, idb, 128, 0 if overlap else 1, C.byref(h)))
        self._h = h
        n, own, off = C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.lib().hexbp_dist_info(self._h, None, None, None, C.byref(n), C.byref(own), C.byref(off)))
        self.n_local, self.owned_offset, self.global_offset = n.value, own.value, off.value
        self.world, self.rank, self.device = world, rank, device
        self.set_mode(mode)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().hexbp_dist_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def set_mode(self, mode: str) -> None:
        _check(_lib.lib().hexbp_dist_set_mode(self._h, {"reference": 0, "fast": 1}[mode]))

    def _stream(self):
        import torch

        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def apply(self, u, w, constrained: bool = False):
        """w = the assembled local part of A u (device tensors); collective."""
        _check(_lib.lib().hexbp_dist_apply(self._h, C.c_void_p(u.data_ptr()), C.c_void_p(w.data_ptr()),
                                           int(constrained), self._stream()))
        return w

    def cg(self, b, x, rel_tol: float = 1e-8, max_iter: int = 2000, constrained: bool = True) -> CGReport:
        """cg (solver.hpp:91-153) on the partition (device tensors; x holds x0);
        every rank returns the same report; collective."""
        rep = _lib.CGReportC()
        hist = np.zeros(max_iter + 1)
        t0 = time.perf_counter()
        _check(_lib.lib().hexbp_dist_cg(self._h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), rel_tol, max_iter,
                                        int(constrained), C.byref(rep), hist.ctypes.data_as(C.POINTER(C.c_double)),
                                        self._stream()))
        return CGReport(rep.iterations, bool(rep.converged), rep.final_rel_residual, hist[: rep.iterations + 1].copy(),
                        time.perf_counter() - t0)


class DistributedOperator:
    """OperatorHandle semantics on a z-slab partition: apply() returns the
    fully assembled local part of A u (interface planes halo-summed)."""

    def __init__(self, part: SlabPartition, comm: Comm, ops):
        self.part, self.comm, self.ops = part, comm, ops
        import torch

        dev = getattr(ops, "device", "cpu")
        self._rup = torch.empty(part.plane, dtype=torch.float64, device=dev)
        self._rdown = torch.empty(part.plane, dtype=torch.float64, device=dev)

    def _plane(self, v, top: bool):
        pl, n = self.part.plane, self.part.n_local
        return v[n - pl:] if top else v[:pl]

    def apply(self, u, w, constrained: bool = False):
        self.ops.apply_partial(u, w, constrained)
        self.halo(u, w, constrained)
        return w

    def halo(self, u, w, constrained: bool):
        part = self.part
        if part.world == 1:
            return
        up = self._plane(w, True) if part.has_up else None
        down = self._plane(w, False) if part.has_down else None
        # no send copies: exchange_planes waits for its sends (NCCL: the
        # current stream is ordered after them; gloo: host-staged), so the
        # in-place combines below cannot race them
        self.comm.exchange_planes(up, down, self._rup if up is not None else None,
                                  self._rdown if down is not None else None)
        if up is not None:
            self.ops.plane_combine(up, self._rup, self._plane(u, True), constrained)
        if down is not None:
            self.ops.plane_combine(down, self._rdown, self._plane(u, False), constrained)


def dist_cg(dop: DistributedOperator, b, x, rel_tol: float = 1e-8, max_iter: int = 2000,
            constrained: bool = True, check_every: int = 8) -> CGReport:
    """cg (solver.hpp:91-153) on the slab partition; every rank returns the
    same report. b, x: this rank's local vectors (x holds x0)."""
    ops, comm = dop.ops, dop.comm
    t0 = time.perf_counter()
    Ap = ops.view("Ap")
    p = ops.view("p")
    dop.apply(x, Ap, constrained)  # r0 = b - A x0
    ops.finish(HEXBP_CGD_INIT, comm.allgather_scalar(ops.reduce(HEXBP_CGD_INIT, b)), comm.world, rel_tol, max_iter)
    fused = getattr(ops, "fused", False)
    for k in range(1, max_iter + 1):
        if fused:
            # the single-GPU fast iteration split at its two reductions: p.Ap
            # inside the operator kernel, ring sums inside the r-update
            pap = ops.apply_fused(constrained)
            dop.halo(p, Ap, constrained)
            ops.finish(HEXBP_CGD_PAP, comm.allgather_scalar(pap), comm.world, rel_tol, max_iter)
            rr = ops.update_r_fused(constrained)
            ops.finish(HEXBP_CGD_UPDATE_R, comm.allgather_scalar(rr), comm.world, rel_tol, max_iter)
        else:
            dop.apply(p, Ap, constrained)
            ops.finish(HEXBP_CGD_PAP, comm.allgather_scalar(ops.reduce(HEXBP_CGD_PAP)), comm.world, rel_tol,
                       max_iter)
            ops.finish(HEXBP_CGD_UPDATE_R, comm.allgather_scalar(ops.reduce(HEXBP_CGD_UPDATE_R)), comm.world,
                       rel_tol, max_iter)
        ops.update_xp(x)
        if rel_tol > 0.0 and k % check_every == 0 and k < max_iter and ops.status() != ST_RUNNING:
            break
    rep = ops.report(max_iter)
    rep.seconds = time.perf_counter() - t0
    return rep


def bench_weak(bp: int, p: int, dims, K: int, W: int, amplitude: float = 0.0, clock=None) -> dict:
    """Weak scaling: each rank owns a dims-sized slab of a (ex, ey, world*ez) box.
    `clock`: optional context-manager factory sampling SM clocks around the
    timed region (bench.py's ClockSampler)."""
    import contextlib

    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group("nccl")
    comm = Comm()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    gdims = (dims[0], dims[1], dims[2] * comm.world)
    part = SlabPartition(gdims, p, comm.world, comm.rank)
    # the library's distributed solve (hexbp_dist_cg): NCCL communicator owned
    # by the library, plane exchange overlapped with the interior layers
    dop = NcclSlabOperator(bp, p, gdims, comm.world, comm.rank, local, amplitude)
    assert dop.n_local == part.n_local and dop.global_offset == part.global_offset
    from .api import bench_rhs

    b_host = torch.from_numpy(bench_rhs(bp, p, gdims, offset=part.global_offset, count=part.n_local))
    b = b_host.cuda(local)
    x = torch.zeros_like(b)
    dop.cg(b, x, 0.0, W, constrained=bp != 1)
    x.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with (clock() if clock else contextlib.nullcontext()) as clk:
        ev0.record()
        rep = dop.cg(b, x, 0.0, K, constrained=bp != 1)
        ev1.record()
        torch.cuda.synchronize()
    dist.barrier()
    t = comm.max_scalar(ev0.elapsed_time(ev1) / 1e3)
    value = part.n_global * K / t / 1e9

    # end to end with host buffers: this rank's b slice in (pinned), x out, copies timed
    bh = b_host.pin_memory()
    xh = torch.empty(part.n_local, dtype=torch.float64).pin_memory()
    x.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    ev0.record()
    b.copy_(bh, non_blocking=True)
    dop.cg(b, x, 0.0, K, constrained=bp != 1)
    xh.copy_(x, non_blocking=True)
    ev1.record()
    torch.cuda.synchronize()
    dist.barrier()
    te = comm.max_scalar(ev0.elapsed_time(ev1) / 1e3)
    planes = int(part.has_up) + int(part.has_down)
    # our kernels per fused iteration: operator (overlapped: two boundary launches,
    # the interior launch and the carry combine), shared-plane ring sums and halo
    # combines, finish(PAP), r-update, finish(UPDATE_R), x/p update; plus the
    # initial residual (operator, ring fix-up, plane combines, reduce, finish)
    op_launches = 4 if (bp == 3 and p == 7 and dims[2] >= 2) else 1
    launches = K * (op_launches + 4 + 2 * planes) + 4 + planes
    return {
        "metric": "BP3 GDOF/s (DOFs x CG iters/sec), fp64, % HBM roofline", "value": value, "unit": "GDOF/s",
        "n_gpus": comm.world, "steps": K, "warmup": W, "ms_per_step": t / K * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference bench RHS slice per rank; device-generated box mesh)",
        "config": {"workload": f"bp{bp} Q_{p}: {dims[0]}x{dims[1]}x{dims[2]} elements per GPU, global box "
                               f"{gdims[0]}x{gdims[1]}x{gdims[2]}, {part.n_global} DOFs, {K} fixed CG iterations",
                   "bp": bp, "p": p, "dims_per_gpu": list(dims), "global_dims": list(gdims),
                   "parallelism": f"z-slab x{comm.world}, hexbp_dist_cg: NCCL plane exchange overlapped with the "
                                  f"interior layers + scalar all-gathers, fused CG iteration",
                   "l2": "inputs larger than L2"},
        "e2e": {"value": part.n_global * K / te / 1e9, "unit": "GDOF/s",
                "h2d_bytes_per_step": part.n_global * 8 / K, "d2h_bytes_per_step": part.n_global * 8 / K,
                "path": "hexbp_dist_cg per rank: pinned b slice in, x slice out, copies inside the timed region"},
        "gpu_launches": launches,
        "clocks": clk.summary() if clk is not None and hasattr(clk, "summary") else None,
        "cg_report": {"iterations": rep.iterations, "final_rel_residual": rep.final_rel_residual},
    }
