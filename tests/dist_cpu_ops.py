"""TEST DOUBLE of parallel.CudaSlabOps for the world_size > 1 gloo tests on
CPU: the same primitive semantics (cgd reduce / finish / update_xp, plane
combine), with the oracle slab problem as the local operator. The
orchestration under test (partition, halo exchange, owned-range reductions,
rank-order combination, CG control flow) is the product's parallel.py."""
import math

import numpy as np
import torch

import oracle

INIT, PAP, UPDATE_R = 0, 1, 2
RUNNING, CONVERGED, DIVERGED, MAXITER = 0, 1, 2, 3


class OracleSlabOps:
    def __init__(self, bp, p, gdims, part, amplitude=0.0):
        self.part = part
        self.device = torch.device("cpu")
        self.o = oracle.OracleSlab(bp, p, gdims, part.z0, part.z1, amplitude)
        assert self.o.n == part.n_local
        n = part.n_local
        self.vec = {k: torch.zeros(n, dtype=torch.float64) for k in ("r", "p", "Ap")}
        self.partial = torch.zeros(1, dtype=torch.float64)
        self.sc = {}
        self.hist = []

    def view(self, name):
        return self.vec[name]

    def apply_partial(self, u, w, constrained):
        w.copy_(torch.from_numpy(self.o.apply(u.numpy(), constrained)))

    def plane_combine(self, dst, src, u, constrained):
        nx, ny = self.part.Nx, self.part.Ny
        out = dst + src
        if constrained:
            X = torch.arange(nx * ny) % nx
            Y = torch.arange(nx * ny) // nx
            edge = (X == 0) | (X == nx - 1) | (Y == 0) | (Y == ny - 1)
            out = torch.where(edge, u, out)
        dst.copy_(out)

    def _owned_dot(self, a, b):
        a = a.numpy().copy()
        a[: self.part.owned_offset] = 0.0  # products of non-owned entries enter as +-0.0
        return oracle.dot(a, b.numpy())

    def reduce(self, op, b=None):
        r, p, Ap = self.vec["r"], self.vec["p"], self.vec["Ap"]
        if op == INIT:
            r.copy_(b - Ap)
            p.copy_(r)
            v = self._owned_dot(r, r)
        elif op == PAP:
            if self.sc["status"] != RUNNING:
                return self.partial
            v = self._owned_dot(p, Ap)
        else:
            if self.sc["status"] != RUNNING:
                return self.partial
            r.copy_(r - self.sc["alpha"] * Ap)
            v = self._owned_dot(r, r)
        self.partial[0] = v
        return self.partial

    def finish(self, op, gathered, world, rel_tol, max_iter):
        sc = self.sc
        if op != INIT and sc["status"] != RUNNING:
            return
        tot = 0.0
        for k in range(world):
            tot += float(gathered[k])
        if op == INIT:
            r0 = math.sqrt(tot)
            self.hist = [r0]
            sc.update(r0=r0, rz=tot, iterations=0, x_pending=0, rel_tol=rel_tol, max_iter=max_iter)
            sc["status"] = DIVERGED if not math.isfinite(r0) else (CONVERGED if r0 == 0 else RUNNING)
        elif op == PAP:
            if not math.isfinite(tot) or tot <= 0:
                sc["status"] = DIVERGED
            else:
                sc["alpha"] = sc["rz"] / tot
        else:
            rn = math.sqrt(tot)
            sc["iterations"] += 1
            self.hist.append(rn)
            sc["x_pending"] = 1
            if not math.isfinite(rn):
                sc["status"] = DIVERGED
            elif rn / sc["r0"] <= sc["rel_tol"]:
                sc["status"] = CONVERGED
            else:
                sc["beta"] = tot / sc["rz"]
                sc["rz"] = tot
                if sc["iterations"] >= sc["max_iter"]:
                    sc["status"] = MAXITER

    def update_xp(self, x):
        sc = self.sc
        if not sc.get("x_pending"):
            return
        p, r = self.vec["p"], self.vec["r"]
        x.add_(sc["alpha"] * p)
        if sc["status"] == RUNNING:
            p.copy_(r + sc["beta"] * p)
        sc["x_pending"] = 0

    def status(self):
        return self.sc["status"]

    def report(self, max_iter):
        from paper_2109_05072_b200.api import CGReport

        h = np.array(self.hist)
        return CGReport(self.sc["iterations"], self.sc["status"] == CONVERGED, h[-1] / h[0] if h[0] else 0.0, h, 0.0)
