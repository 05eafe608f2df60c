"""Multi-rank (world_size 2 and 3) tests of the z-slab partition on CPU with
the gloo backend: the product orchestration (paper_2109_05072_b200/parallel.py:
partition, interface-plane halo sum, owned-range reductions, rank-order CG
scalars) driven with the oracle slab problem as the local operator
(tests/dist_cpu_ops.py), checked against the single-domain oracle."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_cpu_ops import OracleSlabOps

        import oracle
        from paper_2109_05072_b200.parallel import Comm, DistributedOperator, SlabPartition, dist_cg

        bp, p, gdims, a = case
        part = SlabPartition(gdims, p, world, rank)
        comm = Comm()
        ops = OracleSlabOps(bp, p, gdims, part, a)
        dop = DistributedOperator(part, comm, ops)
        glob = oracle.Oracle(bp, p, gdims, a)
        u_g = oracle.random_vector(99, glob.n)
        sl = slice(part.global_offset, part.global_offset + part.n_local)
        res = {}
        for constrained in (False, True):
            w = torch.zeros(part.n_local, dtype=torch.float64)
            dop.apply(torch.from_numpy(u_g[sl].copy()), w, constrained)
            ref = glob.apply(u_g, constrained)[sl]
            res[f"apply{int(constrained)}"] = float(np.abs(w.numpy() - ref).max() / np.abs(ref).max())
        b_g = glob.bench_rhs()
        x = torch.zeros(part.n_local, dtype=torch.float64)
        rep = dist_cg(dop, torch.from_numpy(b_g[sl].copy()), x, rel_tol=1e-8, max_iter=500, constrained=bp != 1)
        ref = glob.cg(b_g, rel_tol=1e-8, max_iter=500, constrained=bp != 1)
        res.update(iters=rep.iterations, ref_iters=ref["iterations"], final=rep.final_rel_residual,
                   ref_final=ref["final_rel_residual"],
                   xerr=float(np.abs(x.numpy() - ref["x"][sl]).max() / np.abs(ref["x"]).max()),
                   owned=part.owned_global_range())
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return results


@pytest.mark.parametrize("world,case", [
    (2, (3, 2, (3, 2, 4), 0.1)),
    (3, (3, 3, (2, 2, 5), 0.05)),
    (2, (5, 2, (2, 3, 3), 0.1)),
    (2, (1, 2, (2, 2, 3), 0.1)),
])
def test_slab_partition_matches_single_domain(world, case):
    res = _run(world, case)
    bp, p, gdims, a = case
    n_global = (gdims[0] * p + 1) * (gdims[1] * p + 1) * (gdims[2] * p + 1)
    # owned ranges tile the global L-vector exactly once
    spans = sorted(r["owned"] for r in res.values())
    assert spans[0][0] == 0 and spans[-1][1] == n_global
    assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))
    for r in res.values():
        assert r["apply0"] < 1e-14 and r["apply1"] < 1e-14
        # every rank runs the identical scalar recurrence
        assert r["iters"] == res[0]["iters"] and r["final"] == res[0]["final"]
        # iteration count of the single domain; the slab
        # reductions group the sums per rank, so iterates agree to
        # rounding-level drift (cf. tools/parity_diag.py), not bitwise: the
        # count may move by one when the reference stops within a hair of tol.
        assert abs(r["iters"] - r["ref_iters"]) <= 1
        if r["iters"] == r["ref_iters"]:
            assert abs(r["final"] - r["ref_final"]) < 5e-10
        assert r["xerr"] < 1e-8


def test_partition_bookkeeping():
    from paper_2109_05072_b200.parallel import SlabPartition

    for ez, world in [(13, 8), (105, 8), (8, 8), (66, 4)]:
        parts = [SlabPartition((4, 3, ez), 7, world, r) for r in range(world)]
        assert sum(pt.nzl for pt in parts) == ez
        assert max(pt.nzl for pt in parts) - min(pt.nzl for pt in parts) <= 1
        for a, b in zip(parts, parts[1:]):
            assert a.z1 == b.z0
            # the top plane of a is the bottom plane of b
            assert a.global_offset + a.n_local - a.plane == b.global_offset
    with pytest.raises(ValueError):
        SlabPartition((2, 2, 3), 2, 4, 0)
