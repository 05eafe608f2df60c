#!/usr/bin/env python
"""Benchmark: BP3 GDOF/s (DOFs x CG iterations / s) of the device-resident CG
on the reference's bench problem, plus the HBM-roofline fraction of the fused
operator kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--bp 3] [--p 7] [--dims 66,66,66]

A "step" is one CG iteration (operator apply + fused vector updates) over the
whole mesh; the timed region is one fixed-iteration solve of K iterations
(rel_tol = 0, exactly the reference's run_bench protocol, bench.hpp:251-267,
including the initial residual), inputs already resident in HBM. Default
workload = BASELINE config 3: BP3, Q_7, 66^3 elements, 99,252,847 DOFs, fp64.
The geometric factors (10 GB) exceed L2 (126 MB), so every timed iteration
streams from HBM (no L2 flush needed).

N > 1 (torchrun, one rank per GPU): weak scaling; rank r owns the z-slab
[r*ez, (r+1)*ez) of a (ex, ey, N*ez) box; the interface-plane halo sum and the
CG dot products go over NCCL (paper_2109_05072_b200/parallel.py).

--impl reference times the reference's own CPU implementation (the
unmodified headers compiled in place, oracle/_ref) on this host's cores with
all threads, on a bounded sample of the same workload (same bp/p, smaller mesh).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BP3 GDOF/s (DOFs x CG iters/sec), fp64, % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--bp", type=int, default=3)
    ap.add_argument("--p", type=int, default=7)
    ap.add_argument("--dims", default=None, help="ex,ey,ez per GPU (default 66,66,66 for p=7)")
    ap.add_argument("--amplitude", type=float, default=0.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="run the multi-GPU (hexbp_dist_cg) path even at N = 1 (single-GPU box check of that path)")
    return ap.parse_args()


def default_dims(p: int):
    # ~100M DOFs per GPU: (e*p+1)^3 <= 1e8 (auto_size_dims, bench.hpp:179-187)
    e = 1
    while ((e + 1) * p + 1) ** 3 <= 100_000_000:
        e += 1
    return (e, e, e)


def kernel_sources_sha(files) -> str:
    """Hash stamp of the kernel sources a profile was captured on (profiles/traffic.json)."""
    import hashlib

    h = hashlib.sha256()
    for f in files:
        h.update(open(os.path.join(ROOT, "paper_2109_05072_b200", "csrc", f), "rb").read())
    return h.hexdigest()[:16]


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(bp: int, p: int, dims):
    """per apply 8(c E q^3 + 2 n_L); per CG iteration 8(c E q^3 + 10 n_L)."""
    q = p + 1 if bp == 5 else p + 2
    c = 1 if bp == 1 else 6
    E = dims[0] * dims[1] * dims[2]
    nL = (dims[0] * p + 1) * (dims[1] * p + 1) * (dims[2] * p + 1)
    return 8 * (c * E * q**3 + 2 * nL), 8 * (c * E * q**3 + 10 * nL), nL, E


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML every
    10 ms (a timed region of 20 CG iterations lasts ~0.1 s), nvidia-smi if NVML
    is unavailable."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, sm_max_mhz, [reasons])
        self._stop = threading.Event()
        self._t = None

    def _sample_nvml(self):
        import pynvml as N

        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        bits = {"hw_slowdown": N.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": N.nvmlClocksThrottleReasonSwPowerCap}
        while not self._stop.is_set():
            sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.rows.append((float(sm), float(mx), [k for k, b in bits.items() if r & b]))
            self._stop.wait(0.01)

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            f = [x.strip() for x in out.split(",")]
            if len(f) >= 6 and f[0].replace(".", "").isdigit():
                self.rows.append((float(f[0]), float(f[1]),
                                  [names[i] for i in range(4) if "Active" in f[2 + i] and "Not" not in f[2 + i]]))
            self._stop.wait(0.05)

    def _run(self):
        try:
            self._sample_nvml()
        except Exception:
            try:
                self._sample_smi()
            except Exception:
                pass

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({x for r in self.rows for x in r[2]}), "samples": len(self.rows)}


def cpu_baseline(bp: int, p: int, iters: int = 20, warmup: int = 1, repeats: int = 3, cfg1: bool = True) -> dict:
    """The reference's own run_bench (oracle/_ref, unmodified headers compiled in
    place) on this host as BASELINE.md section 2 plans it: same bp/p at ~10M DOFs,
    `iters` fixed CG iterations, OMP_NUM_THREADS = physical cores with
    OMP_PROC_BIND=close / OMP_PLACES=cores, plus BASELINE configs[0] in full
    (cfg1). Run in a subprocess so the OpenMP settings take effect."""
    import oracle
    from oracle import cpu_baseline as cb

    oracle.build()
    cores = cb.physical_cores()
    env = dict(os.environ, OMP_NUM_THREADS=str(cores), OMP_PROC_BIND="close", OMP_PLACES="cores")
    cmd = [sys.executable, "-m", "oracle.cpu_baseline", "--bp", str(bp), "--p", str(p), "--iters", str(iters),
           "--warmup", str(warmup), "--repeats", str(repeats)] + (["--cfg1"] if cfg1 else [])
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    if out.returncode != 0:
        raise RuntimeError((out.stderr or out.stdout)[-300:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the reference's own CPU path on this host's cores: K fixed CG iterations
    # per solve (the steps), W warm-up solves, best of 3 timed solves, on the
    # ~10M-DOF sample of the same bp / p
    cb = cpu_baseline(args.bp, args.p, iters=args.steps, warmup=max(1, min(args.warmup, 3)), repeats=3, cfg1=False)
    dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else default_dims(args.p)
    hs = cb["headline_sample"]
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "GDOF/s", "n_gpus": args.gpus,
        "steps": hs["fixed_cg_iters"], "warmup": hs["warmup_solves"] * hs["fixed_cg_iters"],
        "ms_per_step": hs["best_solve_s"] / hs["fixed_cg_iters"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"bp{args.bp} p={args.p}: the ours arm runs {dims[0]}x{dims[1]}x{dims[2]} per GPU; "
                               f"this CPU arm a bounded sample of it ({cb['sample']})", "bp": args.bp, "p": args.p},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import ctypes as C

    import numpy as np
    import torch

    import paper_2109_05072_b200 as hx
    from paper_2109_05072_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    p, bp = args.p, args.bp
    dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else default_dims(p)
    K, W = args.steps, max(args.warmup, 3)
    L = _lib.lib()

    if world > 1 or args.dist:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        from paper_2109_05072_b200 import parallel

        res = parallel.bench_weak(bp, p, dims, K, W, args.amplitude, clock=lambda: ClockSampler(local))
        if rank != 0:
            return
        b_op, b_it, nL, E = algorithmic_bytes(bp, p, dims)  # per GPU (its slab)
        peak, peak_kind = load_peaks()
        t_it = res["ms_per_step"] / 1e3
        res["cg_iteration_roofline"] = {"algorithmic_bytes_per_iter_per_gpu": b_it,
                                        "achieved_GBps_per_gpu": b_it / t_it / 1e9,
                                        "frac": b_it / t_it / 1e9 / peak}
        res["roofline"] = {"bound": "hbm", "achieved": b_it / t_it / 1e9, "peak": peak, "unit": "GB/s",
                           "frac": b_it / t_it / 1e9 / peak, "traffic": None,
                           "note": "whole CG iteration per GPU (N > 1 runs time no separate kernel)",
                           "peak_source": f"{peak_kind} hbm_gbs"}
        print(json.dumps(res), flush=True)
        return

    # ------------------------------------------------------------ single GPU
    mesh = hx.build_box_mesh(dims, p, (1.0, 1.0, 1.0), args.amplitude)
    t0 = time.perf_counter()
    setup = hx.make_setup(hx.BPKind(bp), mesh, device=local)
    op = hx.OperatorHandle(hx.Backend.Cuda, setup)
    setup_s = time.perf_counter() - t0
    n = op.size()
    b_host = hx.bench_rhs(bp, p, dims)
    b = torch.from_numpy(b_host).to(dev)
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    A = hx.ConstrainedOperator(op) if bp != 1 else op
    st = torch.cuda.current_stream(dev)

    # warm-up solve, then the timed fixed-iteration solve (device-resident inputs).
    # Headline = fast mode (FMA/DMMA operator, fused p.Ap); reference mode
    # (bit-exact reference arithmetic) is timed beside it. Warm-ups run at
    # least one 8-iteration block (WG), so the solve's CUDA graph is captured
    # before the timed region (capi.cu pcg_run).
    WG = max(W, 8)
    hx.cg(A, b, x, rel_tol=0.0, max_iter=WG, mode="fast")
    x.zero_()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(st)
        rep = hx.cg(A, b, x, rel_tol=0.0, max_iter=K, mode="fast")
        ev1.record(st)
        torch.cuda.synchronize()
    t_dev = ev0.elapsed_time(ev1) / 1e3
    value = n * K / t_dev / 1e9
    x.zero_()
    hx.cg(A, b, x, rel_tol=0.0, max_iter=WG, mode="reference")
    x.zero_()
    torch.cuda.synchronize()
    ev0.record(st)
    rep_ref = hx.cg(A, b, x, rel_tol=0.0, max_iter=K, mode="reference")
    ev1.record(st)
    torch.cuda.synchronize()
    t_ref = ev0.elapsed_time(ev1) / 1e3
    op.workspace().set_mode("fast")

    # the dominant kernel alone: CUDA events around R back-to-back launches of
    # the operator kernel on the launch stream, in the form the CG runs it
    # (hexbp_apply_cg_form: ring nodes left as column partials for the
    # r-update, input = the workspace's search direction -- row-pitched and
    # TMA-staged on the DMMA degrees -- loaded once before the timed launches)
    u = torch.empty_like(b).uniform_(-1, 1)
    w = torch.empty_like(b)
    con = 1 if bp != 1 else 0
    sp = C.c_void_p(st.cuda_stream)
    assert L.hexbp_apply_cg_form(setup._h, op.workspace()._h, C.c_void_p(u.data_ptr()), C.c_void_p(w.data_ptr()),
                                 con, sp) == 0, L.hexbp_last_error()

    def kernel_once():
        rc = L.hexbp_apply_cg_form(setup._h, op.workspace()._h, None, C.c_void_p(w.data_ptr()), con, sp)
        assert rc == 0, L.hexbp_last_error()

    for _ in range(3):
        kernel_once()
    R = 10
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(st)
    for _ in range(R):
        kernel_once()
    eb.record(st)
    torch.cuda.synchronize()
    t_apply = ea.elapsed_time(eb) / 1e3 / R
    b_op, b_it, nL, E = algorithmic_bytes(bp, p, dims)
    peak, peak_kind = load_peaks()
    achieved = b_op / t_apply / 1e9
    # DRAM bytes per launch from the committed ncu capture -- used only if it was
    # taken on the kernel sources now built (hash stamp), else reported stale
    traffic, traffic_note = None, "no capture for this configuration"
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        tr = json.load(open(prof)).get(f"bp{bp}_p{p}_{dims[0]}x{dims[1]}x{dims[2]}")
        if tr:
            if tr.get("source_sha256_16") == kernel_sources_sha(tr.get("kernel_sources", [])):
                traffic, traffic_note = tr.get("dram_bytes_per_launch"), tr.get("source")
            else:
                traffic_note = "stale: the capture's kernel sources differ from the built ones"

    # end to end through the C ABI with host buffers (pinned), copies inside the timed region
    bh = torch.from_numpy(b_host).pin_memory()
    xh = torch.zeros(n, dtype=torch.float64).pin_memory()
    _dp = C.POINTER(C.c_double)
    repc = _lib.CGReportC()
    ws = op.workspace()
    ws.set_mode("fast")
    L.hexbp_cg_host(setup._h, ws._h, C.cast(bh.data_ptr(), _dp), C.cast(xh.data_ptr(), _dp), n, 0.0, WG,
                    1 if bp != 1 else 0, C.byref(repc), None)
    xh.zero_()
    torch.cuda.synchronize()
    te = time.perf_counter()
    rc = L.hexbp_cg_host(setup._h, ws._h, C.cast(bh.data_ptr(), _dp), C.cast(xh.data_ptr(), _dp), n, 0.0, K,
                         1 if bp != 1 else 0, C.byref(repc), None)
    te = time.perf_counter() - te
    assert rc == 0, L.hexbp_last_error()
    e2e = n * K / te / 1e9

    kinfo = ws.kernel_info()
    line = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": 1, "steps": K, "warmup": W, "warmup_iterations_run": WG,
        "ms_per_step": t_dev / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference bench RHS, bench.hpp:234-243; device-generated box mesh)",
        "config": {"workload": f"BP3-family bp{bp} Q_{p} box {dims[0]}x{dims[1]}x{dims[2]} elements, {n} DOFs, "
                               f"{K} fixed CG iterations (BASELINE configs[2])" if bp == 3 and p == 7 else
                               f"bp{bp} Q_{p} box {dims[0]}x{dims[1]}x{dims[2]}, {n} DOFs, {K} fixed CG iterations",
                   "bp": bp, "p": p, "q": setup.q, "dims": list(dims), "dofs": n, "elements": E,
                   "deform_amplitude": args.amplitude, "parallelism": "single GPU",
                   "l2": "inputs larger than L2 (factors %.2f GB)" % (setup.factor_bytes / 1e9)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_note,
                     "kernel": ("bp3_p7_mma_kernel (DMMA)" if (bp == 3 and p == 7) else "bp_apply_kernel") +
                               " (ring nodes as column partials, summed by the CG r-update)",
                     "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                     "algorithmic_bytes_per_launch": b_op, "kernel_ms": t_apply * 1e3},
        "cg_iteration_roofline": {"algorithmic_bytes_per_iter": b_it, "achieved_GBps": b_it * K / t_dev / 1e9,
                                  "frac": b_it * K / t_dev / 1e9 / peak,
                                  "roofline_GDOFps": peak * 1e9 / (b_it / nL) / 1e9},
        "e2e": {"value": e2e, "unit": "GDOF/s", "h2d_bytes_per_step": 2 * n * 8 / K, "d2h_bytes_per_step": n * 8 / K,
                "path": "hexbp_cg_host (C ABI, pinned host b/x; x0 in, then b in on a copy stream overlapping the initial "
                        "A x0; x out; per solve, amortised per step)"},
        # per CG iteration: operator, ring-summing r-update, x/p update; plus the
        # preconditioner flag store and the initial residual (operator, ring-summing init)
        "gpu_launches": 3 * K + 3,
        "reference_mode": {"GDOFps": n * K / t_ref / 1e9, "ms_per_step": t_ref / K * 1e3,
                           "note": "bit-exact reference arithmetic (same iterates as the CPU reference)",
                           "final_rel_residual": rep_ref.final_rel_residual},
        "clocks": clk.summary(),
        "kernel": kinfo,
        "setup_seconds": setup_s,
        "cg_report": {"iterations": rep.iterations, "r0": float(rep.residual_history[0]),
                      "final_rel_residual": rep.final_rel_residual},
    }
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(bp, p)
        except Exception as ex:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    del setup, op, A, b, x, u, w
    torch.cuda.empty_cache()
    if not args.no_sweep:
        line["p_sweep"] = p_sweep(bp, K, local)
        # BASELINE configs[1]: BP1 mass operator, p = 1..8, ~10M DOFs; and the
        # BP5 (collocated) operator of configs[3] at p = 7 on one GPU
        line["bp1_sweep_10M"] = p_sweep(1, K, local, ps=tuple(range(1, 9)), dofs=10_000_000)
        line["bp5_p7_50M"] = p_sweep(5, K, local, ps=(7,))
        # the paper's fusion comparison: fused single-kernel operator vs the
        # five-pass (gather / grad / factor / grad^T / scatter) pipeline
        line["fusion_vs_multipass"] = {f"bp{bp_}_p{p_}": fusion_compare(bp_, p_, K, local)
                                       for bp_, p_ in ((3, 7), (5, 7), (3, 4))}
        # BASELINE configs[4] (per GPU): BP3 p = 3, 5, 7 at ~50M DOFs, CG to 1e-8
        line["bp3_cg_to_1e-8_50M"] = {str(p_): cg_to_tol(3, p_, local) for p_ in (3, 5, 7)}
    print(json.dumps(line), flush=True)


def p_sweep(bp: int, K: int, local: int, ps=(2, 3, 4, 5, 6, 8), dofs: float = 50_000_000):
    """GDOF/s vs p (the metric is quoted 'vs p') at ~`dofs` DOFs per GPU,
    fixed-iteration fast CG timed with CUDA events."""
    import torch

    import paper_2109_05072_b200 as hx

    out = {}
    peak, _ = load_peaks()
    for p in ps:
        e = 1
        while ((e + 1) * p + 1) ** 3 <= dofs:
            e += 1
        dims = (e, e, e)
        try:
            op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p),
                                                                 device=local))
            A = hx.ConstrainedOperator(op) if bp != 1 else op
            b = torch.from_numpy(hx.bench_rhs(bp, p, dims)).cuda(local)
            x = torch.zeros_like(b)
            hx.cg(A, b, x, 0.0, 8, mode="fast")  # one graph block: capture before timing
            x.zero_()
            torch.cuda.synchronize()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record()
            hx.cg(A, b, x, 0.0, K, mode="fast")
            eb.record()
            torch.cuda.synchronize()
            dt = ea.elapsed_time(eb) / 1e3
            _, b_it, nL, _ = algorithmic_bytes(bp, p, dims)
            out[str(p)] = {"GDOFps": nL * K / dt / 1e9, "dofs": nL, "roofline_frac": b_it * K / dt / 1e9 / peak}
            del op, A, b, x
            torch.cuda.empty_cache()
        except Exception as ex:
            out[str(p)] = {"error": str(ex)[:120]}
    return out


def cg_to_tol(bp: int, p: int, local: int, dofs: float = 50_000_000, rel_tol: float = 1e-8,
              max_iter: int = 6000):
    """Time to solution of the fast CG (rel_tol, bench RHS, x0 = 0), CUDA events."""
    import torch

    import paper_2109_05072_b200 as hx

    e = 1
    while ((e + 1) * p + 1) ** 3 <= dofs:
        e += 1
    dims = (e, e, e)
    try:
        op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p),
                                                             device=local))
        A = hx.ConstrainedOperator(op) if bp != 1 else op
        b = torch.from_numpy(hx.bench_rhs(bp, p, dims)).cuda(local)
        x = torch.zeros_like(b)
        hx.cg(A, b, x, 0.0, 8, mode="fast")  # one graph block: capture before timing
        x.zero_()
        torch.cuda.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        rep = hx.cg(A, b, x, rel_tol, max_iter, mode="fast")
        eb.record()
        torch.cuda.synchronize()
        dt = ea.elapsed_time(eb) / 1e3
        n = b.numel()
        out = {"dims": list(dims), "dofs": n, "iterations": rep.iterations, "converged": bool(rep.converged),
               "final_rel_residual": rep.final_rel_residual, "seconds": dt,
               "GDOFps": n * max(rep.iterations, 1) / dt / 1e9}
        del op, A, b, x
        torch.cuda.empty_cache()
        return out
    except Exception as ex:
        return {"error": str(ex)[:160]}


def fusion_compare(bp: int, p: int, K: int, local: int, dofs: float = 30_000_000):
    """ms per constrained operator apply and per CG iteration on one mesh,
    fused kernel (fast and reference arithmetic) vs the multipass backend
    (always reference arithmetic), CUDA events on the launching stream."""
    import torch

    import paper_2109_05072_b200 as hx

    e = 1
    while ((e + 1) * p + 1) ** 3 <= dofs:
        e += 1
    dims = (e, e, e)
    out = {"dims": list(dims)}
    try:
        setup = hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p), device=local)
        b = torch.from_numpy(hx.bench_rhs(bp, p, dims)).cuda(local)
        u = torch.rand_like(b)
        w = torch.empty_like(b)
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        for name, backend, mode in (("fused_fast", hx.Backend.Cuda, "fast"),
                                    ("fused_reference", hx.Backend.Cuda, "reference"),
                                    ("multipass", hx.Backend.CudaMultipass, "reference")):
            op = hx.OperatorHandle(backend, setup)
            op.workspace().set_mode(mode)
            A = hx.ConstrainedOperator(op) if bp != 1 else op
            for _ in range(3):
                A.apply(u, w)
            torch.cuda.synchronize()
            ea, eb = ev(), ev()
            ea.record()
            for _ in range(K):
                A.apply(u, w)
            eb.record()
            torch.cuda.synchronize()
            t_apply = ea.elapsed_time(eb) / K
            x = torch.zeros_like(b)
            hx.cg(A, b, x, 0.0, 8, mode=mode)  # one graph block: capture before timing
            x.zero_()
            torch.cuda.synchronize()
            ea.record()
            hx.cg(A, b, x, 0.0, K, mode=mode)
            eb.record()
            torch.cuda.synchronize()
            t_it = ea.elapsed_time(eb) / K
            out[name] = {"ms_per_apply": t_apply, "ms_per_cg_iter": t_it, "cg_GDOFps": b.numel() / t_it / 1e6}
            del op, A, x
            torch.cuda.empty_cache()
        out["apply_speedup_fused_fast_vs_multipass"] = out["multipass"]["ms_per_apply"] / out["fused_fast"]["ms_per_apply"]
        del setup, b, u, w
        torch.cuda.empty_cache()
    except Exception as ex:
        out["error"] = str(ex)[:160]
    return out


if __name__ == "__main__":
    main()
