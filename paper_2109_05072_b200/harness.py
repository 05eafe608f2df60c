"""The reference's benchmark harness (bench.hpp) with a CUDA backend
(SURVEY §8(f) row 3): the same JSON campaign config and validation
(bench.hpp:38-153), BENCH_SEED semantics (:155-164), auto-sizing (:166-178),
seeded right-hand side (:181-204, 234-243), timing protocol -- warm-up solves,
then the best of `timed_repeats` solves of exactly `fixed_cg_iters`
unpreconditioned CG iterations (:206-295) -- and the 13-column CSV / plot-data
emitters (:297-390), unchanged, so the reference's plotting and comparison
tooling reads our rows as is.

Backends: the reference's names are accepted by the parser ("multipass",
"fused", "oracle": CPU backends of the reference, not run here) plus
  "cuda"        -- the B200 path, fast mode (DMMA / FMA kernels, fused CG),
  "cuda-exact"  -- the B200 path in reference arithmetic (its residual
                   histories equal the reference's fused backend bit for bit),
  "cuda-multipass" -- the unfused five-pass pipeline on the GPU (multipass.cu,
                   the paper's cuda-ref comparison point), reference arithmetic.
Timing uses CUDA events around each device-resident solve.

The CLI mirrors bench_main.cpp:
    python -m paper_2109_05072_b200.harness [run] config.json [--csv out.csv] [--plot out.dat]
    python -m paper_2109_05072_b200.harness verify [--p P] [--mesh EXxEYxEZ] [--bp bp1|bp3|bp5]
    python -m paper_2109_05072_b200.harness model [--p-min 1] [--p-max 8] [--collocated]
`verify` runs check_equivalence (verify.hpp:50-108) for the device backends.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from dataclasses import dataclass, field
from typing import List, Optional

import ctypes as C

from . import _lib
from .api import (BPKind, ConstrainedOperator, DegenerateElementError, OperatorHandle, Backend, _check, bench_rhs,
                  build_box_mesh, cg, is_diffusion, make_setup, parse_bp, to_string)

K_MAX_DEFORM_AMPLITUDE = 0.15  # mesh.hpp:53
CSV_HEADER = ("bp,backend,p,q,elements,dofs,cg_iters,seconds,throughput,"
              "model_flops_per_elem,model_reads_per_elem,model_ai,threads")
CPU_BACKENDS = ("multipass", "fused", "oracle")
GPU_BACKENDS = ("cuda", "cuda-exact", "cuda-multipass")


class ConfigError(RuntimeError):
    """config_error (bench.hpp:33-36)."""


@dataclass
class BenchConfig:
    """bench.hpp:41-54"""

    bp: str = "bp1"
    degrees: List[int] = field(default_factory=list)
    dims: Optional[tuple] = None
    target_dofs: Optional[int] = None
    deform_amplitude: float = 0.0
    backends: List[str] = field(default_factory=lambda: ["cuda"])
    fixed_cg_iters: int = 20
    warmup_repeats: int = 2
    timed_repeats: int = 5
    threads: int = 0
    output_path: str = ""


@dataclass
class BenchRecord:
    """bench.hpp:56-70"""

    bp: str = ""
    backend: str = ""
    p: int = 0
    q: int = 0
    elements: int = 0
    dofs: int = 0
    cg_iters: int = 0
    seconds: float = 0.0
    throughput: float = 0.0
    model_flops_per_elem: float = 0.0
    model_reads_per_elem: float = 0.0
    model_ai: float = 0.0
    threads: int = 1


@dataclass
class RunOutput:
    """bench.hpp:72-77"""

    records: List[BenchRecord] = field(default_factory=list)
    histories: List[list] = field(default_factory=list)
    seed: int = 0
    errors: List[str] = field(default_factory=list)


_KNOWN = ("bp", "degrees", "dims", "target_dofs", "deform_amplitude", "backends", "fixed_cg_iters",
          "warmup_repeats", "timed_repeats", "threads", "output_path")


def _int(v, name):
    if isinstance(v, bool) or not isinstance(v, int):
        raise ConfigError(f"malformed config value: '{name}' must be an integer")
    return v


def parse_config(j) -> BenchConfig:
    """parse_config (bench.hpp:93-153): unknown keys rejected, exactly one of
    dims / target_dofs, value ranges as the reference."""
    if not isinstance(j, dict):
        raise ConfigError("config must be a JSON object")
    for key in j:
        if key not in _KNOWN:
            raise ConfigError(f"unknown config key '{key}'")
    cfg = BenchConfig()
    if "bp" not in j:
        raise ConfigError("missing required key 'bp'")
    if j["bp"] not in ("bp1", "bp3", "bp5"):
        raise ConfigError(f"unknown bp kind '{j['bp']}' (expected bp1, bp3 or bp5)")
    cfg.bp = j["bp"]
    if "degrees" not in j:
        raise ConfigError("missing required key 'degrees'")
    if not isinstance(j["degrees"], list):
        raise ConfigError("malformed config value: 'degrees' must be an array")
    cfg.degrees = [_int(p, "degrees") for p in j["degrees"]]
    if not cfg.degrees:
        raise ConfigError("'degrees' must be a non-empty array")
    if any(p < 1 for p in cfg.degrees):
        raise ConfigError("degrees must be >= 1")
    if "dims" in j:
        d = j["dims"]
        if not isinstance(d, list) or len(d) != 3:
            raise ConfigError("'dims' must have exactly three entries")
        cfg.dims = tuple(_int(e, "dims") for e in d)
        if any(e < 1 for e in cfg.dims):
            raise ConfigError("dims entries must be >= 1")
    if "target_dofs" in j:
        cfg.target_dofs = _int(j["target_dofs"], "target_dofs")
        if cfg.target_dofs < 1:
            raise ConfigError("target_dofs must be >= 1")
    if (cfg.dims is not None) == (cfg.target_dofs is not None):
        raise ConfigError("exactly one of 'dims' and 'target_dofs' is required")
    if "deform_amplitude" in j:
        cfg.deform_amplitude = float(j["deform_amplitude"])
    if not (0.0 <= cfg.deform_amplitude <= K_MAX_DEFORM_AMPLITUDE):
        raise ConfigError("deform_amplitude must lie in [0, 0.15]")
    if "backends" in j:
        cfg.backends = []
        for b in j["backends"]:
            if b not in CPU_BACKENDS + GPU_BACKENDS:
                raise ConfigError(f"unknown backend '{b}' (expected multipass, fused, oracle, cuda, cuda-exact "
                                  "or cuda-multipass)")
            cfg.backends.append(b)
        if not cfg.backends:
            raise ConfigError("'backends' must be non-empty")
    for key, lo in (("fixed_cg_iters", 1), ("warmup_repeats", 0), ("timed_repeats", 1), ("threads", 0)):
        if key in j:
            setattr(cfg, key, _int(j[key], key))
        if getattr(cfg, key) < lo:
            raise ConfigError(f"{key} must be >= {lo}")
    if "output_path" in j:
        cfg.output_path = str(j["output_path"])
    return cfg


def load_config(path: str) -> BenchConfig:
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise ConfigError(f"cannot open config file '{path}'")
    except json.JSONDecodeError as e:
        raise ConfigError(f"config is not valid JSON: {e}")
    return parse_config(j)


def bench_seed() -> int:
    """BENCH_SEED (decimal unsigned) when set, else 20240101 (bench.hpp:155-164)."""
    env = os.environ.get("BENCH_SEED", "")
    if not env:
        return 20240101
    if not env.isdigit() or int(env) >= 2**64:
        raise ConfigError("BENCH_SEED must be a decimal unsigned integer")
    return int(env)


def auto_size_dims(p: int, target_dofs: int):
    """Largest (e, e, e) box with (e p + 1)^3 <= target, at least one element (bench.hpp:166-178)."""
    e = 1
    while ((e + 1) * p + 1) ** 3 <= target_dofs:
        e += 1
    return (e, e, e)


def cost_model(p: int, collocated: bool):
    """cost_model (cost_model.hpp:27-40): (flops, reads, arithmetic intensity) per element."""
    if p < 1:
        raise ValueError("cost_model: degree must be >= 1")
    n = p + 1
    n3 = n**3
    flops = (12 if collocated else 24) * n3 * n + 15 * n3
    reads = 7 * n3
    return flops, reads, flops / reads


def run_bench(config: BenchConfig, device: int = 0) -> RunOutput:
    """run_bench (bench.hpp:206-295) for the GPU backends; CPU backend names
    are recorded as errors (they are the reference's own, not run here)."""
    import torch

    out = RunOutput(seed=bench_seed())
    for p in config.degrees:
        dims = config.dims if config.dims is not None else auto_size_dims(p, config.target_dofs)
        for backend in config.backends:
            try:
                if backend not in GPU_BACKENDS:
                    raise ConfigError(f"backend '{backend}' is a CPU backend of the reference (not run here)")
                kind = BPKind({"bp1": 1, "bp3": 3, "bp5": 5}[config.bp])
                mesh = build_box_mesh(dims, p, (1.0, 1.0, 1.0), config.deform_amplitude)
                op = OperatorHandle(Backend.CudaMultipass if backend == "cuda-multipass" else Backend.Cuda,
                                    make_setup(kind, mesh, device=device))
                mode = "fast" if backend == "cuda" else "reference"
                A = ConstrainedOperator(op) if kind != BPKind.BP1 else op
                dev = torch.device("cuda", device)
                b = torch.from_numpy(bench_rhs(kind, p, dims, seed=out.seed)).to(dev)
                x = torch.zeros_like(b)
                for _ in range(config.warmup_repeats):
                    x.zero_()
                    cg(A, b, x, 0.0, config.fixed_cg_iters, mode=mode)
                best, report = float("inf"), None
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                for _ in range(config.timed_repeats):
                    x.zero_()
                    torch.cuda.synchronize(dev)
                    ev0.record()
                    r = cg(A, b, x, 0.0, config.fixed_cg_iters, mode=mode)
                    ev1.record()
                    torch.cuda.synchronize(dev)
                    dt = ev0.elapsed_time(ev1) / 1e3
                    if dt < best:
                        best, report = dt, r
                flops, reads, ai = cost_model(p, config.bp == "bp5")
                out.records.append(BenchRecord(
                    bp=config.bp, backend=backend, p=p, q=op.setup().q, elements=mesh.num_elements(),
                    dofs=op.size(), cg_iters=config.fixed_cg_iters, seconds=best,
                    throughput=op.size() * config.fixed_cg_iters / best, model_flops_per_elem=float(flops),
                    model_reads_per_elem=float(reads), model_ai=ai, threads=1))
                out.histories.append([float(v) for v in report.residual_history])
            except Exception as e:  # per-run failures are recorded, the sweep continues
                out.errors.append(f"{config.bp} p={p} backend={backend}: {e}")
    return out


def emit_csv(records, f) -> None:
    """emit_csv (bench.hpp:297-315): header + one 13-column row per record, %.17g."""
    f.write(CSV_HEADER + "\n")
    for r in records:
        f.write("%s,%s,%d,%d,%d,%d,%d,%.17g,%.17g,%.17g,%.17g,%.17g,%d\n" % (
            r.bp, r.backend, r.p, r.q, r.elements, r.dofs, r.cg_iters, r.seconds, r.throughput,
            r.model_flops_per_elem, r.model_reads_per_elem, r.model_ai, r.threads))


def parse_csv(f) -> List[BenchRecord]:
    """parse_csv (bench.hpp:317-349)."""
    lines = f.read().split("\n")
    if not lines or lines[0] == "" and len(lines) == 1:
        raise RuntimeError("parse_csv: empty input")
    if lines[0] != CSV_HEADER:
        raise RuntimeError("parse_csv: unexpected header")
    recs = []
    for line in lines[1:]:
        if not line:
            continue
        c = line.split(",")
        if len(c) != 13:
            raise RuntimeError("parse_csv: expected 13 columns")
        recs.append(BenchRecord(c[0], c[1], int(c[2]), int(c[3]), int(c[4]), int(c[5]), int(c[6]), float(c[7]),
                                float(c[8]), float(c[9]), float(c[10]), float(c[11]), int(c[12])))
    return recs


def emit_plotdata(records, f) -> None:
    """emit_plotdata (bench.hpp:351-383): one block per (backend, p), dofs strictly increasing."""
    s = sorted(records, key=lambda r: (r.backend, r.p, r.dofs))  # stable, as std::stable_sort
    i, first = 0, True
    while i < len(s):
        backend, p = s[i].backend, s[i].p
        if not first:
            f.write("\n")
        first = False
        f.write(f"# backend={backend} p={p}\n")
        last = -1
        while i < len(s) and s[i].backend == backend and s[i].p == p:
            if s[i].dofs != last:
                last = s[i].dofs
                f.write("%d %.17g\n" % (s[i].dofs, s[i].throughput))
            i += 1


# ---------------------------------------------------------------- verify
K_EQUIVALENCE_TOL = 1e-12  # verify.hpp:15


@dataclass
class EquivalenceCase:
    """verify.hpp:17-22"""

    bp: BPKind = BPKind.BP1
    p: int = 1
    dims: tuple = (1, 1, 1)
    amplitude: float = 0.0


def default_equivalence_cases() -> List[EquivalenceCase]:
    """verify.hpp:38-46: every BP, p = 1..4, three box shapes, undeformed and deformed."""
    return [EquivalenceCase(bp, p, dims, a) for bp in (BPKind.BP1, BPKind.BP3, BPKind.BP5) for p in (1, 2, 3, 4)
            for dims in ((1, 1, 1), (2, 2, 2), (3, 2, 1)) for a in (0.0, 0.1)]


def _uniform_stream(seed: int, count: int):
    import numpy as np

    out = np.empty(count)
    _check(_lib.lib().hexbp_uniform_stream(C.c_uint64(seed & (2**64 - 1)), -1.0, 1.0, count,
                                           out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def check_equivalence(c: EquivalenceCase, num_vectors: int = 10, tol: float = K_EQUIVALENCE_TOL,
                      seed: int = 2024, device: int = 0) -> dict:
    """check_equivalence (verify.hpp:50-108) for the device backends. The
    comparison operator is the device operator in reference arithmetic,
    which equals the reference's Fused backend bit for bit
    (tests/test_gpu_parity.py) -- the assembled Backend::Oracle matrix is not
    part of the hot path. Compared: "cuda" (fast kernels) and "cuda-multipass";
    the probes are the reference's (mt19937_64(seed ^ p << 32 ^ n), U(-1, 1))."""
    import numpy as np

    mesh = build_box_mesh(c.dims, c.p, (1.0, 1.0, 1.0), c.amplitude)
    setup = make_setup(c.bp, mesh, device=device)
    exact = OperatorHandle(Backend.Cuda, setup)
    fast = OperatorHandle(Backend.Cuda, setup)
    fast.workspace().set_mode("fast")
    multi = OperatorHandle(Backend.CudaMultipass, setup)
    n = exact.size()
    draws = _uniform_stream(seed ^ (c.p << 32) ^ n, 2 * num_vectors * n)
    res = {"max_rel_multipass": 0.0, "max_rel_fused": 0.0, "max_symmetry": 0.0, "nullspace_residual": 0.0,
           "min_quadratic_form": float("inf")}
    for trial in range(num_vectors):
        u = draws[2 * trial * n:(2 * trial + 1) * n]
        v = draws[(2 * trial + 1) * n:(2 * trial + 2) * n]
        wo, wm, wf = exact.apply(u), multi.apply(u), fast.apply(u)
        ref = float(np.sqrt(wo @ wo))
        res["max_rel_multipass"] = max(res["max_rel_multipass"], float(np.linalg.norm(wm - wo)) / ref)
        res["max_rel_fused"] = max(res["max_rel_fused"], float(np.linalg.norm(wf - wo)) / ref)
        wv = fast.apply(v)
        uav, vau = float(u @ wv), float(v @ wf)
        res["max_symmetry"] = max(res["max_symmetry"],
                                  abs(uav - vau) / (float(np.linalg.norm(wf)) * float(np.linalg.norm(v))))
        if c.bp == BPKind.BP1:
            res["min_quadratic_form"] = min(res["min_quadratic_form"], float(u @ wf) / float(u @ u))
    ok = res["max_rel_multipass"] <= tol and res["max_rel_fused"] <= tol and res["max_symmetry"] <= tol
    if is_diffusion(c.bp):
        from .api import jacobi_diagonal

        w1 = fast.apply(np.ones(n))
        # |A 1|_inf / |A|_inf; without the assembled matrix max_i |A_ii| <= |A|_inf
        # stands in for the norm (a stricter test than the reference's)
        scale = float(np.abs(jacobi_diagonal(exact, device=False)).max())
        res["nullspace_residual"] = float(np.abs(w1).max()) / max(scale, 1e-300)
        ok = ok and res["nullspace_residual"] <= tol
    else:
        ok = ok and res["min_quadratic_form"] > 0.0
    res["pass"] = ok
    return res


def parse_mesh_dims(s: str) -> tuple:
    """bench_main.cpp:27-37"""
    parts = s.split("x")
    if len(parts) != 3 or not all(x.strip().lstrip("-").isdigit() for x in parts):
        raise ConfigError("mesh must look like EXxEYxEZ, e.g. 2x2x2")
    dims = tuple(int(x) for x in parts)
    if any(d < 1 for d in dims):
        raise ConfigError("mesh dimensions must be >= 1")
    return dims


def verify_command(p: Optional[int] = None, mesh: Optional[str] = None, bp: Optional[str] = None,
                   device: int = 0, out=None) -> int:
    """bench_main.cpp:60-104: same case filtering, per-case line and summary."""
    out = out or sys.stdout
    cases = default_equivalence_cases()
    if p is not None:
        if p < 1:
            raise ConfigError("--p must be >= 1")
        cases = [c for c in cases if c.p == p]
        if not cases:  # degree outside the default sweep: test it directly
            cases = [EquivalenceCase(k, p, (2, 2, 2), a) for k in (BPKind.BP1, BPKind.BP3, BPKind.BP5)
                     for a in (0.0, 0.1)]
    if mesh:
        dims = parse_mesh_dims(mesh)
        for c in cases:
            c.dims = dims
    if bp:
        kind = parse_bp(bp)
        cases = [c for c in cases if c.bp == kind]
    all_pass, worst = True, 0.0
    for c in cases:
        tag = f"{to_string(c.bp):<4} p={c.p} mesh={c.dims[0]}x{c.dims[1]}x{c.dims[2]} a={c.amplitude:.2f}"
        try:
            r = check_equivalence(c, device=device)
            rel = max(r["max_rel_fused"], r["max_rel_multipass"])
            worst = max(worst, rel)
            print(f"{tag}  rel={rel:.3e} sym={r['max_symmetry']:.3e} {'ok' if r['pass'] else 'FAIL'}", file=out)
            all_pass = all_pass and r["pass"]
        except DegenerateElementError as e:
            print(f"{tag}  DEGENERATE: {e}", file=out)
            all_pass = False
    print(f"{len(cases)} cases, worst backend/oracle deviation {worst:.3e}, tolerance {K_EQUIVALENCE_TOL:.1e}: "
          f"{'PASS' if all_pass else 'FAIL'}", file=out)
    return 0 if all_pass else 1  # kExitVerifyFailed (bench_main.cpp:25)


def model_command(p_min: int = 1, p_max: int = 8, collocated: bool = False, out=None) -> int:
    """bench_main.cpp:106-117"""
    out = out or sys.stdout
    if p_min < 1 or p_max < p_min:
        raise ConfigError("need 1 <= --p-min <= --p-max")
    print("p,collocated,flops_per_elem,reads_per_elem,ai", file=out)
    for p in range(p_min, p_max + 1):
        m = cost_model(p, collocated)
        print(f"{p},{1 if collocated else 0},{m[0]},{m[1]},{m[2]:.17g}", file=out)
    return 0


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if argv and argv[0] == "verify":
        ap = argparse.ArgumentParser(prog="harness verify")
        ap.add_argument("--p", type=int, default=None)
        ap.add_argument("--mesh", default=None)
        ap.add_argument("--bp", default=None)
        ap.add_argument("--device", type=int, default=0)
        a = ap.parse_args(argv[1:])
        try:
            return verify_command(a.p, a.mesh, a.bp, a.device)
        except (ConfigError, ValueError) as e:
            print(f"config error: {e}", file=sys.stderr)
            return 2
    if argv and argv[0] == "model":
        ap = argparse.ArgumentParser(prog="harness model")
        ap.add_argument("--p-min", type=int, default=1)
        ap.add_argument("--p-max", type=int, default=8)
        ap.add_argument("--collocated", action="store_true")
        a = ap.parse_args(argv[1:])
        try:
            return model_command(a.p_min, a.p_max, a.collocated)
        except ConfigError as e:
            print(f"config error: {e}", file=sys.stderr)
            return 2
    if argv and argv[0] == "run":
        argv = argv[1:]
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("config")
    ap.add_argument("--csv", default=None)
    ap.add_argument("--plot", default=None)
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        cfg = load_config(a.config)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    out = run_bench(cfg, a.device)
    for e in out.errors:
        print(f"error: {e}", file=sys.stderr)
    path = a.csv or cfg.output_path
    if path:
        with open(path, "w", newline="\n") as f:
            emit_csv(out.records, f)
    else:
        emit_csv(out.records, sys.stdout)
    if a.plot:
        with open(a.plot, "w", newline="\n") as f:
            emit_plotdata(out.records, f)
    return 1 if out.errors and not out.records else 0


if __name__ == "__main__":
    sys.exit(main())
