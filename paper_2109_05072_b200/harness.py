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

    python -m paper_2109_05072_b200.harness config.json [--csv out.csv] [--plot out.dat]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from dataclasses import dataclass, field
from typing import List, Optional

from .api import BPKind, ConstrainedOperator, OperatorHandle, Backend, bench_rhs, build_box_mesh, cg, make_setup

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


def main(argv=None) -> int:
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
