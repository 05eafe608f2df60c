"""Harness integration: the reference's run_bench /
config / CSV / plot-data semantics with the CUDA backends. CPU tests mirror
tests/unit/test_bench.cpp (bench.hpp:38-390); the GPU test checks that the
cuda-exact backend reproduces the reference's residual history bit for bit
(RunBench.BackendsShareResidualHistories, test_bench.cpp:221-264)."""
import io
import json
import os

import numpy as np
import pytest

from paper_2109_05072_b200 import harness as H


def minimal():
    return {"bp": "bp3", "degrees": [1, 2], "dims": [2, 2, 2]}


def test_config_minimal_and_defaults():
    cfg = H.parse_config(minimal())
    assert cfg.bp == "bp3" and cfg.degrees == [1, 2] and cfg.dims == (2, 2, 2)
    assert (cfg.fixed_cg_iters, cfg.warmup_repeats, cfg.timed_repeats) == (20, 2, 5)


@pytest.mark.parametrize("mut", [
    lambda j: j.update(surprise=1),
    lambda j: j.pop("bp"),
    lambda j: j.pop("degrees"),
    lambda j: j.update(target_dofs=1000),  # both size specs
    lambda j: j.pop("dims"),               # neither
    lambda j: j.update(degrees=[0]),
    lambda j: j.update(bp="bp7"),
    lambda j: j.update(backends=["warp"]),
    lambda j: j.update(fixed_cg_iters=0),
    lambda j: j.update(deform_amplitude=0.5),
    lambda j: j.update(dims=[1, 1]),
])
def test_config_rejections(mut):
    j = minimal()
    mut(j)
    with pytest.raises(H.ConfigError):
        H.parse_config(j)


def test_config_accepts_target_dofs_and_gpu_backends():
    j = minimal()
    j.pop("dims")
    j["target_dofs"] = 1000
    j["backends"] = ["cuda", "cuda-exact", "fused"]
    cfg = H.parse_config(j)
    assert cfg.target_dofs == 1000 and cfg.backends == ["cuda", "cuda-exact", "fused"]


def test_bench_seed(monkeypatch):
    monkeypatch.delenv("BENCH_SEED", raising=False)
    assert H.bench_seed() == 20240101
    monkeypatch.setenv("BENCH_SEED", "12345")
    assert H.bench_seed() == 12345
    monkeypatch.setenv("BENCH_SEED", "12x45")
    with pytest.raises(H.ConfigError):
        H.bench_seed()


def test_auto_size():
    assert H.auto_size_dims(1, 27) == (2, 2, 2)
    assert H.auto_size_dims(1, 26) == (1, 1, 1)
    assert H.auto_size_dims(3, 15625) == (8, 8, 8)
    assert H.auto_size_dims(3, 15624) == (7, 7, 7)
    assert H.auto_size_dims(5, 1) == (1, 1, 1)


def test_cost_model():
    f, r, ai = H.cost_model(2, False)
    assert (f, r) == (24 * 81 + 15 * 27, 7 * 27) and ai == f / r
    with pytest.raises(ValueError):
        H.cost_model(0, True)


def _rec(**kw):
    r = H.BenchRecord(bp="bp5", backend="cuda", p=3, q=4, elements=64, dofs=2197, cg_iters=20,
                      seconds=0.12345678901234567, model_flops_per_elem=4032, model_reads_per_elem=448, model_ai=9.0,
                      threads=4)
    r.throughput = 2197.0 * 20 / r.seconds
    for k, v in kw.items():
        setattr(r, k, v)
    return r


def test_csv_header_roundtrip_and_columns():
    f = io.StringIO()
    H.emit_csv([], f)
    assert f.getvalue() == H.CSV_HEADER + "\n"
    f = io.StringIO()
    H.emit_csv([_rec()], f)
    row = f.getvalue().split("\n")[1]
    assert row.count(",") == 12
    back = H.parse_csv(io.StringIO(f.getvalue()))
    assert back == [_rec()]  # bitwise through %.17g
    with pytest.raises(RuntimeError):
        H.parse_csv(io.StringIO("bad,header\n"))


def test_plotdata_blocks():
    recs = [_rec(backend="cuda", p=2, dofs=100, throughput=1.0), _rec(backend="cuda", p=2, dofs=50, throughput=2.0),
            _rec(backend="cuda", p=2, dofs=50, throughput=3.0), _rec(backend="cuda-exact", p=1, dofs=10,
                                                                     throughput=4.0)]
    f = io.StringIO()
    H.emit_plotdata(recs, f)
    assert f.getvalue() == "# backend=cuda p=2\n50 2\n100 1\n\n# backend=cuda-exact p=1\n10 4\n"


@pytest.mark.skipif(not os.path.exists(__import__("oracle").REF_SO), reason="oracle/_ref not built")
def test_csv_header_is_the_references():
    import ctypes as C

    import oracle

    lib = C.CDLL(oracle.REF_SO)
    lib.ref_csv_header.restype = C.c_char_p
    assert lib.ref_csv_header().decode() == H.CSV_HEADER


@pytest.mark.gpu
def test_run_bench_cuda_backends_and_reference_history():
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cg.json")))["cfg1_fixed50"]
    cfg = H.parse_config({"bp": "bp3", "degrees": [3], "dims": [33, 33, 33], "backends": ["cuda", "cuda-exact"],
                          "fixed_cg_iters": 50, "warmup_repeats": 1, "timed_repeats": 2})
    out = H.run_bench(cfg)
    assert not out.errors, out.errors
    assert [r.backend for r in out.records] == ["cuda", "cuda-exact"]
    for r in out.records:
        assert r.dofs == 1_000_000 and r.q == 5 and r.elements == 33**3 and r.throughput > 0
    # reference arithmetic: the reference's fused-backend history, bit for bit
    assert np.array_equal(np.array(out.histories[1]), np.array(golden["residual_history"]))
    # fast mode tracks it
    assert abs(out.histories[0][-1] / out.histories[0][0] - golden["final_rel_residual"]) < 1e-10
    f = io.StringIO()
    H.emit_csv(out.records, f)
    assert len(H.parse_csv(io.StringIO(f.getvalue()))) == 2
    # CPU backend names are parsed but reported as errors, the sweep continues
    out2 = H.run_bench(H.parse_config({"bp": "bp1", "degrees": [1], "dims": [2, 2, 2], "backends": ["fused", "cuda"],
                                       "warmup_repeats": 0, "timed_repeats": 1}))
    assert len(out2.records) == 1 and len(out2.errors) == 1


def test_model_and_mesh_parsing_cli():
    """bench_main.cpp model / --mesh parsing mirrors (no GPU)."""
    import io

    from paper_2109_05072_b200 import harness as H

    buf = io.StringIO()
    assert H.model_command(1, 3, True, out=buf) == 0
    lines = buf.getvalue().splitlines()
    assert lines[0] == "p,collocated,flops_per_elem,reads_per_elem,ai" and len(lines) == 4
    assert lines[3].startswith("3,1,4032,448,")  # acceptance_main.cpp:159 (p=3 collocated)
    assert H.parse_mesh_dims("3x2x1") == (3, 2, 1)
    for bad in ("3x2", "0x1x1", "axbxc"):
        with pytest.raises(H.ConfigError):
            H.parse_mesh_dims(bad)
    assert len(H.default_equivalence_cases()) == 72


@pytest.mark.gpu
def test_verify_command_on_gpu():
    """bench verify (bench_main.cpp:60-104) for the device backends: the full
    72-case sweep passes at the reference's 1e-12 tolerance."""
    import io

    from paper_2109_05072_b200 import harness as H

    buf = io.StringIO()
    rc = H.verify_command(out=buf)
    out = buf.getvalue().splitlines()
    assert len(out) == 73
    # as in the reference's own sweep, bp5 p=3 on one a=0.1 element is
    # degenerate (tests/golden/equivalence.json) and fails the verify run
    bad = [line for line in out[:-1] if not line.endswith(" ok")]
    assert len(bad) == 1 and bad[0].startswith("bp5  p=3 mesh=1x1x1 a=0.10  DEGENERATE: non-positive Jacobian"), bad
    assert out[-1].startswith("72 cases, worst backend/oracle deviation") and out[-1].endswith("FAIL"), out[-1]
    assert rc == 1
    buf = io.StringIO()
    assert H.verify_command(p=6, bp="bp5", out=buf) == 0  # degree outside the sweep: 2x2x2, a in {0, 0.1}
    assert len(buf.getvalue().splitlines()) == 3
