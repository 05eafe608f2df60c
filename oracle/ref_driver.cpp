// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A thin extern "C" shim over the UNMODIFIED reference headers in
// /root/reference/proj/include/hexbp (compiled in place by oracle/Makefile,
// output only into oracle/_ref/). It lets tests/, bench.py's cpu_baseline /
// `--impl reference` leg, and tests/golden/make_golden.py drive the
// reference's own code:
//   - make_setup + OperatorHandle(Fused)      (operator.hpp:70-77, 244-279)
//   - ConstrainedOperator                     (solver.hpp:48-74)
//   - cg, jacobi_diagonal                     (solver.hpp:91-205)
//   - run_bench (reference timing protocol)   (bench.hpp:214-295)
//   - check_equivalence (72-case sweep)       (verify.hpp:50-108)
// No reference source is copied here; the headers are #included from their
// original location at build time.
#include <cmath>
#include <cstdint>
#include <numbers>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "hexbp/bench.hpp"
#include "hexbp/verify.hpp"

using namespace hexbp;

namespace {

struct RefHandle {
  HexMesh mesh;
  std::shared_ptr<const OperatorSetup> setup;
  std::unique_ptr<OperatorHandle> op;
  std::unique_ptr<ConstrainedOperator> cop;
  BPKind bp;
};

thread_local std::string g_err;

BPKind to_bp(int bp) { return bp == 1 ? BPKind::BP1 : (bp == 3 ? BPKind::BP3 : BPKind::BP5); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// bp in {1,3,5}; backend 0 = multipass, 1 = fused.
void* ref_create(int bp, int p, int ex, int ey, int ez, double amplitude, int backend) {
  try {
    auto h = std::make_unique<RefHandle>();
    h->bp = to_bp(bp);
    h->mesh = build_box_mesh({ex, ey, ez}, p, {1.0, 1.0, 1.0}, amplitude);
    h->setup = make_setup(h->bp, h->mesh);
    h->op = std::make_unique<OperatorHandle>(backend == 0 ? Backend::Multipass : Backend::Fused, h->setup);
    h->cop = std::make_unique<ConstrainedOperator>(*h->op, boundary_bcs(h->mesh));
    return h.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_destroy(void* h) { delete static_cast<RefHandle*>(h); }

int64_t ref_size(void* h) { return static_cast<RefHandle*>(h)->op->size(); }
int ref_num_elements(void* h) { return static_cast<RefHandle*>(h)->setup->num_elements(); }
int ref_q(void* h) { return static_cast<RefHandle*>(h)->setup->basis.num_quad_1d(); }
int ref_components(void* h) { return static_cast<RefHandle*>(h)->setup->factors.components; }

// B and D: q x (p+1) row-major (basis.hpp:21-22).
void ref_basis(void* h, double* B, double* D) {
  const auto& b = static_cast<RefHandle*>(h)->setup->basis;
  std::memcpy(B, b.B.data().data(), sizeof(double) * b.B.data().size());
  std::memcpy(D, b.D.data().data(), sizeof(double) * b.D.data().size());
}

// Quadrature points/weights of the element rule (q each) and GLL nodes (p+1 each).
void ref_rules(void* h, double* qpts, double* qwts, double* npts, double* nwts) {
  const auto& b = static_cast<RefHandle*>(h)->setup->basis;
  std::memcpy(qpts, b.quad.points.data(), sizeof(double) * b.quad.points.size());
  std::memcpy(qwts, b.quad.weights.data(), sizeof(double) * b.quad.weights.size());
  std::memcpy(npts, b.nodes.points.data(), sizeof(double) * b.nodes.points.size());
  std::memcpy(nwts, b.nodes.weights.data(), sizeof(double) * b.nodes.weights.size());
}

// Geometric factors in the reference AoS layout data[(e*q3+qp)*comp+c] (geometry.hpp:48-56).
void ref_factors(void* h, double* out) {
  const auto& f = static_cast<RefHandle*>(h)->setup->factors;
  std::memcpy(out, f.data.data(), sizeof(double) * f.data.size());
}

// Node coordinates, 3 doubles per global node (mesh.hpp:366).
void ref_coords(void* h, double* out) {
  const auto& m = static_cast<RefHandle*>(h)->mesh;
  for (std::size_t i = 0; i < m.coords.size(); ++i)
    for (int c = 0; c < 3; ++c) out[3 * i + c] = m.coords[i][c];
}

// Unconstrained (constrained=0) or ConstrainedOperator (constrained=1) apply.
int ref_apply(void* hv, int constrained, const double* u, double* w) {
  auto* h = static_cast<RefHandle*>(hv);
  try {
    const std::size_t n = h->op->size();
    std::span<const double> us(u, n);
    std::vector<double> wv;
    if (constrained)
      h->cop->apply(us, wv);
    else
      h->op->apply(us, wv);
    std::memcpy(w, wv.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Reference bench right-hand side (bench.hpp:497-506): seeded uniform(-1,1),
// boundary dofs zeroed for the diffusion kinds.
void ref_bench_rhs(void* hv, uint64_t seed, double* b) {
  auto* h = static_cast<RefHandle*>(hv);
  const auto& dims = h->mesh.dims;
  std::mt19937_64 rng(detail::mix_seed(seed, h->bp, h->mesh.degree, dims));
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  const std::size_t n = h->op->size();
  for (std::size_t i = 0; i < n; ++i) b[i] = dist(rng);
  if (is_diffusion(h->bp))
    for (int d : h->cop->bcs().dofs) b[d] = 0.0;
}

// test::random_vector equivalent (tests/unit/test_support.hpp:15-21) via the std engine.
void ref_random_vector(uint64_t seed, int64_t n, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

// cg on the (constrained) operator. history must hold max_iter+1 doubles.
// Returns 0 ok, 2 divergence_error, 1 other error.
int ref_cg(void* hv, int constrained, const double* b, double* x, double rel_tol, int max_iter, int* iterations,
           int* converged, double* final_rel, double* history, double* seconds) {
  auto* h = static_cast<RefHandle*>(hv);
  try {
    const std::size_t n = h->op->size();
    std::vector<double> xv(x, x + n);
    auto apply = [&](std::span<const double> u, std::vector<double>& w) {
      if (constrained)
        h->cop->apply(u, w);
      else
        h->op->apply(u, w);
    };
    CGReport r = cg(apply, std::span<const double>(b, n), xv, rel_tol, max_iter);
    std::memcpy(x, xv.data(), sizeof(double) * n);
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    *final_rel = r.final_rel_residual;
    *seconds = r.seconds;
    for (std::size_t k = 0; k < r.residual_history.size(); ++k) history[k] = r.residual_history[k];
    return 0;
  } catch (const divergence_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// jacobi_diagonal (solver.hpp:155-205) of the operator (constrained = 0) or
// of the ConstrainedOperator (1 on essential dofs).
void ref_jacobi_diagonal(void* hv, int constrained, double* out) {
  auto* h = static_cast<RefHandle*>(hv);
  const std::vector<double> d = constrained ? jacobi_diagonal(*h->cop) : jacobi_diagonal(*h->op);
  std::memcpy(out, d.data(), sizeof(double) * d.size());
}

// cg with the Jacobi diagonal (solver.hpp:91-153, diag != nullptr).
int ref_pcg(void* hv, int constrained, const double* b, double* x, const double* diag, double rel_tol, int max_iter,
            int* iterations, int* converged, double* final_rel, double* history, double* seconds) {
  auto* h = static_cast<RefHandle*>(hv);
  try {
    const std::size_t n = h->op->size();
    std::vector<double> xv(x, x + n);
    const std::vector<double> dv(diag, diag + n);
    auto apply = [&](std::span<const double> u, std::vector<double>& w) {
      if (constrained)
        h->cop->apply(u, w);
      else
        h->op->apply(u, w);
    };
    CGReport r = cg(apply, std::span<const double>(b, n), xv, rel_tol, max_iter, &dv);
    std::memcpy(x, xv.data(), sizeof(double) * n);
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    *final_rel = r.final_rel_residual;
    *seconds = r.seconds;
    for (std::size_t k = 0; k < r.residual_history.size(); ++k) history[k] = r.residual_history[k];
    return 0;
  } catch (const divergence_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The manufactured-solution Poisson problem of acceptance criterion 5
// (proj/tests/acceptance/acceptance_main.cpp:181-200) driven through the
// reference's API: u = sin(pi x) sin(pi y) sin(pi z) on the unit cube, f = 3 pi^2 u,
// BP3 fused operator with the box-boundary constraint, consistent load
// vector (assemble_load, solver.hpp:207-239) with essential rows zeroed,
// Jacobi-preconditioned cg (1e-8, 2000), discrete L2 error
// (solver.hpp:256-300). Outputs: the load vector b (after zeroing), the
// solution x (n = (elems p + 1)^3 each, may be null), the error, iterations.
int ref_poisson(int elems, int p, double* b_out, double* x_out, double* err, int* iterations) {
  try {
    const double pi = std::numbers::pi;
    auto exact = [pi](double x, double y, double z) { return std::sin(pi * x) * std::sin(pi * y) * std::sin(pi * z); };
    auto rhs = [pi, exact](double x, double y, double z) { return 3.0 * pi * pi * exact(x, y, z); };
    const HexMesh mesh = build_box_mesh({elems, elems, elems}, p, {1, 1, 1}, 0.0);
    auto setup = make_setup(BPKind::BP3, mesh);
    const OperatorHandle op(Backend::Fused, setup);
    const ConstrainedOperator cop(op, boundary_bcs(mesh));
    const GeomFactors mass = mass_factors(mesh, setup->basis);
    std::vector<double> b = assemble_load(mesh, setup->basis, mass, setup->restriction, rhs);
    for (int d : cop.bcs().dofs) b[d] = 0.0;
    auto apply = [&](std::span<const double> u, std::vector<double>& w) { cop.apply(u, w); };
    std::vector<double> x(op.size(), 0.0);
    const std::vector<double> diag = jacobi_diagonal(cop);
    const CGReport report = cg(apply, b, x, 1e-8, 2000, &diag);
    if (b_out) std::memcpy(b_out, b.data(), sizeof(double) * b.size());
    if (x_out) std::memcpy(x_out, x.data(), sizeof(double) * x.size());
    *iterations = report.iterations;
    *err = discrete_l2_error(mesh, setup->basis, mass, setup->restriction, x, exact);
    return report.converged ? 0 : 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// kCsvHeader (bench.hpp:297-299): the CSV schema the harness mirror must keep.
const char* ref_csv_header() { return kCsvHeader; }

// run_bench through the reference's JSON config parser (bench.hpp:93-153,
// 214-295). Writes up to `cap` records: throughput (dofs*iters/s), seconds,
// dofs, threads. Returns the record count, or -1 on error (see ref_last_error).
int ref_run_bench_json(const char* json_text, double* throughput, double* seconds, int64_t* dofs, int* threads,
                       int cap) {
  try {
    const BenchConfig cfg = parse_config(nlohmann::json::parse(json_text));
    const RunOutput out = run_bench(cfg);
    if (!out.errors.empty()) {
      g_err = out.errors.front();
      return -1;
    }
    const int n = static_cast<int>(out.records.size());
    for (int i = 0; i < n && i < cap; ++i) {
      throughput[i] = out.records[i].throughput;
      seconds[i] = out.records[i].seconds;
      dofs[i] = out.records[i].dofs;
      threads[i] = out.records[i].threads;
    }
    return n;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// One case of the reference 72-case equivalence sweep (verify.hpp:50-108).
// out: [max_rel_multipass, max_rel_fused, max_symmetry, max_asymmetry_matrix,
//       nullspace_residual, min_quadratic_form, pass]
int ref_check_equivalence(int bp, int p, int ex, int ey, int ez, double a, double* out) {
  try {
    const EquivalenceResult r = check_equivalence({to_bp(bp), p, {ex, ey, ez}, a});
    out[0] = r.max_rel_multipass;
    out[1] = r.max_rel_fused;
    out[2] = r.max_symmetry;
    out[3] = r.max_asymmetry_matrix;
    out[4] = r.nullspace_residual;
    out[5] = r.min_quadratic_form;
    out[6] = r.pass ? 1.0 : 0.0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Per-element flop count of the reference fused kernel (operator.hpp:283-294).
void ref_count_flops(void* hv, uint64_t* mul, uint64_t* add) {
  auto* h = static_cast<RefHandle*>(hv);
  const FlopCount f = h->op->count_flops();
  *mul = f.mul;
  *add = f.add;
}

}  // extern "C"
