// The drop-in, exercised from the reference's side: compiled against the
// UNMODIFIED reference headers (/root/reference/proj/include, where they lie)
// and the C ABI, the way INTEGRATION.md's Backend::Cuda binding would be.
//
//  * a reference OperatorSetup built by the reference's own make_setup
//    (operator.hpp:70-77) is adopted by hexbp_setup_create -- basis.B / D
//    (basis.hpp:21-22) and factors.data (geometry.hpp:48-56) as they are --
//    and its ElementRestriction::elem_to_global is validated by
//    hexbp_setup_check_restriction (restriction.hpp:22-53);
//  * CudaBackend::apply (hexbp_apply_host) stands where OperatorHandle::apply
//    dispatches (operator.hpp:274-278): bit for bit OperatorHandle(Fused) in
//    reference arithmetic, within 1e-12 (verify.hpp:76-83) in fast mode;
//  * the reference's own cg (solver.hpp:91-153) drives CudaBackend::apply
//    through its ApplyFn parameter on host vectors -- the run_bench lambda
//    path (bench.hpp:244-262), 2 PCIe copies per apply -- and reproduces the
//    residual history of cg over OperatorHandle(Fused) bit for bit;
//  * the constrained apply (ConstrainedOperator, solver.hpp:60-65, with
//    boundary_bcs(mesh, value) for any value: the values are not used) equals
//    the reference's ConstrainedOperator bit for bit.
// TEST INFRASTRUCTURE: built by oracle/Makefile (target dropin) into
// oracle/_ref/ only when /root/reference is present; the GPU box runs the
// prebuilt binary (tests/test_dropin_ref.py).
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "hexbp/mesh.hpp"
#include "hexbp/operator.hpp"
#include "hexbp/solver.hpp"
#include "hexbp_b200.h"

namespace {

int failures = 0;
#define EXPECT(cond, ...)              \
  do {                                 \
    if (!(cond)) {                     \
      std::printf("FAIL %s: ", #cond); \
      std::printf(__VA_ARGS__);        \
      std::printf("\n");               \
      ++failures;                      \
    }                                  \
  } while (0)

void check(int rc) {
  if (rc != HEXBP_OK) throw std::runtime_error(hexbp_last_error());
}

int bp_of(hexbp::BPKind k) { return k == hexbp::BPKind::BP1 ? 1 : (k == hexbp::BPKind::BP3 ? 3 : 5); }

// What OperatorHandle would hold for Backend::Cuda: the
// device setup adopted from the reference's host setup, and a workspace.
struct CudaBackend {
  hexbp_setup_t s = nullptr;
  hexbp_workspace_t w = nullptr;
  CudaBackend(const hexbp::OperatorSetup& setup, const hexbp::HexMesh& mesh, int mode) {
    const auto& b = setup.basis;
    check(hexbp_setup_create(bp_of(setup.kind), b.p, b.num_quad_1d(), mesh.dims.data(), b.B.data().data(),
                             b.D.data().data(), setup.factors.data.data(), 0, &s));
    check(hexbp_setup_check_restriction(s, setup.restriction.elem_to_global.data(),
                                        static_cast<int64_t>(setup.restriction.elem_to_global.size())));
    check(hexbp_workspace_create(s, &w));
    check(hexbp_workspace_set_mode(w, mode));
    check(hexbp_workspace_reserve(w, 4096, 1));
  }
  ~CudaBackend() {
    hexbp_workspace_destroy(w);
    hexbp_setup_destroy(s);
  }
  // OperatorHandle::apply(span, vector&) semantics (operator.hpp:265-279)
  void apply(std::span<const double> u, std::vector<double>& out, int constrained = 0) const {
    out.resize(u.size());
    check(hexbp_apply_host(s, w, u.data(), out.data(), static_cast<int64_t>(u.size()), constrained));
  }
};

double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1.0));
}

void run_case(hexbp::BPKind kind, int p, std::array<int, 3> dims, double a) {
  const hexbp::HexMesh mesh = hexbp::build_box_mesh(dims, p, {1.0, 1.0, 1.0}, a);
  const auto setup = hexbp::make_setup(kind, mesh);
  const hexbp::OperatorHandle ref(hexbp::Backend::Fused, setup);
  std::vector<double> u(static_cast<std::size_t>(ref.size()));
  for (std::size_t i = 0; i < u.size(); ++i) u[i] = std::cos(0.11 * static_cast<double>(i)) - 0.3;
  std::vector<double> wr, wc;
  ref.apply(u, wr);
  const std::string tag = "bp" + std::to_string(bp_of(kind)) + " p=" + std::to_string(p) + " " +
                          std::to_string(dims[0]) + "x" + std::to_string(dims[1]) + "x" + std::to_string(dims[2]);
  {
    CudaBackend cuda(*setup, mesh, HEXBP_MODE_REFERENCE);
    cuda.apply(u, wc);
    EXPECT(wc == wr, "%s: reference-mode apply differs from OperatorHandle(Fused)::apply", tag.c_str());
    if (kind != hexbp::BPKind::BP1) {
      for (double value : {0.0, 2.5}) {  // boundary values are not used by the apply (solver.hpp:60-65)
        const hexbp::ConstrainedOperator rc(ref, hexbp::boundary_bcs(mesh, value));
        std::vector<double> cr, cc;
        rc.apply(u, cr);
        cuda.apply(u, cc, 1);
        EXPECT(cc == cr, "%s: constrained apply differs (bc value %g)", tag.c_str(), value);
      }
    }
    // the reference's own cg driving the device apply through its ApplyFn
    const std::vector<double> b(u.size(), 1.0 / static_cast<double>(u.size()));
    std::vector<double> x1(u.size(), 0.0), x2(u.size(), 0.0);
    const int con = kind != hexbp::BPKind::BP1;
    const hexbp::ConstrainedOperator rcop(ref, hexbp::boundary_bcs(mesh, 0.0));
    std::vector<double> bb = b;
    if (con)
      for (int d : rcop.bcs().dofs) bb[d] = 0.0;
    const hexbp::CGReport r1 = con ? hexbp::cg([&](std::span<const double> v, std::vector<double>& o) { rcop.apply(v, o); },
                                               bb, x1, 1e-8, 3000)
                                   : hexbp::cg([&](std::span<const double> v, std::vector<double>& o) { ref.apply(v, o); },
                                               bb, x1, 1e-8, 3000);
    const hexbp::CGReport r2 =
        hexbp::cg([&](std::span<const double> v, std::vector<double>& o) { cuda.apply(v, o, con); }, bb, x2, 1e-8, 3000);
    EXPECT(r1.iterations == r2.iterations && r1.residual_history == r2.residual_history && x1 == x2,
           "%s: reference cg over the device apply: %d iterations vs %d", tag.c_str(), r2.iterations, r1.iterations);
    std::printf("%s: bitwise apply, reference cg %d iterations bit for bit\n", tag.c_str(), r2.iterations);
  }
  {
    CudaBackend fast(*setup, mesh, HEXBP_MODE_FAST);
    fast.apply(u, wc);
    const double e = rel(wc, wr);
    EXPECT(e <= 1e-12, "%s: fast-mode apply deviation %.3e", tag.c_str(), e);
  }
}

}  // namespace

int main() {
  run_case(hexbp::BPKind::BP3, 7, {3, 2, 3}, 0.1);
  run_case(hexbp::BPKind::BP5, 7, {2, 3, 2}, 0.1);
  run_case(hexbp::BPKind::BP1, 3, {4, 3, 2}, 0.05);
  run_case(hexbp::BPKind::BP3, 2, {5, 4, 3}, 0.0);
  // a restriction that is not the structured box numbering is refused
  {
    const hexbp::HexMesh mesh = hexbp::build_box_mesh({2, 2, 2}, 2, {1.0, 1.0, 1.0}, 0.0);
    auto setup = hexbp::make_setup(hexbp::BPKind::BP3, mesh);
    std::vector<int> perm = setup->restriction.elem_to_global;
    std::swap(perm[3], perm[4]);
    hexbp_setup_t s = nullptr;
    const auto& b = setup->basis;
    check(hexbp_setup_create(3, 2, b.num_quad_1d(), mesh.dims.data(), b.B.data().data(), b.D.data().data(),
                             setup->factors.data.data(), 0, &s));
    EXPECT(hexbp_setup_check_restriction(s, setup->restriction.elem_to_global.data(),
                                         static_cast<int64_t>(perm.size())) == HEXBP_OK,
           "structured table accepted");
    EXPECT(hexbp_setup_check_restriction(s, perm.data(), static_cast<int64_t>(perm.size())) ==
               HEXBP_INVALID_ARGUMENT,
           "permuted table refused");
    EXPECT(hexbp_setup_check_restriction(s, perm.data(), static_cast<int64_t>(perm.size()) - 1) ==
               HEXBP_INVALID_ARGUMENT,
           "short table refused");
    hexbp_setup_destroy(s);
  }
  std::printf("%s\n", failures ? "FAILED" : "ALL PASS");
  return failures ? 1 : 0;
}
