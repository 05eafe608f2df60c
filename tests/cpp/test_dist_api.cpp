// The multi-GPU entry of the C++ host mirror (hexbp::b200::DistributedOperator
// over hexbp_dist_*, NCCL owned by the library), driven like a reference
// caller drives OperatorHandle / cg (operator.hpp:265-279, solver.hpp:91-153).
// One GPU is available to the test box, so the communicator has one rank;
// the boundary / interior split of the overlapped apply (overlap.cu) and the
// NCCL collectives of the CG (all-gather of the scalar partials) still run.
// Checks: the distributed apply equals the single-GPU fast apply bit for bit
// (overlapped and not); the distributed CG reproduces the single-GPU fast
// CG's iteration count and final residual.
#include <cmath>
#include <cstdio>
#include <vector>

#include "hexbp_b200.hpp"

using namespace hexbp::b200;

static int failures = 0;
#define EXPECT(cond, ...)                  \
  do {                                     \
    if (!(cond)) {                         \
      std::printf("FAIL %s: ", #cond);     \
      std::printf(__VA_ARGS__);            \
      std::printf("\n");                   \
      ++failures;                          \
    }                                      \
  } while (0)

static void run_case(BPKind kind, int p, std::array<int, 3> dims) {
  const HexMesh mesh = build_box_mesh(dims, p, {1.0, 1.0, 1.0}, 0.1);
  const OperatorHandle op(Backend::Cuda, make_setup(kind, mesh));
  op.workspace().set_mode(Mode::Fast);
  std::vector<double> u(static_cast<std::size_t>(op.size()));
  for (std::size_t i = 0; i < u.size(); ++i) u[i] = std::sin(0.37 * static_cast<double>(i)) + 0.25;
  const std::vector<double> b = bench_rhs(kind, p, dims);
  for (int overlap = 0; overlap < 2; ++overlap) {
    const NcclId id = nccl_unique_id();
    DistributedOperator dop(kind, mesh, 1, 0, id, 0, overlap != 0);
    EXPECT(dop.size() == op.size() && dop.owned_offset() == 0 && dop.global_offset() == 0, "sizes");
    for (int con = 0; con < 2; ++con) {
      std::vector<double> w, wd;
      if (con) ConstrainedOperator(op).apply(u, w); else op.apply(u, w);
      dop.apply(u, wd, con != 0);
      bool same = w.size() == wd.size();
      for (std::size_t i = 0; same && i < w.size(); ++i) same = w[i] == wd[i];
      EXPECT(same, "bp%d p=%d %dx%dx%d overlap=%d constrained=%d: distributed apply != single-GPU apply",
             kind == BPKind::BP3 ? 3 : 5, p, dims[0], dims[1], dims[2], overlap, con);
    }
    std::vector<double> x(b.size(), 0.0), xd(b.size(), 0.0);
    const CGReport r = kind == BPKind::BP1 ? cg(op, b, x, 1e-8, 3000) : cg(ConstrainedOperator(op), b, x, 1e-8, 3000);
    const CGReport rd = dop.cg(b, xd, 1e-8, 3000, kind != BPKind::BP1);
    EXPECT(rd.iterations == r.iterations && rd.converged, "CG iterations %d vs %d", rd.iterations, r.iterations);
    // two fast-mode solves with different reduction trees (rank partials over
    // owned nodes vs the single-GPU fused tree): equal counts, residuals equal
    // up to the chaotic amplification of rounding (the north-star comparison
    // against the reference itself is tests/test_dist_nccl.py on the goldens)
    EXPECT(std::fabs(rd.final_rel_residual - r.final_rel_residual) <= 5e-10, "final %.17g vs %.17g",
           rd.final_rel_residual, r.final_rel_residual);
    double dx = 0.0, nx = 0.0;
    for (std::size_t i = 0; i < x.size(); ++i) {
      dx = std::fmax(dx, std::fabs(x[i] - xd[i]));
      nx = std::fmax(nx, std::fabs(x[i]));
    }
    EXPECT(dx <= 1e-8 * nx, "solution max deviation %.3e", dx / nx);
    std::printf("bp%d p=%d %dx%dx%d overlap=%d: %d iterations (single GPU %d), final %.6e\n",
                kind == BPKind::BP3 ? 3 : 5, p, dims[0], dims[1], dims[2], overlap, rd.iterations, r.iterations,
                rd.final_rel_residual);
  }
}

int main() {
  run_case(BPKind::BP3, 7, {4, 3, 6});  // DMMA kernel: boundary / interior split with two inner planes
  run_case(BPKind::BP3, 7, {3, 4, 2});  // one inner plane
  run_case(BPKind::BP5, 4, {3, 3, 4});  // kernels without range support: single launch, exchange after
  bool threw = false;
  try {
    const NcclId id = nccl_unique_id();
    DistributedOperator bad(BPKind::BP3, build_box_mesh({2, 2, 1}, 2, {1.0, 1.0, 1.0}, 0.0), 2, 0, id);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw, "fewer element layers than ranks throws std::invalid_argument");
  std::printf("%s\n", failures ? "FAILED" : "ALL PASS");
  return failures ? 1 : 0;
}
