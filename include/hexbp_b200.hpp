// include/hexbp_b200.hpp -- C++ host mirror of the hexbp operator API over
// the C ABI (hexbp_b200.h). Header-only; link libhexbp_b200.so.
//
// A caller of the reference (/root/reference/proj/include/hexbp) finds the
// same surface, with Backend::Cuda as the new plugin value:
//   build_box_mesh (mesh.hpp:86)      -> hexbp::b200::build_box_mesh (metadata)
//   make_setup (operator.hpp:70)      -> hexbp::b200::make_setup (device geometry)
//   OperatorHandle (operator.hpp:244) -> apply(span, vector&), apply(..., Workspace&),
//                                        size(), make_workspace(), count_flops()
//   ConstrainedOperator (solver.hpp:48), cg / CGReport (solver.hpp:76-153)
//   divergence_error (solver.hpp:17), degenerate_element_error (geometry.hpp:19)
// Error codes of the C ABI are rethrown as the reference's exception types.
#pragma once

#include <array>
#include <chrono>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hexbp_b200.h"

namespace hexbp::b200 {

enum class BPKind { BP1, BP3, BP5 };
enum class Backend { Cuda, CudaMultipass };  // Backend::Fused / Backend::Multipass on the GPU
enum class Mode { Reference = HEXBP_MODE_REFERENCE, Fast = HEXBP_MODE_FAST, FastOperator = HEXBP_MODE_FAST_OPERATOR };

class divergence_error : public std::runtime_error {
 public:
  explicit divergence_error(const std::string& w) : std::runtime_error(w) {}
};
class degenerate_element_error : public std::runtime_error {
 public:
  explicit degenerate_element_error(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
  if (rc == HEXBP_OK) return;
  const std::string msg = hexbp_last_error();
  switch (rc) {
    case HEXBP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case HEXBP_DIVERGENCE: throw divergence_error(msg);
    case HEXBP_DEGENERATE: throw degenerate_element_error(msg);
    case HEXBP_LOGIC: throw std::logic_error(msg);
    case HEXBP_OUT_OF_MEMORY: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}

inline int bp_code(BPKind k) { return k == BPKind::BP1 ? 1 : (k == BPKind::BP3 ? 3 : 5); }

struct HexMesh {  // mesh.hpp:29-51 (coordinates are generated on the device)
  std::array<int, 3> dims{1, 1, 1};
  int degree = 1;
  std::array<double, 3> extent{1.0, 1.0, 1.0};
  double deform_amplitude = 0.0;
  int num_elements() const { return dims[0] * dims[1] * dims[2]; }
  int nodes_per_elem() const { return (degree + 1) * (degree + 1) * (degree + 1); }
  std::array<int, 3> node_grid() const {
    return {dims[0] * degree + 1, dims[1] * degree + 1, dims[2] * degree + 1};
  }
  int64_t num_nodes() const {
    const auto g = node_grid();
    return static_cast<int64_t>(g[0]) * g[1] * g[2];
  }
};

inline HexMesh build_box_mesh(std::array<int, 3> dims, int p, std::array<double, 3> extent, double a) {
  for (int d = 0; d < 3; ++d) {
    if (dims[d] < 1) throw std::invalid_argument("build_box_mesh: element counts must be >= 1");
    if (!(extent[d] > 0.0)) throw std::invalid_argument("build_box_mesh: extents must be positive");
  }
  if (p < 1) throw std::invalid_argument("build_box_mesh: degree must be >= 1");
  if (!(a >= 0.0 && a <= 0.15)) throw std::invalid_argument("build_box_mesh: deform amplitude outside [0, 0.15]");
  return HexMesh{dims, p, extent, a};
}

class OperatorSetup {  // operator.hpp:60-68, device resident
 public:
  explicit OperatorSetup(hexbp_setup_t h) : h_(h) { check(hexbp_setup_get_info(h_, &info_)); }
  ~OperatorSetup() { hexbp_setup_destroy(h_); }
  OperatorSetup(const OperatorSetup&) = delete;
  OperatorSetup& operator=(const OperatorSetup&) = delete;
  int l_size() const { return static_cast<int>(info_.l_size); }
  int num_elements() const { return static_cast<int>(info_.elements); }
  const hexbp_setup_info& info() const { return info_; }
  hexbp_setup_t handle() const { return h_; }

 private:
  hexbp_setup_t h_;
  hexbp_setup_info info_{};
};

inline std::shared_ptr<const OperatorSetup> make_setup(BPKind kind, const HexMesh& mesh, int device = 0) {
  hexbp_setup_t h = nullptr;
  check(hexbp_setup_create_box(bp_code(kind), mesh.degree, mesh.dims.data(), mesh.extent.data(),
                               mesh.deform_amplitude, device, &h));
  return std::make_shared<const OperatorSetup>(h);
}

class Workspace {  // operator.hpp:148-211
 public:
  explicit Workspace(const OperatorSetup& s) { check(hexbp_workspace_create(s.handle(), &h_)); }
  ~Workspace() {
    if (h_) hexbp_workspace_destroy(h_);
  }
  Workspace(Workspace&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  Workspace(const Workspace&) = delete;
  void set_mode(Mode m) { check(hexbp_workspace_set_mode(h_, static_cast<int>(m))); }
  void set_backend(Backend b) {
    check(hexbp_workspace_set_backend(h_, b == Backend::CudaMultipass ? HEXBP_BACKEND_MULTIPASS
                                                                      : HEXBP_BACKEND_FUSED));
  }
  int qpoint_fields() const {  // operator.hpp:193-194
    int q = 0;
    uint64_t b = 0;
    check(hexbp_workspace_info(h_, &q, &b));
    return q;
  }
  std::size_t global_bytes() const {  // operator.hpp:196-201
    int q = 0;
    uint64_t b = 0;
    check(hexbp_workspace_info(h_, &q, &b));
    return static_cast<std::size_t>(b);
  }
  hexbp_workspace_t handle() const { return h_; }

 private:
  hexbp_workspace_t h_ = nullptr;
};

struct FlopCount {  // tensor.hpp:19-29
  std::uint64_t mul = 0;
  std::uint64_t add = 0;
  std::uint64_t total() const { return mul + add; }
};

class OperatorHandle {
 public:
  OperatorHandle(Backend backend, std::shared_ptr<const OperatorSetup> setup)
      : backend_(backend), setup_(std::move(setup)), ws_(std::make_unique<Workspace>(make_workspace())) {}

  int size() const { return setup_->l_size(); }
  const OperatorSetup& setup() const { return *setup_; }
  Workspace make_workspace() const {  // operator.hpp:262
    Workspace w(*setup_);
    if (backend_ == Backend::CudaMultipass) w.set_backend(backend_);
    return w;
  }
  Backend backend() const { return backend_; }
  Workspace& workspace() const { return *ws_; }

  // operator.hpp:265-279 (host vectors; w is resized like the reference's :273)
  void apply(std::span<const double> u, std::vector<double>& w) const { apply(u, w, *ws_); }
  void apply(std::span<const double> u, std::vector<double>& w, Workspace& ws, FlopCount* flops = nullptr) const {
    apply_impl(u, w, ws, 0);
    if (flops) {
      const FlopCount f = count_flops();
      flops->mul += f.mul * setup_->num_elements();
      flops->add += f.add * setup_->num_elements();
    }
  }
  // device vectors, asynchronous on `stream`
  void apply_device(const double* u, double* w, bool constrained = false, void* stream = nullptr) const {
    check(hexbp_apply(setup_->handle(), ws_->handle(), u, w, constrained ? 1 : 0, stream));
  }
  FlopCount count_flops() const {  // operator.hpp:283-294
    FlopCount f;
    uint64_t m = 0, a = 0;
    check(hexbp_count_flops(setup_->handle(), &m, &a));
    f.mul = m;
    f.add = a;
    return f;
  }
  void apply_impl(std::span<const double> u, std::vector<double>& w, Workspace& ws, int constrained) const {
    if (static_cast<int>(u.size()) != size()) throw std::invalid_argument("apply: L-vector length mismatch");
    w.resize(u.size());
    check(hexbp_apply_host(setup_->handle(), ws.handle(), u.data(), w.data(), static_cast<int64_t>(u.size()),
                           constrained));
  }

 private:
  Backend backend_ = Backend::Cuda;
  std::shared_ptr<const OperatorSetup> setup_;
  std::unique_ptr<Workspace> ws_;
};

// solver.hpp:48-74 for the homogeneous box-surface constraints (boundary_bcs)
class ConstrainedOperator {
 public:
  explicit ConstrainedOperator(const OperatorHandle& op) : op_(op) {}
  int size() const { return op_.size(); }
  const OperatorHandle& raw() const { return op_; }
  void apply(std::span<const double> u, std::vector<double>& w) const { op_.apply_impl(u, w, op_.workspace(), 1); }

 private:
  const OperatorHandle& op_;
};

struct CGReport {  // solver.hpp:76-82
  int iterations = 0;
  bool converged = false;
  double final_rel_residual = 0.0;
  std::vector<double> residual_history;
  double seconds = 0.0;
};

namespace detail {
inline CGReport run_cg(const OperatorHandle& op, int constrained, std::span<const double> b, std::vector<double>& x,
                       double rel_tol, int max_iter, const std::vector<double>* diag = nullptr) {
  const auto t0 = std::chrono::steady_clock::now();
  if (x.size() != b.size()) throw std::invalid_argument("cg: x0 length mismatch");
  if (diag && diag->size() != b.size()) throw std::invalid_argument("cg: diagonal length mismatch");
  if (max_iter < 0) throw std::invalid_argument("cg: max_iter must be >= 0");
  CGReport r;
  std::vector<double> hist(static_cast<std::size_t>(max_iter) + 1);
  hexbp_cg_report rep{};
  check(hexbp_pcg_host(op.setup().handle(), op.workspace().handle(), b.data(), x.data(),
                       diag ? diag->data() : nullptr, static_cast<int64_t>(b.size()), rel_tol, max_iter, constrained,
                       &rep, hist.data()));
  r.iterations = rep.iterations;
  r.converged = rep.converged != 0;
  r.final_rel_residual = rep.final_rel_residual;
  hist.resize(static_cast<std::size_t>(rep.iterations) + 1);
  r.residual_history = std::move(hist);
  r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return r;
}
}  // namespace detail

// cg (solver.hpp:91-153) for device operators: the recurrence runs on the
// device; `diag` = Jacobi preconditioner (solver.hpp:105-108), as the reference.
inline CGReport cg(const OperatorHandle& op, std::span<const double> b, std::vector<double>& x, double rel_tol = 1e-8,
                   int max_iter = 2000, const std::vector<double>* diag = nullptr) {
  return detail::run_cg(op, 0, b, x, rel_tol, max_iter, diag);
}
inline CGReport cg(const ConstrainedOperator& op, std::span<const double> b, std::vector<double>& x,
                   double rel_tol = 1e-8, int max_iter = 2000, const std::vector<double>* diag = nullptr) {
  return detail::run_cg(op.raw(), 1, b, x, rel_tol, max_iter, diag);
}

// jacobi_diagonal (solver.hpp:155-205), computed on the device, bit for bit.
namespace detail {
inline std::vector<double> jacobi(const OperatorHandle& op, int constrained) {
  std::vector<double> out(static_cast<std::size_t>(op.size()));
  check(hexbp_jacobi_diagonal_host(op.setup().handle(), constrained, out.data()));
  return out;
}
}  // namespace detail
inline std::vector<double> jacobi_diagonal(const OperatorHandle& op) { return detail::jacobi(op, 0); }
inline std::vector<double> jacobi_diagonal(const ConstrainedOperator& op) { return detail::jacobi(op.raw(), 1); }

// ---- Multi-GPU: the z-slab operator and CG of one rank (hexbp_dist_*, NCCL
// owned by the library; one process per GPU). Rank 0 makes the id with
// nccl_unique_id() and the caller broadcasts its 128 bytes to the other ranks.
using NcclId = std::array<unsigned char, 128>;
inline NcclId nccl_unique_id() {
  NcclId id{};
  check(hexbp_dist_unique_id(id.data(), static_cast<int64_t>(id.size())));
  return id;
}

class DistributedOperator {
 public:
  // This rank's share (balanced split of the element layers, rank order = z
  // order) of the operator on build_box_mesh(global dims); collective.
  DistributedOperator(BPKind kind, const HexMesh& global_mesh, int world, int rank, const NcclId& id,
                      int device = 0, bool overlap = true) {
    check(hexbp_dist_create_box(bp_code(kind), global_mesh.degree, global_mesh.dims.data(), global_mesh.extent.data(),
                                global_mesh.deform_amplitude, world, rank, device, id.data(),
                                static_cast<int64_t>(id.size()), overlap ? 0 : HEXBP_DIST_NO_OVERLAP, &h_));
    check(hexbp_dist_info(h_, nullptr, &world_, &rank_, &n_, &owned_, &offset_));
  }
  ~DistributedOperator() {
    if (h_) hexbp_dist_destroy(h_);
  }
  DistributedOperator(const DistributedOperator&) = delete;
  DistributedOperator& operator=(const DistributedOperator&) = delete;

  int size() const { return static_cast<int>(n_); }        // local L-vector length
  int64_t owned_offset() const { return owned_; }          // plane 0 belongs to the rank below
  int64_t global_offset() const { return offset_; }        // global index of local node 0
  int world() const { return world_; }
  int rank() const { return rank_; }
  void set_mode(Mode m) { check(hexbp_dist_set_mode(h_, static_cast<int>(m))); }

  // OperatorHandle::apply / ConstrainedOperator::apply on this rank's slice
  // (w = the assembled local part of A u); collective
  void apply(std::span<const double> u, std::vector<double>& w, bool constrained = false) const {
    if (static_cast<int64_t>(u.size()) != n_) throw std::invalid_argument("apply: L-vector length mismatch");
    w.resize(u.size());
    check(hexbp_dist_apply_host(h_, u.data(), w.data(), n_, constrained ? 1 : 0));
  }
  void apply_device(const double* u, double* w, bool constrained = false, void* stream = nullptr) const {
    check(hexbp_dist_apply(h_, u, w, constrained ? 1 : 0, stream));
  }
  // cg (solver.hpp:91-153) on the partition; every rank returns the same report
  CGReport cg(std::span<const double> b, std::vector<double>& x, double rel_tol = 1e-8, int max_iter = 2000,
              bool constrained = true) const {
    const auto t0 = std::chrono::steady_clock::now();
    if (static_cast<int64_t>(b.size()) != n_ || x.size() != b.size())
      throw std::invalid_argument("cg: x0 length mismatch");
    if (max_iter < 0) throw std::invalid_argument("cg: max_iter must be >= 0");
    std::vector<double> hist(static_cast<std::size_t>(max_iter) + 1);
    hexbp_cg_report rep{};
    check(hexbp_dist_cg_host(h_, b.data(), x.data(), n_, rel_tol, max_iter, constrained ? 1 : 0, &rep, hist.data()));
    CGReport r;
    r.iterations = rep.iterations;
    r.converged = rep.converged != 0;
    r.final_rel_residual = rep.final_rel_residual;
    hist.resize(static_cast<std::size_t>(rep.iterations) + 1);
    r.residual_history = std::move(hist);
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return r;
  }
  hexbp_dist_t handle() const { return h_; }

 private:
  hexbp_dist_t h_ = nullptr;
  int world_ = 1, rank_ = 0;
  int64_t n_ = 0, owned_ = 0, offset_ = 0;
};

// run_bench's right-hand side (bench.hpp:234-243), BENCH_SEED default 20240101
inline std::vector<double> bench_rhs(BPKind kind, int p, std::array<int, 3> dims, uint64_t seed = 20240101ull) {
  const int64_t n = static_cast<int64_t>(dims[0] * p + 1) * (dims[1] * p + 1) * (dims[2] * p + 1);
  std::vector<double> b(static_cast<std::size_t>(n));
  check(hexbp_bench_rhs(bp_code(kind), p, dims.data(), seed, 0, n, b.data()));
  return b;
}

}  // namespace hexbp::b200
