// Internal declarations shared by the hexbp-b200 translation units.
// Public C ABI: include/hexbp_b200.h.
#pragma once

#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point; no -lcuda)
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hexbp_b200.h"

namespace hxb {

// Element kernel families (operator.hpp:29,51,55-56):
//   MASS   = BP1, q = p+2 Gauss, one factor per point (wdetJ)
//   DIFF   = BP3, q = p+2 Gauss, six factors per point (G)
//   COLLOC = BP5, q = p+1 GLL (B = I exactly, basis.hpp:55-66), six factors
enum Kind : int { KIND_MASS = 0, KIND_DIFF = 1, KIND_COLLOC = 2 };

// Opt a kernel in to more than 48 KB of dynamic shared memory. The attribute
// is per device, so it is set once per (call site, device): `mask` is the call
// site's bit set of devices already configured.
inline void set_smem_attr_once(std::atomic<uint64_t>& mask, const void* fn, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  mask.fetch_or(bit, std::memory_order_release);
}

constexpr int kMaxP = 8;            // the fused kernels (apply*.cu): p = 1..8, the BASELINE range
constexpr int kMaxPG = 10;          // generic degrees 9..10: the multipass pipeline (multipass.cu)
constexpr int kMaxQ = kMaxPG + 2;   // basis table storage

// Device-resident CG state (solver.hpp:91-153); read/written only by kernels.
struct DevScalars {
  double rz, pAp, alpha, beta, r0, rnorm, rel_tol, pad0;
  int status, iterations, x_pending, max_iter;
  int precond, pad1;  // precond: Jacobi z = r / diag (beta from r.z, not r.r)
};
enum : int { ST_RUNNING = 0, ST_CONVERGED = 1, ST_DIVERGED = 2, ST_MAXITER = 3 };

// Position of node (i, j) of a column footprint on its lateral ring
// (4p nodes with i or j in {0, p}); see apply.cu.
__host__ __device__ inline int ring_index(int P, int i, int j) {
  if (j == 0 && i < P) return i;
  if (i == P && j < P) return P + j;
  if (j == P && i > 0) return 2 * P + (P - i);
  if (i == 0 && j > 0) return 3 * P + (P - j);
  return 0;
}

// Arguments of the fused operator kernel (passed by value, __grid_constant__).
struct ApplyArgs {
  const double* u;
  double* w;
  const double* G;          // factors, device layout (setup.cu)
  long long gstride;        // doubles per element block of G
  int g_aos;                // element block layout: 1 = [qp][comp] (DMMA kernel), 0 = [comp][a][b+q*c]
  int nx, ny, nz;           // elements of this (slab) mesh
  int Nx, Ny, Nz;           // local node grid
  int ncols;                // nx * ny
  int constrained;          // ConstrainedOperator semantics (solver.hpp:60-65)
  int bc_zlo, bc_zhi;       // z-faces that are essential (slab partitions)
  double* lateral;          // ring partials: exact mode [Z][column][4p]; fast mode latY (ring.cuh)
  double* zupper;           // exact mode: upper-layer ring partials of z-shared planes [ez][column][4p]
  double* col_dot;          // per-column partial p.Ap (nullptr: no dot)
  double* fix_partials;     // per-block partial p.Ap of the lateral fix-up
  unsigned int* fix_done;
  DevScalars* sc;           // CG scalars (nullptr: plain apply)
  double* dot_out;          // where the final dot lands (nullptr: CG alpha logic only)
  double* lat_x;            // fast mode: latX (ring.cuh)
  int zlo_shared;           // z-slab partition: node plane Z = 0 is owned by the rank below (its
                            // constrained nodes' u.u share of p.Ap is counted there)
  // Element range [zr0, zr1) of every column this launch marches (default
  // [0, nz)); kernels without range support (apply_overlap_supported) ignore it.
  int zr0, zr1;
  // Non-null: the range's bottom (carry_lo) / top (carry_hi) node plane is
  // not stored but left as this launch's share in [column][(p+1)^2] (j-major
  // footprint order), to be summed with the neighbouring launch's share by
  // launch_carry_combine -- the multi-GPU overlap of dist.cu.
  double* carry_lo;
  double* carry_hi;
  // Row-pitched input (the single-GPU fast CG's search direction, Workspace::pt):
  // node (X, Y, Z) of u at X + u_pitch (Y + Ny Z). u_pitch = 0: unpadded (Nx).
  // With u_tmap (host pointer, read by the launcher) the DMMA kernels stage
  // each element's 8^3 node block by one TMA tensor copy.
  int u_pitch;
  const CUtensorMap* u_tmap;
  int w_pitch;  // row pitch of w (0: Nx); the pitched fast CG's A p (Workspace::Apt)
};

struct Setup {
  int bp = 3, p = 1, q = 3, kind = KIND_DIFF, comp = 6;
  int dims[3] = {1, 1, 1};   // local element counts
  int gdims[3] = {1, 1, 1};  // global element counts
  int z0 = 0;                // first global element layer of this slab
  int bc_zlo = 1, bc_zhi = 1;
  int64_t nL = 0;
  int64_t E = 0;
  int device = 0;
  long long gstride = 0;
  int g_aos = 0;  // see ApplyArgs::g_aos; chosen per (kind, p) at setup (setup.cu)
  double B[kMaxQ * (kMaxPG + 1)] = {};
  double D[kMaxQ * (kMaxPG + 1)] = {};
  double qw[kMaxQ] = {};
  double* G = nullptr;  // device
  // box meshes (hexbp_setup_create_box*): the mesh parameters, so that node
  // coordinates can be regenerated on the device (fe_tools.cu)
  int box = 0;
  double ext[3] = {1.0, 1.0, 1.0};
  double amplitude = 0.0;
};

struct Workspace {
  const Setup* s = nullptr;
  int device = 0;
  double* lateral = nullptr;
  double* zupper = nullptr;
  double* col_dot = nullptr;
  double* fix_partials = nullptr;
  unsigned int* fix_done = nullptr;
  int fixup_grid = 0;
  DevScalars* sc = nullptr;
  double* r = nullptr;
  double* p = nullptr;
  double* Ap = nullptr;
  // Row-pitched copy of the search direction for the single-GPU fast CG on
  // the DMMA degrees (row pitch Nx rounded up to even: 16-byte row strides,
  // as a TMA tensor map requires), and its 3D tensor map (box = one element).
  // With it the solve keeps x, r and A p row-pitched as well (xt, rt, Apt),
  // so every vector kernel of the iteration is 32-byte aligned across its
  // operands; x is copied in and out once per solve.
  double* pt = nullptr;
  double* xt = nullptr;
  double* rt = nullptr;
  double* Apt = nullptr;
  int pt_pitch = 0;
  CUtensorMap pt_map;
  int use_pt = 0;  // set by the fast CG for the duration of a solve (capi.cu pcg_run)
  double* tmp_u = nullptr;  // host-API staging
  double* tmp_w = nullptr;
  double* tmp_d = nullptr;  // host-API Jacobi diagonal staging
  double* vec_partials = nullptr;
  unsigned int* vec_done = nullptr;
  double* history = nullptr;
  int history_cap = 0;
  int vec_blocks = 0;
  int exact = 1;                  // reduction mode (cg.cu): 1 = reference order, 0 = fused
  int fast_op = 0;                // HEXBP_MODE_FAST_OPERATOR: fast operator kernel under the exact CG
  const double* diag = nullptr;   // Jacobi diagonal of the running solve (nullptr: no preconditioner)
  int multipass = 0;              // HEXBP_BACKEND_MULTIPASS (multipass.cu)
  double* mp_buf = nullptr;       // its E-vectors, quadrature fields and basis tables
  double* dot_result = nullptr;
  DevScalars* host_sc = nullptr;  // pinned mirror
  // host-API solves: b streams in on copy_st while the initial A x0 runs
  size_t scatter_bytes = 0;  // transpose-restriction scratch (lateral + zupper): Workspace::global_bytes analog
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ev_x = nullptr, ev_b = nullptr;
  // fixed-iteration fast solves replay a CUDA graph of kCgGraphBlock
  // iterations (capi.cu pcg_run), captured on graph_st and cached per
  // (x, p, A p, Jacobi diagonal, constrained, arithmetic mode) -- the only
  // arguments the iteration's kernels take that can change between solves
  cudaStream_t graph_st = nullptr;
  cudaEvent_t ev_g0 = nullptr, ev_g1 = nullptr;
  struct CgGraph {
    cudaGraphExec_t exec = nullptr;
    const void* key[4] = {nullptr, nullptr, nullptr, nullptr};
    int con = -1;
  };
  CgGraph cg_graphs[4];  // a few argument sets (modes, vectors) stay captured
  int cg_graph_next = 0;
  int cg_graph_failed = 0;
};

// ---- apply.cu
// Setups whose fast operator kernel stages u by TMA tensor copies from a
// row-pitched vector (the DMMA kernels); tma.cu encodes the maps.
bool tma_u_supported(const Setup& s);
bool tma_u_staging_enabled();
int tma_u_pitch(const Setup& s);
cudaError_t encode_u_tensor_map(const Setup& s, const double* u, int pitch, CUtensorMap* map);
// finish_ring = false leaves the ring nodes of w as lateral partials (CG fast
// mode: launch_cg_update_r sums them).
ApplyArgs make_apply_args(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                          double* dot_out, DevScalars* sc);
cudaError_t launch_apply(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                         double* dot_out, DevScalars* sc, cudaStream_t st, bool finish_ring = true);
int fixup_grid(const Setup& s);
// ---- overlap.cu: boundary / interior split of a slab apply (dist.cu overlap)
struct OverlapBuffers {
  double* carry;         // overlap_carry_doubles(s)
  double* slots;         // [3] p.Ap partials of the boundary (2) and interior launches
  double* coldot;        // [3 * ncols] per-launch column partials
  unsigned int* tickets; // [4] zeroed last-CTA tickets
  double* partials;      // [overlap_partials_capacity()]
};
bool apply_overlap_supported(const Setup& s);
int64_t overlap_carry_doubles(const Setup& s);
int overlap_partials_capacity();
cudaError_t launch_apply_boundary(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                                  const OverlapBuffers& ob, cudaStream_t st);
cudaError_t launch_apply_interior(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                                  const OverlapBuffers& ob, cudaStream_t st);
// inner planes from the carries + their p.Ap share; *out = the rank's whole p.Ap share
cudaError_t launch_carry_combine(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                                 const OverlapBuffers& ob, double* out, cudaStream_t st);

// ---- apply_mma.cu (FP64 tensor-core kernel, BP3 p = 7)
bool mma_kernel_applies(const Setup& s);
// ---- apply_mma5.cu (FP64 tensor-core kernel, BP5 p = 7)
bool mma5_kernel_applies(const Setup& s);
cudaError_t launch_apply_mma5(const Setup& s, const ApplyArgs& a, cudaStream_t st);
void mma5_kernel_info(int* regs, int* smem, int* threads, int* blocks_per_sm);
cudaError_t launch_apply_mma(const Setup& s, const ApplyArgs& a, cudaStream_t st);
void mma_kernel_info(int* regs, int* smem, int* threads, int* blocks_per_sm);
// ---- apply_exact.cu (bit-exact reference arithmetic)
cudaError_t launch_apply_exact(const Setup& s, const ApplyArgs& a, int fix_grid, cudaStream_t st);
void apply_kernel_info(const Setup& s, int* regs, int* smem, int* threads, int* blocks_per_sm);

// ---- cg.cu
cudaError_t launch_cg_init(const Workspace& ws, const double* b, int64_t n, double rel_tol, int max_iter,
                           cudaStream_t st);
cudaError_t launch_cg_update_r(const Workspace& ws, int64_t n, cudaStream_t st, int constrained = 1);
// z-slab CG, fast mode: the r-update with the shared node planes already
// assembled in Ap (halo-summed), r.r over owned nodes only -> *rank_partial
cudaError_t launch_cgd_update_r_fused(const Workspace& ws, int constrained, double* rank_partial, cudaStream_t st);
// stream-ordered store of one int (a pageable cudaMemcpyAsync would synchronise the stream)
cudaError_t launch_set_int(int* p, int v, cudaStream_t st);
// transpose restriction part 2 for the node planes Z in [z_begin, z_end) only
cudaError_t launch_lateral_fixup_planes(const Setup& s, const Workspace& ws, const double* u, double* w,
                                        int constrained, int z_begin, int z_end, cudaStream_t st);
cudaError_t launch_cg_pap(const Workspace& ws, int64_t n, cudaStream_t st);
// fast mode: r = b - A x with A x from launch_apply(x, ..., finish_ring = false)
cudaError_t launch_cg_init_ring(const Workspace& ws, const double* b, const double* x, int64_t n, double rel_tol,
                                int max_iter, int constrained, cudaStream_t st);
// Jacobi PCG: rz = r.(r / diag) (reference order); at init sets rz, after an
// r-update sets beta = rz_next / rz (solver.hpp:105-108, 145-147)
cudaError_t launch_cg_rz(const Workspace& ws, int64_t n, cudaStream_t st);
// ---- multipass.cu: apply_multipass (operator.hpp:318-394) on the GPU
int64_t multipass_doubles(const Setup& s);
// upload = true: store the basis tables into buf's tail (once, synchronous) and return
cudaError_t launch_apply_multipass(const Setup& s, double* buf, const double* u, double* w, int constrained,
                                   cudaStream_t st, bool upload = false);
// ---- jacobi.cu: jacobi_diagonal (solver.hpp:155-205) in reference arithmetic
cudaError_t launch_jacobi_diagonal(const Setup& s, int constrained, double* diag, cudaStream_t st);
int64_t reduction_partials(int64_t n);
// Longest vector hexbp_dot can reduce with a workspace made for an L-vector of nL
// entries: one deterministic_dot chunk partial per vec_partials slot.
int64_t dot_capacity(int64_t nL);
cudaError_t launch_cgd_reduce(const Workspace& ws, int op, const double* b, int64_t n, int64_t owned, double* out,
                              cudaStream_t st);
cudaError_t launch_cgd_finish(const Workspace& ws, int op, const double* gathered, int world, double rel_tol,
                              int max_iter, cudaStream_t st);
cudaError_t launch_plane_combine(double* dst, const double* src, const double* u, int nxn, int nyn, int constrained,
                                 cudaStream_t st);
cudaError_t launch_cg_update_xp(const Workspace& ws, double* x, int64_t n, cudaStream_t st, double* p = nullptr);
cudaError_t launch_dot(const Workspace& ws, const double* a, const double* b, int64_t n, double* out,
                       cudaStream_t st);
int vec_grid(int64_t n);
cudaError_t launch_copy_rows(double* dst, int dst_pitch, const double* src, int src_pitch, int Nx, int64_t rows,
                             cudaStream_t st);

// ---- setup.cu
struct BoxGeometryArgs {
  const double* ax;  // axis node coordinates (global index)
  const double* ay;
  const double* az;
  const double* sx;  // sin(2 pi x / Lx) per axis node, host libm (mesh.hpp:107-116)
  const double* sy;
  const double* sz;
  double amplitude;
  double ext[3];
};
cudaError_t launch_box_geometry(const Setup& s, const BoxGeometryArgs& g, unsigned long long* bad_key,
                                double* bad_det, cudaStream_t st);
cudaError_t launch_factors_from_aos(const Setup& s, const double* aos, cudaStream_t st);
cudaError_t launch_factors_to_aos(const Setup& s, double* aos, cudaStream_t st);
// ---- fe_tools.cu: finite-element helpers of the Poisson check (solver.hpp:207-300)
cudaError_t launch_node_coords(const Setup& s, const BoxGeometryArgs& g, double* out, cudaStream_t st);
cudaError_t launch_interp_to_qpts(const Setup& s, const double* v, double* out, cudaStream_t st);
cudaError_t launch_interp_transpose(const Setup& s, const double* vq, double* out, cudaStream_t st);

// ---- basis.cpp (host)
void gl_rule(int n, double* pts, double* wts);
void gll_rule(int n, double* pts, double* wts);
void build_basis(int p, int q, bool gll, double* B, double* D, double* qpts, double* qwts, double* npts,
                 double* nwts);
std::vector<double> axis_node_coords(int elems, int p, double length);

void set_error(const std::string& msg);

}  // namespace hxb
