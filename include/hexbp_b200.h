/* include/hexbp_b200.h -- C ABI of the B200-native hexbp hot path.
 *
 * Plain pointers and sizes only (no torch / CUDA types in the signatures;
 * streams are passed as `void*` holding a cudaStream_t, NULL = legacy
 * default stream). Every entry point names the reference interface it
 * replaces (paths under /root/reference/proj/include/hexbp/).
 *
 * Status codes map to the reference's exception types:
 *   HEXBP_OK                0
 *   HEXBP_INVALID_ARGUMENT  1  std::invalid_argument   (e.g. operator.hpp:268)
 *   HEXBP_DIVERGENCE        2  hexbp::divergence_error (solver.hpp:17-20,114,129-130,136)
 *   HEXBP_CUDA_ERROR        3  std::runtime_error
 *   HEXBP_OUT_OF_MEMORY     4  std::bad_alloc
 *   HEXBP_DEGENERATE        5  hexbp::degenerate_element_error (geometry.hpp:19-32,129)
 *   HEXBP_LOGIC             6  std::logic_error        (operator.hpp:258,284)
 * A human-readable message for the last failure on the calling thread is
 * returned by hexbp_last_error().
 */
#ifndef HEXBP_B200_H
#define HEXBP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HEXBP_OK = 0,
  HEXBP_INVALID_ARGUMENT = 1,
  HEXBP_DIVERGENCE = 2,
  HEXBP_CUDA_ERROR = 3,
  HEXBP_OUT_OF_MEMORY = 4,
  HEXBP_DEGENERATE = 5,
  HEXBP_LOGIC = 6
};

typedef struct hexbp_setup_s* hexbp_setup_t;         /* device OperatorSetup (operator.hpp:60-68) */
typedef struct hexbp_workspace_s* hexbp_workspace_t; /* device Workspace (operator.hpp:148-211)   */
typedef struct hexbp_dist_s* hexbp_dist_t;           /* z-slab operator + CG of one rank (NCCL)  */

typedef struct {
  int bp;            /* 1, 3 or 5 (BPKind, operator.hpp:29) */
  int p, q;          /* degree, quadrature points per axis (operator.hpp:55) */
  int dims[3];       /* local element counts */
  int gdims[3];      /* global element counts (== dims unless a slab) */
  int z0;            /* first global element layer of this slab */
  int components;    /* 1 (BP1 wdetJ) or 6 (BP3/BP5 G) (geometry.hpp:41-57) */
  int64_t l_size;    /* OperatorSetup::l_size (operator.hpp:66) */
  int64_t elements;  /* OperatorSetup::num_elements (operator.hpp:67) */
  int64_t factor_bytes;
} hexbp_setup_info;

typedef struct {
  int iterations;            /* CGReport::iterations       (solver.hpp:76-82) */
  int converged;             /* CGReport::converged        */
  double final_rel_residual; /* CGReport::final_rel_residual */
  double r0_norm;            /* residual_history[0]        */
  double seconds;            /* CGReport::seconds (host wall clock of the call) */
} hexbp_cg_report;

const char* hexbp_last_error(void);
int hexbp_device_count(void);

/* Replaces make_setup(kind, mesh) for the reference's structured box mesh
 * (operator.hpp:70-77, mesh.hpp:86-123, geometry.hpp:78-193): the mesh
 * coordinates, Jacobians and geometric factors are generated ON THE DEVICE
 * with the reference's operation order. extent = NULL means {1,1,1}.
 * Degrees: p = 1..8 run the fused kernels; p = 9, 10 (the reference accepts
 * any p, basis.hpp:86-111) run the multipass pipeline in reference
 * arithmetic -- their workspaces are created on HEXBP_BACKEND_MULTIPASS and
 * accept HEXBP_MODE_REFERENCE only; p > 10 is HEXBP_INVALID_ARGUMENT. */
int hexbp_setup_create_box(int bp, int p, const int dims[3], const double extent[3], double amplitude,
                           int device, hexbp_setup_t* out);

/* Slab of the same global box (z element layers [z0, z1)) for the multi-GPU
 * partition; its node planes are [z0*p, z1*p] of the global grid. */
int hexbp_setup_create_box_slab(int bp, int p, const int gdims[3], int z0, int z1, const double extent[3],
                                double amplitude, int device, hexbp_setup_t* out);

/* Replaces an existing host OperatorSetup: uploads the reference's own
 * tables -- B, D (q x (p+1) row-major, basis.hpp:21-22) and the factors in
 * the reference AoS layout data[(e*q^3+qp)*comp + c] (geometry.hpp:48-56) --
 * and re-lays them out for the device kernel. */
int hexbp_setup_create(int bp, int p, int q, const int dims[3], const double* B, const double* D,
                       const double* factors_aos, int device, hexbp_setup_t* out);

void hexbp_setup_destroy(hexbp_setup_t s);
/* The device kernels compute the structured restriction arithmetically
 * (global id of node (i,j,k) of element (ex,ey,ez), mesh.hpp:74-82) instead
 * of streaming ElementRestriction::elem_to_global (restriction.hpp:22-53).
 * A caller adopting a reference OperatorSetup passes its table here: OK iff it
 * is exactly that numbering for this setup's box (slab: the global ids of its
 * element layers); HEXBP_INVALID_ARGUMENT (with the first mismatching slot in
 * hexbp_last_error) otherwise -- a non-box restriction would give wrong results. */
int hexbp_setup_check_restriction(hexbp_setup_t s, const int32_t* elem_to_global, int64_t n);
int hexbp_setup_get_info(hexbp_setup_t s, hexbp_setup_info* out);
/* B, D as used by the kernels (q x (p+1) row-major). */
int hexbp_setup_basis(hexbp_setup_t s, double* B, double* D);
/* Factors downloaded back into the reference AoS layout (validation). */
int hexbp_setup_factors(hexbp_setup_t s, double* factors_aos);
/* Finite-element helpers of the manufactured-solution Poisson check
 * (acceptance_main.cpp:181-222; device, reference arithmetic). Element order
 * e = ex + nx (ey + ny ez) (mesh.hpp:71-82), quadrature point order
 * a + q (b + q c); all pointers are device memory.
 *   factors_device: the factors in the reference AoS layout (E x q^3 x comp)
 *   node_coords:    box setups only: out[c * l_size + node] = mesh.coords[node][c]
 *                   (mesh.hpp:107-119), bitwise
 *   interp_to_qpts: gather + elem_interp (restriction.hpp:55-65,
 *                   tensor.hpp:141-153): L-vector -> E x q^3
 *   interp_transpose: elem_interp_transpose + scatter_add (tensor.hpp:155-172,
 *                   restriction.hpp:67-80): E x q^3 -> L-vector (overwritten)
 * assemble_load (solver.hpp:207-239) = interp_transpose(wdetJ * f(x_q)) and
 * discrete_l2_error (solver.hpp:256-300) compose them (api.py). */
int hexbp_setup_factors_device(hexbp_setup_t s, double* out_dev, void* stream);
int hexbp_setup_node_coords(hexbp_setup_t s, double* out_dev, void* stream);
int hexbp_interp_to_qpts(hexbp_setup_t s, const double* v_dev, double* out_dev, void* stream);
int hexbp_interp_transpose(hexbp_setup_t s, const double* vq_dev, double* out_dev, void* stream);

/* Replaces OperatorHandle::make_workspace (operator.hpp:262): ticket/progress
 * flags, per-column partial sums, CG vectors and scalars, a 4096-iteration CG
 * history. Device-pointer apply / cg never allocate (cg within the reserved
 * history); the host-pointer entry points allocate their L-vector staging on
 * first use unless hexbp_workspace_reserve was called. */
int hexbp_workspace_create(hexbp_setup_t s, hexbp_workspace_t* out);
void hexbp_workspace_destroy(hexbp_workspace_t ws);
/* Optional explicit reservation (Workspace construction, operator.hpp:148-211,
 * allocates everything up front; test_operator.cpp:184-194): the device CG
 * history for solves of up to max_iter iterations (4096 are reserved at
 * creation) and, with host_staging != 0, the two L-vector staging buffers
 * of the host-pointer entry points (hexbp_apply_host / hexbp_cg_host /
 * hexbp_pcg_host, which otherwise allocate them on first use). After a
 * successful reserve, those calls allocate nothing for solves within it. */
int hexbp_workspace_reserve(hexbp_workspace_t ws, int max_iter, int host_staging);

/* Arithmetic mode of hexbp_apply / hexbp_cg on this workspace:
 *  HEXBP_MODE_REFERENCE (default): bit-exact reference arithmetic. The
 *    operator follows elem_grad / elem_grad_transpose / scatter_add's
 *    operation order with unfused multiply and add (tensor.hpp:50-235,
 *    restriction.hpp:67-80), the inner products follow deterministic_dot
 *    (dense.hpp:52-81) and the vector updates solver.hpp:103,132-147. The
 *    device CG reproduces the reference's iterates bit for bit (same
 *    iteration counts, same residual history).
 *  HEXBP_MODE_FAST: the throughput path. FMA sum-factorised kernel, p.Ap
 *    fused into the operator kernel, FMA updates, fixed-order tree
 *    reductions: operator within ~3e-16 of the reference per entry, bitwise
 *    reproducible run to run, iterates equal to the reference's up to
 *    rounding. hexbp_dot always uses the reference order.
 *  HEXBP_MODE_FAST_OPERATOR: the fast operator kernel under the reference's
 *    CG recurrence -- deterministic_dot-order inner products and the
 *    unfused vector updates of REFERENCE mode -- so a solve differs from the
 *    reference only by the operator's rounding (the parity-diagnosis mode). */
enum { HEXBP_MODE_REFERENCE = 0, HEXBP_MODE_FAST = 1, HEXBP_MODE_FAST_OPERATOR = 2 };

/* Operator backend of a workspace (Backend, operator.hpp:31):
 *  HEXBP_BACKEND_FUSED (default): one fused kernel per apply (Backend::Fused).
 *  HEXBP_BACKEND_MULTIPASS: OperatorHandle::apply_multipass (operator.hpp:
 *    318-394) on the GPU -- gather, gradient pass, factor pass, transpose
 *    pass, scatter_add, with the E-vectors and quadrature fields in HBM (the
 *    cuda-ref analog); always in reference arithmetic (bit
 *    for bit the reference's Multipass). Allocates 2 E (p+1)^3 + 6 E q^3
 *    doubles here (apply never allocates). */
enum { HEXBP_BACKEND_FUSED = 0, HEXBP_BACKEND_MULTIPASS = 1 };
int hexbp_workspace_set_backend(hexbp_workspace_t ws, int backend);
/* Workspace::qpoint_fields / global_bytes (operator.hpp:193-202): the global
 * quadrature-point fields owned (multipass: 2 x fields, fused: 0) and the
 * bytes of element-level global scratch (fused: the transpose-restriction
 * partial buffers, which replace the reference's E-vector; multipass: the
 * E-vectors and quadrature fields as well). */
int hexbp_workspace_info(hexbp_workspace_t ws, int* qpoint_fields, uint64_t* global_bytes);
int hexbp_workspace_set_mode(hexbp_workspace_t ws, int mode);

/* Replaces OperatorHandle::apply(u, w, ws) (operator.hpp:265-279) and, with
 * constrained = 1, ConstrainedOperator::apply (solver.hpp:60-65). Device
 * pointers of l_size doubles, asynchronous on `stream`. u and w must not
 * alias. */
int hexbp_apply(hexbp_setup_t s, hexbp_workspace_t ws, const double* u_dev, double* w_dev, int constrained,
                void* stream);

/* The fast-mode operator kernel alone (HEXBP_MODE_FAST workspaces only): as
 * hexbp_apply, except that the nodes shared between element columns (the
 * "ring" of each column footprint, 4p per node plane) are left as column
 * partial sums in the workspace instead of being summed into w -- the form
 * the fast CG consumes (its r-update adds them, restriction.hpp:67-80 order).
 * w is final on every other node. For fused callers and for timing the
 * dominant kernel. */
int hexbp_apply_ring_deferred(hexbp_setup_t s, hexbp_workspace_t ws, const double* u_dev, double* w_dev,
                              int constrained, void* stream);

/* The operator in the form the single-GPU fast CG launches it, on the
 * workspace's own search-direction buffer: ring nodes deferred as above and,
 * on the DMMA degrees (BP3 / BP5, p = 7), u staged by one TMA tensor copy per
 * element from the row-pitched search direction (tma.cu). u_dev (n unpadded
 * doubles) is first copied into that buffer; u_dev = NULL applies to its
 * current contents (timing loops). Clobbers the search direction of a solve
 * on this workspace. constrained = 0 / 1 as elsewhere; | 2 adds the CG's
 * fused p.Ap (the exact kernel variant the solve launches; result discarded). */
int hexbp_apply_cg_form(hexbp_setup_t s, hexbp_workspace_t ws, const double* u_dev, double* w_dev, int constrained,
                        void* stream);

/* Same, with HOST buffers of n doubles; synchronous (drop-in for the
 * reference's std::span / std::vector signature). */
int hexbp_apply_host(hexbp_setup_t s, hexbp_workspace_t ws, const double* u, double* w, int64_t n, int constrained);

/* Replaces cg(apply, b, x, rel_tol, max_iter) (solver.hpp:91-153) for a device
 * operator: the whole recurrence runs on the device (fused AXPY + fixed-order
 * reductions, p.Ap fused into the operator kernel). b_dev, x_dev: l_size
 * doubles on the device; x_dev holds x0 on entry. `history` (host, may be
 * NULL) receives residual_history (iterations+1 entries, capacity
 * max_iter+1). Synchronous. */
int hexbp_cg(hexbp_setup_t s, hexbp_workspace_t ws, const double* b_dev, double* x_dev, double rel_tol, int max_iter,
             int constrained, hexbp_cg_report* report, double* history, void* stream);

/* cg with the Jacobi preconditioner z = r / diag (solver.hpp:91-153 with
 * `diag`, :105-108): diag_dev holds l_size doubles on the device, NULL gives
 * hexbp_cg. Same reports, modes and error semantics as hexbp_cg; reference
 * mode reproduces the reference's preconditioned iterates bit for bit. */
int hexbp_pcg(hexbp_setup_t s, hexbp_workspace_t ws, const double* b_dev, double* x_dev, const double* diag_dev,
              double rel_tol, int max_iter, int constrained, hexbp_cg_report* report, double* history, void* stream);

/* jacobi_diagonal (solver.hpp:155-205) computed on the device in the
 * reference's arithmetic (bit for bit): the operator's diagonal, or with
 * constrained = 1 the ConstrainedOperator's (1 on the essential dofs).
 * diag_dev: l_size doubles. Setup-time call: allocates a temporary element
 * vector; synchronous. */
int hexbp_jacobi_diagonal(hexbp_setup_t s, int constrained, double* diag_dev, void* stream);

/* Same, into a HOST vector of l_size doubles. */
int hexbp_jacobi_diagonal_host(hexbp_setup_t s, int constrained, double* diag);

/* Same as hexbp_pcg with HOST b, x and diag (diag may be NULL). */
int hexbp_pcg_host(hexbp_setup_t s, hexbp_workspace_t ws, const double* b, double* x, const double* diag, int64_t n,
                   double rel_tol, int max_iter, int constrained, hexbp_cg_report* report, double* history);

/* Same with HOST b and x (x0 in, solution out). */
int hexbp_cg_host(hexbp_setup_t s, hexbp_workspace_t ws, const double* b, double* x, int64_t n, double rel_tol,
                  int max_iter, int constrained, hexbp_cg_report* report, double* history);

/* deterministic_dot (dense.hpp:74-81) on device vectors: fixed-order
 * partition, bitwise reproducible run to run. Synchronous. */
int hexbp_dot(hexbp_workspace_t ws, const double* a_dev, const double* b_dev, int64_t n, double* out, void* stream);

/* OperatorHandle::count_flops (operator.hpp:283-294): per-element multiplies
 * and adds executed by the device kernel (analytic trip counts). */
int hexbp_count_flops(hexbp_setup_t s, uint64_t* mul, uint64_t* add);

/* Seeded right-hand side of the reference benchmark (bench.hpp:234-243,
 * seed mixing bench.hpp:193-204; BENCH_SEED default 20240101): entries
 * [offset, offset+count) of the global L-vector of the (bp, p, dims) box,
 * boundary dofs zeroed for BP3/BP5. Generated with the same std::mt19937_64 /
 * uniform_real_distribution so the device solves the reference's system. */
int hexbp_bench_rhs(int bp, int p, const int dims[3], uint64_t seed, int64_t offset, int64_t count, double* out);
/* `count` draws of std::uniform_real_distribution<double>(lo, hi) over
 * std::mt19937_64(seed): check_equivalence's probe vectors (verify.hpp:64-70). */
int hexbp_uniform_stream(uint64_t seed, double lo, double hi, int64_t count, double* out);

/* ---- Multi-GPU z-slab building blocks (paper_2109_05072_b200/parallel.py).
 * The reference has no distributed path; these split hexbp_cg at its
 * reductions so that the rank partials can be all-gathered (NCCL) and
 * combined in rank order on every rank:
 *   apply(p) -> halo (plane exchange + hexbp_plane_combine) ->
 *   hexbp_cgd_reduce(PAP) -> all-gather -> hexbp_cgd_finish(PAP) ->
 *   hexbp_cgd_reduce(UPDATE_R) -> all-gather -> hexbp_cgd_finish(UPDATE_R) ->
 *   hexbp_cgd_update_xp.
 * Partials sum entries [owned_offset, l_size) in deterministic_dot order. */
enum { HEXBP_CGD_INIT = 0, HEXBP_CGD_PAP = 1, HEXBP_CGD_UPDATE_R = 2 };
/* Device pointers of the workspace CG vectors (l_size doubles each). */
int hexbp_workspace_vectors(hexbp_workspace_t ws, double** r, double** p, double** Ap);
/* INIT: r = b - Ap, p = r, partial r.r; PAP: partial p.Ap; UPDATE_R: r -= alpha Ap, partial r.r.
 * partial_dev: one device double. */
int hexbp_cgd_reduce(hexbp_workspace_t ws, int op, const double* b_dev, int64_t owned_offset, double* partial_dev,
                     void* stream);
/* Rank-order sum of `world` gathered partials (device) + the scalar recurrence. */
int hexbp_cgd_finish(hexbp_workspace_t ws, int op, const double* gathered_dev, int world, double rel_tol, int max_iter,
                     void* stream);
int hexbp_cgd_update_xp(hexbp_workspace_t ws, double* x_dev, void* stream);
/* Synchronous read of the device CG state: status 0 running, 1 converged, 2 diverged, 3 max_iter. */
int hexbp_cgd_report(hexbp_workspace_t ws, int* status, hexbp_cg_report* report, double* history, int history_cap);
/* Halo sum of one interface node plane (nxn x nyn): dst += src, box-boundary
 * nodes keep u when constrained. */
int hexbp_plane_combine(double* dst_dev, const double* src_dev, const double* u_dev, int nxn, int nyn, int constrained,
                        void* stream);
/* Fused z-slab iteration (fast mode; the single-GPU fast CG split at its two
 * global reductions):
 *   hexbp_cgd_apply_fused -> halo (plane exchange + hexbp_plane_combine on Ap)
 *   -> all-gather -> hexbp_cgd_finish(PAP) -> hexbp_cgd_update_r_fused ->
 *   all-gather -> hexbp_cgd_finish(UPDATE_R) -> hexbp_cgd_update_xp.
 * apply_fused: Ap = A p (workspace p) with this rank's share of p.Ap in
 * *partial_dev, fused into the operator kernel (the shares of the shared node
 * planes add up across ranks by linearity; constrained nodes of plane 0 count
 * on the rank below); the ring nodes of the shared planes are summed locally
 * so that Ap holds this rank's partial plane for the halo exchange. */
int hexbp_cgd_apply_fused(hexbp_setup_t setup, hexbp_workspace_t ws, int constrained, double* partial_dev,
                          void* stream);
/* r -= alpha Ap with the ring sums fused (shared planes read from the
 * halo-summed Ap); this rank's r.r over owned nodes -> *partial_dev. */
int hexbp_cgd_update_r_fused(hexbp_workspace_t ws, int constrained, double* partial_dev, void* stream);

/* ---- Multi-GPU z-slab operator and CG over NCCL (one process per GPU).
 * The reference's OperatorHandle::apply / cg (operator.hpp:265-279,
 * solver.hpp:91-153) on a partition of the box into contiguous element
 * layers per rank (rank order = z order); the library owns the NCCL
 * communicator. Rank 0 creates the id with hexbp_dist_unique_id and the
 * caller broadcasts its bytes (MPI, a file, torch.distributed) before every
 * rank calls hexbp_dist_create[_box]. Per operator apply: the boundary
 * element layers first, the shared-plane exchange (ncclSend/ncclRecv) while
 * the interior layers compute on a second stream, then the planes' halo sum
 * (dst + src on both ranks: bitwise equal copies). CG scalars: rank partials
 * over owned nodes, ncclAllGather, rank-order sum -- every rank runs the same
 * recurrence. HEXBP_DIST_NO_OVERLAP: one launch per apply, exchange after. */
enum { HEXBP_DIST_NO_OVERLAP = 1 };
int hexbp_dist_unique_id(void* id, int64_t bytes); /* >= 128 bytes (ncclUniqueId) */
/* Adopt this rank's slab setup (hexbp_setup_create_box_slab: layers [z0, z1)
 * of the global box); collective over the `world` ranks. */
int hexbp_dist_create(hexbp_setup_t slab, int world, int rank, const void* id, int64_t id_bytes, int flags,
                      hexbp_dist_t* out);
/* Same, building this rank's share of build_box_mesh(gdims, p, extent, amplitude)
 * (balanced split: rank r gets layers [r*b + min(r, m), ...) with gz = b*world + m). */
int hexbp_dist_create_box(int bp, int p, const int gdims[3], const double extent[3], double amplitude, int world,
                          int rank, int device, const void* id, int64_t id_bytes, int flags, hexbp_dist_t* out);
void hexbp_dist_destroy(hexbp_dist_t d);
/* This rank's setup, world, rank, local L-vector length, first owned local
 * index (plane 0 belongs to the rank below) and global index of local node 0. */
int hexbp_dist_info(hexbp_dist_t d, hexbp_setup_t* setup, int* world, int* rank, int64_t* l_size,
                    int64_t* owned_offset, int64_t* global_offset);
/* HEXBP_MODE_FAST (default: the fused iteration) or HEXBP_MODE_REFERENCE
 * (reference-arithmetic operator, deterministic_dot-order rank partials). */
int hexbp_dist_set_mode(hexbp_dist_t d, int mode);
/* w = assembled local part of A u (OperatorHandle::apply on the partition). Collective. */
int hexbp_dist_apply(hexbp_dist_t d, const double* u_dev, double* w_dev, int constrained, void* stream);
/* cg (solver.hpp:91-153) on the partition: b, x = this rank's local vectors
 * (x holds x0); every rank returns the same report. Collective. */
int hexbp_dist_cg(hexbp_dist_t d, const double* b_dev, double* x_dev, double rel_tol, int max_iter, int constrained,
                  hexbp_cg_report* report, double* history, void* stream);
/* The same with HOST vectors (this rank's slices; staged through the workspace). */
int hexbp_dist_apply_host(hexbp_dist_t d, const double* u, double* w, int64_t n, int constrained);
int hexbp_dist_cg_host(hexbp_dist_t d, const double* b, double* x, int64_t n, double rel_tol, int max_iter,
                       int constrained, hexbp_cg_report* report, double* history);

/* Kernel resource report: registers/thread, static+dynamic smem bytes,
 * threads per CTA, resident CTAs per SM. */
int hexbp_kernel_info(hexbp_setup_t s, int* regs, int* smem_bytes, int* threads, int* ctas_per_sm);

#ifdef __cplusplus
}
#endif
#endif /* HEXBP_B200_H */
