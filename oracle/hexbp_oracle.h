/* oracle/hexbp_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hexbp CPU path (quadrature, basis,
 * structured mesh, geometric factors, sum-factorised element kernels,
 * restriction, constrained operator, CG, deterministic reductions). It is
 * the parity checker for the CUDA product path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * Every function cites the reference file:line it restates; the arithmetic
 * follows the reference's operation order (no FMA contraction), and
 * tests/test_oracle.py pins it bitwise against oracle/_ref (the reference
 * compiled in place) through the committed fixtures in tests/golden/.
 */
#ifndef HEXBP_ORACLE_H
#define HEXBP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* bp in {1,3,5}. Returns NULL on invalid input or degenerate geometry
 * (message via or_last_error()). */
void* or_create(int bp, int p, int ex, int ey, int ez, double amplitude);
/* element layers [z0, z1) of the (ex, ey, gez) box (multi-GPU slab) */
void* or_create_slab(int bp, int p, int ex, int ey, int gez, int z0, int z1, double amplitude);
void or_destroy(void* h);
const char* or_last_error(void);

int64_t or_size(void* h);
int or_num_elements(void* h);
int or_q(void* h);
int or_components(void* h);
void or_basis(void* h, double* B, double* D);
void or_rules(void* h, double* qpts, double* qwts, double* npts, double* nwts);
void or_factors(void* h, double* out); /* reference AoS layout */
void or_coords(void* h, double* out);  /* 3 doubles per node */
int64_t or_num_boundary(void* h);
void or_boundary(void* h, int32_t* out);

/* constrained: 0 = OperatorHandle::apply, 1 = ConstrainedOperator::apply */
int or_apply(void* h, int constrained, const double* u, double* w);
/* 0 ok, 2 divergence (pAp <= 0 or non-finite) */
int or_cg(void* h, int constrained, const double* b, double* x, double rel_tol, int max_iter, int* iterations,
          int* converged, double* final_rel, double* history);

/* jacobi_diagonal (solver.hpp:155-205); constrained: 1 on essential dofs */
void or_jacobi_diagonal(void* h, int constrained, double* out);
/* cg with Jacobi preconditioner z = r / diag (diag may be NULL) */
int or_pcg(void* h, int constrained, const double* b, double* x, const double* diag, double rel_tol, int max_iter,
           int* iterations, int* converged, double* final_rel, double* history);

double or_dot(const double* a, const double* b, int64_t n);
void or_bench_rhs(void* h, uint64_t seed, double* b);
void or_random_vector(uint64_t seed, int64_t n, double* out);
uint64_t or_mix_seed(uint64_t seed, int bp, int p, int ex, int ey, int ez);
int or_gl_rule(int n, double* pts, double* wts);
int or_gll_rule(int n, double* pts, double* wts);

#ifdef __cplusplus
}
#endif
#endif
