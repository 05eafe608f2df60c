// Device-resident conjugate-gradient recurrence (solver.hpp:91-153, no
// preconditioner, z = r). Per iteration (p.Ap and alpha are produced by the
// operator kernel, apply.cu):
//   cg_update_r  : r -= alpha Ap; ||r||^2 (fixed-order reduction); the last
//                  block records the residual history, applies the stopping
//                  rule rnorm/r0 <= rel_tol and computes beta = rr/rz.
//   cg_update_xp : x += alpha p (deferred from the reference's :132 so it
//                  fuses with the search-direction update); p = r + beta p.
// HBM traffic per iteration: 2 n (apply) + 3 n + 5 n = 10 n doubles + factors.
// All reductions use a fixed grid and fixed summation order, so the whole
// recurrence is bitwise reproducible run to run (solver.hpp:87-90).
#include <cuda_runtime.h>

#include "device_util.cuh"
#include "internal.h"

namespace hxb {
namespace {

constexpr int VT = 256;

__device__ __forceinline__ bool last_block(unsigned int* done) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  return s_last;
}

__device__ __forceinline__ double reduce_partials(const double* part, int nblk, double* red) {
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += VT) s += __ldcg(part + b);
  return block_sum<VT>(s, red);
}

// r = b - Ap; p = r; rr = r.r; r0 = sqrt(rr) (solver.hpp:102-124).
__global__ void __launch_bounds__(VT) cg_init_kernel(const double* __restrict__ b, const double* __restrict__ Ap,
                                                     double* __restrict__ r, double* __restrict__ p, long long n,
                                                     double* part, unsigned int* done, DevScalars* sc,
                                                     double* hist, double rel_tol, int max_iter) {
  __shared__ double red[VT / 32];
  double acc = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * VT;
  for (long long i = blockIdx.x * static_cast<long long>(VT) + threadIdx.x; i < n; i += stride) {
    const double v = b[i] - Ap[i];
    r[i] = v;
    p[i] = v;
    acc = fma(v, v, acc);
  }
  const double s = block_sum<VT>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (!last_block(done)) return;
  __threadfence();
  const double rr = reduce_partials(part, gridDim.x, red);
  if (threadIdx.x == 0) {
    const double r0 = sqrt(rr);
    hist[0] = r0;
    sc->r0 = r0;
    sc->rnorm = r0;
    sc->rz = rr;
    sc->rel_tol = rel_tol;
    sc->max_iter = max_iter;
    sc->iterations = 0;
    sc->x_pending = 0;
    if (!isfinite(r0))
      sc->status = ST_DIVERGED;
    else if (r0 == 0.0)
      sc->status = ST_CONVERGED;
    else if (max_iter <= 0)
      sc->status = ST_MAXITER;
    else
      sc->status = ST_RUNNING;
    *done = 0;
  }
}

// r -= alpha Ap; rr = r.r; stopping rule and beta (solver.hpp:133-147).
__global__ void __launch_bounds__(VT) cg_update_r_kernel(const double* __restrict__ Ap, double* __restrict__ r,
                                                         long long n, double* part, unsigned int* done,
                                                         DevScalars* sc, double* hist) {
  __shared__ double red[VT / 32];
  if (*(volatile int*)&sc->status != ST_RUNNING) return;
  const double alpha = sc->alpha;
  double acc = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * VT;
  for (long long i = blockIdx.x * static_cast<long long>(VT) + threadIdx.x; i < n; i += stride) {
    const double v = fma(-alpha, Ap[i], r[i]);
    r[i] = v;
    acc = fma(v, v, acc);
  }
  const double s = block_sum<VT>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (!last_block(done)) return;
  __threadfence();
  const double rr = reduce_partials(part, gridDim.x, red);
  if (threadIdx.x == 0) {
    const double rnorm = sqrt(rr);
    const int k = sc->iterations + 1;
    sc->iterations = k;
    sc->rnorm = rnorm;
    hist[k] = rnorm;
    sc->x_pending = 1;
    if (!isfinite(rnorm)) {
      sc->status = ST_DIVERGED;
    } else if (rnorm / sc->r0 <= sc->rel_tol) {
      sc->status = ST_CONVERGED;
    } else {
      sc->beta = rr / sc->rz;  // z = r: rz_next == r.r (solver.hpp:143-146)
      sc->rz = rr;
      if (k >= sc->max_iter) sc->status = ST_MAXITER;
    }
    *done = 0;
  }
}

// x += alpha p; p = r + beta p (solver.hpp:132,147).
__global__ void __launch_bounds__(VT) cg_update_xp_kernel(double* __restrict__ x, double* __restrict__ p,
                                                          const double* __restrict__ r, long long n,
                                                          unsigned int* done, DevScalars* sc) {
  if (*(volatile int*)&sc->x_pending == 0) return;
  const double alpha = sc->alpha, beta = sc->beta;
  const bool update_p = *(volatile int*)&sc->status == ST_RUNNING;
  const long long stride = static_cast<long long>(gridDim.x) * VT;
  if (update_p) {
    for (long long i = blockIdx.x * static_cast<long long>(VT) + threadIdx.x; i < n; i += stride) {
      const double pi = p[i];
      x[i] = fma(alpha, pi, x[i]);
      p[i] = fma(beta, pi, r[i]);
    }
  } else {
    for (long long i = blockIdx.x * static_cast<long long>(VT) + threadIdx.x; i < n; i += stride)
      x[i] = fma(alpha, p[i], x[i]);
  }
  if (!last_block(done)) return;
  if (threadIdx.x == 0) {
    sc->x_pending = 0;
    *done = 0;
  }
}

__global__ void __launch_bounds__(VT) dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                 long long n, double* part, unsigned int* done, double* out) {
  __shared__ double red[VT / 32];
  double acc = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * VT;
  for (long long i = blockIdx.x * static_cast<long long>(VT) + threadIdx.x; i < n; i += stride)
    acc = fma(a[i], b[i], acc);
  const double s = block_sum<VT>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (!last_block(done)) return;
  __threadfence();
  const double tot = reduce_partials(part, gridDim.x, red);
  if (threadIdx.x == 0) {
    *out = tot;
    *done = 0;
  }
}

}  // namespace

int vec_grid(int64_t n) {
  // Fixed function of n (never of timing): 148 SMs x 8 blocks of 256 threads,
  // fewer for small vectors.
  long long g = (n + VT - 1) / VT;
  if (g > 148 * 8) g = 148 * 8;
  return static_cast<int>(g < 1 ? 1 : g);
}

cudaError_t launch_cg_init(const Workspace& ws, const double* b, int64_t n, double rel_tol, int max_iter,
                           cudaStream_t st) {
  cg_init_kernel<<<vec_grid(n), VT, 0, st>>>(b, ws.Ap, ws.r, ws.p, n, ws.vec_partials, ws.vec_done, ws.sc,
                                             ws.history, rel_tol, max_iter);
  return cudaGetLastError();
}

cudaError_t launch_cg_update_r(const Workspace& ws, int64_t n, cudaStream_t st) {
  cg_update_r_kernel<<<vec_grid(n), VT, 0, st>>>(ws.Ap, ws.r, n, ws.vec_partials, ws.vec_done, ws.sc, ws.history);
  return cudaGetLastError();
}

cudaError_t launch_cg_update_xp(const Workspace& ws, double* x, int64_t n, cudaStream_t st) {
  cg_update_xp_kernel<<<vec_grid(n), VT, 0, st>>>(x, ws.p, ws.r, n, ws.vec_done, ws.sc);
  return cudaGetLastError();
}

cudaError_t launch_dot(const Workspace& ws, const double* a, const double* b, int64_t n, double* out,
                       cudaStream_t st) {
  dot_kernel<<<vec_grid(n), VT, 0, st>>>(a, b, n, ws.vec_partials, ws.vec_done, out);
  return cudaGetLastError();
}

}  // namespace hxb
