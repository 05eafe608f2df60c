// Device restatement of the reference's element tensor kernels in its exact
// arithmetic (tensor.hpp:50-235): every output entry is produced by one
// thread with contract_dim's summation order and unfused multiply / add, so
// results are bitwise identical to the host code. Used by the device
// geometry setup (setup.cu) and the multipass backend (multipass.cu).
// All threads of the CTA cooperate; each call ends with __syncthreads().
#pragma once
#include <cuda_runtime.h>

namespace hxb {
namespace tdev {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }

// contract_dim (tensor.hpp:50-114): Y[.. a ..] (+)= sum_m A(a, m) X[.. m ..]
// along `axis` of the x-fastest (n0, n1, n2) tensor x; A is m x n row-major.
__device__ inline void contract_dim_dev(const double* A, int m, int n, int axis, const double* x, int n0, int n1,
                                        int n2, double* y, bool accumulate) {
  if (axis == 0) {
    const int rest = n1 * n2;
    for (int o = threadIdx.x; o < rest * m; o += blockDim.x) {
      const int c = o / m, a = o % m;
      double sum = 0.0;
      for (int i = 0; i < n; ++i) sum = da(sum, dm(A[a * n + i], x[c * n0 + i]));
      y[c * m + a] = accumulate ? da(y[c * m + a], sum) : sum;
    }
  } else if (axis == 1) {
    for (int o = threadIdx.x; o < n2 * m * n0; o += blockDim.x) {
      const int i = o % n0, a = (o / n0) % m, k = o / (n0 * m);
      double* yp = y + k * n0 * m + a * n0 + i;
      double v = accumulate ? *yp : 0.0;
      for (int j = 0; j < n; ++j) v = da(v, dm(A[a * n + j], x[k * n0 * n1 + j * n0 + i]));
      *yp = v;
    }
  } else {
    const int plane = n0 * n1;
    for (int o = threadIdx.x; o < m * plane; o += blockDim.x) {
      const int i = o % plane, a = o / plane;
      double* yp = y + a * plane + i;
      double v = accumulate ? *yp : 0.0;
      for (int k = 0; k < n; ++k) v = da(v, dm(A[a * n + k], x[k * plane + i]));
      *yp = v;
    }
  }
  __syncthreads();
}

// elem_grad (tensor.hpp:177-203); ta: q n n, tb: q q n doubles.
__device__ inline void elem_grad_dev(const double* B, const double* D, int n, int q, bool colloc, const double* u,
                                     double* gr, double* gs, double* gt, double* ta, double* tb) {
  if (colloc) {
    contract_dim_dev(D, q, n, 0, u, n, n, n, gr, false);
    contract_dim_dev(D, q, n, 1, u, n, n, n, gs, false);
    contract_dim_dev(D, q, n, 2, u, n, n, n, gt, false);
    return;
  }
  contract_dim_dev(D, q, n, 0, u, n, n, n, ta, false);
  contract_dim_dev(B, q, n, 1, ta, q, n, n, tb, false);
  contract_dim_dev(B, q, n, 2, tb, q, q, n, gr, false);
  contract_dim_dev(B, q, n, 0, u, n, n, n, ta, false);
  contract_dim_dev(D, q, n, 1, ta, q, n, n, tb, false);
  contract_dim_dev(B, q, n, 2, tb, q, q, n, gs, false);
  contract_dim_dev(B, q, n, 1, ta, q, n, n, tb, false);
  contract_dim_dev(D, q, n, 2, tb, q, q, n, gt, false);
}

// elem_grad_transpose (tensor.hpp:207-235); Bt, Dt: n x q; ta, tc: q q n; tb: q n n.
__device__ inline void elem_grad_transpose_dev(const double* Bt, const double* Dt, int n, int q, bool colloc,
                                               const double* gr, const double* gs, const double* gt, double* out,
                                               double* ta, double* tb, double* tc) {
  if (colloc) {
    contract_dim_dev(Dt, n, q, 0, gr, q, q, q, out, false);
    contract_dim_dev(Dt, n, q, 1, gs, q, q, q, out, true);
    contract_dim_dev(Dt, n, q, 2, gt, q, q, q, out, true);
    return;
  }
  contract_dim_dev(Bt, n, q, 2, gs, q, q, q, ta, false);
  contract_dim_dev(Dt, n, q, 1, ta, q, q, n, tb, false);
  contract_dim_dev(Dt, n, q, 2, gt, q, q, q, tc, false);
  contract_dim_dev(Bt, n, q, 1, tc, q, q, n, tb, true);
  contract_dim_dev(Bt, n, q, 0, tb, q, n, n, out, false);
  contract_dim_dev(Bt, n, q, 2, gr, q, q, q, ta, false);
  contract_dim_dev(Bt, n, q, 1, ta, q, q, n, tb, false);
  contract_dim_dev(Dt, n, q, 0, tb, q, n, n, out, true);
}

// elem_interp / elem_interp_transpose (tensor.hpp:141-172); collocated: copy.
__device__ inline void elem_interp_dev(const double* B, int n, int q, bool colloc, const double* u, double* out,
                                       double* t0, double* t1) {
  if (colloc) {
    for (int o = threadIdx.x; o < n * n * n; o += blockDim.x) out[o] = u[o];
    __syncthreads();
    return;
  }
  contract_dim_dev(B, q, n, 0, u, n, n, n, t0, false);
  contract_dim_dev(B, q, n, 1, t0, q, n, n, t1, false);
  contract_dim_dev(B, q, n, 2, t1, q, q, n, out, false);
}

__device__ inline void elem_interp_transpose_dev(const double* Bt, int n, int q, bool colloc, const double* v,
                                                 double* out, double* t0, double* t1) {
  if (colloc) {
    for (int o = threadIdx.x; o < q * q * q; o += blockDim.x) out[o] = v[o];
    __syncthreads();
    return;
  }
  contract_dim_dev(Bt, n, q, 2, v, q, q, q, t0, false);
  contract_dim_dev(Bt, n, q, 1, t0, q, q, n, t1, false);
  contract_dim_dev(Bt, n, q, 0, t1, q, n, n, out, false);
}

}  // namespace tdev
}  // namespace hxb
