// GPU multipass backend: the unfused pipeline of
// OperatorHandle::apply_multipass (operator.hpp:318-394) as one kernel per
// pass, with the E-vectors and quadrature-point fields in HBM -- the B200
// analog of libCEED's cuda-ref backend, kept to reproduce the paper's
// fusion comparison (fused kernels vs a sequence of
// kernels with temporaries in global memory):
//   gather (restriction.hpp:55-65)          u      -> u_e       E n^3
//   gradient pass (elem_grad / elem_interp) u_e    -> grad_q    3 E q^3 (1 for BP1)
//   factor pass (copy + apply_*_factors)    grad_q -> flux_q    3 E q^3
//   transpose pass (elem_grad_transpose)    flux_q -> w_e       E n^3
//   scatter_add (restriction.hpp:67-80)     w_e    -> w         ascending slots
// In the reference's arithmetic (tensor_dev.cuh, unfused, reference loop
// orders), so the output equals the reference's Multipass backend bit for bit.
#include <cuda_runtime.h>

#include "device_util.cuh"
#include "internal.h"
#include "tensor_dev.cuh"

namespace hxb {
namespace {

using tdev::da;
using tdev::dm;

struct MpCfg {
  int p, n, q, comp, nx, ny, nz, Nx, Ny, Nz, aos, colloc, diff, constrained, bc_zlo, bc_zhi;
  long long gstride;
};

__device__ __forceinline__ long long fidx(const MpCfg& c, int m, int a, int b, int cc) {
  const int q = c.q;
  if (c.aos == 2) return ((static_cast<long long>(cc) * c.comp + m) * q + b) * q + a;
  if (c.aos) return static_cast<long long>(a + q * (b + q * cc)) * c.comp + m;
  return static_cast<long long>(m) * q * q * q + static_cast<long long>(a) * q * q + (b + q * cc);
}

__device__ __forceinline__ bool essential(const MpCfg& c, int X, int Y, int Z) {
  return c.constrained && (X == 0 || X == c.Nx - 1 || Y == 0 || Y == c.Ny - 1 || (Z == 0 && c.bc_zlo) ||
                           (Z == c.Nz - 1 && c.bc_zhi));
}

// gather: u_e[e nen + l] = u[node(e, l)], element order e = ex + nx (ey + ny ez);
// ConstrainedOperator: the essential entries of the copy are zeroed (solver.hpp:60-63)
__global__ void mp_gather_kernel(const MpCfg c, const double* __restrict__ u, double* __restrict__ ue, long long E) {
  const int n = c.n, nen = n * n * n;
  const long long total = E * nen;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long e = o / nen;
    const int l = static_cast<int>(o - e * nen);
    const int i = l % n, j = (l / n) % n, k = l / (n * n);
    const int ex = static_cast<int>(e % c.nx), ey = static_cast<int>((e / c.nx) % c.ny),
              ez = static_cast<int>(e / (static_cast<long long>(c.nx) * c.ny));
    const int X = ex * c.p + i, Y = ey * c.p + j, Z = ez * c.p + k;
    ue[o] = essential(c, X, Y, Z) ? 0.0 : u[X + static_cast<long long>(c.Nx) * (Y + static_cast<long long>(c.Ny) * Z)];
  }
}

// gradient pass (or interpolation for BP1): one CTA per element
__global__ void mp_grad_kernel(const MpCfg c, const double* __restrict__ Bg, const double* __restrict__ Dg,
                               const double* __restrict__ ue, double* __restrict__ gq) {
  extern __shared__ double sm[];
  const int n = c.n, q = c.q, nen = n * n * n, q3 = q * q * q, big = n > q ? n : q;
  double* B = sm;
  double* D = B + q * n;
  double* u = D + q * n;
  double* ta = u + nen;
  double* tb = ta + big * big * big;
  double* g = tb + big * big * big;  // 3 q3
  const long long e = blockIdx.x;
  for (int t = threadIdx.x; t < q * n; t += blockDim.x) {
    B[t] = Bg[t];
    D[t] = Dg[t];
  }
  for (int t = threadIdx.x; t < nen; t += blockDim.x) u[t] = ue[e * nen + t];
  __syncthreads();
  const long long E = static_cast<long long>(c.nx) * c.ny * c.nz;
  if (c.diff) {
    tdev::elem_grad_dev(B, D, n, q, c.colloc, u, g, g + q3, g + 2 * q3, ta, tb);
    for (int t = threadIdx.x; t < 3 * q3; t += blockDim.x) {
      const int f = t / q3, qp = t - f * q3;
      gq[(f * E + e) * q3 + qp] = g[t];
    }
  } else {
    tdev::elem_interp_dev(B, n, q, c.colloc, u, g, ta, tb);
    for (int t = threadIdx.x; t < q3; t += blockDim.x) gq[e * q3 + t] = g[t];
  }
}

// factor pass: flux = copy of grad, then apply_diffusion_factors / apply_mass_factors
// (operator.hpp:124-142) with the factors of the element's device slot
__global__ void mp_factor_kernel(const MpCfg c, const double* __restrict__ G, const double* __restrict__ gq,
                                 double* __restrict__ fq, long long E) {
  const int q = c.q, q3 = q * q * q;
  const long long total = E * q3;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long e = o / q3;
    const int qp = static_cast<int>(o - e * q3);
    const int a = qp % q, b = (qp / q) % q, cc = qp / (q * q);
    const int ex = static_cast<int>(e % c.nx), ey = static_cast<int>((e / c.nx) % c.ny),
              ez = static_cast<int>(e / (static_cast<long long>(c.nx) * c.ny));
    const double* Ge = G + ((static_cast<long long>(ex) + static_cast<long long>(c.nx) * ey) * c.nz + ez) * c.gstride;
    if (c.diff) {
      const double r = gq[o], s = gq[E * q3 + o], t = gq[2 * E * q3 + o];
      double gv[6];
      for (int m = 0; m < 6; ++m) gv[m] = Ge[fidx(c, m, a, b, cc)];
      fq[o] = da(da(dm(gv[0], r), dm(gv[1], s)), dm(gv[2], t));
      fq[E * q3 + o] = da(da(dm(gv[1], r), dm(gv[3], s)), dm(gv[4], t));
      fq[2 * E * q3 + o] = da(da(dm(gv[2], r), dm(gv[4], s)), dm(gv[5], t));
    } else {
      fq[o] = dm(gq[o], Ge[fidx(c, 0, a, b, cc)]);
    }
  }
}

// transpose pass: one CTA per element, flux -> w_e
__global__ void mp_gradT_kernel(const MpCfg c, const double* __restrict__ Btg, const double* __restrict__ Dtg,
                                const double* __restrict__ fq, double* __restrict__ we) {
  extern __shared__ double sm[];
  const int n = c.n, q = c.q, nen = n * n * n, q3 = q * q * q, big = n > q ? n : q;
  double* Bt = sm;
  double* Dt = Bt + q * n;
  double* f = Dt + q * n;  // 3 q3
  double* out = f + 3 * q3;
  double* ta = out + nen;
  double* tb = ta + big * big * big;
  double* tc = tb + big * big * big;
  const long long e = blockIdx.x;
  const long long E = static_cast<long long>(c.nx) * c.ny * c.nz;
  for (int t = threadIdx.x; t < q * n; t += blockDim.x) {
    Bt[t] = Btg[t];
    Dt[t] = Dtg[t];
  }
  const int nf = c.diff ? 3 : 1;
  for (int t = threadIdx.x; t < nf * q3; t += blockDim.x) {
    const int fi = t / q3, qp = t - fi * q3;
    f[t] = fq[(fi * E + e) * q3 + qp];
  }
  __syncthreads();
  if (c.diff)
    tdev::elem_grad_transpose_dev(Bt, Dt, n, q, c.colloc, f, f + q3, f + 2 * q3, out, ta, tb, tc);
  else
    tdev::elem_interp_transpose_dev(Bt, n, q, c.colloc, f, out, ta, tb);
  for (int t = threadIdx.x; t < nen; t += blockDim.x) we[e * nen + t] = out[t];
}

// scatter_add: every node sums its element slots in ascending slot order;
// ConstrainedOperator rows w = u (solver.hpp:64)
__global__ void mp_scatter_kernel(const MpCfg c, const double* __restrict__ we, const double* __restrict__ u,
                                  double* __restrict__ w) {
  const int P = c.p, n = c.n, nen = n * n * n;
  const long long total = static_cast<long long>(c.Nx) * c.Ny * c.Nz;
  for (long long node = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; node < total;
       node += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int X = static_cast<int>(node % c.Nx);
    const int Y = static_cast<int>((node / c.Nx) % c.Ny);
    const int Z = static_cast<int>(node / (static_cast<long long>(c.Nx) * c.Ny));
    if (essential(c, X, Y, Z)) {
      w[node] = u[node];
      continue;
    }
    auto range = [&](int V, int ne, int& lo, int& hi) {
      hi = V / P < ne ? V / P : ne - 1;
      lo = (V % P == 0 && V > 0) ? V / P - 1 : hi;
    };
    int xl, xh, yl, yh, zl, zh;
    range(X, c.nx, xl, xh);
    range(Y, c.ny, yl, yh);
    range(Z, c.nz, zl, zh);
    double s = 0.0;
    for (int ez = zl; ez <= zh; ++ez)
      for (int ey = yl; ey <= yh; ++ey)
        for (int ex = xl; ex <= xh; ++ex) {
          const long long e = ex + static_cast<long long>(c.nx) * (ey + static_cast<long long>(c.ny) * ez);
          s = da(s, we[e * nen + (X - ex * P) + n * ((Y - ey * P) + n * (Z - ez * P))]);
        }
    w[node] = s;
  }
}

}  // namespace

int64_t multipass_doubles(const Setup& s) {
  const int64_t nen = static_cast<int64_t>(s.p + 1) * (s.p + 1) * (s.p + 1);
  const int64_t q3 = static_cast<int64_t>(s.q) * s.q * s.q;
  const int nf = s.kind == KIND_MASS ? 1 : 3;
  return 2 * s.E * nen + 2 * nf * s.E * q3 + 4 * static_cast<int64_t>(s.q) * (s.p + 1);
}

cudaError_t launch_apply_multipass(const Setup& s, double* buf, const double* u, double* w, int constrained,
                                   cudaStream_t st, bool upload) {
  MpCfg c{};
  c.p = s.p;
  c.n = s.p + 1;
  c.q = s.q;
  c.comp = s.comp;
  c.nx = s.dims[0];
  c.ny = s.dims[1];
  c.nz = s.dims[2];
  c.Nx = c.nx * c.p + 1;
  c.Ny = c.ny * c.p + 1;
  c.Nz = c.nz * c.p + 1;
  c.aos = s.g_aos;
  c.colloc = s.kind == KIND_COLLOC;
  c.diff = s.kind != KIND_MASS;
  c.constrained = constrained;
  c.bc_zlo = s.bc_zlo;
  c.bc_zhi = s.bc_zhi;
  c.gstride = s.gstride;
  const int n = c.n, q = c.q, nen = n * n * n, q3 = q * q * q, big = n > q ? n : q;
  const int nf = c.diff ? 3 : 1;
  // workspace: u_e, w_e (E nen each), grad_q, flux_q (nf E q3 each), B, D, Bt, Dt
  double* ue = buf;
  double* we = ue + s.E * nen;
  double* gq = we + s.E * nen;
  double* fq = gq + nf * s.E * q3;
  double* dB = fq + nf * s.E * q3;
  double* dD = dB + q * n;
  double* dBt = dD + q * n;
  double* dDt = dBt + q * n;
  double Bt[kMaxQ * (kMaxPG + 1)], Dt[kMaxQ * (kMaxPG + 1)];
  for (int a = 0; a < q; ++a)
    for (int i = 0; i < n; ++i) {
      Bt[i * q + a] = s.B[a * n + i];
      Dt[i * q + a] = s.D[a * n + i];
    }
  if (upload) {  // once, at hexbp_workspace_set_backend (a pageable copy synchronises the stream)
    cudaError_t e = cudaMemcpy(dB, s.B, sizeof(double) * q * n, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemcpy(dD, s.D, sizeof(double) * q * n, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemcpy(dBt, Bt, sizeof(double) * q * n, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemcpy(dDt, Dt, sizeof(double) * q * n, cudaMemcpyHostToDevice);
    return e;
  }
  const size_t smg = sizeof(double) * (2 * q * n + nen + 2 * big * big * big + 3 * q3);
  const size_t smt = sizeof(double) * (2 * q * n + 3 * q3 + nen + 3 * big * big * big);
  static std::atomic<uint64_t> cfg_grad{0}, cfg_gradT{0};
  // 100 KB covers both passes up to p = 10 (BP3: 82 / 96 KB)
  set_smem_attr_once(cfg_grad, reinterpret_cast<const void*>(&mp_grad_kernel), 100 * 1024);
  set_smem_attr_once(cfg_gradT, reinterpret_cast<const void*>(&mp_gradT_kernel), 100 * 1024);
  if (smg > 100 * 1024 || smt > 100 * 1024) return cudaErrorInvalidValue;
  const int grid = 148 * 8;
  mp_gather_kernel<<<grid, 256, 0, st>>>(c, u, ue, s.E);
  mp_grad_kernel<<<static_cast<unsigned>(s.E), 256, smg, st>>>(c, dB, dD, ue, gq);
  mp_factor_kernel<<<grid, 256, 0, st>>>(c, s.G, gq, fq, s.E);
  mp_gradT_kernel<<<static_cast<unsigned>(s.E), 256, smt, st>>>(c, dBt, dDt, fq, we);
  mp_scatter_kernel<<<grid, 256, 0, st>>>(c, we, u, w);
  return cudaGetLastError();
}

}  // namespace hxb
