// Finite-element helpers of the manufactured-solution Poisson check
// (acceptance_main.cpp:181-222), on the device in the
// reference's arithmetic:
//   node coordinates      mesh.hpp:107-119 (box meshes; bitwise mesh.coords)
//   interp to quadrature  gather + elem_interp          (restriction.hpp:55-65,
//                         tensor.hpp:141-153): L-vector -> E x q^3
//   interp transpose      elem_interp_transpose + scatter_add
//                         (tensor.hpp:155-172, restriction.hpp:67-80):
//                         E x q^3 -> L-vector, ascending element order
// With them assemble_load (solver.hpp:207-239) and discrete_l2_error
// (solver.hpp:256-300) are compositions with a user function evaluated at the
// mapped quadrature points (api.py). Element order e = ex + nx (ey + ny ez)
// (mesh.hpp:71-82), point order a + q (b + q c).
#include <cuda_runtime.h>

#include "internal.h"
#include "tensor_dev.cuh"

namespace hxb {
namespace {

using tdev::da;
using tdev::dm;

struct FeCfg {
  int p, n, q, nx, ny, nz, Nx, Ny, Nz, colloc;
};

FeCfg fe_cfg(const Setup& s) {
  FeCfg c{};
  c.p = s.p;
  c.n = s.p + 1;
  c.q = s.q;
  c.nx = s.dims[0];
  c.ny = s.dims[1];
  c.nz = s.dims[2];
  c.Nx = c.nx * c.p + 1;
  c.Ny = c.ny * c.p + 1;
  c.Nz = c.nz * c.p + 1;
  c.colloc = s.kind == KIND_COLLOC;
  return c;
}

// mesh.hpp:107-119: x + L_d * a sin(2 pi x/Lx) sin(2 pi y/Ly) sin(2 pi z/Lz),
// the sines from the host (libm), products unfused in the reference's order
__global__ void node_coords_kernel(const FeCfg c, BoxGeometryArgs g, int z0n, double* __restrict__ out) {
  const long long n = static_cast<long long>(c.Nx) * c.Ny * c.Nz;
  for (long long node = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; node < n;
       node += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int X = static_cast<int>(node % c.Nx);
    const int Y = static_cast<int>((node / c.Nx) % c.Ny);
    const int Z = static_cast<int>(node / (static_cast<long long>(c.Nx) * c.Ny)) + z0n;
    double disp = 0.0;
    if (g.amplitude > 0.0) disp = dm(dm(dm(g.amplitude, g.sx[X]), g.sy[Y]), g.sz[Z]);
    out[node] = da(g.ax[X], dm(g.ext[0], disp));
    out[n + node] = da(g.ay[Y], dm(g.ext[1], disp));
    out[2 * n + node] = da(g.az[Z], dm(g.ext[2], disp));
  }
}

// one CTA per element: gather the nodal values, elem_interp -> out[e][qp]
__global__ void interp_qpts_kernel(const FeCfg c, const double* __restrict__ Bg, const double* __restrict__ v,
                                   double* __restrict__ out) {
  extern __shared__ double sm[];
  const int n = c.n, q = c.q, nen = n * n * n, q3 = q * q * q, big = n > q ? n : q;
  double* B = sm;
  double* u = B + q * n;
  double* t0 = u + nen;
  double* t1 = t0 + big * big * big;
  double* o = t1 + big * big * big;
  const long long e = blockIdx.x;
  const int ex = static_cast<int>(e % c.nx), ey = static_cast<int>((e / c.nx) % c.ny),
            ez = static_cast<int>(e / (static_cast<long long>(c.nx) * c.ny));
  for (int t = threadIdx.x; t < q * n; t += blockDim.x) B[t] = Bg[t];
  for (int l = threadIdx.x; l < nen; l += blockDim.x) {
    const int i = l % n, j = (l / n) % n, k = l / (n * n);
    const int X = ex * c.p + i, Y = ey * c.p + j, Z = ez * c.p + k;
    u[l] = v[X + static_cast<long long>(c.Nx) * (Y + static_cast<long long>(c.Ny) * Z)];
  }
  __syncthreads();
  tdev::elem_interp_dev(B, n, q, c.colloc, u, o, t0, t1);
  for (int t = threadIdx.x; t < q3; t += blockDim.x) out[e * q3 + t] = o[t];
}

// one CTA per element: elem_interp_transpose -> E-vector
__global__ void interp_transpose_kernel(const FeCfg c, const double* __restrict__ Btg, const double* __restrict__ vq,
                                        double* __restrict__ we) {
  extern __shared__ double sm[];
  const int n = c.n, q = c.q, nen = n * n * n, q3 = q * q * q, big = n > q ? n : q;
  double* Bt = sm;
  double* vs = Bt + q * n;
  double* t0 = vs + q3;
  double* t1 = t0 + big * big * big;
  double* o = t1 + big * big * big;
  const long long e = blockIdx.x;
  for (int t = threadIdx.x; t < q * n; t += blockDim.x) Bt[t] = Btg[t];
  for (int t = threadIdx.x; t < q3; t += blockDim.x) vs[t] = vq[e * q3 + t];
  __syncthreads();
  tdev::elem_interp_transpose_dev(Bt, n, q, c.colloc, vs, o, t0, t1);
  for (int t = threadIdx.x; t < nen; t += blockDim.x) we[e * nen + t] = o[t];
}

// scatter_add: every node sums its 1-8 element entries in ascending element order
__global__ void scatter_add_kernel(const FeCfg c, const double* __restrict__ we, double* __restrict__ w) {
  const int P = c.p, n = c.n, nen = n * n * n;
  const long long total = static_cast<long long>(c.Nx) * c.Ny * c.Nz;
  for (long long node = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; node < total;
       node += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int X = static_cast<int>(node % c.Nx);
    const int Y = static_cast<int>((node / c.Nx) % c.Ny);
    const int Z = static_cast<int>(node / (static_cast<long long>(c.Nx) * c.Ny));
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

size_t interp_smem(const FeCfg& c, bool transpose) {
  const int n = c.n, q = c.q, big = n > q ? n : q;
  return sizeof(double) * (q * n + (transpose ? q * q * q + n * n * n : n * n * n + q * q * q) + 2 * big * big * big);
}

}  // namespace

cudaError_t launch_node_coords(const Setup& s, const BoxGeometryArgs& g, double* out, cudaStream_t st) {
  const FeCfg c = fe_cfg(s);
  node_coords_kernel<<<148 * 8, 256, 0, st>>>(c, g, s.z0 * s.p, out);
  return cudaGetLastError();
}

cudaError_t launch_interp_to_qpts(const Setup& s, const double* v, double* out, cudaStream_t st) {
  const FeCfg c = fe_cfg(s);
  double* dB = nullptr;
  cudaError_t e = cudaMallocAsync(&dB, sizeof(double) * c.q * c.n, st);
  if (!e) e = cudaMemcpyAsync(dB, s.B, sizeof(double) * c.q * c.n, cudaMemcpyHostToDevice, st);
  if (!e) {
    const size_t sm = interp_smem(c, false);
    cudaFuncSetAttribute(&interp_qpts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    interp_qpts_kernel<<<static_cast<unsigned>(s.E), 128, sm, st>>>(c, dB, v, out);
    e = cudaGetLastError();
  }
  cudaFreeAsync(dB, st);
  return e;
}

cudaError_t launch_interp_transpose(const Setup& s, const double* vq, double* out, cudaStream_t st) {
  const FeCfg c = fe_cfg(s);
  const int n = c.n, q = c.q;
  double Bt[kMaxQ * (kMaxPG + 1)];
  for (int a = 0; a < q; ++a)
    for (int i = 0; i < n; ++i) Bt[i * q + a] = s.B[a * n + i];
  double *dBt = nullptr, *we = nullptr;
  cudaError_t e = cudaMallocAsync(&dBt, sizeof(double) * q * n, st);
  if (!e) e = cudaMallocAsync(&we, sizeof(double) * s.E * n * n * n, st);
  if (!e) e = cudaMemcpyAsync(dBt, Bt, sizeof(double) * q * n, cudaMemcpyHostToDevice, st);
  if (!e) {
    const size_t sm = interp_smem(c, true);
    cudaFuncSetAttribute(&interp_transpose_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm));
    interp_transpose_kernel<<<static_cast<unsigned>(s.E), 128, sm, st>>>(c, dBt, vq, we);
    e = cudaGetLastError();
  }
  if (!e) {
    scatter_add_kernel<<<148 * 8, 256, 0, st>>>(c, we, out);
    e = cudaGetLastError();
  }
  cudaFreeAsync(dBt, st);
  cudaFreeAsync(we, st);
  return e;
}

}  // namespace hxb
