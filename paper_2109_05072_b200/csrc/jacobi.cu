// jacobi_diagonal (solver.hpp:155-205) on the device, in the reference's
// arithmetic: the diagonal entry of A^e at local node (i, j, k) is
//   BP3/BP5: sum_{c,b,a} g0 dr^2 + g3 ds^2 + g5 dt^2 + 2 (g1 dr ds + g2 dr dt + g4 ds dt)
//            dr = D(a,i) B(b,j) B(c,k), ds = B(a,i) D(b,j) B(c,k), dt = B(a,i) B(b,j) D(c,k)
//   BP1:     sum_{c,b,a} wdetJ phi^2, phi = B(a,i) B(b,j) B(c,k)
// with the loops (k, j, i outside; c, b, a inside) and the expression
// evaluated in the reference's order with unfused multiply / add
// (solver.hpp:175-190), then scatter_add's ascending-element summation
// (restriction.hpp:67-80). The result equals the reference's vector bit for
// bit. Setup-time work (O(E n^3 q^3) flops, like the reference); the element
// diagonals go through a temporary E-vector.
#include <cuda_runtime.h>

#include "device_util.cuh"
#include "internal.h"

namespace hxb {
namespace {

#define DM(a, b) __dmul_rn((a), (b))
#define DA(a, b) __dadd_rn((a), (b))

struct JacCfg {
  int p, n, q, comp, nx, ny, nz, aos, diff;
  long long gstride;
};

// one CTA per element slot (column-major, setup.cu), one thread per local node
__global__ void jacobi_elem_kernel(const JacCfg c, const double* __restrict__ G, const double* __restrict__ Bg,
                                   const double* __restrict__ Dg, double* __restrict__ de) {
  extern __shared__ double sm[];
  const int n = c.n, q = c.q, q3 = q * q * q, nen = n * n * n;
  double* B = sm;           // q x n
  double* D = B + q * n;    // q x n
  double* g = D + q * n;    // [qp][comp], qp = a + q (b + q c)
  const long long slot = blockIdx.x;
  const int ez = static_cast<int>(slot % c.nz), col = static_cast<int>(slot / c.nz);
  const int ex = col % c.nx, ey = col / c.nx;
  for (int t = threadIdx.x; t < q * n; t += blockDim.x) {
    B[t] = Bg[t];
    D[t] = Dg[t];
  }
  const double* Ge = G + slot * c.gstride;
  for (int t = threadIdx.x; t < q3 * c.comp; t += blockDim.x) {
    const int qp = t / c.comp, m = t - qp * c.comp;
    const int a = qp % q, b = (qp / q) % q, cc = qp / (q * q);
    const long long off = c.aos == 2 ? ((static_cast<long long>(cc) * c.comp + m) * q + b) * q + a
                          : c.aos    ? static_cast<long long>(qp) * c.comp + m
                                     : static_cast<long long>(m) * q3 + static_cast<long long>(a) * q * q + (b + q * cc);
    g[t] = Ge[off];
  }
  __syncthreads();
  for (int l = threadIdx.x; l < nen; l += blockDim.x) {
  const int i = l % n, j = (l / n) % n, k = l / (n * n);
  double sum = 0.0;
  for (int cc = 0; cc < q; ++cc)
    for (int b = 0; b < q; ++b)
      for (int a = 0; a < q; ++a) {
        const int qp = a + q * (b + q * cc);
        if (c.diff) {
          const double* gq = g + qp * 6;
          const double dr = DM(DM(D[a * n + i], B[b * n + j]), B[cc * n + k]);
          const double ds = DM(DM(B[a * n + i], D[b * n + j]), B[cc * n + k]);
          const double dt = DM(DM(B[a * n + i], B[b * n + j]), D[cc * n + k]);
          const double t1 = DA(DA(DM(DM(gq[0], dr), dr), DM(DM(gq[3], ds), ds)), DM(DM(gq[5], dt), dt));
          const double t2 = DA(DA(DM(DM(gq[1], dr), ds), DM(DM(gq[2], dr), dt)), DM(DM(gq[4], ds), dt));
          sum = DA(sum, DA(t1, DM(2.0, t2)));
        } else {
          const double phi = DM(DM(B[a * n + i], B[b * n + j]), B[cc * n + k]);
          sum = DA(sum, DM(DM(g[qp], phi), phi));
        }
      }
  // E-vector in the reference's element order e = ex + nx (ey + ny ez)
  const long long e = ex + static_cast<long long>(c.nx) * (ey + static_cast<long long>(c.ny) * ez);
  de[e * nen + l] = sum;
  }
}

// scatter_add: each node sums its 1-8 element entries in ascending element
// order (ez, then ey, then ex); ConstrainedOperator diagonal: 1 on essential dofs.
__global__ void jacobi_gather_kernel(const JacCfg c, const double* __restrict__ de, double* __restrict__ diag,
                                     int constrained, int bc_zlo, int bc_zhi) {
  const int P = c.p, n = c.n, nen = n * n * n;
  const int Nx = c.nx * P + 1, Ny = c.ny * P + 1, Nz = c.nz * P + 1;
  const long long total = static_cast<long long>(Nx) * Ny * Nz;
  for (long long node = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; node < total;
       node += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int X = static_cast<int>(node % Nx);
    const int Y = static_cast<int>((node / Nx) % Ny);
    const int Z = static_cast<int>(node / (static_cast<long long>(Nx) * Ny));
    if (constrained && (X == 0 || X == Nx - 1 || Y == 0 || Y == Ny - 1 || (Z == 0 && bc_zlo) ||
                        (Z == Nz - 1 && bc_zhi))) {
      diag[node] = 1.0;
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
          const int loc = (X - ex * P) + n * ((Y - ey * P) + n * (Z - ez * P));
          s = DA(s, de[e * nen + loc]);
        }
    diag[node] = s;
  }
}

}  // namespace

cudaError_t launch_jacobi_diagonal(const Setup& s, int constrained, double* diag, cudaStream_t st) {
  JacCfg c{};
  c.p = s.p;
  c.n = s.p + 1;
  c.q = s.q;
  c.comp = s.comp;
  c.nx = s.dims[0];
  c.ny = s.dims[1];
  c.nz = s.dims[2];
  c.aos = s.g_aos;
  c.diff = s.kind != KIND_MASS;
  c.gstride = s.gstride;
  const int nen = c.n * c.n * c.n;
  const size_t smem = sizeof(double) * (2 * c.q * c.n + static_cast<size_t>(c.q) * c.q * c.q * c.comp);
  double *de = nullptr, *dB = nullptr, *dD = nullptr;
  cudaError_t e = cudaMalloc(&de, sizeof(double) * static_cast<size_t>(s.E) * nen);
  if (!e) e = cudaMalloc(&dB, sizeof(double) * c.q * c.n);
  if (!e) e = cudaMalloc(&dD, sizeof(double) * c.q * c.n);
  if (!e) e = cudaMemcpyAsync(dB, s.B, sizeof(double) * c.q * c.n, cudaMemcpyHostToDevice, st);
  if (!e) e = cudaMemcpyAsync(dD, s.D, sizeof(double) * c.q * c.n, cudaMemcpyHostToDevice, st);
  if (!e) e = cudaFuncSetAttribute(&jacobi_elem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem));
  if (!e) {
    const int threads = nen < 1024 ? (nen + 31) / 32 * 32 : 1024;  // p >= 10: nodes strided over the CTA
    jacobi_elem_kernel<<<static_cast<unsigned>(s.E), threads, smem, st>>>(c, s.G, dB, dD, de);
    e = cudaGetLastError();
  }
  if (!e) {
    jacobi_gather_kernel<<<148 * 8, 256, 0, st>>>(c, de, diag, constrained, s.bc_zlo, s.bc_zhi);
    e = cudaGetLastError();
  }
  if (!e) e = cudaStreamSynchronize(st);
  cudaFree(de);
  cudaFree(dB);
  cudaFree(dD);
  return e;
}

}  // namespace hxb
