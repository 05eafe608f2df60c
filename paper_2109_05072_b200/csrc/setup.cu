// Device-side setup of the geometric factors.
//
// build_box_mesh (mesh.hpp:86-123) + compute_jacobians (geometry.hpp:78-131)
// + mass_factors / diffusion_factors (geometry.hpp:144-193), one CTA per
// element. Every contraction reproduces contract_dim's loop order
// (tensor.hpp:50-114) with explicit non-fused double operations
// (__dmul_rn/__dadd_rn never contract to FMA), so the factors are bitwise
// identical to the reference's host make_setup. This removes the host RAM /
// time wall of the 100M-400M DOF configurations (E*q^3*16 doubles of host
// Jacobians, geometry.hpp:87-88).
//
// Device factor layout (what the operator kernel streams):
//   element slot  s = (ex + nx*ey) * nz + ez      (column-major: a column's
//                                                  elements are contiguous)
//   within slot   ((m*q + a) * q + b) * q + c'... stored as (m*q + a)*q*q + (b + q*c)
//   i.e. component m, then the x-index a of the point, then the (y,z) pair,
//   so the x-pencil thread (b,c) of the kernel reads coalesced rows.
//   Slot stride gstride = comp*q^3 rounded up to an even count (16 B).
// The DMMA kernels use their own element-block orders (Setup::g_aos):
//   1 = [qp][comp] (BP3 p=7, apply_mma.cu), 2 = [c][comp][b][a] (BP5 p=7,
//   apply_mma5.cu: one z-plane of all components is a contiguous block).
#include <cuda_runtime.h>

#include "internal.h"
#include "tensor_dev.cuh"

namespace hxb {
namespace {

#define DM(a, b) __dmul_rn((a), (b))
#define DA(a, b) __dadd_rn((a), (b))
#define DS(a, b) __dsub_rn((a), (b))

struct GeomCfg {
  int p, n, q, comp, nx, ny, nz, z0;  // z0: global element layer offset of the slab
  long long gstride;
  int aos;
};

// Offset of component m of quadrature point (a, b, c) inside an element block.
__device__ __forceinline__ long long gidx(const GeomCfg& cfg, int m, int a, int b, int c) {
  const int q = cfg.q;
  if (cfg.aos == 2) return ((static_cast<long long>(c) * cfg.comp + m) * q + b) * q + a;  // [c][comp][b][a]
  if (cfg.aos) return static_cast<long long>(a + q * (b + q * c)) * cfg.comp + m;           // [qp][comp]
  return static_cast<long long>(m) * q * q * q + static_cast<long long>(a) * q * q + (b + q * c);
}

using tdev::elem_grad_dev;

__global__ void box_geometry_kernel(GeomCfg cfg, const double* __restrict__ Bg, const double* __restrict__ Dg,
                                    const double* __restrict__ qw, BoxGeometryArgs g, double* __restrict__ G,
                                    unsigned long long* bad_key, double* bad_det) {
  extern __shared__ double sm[];
  const int n = cfg.n, q = cfg.q, n3 = n * n * n, q3 = q * q * q;
  const int big = n > q ? n : q;
  double* Bs = sm;                 // q*n
  double* Ds = Bs + q * n;         // q*n
  double* nodal = Ds + q * n;      // n3
  double* ta = nodal + n3;         // big^3
  double* tb = ta + big * big * big;
  double* gf = tb + big * big * big;  // 3 * q3
  double* J = gf + 3 * q3;            // 9 * q3
  for (int i = threadIdx.x; i < q * n; i += blockDim.x) {
    Bs[i] = Bg[i];
    Ds[i] = Dg[i];
  }
  const long long slot = blockIdx.x;  // column-major element slot
  const int ez = static_cast<int>(slot % cfg.nz);
  const int col = static_cast<int>(slot / cfg.nz);
  const int ex = col % cfg.nx, ey = col / cfg.nx;
  const int gez = ez + cfg.z0;  // global element layer
  const int p = cfg.p;
  const bool colloc = cfg.comp == 6 && q == n;
  __syncthreads();

  for (int c = 0; c < 3; ++c) {
    // gather_coords (geometry.hpp:73-77) of the analytic box node positions
    // (mesh.hpp:107-119): x + L * a*sin(2pi x/Lx)*sin(2pi y/Ly)*sin(2pi z/Lz)
    for (int l = threadIdx.x; l < n3; l += blockDim.x) {
      const int i = l % n, j = (l / n) % n, k = l / (n * n);
      const int X = ex * p + i, Y = ey * p + j, Z = gez * p + k;
      const double base = c == 0 ? g.ax[X] : (c == 1 ? g.ay[Y] : g.az[Z]);
      double disp = 0.0;
      if (g.amplitude > 0.0) disp = DM(DM(DM(g.amplitude, g.sx[X]), g.sy[Y]), g.sz[Z]);
      nodal[l] = DA(base, DM(g.ext[c], disp));
    }
    __syncthreads();
    elem_grad_dev(Bs, Ds, n, q, q == n && colloc, nodal, gf, gf + q3, gf + 2 * q3, ta, tb);
    for (int qp = threadIdx.x; qp < q3; qp += blockDim.x)
      for (int d = 0; d < 3; ++d) J[qp * 9 + c * 3 + d] = gf[d * q3 + qp];
    __syncthreads();
  }

  double* Ge = G + slot * cfg.gstride;
  for (int qp = threadIdx.x; qp < q3; qp += blockDim.x) {
    const double* j = J + qp * 9;
    // geometry.hpp:113-115
    const double det = DA(DS(DM(j[0], DS(DM(j[4], j[8]), DM(j[5], j[7]))), DM(j[1], DS(DM(j[3], j[8]), DM(j[5], j[6])))),
                          DM(j[2], DS(DM(j[3], j[7]), DM(j[4], j[6]))));
    if (!(det > 0.0)) {
      const long long e_ref = ex + static_cast<long long>(cfg.nx) * (ey + static_cast<long long>(cfg.ny) * ez);
      const unsigned long long key = (static_cast<unsigned long long>(e_ref) << 20) | static_cast<unsigned>(qp);
      const unsigned long long old = atomicMin(bad_key, key);
      if (key < old) *bad_det = det;  // best effort message detail
    }
    const int a = qp % q, b = (qp / q) % q, cc = qp / (q * q);
    const double w = DM(DM(qw[a], qw[b]), qw[cc]);  // tensor_weight, geometry.hpp:139-143
    if (cfg.comp == 1) {
      Ge[gidx(cfg, 0, a, b, cc)] = DM(w, det);  // geometry.hpp:156-158
    } else {
      // geometry.hpp:178-191
      const double inv[9] = {
          __ddiv_rn(DS(DM(j[4], j[8]), DM(j[5], j[7])), det), __ddiv_rn(DS(DM(j[2], j[7]), DM(j[1], j[8])), det),
          __ddiv_rn(DS(DM(j[1], j[5]), DM(j[2], j[4])), det), __ddiv_rn(DS(DM(j[5], j[6]), DM(j[3], j[8])), det),
          __ddiv_rn(DS(DM(j[0], j[8]), DM(j[2], j[6])), det), __ddiv_rn(DS(DM(j[2], j[3]), DM(j[0], j[5])), det),
          __ddiv_rn(DS(DM(j[3], j[7]), DM(j[4], j[6])), det), __ddiv_rn(DS(DM(j[1], j[6]), DM(j[0], j[7])), det),
          __ddiv_rn(DS(DM(j[0], j[4]), DM(j[1], j[3])), det)};
      const double wd = DM(w, det);
      int m = 0;
      for (int r = 0; r < 3; ++r)
        for (int s = r; s < 3; ++s) {
          double dot = 0.0;
          for (int k = 0; k < 3; ++k) dot = DA(dot, DM(inv[r * 3 + k], inv[s * 3 + k]));
          Ge[gidx(cfg, m, a, b, cc)] = DM(wd, dot);
          ++m;
        }
    }
  }
}

// Reference AoS (geometry.hpp:48-56, element order mesh.hpp:71-82) <-> device layout.
__global__ void factors_relayout_kernel(GeomCfg cfg, const double* __restrict__ src, double* __restrict__ dst,
                                        int to_device) {
  const int q = cfg.q, q3 = q * q * q, comp = cfg.comp;
  const long long slot = blockIdx.x;
  const int ez = static_cast<int>(slot % cfg.nz);
  const int col = static_cast<int>(slot / cfg.nz);
  const int ex = col % cfg.nx, ey = col / cfg.nx;
  const long long e_ref = ex + static_cast<long long>(cfg.nx) * (ey + static_cast<long long>(cfg.ny) * ez);
  for (int l = threadIdx.x; l < q3 * comp; l += blockDim.x) {
    const int qp = l / comp, m = l % comp;
    const int a = qp % q, b = (qp / q) % q, c = qp / (q * q);
    const long long aos = (e_ref * q3 + qp) * comp + m;
    const long long dev = slot * cfg.gstride + gidx(cfg, m, a, b, c);
    if (to_device)
      dst[dev] = src[aos];
    else
      dst[aos] = src[dev];
  }
}

GeomCfg cfg_of(const Setup& s) {
  GeomCfg c{};
  c.p = s.p;
  c.n = s.p + 1;
  c.q = s.q;
  c.comp = s.comp;
  c.nx = s.dims[0];
  c.ny = s.dims[1];
  c.nz = s.dims[2];
  c.z0 = s.z0;
  c.gstride = s.gstride;
  c.aos = s.g_aos;
  return c;
}

}  // namespace

cudaError_t launch_box_geometry(const Setup& s, const BoxGeometryArgs& g, unsigned long long* bad_key,
                                double* bad_det, cudaStream_t st) {
  const GeomCfg c = cfg_of(s);
  const int n = c.n, q = c.q, big = n > q ? n : q;
  const size_t smem = sizeof(double) * (2 * q * n + n * n * n + 2 * big * big * big + 12 * q * q * q);
  double *dB = nullptr, *dD = nullptr, *dw = nullptr;
  cudaError_t err = cudaMallocAsync(&dB, sizeof(double) * q * n, st);
  if (err) return err;
  cudaMallocAsync(&dD, sizeof(double) * q * n, st);
  cudaMallocAsync(&dw, sizeof(double) * q, st);
  cudaMemcpyAsync(dB, s.B, sizeof(double) * q * n, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dD, s.D, sizeof(double) * q * n, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dw, s.qw, sizeof(double) * q, cudaMemcpyHostToDevice, st);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(box_geometry_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const long long nslots = static_cast<long long>(s.dims[0]) * s.dims[1] * s.dims[2];
  box_geometry_kernel<<<static_cast<unsigned>(nslots), 128, smem, st>>>(c, dB, dD, dw, g, s.G, bad_key, bad_det);
  err = cudaGetLastError();
  cudaFreeAsync(dB, st);
  cudaFreeAsync(dD, st);
  cudaFreeAsync(dw, st);
  return err;
}

cudaError_t launch_factors_from_aos(const Setup& s, const double* aos, cudaStream_t st) {
  const long long nslots = static_cast<long long>(s.dims[0]) * s.dims[1] * s.dims[2];
  factors_relayout_kernel<<<static_cast<unsigned>(nslots), 256, 0, st>>>(cfg_of(s), aos, s.G, 1);
  return cudaGetLastError();
}

cudaError_t launch_factors_to_aos(const Setup& s, double* aos, cudaStream_t st) {
  const long long nslots = static_cast<long long>(s.dims[0]) * s.dims[1] * s.dims[2];
  factors_relayout_kernel<<<static_cast<unsigned>(nslots), 256, 0, st>>>(cfg_of(s), s.G, aos, 0);
  return cudaGetLastError();
}

}  // namespace hxb
