// C ABI of the B200 hot path (include/hexbp_b200.h): setup / workspace
// lifetime, operator apply, device-resident CG, deterministic dot.
#include <cuda_runtime.h>

#include <chrono>
#include <cstddef>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "capi_util.h"
#include "internal.h"
#include "ring.cuh"

namespace hxb {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

}  // namespace hxb

using namespace hxb;

namespace {

int kind_of(int bp) { return bp == 1 ? KIND_MASS : (bp == 3 ? KIND_DIFF : KIND_COLLOC); }

int default_q(int bp, int p) { return bp == 5 ? p + 1 : p + 2; }  // operator.hpp:55

int init_setup(Setup& s, int bp, int p, const int gdims[3], int z0, int z1, int device) {
  if (!(bp == 1 || bp == 3 || bp == 5)) return invalid("setup: bp must be 1, 3 or 5");
  if (p < 1 || p > kMaxPG) return invalid("setup: degree must be in [1, 10] for the device kernels");
  for (int d = 0; d < 3; ++d)
    if (gdims[d] < 1) return invalid("build_box_mesh: element counts must be >= 1");
  if (z0 < 0 || z1 <= z0 || z1 > gdims[2]) return invalid("setup: bad slab range");
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  if (ndev == 0) {
    set_error("no CUDA device available: the hexbp-b200 operator has no CPU fallback");
    return HEXBP_CUDA_ERROR;
  }
  if (device < 0 || device >= ndev) return invalid("setup: bad device ordinal");
  s.bp = bp;
  s.p = p;
  s.q = default_q(bp, p);
  s.kind = kind_of(bp);
  s.comp = bp == 1 ? 1 : 6;
  for (int d = 0; d < 3; ++d) s.gdims[d] = gdims[d];
  s.dims[0] = gdims[0];
  s.dims[1] = gdims[1];
  s.dims[2] = z1 - z0;
  s.z0 = z0;
  s.bc_zlo = z0 == 0;
  s.bc_zhi = z1 == gdims[2];
  s.device = device;
  s.nL = static_cast<int64_t>(s.dims[0] * p + 1) * (s.dims[1] * p + 1) * (s.dims[2] * p + 1);
  s.E = static_cast<int64_t>(s.dims[0]) * s.dims[1] * s.dims[2];
  const long long per = static_cast<long long>(s.comp) * s.q * s.q * s.q;
  s.gstride = (per + 1) / 2 * 2;
  // DMMA kernels' factor block orders: [qp][6] (BP3 p=7, apply_mma.cu), [c][6][b][a] (BP5 p=7, apply_mma5.cu)
  // (HEXBP_NO_DMMA=1: the DFMA kernels' layout for A/B comparisons)
  const char* no_dmma = std::getenv("HEXBP_NO_DMMA");
  const bool dmma = !(no_dmma && *no_dmma && *no_dmma != '0');
  s.g_aos = !dmma ? 0 : (s.kind == KIND_DIFF && p == 7) ? 1 : ((s.kind == KIND_COLLOC && p == 7) ? 2 : 0);
  std::vector<double> qp(s.q), npn(p + 1), nw(p + 1);
  try {
    build_basis(p, s.q, bp == 5, s.B, s.D, qp.data(), s.qw, npn.data(), nw.data());
  } catch (const std::exception& e) {
    return invalid(e.what());
  }
  return HEXBP_OK;
}

int create_box(int bp, int p, const int gdims[3], int z0, int z1, const double extent[3], double amplitude,
               int device, hexbp_setup_t* out) {
  if (!out) return invalid("setup: null output handle");
  *out = nullptr;
  const double ext[3] = {extent ? extent[0] : 1.0, extent ? extent[1] : 1.0, extent ? extent[2] : 1.0};
  for (int d = 0; d < 3; ++d)
    if (!(ext[d] > 0.0)) return invalid("build_box_mesh: extents must be positive");
  if (!(amplitude >= 0.0 && amplitude <= 0.15))  // mesh.hpp:84,104-105
    return invalid("build_box_mesh: deform amplitude outside [0, 0.15]");
  auto* h = new (std::nothrow) hexbp_setup_s;
  if (!h) return HEXBP_OUT_OF_MEMORY;
  Setup& s = h->s;
  int rc = init_setup(s, bp, p, gdims, z0, z1, device);
  if (rc) {
    delete h;
    return rc;
  }
  DeviceGuard g(device);
  // Global axis coordinates and the separable deformation factors, on the
  // host with libm exactly as mesh.hpp:59-67,107-116 evaluates them.
  constexpr double kPi = 3.141592653589793;
  std::vector<double> axis[3], sn[3];
  for (int d = 0; d < 3; ++d) {
    axis[d] = axis_node_coords(gdims[d], p, ext[d]);
    sn[d].resize(axis[d].size());
    for (std::size_t i = 0; i < axis[d].size(); ++i) sn[d][i] = std::sin(2.0 * kPi * axis[d][i] / ext[d]);
  }
  double* dbuf = nullptr;
  std::size_t tot = 0;
  for (int d = 0; d < 3; ++d) tot += 2 * axis[d].size();
  const std::size_t gbytes = sizeof(double) * static_cast<std::size_t>(s.gstride) * s.E;
  cudaError_t e = cudaMalloc(&s.G, gbytes);
  if (e) {
    delete h;
    return cuda_status(e, "cudaMalloc(factors)");
  }
  unsigned long long* bad = nullptr;
  double* bad_det = nullptr;
  e = cudaMalloc(&dbuf, sizeof(double) * tot + 16 + sizeof(double));
  if (e) {
    cudaFree(s.G);
    delete h;
    return cuda_status(e, "cudaMalloc(axis)");
  }
  std::vector<double> host(tot);
  BoxGeometryArgs ga{};
  std::size_t off = 0;
  const double** ap[3] = {&ga.ax, &ga.ay, &ga.az};
  const double** sp[3] = {&ga.sx, &ga.sy, &ga.sz};
  for (int d = 0; d < 3; ++d) {
    std::memcpy(host.data() + off, axis[d].data(), sizeof(double) * axis[d].size());
    *ap[d] = dbuf + off;
    off += axis[d].size();
    std::memcpy(host.data() + off, sn[d].data(), sizeof(double) * sn[d].size());
    *sp[d] = dbuf + off;
    off += sn[d].size();
  }
  ga.amplitude = amplitude;
  for (int d = 0; d < 3; ++d) ga.ext[d] = ext[d];
  s.box = 1;
  s.amplitude = amplitude;
  for (int d = 0; d < 3; ++d) s.ext[d] = ext[d];
  bad = reinterpret_cast<unsigned long long*>(dbuf + tot);
  bad_det = dbuf + tot + 2;
  cudaMemcpy(dbuf, host.data(), sizeof(double) * tot, cudaMemcpyHostToDevice);
  cudaMemset(bad, 0xff, sizeof(unsigned long long));
  e = launch_box_geometry(s, ga, bad, bad_det, nullptr);
  if (!e) e = cudaDeviceSynchronize();
  unsigned long long hbad = ~0ull;
  double hdet = 0.0;
  if (!e) {
    cudaMemcpy(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hdet, bad_det, sizeof hdet, cudaMemcpyDeviceToHost);
  }
  cudaFree(dbuf);
  if (e) {
    cudaFree(s.G);
    delete h;
    return cuda_status(e, "box geometry");
  }
  if (hbad != ~0ull) {
    const long long elem = static_cast<long long>(hbad >> 20);
    const int qpt = static_cast<int>(hbad & 0xfffff);
    set_error("non-positive Jacobian determinant " + std::to_string(hdet) + " at element " + std::to_string(elem) +
              ", quadrature point " + std::to_string(qpt));
    cudaFree(s.G);
    delete h;
    return HEXBP_DEGENERATE;
  }
  *out = h;
  return HEXBP_OK;
}

int ensure_history(Workspace& w, int max_iter) {
  if (max_iter + 1 <= w.history_cap) return HEXBP_OK;
  CK(cudaFree(w.history));
  w.history = nullptr;
  w.history_cap = 0;
  CK(cudaMalloc(&w.history, sizeof(double) * (max_iter + 1)));
  w.history_cap = max_iter + 1;
  return HEXBP_OK;
}

int ensure_diag_staging(Workspace& w) {
  if (w.tmp_d) return HEXBP_OK;
  CK(cudaMalloc(&w.tmp_d, sizeof(double) * w.s->nL));
  return HEXBP_OK;
}

int ensure_host_staging(Workspace& w) {
  if (w.tmp_u) return HEXBP_OK;
  CK(cudaMalloc(&w.tmp_u, sizeof(double) * w.s->nL));
  CK(cudaMalloc(&w.tmp_w, sizeof(double) * w.s->nL));
  CK(cudaStreamCreateWithFlags(&w.copy_st, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&w.ev_x, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&w.ev_b, cudaEventDisableTiming));
  return HEXBP_OK;
}

// Host-API staging of a solve's inputs: x0 first on the compute stream, then
// b on the copy stream (after x0: the two would otherwise share PCIe and delay
// the initial apply), so b's transfer overlaps the initial A x0. Returns the
// event the residual kernel waits on.
cudaError_t stage_solve_inputs(Workspace& w, const double* b, const double* x, int64_t n, cudaStream_t st) {
  const size_t bytes = sizeof(double) * static_cast<size_t>(n);
  cudaError_t e = cudaMemcpyAsync(w.tmp_w, x, bytes, cudaMemcpyHostToDevice, st);
  if (!e) e = cudaEventRecord(w.ev_x, st);
  if (!e) e = cudaStreamWaitEvent(w.copy_st, w.ev_x, 0);
  if (!e) e = cudaMemcpyAsync(w.tmp_u, b, bytes, cudaMemcpyHostToDevice, w.copy_st);
  if (!e) e = cudaEventRecord(w.ev_b, w.copy_st);
  return e;
}

int pcg_run(hexbp_setup_t h, hexbp_workspace_t wh, const double* b, double* x, const double* diag, double rel_tol,
            int max_iter, int constrained, hexbp_cg_report* report, double* history, cudaStream_t st,
            cudaEvent_t b_ready);

}  // namespace

extern "C" {

const char* hexbp_last_error(void) { return g_last_error.c_str(); }

int hexbp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int hexbp_setup_create_box(int bp, int p, const int dims[3], const double extent[3], double amplitude, int device,
                           hexbp_setup_t* out) {
  if (!dims) return invalid("setup: null dims");
  return create_box(bp, p, dims, 0, dims[2], extent, amplitude, device, out);
}

int hexbp_setup_create_box_slab(int bp, int p, const int gdims[3], int z0, int z1, const double extent[3],
                                double amplitude, int device, hexbp_setup_t* out) {
  if (!gdims) return invalid("setup: null dims");
  return create_box(bp, p, gdims, z0, z1, extent, amplitude, device, out);
}

int hexbp_setup_create(int bp, int p, int q, const int dims[3], const double* B, const double* D,
                       const double* factors_aos, int device, hexbp_setup_t* out) {
  if (!out || !dims || !B || !D || !factors_aos) return invalid("setup: null argument");
  *out = nullptr;
  auto* h = new (std::nothrow) hexbp_setup_s;
  if (!h) return HEXBP_OUT_OF_MEMORY;
  Setup& s = h->s;
  int rc = init_setup(s, bp, p, dims, 0, dims[2], device);
  if (rc) {
    delete h;
    return rc;
  }
  if (q != s.q) {
    delete h;
    return invalid("setup: the device kernels implement the reference quadrature convention q = p+2 (BP1/BP3), "
                   "p+1 (BP5) (operator.hpp:55)");
  }
  const int n = p + 1;
  std::memcpy(s.B, B, sizeof(double) * q * n);
  std::memcpy(s.D, D, sizeof(double) * q * n);
  DeviceGuard g(device);
  const std::size_t aos_n = static_cast<std::size_t>(s.E) * q * q * q * s.comp;
  double* tmp = nullptr;
  cudaError_t e = cudaMalloc(&s.G, sizeof(double) * static_cast<std::size_t>(s.gstride) * s.E);
  if (!e) e = cudaMalloc(&tmp, sizeof(double) * aos_n);
  if (!e) e = cudaMemcpy(tmp, factors_aos, sizeof(double) * aos_n, cudaMemcpyHostToDevice);
  if (!e) e = launch_factors_from_aos(s, tmp, nullptr);
  if (!e) e = cudaDeviceSynchronize();
  if (tmp) cudaFree(tmp);
  if (e) {
    if (s.G) cudaFree(s.G);
    delete h;
    return cuda_status(e, "setup upload");
  }
  *out = h;
  return HEXBP_OK;
}

int hexbp_setup_check_restriction(hexbp_setup_t h, const int32_t* elem_to_global, int64_t n) {
  if (!h || (!elem_to_global && n)) return invalid("check_restriction: null argument");
  const Setup& s = h->s;
  const int p = s.p, nn = p + 1;
  const int64_t nen = static_cast<int64_t>(nn) * nn * nn;
  if (n != s.E * nen)
    return invalid("check_restriction: table length " + std::to_string(n) + " != elements x (p+1)^3 = " +
                   std::to_string(s.E * nen));
  const int64_t gx = static_cast<int64_t>(s.gdims[0]) * p + 1, gy = static_cast<int64_t>(s.gdims[1]) * p + 1;
  int64_t pos = 0;
  for (int ez = s.z0; ez < s.z0 + s.dims[2]; ++ez)  // mesh.hpp:74-82 element and node order
    for (int ey = 0; ey < s.dims[1]; ++ey)
      for (int ex = 0; ex < s.dims[0]; ++ex)
        for (int k = 0; k <= p; ++k)
          for (int j = 0; j <= p; ++j)
            for (int i = 0; i <= p; ++i, ++pos) {
              const int64_t g = (static_cast<int64_t>(ex) * p + i) + gx * ((static_cast<int64_t>(ey) * p + j) +
                                                                           gy * (static_cast<int64_t>(ez) * p + k));
              if (elem_to_global[pos] != g)
                return invalid("check_restriction: elem_to_global[" + std::to_string(pos) + "] = " +
                               std::to_string(elem_to_global[pos]) + ", the structured box numbering has " +
                               std::to_string(g) + " (the device kernels support box meshes only)");
            }
  return HEXBP_OK;
}

void hexbp_setup_destroy(hexbp_setup_t h) {
  if (!h) return;
  DeviceGuard g(h->s.device);
  if (h->s.G) cudaFree(h->s.G);
  delete h;
}

int hexbp_setup_get_info(hexbp_setup_t h, hexbp_setup_info* out) {
  if (!h || !out) return invalid("null argument");
  const Setup& s = h->s;
  out->bp = s.bp;
  out->p = s.p;
  out->q = s.q;
  for (int d = 0; d < 3; ++d) {
    out->dims[d] = s.dims[d];
    out->gdims[d] = s.gdims[d];
  }
  out->z0 = s.z0;
  out->components = s.comp;
  out->l_size = s.nL;
  out->elements = s.E;
  out->factor_bytes = static_cast<int64_t>(s.E) * s.q * s.q * s.q * s.comp * 8;
  return HEXBP_OK;
}

int hexbp_setup_basis(hexbp_setup_t h, double* B, double* D) {
  if (!h || !B || !D) return invalid("null argument");
  const int nq = h->s.q * (h->s.p + 1);
  std::memcpy(B, h->s.B, sizeof(double) * nq);
  std::memcpy(D, h->s.D, sizeof(double) * nq);
  return HEXBP_OK;
}

int hexbp_setup_factors(hexbp_setup_t h, double* aos) {
  if (!h || !aos) return invalid("null argument");
  const Setup& s = h->s;
  DeviceGuard g(s.device);
  const std::size_t n = static_cast<std::size_t>(s.E) * s.q * s.q * s.q * s.comp;
  double* tmp = nullptr;
  CK(cudaMalloc(&tmp, sizeof(double) * n));
  cudaError_t e = launch_factors_to_aos(s, tmp, nullptr);
  if (!e) e = cudaMemcpy(aos, tmp, sizeof(double) * n, cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  return cuda_status(e, "factors download");
}

int hexbp_setup_factors_device(hexbp_setup_t h, double* out, void* stream) {
  if (!h || !out) return invalid("null argument");
  DeviceGuard g(h->s.device);
  CK(launch_factors_to_aos(h->s, out, static_cast<cudaStream_t>(stream)));
  return HEXBP_OK;
}

int hexbp_setup_node_coords(hexbp_setup_t h, double* out, void* stream) {
  if (!h || !out) return invalid("null argument");
  const Setup& s = h->s;
  if (!s.box) return invalid("node_coords: setup was not created from a box mesh");
  DeviceGuard g(s.device);
  constexpr double kPi = 3.141592653589793;
  std::vector<double> host;
  std::size_t off[6];
  for (int d = 0; d < 3; ++d) {  // mesh.hpp:59-67,107-116 on the host, as at setup
    const std::vector<double> ax = axis_node_coords(s.gdims[d], s.p, s.ext[d]);
    off[2 * d] = host.size();
    host.insert(host.end(), ax.begin(), ax.end());
    off[2 * d + 1] = host.size();
    for (double x : ax) host.push_back(std::sin(2.0 * kPi * x / s.ext[d]));
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* dbuf = nullptr;
  CK(cudaMallocAsync(&dbuf, sizeof(double) * host.size(), st));
  cudaError_t e = cudaMemcpyAsync(dbuf, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, st);
  BoxGeometryArgs ga{};
  ga.ax = dbuf + off[0];
  ga.sx = dbuf + off[1];
  ga.ay = dbuf + off[2];
  ga.sy = dbuf + off[3];
  ga.az = dbuf + off[4];
  ga.sz = dbuf + off[5];
  ga.amplitude = s.amplitude;
  for (int d = 0; d < 3; ++d) ga.ext[d] = s.ext[d];
  if (!e) e = launch_node_coords(s, ga, out, st);
  if (!e) e = cudaStreamSynchronize(st);  // the host staging vector goes out of scope
  cudaFreeAsync(dbuf, st);
  return cuda_status(e, "node_coords");
}

int hexbp_interp_to_qpts(hexbp_setup_t h, const double* v, double* out, void* stream) {
  if (!h || !v || !out) return invalid("null argument");
  DeviceGuard g(h->s.device);
  CK(launch_interp_to_qpts(h->s, v, out, static_cast<cudaStream_t>(stream)));
  return HEXBP_OK;
}

int hexbp_interp_transpose(hexbp_setup_t h, const double* vq, double* out, void* stream) {
  if (!h || !vq || !out) return invalid("null argument");
  DeviceGuard g(h->s.device);
  CK(launch_interp_transpose(h->s, vq, out, static_cast<cudaStream_t>(stream)));
  return HEXBP_OK;
}

int hexbp_workspace_create(hexbp_setup_t h, hexbp_workspace_t* out) {
  if (!h || !out) return invalid("null argument");
  *out = nullptr;
  auto* wh = new (std::nothrow) hexbp_workspace_s;
  if (!wh) return HEXBP_OUT_OF_MEMORY;
  Workspace& w = wh->w;
  const Setup& s = h->s;
  w.s = &s;
  w.device = s.device;
  DeviceGuard g(s.device);
  const int ncols = s.dims[0] * s.dims[1];
  const std::size_t n = static_cast<std::size_t>(s.nL);
  w.vec_blocks = vec_grid(s.nL);
  w.history_cap = 4097;
  cudaError_t e = cudaSuccess;
  auto al = [&](void** p, std::size_t bytes) {
    if (!e) e = cudaMalloc(p, bytes);
    if (!e) e = cudaMemset(*p, 0, bytes);
  };
  w.fixup_grid = fixup_grid(s);
  {
    const std::size_t nz_nodes = static_cast<std::size_t>(s.dims[2]) * s.p + 1;
    const std::size_t exact = static_cast<std::size_t>(ncols) * 4 * s.p * nz_nodes;
    const std::size_t fast = static_cast<std::size_t>(lat_fast_doubles(s.p, s.dims[0], s.dims[1], nz_nodes));
    al(reinterpret_cast<void**>(&w.lateral), sizeof(double) * (exact > fast ? exact : fast));
    w.scatter_bytes += sizeof(double) * (exact > fast ? exact : fast);
  }
  al(reinterpret_cast<void**>(&w.zupper), sizeof(double) * static_cast<std::size_t>(ncols) * 4 * s.p * s.dims[2]);
  w.scatter_bytes += sizeof(double) * static_cast<std::size_t>(ncols) * 4 * s.p * s.dims[2];
  // one partial p.Ap per operator CTA: at most one per (column, z-segment) <= E
  al(reinterpret_cast<void**>(&w.col_dot), sizeof(double) * static_cast<std::size_t>(ncols) * s.dims[2]);
  al(reinterpret_cast<void**>(&w.fix_partials), sizeof(double) * w.fixup_grid);
  al(reinterpret_cast<void**>(&w.fix_done), sizeof(unsigned int) * 4);
  al(reinterpret_cast<void**>(&w.sc), sizeof(DevScalars));
  al(reinterpret_cast<void**>(&w.r), sizeof(double) * n);
  al(reinterpret_cast<void**>(&w.p), sizeof(double) * n);
  al(reinterpret_cast<void**>(&w.Ap), sizeof(double) * n);
  al(reinterpret_cast<void**>(&w.vec_partials), sizeof(double) * reduction_partials(s.nL));
  al(reinterpret_cast<void**>(&w.dot_result), sizeof(double) * 2);
  al(reinterpret_cast<void**>(&w.vec_done), sizeof(unsigned int) * 4);
  al(reinterpret_cast<void**>(&w.history), sizeof(double) * w.history_cap);
  if (!e && tma_u_supported(s)) {  // row-pitched vectors of the fast CG (tma.cu)
    w.pt_pitch = tma_u_pitch(s);
    const std::size_t np = sizeof(double) * static_cast<std::size_t>(w.pt_pitch) *
                           (static_cast<std::size_t>(s.dims[1]) * s.p + 1) * (static_cast<std::size_t>(s.dims[2]) * s.p + 1);
    al(reinterpret_cast<void**>(&w.pt), np);
    al(reinterpret_cast<void**>(&w.xt), np);
    al(reinterpret_cast<void**>(&w.rt), np);
    al(reinterpret_cast<void**>(&w.Apt), np);
    // no tensor map (driver without cuTensorMapEncodeTiled): the fast CG keeps
    // the unpadded p and the cp.async-staged kernels
    if (!e && encode_u_tensor_map(s, w.pt, w.pt_pitch, &w.pt_map) != cudaSuccess) {
      for (double** b : {&w.pt, &w.xt, &w.rt, &w.Apt}) {
        cudaFree(*b);
        *b = nullptr;
      }
      w.pt_pitch = 0;
    }
  }
  if (!e) e = cudaMallocHost(reinterpret_cast<void**>(&w.host_sc), sizeof(DevScalars));
  if (e) {
    hexbp_workspace_destroy(wh);
    return cuda_status(e, "workspace allocation");
  }
  if (s.p > kMaxP) {  // generic degree: the fused kernels stop at p = 8; the multipass pipeline serves it
    const int rc = hexbp_workspace_set_backend(wh, HEXBP_BACKEND_MULTIPASS);
    if (rc) {
      hexbp_workspace_destroy(wh);
      return rc;
    }
  }
  *out = wh;
  return HEXBP_OK;
}

int hexbp_workspace_reserve(hexbp_workspace_t wh, int max_iter, int host_staging) {
  if (!wh || max_iter < 0) return invalid("workspace_reserve: bad argument");
  Workspace& w = wh->w;
  DeviceGuard g(w.device);
  int rc = ensure_history(w, max_iter);
  if (!rc && (host_staging & 1)) rc = ensure_host_staging(w);
  if (!rc && (host_staging & 2)) rc = ensure_diag_staging(w);
  return rc;
}

void hexbp_workspace_destroy(hexbp_workspace_t wh) {
  if (!wh) return;
  Workspace& w = wh->w;
  DeviceGuard g(w.device);
  void* bufs[] = {w.mp_buf, w.lateral, w.zupper, w.fix_partials, w.fix_done,  w.col_dot, w.sc, w.r, w.p, w.Ap, w.tmp_u, w.tmp_w, w.tmp_d, w.vec_partials,
                  w.vec_done, w.history, w.dot_result, w.pt, w.xt, w.rt, w.Apt};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (w.host_sc) cudaFreeHost(w.host_sc);
  if (w.copy_st) cudaStreamDestroy(w.copy_st);
  for (auto& cg : w.cg_graphs)
    if (cg.exec) cudaGraphExecDestroy(cg.exec);
  if (w.graph_st) cudaStreamDestroy(w.graph_st);
  if (w.ev_g0) cudaEventDestroy(w.ev_g0);
  if (w.ev_g1) cudaEventDestroy(w.ev_g1);
  if (w.ev_x) cudaEventDestroy(w.ev_x);
  if (w.ev_b) cudaEventDestroy(w.ev_b);
  delete wh;
}

int hexbp_apply(hexbp_setup_t h, hexbp_workspace_t wh, const double* u, double* w, int constrained, void* stream) {
  if (!h || !wh || !u || !w) return invalid("apply: null argument");
  if (wh->w.s != &h->s) return invalid("apply: workspace belongs to another setup");
  if (u == w) return invalid("apply: u and w must not alias");
  DeviceGuard g(h->s.device);
  CK(launch_apply(h->s, wh->w, u, w, constrained, nullptr, nullptr, static_cast<cudaStream_t>(stream)));
  return HEXBP_OK;
}

int hexbp_apply_cg_form(hexbp_setup_t h, hexbp_workspace_t wh, const double* u, double* w, int constrained,
                        void* stream) {
  if (!h || !wh || !w) return invalid("apply_cg_form: null argument");
  if (wh->w.s != &h->s) return invalid("apply: workspace belongs to another setup");
  Workspace& ws = wh->w;
  if (ws.exact && !ws.fast_op) return invalid("apply_cg_form: fast-mode workspaces only");
  const Setup& s = h->s;
  DeviceGuard g(s.device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* pv = ws.pt && !ws.exact ? ws.pt : ws.p;
  if (u == w || pv == w) return invalid("apply_cg_form: u / the search direction and w must not alias");
  if (u) {
    const size_t Nx = static_cast<size_t>(s.dims[0]) * s.p + 1;
    const size_t rows = static_cast<size_t>(s.nL) / Nx;
    const size_t pitch = pv == ws.pt ? static_cast<size_t>(ws.pt_pitch) : Nx;
    CK(launch_copy_rows(pv, static_cast<int>(pitch), u, static_cast<int>(Nx), static_cast<int>(Nx), rows, st));
  }
  // constrained bit 1: also the fused p.Ap of the CG form (into the
  // workspace's dot scratch), i.e. exactly the kernel variant the solve runs
  CK(launch_apply(s, ws, pv, w, constrained & 1, (constrained & 2) ? ws.dot_result : nullptr, nullptr, st, false));
  return HEXBP_OK;
}

int hexbp_apply_ring_deferred(hexbp_setup_t h, hexbp_workspace_t wh, const double* u, double* w, int constrained,
                              void* stream) {
  if (!h || !wh || !u || !w) return invalid("apply: null argument");
  if (wh->w.s != &h->s) return invalid("apply: workspace belongs to another setup");
  if (u == w) return invalid("apply: u and w must not alias");
  if (wh->w.exact && !wh->w.fast_op) return invalid("apply_ring_deferred: fast-mode workspaces only");
  DeviceGuard g(h->s.device);
  CK(launch_apply(h->s, wh->w, u, w, constrained, nullptr, nullptr, static_cast<cudaStream_t>(stream), false));
  return HEXBP_OK;
}

int hexbp_apply_host(hexbp_setup_t h, hexbp_workspace_t wh, const double* u, double* w, int64_t n, int constrained) {
  if (!h || !wh || !u || !w) return invalid("apply: null argument");
  if (n != h->s.nL) return invalid("apply: L-vector length mismatch");  // operator.hpp:268
  DeviceGuard g(h->s.device);
  Workspace& ws = wh->w;
  int rc = ensure_host_staging(ws);
  if (rc) return rc;
  CK(cudaMemcpy(ws.tmp_u, u, sizeof(double) * n, cudaMemcpyHostToDevice));
  CK(launch_apply(h->s, ws, ws.tmp_u, ws.tmp_w, constrained, nullptr, nullptr, nullptr));
  CK(cudaMemcpy(w, ws.tmp_w, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return HEXBP_OK;
}

int hexbp_cg(hexbp_setup_t h, hexbp_workspace_t wh, const double* b, double* x, double rel_tol, int max_iter,
             int constrained, hexbp_cg_report* report, double* history, void* stream) {
  return hexbp_pcg(h, wh, b, x, nullptr, rel_tol, max_iter, constrained, report, history, stream);
}

int hexbp_jacobi_diagonal(hexbp_setup_t h, int constrained, double* diag, void* stream) {
  if (!h || !diag) return invalid("jacobi_diagonal: null argument");
  DeviceGuard g(h->s.device);
  const cudaError_t e = launch_jacobi_diagonal(h->s, constrained, diag, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorMemoryAllocation) return cuda_status(e, "jacobi_diagonal: element vector");
  CK(e);
  return HEXBP_OK;
}

int hexbp_jacobi_diagonal_host(hexbp_setup_t h, int constrained, double* diag) {
  if (!h || !diag) return invalid("jacobi_diagonal: null argument");
  DeviceGuard g(h->s.device);
  double* d = nullptr;
  const size_t bytes = sizeof(double) * static_cast<size_t>(h->s.nL);
  if (cudaMalloc(&d, bytes) != cudaSuccess) return cuda_status(cudaErrorMemoryAllocation, "jacobi_diagonal");
  int rc = hexbp_jacobi_diagonal(h, constrained, d, nullptr);
  if (rc == HEXBP_OK) {
    const cudaError_t e = cudaMemcpy(diag, d, bytes, cudaMemcpyDeviceToHost);
    if (e) rc = cuda_status(e, "jacobi_diagonal: copy");
  }
  cudaFree(d);
  return rc;
}

int hexbp_pcg_host(hexbp_setup_t h, hexbp_workspace_t wh, const double* b, double* x, const double* diag, int64_t n,
                   double rel_tol, int max_iter, int constrained, hexbp_cg_report* report, double* history) {
  if (!h || !wh || !b || !x) return invalid("cg: null argument");
  if (n != h->s.nL) return invalid("cg: x0 length mismatch");  // solver.hpp:96
  DeviceGuard g(h->s.device);
  Workspace& w = wh->w;
  int rc = ensure_host_staging(w);
  if (rc) return rc;
  double* dd = nullptr;
  if (diag) {
    if ((rc = ensure_diag_staging(w))) return rc;
    dd = w.tmp_d;
    CK(cudaMemcpy(dd, diag, sizeof(double) * n, cudaMemcpyHostToDevice));
  }
  CK(stage_solve_inputs(w, b, x, n, nullptr));
  rc = pcg_run(h, wh, w.tmp_u, w.tmp_w, dd, rel_tol, max_iter, constrained, report, history, nullptr, w.ev_b);
  if (rc == HEXBP_OK || rc == HEXBP_DIVERGENCE) CK(cudaMemcpy(x, w.tmp_w, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return rc;
}

int hexbp_pcg(hexbp_setup_t h, hexbp_workspace_t wh, const double* b, double* x, const double* diag, double rel_tol,
              int max_iter, int constrained, hexbp_cg_report* report, double* history, void* stream) {
  return pcg_run(h, wh, b, x, diag, rel_tol, max_iter, constrained, report, history,
                 static_cast<cudaStream_t>(stream), nullptr);
}

}  // extern "C"

namespace {

constexpr int kCgGraphBlock = 8;  // iterations per captured graph

// HEXBP_CG_GRAPH=0 keeps the eager launch loop (A/B switch)
bool cg_graph_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("HEXBP_CG_GRAPH");
    return !(v && *v == '0');
  }();
  return on;
}

int pcg_run(hexbp_setup_t h, hexbp_workspace_t wh, const double* b, double* x, const double* diag, double rel_tol,
            int max_iter, int constrained, hexbp_cg_report* report, double* history, cudaStream_t st,
            cudaEvent_t b_ready) {
  if (!h || !wh || !b || !x) return invalid("cg: null argument");
  if (max_iter < 0) return invalid("cg: max_iter must be >= 0");
  const auto t0 = std::chrono::steady_clock::now();
  const Setup& s = h->s;
  Workspace& w = wh->w;
  DeviceGuard g(s.device);
  int hrc = ensure_history(w, max_iter);  // no-op within the reserved capacity
  if (hrc) return hrc;
  const int64_t n = s.nL;
  // Jacobi preconditioner for this solve (DevScalars::precond selects the
  // r.z recurrence of beta in the kernels' scalar logic)
  w.diag = diag;
  CK(launch_set_int(&w.sc->precond, diag ? 1 : 0, st));
  struct ClearDiag {  // the workspace's other solvers (multi-GPU CG) run unpreconditioned
    Workspace& w;
    cudaStream_t st;
    ~ClearDiag() {
      w.diag = nullptr;
      cudaMemsetAsync(reinterpret_cast<char*>(w.sc) + offsetof(DevScalars, precond), 0, sizeof(int), st);
    }
  } clear_diag{w, st};
  // fast CG on the DMMA degrees (unpreconditioned): the search direction
  // lives row-pitched in Workspace::pt so the operator stages it by TMA
  // tensor copies (tma.cu), and x, r, A p share that pitch (xt, rt, Apt) so
  // the vector kernels stay 32-byte aligned across operands; x is copied in
  // here and out after the loop
  struct UsePt {
    Workspace& w;
    ~UsePt() { w.use_pt = 0; }
  } use_pt{w};
  w.use_pt = !w.exact && w.pt != nullptr && diag == nullptr;
  double* const pv = w.use_pt ? w.pt : w.p;
  double* const xv = w.use_pt ? w.xt : x;
  double* const apv = w.use_pt ? w.Apt : w.Ap;
  const size_t Nx = static_cast<size_t>(s.dims[0]) * s.p + 1, rows = static_cast<size_t>(n) / Nx;
  if (w.use_pt)
    CK(launch_copy_rows(w.xt, w.pt_pitch, x, static_cast<int>(Nx), static_cast<int>(Nx), rows, st));
  // r0 = b - A x0 (solver.hpp:102-103); fast mode sums the ring in the init kernel
  if (w.exact) {
    CK(launch_apply(s, w, x, w.Ap, constrained, nullptr, nullptr, st));
    if (b_ready) CK(cudaStreamWaitEvent(st, b_ready, 0));
    CK(launch_cg_init(w, b, n, rel_tol, max_iter, st));
  } else {
    CK(launch_apply(s, w, x, apv, constrained, nullptr, nullptr, st, /*finish_ring=*/false));
    if (b_ready) CK(cudaStreamWaitEvent(st, b_ready, 0));
    CK(launch_cg_init_ring(w, b, x, n, rel_tol, max_iter, constrained, st));
  }
  if (diag && w.exact) CK(launch_cg_rz(w, n, st));  // rz = r0.z0 (solver.hpp:124)
  const int check_every = rel_tol > 0.0 ? 8 : (1 << 30);
  // one CG iteration (solver.hpp:126-148) on stream q
  auto iteration = [&](cudaStream_t q) -> cudaError_t {
    cudaError_t e = cudaSuccess;
    if (w.exact) {
      e = launch_apply(s, w, w.p, w.Ap, constrained, nullptr, nullptr, q);
      if (!e) e = launch_cg_pap(w, n, q);
    } else {
      e = launch_apply(s, w, pv, apv, constrained, nullptr, w.sc, q, /*finish_ring=*/false);
    }
    if (!e) e = launch_cg_update_r(w, n, q, constrained);
    if (!e && diag && w.exact) e = launch_cg_rz(w, n, q);  // rz_next = r.z, beta (solver.hpp:145-147)
    if (!e) e = launch_cg_update_xp(w, xv, n, q);
    return e;
  };
  int k0 = 1;  // first iteration the eager loop below runs
  static_assert(kCgGraphBlock == 8, "graph blocks end where the eager loop checks convergence");
  if (max_iter >= kCgGraphBlock && cg_graph_enabled() && !w.cg_graph_failed) {
    // replay a captured block of iterations (the kernels read alpha, beta and
    // the stopping state from device scalars, so every replay is the launch
    // sequence of the eager loop; a converged solve's remaining launches
    // return at once); with a tolerance the host checks the stopping state
    // after every block, where the eager loop checks it
    const int con = (constrained ? 1 : 0) + (w.exact ? 2 : 0) + (w.fast_op ? 4 : 0) + (w.multipass ? 8 : 0);
    const void* key[4] = {xv, pv, apv, diag};
    Workspace::CgGraph* hit = nullptr;
    for (auto& cg : w.cg_graphs)
      if (cg.exec && cg.con == con && std::memcmp(cg.key, key, sizeof key) == 0) hit = &cg;
    if (!hit) {
      Workspace::CgGraph& slot = w.cg_graphs[w.cg_graph_next];
      w.cg_graph_next = (w.cg_graph_next + 1) % 4;
      if (slot.exec) cudaGraphExecDestroy(slot.exec);
      slot.exec = nullptr;
      cudaError_t ge = cudaSuccess;
      if (!w.graph_st) ge = cudaStreamCreateWithFlags(&w.graph_st, cudaStreamNonBlocking);
      if (!ge && !w.ev_g0) ge = cudaEventCreateWithFlags(&w.ev_g0, cudaEventDisableTiming);
      if (!ge && !w.ev_g1) ge = cudaEventCreateWithFlags(&w.ev_g1, cudaEventDisableTiming);
      cudaGraph_t graph = nullptr;
      if (!ge) ge = cudaStreamBeginCapture(w.graph_st, cudaStreamCaptureModeThreadLocal);
      if (!ge) {
        cudaError_t le = cudaSuccess;
        for (int i = 0; i < kCgGraphBlock && !le; ++i) le = iteration(w.graph_st);
        ge = cudaStreamEndCapture(w.graph_st, &graph);
        if (!ge) ge = le;
      }
      if (!ge) ge = cudaGraphInstantiate(&slot.exec, graph, 0);
      if (!ge) ge = cudaGraphUpload(slot.exec, w.graph_st);
      if (graph) cudaGraphDestroy(graph);
      if (ge) {  // no graph on this system / configuration: the eager loop
        cudaGetLastError();
        if (slot.exec) cudaGraphExecDestroy(slot.exec);
        slot.exec = nullptr;
        w.cg_graph_failed = 1;
      } else {
        std::memcpy(slot.key, key, sizeof key);
        slot.con = con;
        hit = &slot;
      }
    }
    if (hit) {
      CK(cudaEventRecord(w.ev_g0, st));
      CK(cudaStreamWaitEvent(w.graph_st, w.ev_g0, 0));
      for (; k0 + kCgGraphBlock - 1 <= max_iter; k0 += kCgGraphBlock) {
        CK(cudaGraphLaunch(hit->exec, w.graph_st));
        if (rel_tol > 0.0 && k0 + kCgGraphBlock - 1 < max_iter) {
          CK(cudaMemcpyAsync(w.host_sc, w.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, w.graph_st));
          CK(cudaStreamSynchronize(w.graph_st));
          if (w.host_sc->status != ST_RUNNING) {
            k0 = max_iter + 1;
            break;
          }
        }
      }
      CK(cudaEventRecord(w.ev_g1, w.graph_st));
      CK(cudaStreamWaitEvent(st, w.ev_g1, 0));
    }
  }
  for (int k = k0; k <= max_iter; ++k) {
    CK(iteration(st));
    if (k % check_every == 0 && k < max_iter) {
      CK(cudaMemcpyAsync(w.host_sc, w.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (w.host_sc->status != ST_RUNNING) break;
    }
  }
  if (w.use_pt)
    CK(launch_copy_rows(x, static_cast<int>(Nx), w.xt, w.pt_pitch, static_cast<int>(Nx), rows, st));
  CK(cudaMemcpyAsync(w.host_sc, w.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const DevScalars hs = *w.host_sc;
  if (history) CK(cudaMemcpy(history, w.history, sizeof(double) * (hs.iterations + 1), cudaMemcpyDeviceToHost));
  if (report) {
    double last = hs.r0;
    if (hs.iterations > 0) CK(cudaMemcpy(&last, w.history + hs.iterations, sizeof(double), cudaMemcpyDeviceToHost));
    report->iterations = hs.iterations;
    report->converged = hs.status == ST_CONVERGED;
    report->r0_norm = hs.r0;
    report->final_rel_residual = hs.r0 == 0.0 ? 0.0 : last / hs.r0;
    report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  if (hs.status == ST_DIVERGED) {
    set_error(hs.iterations == 0 && !std::isfinite(hs.r0) ? "cg: non-finite initial residual"
                                                          : "cg: operator not positive definite on the search space "
                                                            "or non-finite residual");
    return HEXBP_DIVERGENCE;
  }
  return HEXBP_OK;
}

}  // namespace

extern "C" {

int hexbp_cg_host(hexbp_setup_t h, hexbp_workspace_t wh, const double* b, double* x, int64_t n, double rel_tol,
                  int max_iter, int constrained, hexbp_cg_report* report, double* history) {
  if (!h || !wh || !b || !x) return invalid("cg: null argument");
  if (n != h->s.nL) return invalid("cg: x0 length mismatch");  // solver.hpp:96
  DeviceGuard g(h->s.device);
  Workspace& w = wh->w;
  int rc = ensure_host_staging(w);
  if (rc) return rc;
  CK(stage_solve_inputs(w, b, x, n, nullptr));
  rc = pcg_run(h, wh, w.tmp_u, w.tmp_w, nullptr, rel_tol, max_iter, constrained, report, history, nullptr, w.ev_b);
  if (rc == HEXBP_OK || rc == HEXBP_DIVERGENCE) CK(cudaMemcpy(x, w.tmp_w, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return rc;
}

int hexbp_dot(hexbp_workspace_t wh, const double* a, const double* b, int64_t n, double* out, void* stream) {
  if (!wh || !a || !b || !out) return invalid("dot: null argument");
  Workspace& w = wh->w;
  // the chunk partials live in the workspace's vec_partials (sized for the
  // setup's L-vector at workspace creation)
  if (n < 0 || n > dot_capacity(w.s->nL)) return invalid("dot: length exceeds the workspace's reduction buffer");
  DeviceGuard g(w.device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* dres = w.dot_result;
  CK(launch_dot(w, a, b, n, dres, st));
  CK(cudaMemcpyAsync(out, dres, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return HEXBP_OK;
}

int hexbp_workspace_vectors(hexbp_workspace_t wh, double** r, double** p, double** Ap) {
  if (!wh || !r || !p || !Ap) return invalid("null argument");
  *r = wh->w.r;
  *p = wh->w.p;
  *Ap = wh->w.Ap;
  return HEXBP_OK;
}

int hexbp_cgd_reduce(hexbp_workspace_t wh, int op, const double* b, int64_t owned, double* partial, void* stream) {
  if (!wh || !partial || op < 0 || op > 2 || (op == 0 && !b)) return invalid("cgd_reduce: bad argument");
  Workspace& w = wh->w;
  if (owned < 0 || owned > w.s->nL) return invalid("cgd_reduce: owned offset outside the L-vector");
  DeviceGuard g(w.device);
  CK(launch_cgd_reduce(w, op, b, w.s->nL, owned, partial, static_cast<cudaStream_t>(stream)));
  return HEXBP_OK;
}

int hexbp_cgd_finish(hexbp_workspace_t wh, int op, const double* gathered, int world, double rel_tol, int max_iter,
                     void* stream) {
  if (!wh || !gathered || world < 1 || op < 0 || op > 2) return invalid("cgd_finish: bad argument");
  Workspace& w = wh->w;
  DeviceGuard g(w.device);
  if (op == 0) {
    const int rc = ensure_history(w, max_iter);
    if (rc) return rc;
  }
  CK(launch_cgd_finish(w, op, gathered, world, rel_tol, max_iter, static_cast<cudaStream_t>(stream)));
  return HEXBP_OK;
}

int hexbp_cgd_apply_fused(hexbp_setup_t h, hexbp_workspace_t wh, int constrained, double* partial, void* stream) {
  if (!h || !wh || !partial) return invalid("cgd_apply_fused: null argument");
  Workspace& w = wh->w;
  const Setup& s = h->s;
  if (w.s != &s) return invalid("cgd_apply_fused: workspace belongs to another setup");
  if (w.exact || w.multipass) return invalid("cgd_apply_fused: fast mode only");
  DeviceGuard g(s.device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(launch_apply(s, w, w.p, w.Ap, constrained, partial, nullptr, st, /*finish_ring=*/false));
  const int Nz = s.dims[2] * s.p + 1;
  if (s.z0 > 0) CK(launch_lateral_fixup_planes(s, w, w.p, w.Ap, constrained, 0, 1, st));
  if (s.z0 + s.dims[2] < s.gdims[2]) CK(launch_lateral_fixup_planes(s, w, w.p, w.Ap, constrained, Nz - 1, Nz, st));
  return HEXBP_OK;
}

int hexbp_cgd_update_r_fused(hexbp_workspace_t wh, int constrained, double* partial, void* stream) {
  if (!wh || !partial) return invalid("cgd_update_r_fused: null argument");
  Workspace& w = wh->w;
  if (w.exact || w.multipass) return invalid("cgd_update_r_fused: fast mode only");
  DeviceGuard g(w.device);
  CK(launch_cgd_update_r_fused(w, constrained, partial, static_cast<cudaStream_t>(stream)));
  return HEXBP_OK;
}

int hexbp_cgd_update_xp(hexbp_workspace_t wh, double* x, void* stream) {
  if (!wh || !x) return invalid("null argument");
  DeviceGuard g(wh->w.device);
  CK(launch_cg_update_xp(wh->w, x, wh->w.s->nL, static_cast<cudaStream_t>(stream)));
  return HEXBP_OK;
}

int hexbp_cgd_report(hexbp_workspace_t wh, int* status, hexbp_cg_report* report, double* history, int cap) {
  if (!wh) return invalid("null argument");
  Workspace& w = wh->w;
  DeviceGuard g(w.device);
  CK(cudaDeviceSynchronize());
  DevScalars hs;
  CK(cudaMemcpy(&hs, w.sc, sizeof hs, cudaMemcpyDeviceToHost));
  if (status) *status = hs.status;
  if (history && cap > 0) {
    const int m = hs.iterations + 1 < cap ? hs.iterations + 1 : cap;
    CK(cudaMemcpy(history, w.history, sizeof(double) * m, cudaMemcpyDeviceToHost));
  }
  if (report) {
    double last = hs.r0;
    if (hs.iterations > 0) CK(cudaMemcpy(&last, w.history + hs.iterations, sizeof(double), cudaMemcpyDeviceToHost));
    report->iterations = hs.iterations;
    report->converged = hs.status == ST_CONVERGED;
    report->r0_norm = hs.r0;
    report->final_rel_residual = hs.r0 == 0.0 ? 0.0 : last / hs.r0;
    report->seconds = 0.0;
  }
  return hs.status == ST_DIVERGED ? (set_error("cg: divergence"), HEXBP_DIVERGENCE) : HEXBP_OK;
}

int hexbp_plane_combine(double* dst, const double* src, const double* u, int nxn, int nyn, int constrained,
                        void* stream) {
  if (!dst || !src || (constrained && !u) || nxn < 1 || nyn < 1) return invalid("plane_combine: bad argument");
  CK(launch_plane_combine(dst, src, u, nxn, nyn, constrained, static_cast<cudaStream_t>(stream)));
  return HEXBP_OK;
}

int hexbp_workspace_set_mode(hexbp_workspace_t wh, int mode) {
  if (!wh || (mode != HEXBP_MODE_REFERENCE && mode != HEXBP_MODE_FAST && mode != HEXBP_MODE_FAST_OPERATOR))
    return invalid("bad arithmetic mode");
  if (wh->w.multipass && mode != HEXBP_MODE_REFERENCE)
    return invalid(wh->w.s->p > kMaxP ? "degree > 8 runs the multipass pipeline, in reference arithmetic only"
                                      : "the multipass backend runs in reference arithmetic only");
  wh->w.exact = mode != HEXBP_MODE_FAST;
  wh->w.fast_op = mode == HEXBP_MODE_FAST_OPERATOR;
  return HEXBP_OK;
}

int hexbp_workspace_set_backend(hexbp_workspace_t wh, int backend) {
  if (!wh || (backend != HEXBP_BACKEND_FUSED && backend != HEXBP_BACKEND_MULTIPASS)) return invalid("bad backend");
  Workspace& w = wh->w;
  if (backend == HEXBP_BACKEND_FUSED && w.s->p > kMaxP) return invalid("the fused kernels take degrees 1..8");
  DeviceGuard g(w.device);
  if (backend == HEXBP_BACKEND_MULTIPASS && !w.mp_buf) {
    const size_t bytes = sizeof(double) * static_cast<size_t>(multipass_doubles(*w.s));
    if (cudaMalloc(&w.mp_buf, bytes) != cudaSuccess) {
      w.mp_buf = nullptr;
      return cuda_status(cudaErrorMemoryAllocation, "multipass workspace");
    }
    const cudaError_t e = launch_apply_multipass(*w.s, w.mp_buf, nullptr, nullptr, 0, nullptr, /*upload=*/true);
    if (e != cudaSuccess) return cuda_status(e, "multipass basis upload");
  }
  w.multipass = backend == HEXBP_BACKEND_MULTIPASS;
  if (w.multipass) {
    w.exact = 1;
    w.fast_op = 0;
  }
  return HEXBP_OK;
}

int hexbp_workspace_info(hexbp_workspace_t wh, int* qpoint_fields, uint64_t* global_bytes) {
  if (!wh || !qpoint_fields || !global_bytes) return invalid("null argument");
  const Workspace& w = wh->w;
  const int nf = w.s->kind == KIND_MASS ? 1 : 3;
  *qpoint_fields = w.multipass ? 2 * nf : 0;  // operator.hpp:159-172
  *global_bytes = w.multipass ? sizeof(double) * static_cast<uint64_t>(multipass_doubles(*w.s)) + w.scatter_bytes
                              : w.scatter_bytes;
  return HEXBP_OK;
}

int hexbp_count_flops(hexbp_setup_t h, uint64_t* mul, uint64_t* add) {
  if (!h || !mul || !add) return invalid("null argument");
  const uint64_t N = h->s.p + 1, Q = h->s.q;
  uint64_t fma = 0, m = 0, a = 0;
  switch (h->s.kind) {
    case KIND_DIFF:
      fma = 4 * N * N * N * Q + 6 * N * N * Q * Q + 6 * N * Q * Q * Q;
      m = 9 * Q * Q * Q;
      a = 6 * Q * Q * Q;
      break;
    case KIND_COLLOC:
      fma = 6 * N * N * N * N;
      m = 9 * N * N * N;
      a = 6 * N * N * N + 2 * N * N * N;  // + the identity-branch adds of Y'/Z'
      break;
    default:
      fma = 2 * (N * N * N * Q + N * N * Q * Q + N * Q * Q * Q);
      m = Q * Q * Q;
      break;
  }
  *mul = fma + m;
  *add = fma + a;
  return HEXBP_OK;
}

int hexbp_kernel_info(hexbp_setup_t h, int* regs, int* smem, int* threads, int* ctas) {
  if (!h || !regs || !smem || !threads || !ctas) return invalid("null argument");
  DeviceGuard g(h->s.device);
  apply_kernel_info(h->s, regs, smem, threads, ctas);
  return HEXBP_OK;
}

}  // extern "C"
