// Multi-GPU z-slab operator and CG behind the C ABI, one rank
// (process) per GPU, NCCL over NVLink for the two exchange steps the BP
// operator and CG have. The reference is single address space;
// this is the scale-out of its OperatorHandle::apply / cg (operator.hpp:
// 265-279, solver.hpp:91-153) that a C++ caller reaches through
// hexbp_dist_* (include/hexbp_b200.h) or hexbp::b200::DistributedOperator
// (include/hexbp_b200.hpp).
//
// Partition: contiguous element layers [z0, z1) per rank, in rank order. A
// rank owns node planes Z = z0 p .. z1 p; the top plane is shared with rank+1
// (each holds its own partial sum of it).
//
// Halo sum (the shared-node gather-scatter of restriction.hpp:67-80 across
// ranks): the two ranks swap their partial planes (ncclSend/ncclRecv in one
// group) and both add dst + src -- IEEE addition commutes, so the two copies
// are bitwise equal and no ownership fix-up is needed.
//
// CG scalars: each rank reduces over the nodes it owns (plane 0 belongs to the
// rank below), the partials are all-gathered (ncclAllGather, one double) and
// summed in rank order on every rank by the same one-thread kernel, so all
// ranks run the identical scalar recurrence.
//
// Overlap (fast mode, kernels with element-range support): per operator apply
//   stream st : boundary layers (element 0 and nz-1 of every column, their
//               inner node planes to carry buffers) -> ring sums of the two
//               shared planes -> NCCL plane exchange (+ the p.Ap all-gather of
//               the previous step's data is not needed: see below)
//   stream st2: interior layers 1 .. nz-2 (concurrently)
//   join      : the two inner planes assembled from the carries
//               (carry_combine_kernel, exactly the sum the single-launch
//               march forms), the halo planes combined, the rank's p.Ap
//               share summed from the launches' partials in fixed order.
// The halo transfer therefore runs while the interior elements compute.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the entry points are resolved at run time (nccl())

#include <cmath>
#include <cstring>
#include <initializer_list>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "capi_util.h"
#include "internal.h"
#include "ring.cuh"

struct hexbp_dist_s {
  hexbp_setup_t setup = nullptr;
  bool own_setup = false;
  hexbp_workspace_t ws = nullptr;
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
  bool has_up = false, has_down = false;
  int nxn = 0, nyn = 0;
  int64_t plane = 0, nL = 0, owned = 0;
  double* halo_up = nullptr;    // partial plane received from rank + 1
  double* halo_down = nullptr;  // from rank - 1
  double* scal = nullptr;       // [0]: this rank's partial, [1 .. world]: gathered
  hxb::OverlapBuffers ob{};     // boundary / interior split (overlap.cu)
  cudaStream_t st2 = nullptr;   // interior launches
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int overlap = 1;              // HEXBP_DIST_OVERLAP
  int fast = 1;                 // fused fast iteration (HEXBP_MODE_FAST) or reference reductions
};

using namespace hxb;

namespace {

// NCCL is resolved at run time (dlopen of libnccl.so.2 on first use): a
// process that already loaded NCCL -- PyTorch's bundled one -- shares that copy,
// and loading this library never forces a second, older libnccl.so.2 on a
// process whose other libraries need the newer one.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(h, name)); };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.AllGather, "ncclAllGather");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.AllGather && a.GroupStart &&
           a.GroupEnd && a.GetErrorString;
    return a;
  }();
  return api;
}

int nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return HEXBP_OK;
  set_error(std::string(where) + ": " + nccl().GetErrorString(r));
  return HEXBP_CUDA_ERROR;
}

int need_nccl() {
  if (nccl().ok) return HEXBP_OK;
  set_error("dist: libnccl.so.2 not found or incomplete (the multi-GPU path needs NCCL)");
  return HEXBP_CUDA_ERROR;
}

#define NK(call)                                       \
  do {                                                 \
    ncclResult_t _r = (call);                          \
    if (_r != ncclSuccess) return nccl_status(_r, #call); \
  } while (0)

// Balanced z split of gz element layers over `world` ranks (bench.py and
// parallel.SlabPartition use the same rule).
void slab_range(int gz, int world, int rank, int* z0, int* z1) {
  const int base = gz / world, rem = gz % world;
  *z0 = rank * base + (rank < rem ? rank : rem);
  *z1 = *z0 + base + (rank < rem ? 1 : 0);
}

// All ranks' slab parameters must tile the same global box in rank order.
int check_layout(hexbp_dist_s& d, cudaStream_t st) {
  const Setup& s = d.setup->s;
  int mine[8] = {s.bp, s.p, s.gdims[0], s.gdims[1], s.gdims[2], s.z0, s.z0 + s.dims[2], d.rank};
  int* dev = nullptr;
  CK(cudaMalloc(&dev, sizeof(int) * 8 * (d.world + 1)));
  std::vector<int> all(8 * d.world);
  cudaError_t e = cudaMemcpyAsync(dev, mine, sizeof mine, cudaMemcpyHostToDevice, st);
  ncclResult_t r = e ? ncclSuccess : nccl().AllGather(dev, dev + 8, 8, ncclInt32, d.comm, st);
  if (!e && r == ncclSuccess) e = cudaMemcpyAsync(all.data(), dev + 8, sizeof(int) * 8 * d.world,
                                                  cudaMemcpyDeviceToHost, st);
  if (!e && r == ncclSuccess) e = cudaStreamSynchronize(st);
  cudaFree(dev);
  CK(e);
  NK(r);
  int next_z = 0;
  for (int k = 0; k < d.world; ++k) {
    const int* o = all.data() + 8 * k;
    if (o[0] != mine[0] || o[1] != mine[1] || o[2] != mine[2] || o[3] != mine[3] || o[4] != mine[4] || o[7] != k)
      return invalid("dist: ranks disagree on (bp, p, global box)");
    if (o[5] != next_z) return invalid("dist: slabs must tile the box in rank order (z0 of rank k = z1 of rank k-1)");
    next_z = o[6];
  }
  if (next_z != s.gdims[2]) return invalid("dist: slabs do not cover the box");
  return HEXBP_OK;
}

// Halo sum of the shared planes of w (this rank's partials -> assembled).
// One NCCL group: both neighbours' planes, plus (optionally) the all-gather of
// this rank's scalar partial scal[0] -> scal[1 .. world].
int exchange(hexbp_dist_s& d, const double* u, double* w, int constrained, bool gather, cudaStream_t st) {
  if (d.world == 1) {
    if (gather) CK(cudaMemcpyAsync(d.scal + 1, d.scal, sizeof(double), cudaMemcpyDeviceToDevice, st));
    return HEXBP_OK;
  }
  NK(nccl().GroupStart());
  if (d.has_up) {
    NK(nccl().Send(w + d.nL - d.plane, d.plane, ncclDouble, d.rank + 1, d.comm, st));
    NK(nccl().Recv(d.halo_up, d.plane, ncclDouble, d.rank + 1, d.comm, st));
  }
  if (d.has_down) {
    NK(nccl().Send(w, d.plane, ncclDouble, d.rank - 1, d.comm, st));
    NK(nccl().Recv(d.halo_down, d.plane, ncclDouble, d.rank - 1, d.comm, st));
  }
  if (gather) NK(nccl().AllGather(d.scal, d.scal + 1, 1, ncclDouble, d.comm, st));
  NK(nccl().GroupEnd());
  // stream order: the group's sends have completed before the combines write
  if (d.has_up)
    CK(launch_plane_combine(w + d.nL - d.plane, d.halo_up, u + d.nL - d.plane, d.nxn, d.nyn, constrained, st));
  if (d.has_down) CK(launch_plane_combine(w, d.halo_down, u, d.nxn, d.nyn, constrained, st));
  return HEXBP_OK;
}

int gather_scalar(hexbp_dist_s& d, cudaStream_t st) {
  if (d.world == 1) {
    CK(cudaMemcpyAsync(d.scal + 1, d.scal, sizeof(double), cudaMemcpyDeviceToDevice, st));
    return HEXBP_OK;
  }
  NK(nccl().AllGather(d.scal, d.scal + 1, 1, ncclDouble, d.comm, st));
  return HEXBP_OK;
}

// Ap = A p with this rank's p.Ap share in scal[0]; shared planes assembled
// (ring sums of the two shared planes locally, then the halo), partial
// all-gathered into scal[1 ..]. Overlapped when the kernel supports ranges.
int apply_fused(hexbp_dist_s& d, int constrained, cudaStream_t st) {
  Workspace& w = d.ws->w;
  const Setup& s = d.setup->s;
  if (d.overlap && apply_overlap_supported(s)) {
    CK(cudaEventRecord(d.ev_fork, st));
    CK(cudaStreamWaitEvent(d.st2, d.ev_fork, 0));
    const OverlapBuffers& ob = d.ob;
    CK(launch_apply_boundary(s, w, w.p, w.Ap, constrained, ob, st));
    CK(launch_apply_interior(s, w, w.p, w.Ap, constrained, ob, d.st2));
    const int Nz = s.dims[2] * s.p + 1;
    if (d.has_down) CK(launch_lateral_fixup_planes(s, w, w.p, w.Ap, constrained, 0, 1, st));
    if (d.has_up) CK(launch_lateral_fixup_planes(s, w, w.p, w.Ap, constrained, Nz - 1, Nz, st));
    // the plane exchange runs on st while the interior launch computes on st2
    int rc = exchange(d, w.p, w.Ap, constrained, /*gather=*/false, st);
    if (rc) return rc;
    CK(cudaEventRecord(d.ev_join, d.st2));
    CK(cudaStreamWaitEvent(st, d.ev_join, 0));
    CK(launch_carry_combine(s, w, w.p, w.Ap, constrained, ob, d.scal, st));
    return gather_scalar(d, st);
  }
  CK(launch_apply(s, w, w.p, w.Ap, constrained, d.scal, nullptr, st, /*finish_ring=*/false));
  const int Nz = s.dims[2] * s.p + 1;
  if (d.has_down) CK(launch_lateral_fixup_planes(s, w, w.p, w.Ap, constrained, 0, 1, st));
  if (d.has_up) CK(launch_lateral_fixup_planes(s, w, w.p, w.Ap, constrained, Nz - 1, Nz, st));
  return exchange(d, w.p, w.Ap, constrained, /*gather=*/true, st);
}

int finish(hexbp_dist_s& d, int op, double rel_tol, int max_iter, cudaStream_t st) {
  CK(launch_cgd_finish(d.ws->w, op, d.scal + 1, d.world, rel_tol, max_iter, st));
  return HEXBP_OK;
}

int reduce_gather(hexbp_dist_s& d, int op, const double* b, cudaStream_t st) {
  CK(launch_cgd_reduce(d.ws->w, op, b, d.nL, d.owned, d.scal, st));
  return gather_scalar(d, st);
}

}  // namespace

extern "C" {

int hexbp_dist_unique_id(void* id, int64_t bytes) {
  if (!id || bytes < static_cast<int64_t>(sizeof(ncclUniqueId))) return invalid("dist_unique_id: buffer too small");
  if (const int rc = need_nccl()) return rc;
  ncclUniqueId u;
  NK(nccl().GetUniqueId(&u));
  std::memcpy(id, &u, sizeof u);
  return HEXBP_OK;
}

int hexbp_dist_create(hexbp_setup_t slab, int world, int rank, const void* id, int64_t id_bytes, int flags,
                      hexbp_dist_t* out) {
  if (!slab || !id || !out || world < 1 || rank < 0 || rank >= world) return invalid("dist_create: bad argument");
  if (id_bytes < static_cast<int64_t>(sizeof(ncclUniqueId))) return invalid("dist_create: NCCL id too short");
  if (const int rc = need_nccl()) return rc;
  *out = nullptr;
  auto* d = new (std::nothrow) hexbp_dist_s;
  if (!d) return HEXBP_OUT_OF_MEMORY;
  const Setup& s = slab->s;
  d->setup = slab;
  d->world = world;
  d->rank = rank;
  d->device = s.device;
  d->overlap = (flags & HEXBP_DIST_NO_OVERLAP) ? 0 : 1;
  d->has_down = s.z0 > 0;
  d->has_up = s.z0 + s.dims[2] < s.gdims[2];
  d->nxn = s.gdims[0] * s.p + 1;
  d->nyn = s.gdims[1] * s.p + 1;
  d->plane = static_cast<int64_t>(d->nxn) * d->nyn;
  d->nL = s.nL;
  d->owned = d->has_down ? d->plane : 0;
  DeviceGuard g(s.device);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  int rc = HEXBP_OK;
  {
    const ncclResult_t r = nccl().CommInitRank(&d->comm, world, u, rank);
    if (r != ncclSuccess) rc = nccl_status(r, "ncclCommInitRank");
  }
  if (!rc) rc = hexbp_workspace_create(slab, &d->ws);
  if (!rc) rc = hexbp_workspace_set_mode(d->ws, HEXBP_MODE_FAST);
  if (!rc) rc = hexbp_workspace_reserve(d->ws, 0, 0);
  cudaError_t e = cudaSuccess;
  auto al = [&](double** p, int64_t n) {
    if (!e && !rc) e = cudaMalloc(p, sizeof(double) * static_cast<size_t>(n));
    if (!e && !rc) e = cudaMemset(*p, 0, sizeof(double) * static_cast<size_t>(n));
  };
  al(&d->halo_up, d->plane);
  al(&d->halo_down, d->plane);
  al(&d->scal, d->world + 1);
  if (apply_overlap_supported(s)) {
    al(&d->ob.carry, overlap_carry_doubles(s));
    al(&d->ob.slots, 4);
    al(&d->ob.coldot, 3LL * s.dims[0] * s.dims[1]);
    al(&d->ob.partials, overlap_partials_capacity());
    al(reinterpret_cast<double**>(&d->ob.tickets), 2);  // 4 zeroed unsigned ints
  }
  if (!e && !rc) e = cudaStreamCreateWithFlags(&d->st2, cudaStreamNonBlocking);
  if (!e && !rc) e = cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming);
  if (!e && !rc) e = cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming);
  if (e && !rc) rc = cuda_status(e, "dist_create");
  if (!rc) rc = check_layout(*d, nullptr);
  if (rc) {
    const std::string msg = hexbp_last_error();
    hexbp_dist_destroy(d);
    set_error(msg);
    return rc;
  }
  *out = d;
  return HEXBP_OK;
}

int hexbp_dist_create_box(int bp, int p, const int gdims[3], const double extent[3], double amplitude, int world,
                          int rank, int device, const void* id, int64_t id_bytes, int flags, hexbp_dist_t* out) {
  if (!gdims || !out || world < 1 || rank < 0 || rank >= world) return invalid("dist_create_box: bad argument");
  if (gdims[2] < world) return invalid("dist_create_box: fewer element layers than ranks");
  int z0 = 0, z1 = 0;
  slab_range(gdims[2], world, rank, &z0, &z1);
  hexbp_setup_t s = nullptr;
  int rc = hexbp_setup_create_box_slab(bp, p, gdims, z0, z1, extent, amplitude, device, &s);
  if (rc) return rc;
  rc = hexbp_dist_create(s, world, rank, id, id_bytes, flags, out);
  if (rc) {
    hexbp_setup_destroy(s);
    return rc;
  }
  (*out)->own_setup = true;
  return HEXBP_OK;
}

void hexbp_dist_destroy(hexbp_dist_t d) {
  if (!d) return;
  {
    DeviceGuard g(d->device);
    if (d->comm) nccl().CommDestroy(d->comm);
    for (void* b : {static_cast<void*>(d->halo_up), static_cast<void*>(d->halo_down), static_cast<void*>(d->scal),
                    static_cast<void*>(d->ob.carry), static_cast<void*>(d->ob.slots),
                    static_cast<void*>(d->ob.coldot), static_cast<void*>(d->ob.partials),
                    static_cast<void*>(d->ob.tickets)})
      if (b) cudaFree(b);
    if (d->st2) cudaStreamDestroy(d->st2);
    if (d->ev_fork) cudaEventDestroy(d->ev_fork);
    if (d->ev_join) cudaEventDestroy(d->ev_join);
    if (d->ws) hexbp_workspace_destroy(d->ws);
  }
  if (d->own_setup) hexbp_setup_destroy(d->setup);
  delete d;
}

int hexbp_dist_info(hexbp_dist_t d, hexbp_setup_t* setup, int* world, int* rank, int64_t* l_size,
                    int64_t* owned_offset, int64_t* global_offset) {
  if (!d) return invalid("null argument");
  const Setup& s = d->setup->s;
  if (setup) *setup = d->setup;
  if (world) *world = d->world;
  if (rank) *rank = d->rank;
  if (l_size) *l_size = d->nL;
  if (owned_offset) *owned_offset = d->owned;
  if (global_offset) *global_offset = d->plane * static_cast<int64_t>(s.z0) * s.p;
  return HEXBP_OK;
}

int hexbp_dist_set_mode(hexbp_dist_t d, int mode) {
  if (!d || (mode != HEXBP_MODE_REFERENCE && mode != HEXBP_MODE_FAST)) return invalid("dist_set_mode: bad mode");
  const int rc = hexbp_workspace_set_mode(d->ws, mode);
  if (!rc) d->fast = mode == HEXBP_MODE_FAST;
  return rc;
}

int hexbp_dist_apply(hexbp_dist_t d, const double* u, double* w, int constrained, void* stream) {
  if (!d || !u || !w) return invalid("dist_apply: null argument");
  if (u == w) return invalid("dist_apply: u and w must not alias");
  DeviceGuard g(d->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Setup& s = d->setup->s;
  Workspace& ws = d->ws->w;
  if (d->fast && d->overlap && apply_overlap_supported(s)) {
    // boundary layers -> their two planes' ring sums -> plane exchange, while
    // the interior layers compute on st2; then the inner planes and the rest
    // of the ring sums (every plane once, as launch_apply's fix-up)
    const int Nz = s.dims[2] * s.p + 1;
    CK(cudaEventRecord(d->ev_fork, st));
    CK(cudaStreamWaitEvent(d->st2, d->ev_fork, 0));
    CK(launch_apply_boundary(s, ws, u, w, constrained, d->ob, st));
    CK(launch_apply_interior(s, ws, u, w, constrained, d->ob, d->st2));
    CK(launch_lateral_fixup_planes(s, ws, u, w, constrained, 0, 1, st));
    CK(launch_lateral_fixup_planes(s, ws, u, w, constrained, Nz - 1, Nz, st));
    const int rc = exchange(*d, u, w, constrained, /*gather=*/false, st);
    if (rc) return rc;
    CK(cudaEventRecord(d->ev_join, d->st2));
    CK(cudaStreamWaitEvent(st, d->ev_join, 0));
    CK(launch_carry_combine(s, ws, u, w, constrained, d->ob, d->scal, st));
    CK(launch_lateral_fixup_planes(s, ws, u, w, constrained, 1, Nz - 1, st));
    return HEXBP_OK;
  }
  CK(launch_apply(s, ws, u, w, constrained, nullptr, nullptr, st));
  return exchange(*d, u, w, constrained, /*gather=*/false, st);
}

int hexbp_dist_apply_host(hexbp_dist_t d, const double* u, double* w, int64_t n, int constrained) {
  if (!d || !u || !w) return invalid("dist_apply: null argument");
  if (n != d->nL) return invalid("apply: L-vector length mismatch");  // operator.hpp:268
  DeviceGuard g(d->device);
  int rc = hexbp_workspace_reserve(d->ws, 0, 1);
  if (rc) return rc;
  Workspace& ws = d->ws->w;
  CK(cudaMemcpy(ws.tmp_u, u, sizeof(double) * n, cudaMemcpyHostToDevice));
  if ((rc = hexbp_dist_apply(d, ws.tmp_u, ws.tmp_w, constrained, nullptr))) return rc;
  CK(cudaMemcpy(w, ws.tmp_w, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return HEXBP_OK;
}

int hexbp_dist_cg(hexbp_dist_t d, const double* b, double* x, double rel_tol, int max_iter, int constrained,
                  hexbp_cg_report* report, double* history, void* stream) {
  if (!d || !b || !x) return invalid("dist_cg: null argument");
  if (max_iter < 0) return invalid("cg: max_iter must be >= 0");
  DeviceGuard g(d->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Workspace& w = d->ws->w;
  const Setup& s = d->setup->s;
  int rc = hexbp_workspace_reserve(d->ws, max_iter, 0);
  if (rc) return rc;
  // r0 = b - A x0 (solver.hpp:102-103) with the assembled A x0
  CK(launch_apply(s, w, x, w.Ap, constrained, nullptr, nullptr, st));
  if ((rc = exchange(*d, x, w.Ap, constrained, false, st))) return rc;
  if ((rc = reduce_gather(*d, HEXBP_CGD_INIT, b, st))) return rc;
  if ((rc = finish(*d, HEXBP_CGD_INIT, rel_tol, max_iter, st))) return rc;
  const int check_every = rel_tol > 0.0 ? 8 : (1 << 30);
  for (int k = 1; k <= max_iter; ++k) {
    if (d->fast) {
      // the single-GPU fast iteration split at its two global reductions
      if ((rc = apply_fused(*d, constrained, st))) return rc;
      if ((rc = finish(*d, HEXBP_CGD_PAP, rel_tol, max_iter, st))) return rc;
      CK(launch_cgd_update_r_fused(w, constrained, d->scal, st));
      if ((rc = gather_scalar(*d, st))) return rc;
      if ((rc = finish(*d, HEXBP_CGD_UPDATE_R, rel_tol, max_iter, st))) return rc;
    } else {
      CK(launch_apply(s, w, w.p, w.Ap, constrained, nullptr, nullptr, st));
      if ((rc = exchange(*d, w.p, w.Ap, constrained, false, st))) return rc;
      if ((rc = reduce_gather(*d, HEXBP_CGD_PAP, nullptr, st))) return rc;
      if ((rc = finish(*d, HEXBP_CGD_PAP, rel_tol, max_iter, st))) return rc;
      if ((rc = reduce_gather(*d, HEXBP_CGD_UPDATE_R, nullptr, st))) return rc;
      if ((rc = finish(*d, HEXBP_CGD_UPDATE_R, rel_tol, max_iter, st))) return rc;
    }
    CK(launch_cg_update_xp(w, x, d->nL, st));
    if (k % check_every == 0 && k < max_iter) {
      CK(cudaMemcpyAsync(w.host_sc, w.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (w.host_sc->status != ST_RUNNING) break;  // identical on every rank
    }
  }
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
    report->seconds = 0.0;
  }
  if (hs.status == ST_DIVERGED) {
    set_error("cg: operator not positive definite on the search space or non-finite residual");
    return HEXBP_DIVERGENCE;
  }
  return HEXBP_OK;
}

int hexbp_dist_cg_host(hexbp_dist_t d, const double* b, double* x, int64_t n, double rel_tol, int max_iter,
                       int constrained, hexbp_cg_report* report, double* history) {
  if (!d || !b || !x) return invalid("dist_cg: null argument");
  if (n != d->nL) return invalid("cg: x0 length mismatch");  // solver.hpp:96
  DeviceGuard g(d->device);
  int rc = hexbp_workspace_reserve(d->ws, max_iter, 1);
  if (rc) return rc;
  Workspace& ws = d->ws->w;
  CK(cudaMemcpy(ws.tmp_u, b, sizeof(double) * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ws.tmp_w, x, sizeof(double) * n, cudaMemcpyHostToDevice));
  rc = hexbp_dist_cg(d, ws.tmp_u, ws.tmp_w, rel_tol, max_iter, constrained, report, history, nullptr);
  if (rc == HEXBP_OK || rc == HEXBP_DIVERGENCE) CK(cudaMemcpy(x, ws.tmp_w, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return rc;
}

}  // extern "C"
