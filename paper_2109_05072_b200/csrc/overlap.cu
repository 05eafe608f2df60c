// Boundary / interior split of one slab operator apply, for the multi-GPU
// overlap of dist.cu ("boundary layers first, post the plane
// exchange, interior elements, add the neighbour's partial").
//
// The fused element-column kernel marches each column bottom to top and
// carries the z-shared node plane between consecutive elements in registers;
// a slab's two shared planes (Z = 0 and Z = Nz-1) are therefore complete only
// at the very start and the very end of every column. Split per column:
//   boundary : element 0 and element nz-1, one element each (two launches on
//              the caller's stream); their inner planes Z = p and (nz-1) p
//              left as carry shares instead of stored
//   interior : elements 1 .. nz-2 (one launch on a second stream, concurrent
//              with the boundary launches and the halo exchange that follows
//              them), both end planes left as carry shares
//   combine  : inner plane value = share of the element above + share of the
//              element below -- exactly the `o(e) + carry(e-1)` sum of the
//              single-launch march, so the assembled A p is bitwise the
//              single launch's -- then the same store / ring / p.Ap logic as
//              the kernel's Z' epilogue (restriction.hpp:67-80 ordering).
// The rank's p.Ap share: the three launches' partials and the combine's, in
// fixed order (deterministic run to run). Both DMMA kernels (BP3 p = 7 and
// BP5 p = 7; BP5's p.Ap is the element energy form, so its combine adds
// nothing to the dot) and the DFMA element kernel (every other degree but the
// thread-per-column BP1 p = 1, 2 and BP5 p = 1) take ranges.
#include <cuda_runtime.h>

#include "device_util.cuh"
#include "internal.h"
#include "ring.cuh"

namespace hxb {

bool use_mma(const Setup& s);
bool dfma_ranges_supported(const Setup& s);                                       // apply.cu
cudaError_t launch_apply_dfma(const Setup& s, const ApplyArgs& a, cudaStream_t st);  // apply.cu

namespace {

constexpr int CT = 256;  // combine threads per block
constexpr int kMaxCombineBlocks = 296;

struct CombineArgs {
  ApplyArgs a;
  const double* lo[2];  // share of the element above the plane (its bottom plane)
  const double* hi[2];  // share of the element below (its top plane)
  int Z[2];             // node plane index
  int nplanes;
  double* partials;     // [gridDim.x]
  unsigned int* ticket;
  const double* slots;  // the launches' p.Ap partials
  int nslots;
  int nodal_dot;        // BP3: the inner planes' p.Ap share is added here; BP5: energy form (in the launches)
  double* out;          // rank share of p.Ap
};

template <int P>
__global__ void __launch_bounds__(CT) carry_combine_kernel(const __grid_constant__ CombineArgs c) {
  constexpr int NN = (P + 1) * (P + 1);
  const ApplyArgs& A = c.a;
  const LatLayout Lat(P, A.nx, A.ny);
  const long long per_plane = static_cast<long long>(A.ncols) * NN;
  const long long total = per_plane * c.nplanes;
  double dot = 0.0;
  for (long long idx = blockIdx.x * static_cast<long long>(CT) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * CT) {
    const int pl = static_cast<int>(idx / per_plane);
    const long long r = idx - pl * per_plane;
    const int col = static_cast<int>(r / NN), node = static_cast<int>(r - static_cast<long long>(col) * NN);
    const int j = node / (P + 1), i = node - j * (P + 1);
    const int ex = col % A.nx, ey = col / A.nx;
    const int Z = c.Z[pl], X = ex * P + i, Y = ey * P + j;
    const long long off = static_cast<long long>(col) * NN + node;
    const double v = c.lo[pl][off] + c.hi[pl][off];
    const double uv = A.u[X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z)];
    if (i == 0 || i == P || j == 0 || j == P) {  // ring node: this column's partial
      if (j == 0 || j == P)
        A.lateral[Lat.y_index(P, A.nx, Z, ey + (j == P), j == 0, ex, i)] = v;
      else
        A.lat_x[Lat.x_index(A.nx, Z, Y, ex + (i == P), i == 0)] = v;
      if (c.nodal_dot) {
        if (A.constrained && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1)) {
          if (ring_owner(P, i, j, ex, ey, A.nx, A.ny)) dot = fma(uv, uv, dot);  // w = u, counted once
        } else {
          dot = fma(uv, v, dot);
        }
      }
    } else {  // inner planes are never z-boundary planes: no constraint here
      A.w[X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z)] = v;
      if (c.nodal_dot) dot = fma(uv, v, dot);
    }
  }
  __shared__ double red[CT / 32];
  __shared__ int last;
  const double bs = block_sum<CT>(dot, red);
  if (threadIdx.x == 0) {
    c.partials[blockIdx.x] = bs;
    __threadfence();
    last = atomicAdd(c.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double s = 0.0;
  for (int k = 0; k < c.nslots; ++k) s += __ldcg(c.slots + k);
  for (unsigned int b = 0; b < gridDim.x; ++b) s += __ldcg(c.partials + b);
  *c.out = s;
  *c.ticket = 0;
}

}  // namespace

bool apply_overlap_supported(const Setup& s) {
  const bool ranges = use_mma(s) ? (mma_kernel_applies(s) || mma5_kernel_applies(s)) : dfma_ranges_supported(s);
  return ranges && s.dims[2] >= 2;
}

static cudaError_t launch_range(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  if (!use_mma(s)) return launch_apply_dfma(s, a, st);
  return mma5_kernel_applies(s) ? launch_apply_mma5(s, a, st) : launch_apply_mma(s, a, st);
}

int64_t overlap_carry_doubles(const Setup& s) {
  return 4LL * s.dims[0] * s.dims[1] * (s.p + 1) * (s.p + 1);
}

static ApplyArgs range_args(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                            const OverlapBuffers& ob, int launch, int zr0, int zr1, double* lo, double* hi) {
  ApplyArgs a = make_apply_args(s, ws, u, w, constrained, ob.slots + launch, nullptr);
  a.col_dot = ob.coldot + static_cast<long long>(launch) * a.ncols;
  a.fix_done = ob.tickets + launch;
  a.zr0 = zr0;
  a.zr1 = zr1;
  a.carry_lo = lo;
  a.carry_hi = hi;
  return a;
}

static double* carry_plane(const Setup& s, const OverlapBuffers& ob, int k) {
  return ob.carry + static_cast<long long>(k) * s.dims[0] * s.dims[1] * (s.p + 1) * (s.p + 1);
}

// carry planes: 0 = element 0's top, 1 = element nz-1's bottom,
//               2 = interior's bottom (element 1), 3 = interior's top (element nz-2)
cudaError_t launch_apply_boundary(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                                  const OverlapBuffers& ob, cudaStream_t st) {
  const int nz = s.dims[2];
  cudaError_t e = launch_range(s, range_args(s, ws, u, w, constrained, ob, 0, 0, 1, nullptr, carry_plane(s, ob, 0)),
                               st);
  if (e) return e;
  return launch_range(s, range_args(s, ws, u, w, constrained, ob, 1, nz - 1, nz, carry_plane(s, ob, 1), nullptr),
                      st);
}

cudaError_t launch_apply_interior(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                                  const OverlapBuffers& ob, cudaStream_t st) {
  const int nz = s.dims[2];
  if (nz < 3) return cudaMemsetAsync(ob.slots + 2, 0, sizeof(double), st);
  return launch_range(
      s, range_args(s, ws, u, w, constrained, ob, 2, 1, nz - 1, carry_plane(s, ob, 2), carry_plane(s, ob, 3)), st);
}

cudaError_t launch_carry_combine(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                                 const OverlapBuffers& ob, double* out, cudaStream_t st) {
  const int nz = s.dims[2];
  CombineArgs c{};
  c.a = make_apply_args(s, ws, u, w, constrained, nullptr, nullptr);
  if (nz == 2) {  // one inner plane: element 1's bottom + element 0's top
    c.nplanes = 1;
    c.Z[0] = s.p;
    c.lo[0] = carry_plane(s, ob, 1);
    c.hi[0] = carry_plane(s, ob, 0);
  } else {
    c.nplanes = 2;
    c.Z[0] = s.p;
    c.lo[0] = carry_plane(s, ob, 2);
    c.hi[0] = carry_plane(s, ob, 0);
    c.Z[1] = (nz - 1) * s.p;
    c.lo[1] = carry_plane(s, ob, 1);
    c.hi[1] = carry_plane(s, ob, 3);
  }
  c.partials = ob.partials;
  c.ticket = ob.tickets + 3;
  c.slots = ob.slots;
  c.nslots = 3;
  c.nodal_dot = !(use_mma(s) && mma5_kernel_applies(s));  // the BP5 DMMA kernel's p.Ap is the energy form
  c.out = out;
  const long long nodes = static_cast<long long>(c.nplanes) * s.dims[0] * s.dims[1] * (s.p + 1) * (s.p + 1);
  long long blocks = (nodes + CT - 1) / CT;
  if (blocks > kMaxCombineBlocks) blocks = kMaxCombineBlocks;
  switch (s.p) {
#define HXB_CC(PP) \
  case PP: carry_combine_kernel<PP><<<static_cast<int>(blocks), CT, 0, st>>>(c); break;
    HXB_CC(1) HXB_CC(2) HXB_CC(3) HXB_CC(4) HXB_CC(5) HXB_CC(6) HXB_CC(7) HXB_CC(8)
#undef HXB_CC
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int overlap_partials_capacity() { return kMaxCombineBlocks; }

}  // namespace hxb
