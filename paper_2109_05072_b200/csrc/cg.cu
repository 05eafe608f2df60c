// Device-resident conjugate-gradient recurrence (solver.hpp:91-153, no
// preconditioner, z = r).
//
// Two reduction modes (hexbp_cg_set_mode):
//  EXACT (default): every inner product follows deterministic_dot
//    (dense.hpp:52-81) bit for bit -- 4096-entry blocks summed sequentially
//    with separate multiply and add (no FMA, like the reference's default
//    x86-64 build), block partials summed sequentially in block order -- and
//    the vector updates use the reference's unfused arithmetic
//    (solver.hpp:103,132-133,147). Given the same operator outputs the device
//    recurrence is the reference recurrence; the only deviation left is the
//    operator apply itself (<= 3e-16 per entry). Per iteration:
//      apply(p)           -> Ap                         2n doubles + factors
//      cg_pap             -> p.Ap, alpha                2n
//      cg_update_r        -> r -= alpha Ap, r.r, beta   3n
//      cg_update_xp       -> x += alpha p, p = r + beta p   5n
//  FUSED: p.Ap is produced by the operator kernel (column partials + lateral
//    fix-up partials) and the updates use FMA with fixed-order tree
//    reductions: 10n per iteration. Bitwise reproducible run to run, not
//    bitwise equal to the reference's sums.
// In both modes the last CTA of each reduction applies the reference's
// stopping rule and error semantics on the device, so no host round trip is
// needed per iteration.
#include <cuda_runtime.h>

#include <cstdlib>

#include "device_util.cuh"
#include "internal.h"
#include "ring.cuh"

namespace hxb {
namespace {

constexpr int VT = 256;
constexpr int CHUNK = 4096;          // detail::kReductionBlock (dense.hpp:52)
constexpr int RVT = 128;             // blocked_reduce_kernel: threads per CTA
constexpr int RT = 32;               // entries per chunk per tile (one coalesced 256-byte row)
constexpr int CPW = 16;              // chunks per warp (more warps, more loads in flight)

#define DM(a, b) __dmul_rn((a), (b))
#define DA(a, b) __dadd_rn((a), (b))
#define DS(a, b) __dsub_rn((a), (b))
#define DD(a, b) __ddiv_rn((a), (b))

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

// Sequential sum of the chunk partials in chunk order (dense.hpp:70-71), by
// one thread; loads are batched ahead of the dependent add chain.
__device__ __forceinline__ double serial_sum(const double* part, long long n) {
  double s = 0.0;
  long long c = 0;
  for (; c + 8 <= n; c += 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcg(part + c + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) s = DA(s, v[k]);
  }
  for (; c < n; ++c) s = DA(s, __ldcg(part + c));
  return s;
}

// The same sequential chunk-order sum by thread 0 of the (last) CTA, fed
// from shared memory: the CTA stages the partials in double-buffered tiles
// (coalesced loads by every thread) while thread 0 runs the dependent add
// chain over the previous tile -- L2 latency off the chain. `buf`: >= 2 * RSB doubles.
constexpr int RSB = 1024;
__device__ double block_serial_sum(const double* part, long long n, double* buf) {
  double s = 0.0;
  const long long ntiles = (n + RSB - 1) / RSB;
  auto stage = [&](long long t) {
    double* dst = buf + (t & 1) * RSB;
    for (int i = threadIdx.x; i < RSB; i += blockDim.x) {
      const long long g = t * RSB + i;
      dst[i] = g < n ? __ldcg(part + g) : 0.0;
    }
  };
  if (ntiles > 0) stage(0);
  __syncthreads();
  for (long long t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) stage(t + 1);
    if (threadIdx.x == 0) {
      const double* src = buf + (t & 1) * RSB;
      const int m = static_cast<int>(n - t * RSB < RSB ? n - t * RSB : RSB);
#pragma unroll 16
      for (int i = 0; i < m; ++i) s = DA(s, src[i]);
    }
    __syncthreads();
  }
  return s;
}

enum Op : int { OP_DOT = 0, OP_PAP = 1, OP_INIT = 2, OP_UPDATE_R = 3, OP_RZ = 4 };

// Blocked exact reduction with an optional fused elementwise update.
//   OP_DOT      : dot(a, b)                                   -> *out
//   OP_PAP      : dot(p=a, Ap=b); alpha = rz / pAp            (solver.hpp:128-131)
//   OP_INIT     : r = b - Ap (a=b_rhs, b=Ap, w0=r, w1=p); p = r; r.r; r0  (solver.hpp:102-124)
//   OP_UPDATE_R : r = r - alpha Ap (a=r, b=Ap, w0=r); r.r; rnorm, stop, beta (solver.hpp:133-147)
//   OP_RZ       : r.z with z = r / diag (a=r, b=diag) -> rz (init) or beta, rz (solver.hpp:108,145-147)
// With a Jacobi diagonal `dv`, OP_INIT stores p = z = r / diag.
__device__ void scalar_logic(int op, double tot, DevScalars* sc, double* hist, double rel_tol, int max_iter);

// Products / fused updates of one element (reference arithmetic, unfused).
template <int OP>
__device__ __forceinline__ double elem_op(double x, double y, long long g, double alpha, double* w0, double* w1,
                                          const double* dv) {
  if (OP == OP_DOT || OP == OP_PAP) return DM(x, y);
  if (OP == OP_RZ) return DM(x, DD(x, y));  // r * (r / diag)
  if (OP == OP_INIT) {
    const double r = DS(x, y);  // r = b - Ap (solver.hpp:103)
    w0[g] = r;
    w1[g] = dv ? DD(r, dv[g]) : r;  // z = r / diag (or r); p = z (solver.hpp:105-109,123)
    return DM(r, r);
  }
  const double r = DS(x, DM(alpha, y));  // r -= alpha * Ap (solver.hpp:133)
  w0[g] = r;
  return DM(r, r);
}

// Blocked exact reduction (deterministic_dot's order: every 4096-entry chunk
// summed sequentially from 0.0, chunk partials summed in chunk order by the
// last CTA, dense.hpp:52-81) with an optional fused elementwise update.
// A warp owns 32 consecutive chunks; lane c sums chunk c. Per tile of RT
// entries the warp loads each of its chunks' RT-entry segments coalesced (one
// 256-byte row per load), computes the products / fused updates there (the
// updated vectors are written coalesced) and transposes the products through
// a per-warp shared tile; lane c then adds its row in order while the next
// tile's loads are in flight. No CTA barrier: warps run independently.
// `owned` >= 0: elementwise updates run over [0, n) but only entries
// [owned, n) enter the sum (multi-GPU slabs: the bottom interface plane is
// owned by the rank below); the rank partial is written to *out (dist mode).
template <int OP>
__global__ void __launch_bounds__(RVT) blocked_reduce_kernel(const double* a, const double* b, double* w0,
                                                             double* w1, long long n, double* part,
                                                             unsigned int* done, DevScalars* sc, double* hist,
                                                             double* out, double rel_tol, int max_iter,
                                                             long long owned = -1, const double* dv = nullptr) {
  __shared__ double tile[RVT / 32][CPW * (RT + 1)];  // also the staging buffer of the final sum
  static_assert(RVT / 32 * CPW * (RT + 1) >= 2 * RSB, "block_serial_sum buffer");
  const bool dist = owned >= 0;
  const long long lo = dist ? owned : 0;
  if (OP == OP_PAP || OP == OP_UPDATE_R || OP == OP_RZ) {
    if (*(volatile int*)&sc->status != ST_RUNNING) return;
  }
  const double alpha = OP == OP_UPDATE_R ? sc->alpha : 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* T = tile[warp];
  const long long nchunks = (n + CHUNK - 1) / CHUNK;
  const long long c0 = (static_cast<long long>(blockIdx.x) * (RVT / 32) + warp) * CPW;  // first chunk of the warp
  double s = 0.0;
  if (c0 < nchunks) {
    double xa[CPW], xb[CPW];
    auto load = [&](int t) {  // row c: entries [t*RT, t*RT + RT) of chunk c0 + c, lane = entry (RT = 32)
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const long long g = (c0 + c) * CHUNK + static_cast<long long>(t) * RT + lane;
        xa[c] = g < n ? __ldcs(a + g) : 0.0;
        xb[c] = g < n ? __ldcs(b + g) : 1.0;
      }
    };
    load(0);
    for (int t = 0; t < CHUNK / RT; ++t) {
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const long long g = (c0 + c) * CHUNK + static_cast<long long>(t) * RT + lane;
        double pr = 0.0;
        if (g < n) {
          pr = elem_op<OP>(xa[c], xb[c], g, alpha, w0, w1, dv);
          if (g < lo) pr = 0.0;  // not owned by this rank
        }
        T[c * (RT + 1) + lane] = pr;
      }
      if (t + 1 < CHUNK / RT) load(t + 1);  // in flight during the add chain below
      __syncwarp();
      if (lane < CPW) {
        const double* row = T + lane * (RT + 1);
        const long long cend = (c0 + lane) * CHUNK + static_cast<long long>(t) * RT;
#pragma unroll 8
        for (int e = 0; e < RT; ++e) {
          if (cend + e < n) s = DA(s, row[e]);  // exactly the chunk's entries, in order
        }
      }
      __syncwarp();
    }
    if (lane < CPW && c0 + lane < nchunks) {
      part[c0 + lane] = s;
      __threadfence();
    }
  }
  if (!last_block(done)) return;
  __threadfence();
  const double tot = block_serial_sum(part, nchunks, &tile[0][0]);
  if (threadIdx.x != 0) return;
  *done = 0;
  if (OP == OP_DOT || dist) {
    *out = tot;  // distributed CG: the rank partial, combined by cgd_finish_kernel
  } else {
    scalar_logic(OP, tot, sc, hist, rel_tol, max_iter);
  }
}

// The reference's scalar recurrence for one reduced quantity (solver.hpp:102-147).
__device__ void scalar_logic(int op, double tot, DevScalars* sc, double* hist, double rel_tol, int max_iter) {
  if (op == OP_PAP) {
    if (!isfinite(tot) || tot <= 0.0) {
      sc->status = ST_DIVERGED;
    } else {
      sc->pAp = tot;
      sc->alpha = sc->rz / tot;
    }
  } else if (op == OP_RZ) {
    if (sc->iterations == 0) {
      sc->rz = tot;  // rz = r0.z0 (solver.hpp:124)
    } else {
      sc->beta = tot / sc->rz;  // solver.hpp:145-147
      sc->rz = tot;
    }
  } else if (op == OP_INIT) {
    const double r0 = sqrt(tot);
    hist[0] = r0;
    sc->r0 = r0;
    sc->rnorm = r0;
    sc->rz = tot;  // deterministic_dot(r, z) with z = r: the same sum
    sc->rel_tol = rel_tol;
    sc->max_iter = max_iter;
    sc->iterations = 0;
    sc->x_pending = 0;
    sc->status = !isfinite(r0) ? ST_DIVERGED : (r0 == 0.0 ? ST_CONVERGED : (max_iter <= 0 ? ST_MAXITER : ST_RUNNING));
  } else {
    const double rnorm = sqrt(tot);
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
      if (!sc->precond) {  // Jacobi: beta from OP_RZ
        sc->beta = tot / sc->rz;
        sc->rz = tot;
      }
      if (k >= sc->max_iter) sc->status = ST_MAXITER;
    }
  }
}

// x += alpha p; p = z + beta p, z = r / diag or r (solver.hpp:105-108,132,147).
template <bool EXACT, bool PC>
__global__ void __launch_bounds__(VT) cg_update_xp_kernel(double* __restrict__ x, double* __restrict__ p,
                                                          const double* __restrict__ r, long long n,
                                                          unsigned int* done, DevScalars* sc,
                                                          const double* __restrict__ dv) {
  if (*(volatile int*)&sc->x_pending == 0) return;
  const double alpha = sc->alpha, beta = sc->beta;
  const bool update_p = *(volatile int*)&sc->status == ST_RUNNING;
  const long long stride = static_cast<long long>(gridDim.x) * VT;
  long long i = blockIdx.x * static_cast<long long>(VT) + threadIdx.x;
  // 4 independent coalesced streams per thread in flight (memory-level parallelism)
  for (; i + 3 * stride < n; i += 4 * stride) {
    double pv[4], xv[4], rv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      pv[u] = p[i + u * stride];
      xv[u] = x[i + u * stride];
      rv[u] = update_p ? r[i + u * stride] : 0.0;
      if (PC && update_p) rv[u] = EXACT ? DD(rv[u], dv[i + u * stride]) : rv[u] / dv[i + u * stride];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (EXACT) {
        x[i + u * stride] = DA(xv[u], DM(alpha, pv[u]));
        if (update_p) p[i + u * stride] = DA(rv[u], DM(beta, pv[u]));
      } else {
        x[i + u * stride] = fma(alpha, pv[u], xv[u]);
        if (update_p) p[i + u * stride] = fma(beta, pv[u], rv[u]);
      }
    }
  }
  for (; i < n; i += stride) {
    const double pi = p[i];
    const double zi = update_p ? (PC ? (EXACT ? DD(r[i], dv[i]) : r[i] / dv[i]) : r[i]) : 0.0;
    if (EXACT) {
      x[i] = DA(x[i], DM(alpha, pi));
      if (update_p) p[i] = DA(zi, DM(beta, pi));
    } else {
      x[i] = fma(alpha, pi, x[i]);
      if (update_p) p[i] = fma(beta, pi, zi);
    }
  }
  if (!last_block(done)) return;
  if (threadIdx.x == 0) {
    sc->x_pending = 0;
    *done = 0;
  }
}

// ---- FUSED mode: FMA updates and fixed-order tree reductions.
__device__ __forceinline__ double tree_partials(const double* part, int nblk, double* red) {
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += VT) s += __ldcg(part + b);
  return block_sum<VT>(s, red);
}

__global__ void __launch_bounds__(VT) fused_init_kernel(const double* __restrict__ b, const double* __restrict__ Ap,
                                                        double* __restrict__ r, double* __restrict__ p, long long n,
                                                        double* part, unsigned int* done, DevScalars* sc,
                                                        double* hist, double rel_tol, int max_iter,
                                                        const double* __restrict__ dv) {
  __shared__ double red[VT / 32];
  double acc = 0.0, acz = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * VT;
  for (long long i = blockIdx.x * static_cast<long long>(VT) + threadIdx.x; i < n; i += stride) {
    const double v = b[i] - Ap[i];
    r[i] = v;
    const double z = dv ? v / dv[i] : v;
    p[i] = z;
    acc = fma(v, v, acc);
    acz = fma(v, z, acz);
  }
  const double s = block_sum<VT>(acc, red);
  const double sz = dv ? block_sum<VT>(acz, red) : 0.0;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    part[gridDim.x + blockIdx.x] = sz;
  }
  if (!last_block(done)) return;
  __threadfence();
  const double rr = tree_partials(part, gridDim.x, red);
  const double rz = dv ? tree_partials(part + gridDim.x, gridDim.x, red) : rr;
  if (threadIdx.x == 0) {
    const double r0 = sqrt(rr);
    hist[0] = r0;
    sc->r0 = r0;
    sc->rnorm = r0;
    sc->rz = rz;
    sc->rel_tol = rel_tol;
    sc->max_iter = max_iter;
    sc->iterations = 0;
    sc->x_pending = 0;
    sc->status = !isfinite(r0) ? ST_DIVERGED : (r0 == 0.0 ? ST_CONVERGED : (max_iter <= 0 ? ST_MAXITER : ST_RUNNING));
    *done = 0;
  }
}

// FUSED mode, r = r - alpha A p with A p's ring nodes still as column
// partials (launch_apply(..., finish_ring = false)): every ring node sums its
// 1-4 partials in ascending column order (ring.cuh; the values equal the ones
// lateral_fixup_kernel would store, bit for bit) where A p is consumed, so the
// ring never makes a round trip through HBM as A p. One warp per node row
// (Y, Z); four row segments of 32 nodes in flight per warp.
struct RingUpdateArgs {
  const double* Ap;       // final on interior nodes
  const double* p;        // the applied vector (ConstrainedOperator rows: A p = p)
  const double* latY;     // ring partials (ring.cuh layout)
  const double* latX;
  const double* dv;       // Jacobi diagonal (nullptr: plain CG)
  const double* b;        // INIT: right-hand side (r = b - A x)
  double* pout;           // INIT: p = z
  double rel_tol;         // INIT: stopping rule parameters
  int max_iter;
  double* r;
  int nx, ny, Nx, Ny, Nz, constrained, bc_zlo, bc_zhi;
  // z-slab partition: node planes Z = 0 / Nz-1 shared with the rank below /
  // above hold the assembled (halo-summed) A p in Ap; plane 0 belongs to the
  // rank below (not in this rank's r.r). rank_partial != nullptr: the last
  // block stores this rank's r.r there instead of running the scalar step.
  int zlo_asm, zhi_asm;
  double* rank_partial;
  int p_pitch, pout_pitch;  // row pitches of p and pout (Workspace::pt: Nx rounded up to even)
  int v_pitch;              // row pitch of r and Ap (Workspace::rt / Apt in the pitched fast CG)
};

// INIT = true: the initial residual r = b - A x (x applied in CG form), p = z,
// r.r -> r0 and the stopping state, r.z -> rz (solver.hpp:102-124).
#ifndef HX_RING_MINB
#define HX_RING_MINB 4  // 64 registers, no spill: the 16-byte plain-row path keeps 4 pairs in flight
#endif
#ifndef HX_RING_U
#define HX_RING_U 2
#endif
constexpr int RU = HX_RING_U;  // plain-row chunks of 32 nodes in flight per warp
template <int P, bool INIT, bool PC>
__global__ void __launch_bounds__(VT, HX_RING_MINB) fused_ring_update_r_kernel(const __grid_constant__ RingUpdateArgs R, double* part,
                                                                 unsigned int* done, DevScalars* sc, double* hist) {
  __shared__ double red[VT / 32];
  if (!INIT && *(volatile int*)&sc->status != ST_RUNNING) return;
  const double alpha = INIT ? 0.0 : sc->alpha;
  const int lane = threadIdx.x & 31;
  const int rows = R.Ny * R.Nz;  // < 2^31 (n_L < 2^31 checked at setup)
  const LatLayout L(P, R.nx, R.ny);
  double acc = 0.0, acz = 0.0;  // r.r and, with a Jacobi diagonal, r.z
  const int lmod = lane % P;
  for (int row = blockIdx.x * (VT / 32) + (threadIdx.x >> 5); row < rows; row += gridDim.x * (VT / 32)) {
    const int Z = row / R.Ny, Y = row - Z * R.Ny;
    const bool bcrow = R.constrained && (Y == 0 || Y == R.Ny - 1 || (Z == 0 && R.bc_zlo) || (Z == R.Nz - 1 && R.bc_zhi));
    double* rr_ = R.r + static_cast<long long>(R.v_pitch) * row;
    const double* ap = R.Ap + static_cast<long long>(R.v_pitch) * row;
    const double* pp = R.p + static_cast<long long>(R.p_pitch) * row;
    const double* dd = PC ? R.dv + static_cast<long long>(R.Nx) * row : nullptr;
    const double* bb = INIT ? R.b + static_cast<long long>(R.Nx) * row : nullptr;
    double* po = INIT ? R.pout + static_cast<long long>(R.pout_pitch) * row : nullptr;
    if ((Z == 0 && R.zlo_asm) || (Z == R.Nz - 1 && R.zhi_asm)) {
      // shared node plane, already assembled in Ap (constrained nodes: A p = p)
      const bool owned = !(Z == 0 && R.zlo_asm);
      for (int X = lane; X < R.Nx; X += 32) {
        const double a = ap[X];
        const double v = INIT ? bb[X] - a : fma(-alpha, a, rr_[X]);
        rr_[X] = v;
        const double z = PC ? v / dd[X] : v;
        if (owned) {
          acc = fma(v, v, acc);
          if (PC) acz = fma(v, z, acz);
        }
        if (INIT) po[X] = z;
      }
    } else if (Y % P != 0) {
      // plain row: interior nodes read A p; x-face nodes X = fx*P sum the
      // (left, right) partial pair of latX (one 16-byte load)
      const double* xr = R.latX + L.x_index(R.nx, Z, Y, 0, 0);
      if constexpr (!INIT && !PC) {
        // the CG iteration's form with 16-byte accesses: node pairs (X, X+1)
        // at even global index, the odd element at the row start / end alone
        const int head = static_cast<int>((static_cast<long long>(R.v_pitch) * row) & 1);
        auto lat_at = [&](int X) { return __ldcg(reinterpret_cast<const double2*>(xr) + X / P); };
        auto node_a = [&](int X, double a_loaded, double2 lr) -> double {  // A p at node X of the row
          if (X % P != 0) return a_loaded;
          if (R.constrained && (bcrow || X == 0 || X == R.Nx - 1)) return pp[X];  // A p = p
          const int fx = X / P;
          double sum = 0.0;  // ascending column order (ring_node_sum)
          if (fx > 0) sum += lr.x;
          if (fx < R.nx) sum += lr.y;
          return sum;
        };
        auto single = [&](int X) {
          const bool xf = X % P == 0;
          const double rv = rr_[X];
          const double a = node_a(X, xf ? 0.0 : ap[X], xf ? lat_at(X) : make_double2(0.0, 0.0));
          const double v = fma(-alpha, a, rv);
          rr_[X] = v;
          acc = fma(v, v, acc);
        };
        if (head && lane == 0) single(0);
        const int npair = (R.Nx - head) / 2;
        for (int k0 = 0; k0 < npair; k0 += RU * 32) {
          double2 rv[RU], av[RU], l0[RU], l1[RU];
#pragma unroll
          for (int u = 0; u < RU; ++u) {  // every load of the chunk before the first use
            const int k = k0 + 32 * u + lane;
            const bool ok = k < npair;
            const int X = head + 2 * k;
            const bool f0 = ok && X % P == 0, f1 = ok && (X + 1) % P == 0;
            rv[u] = ok ? *reinterpret_cast<const double2*>(rr_ + X) : make_double2(0.0, 0.0);
            av[u] = ok ? *reinterpret_cast<const double2*>(ap + X) : make_double2(0.0, 0.0);
            l0[u] = f0 ? lat_at(X) : make_double2(0.0, 0.0);
            l1[u] = f1 ? lat_at(X + 1) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < RU; ++u) {
            const int k = k0 + 32 * u + lane;
            if (k < npair) {
              const int X = head + 2 * k;
              const double a0 = node_a(X, av[u].x, l0[u]), a1 = node_a(X + 1, av[u].y, l1[u]);
              const double2 v = make_double2(fma(-alpha, a0, rv[u].x), fma(-alpha, a1, rv[u].y));
              *reinterpret_cast<double2*>(rr_ + X) = v;
              acc = fma(v.x, v.x, acc);
              acc = fma(v.y, v.y, acc);
            }
          }
        }
        const int tail = head + 2 * npair;
        if (tail < R.Nx && lane == 0) single(tail);
      } else
      for (int x0 = 0; x0 < R.Nx; x0 += RU * 32) {
        // every load of the chunk is issued before the first use
        double av[RU], rv[RU];
        double2 lr[RU];
        bool xf[RU];
        int xm = (x0 % P + lmod) % P;  // X % P for u = 0
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int X = x0 + 32 * u + lane;
          const bool ok = X < R.Nx;
          xf[u] = ok && xm == 0;
          rv[u] = ok ? rr_[X] : 0.0;
          av[u] = ok && !xf[u] ? ap[X] : 0.0;
          lr[u] = xf[u] ? __ldcg(reinterpret_cast<const double2*>(xr) + X / P) : make_double2(0.0, 0.0);
          xm += 32 % P;
          if (xm >= P) xm -= P;
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int X = x0 + 32 * u + lane;
          if (X < R.Nx) {
            double a = av[u];
            if (xf[u]) {
              if (R.constrained && (bcrow || X == 0 || X == R.Nx - 1)) {
                a = pp[X];  // ConstrainedOperator row: A p = p
              } else {
                const int fx = X / P;
                double sum = 0.0;  // ascending column order (ring_node_sum)
                if (fx > 0) sum += lr[u].x;
                if (fx < R.nx) sum += lr[u].y;
                a = sum;
              }
            }
            const double v = INIT ? bb[X] - a : fma(-alpha, a, rv[u]);
            rr_[X] = v;
            acc = fma(v, v, acc);
            const double z = PC ? v / dd[X] : v;
            if (PC) acz = fma(v, z, acz);
            if (INIT) po[X] = z;
          }
        }
      }
    } else {
      // ring row Y = fy*P: every node sums the latY partials of the columns
      // below / above (and both x-columns at a corner), ascending column order
      const int fy = Y / P;
      const bool below = fy > 0, above = fy < R.ny;
      const double* yb = R.latY + L.y_index(P, R.nx, Z, fy, 0, 0, 0);  // side 0 (column below)
      const double* ya = yb + static_cast<long long>(R.nx) * (P + 1);   // side 1 (column above)
      for (int x0 = 0; x0 < R.Nx; x0 += 2 * 32) {
        double rv[2], q[2][4];
        bool lo[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {  // loads first
          const int X = x0 + 32 * u + lane;
          const bool ok = X < R.Nx;
          const int cxh = X / P < R.nx ? X / P : R.nx - 1;
          const int o = cxh * (P + 1) + (X - cxh * P);  // (cxh, ih) in a side's [cx][i] block
          lo[u] = X % P == 0 && X > 0 && X / P < R.nx;  // interior corner: (cxh-1, P) at o - 1
          rv[u] = ok ? rr_[X] : 0.0;
          q[u][0] = ok && below && lo[u] ? __ldcg(yb + o - 1) : 0.0;
          q[u][1] = ok && below ? __ldcg(yb + o) : 0.0;
          q[u][2] = ok && above && lo[u] ? __ldcg(ya + o - 1) : 0.0;
          q[u][3] = ok && above ? __ldcg(ya + o) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int X = x0 + 32 * u + lane;
          if (X < R.Nx) {
            double a;
            if (R.constrained && (bcrow || X == 0 || X == R.Nx - 1)) {
              a = pp[X];  // ConstrainedOperator row: A p = p
            } else {
              double sum = 0.0;  // ascending column order (ring_node_sum)
              if (below && lo[u]) sum += q[u][0];
              if (below) sum += q[u][1];
              if (above && lo[u]) sum += q[u][2];
              if (above) sum += q[u][3];
              a = sum;
            }
            const double v = INIT ? bb[X] - a : fma(-alpha, a, rv[u]);
            rr_[X] = v;
            acc = fma(v, v, acc);
            const double z = PC ? v / dd[X] : v;
            if (PC) acz = fma(v, z, acz);
            if (INIT) po[X] = z;
          }
        }
      }
    }
  }
  const double s = block_sum<VT>(acc, red);
  const double sz = PC ? block_sum<VT>(acz, red) : 0.0;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    if (PC) part[gridDim.x + blockIdx.x] = sz;
  }
  if (!last_block(done)) return;
  __threadfence();
  const double rr = tree_partials(part, gridDim.x, red);
  const double rz = PC ? tree_partials(part + gridDim.x, gridDim.x, red) : rr;
  if (R.rank_partial) {  // z-slab CG: the ranks' partials are combined by cgd_finish_kernel
    if (threadIdx.x == 0) {
      *R.rank_partial = rr;
      *done = 0;
    }
    return;
  }
  if (INIT) {
    if (threadIdx.x == 0) {
      const double r0 = sqrt(rr);
      hist[0] = r0;
      sc->r0 = r0;
      sc->rnorm = r0;
      sc->rz = rz;
      sc->rel_tol = R.rel_tol;
      sc->max_iter = R.max_iter;
      sc->iterations = 0;
      sc->x_pending = 0;
      sc->status = !isfinite(r0) ? ST_DIVERGED
                                 : (r0 == 0.0 ? ST_CONVERGED : (R.max_iter <= 0 ? ST_MAXITER : ST_RUNNING));
      *done = 0;
    }
    return;
  }
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
      sc->beta = rz / sc->rz;  // solver.hpp:145-147 (rz = r.r without a preconditioner)
      sc->rz = rz;
      if (k >= sc->max_iter) sc->status = ST_MAXITER;
    }
    *done = 0;
  }
}

int chunk_grid(int64_t n) {
  const long long nch = (n + CHUNK - 1) / CHUNK;
  const long long per_cta = RVT / 32 * CPW;
  return static_cast<int>((nch + per_cta - 1) / per_cta);
}

// Multi-GPU: sum the all-gathered rank partials in rank order (identical on
// every rank) and apply the scalar recurrence.
__global__ void cgd_finish_kernel(int op, const double* gathered, int world, DevScalars* sc, double* hist,
                                  double rel_tol, int max_iter) {
  if (op != OP_INIT && *(volatile int*)&sc->status != ST_RUNNING) return;
  double tot = 0.0;
  for (int r = 0; r < world; ++r) tot = DA(tot, gathered[r]);
  scalar_logic(op, tot, sc, hist, rel_tol, max_iter);
}

// Interface-plane halo sum of the z-slab partition: dst = dst + src (IEEE
// addition commutes, so the two ranks sharing the plane obtain identical
// sums); with ConstrainedOperator semantics the plane's box-boundary nodes
// keep w = u (both ranks already hold u there).
__global__ void plane_combine_kernel(double* dst, const double* src, const double* u, int nxn, int nyn,
                                     int constrained) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nxn * nyn) return;
  const int X = i % nxn, Y = i / nxn;
  if (constrained && (X == 0 || X == nxn - 1 || Y == 0 || Y == nyn - 1))
    dst[i] = u[i];
  else
    dst[i] = dst[i] + src[i];
}

}  // namespace

cudaError_t launch_cgd_reduce(const Workspace& ws, int op, const double* b, int64_t n, int64_t owned,
                              double* out, cudaStream_t st) {
  const int grid = chunk_grid(n);
  if (op == 0)
    blocked_reduce_kernel<OP_INIT><<<grid, RVT, 0, st>>>(b, ws.Ap, ws.r, ws.p, n, ws.vec_partials, ws.vec_done, ws.sc,
                                                       ws.history, out, 0.0, 0, owned);
  else if (op == 1)
    blocked_reduce_kernel<OP_PAP><<<grid, RVT, 0, st>>>(ws.p, ws.Ap, nullptr, nullptr, n, ws.vec_partials, ws.vec_done,
                                                      ws.sc, ws.history, out, 0.0, 0, owned);
  else
    blocked_reduce_kernel<OP_UPDATE_R><<<grid, RVT, 0, st>>>(ws.r, ws.Ap, ws.r, nullptr, n, ws.vec_partials,
                                                           ws.vec_done, ws.sc, ws.history, out, 0.0, 0, owned);
  return cudaGetLastError();
}

cudaError_t launch_cgd_finish(const Workspace& ws, int op, const double* gathered, int world, double rel_tol,
                              int max_iter, cudaStream_t st) {
  const int opk = op == 0 ? OP_INIT : (op == 1 ? OP_PAP : OP_UPDATE_R);
  cgd_finish_kernel<<<1, 1, 0, st>>>(opk, gathered, world, ws.sc, ws.history, rel_tol, max_iter);
  return cudaGetLastError();
}

cudaError_t launch_plane_combine(double* dst, const double* src, const double* u, int nxn, int nyn, int constrained,
                                 cudaStream_t st) {
  const int n = nxn * nyn;
  plane_combine_kernel<<<(n + 255) / 256, 256, 0, st>>>(dst, src, u, nxn, nyn, constrained);
  return cudaGetLastError();
}

int vec_grid(int64_t n) {
  // Fixed function of n (never of timing): at most 148 SMs x 8 blocks.
  long long g = (n + VT - 1) / VT;
  if (g > 148 * 8) g = 148 * 8;
  return static_cast<int>(g < 1 ? 1 : g);
}

// Exactly one full wave of a grid-stride kernel (the ring r-update: 10% faster
// than the 1.6 waves of vec_grid at 48 registers; the plain streaming kernels
// measured best with vec_grid): resident CTAs per SM (from
// its register / shared-memory footprint) x SMs, capped by vec_grid. A fixed
// function of (kernel, device, n), so reductions stay run-to-run identical.
template <typename K>
int wave_grid(K kernel, int64_t n) {
  // cache per (kernel, device); kernels of one signature share the type K
  struct Entry {
    const void* fn;
    int dev, cap;
  };
  static Entry cache[64];
  static int used = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const void* fn = reinterpret_cast<const void*>(kernel);
  int cap = 0;
  for (int i = 0; i < used; ++i)
    if (cache[i].fn == fn && cache[i].dev == dev) cap = cache[i].cap;
  if (cap == 0) {
    int sms = 148, bps = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, VT, 0);
    cap = (bps > 0 ? bps : 8) * sms;
    if (cap > 148 * 8) cap = 148 * 8;  // vec_partials capacity (reduction_partials)
    if (used < 64) cache[used++] = {fn, dev, cap};
  }
  const int g = vec_grid(n);
  return g < cap ? g : cap;
}

int64_t dot_capacity(int64_t nL) { return reduction_partials(nL) * CHUNK; }

int64_t reduction_partials(int64_t n) {
  // exact-mode chunk partials, or two partials per CTA of the fused kernels
  const int64_t nch = (n + CHUNK - 1) / CHUNK;
  return nch > 2 * 148 * 8 ? nch : 2 * 148 * 8;
}

cudaError_t launch_cg_init(const Workspace& ws, const double* b, int64_t n, double rel_tol, int max_iter,
                           cudaStream_t st) {
  if (ws.exact) {
    blocked_reduce_kernel<OP_INIT><<<chunk_grid(n), RVT, 0, st>>>(b, ws.Ap, ws.r, ws.p, n, ws.vec_partials,
                                                                 ws.vec_done, ws.sc, ws.history, nullptr, rel_tol,
                                                                 max_iter, -1, ws.diag);
  } else {
    fused_init_kernel<<<vec_grid(n), VT, 0, st>>>(b, ws.Ap, ws.r, ws.p, n, ws.vec_partials, ws.vec_done, ws.sc,
                                                  ws.history, rel_tol, max_iter, ws.diag);
  }
  return cudaGetLastError();
}

cudaError_t launch_cg_pap(const Workspace& ws, int64_t n, cudaStream_t st) {
  blocked_reduce_kernel<OP_PAP><<<chunk_grid(n), RVT, 0, st>>>(ws.p, ws.Ap, nullptr, nullptr, n, ws.vec_partials,
                                                              ws.vec_done, ws.sc, ws.history, nullptr, 0.0, 0);
  return cudaGetLastError();
}

cudaError_t launch_cg_rz(const Workspace& ws, int64_t n, cudaStream_t st) {
  blocked_reduce_kernel<OP_RZ><<<chunk_grid(n), RVT, 0, st>>>(ws.r, ws.diag, nullptr, nullptr, n, ws.vec_partials,
                                                             ws.vec_done, ws.sc, ws.history, nullptr, 0.0, 0);
  return cudaGetLastError();
}

namespace {
template <bool INIT>
cudaError_t launch_ring_r(const Workspace& ws, int64_t n, cudaStream_t st, int constrained, const double* p_applied,
                          const double* b, double rel_tol, int max_iter, int zlo_asm = 0, int zhi_asm = 0,
                          double* rank_partial = nullptr) {
  const Setup& s = *ws.s;
  RingUpdateArgs R;
  const int Nx = s.dims[0] * s.p + 1;
  // the pitched fast CG (Workspace::use_pt): r, Ap and p row-pitched
  R.Ap = ws.use_pt ? ws.Apt : ws.Ap;
  R.v_pitch = ws.use_pt ? ws.pt_pitch : Nx;
  R.p = p_applied;
  R.p_pitch = ws.pt != nullptr && p_applied == ws.pt ? ws.pt_pitch : Nx;
  R.latY = ws.lateral;
  R.latX = ws.lateral + LatLayout(s.p, s.dims[0], s.dims[1]).y_zstride * (s.dims[2] * s.p + 1);
  R.dv = ws.diag;
  R.b = b;
  R.pout = ws.use_pt ? ws.pt : ws.p;
  R.pout_pitch = ws.use_pt ? ws.pt_pitch : Nx;
  R.rel_tol = rel_tol;
  R.max_iter = max_iter;
  R.r = ws.use_pt ? ws.rt : ws.r;
  R.nx = s.dims[0];
  R.ny = s.dims[1];
  R.Nx = s.dims[0] * s.p + 1;
  R.Ny = s.dims[1] * s.p + 1;
  R.Nz = s.dims[2] * s.p + 1;
  R.constrained = constrained;
  R.bc_zlo = s.bc_zlo;
  R.bc_zhi = s.bc_zhi;
  R.zlo_asm = zlo_asm;
  R.zhi_asm = zhi_asm;
  R.rank_partial = rank_partial;
  switch (s.p) {
#define HXB_RING_CASE(PP)                                                                                             \
  case PP:                                                                                                             \
    if (R.dv)                                                                                                          \
      fused_ring_update_r_kernel<PP, INIT, true><<<wave_grid(fused_ring_update_r_kernel<PP, INIT, true>, n), VT, 0,     \
                                                   st>>>(R, ws.vec_partials, ws.vec_done, ws.sc, ws.history);          \
    else                                                                                                               \
      fused_ring_update_r_kernel<PP, INIT, false><<<wave_grid(fused_ring_update_r_kernel<PP, INIT, false>, n), VT, 0,   \
                                                    st>>>(R, ws.vec_partials, ws.vec_done, ws.sc, ws.history);         \
    break;
    HXB_RING_CASE(1)
    HXB_RING_CASE(2)
    HXB_RING_CASE(3)
    HXB_RING_CASE(4)
    HXB_RING_CASE(5)
    HXB_RING_CASE(6)
    HXB_RING_CASE(7)
    HXB_RING_CASE(8)
#undef HXB_RING_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_cg_update_r(const Workspace& ws, int64_t n, cudaStream_t st, int constrained) {
  if (ws.exact) {
    blocked_reduce_kernel<OP_UPDATE_R><<<chunk_grid(n), RVT, 0, st>>>(ws.r, ws.Ap, ws.r, nullptr, n, ws.vec_partials,
                                                                     ws.vec_done, ws.sc, ws.history, nullptr, 0.0, 0);
    return cudaGetLastError();
  }
  // fast mode: A p comes from launch_apply(..., finish_ring = false)
  return launch_ring_r<false>(ws, n, st, constrained, ws.use_pt ? ws.pt : ws.p, nullptr, 0.0, 0);
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

// Row copy between pitches (the pitched fast CG's x in / out, tma.cu): one
// warp per node row, four 32-node chunks loaded before they are stored
// (cudaMemcpy2DAsync ran at half the bandwidth on these 3.7 KB rows).
__global__ void __launch_bounds__(VT) copy_rows_kernel(double* __restrict__ dst, int dst_pitch,
                                                       const double* __restrict__ src, int src_pitch, int Nx, int rows) {
  const int lane = threadIdx.x & 31;
  for (int row = blockIdx.x * (VT / 32) + (threadIdx.x >> 5); row < rows; row += gridDim.x * (VT / 32)) {
    const double* s = src + static_cast<long long>(src_pitch) * row;
    double* d = dst + static_cast<long long>(dst_pitch) * row;
    for (int x0 = 0; x0 < Nx; x0 += 4 * 32) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int X = x0 + 32 * u + lane;
        v[u] = X < Nx ? s[X] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int X = x0 + 32 * u + lane;
        if (X < Nx) d[X] = v[u];
      }
    }
  }
}

cudaError_t launch_copy_rows(double* dst, int dst_pitch, const double* src, int src_pitch, int Nx, int64_t rows,
                             cudaStream_t st) {
  long long g = (rows + VT / 32 - 1) / (VT / 32);
  if (g > 148 * 16) g = 148 * 16;
  copy_rows_kernel<<<static_cast<int>(g < 1 ? 1 : g), VT, 0, st>>>(dst, dst_pitch, src, src_pitch, Nx,
                                                                   static_cast<int>(rows));
  return cudaGetLastError();
}

cudaError_t launch_set_int(int* p, int v, cudaStream_t st) {
  set_int_kernel<<<1, 1, 0, st>>>(p, v);
  return cudaGetLastError();
}

cudaError_t launch_cgd_update_r_fused(const Workspace& ws, int constrained, double* rank_partial, cudaStream_t st) {
  const Setup& s = *ws.s;
  const int has_down = s.z0 > 0, has_up = s.z0 + s.dims[2] < s.gdims[2];
  return launch_ring_r<false>(ws, s.nL, st, constrained, ws.p, nullptr, 0.0, 0, has_down, has_up, rank_partial);
}

cudaError_t launch_cg_init_ring(const Workspace& ws, const double* b, const double* x, int64_t n, double rel_tol,
                                int max_iter, int constrained, cudaStream_t st) {
  return launch_ring_r<true>(ws, n, st, constrained, x, b, rel_tol, max_iter);
}

cudaError_t launch_cg_update_xp(const Workspace& ws, double* x, int64_t n, cudaStream_t st, double* p) {
  if (!p) p = ws.use_pt ? ws.pt : ws.p;
  const int g = vec_grid(n);
  const int Nx = ws.s->dims[0] * ws.s->p + 1;
  if (ws.use_pt) {
    if (p != ws.pt || x != ws.xt) return cudaErrorInvalidValue;
    // pitched fast CG: x, p, r share the row pitch, so the flat update runs
    // over the pitched index space (the pad column is updated too, never read)
    const int64_t np = static_cast<int64_t>(ws.pt_pitch) * (n / Nx);
    const int gp = vec_grid(np);
    cg_update_xp_kernel<false, false><<<gp, VT, 0, st>>>(x, p, ws.rt, np, ws.vec_done, ws.sc, nullptr);
    return cudaGetLastError();
  }
  if (ws.exact) {
    if (ws.diag)
      cg_update_xp_kernel<true, true><<<g, VT, 0, st>>>(x, p, ws.r, n, ws.vec_done, ws.sc, ws.diag);
    else
      cg_update_xp_kernel<true, false><<<g, VT, 0, st>>>(x, p, ws.r, n, ws.vec_done, ws.sc, nullptr);
  } else {
    if (ws.diag)
      cg_update_xp_kernel<false, true><<<g, VT, 0, st>>>(x, p, ws.r, n, ws.vec_done, ws.sc, ws.diag);
    else
      cg_update_xp_kernel<false, false><<<g, VT, 0, st>>>(x, p, ws.r, n, ws.vec_done, ws.sc, nullptr);
  }
  return cudaGetLastError();
}

cudaError_t launch_dot(const Workspace& ws, const double* a, const double* b, int64_t n, double* out,
                       cudaStream_t st) {
  blocked_reduce_kernel<OP_DOT><<<chunk_grid(n), RVT, 0, st>>>(a, b, nullptr, nullptr, n, ws.vec_partials,
                                                              ws.vec_done, ws.sc, ws.history, out, 0.0, 0);
  return cudaGetLastError();
}

}  // namespace hxb
