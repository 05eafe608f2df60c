// Transpose restriction, part 2 (ring nodes), for the fast operator kernels.
//
// Part 1 (the element-column kernels) writes final values of the nodes
// strictly inside each column footprint and, for the 4p "ring" nodes shared
// with neighbouring columns, the column's partial sum into the lateral buffer
// lat[Z][col][4p]. A ring node's value is the sum of its 1-4 column partials
// in ascending column order (scatter_add's element order, restriction.hpp:
// 67-80), so it is bitwise reproducible.
//
// Who adds the partials:
//  * plain applies: lateral_fixup_kernel (apply.cu), one extra pass;
//  * CG: the r-update kernel (cg.cu) sums them where it needs A p -- no
//    extra pass over HBM, and A p is never materialised on the ring.
// p.Ap needs no ring sums: p.(A p) over the ring equals the sum over columns
// of p_n * (column partial)_n, so every column adds its own ring partials to
// its dot (constrained ring nodes, w = u, are counted once, by the node's
// owner column). The last CTA of the operator kernel sums the column partials
// in index order and applies alpha = rz / pAp (solver.hpp:127-131), so alpha
// is known when the operator kernel ends.
#pragma once
#include <cuda_runtime.h>

#include "device_util.cuh"
#include "internal.h"

namespace hxb {

// Does column (ex, ey) own its footprint node (i, j)? Owner = the column in
// which the node has local index < p (at the upper domain edge the last
// column keeps its far side).
__device__ __forceinline__ bool ring_owner(int P, int i, int j, int ex, int ey, int nx, int ny) {
  return (i != P || ex == nx - 1) && (j != P || ey == ny - 1);
}

// Lateral buffer layout (fast kernels), by node rows so that both the
// element-column producers and the row-streaming consumers are coalesced:
//   latY[Z][fy][side][cx][i], i = 0..P : ring rows Y = fy*P; side 0 = the
//       column below the row (cy = fy-1, local j = P), side 1 = the column
//       above (cy = fy, j = 0); each column stores its P+1 row nodes
//       (corners included), X = cx*P + i.
//   latX[Z][Y][fx][side] : x-face nodes X = fx*P on rows Y % P != 0; side 0 =
//       the column left of the face (cx = fx-1, i = P), side 1 = right (i = 0).
struct LatLayout {
  long long y_zstride, x_zstride;
  __host__ __device__ LatLayout(int P, int nx, int ny) {
    y_zstride = static_cast<long long>(ny + 1) * 2 * nx * (P + 1);
    x_zstride = static_cast<long long>(ny * P + 1) * (nx + 1) * 2;
  }
  __host__ __device__ long long y_index(int P, int nx, int Z, int fy, int side, int cx, int i) const {
    return Z * y_zstride + ((static_cast<long long>(fy) * 2 + side) * nx + cx) * (P + 1) + i;
  }
  __host__ __device__ long long x_index(int nx, int Z, int Y, int fx, int side) const {
    return Z * x_zstride + (static_cast<long long>(Y) * (nx + 1) + fx) * 2 + side;
  }
};

// Doubles of the fast lateral buffer: latY then latX.
__host__ __device__ inline long long lat_fast_doubles(int P, int nx, int ny, int Nz) {
  const LatLayout L(P, nx, ny);
  return (L.y_zstride + L.x_zstride) * Nz;
}

// Where column (ex, ey) stores the partial of its footprint node (i, j) on
// plane Z (ring nodes only): index into latY (is_y) or latX.
__device__ __forceinline__ long long lat_store_index(const LatLayout& L, int P, int nx, int ex, int ey, int i, int j,
                                                     int Z, bool& is_y) {
  if (j == 0 || j == P) {
    is_y = true;
    return L.y_index(P, nx, Z, ey + (j == P), j == 0, ex, i);
  }
  is_y = false;
  return L.x_index(nx, Z, ey * P + j, ex + (i == P), i == 0);
}

// Sum of the column partials of ring node (X, Y, Z) in ascending column index
// order -- for a corner (cy_lo, cx_lo), (cy_lo, cx_hi), (cy_hi, cx_lo),
// (cy_hi, cx_hi) -- each present partial once; loads issued before the sum.
__device__ __forceinline__ double ring_node_sum(const double* latY, const double* latX, const LatLayout& L, int P,
                                                int nx, int ny, int X, int Y, int Z) {
  double s = 0.0;
  if (Y % P == 0) {
    const int fy = Y / P;
    const int cxh = X / P < nx ? X / P : nx - 1;
    const int ih = X - cxh * P;
    const bool lo = X % P == 0 && X > 0 && X / P < nx;  // interior corner: column cxh-1 at i = P too
    const bool below = fy > 0, above = fy < ny;
    const double b0 = below && lo ? __ldcg(latY + L.y_index(P, nx, Z, fy, 0, cxh - 1, P)) : 0.0;
    const double b1 = below ? __ldcg(latY + L.y_index(P, nx, Z, fy, 0, cxh, ih)) : 0.0;
    const double a0 = above && lo ? __ldcg(latY + L.y_index(P, nx, Z, fy, 1, cxh - 1, P)) : 0.0;
    const double a1 = above ? __ldcg(latY + L.y_index(P, nx, Z, fy, 1, cxh, ih)) : 0.0;
    if (below && lo) s += b0;
    if (below) s += b1;
    if (above && lo) s += a0;
    if (above) s += a1;
  } else {
    const int fx = X / P;
    const double l = fx > 0 ? __ldcg(latX + L.x_index(nx, Z, Y, fx, 0)) : 0.0;
    const double r = fx < nx ? __ldcg(latX + L.x_index(nx, Z, Y, fx, 1)) : 0.0;
    if (fx > 0) s += l;
    if (fx < nx) s += r;
  }
  return s;
}

// Global completion of a fused p.Ap: the last CTA sums the column partials in
// index order and applies the CG scalar step. `coldot`: thread 0's sum over the
// CTA's columns; `col`: the CTA index (one partial per CTA).
template <int NT>
__device__ void ring_dot_finish(const ApplyArgs& A, int col, double coldot, double* red) {
  __shared__ int s_last;
  if (A.col_dot == nullptr) return;
  if (threadIdx.x == 0) {
    A.col_dot[col] = coldot;
    __threadfence();
    s_last = atomicAdd(A.fix_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double s = 0.0;
  for (int c = threadIdx.x; c < static_cast<int>(gridDim.x); c += NT) s += __ldcg(A.col_dot + c);
  const double pAp = block_sum<NT>(s, red);
  if (threadIdx.x == 0) {
    *A.fix_done = 0;
    if (A.dot_out) *A.dot_out = pAp;
    if (A.sc) {
      if (!isfinite(pAp) || pAp <= 0.0) {
        A.sc->status = ST_DIVERGED;
      } else {
        A.sc->pAp = pAp;
        A.sc->alpha = A.sc->rz / pAp;
      }
    }
  }
}

}  // namespace hxb
