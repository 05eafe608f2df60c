// Fused matrix-free BP operator apply for sm_100a.
//
// Replaces OperatorHandle::apply_fused (operator.hpp:396-414) =
//   gather (restriction.hpp:55-65, inlined operator.hpp:223-225)
//   -> elem_grad / elem_interp        (tensor.hpp:141-203)
//   -> apply_{diffusion,mass}_factors (operator.hpp:124-142)
//   -> elem_grad_transpose / interp^T (tensor.hpp:155-172, 207-235)
//   -> scatter_add                    (restriction.hpp:67-80)
// plus the ConstrainedOperator wrapper (solver.hpp:60-65) and, in CG mode,
// the p.Ap reduction and alpha = rz / pAp (solver.hpp:127-131).
//
// Work decomposition ("element columns"): CTA c owns the (ex, ey) column of
// elements and marches it along z. The structured-mesh gather is index
// arithmetic (mesh.hpp:81); no connectivity table is read.
//
// Deterministic transpose restriction (K4), one launch:
//  1. z-shared node planes are summed in registers (carry of the previous
//     element's top plane, element order). Nodes strictly inside the
//     column's (p+1)x(p+1) footprint belong to it alone: final values are
//     written to w once. Each of the 4p "ring" nodes of the footprint is shared
//     with 1-3 neighbouring columns: the column writes its partial to the
//     lateral buffer lat[Z][column][ring position].
//  2. the ring nodes sum their 1-4 column partials in ascending column order
//     (ring.cuh): lateral_fixup_kernel for plain applies; inside the CG
//     r-update for CG (cg.cu). p.Ap and alpha are complete after part 1.
// Every node's partials are therefore added in one fixed order: results are
// bitwise identical run to run (restriction.hpp:18-21) with no inter-CTA
// waiting.
//
// Element pipeline (q x q threads per column, z-pencil -> y -> x pencils):
//   Z : thread (i,j) holds u(i,j,:) in registers; B_z u, D_z u        -> smem A
//   Y : thread (i,c) holds a y-pencil; B_y, D_y                         -> smem B
//   X : thread (b,c) holds x-pencils; gr, gs, gt at the q points of its x-line,
//       G streamed from HBM straight to registers (coalesced, L2 evict-first,
//       bulk-prefetched two elements ahead), then D_x^T / B_x^T          -> smem B
//   Y': B_y^T, D_y^T                                                     -> smem A
//   Z': B_z^T, D_z^T into the z-pencil registers = the element's result.
// The contraction order is the reference's (D,B,B),(B,D,B),(B,B,D) with the
// shared sweeps of tensor.hpp:193-202 / 226-234.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "device_util.cuh"
#include "internal.h"
#include "ring.cuh"

namespace hxb {

namespace {

// ---- shared-memory padding chosen at compile time to minimise bank conflicts
// for the two strided patterns (8-byte words: a half-warp must touch 16
// distinct word-mod-16 slots to be conflict free).
constexpr int pattern_cost(int N, int Q, int S, int kind) {
  int total = 0;
  const int nact = N * Q;
  for (int h0 = 0; h0 < nact; h0 += 16) {
    int words[16] = {};
    int nw = 0;
    for (int t = h0; t < h0 + 16 && t < nact; ++t) {
      const int i = t % N, c = t / N;
      const int w = kind == 0 ? c * S + i : i * S + c * Q;
      bool dup = false;
      for (int k = 0; k < nw; ++k)
        if (words[k] == w) dup = true;
      if (!dup) words[nw++] = w;
    }
    int cnt[16] = {};
    int deg = 0;
    for (int k = 0; k < nw; ++k) {
      const int b = words[k] % 16;
      cnt[b]++;
      if (cnt[b] > deg) deg = cnt[b];
    }
    total += deg;
  }
  return total;
}

constexpr int best_stride(int N, int Q, int base, int kind) {
  int best = base, bc = 1 << 30;
  for (int pad = 0; pad < 16; ++pad) {
    const int c = pattern_cost(N, Q, base + pad, kind);
    if (c < bc) {
      bc = c;
      best = base + pad;
    }
  }
  return best;
}

template <int P, int Q>
struct alignas(16) BasisT {  // 16-byte aligned kernel parameter: paired constant loads (LDCU.128)
  double B[Q][P + 1];
  double D[Q][P + 1];
};

template <int P, int Q, int KIND>
struct Cfg {
  static constexpr int N = P + 1;
  static constexpr int QQ = Q * Q;
  static constexpr int NT = ((QQ + 31) / 32) * 32;
  static constexpr int FA = KIND == KIND_MASS ? 1 : 2;  // fields in smem A ([f][c][j][i])
  static constexpr int FB = KIND == KIND_MASS ? 1 : 3;  // fields in smem B ([f][i][c][b])
  static constexpr int SA_CS = best_stride(N, Q, N * N, 0);
  static constexpr int SB_IS = best_stride(N, Q, Q * Q, 1);
  static constexpr int SA_SIZE = FA * Q * SA_CS;
  static constexpr int SB_SIZE = FB * N * SB_IS;
  static constexpr int COMP = KIND == KIND_MASS ? 1 : 6;
  static constexpr int GS = (COMP * Q * Q * Q + 1) / 2 * 2;  // element block of G (== Setup::gstride)
  static constexpr int G_OFF = (SA_SIZE + SB_SIZE + 1) / 2 * 2;  // 16-byte aligned TMA destination
  static constexpr int U_OFF = G_OFF + GS;                       // two u slabs (cp.async double buffer)
  static constexpr int BAR_OFF = U_OFF + 2 * N * N * N;
  static constexpr int SMEM_BYTES = (BAR_OFF + 1) * 8;
  // ptxas sizes the register cap as if CTAs were whole 4-warp groups; these
  // values leave the cap at 255 and let registers/smem set the occupancy.
  // (P = 4 stiffness: ptxas spills uniform registers into vector registers
  // (R2UR per basis coefficient) and reaches 194 registers unless capped; six
  // CTAs per SM measured faster despite a small spill.)
  static constexpr int MIN_BLOCKS =
      NT <= 32 ? 8 : (NT <= 64 ? (P == 4 && KIND != KIND_MASS ? 6 : 4) : (NT <= 96 ? 3 : 2));
};

template <int P, int Q, int KIND>
__global__ void __launch_bounds__(Cfg<P, Q, KIND>::NT, Cfg<P, Q, KIND>::MIN_BLOCKS)
    bp_apply_kernel(const __grid_constant__ ApplyArgs A, const __grid_constant__ BasisT<P, Q> bs) {
  using K = Cfg<P, Q, KIND>;
  constexpr int N = K::N, QQ = K::QQ, NT = K::NT;
  constexpr bool COLLOC = KIND == KIND_COLLOC;
  constexpr bool MASS = KIND == KIND_MASS;

  extern __shared__ double smem[];
  double* SA = smem;
  double* SB = smem + K::SA_SIZE;
  __shared__ double s_red[NT / 32];

  if (A.sc != nullptr && *(volatile int*)&A.sc->status != ST_RUNNING) return;  // CG already stopped

  const int t = threadIdx.x;
  const uint64_t pol = policy_evict_first();
  const bool do_dot = A.col_dot != nullptr;
  const bool zrole = t < N * N;
  const int zi = t % N, zj = t / N;
  const int col = blockIdx.x;
  const int ex = col % A.nx, ey = col / A.nx;
  const int X = ex * P + zi, Y = ey * P + zj;
  const bool bcxy = A.constrained && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1);
  const bool ring = zi == 0 || zi == P || zj == 0 || zj == P;
  const bool owner = ring_owner(P, zi, zj, ex, ey, A.nx, A.ny);
  const LatLayout L(P, A.nx, A.ny);
  bool lat_is_y = false;
  const long long lat0 = ring ? lat_store_index(L, P, A.nx, ex, ey, zi, zj, 0, lat_is_y) : 0;
  double* lat = (lat_is_y ? A.lateral : A.lat_x) + lat0;
  const long long lat_stride = lat_is_y ? L.y_zstride : L.x_zstride;
  double carry = 0.0, dot = 0.0;

  // Staging: the element's factor block G_e is copied global -> shared by the
  // TMA bulk engine (one elected thread, mbarrier completion), issued as soon
  // as the previous element's phase X has consumed the buffer; the z-pencil of
  // u for element ez+1 is fetched by LDGSTS (cp.async) into the other half of a
  // double buffer while element ez computes. Neither costs registers.
  const double* Gcol = A.G + static_cast<long long>(col) * A.nz * K::GS;
  constexpr uint32_t gbytes = K::GS * 8;
  double* Gs = smem + K::G_OFF;
  double* Us = smem + K::U_OFF;
  const uint32_t bar = smem_u32(smem + K::BAR_OFF);
  const uint32_t gs_addr = smem_u32(Gs);
  if (t == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t == 0) {
    mbar_arrive_expect_tx(bar, gbytes);
    bulk_g2s(gs_addr, Gcol, gbytes, bar, pol);
    if (A.nz > 1) prefetch_l2_bulk(Gcol + K::GS, gbytes);
  }
  auto fetch_u = [&](int ez, int buf) {
    if (zrole) {
      const uint32_t dst = smem_u32(Us + buf * N * N * N + t);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const long long node =
            X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * (ez * P + k));
        cp_async8(dst + k * N * N * 8, A.u + node);
      }
    }
    cp_async_commit();
  };
  fetch_u(0, 0);

  for (int ez = 0; ez < A.nz; ++ez) {
    if (t == 0 && ez + 2 < A.nz) prefetch_l2_bulk(Gcol + (ez + 2) * K::GS, gbytes);
    const double* Ge = Gs;
    double out[N];
    if (ez + 1 < A.nz) {
      fetch_u(ez + 1, (ez + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }

    // ---------------- phase Z: gather the z-pencil, contract along z
    if (zrole) {
      double uk[N];
      const double* us = Us + (ez & 1) * N * N * N + t;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int Z = ez * P + k;
        double v = us[k * N * N];
        if (A.constrained && (bcxy || (Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi))) v = 0.0;
        uk[k] = v;
      }
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        double s0;
        if constexpr (COLLOC) {
          s0 = uk[c];
        } else {
          s0 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) s0 = fma(bs.B[c][k], uk[k], s0);
        }
        SA[c * K::SA_CS + t] = s0;
        if constexpr (!MASS) {
          double s1 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) s1 = fma(bs.D[c][k], uk[k], s1);
          SA[(Q + c) * K::SA_CS + t] = s1;
        }
      }
    }
    __syncthreads();

    // ---------------- phase Y: y-pencils
    if (t < N * Q) {
      const int i = t % N, c = t / N;
      double y0[N], y1[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        y0[j] = SA[c * K::SA_CS + j * N + i];
        if constexpr (!MASS) y1[j] = SA[(Q + c) * K::SA_CS + j * N + i];
      }
      double* sb = SB + i * K::SB_IS + c * Q;
#pragma unroll
      for (int b = 0; b < Q; ++b) {
        double bb = 0.0, db = 0.0, bd = 0.0;
        if constexpr (COLLOC) {
          bb = y0[b];
          bd = y1[b];
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) bb = fma(bs.B[b][j], y0[j], bb);
          if constexpr (!MASS) {
#pragma unroll
            for (int j = 0; j < N; ++j) bd = fma(bs.B[b][j], y1[j], bd);
          }
        }
        sb[b] = bb;
        if constexpr (!MASS) {
#pragma unroll
          for (int j = 0; j < N; ++j) db = fma(bs.D[b][j], y0[j], db);
          sb[N * K::SB_IS + b] = db;
          sb[2 * N * K::SB_IS + b] = bd;
        }
      }
    }
    __syncthreads();

    // ---------------- phase X: x-pencils, pointwise factors, back along x
    mbar_wait_parity(bar, ez & 1);  // G_e has landed in shared memory
    if (t < QQ) {
      if constexpr (MASS) {
        double x0[N], v[Q];
#pragma unroll
        for (int i = 0; i < N; ++i) x0[i] = SB[i * K::SB_IS + t];
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) s = fma(bs.B[a][i], x0[i], s);
          v[a] = s * Ge[a * QQ + t];
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < Q; ++a) s = fma(bs.B[a][i], v[a], s);
          SB[i * K::SB_IS + t] = s;
        }
      } else {
        double gr[Q], gs[Q], gt[Q];
        {
          double x0[N], x1[N], x2[N];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            x0[i] = SB[i * K::SB_IS + t];
            x1[i] = SB[(N + i) * K::SB_IS + t];
            x2[i] = SB[(2 * N + i) * K::SB_IS + t];
          }
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            double r = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) r = fma(bs.D[a][i], x0[i], r);
            gr[a] = r;
            if constexpr (COLLOC) {
              gs[a] = x1[a];
              gt[a] = x2[a];
            } else {
              double s = 0.0, u = 0.0;
#pragma unroll
              for (int i = 0; i < N; ++i) {
                s = fma(bs.B[a][i], x1[i], s);
                u = fma(bs.B[a][i], x2[i], u);
              }
              gs[a] = s;
              gt[a] = u;
            }
          }
        }
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          const double* g = Ge + a * QQ + t;
          const double g0 = g[0 * Q * QQ], g1 = g[1 * Q * QQ], g2 = g[2 * Q * QQ];
          const double g3 = g[3 * Q * QQ], g4 = g[4 * Q * QQ], g5 = g[5 * Q * QQ];
          const double r = gr[a], s = gs[a], u = gt[a];
          gr[a] = g0 * r + g1 * s + g2 * u;  // operator.hpp:129-131
          gs[a] = g1 * r + g3 * s + g4 * u;
          gt[a] = g2 * r + g4 * s + g5 * u;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int a = 0; a < Q; ++a) a1 = fma(bs.D[a][i], gr[a], a1);
          if constexpr (COLLOC) {
            a2 = gs[i];
            a3 = gt[i];
          } else {
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              a2 = fma(bs.B[a][i], gs[a], a2);
              a3 = fma(bs.B[a][i], gt[a], a3);
            }
          }
          SB[i * K::SB_IS + t] = a1;
          SB[(N + i) * K::SB_IS + t] = a2;
          SB[(2 * N + i) * K::SB_IS + t] = a3;
        }
      }
    }
    __syncthreads();
    if (t == 0 && ez + 1 < A.nz) {  // G buffer consumed: stream the next element's block
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, gbytes);
      bulk_g2s(gs_addr, Gcol + (ez + 1) * K::GS, gbytes, bar, pol);
    }

    // ---------------- phase Y': back along y
    if (t < N * Q) {
      const int i = t % N, c = t / N;
      const double* sb = SB + i * K::SB_IS + c * Q;
      double a0[Q], a1[Q], a2[Q];
#pragma unroll
      for (int b = 0; b < Q; ++b) {
        a0[b] = sb[b];
        if constexpr (!MASS) {
          a1[b] = sb[N * K::SB_IS + b];
          a2[b] = sb[2 * N * K::SB_IS + b];
        }
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double c1 = 0.0, c2 = 0.0;
        if constexpr (MASS) {
#pragma unroll
          for (int b = 0; b < Q; ++b) c1 = fma(bs.B[b][j], a0[b], c1);
        } else if constexpr (COLLOC) {
          c1 = a0[j];
#pragma unroll
          for (int b = 0; b < Q; ++b) c1 = fma(bs.D[b][j], a1[b], c1);
          c2 = a2[j];
        } else {
#pragma unroll
          for (int b = 0; b < Q; ++b) {
            c1 = fma(bs.B[b][j], a0[b], c1);
            c2 = fma(bs.B[b][j], a2[b], c2);
          }
#pragma unroll
          for (int b = 0; b < Q; ++b) c1 = fma(bs.D[b][j], a1[b], c1);
        }
        SA[c * K::SA_CS + j * N + i] = c1;
        if constexpr (!MASS) SA[(Q + c) * K::SA_CS + j * N + i] = c2;
      }
    }
    __syncthreads();

    // ---------------- phase Z': back along z into the z-pencil
    if (zrole) {
      double c1[Q], c2[Q];
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        c1[c] = SA[c * K::SA_CS + t];
        if constexpr (!MASS) c2[c] = SA[(Q + c) * K::SA_CS + t];
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
        if constexpr (COLLOC) {
          s = c1[k];
        } else {
#pragma unroll
          for (int c = 0; c < Q; ++c) s = fma(bs.B[c][k], c1[c], s);
        }
        if constexpr (!MASS) {
#pragma unroll
          for (int c = 0; c < Q; ++c) s = fma(bs.D[c][k], c2[c], s);
        }
        out[k] = s;
      }

      // ---------------- transpose restriction, part 1 (see header)
      out[0] += carry;
      const int kend = (ez == A.nz - 1) ? N : P;
      const double* usz = Us + (ez & 1) * N * N * N + t;  // u of this element, still staged
      if (!do_dot) {  // plain apply: the lean epilogue (keeps ptxas' uniform registers for the basis)
#pragma unroll
        for (int k = 0; k < N; ++k) {
          if (k < kend) {
            const int Z = ez * P + k;
            if (ring) {
              lat[Z * lat_stride] = out[k];
            } else {
              const long long node = X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
              double v = out[k];
              if (A.constrained && ((Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi))) v = usz[k * N * N];
              A.w[node] = v;
            }
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          if (k < kend) {
            const int Z = ez * P + k;
            const double uv = usz[k * N * N];
            const bool zbc = A.constrained && ((Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi));
            if (ring) {
              lat[Z * lat_stride] = out[k];
              // column-local share of p.Ap on the ring (ring.cuh); w = u rows counted once
              if (bcxy || zbc)
                dot = owner ? fma(uv, uv, dot) : dot;
              else
                dot = fma(uv, out[k], dot);
            } else {
              const long long node = X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
              const double v = zbc ? uv : out[k];
              A.w[node] = v;
              dot = fma(uv, v, dot);
            }
          }
        }
      }
      carry = out[P];
    }
    __syncthreads();  // smem A is rewritten by the next element's phase Z
  }
  const double cdot = do_dot ? block_sum<NT>(dot, s_red) : 0.0;
  ring_dot_finish<NT>(A, col, cdot, s_red);
}

// Transpose restriction, part 2, for plain applies: every ring node sums its
// 1-4 column partials in ascending column order (ring.cuh). (CG fuses this
// into its r-update, cg.cu; p.Ap is complete after part 1.)
constexpr int FT = 256;

__global__ void __launch_bounds__(FT) lateral_fixup_kernel(const __grid_constant__ ApplyArgs A, int P) {
  // one warp per node row (Y, Z): ring rows (Y % P == 0) finish every node,
  // other rows their x-face nodes X = fx*P
  const LatLayout L(P, A.nx, A.ny);
  const int lane = threadIdx.x & 31;
  const long long rows = static_cast<long long>(A.Ny) * A.Nz;
  for (long long row = blockIdx.x * (FT / 32) + (threadIdx.x >> 5); row < rows;
       row += static_cast<long long>(gridDim.x) * (FT / 32)) {
    const int Z = static_cast<int>(row / A.Ny), Y = static_cast<int>(row - static_cast<long long>(Z) * A.Ny);
    const bool yring = Y % P == 0;
    const int count = yring ? A.Nx : A.nx + 1;
    const bool bcrow = A.constrained && (Y == 0 || Y == A.Ny - 1 || (Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi));
    for (int q = lane; q < count; q += 32) {
      const int X = yring ? q : q * P;
      const long long node = X + static_cast<long long>(A.Nx) * row;
      double s;
      if (A.constrained && (bcrow || X == 0 || X == A.Nx - 1))
        s = A.u[node];
      else
        s = ring_node_sum(A.lateral, A.lat_x, L, P, A.nx, A.ny, X, Y, Z);
      A.w[node] = s;
    }
  }
}

template <int P, int Q, int KIND>
void* kernel_ptr() {
  static bool configured = false;  // opt in to > 48 KB dynamic shared memory once per instantiation
  if (!configured) {
    cudaFuncSetAttribute(&bp_apply_kernel<P, Q, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg<P, Q, KIND>::SMEM_BYTES);
    configured = true;
  }
  return reinterpret_cast<void*>(&bp_apply_kernel<P, Q, KIND>);
}

template <int P, int Q, int KIND>
cudaError_t launch_t(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  using K = Cfg<P, Q, KIND>;
  kernel_ptr<P, Q, KIND>();
  if (s.gstride != K::GS) return cudaErrorInvalidValue;
  BasisT<P, Q> bs;
  for (int i = 0; i < Q; ++i)
    for (int j = 0; j <= P; ++j) {
      bs.B[i][j] = s.B[i * (P + 1) + j];
      bs.D[i][j] = s.D[i * (P + 1) + j];
    }
  bp_apply_kernel<P, Q, KIND><<<a.ncols, K::NT, K::SMEM_BYTES, st>>>(a, bs);
  return cudaGetLastError();
}

struct KInfo {
  void* fn;
  int nt;
  int smem;
};

template <int P, int KIND>
KInfo info_t() {
  constexpr int Q = KIND == KIND_COLLOC ? P + 1 : P + 2;
  using K = Cfg<P, Q, KIND>;
  return {kernel_ptr<P, Q, KIND>(), K::NT, K::SMEM_BYTES};
}

template <int KIND>
KInfo info_k(int p) {
  switch (p) {
    case 1: return info_t<1, KIND>();
    case 2: return info_t<2, KIND>();
    case 3: return info_t<3, KIND>();
    case 4: return info_t<4, KIND>();
    case 5: return info_t<5, KIND>();
    case 6: return info_t<6, KIND>();
    case 7: return info_t<7, KIND>();
    case 8: return info_t<8, KIND>();
  }
  return {nullptr, 0, 0};
}

KInfo info_for(const Setup& s) {
  switch (s.kind) {
    case KIND_MASS: return info_k<KIND_MASS>(s.p);
    case KIND_DIFF: return info_k<KIND_DIFF>(s.p);
    case KIND_COLLOC: return info_k<KIND_COLLOC>(s.p);
  }
  return {nullptr, 0, 0};
}

template <int KIND>
cudaError_t launch_k(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  constexpr int D = KIND == KIND_COLLOC ? 1 : 2;
  switch (s.p) {
    case 1: return launch_t<1, 1 + D, KIND>(s, a, st);
    case 2: return launch_t<2, 2 + D, KIND>(s, a, st);
    case 3: return launch_t<3, 3 + D, KIND>(s, a, st);
    case 4: return launch_t<4, 4 + D, KIND>(s, a, st);
    case 5: return launch_t<5, 5 + D, KIND>(s, a, st);
    case 6: return launch_t<6, 6 + D, KIND>(s, a, st);
    case 7: return launch_t<7, 7 + D, KIND>(s, a, st);
    case 8: return launch_t<8, 8 + D, KIND>(s, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int fixup_grid(const Setup& s) {
  const long long P = s.p;
  const long long nx = s.dims[0], ny = s.dims[1];
  const long long per_plane = (ny + 1) * (nx * P + 1) + (nx + 1) * ny * (P - 1);
  const long long total = per_plane * (s.dims[2] * P + 1);
  long long g = (total + FT - 1) / FT;
  if (g > 148 * 8) g = 148 * 8;
  return static_cast<int>(g < 1 ? 1 : g);
}

// DMMA kernel for BP3 p = 7 unless HEXBP_NO_DMMA=1 (A/B comparisons).
bool use_mma(const Setup& s) {
  static const bool disabled = [] {
    const char* v = std::getenv("HEXBP_NO_DMMA");
    return v && *v && *v != '0';
  }();
  // the [qp][6] factor layout of BP3 p=7 setups is read by the DMMA kernel only
  return (s.g_aos || !disabled) && (mma_kernel_applies(s) || mma5_kernel_applies(s));
}

void apply_kernel_info(const Setup& s, int* regs, int* smem, int* threads, int* blocks_per_sm) {
  if (use_mma(s)) {
    if (mma5_kernel_applies(s))
      mma5_kernel_info(regs, smem, threads, blocks_per_sm);
    else
      mma_kernel_info(regs, smem, threads, blocks_per_sm);
    return;
  }
  const KInfo ki = info_for(s);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, ki.fn);
  *regs = fa.numRegs;
  *smem = static_cast<int>(fa.sharedSizeBytes) + ki.smem;
  *threads = ki.nt;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, ki.fn, ki.nt, ki.smem);
}

cudaError_t launch_apply(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                         double* dot_out, DevScalars* sc, cudaStream_t st, bool finish_ring) {
  ApplyArgs a{};
  a.u = u;
  a.w = w;
  a.G = s.G;
  a.gstride = s.gstride;
  a.g_aos = s.g_aos;
  a.nx = s.dims[0];
  a.ny = s.dims[1];
  a.nz = s.dims[2];
  a.Nx = s.dims[0] * s.p + 1;
  a.Ny = s.dims[1] * s.p + 1;
  a.Nz = s.dims[2] * s.p + 1;
  a.ncols = s.dims[0] * s.dims[1];
  a.constrained = constrained;
  a.bc_zlo = s.bc_zlo;
  a.bc_zhi = s.bc_zhi;
  a.lateral = ws.lateral;
  a.lat_x = ws.lateral + LatLayout(s.p, s.dims[0], s.dims[1]).y_zstride * (s.dims[2] * s.p + 1);
  a.zupper = ws.zupper;
  a.col_dot = (dot_out || sc) ? ws.col_dot : nullptr;
  a.fix_partials = ws.fix_partials;
  a.fix_done = ws.fix_done;
  a.sc = sc;
  a.dot_out = dot_out;
  if (ws.multipass) {  // Backend::Multipass analog (reference arithmetic; CG reduces in cg.cu)
    if (dot_out || sc) return cudaErrorInvalidValue;
    return launch_apply_multipass(s, ws.mp_buf, u, w, constrained, st);
  }
  if (ws.exact) {
    if (dot_out || sc) return cudaErrorInvalidValue;  // the exact path reduces in cg.cu
    return launch_apply_exact(s, a, ws.fixup_grid, st);
  }
  cudaError_t e = cudaErrorInvalidValue;
  if (use_mma(s)) {
    e = mma5_kernel_applies(s) ? launch_apply_mma5(s, a, st) : launch_apply_mma(s, a, st);
  } else {
    switch (s.kind) {
      case KIND_MASS: e = launch_k<KIND_MASS>(s, a, st); break;
      case KIND_DIFF: e = launch_k<KIND_DIFF>(s, a, st); break;
      case KIND_COLLOC: e = launch_k<KIND_COLLOC>(s, a, st); break;
    }
  }
  if (e != cudaSuccess || !finish_ring) return e;  // CG: the r-update sums the ring (cg.cu)
  lateral_fixup_kernel<<<ws.fixup_grid, FT, 0, st>>>(a, s.p);
  return cudaGetLastError();
}

}  // namespace hxb
