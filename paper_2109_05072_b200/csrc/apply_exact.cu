// Bit-exact operator apply (reference arithmetic) for sm_100a.
//
// Same work decomposition, staging and lateral fix-up as the fast kernel
// (apply.cu), but every floating-point operation is the reference's:
//  * the contraction ORDER of elem_grad / elem_grad_transpose / elem_interp
//    (tensor.hpp:141-235): x first on the way in, z first on the way out,
//    with the accumulate semantics of contract_dim (tensor.hpp:50-114:
//    axis-0 outputs are fresh sums added to the destination, axis-1/2 outputs
//    continue the destination's running sum);
//  * every product and sum rounded separately (__dmul_rn / __dadd_rn never
//    contract to FMA), as the reference's default x86-64 build computes;
//  * apply_diffusion_factors' expression order (operator.hpp:129-131);
//  * scatter_add's summation order (restriction.hpp:67-80): every node sums
//    its element contributions from 0.0 in ascending element index, i.e. the
//    lower z-layer's columns (ascending) before the upper layer's.
// Given identical inputs the device output is bitwise identical to
// OperatorHandle::apply (Backend::Fused) and ConstrainedOperator::apply.
// Together with the reference-order reductions of cg.cu, the whole device CG
// recurrence reproduces the reference's iterates bit for bit.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_util.cuh"
#include "internal.h"

namespace hxb {
namespace {

#define DM(a, b) __dmul_rn((a), (b))
#define DA(a, b) __dadd_rn((a), (b))

template <int P, int Q>
struct BasisX {
  double B[Q][P + 1];
  double D[Q][P + 1];
};

template <int P, int Q, int KIND>
struct XCfg {
  static constexpr int N = P + 1;
  static constexpr int NQ = N > Q ? N : Q;
  static constexpr int NT = ((NQ * NQ + 31) / 32) * 32;
  static constexpr int COMP = KIND == KIND_MASS ? 1 : 6;
  static constexpr int GS = (COMP * Q * Q * Q + 1) / 2 * 2;
  // Scratch tensors T0..T2: each holds up to max(n,q)^3 doubles, addressed
  // [k][j][i] with i fastest (the x index), row stride R = NQ+1, plane NQ*R+1.
  static constexpr int R = NQ + 1;
  static constexpr int PL = NQ * R + 1;
  static constexpr int TS = NQ * PL + 1;
  static constexpr int NTS = 3;
  static constexpr int G_OFF = (NTS * TS + 1) / 2 * 2;
  static constexpr int U_OFF = G_OFF + GS;
  static constexpr int CZ_OFF = U_OFF + 2 * N * N * N;  // z-carry, double buffered
  static constexpr int BAR_OFF = CZ_OFF + 2 * N * N;
  static constexpr int SMEM_BYTES = (BAR_OFF + 1) * 8;
};

// CTAs per SM the register allocation targets (measured on a B200: the
// kernel spills either way at p >= 7; more resident CTAs win for BP1 at p = 7
// and p = 8, lose for BP3 p = 8; BP3 p = 7 fits three CTAs by shared memory
// and, with the 16-byte factor loads, runs best at that register target:
// reference-mode CG 11.30 -> 10.83 ms/it at cfg3, same iterates)
constexpr int exact_min_blocks(int p, int kind) {
  return (p == 7 && kind == KIND_DIFF) ? 3 : (p == 7 && kind == KIND_MASS) ? 4 : (p == 8 && kind == KIND_MASS) ? 3 : 1;
}
template <int P, int Q, int KIND>
__global__ void __launch_bounds__(XCfg<P, Q, KIND>::NT, exact_min_blocks(P, KIND))
    bp_apply_exact_kernel(const __grid_constant__ ApplyArgs A, const __grid_constant__ BasisX<P, Q> bs) {
  using K = XCfg<P, Q, KIND>;
  constexpr int N = K::N, NT = K::NT, QQ = Q * Q;
  constexpr bool COLLOC = KIND == KIND_COLLOC;
  constexpr bool MASS = KIND == KIND_MASS;
  extern __shared__ double smem[];
  double* T0 = smem;
  double* T1 = smem + K::TS;
  double* T2 = smem + 2 * K::TS;
  double* Gs = smem + K::G_OFF;
  double* Us = smem + K::U_OFF;
  double* Cz = smem + K::CZ_OFF;
  auto at = [](int i, int j, int k) { return k * K::PL + j * K::R + i; };

  const int t = threadIdx.x;
  const uint64_t pol = policy_evict_first();
  const int col = blockIdx.x;
  const int ex = col % A.nx, ey = col / A.nx;
  const double* Gcol = A.G + static_cast<long long>(col) * A.nz * K::GS;
  constexpr uint32_t gbytes = K::GS * 8;
  const uint32_t bar = smem_u32(smem + K::BAR_OFF);
  const long long lat_stride = static_cast<long long>(A.ncols) * (4 * P);
  if (t == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t == 0) {
    mbar_arrive_expect_tx(bar, gbytes);
    bulk_g2s(smem_u32(Gs), Gcol, gbytes, bar, pol);
  }
  // u staging: thread (i,j) of the footprint copies its z-pencil (layout [k][j][i]).
  auto fetch_u = [&](int ez, int buf) {
    if (t < N * N) {
      const int i = t % N, j = t / N;
      const uint32_t dst = smem_u32(Us + buf * N * N * N + t);
      for (int k = 0; k < N; ++k) {
        const long long node = (ex * P + i) + static_cast<long long>(A.Nx) *
                                                  ((ey * P + j) + static_cast<long long>(A.Ny) * (ez * P + k));
        cp_async8(dst + k * N * N * 8, A.u + node);
      }
    }
    cp_async_commit();
  };
  fetch_u(0, 0);

  for (int ez = 0; ez < A.nz; ++ez) {
    if (ez + 1 < A.nz) {
      fetch_u(ez + 1, (ez + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    // nodal values with the ConstrainedOperator mask (solver.hpp:61-62), into T0 as [k][j][i]
    if (t < N * N) {
      const int i = t % N, j = t / N;
      const int X = ex * P + i, Y = ey * P + j;
      const bool bcxy = A.constrained && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1);
      const double* us = Us + (ez & 1) * N * N * N + t;
      for (int k = 0; k < N; ++k) {
        const int Z = ez * P + k;
        double v = us[k * N * N];
        if (A.constrained && (bcxy || (Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi))) v = 0.0;
        T0[at(i, j, k)] = v;
      }
    }
    __syncthreads();

    if constexpr (MASS) {
      // elem_interp (tensor.hpp:141-152): B along x, y, z
      if (t < N * N) {  // x: thread (j,k)
        const int j = t % N, k = t / N;
        double x[N];
        for (int i = 0; i < N; ++i) x[i] = T0[at(i, j, k)];
        for (int a = 0; a < Q; ++a) {
          double s = 0.0;
          for (int i = 0; i < N; ++i) s = DA(s, DM(bs.B[a][i], x[i]));
          T1[at(a, j, k)] = s;
        }
      }
      __syncthreads();
      if (t < Q * N) {  // y: thread (a,k)
        const int a = t % Q, k = t / Q;
        double x[N];
        for (int j = 0; j < N; ++j) x[j] = T1[at(a, j, k)];
        for (int b = 0; b < Q; ++b) {
          double s = 0.0;
          for (int j = 0; j < N; ++j) s = DA(s, DM(bs.B[b][j], x[j]));
          T2[at(a, b, k)] = s;
        }
      }
      __syncthreads();
      mbar_wait_parity(bar, ez & 1);
      if (t < QQ) {  // z, factor, z^T: thread (a,b)
        const int a = t % Q, b = t / Q;
        double x[N], v[Q];
        for (int k = 0; k < N; ++k) x[k] = T2[at(a, b, k)];
        for (int c = 0; c < Q; ++c) {
          double s = 0.0;
          for (int k = 0; k < N; ++k) s = DA(s, DM(bs.B[c][k], x[k]));
          v[c] = DM(s, Gs[a * QQ + b + Q * c]);  // apply_mass_factors (operator.hpp:140)
        }
        // elem_interp_transpose (tensor.hpp:155-172): Bt along z, y, x
        for (int kk = 0; kk < N; ++kk) {
          double s = 0.0;
          for (int c = 0; c < Q; ++c) s = DA(s, DM(bs.B[c][kk], v[c]));
          T1[at(a, b, kk)] = s;
        }
      }
      __syncthreads();
      if (t == 0 && ez + 1 < A.nz) {
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, gbytes);
        bulk_g2s(smem_u32(Gs), Gcol + (ez + 1) * K::GS, gbytes, bar, pol);
      }
      if (t < Q * N) {  // y^T: thread (a,kk)
        const int a = t % Q, kk = t / Q;
        double x[Q];
        for (int b = 0; b < Q; ++b) x[b] = T1[at(a, b, kk)];
        for (int jj = 0; jj < N; ++jj) {
          double s = 0.0;
          for (int b = 0; b < Q; ++b) s = DA(s, DM(bs.B[b][jj], x[b]));
          T2[at(a, jj, kk)] = s;
        }
      }
      __syncthreads();
      if (t < N * N) {  // x^T: thread (jj,kk) -> result in T0 [kk][jj][ii]
        const int jj = t % N, kk = t / N;
        double x[Q];
        for (int a = 0; a < Q; ++a) x[a] = T2[at(a, jj, kk)];
        for (int ii = 0; ii < N; ++ii) {
          double s = 0.0;
          for (int a = 0; a < Q; ++a) s = DA(s, DM(bs.B[a][ii], x[a]));
          T0[at(ii, jj, kk)] = s;
        }
      }
    } else if constexpr (!COLLOC) {
      // ---- elem_grad (tensor.hpp:190-202): ta=D_x u; tb=B_y ta; gr=B_z tb;
      //      ta=B_x u; tb=D_y ta; gs=B_z tb; tb=B_y ta; gt=D_z tb
      if (t < N * N) {  // x: thread (j,k); T1 = D_x u, T2 = B_x u
        const int j = t % N, k = t / N;
        double x[N];
        for (int i = 0; i < N; ++i) x[i] = T0[at(i, j, k)];
        for (int a = 0; a < Q; ++a) {
          double s1 = 0.0, s2 = 0.0;
          for (int i = 0; i < N; ++i) {
            s1 = DA(s1, DM(bs.D[a][i], x[i]));
            s2 = DA(s2, DM(bs.B[a][i], x[i]));
          }
          T1[at(a, j, k)] = s1;
          T2[at(a, j, k)] = s2;
        }
      }
      __syncthreads();
      // y: thread (a,k): y0 = D_x u pencil, y1 = B_x u pencil.
      // outputs (in registers across the barrier): rB = B_y y0, sD = D_y y1, tB = B_y y1
      double ry[Q], sy[Q], ty[Q];
      if (t < Q * N) {
        const int a = t % Q, k = t / Q;
        double y0[N], y1[N];
        for (int j = 0; j < N; ++j) {
          y0[j] = T1[at(a, j, k)];
          y1[j] = T2[at(a, j, k)];
        }
        for (int b = 0; b < Q; ++b) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
          for (int j = 0; j < N; ++j) {
            s0 = DA(s0, DM(bs.B[b][j], y0[j]));
            s1 = DA(s1, DM(bs.D[b][j], y1[j]));
            s2 = DA(s2, DM(bs.B[b][j], y1[j]));
          }
          ry[b] = s0;
          sy[b] = s1;
          ty[b] = s2;
        }
      }
      __syncthreads();
      if (t < Q * N) {
        const int a = t % Q, k = t / Q;
        for (int b = 0; b < Q; ++b) {
          T0[at(a, b, k)] = ry[b];
          T1[at(a, b, k)] = sy[b];
          T2[at(a, b, k)] = ty[b];
        }
      }
      __syncthreads();
      mbar_wait_parity(bar, ez & 1);
      if (t < QQ) {  // z: thread (a,b): gr = B_z T0, gs = B_z T1, gt = D_z T2; factors; z^T
        const int a = t % Q, b = t / Q;
        double z0[N], z1[N], z2[N];
        for (int k = 0; k < N; ++k) {
          z0[k] = T0[at(a, b, k)];
          z1[k] = T1[at(a, b, k)];
          z2[k] = T2[at(a, b, k)];
        }
        double vr[Q], vs[Q], vt[Q];
        for (int c = 0; c < Q; ++c) {
          double r = 0.0, s = 0.0, u = 0.0;
          for (int k = 0; k < N; ++k) {
            r = DA(r, DM(bs.B[c][k], z0[k]));
            s = DA(s, DM(bs.B[c][k], z1[k]));
            u = DA(u, DM(bs.D[c][k], z2[k]));
          }
          // apply_diffusion_factors (operator.hpp:129-131); G at point (a,b,c)
          const int qp = a + Q * (b + Q * c);
          double g0, g1, g2, g3, g4, g5;
          if (A.g_aos) {  // [qp][6]: the point's six components as three 16-byte loads
            const double2* g = reinterpret_cast<const double2*>(Gs + qp * 6);
            const double2 ga = g[0], gb = g[1], gc = g[2];
            g0 = ga.x, g1 = ga.y, g2 = gb.x, g3 = gb.y, g4 = gc.x, g5 = gc.y;
          } else {
            const double* g = A.g_aos ? Gs + qp * 6 : Gs + a * QQ + b + Q * c;
            const int cs = A.g_aos ? 1 : Q * QQ;  // component stride
            g0 = g[0], g1 = g[cs], g2 = g[2 * cs], g3 = g[3 * cs], g4 = g[4 * cs], g5 = g[5 * cs];
          }
          vr[c] = DA(DA(DM(g0, r), DM(g1, s)), DM(g2, u));
          vs[c] = DA(DA(DM(g1, r), DM(g3, s)), DM(g4, u));
          vt[c] = DA(DA(DM(g2, r), DM(g4, s)), DM(g5, u));
        }
        // elem_grad_transpose (tensor.hpp:226-234), z parts:
        //   ta = Bt_z gs  -> T0;  tc = Dt_z gt -> T1;  ta' = Bt_z gr -> T2
        for (int kk = 0; kk < N; ++kk) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
          for (int c = 0; c < Q; ++c) {
            s0 = DA(s0, DM(bs.B[c][kk], vs[c]));
            s1 = DA(s1, DM(bs.D[c][kk], vt[c]));
            s2 = DA(s2, DM(bs.B[c][kk], vr[c]));
          }
          T0[at(a, b, kk)] = s0;
          T1[at(a, b, kk)] = s1;
          T2[at(a, b, kk)] = s2;
        }
      }
      __syncthreads();
      if (t == 0 && ez + 1 < A.nz) {
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, gbytes);
        bulk_g2s(smem_u32(Gs), Gcol + (ez + 1) * K::GS, gbytes, bar, pol);
      }
      // y^T: thread (a,kk): tb = Dt_y ta; tb += Bt_y tc (continuing); tb' = Bt_y ta'
      double c1[N], c2[N];
      if (t < Q * N) {
        const int a = t % Q, kk = t / Q;
        double y0[Q], y1[Q], y2[Q];
        for (int b = 0; b < Q; ++b) {
          y0[b] = T0[at(a, b, kk)];
          y1[b] = T1[at(a, b, kk)];
          y2[b] = T2[at(a, b, kk)];
        }
        for (int jj = 0; jj < N; ++jj) {
          double s = 0.0, s2 = 0.0;
          for (int b = 0; b < Q; ++b) s = DA(s, DM(bs.D[b][jj], y0[b]));
          for (int b = 0; b < Q; ++b) s = DA(s, DM(bs.B[b][jj], y1[b]));
          for (int b = 0; b < Q; ++b) s2 = DA(s2, DM(bs.B[b][jj], y2[b]));
          c1[jj] = s;
          c2[jj] = s2;
        }
      }
      __syncthreads();
      if (t < Q * N) {
        const int a = t % Q, kk = t / Q;
        for (int jj = 0; jj < N; ++jj) {
          T1[at(a, jj, kk)] = c1[jj];
          T2[at(a, jj, kk)] = c2[jj];
        }
      }
      __syncthreads();
      if (t < N * N) {  // x^T: out = Bt_x tb (fresh); out = out + (Dt_x tb') (axis-0 accumulate)
        const int jj = t % N, kk = t / N;
        double x1[Q], x2[Q];
        for (int a = 0; a < Q; ++a) {
          x1[a] = T1[at(a, jj, kk)];
          x2[a] = T2[at(a, jj, kk)];
        }
        for (int ii = 0; ii < N; ++ii) {
          double s = 0.0, s2 = 0.0;
          for (int a = 0; a < Q; ++a) s = DA(s, DM(bs.B[a][ii], x1[a]));
          for (int a = 0; a < Q; ++a) s2 = DA(s2, DM(bs.D[a][ii], x2[a]));
          T0[at(ii, jj, kk)] = DA(s, s2);
        }
      }
    } else {
      // ---- collocated (tensor.hpp:183-187, 214-218): gr = D_x u, gs = D_y u, gt = D_z u;
      //      out = Dt_x gr; out += Dt_y gs (continuing); out += Dt_z gt (continuing)
      if (t < N * N) {  // x: thread (j,k): gr -> T1
        const int j = t % N, k = t / N;
        double x[N];
        for (int i = 0; i < N; ++i) x[i] = T0[at(i, j, k)];
        for (int a = 0; a < N; ++a) {
          double s = 0.0;
          for (int i = 0; i < N; ++i) s = DA(s, DM(bs.D[a][i], x[i]));
          T1[at(a, j, k)] = s;
        }
      }
      if (t < N * N) {  // y: thread (i,k): gs -> T2
        const int i = t % N, k = t / N;
        double x[N];
        for (int j = 0; j < N; ++j) x[j] = T0[at(i, j, k)];
        for (int b = 0; b < N; ++b) {
          double s = 0.0;
          for (int j = 0; j < N; ++j) s = DA(s, DM(bs.D[b][j], x[j]));
          T2[at(i, b, k)] = s;
        }
      }
      __syncthreads();
      mbar_wait_parity(bar, ez & 1);
      double vt[N];
      if (t < N * N) {  // z: thread (a,b): gt, factors -> vr, vs in T1/T2 (in place), vt kept
        const int a = t % N, b = t / N;
        double x[N];
        for (int k = 0; k < N; ++k) x[k] = T0[at(a, b, k)];
        for (int c = 0; c < N; ++c) {
          double u = 0.0;
          for (int k = 0; k < N; ++k) u = DA(u, DM(bs.D[c][k], x[k]));
          const double r = T1[at(a, b, c)], s = T2[at(a, b, c)];
          // factor layout: [m][a][b + q c] (0) or [c][m][b][a] (2, BP5 p=7 DMMA setups)
          const double* g = A.g_aos == 2 ? Gs + (c * 6 * N + b) * N + a : Gs + a * N * N + b + N * c;
          const int cs = A.g_aos == 2 ? N * N : N * N * N;  // component stride
          const double g0 = g[0], g1 = g[cs], g2 = g[2 * cs], g3 = g[3 * cs], g4 = g[4 * cs], g5 = g[5 * cs];
          T1[at(a, b, c)] = DA(DA(DM(g0, r), DM(g1, s)), DM(g2, u));
          T2[at(a, b, c)] = DA(DA(DM(g1, r), DM(g3, s)), DM(g4, u));
          vt[c] = DA(DA(DM(g2, r), DM(g4, s)), DM(g5, u));
        }
      }
      __syncthreads();
      if (t == 0 && ez + 1 < A.nz) {
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, gbytes);
        bulk_g2s(smem_u32(Gs), Gcol + (ez + 1) * K::GS, gbytes, bar, pol);
      }
      if (t < N * N) {  // x^T: thread (j,k): out = Dt_x vr -> T0
        const int j = t % N, k = t / N;
        double x[N];
        for (int a = 0; a < N; ++a) x[a] = T1[at(a, j, k)];
        for (int ii = 0; ii < N; ++ii) {
          double s = 0.0;
          for (int a = 0; a < N; ++a) s = DA(s, DM(bs.D[a][ii], x[a]));
          T0[at(ii, j, k)] = s;
        }
      }
      __syncthreads();
      if (t < N * N) {  // y^T: thread (i,k): out += Dt_y vs, continuing per output
        const int i = t % N, k = t / N;
        double x[N];
        for (int b = 0; b < N; ++b) x[b] = T2[at(i, b, k)];
        for (int jj = 0; jj < N; ++jj) {
          double s = T0[at(i, jj, k)];
          for (int b = 0; b < N; ++b) s = DA(s, DM(bs.D[b][jj], x[b]));
          T0[at(i, jj, k)] = s;
        }
      }
      __syncthreads();
      if (t < N * N) {  // z^T: thread (i,j): out += Dt_z vt, continuing
        const int i = t % N, j = t / N;
        for (int kk = 0; kk < N; ++kk) {
          double s = T0[at(i, j, kk)];
          for (int c = 0; c < N; ++c) s = DA(s, DM(bs.D[c][kk], vt[c]));
          T0[at(i, j, kk)] = s;
        }
      }
    }
    __syncthreads();

    // ---- scatter in reference order (restriction.hpp:75-79). Result in T0 [k][j][i].
    if (t < N * N) {
      const int ii = t % N, jj = t / N;  // thread owns node column (ii, jj) of the footprint
      const int X = ex * P + ii, Y = ey * P + jj;
      const bool ring = ii == 0 || ii == P || jj == 0 || jj == P;
      const bool bcxy = A.constrained && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1);
      double* lat = A.lateral + static_cast<long long>(col) * (4 * P) + ring_index(P, ii, jj);
      const double* cz_in = Cz + (ez & 1) * N * N;
      double* cz_out = Cz + ((ez + 1) & 1) * N * N;
      for (int kk = 0; kk < N; ++kk) {
        const int Z = ez * P + kk;
        const double v = T0[at(ii, jj, kk)];
        if (ring) {
          if (kk == 0 && ez > 0)
            A.zupper[(static_cast<long long>(ez) * A.ncols + col) * (4 * P) + ring_index(P, ii, jj)] = v;
          else
            lat[Z * lat_stride] = v;  // kk == P: lower contribution of plane (ez+1)*P
        } else {
          if (kk == P && ez + 1 < A.nz) {
            cz_out[t] = DA(0.0, v);  // (0 + lower), upper added by the next element
            continue;
          }
          double s = (kk == 0 && ez > 0) ? DA(cz_in[t], v) : DA(0.0, v);
          const long long node = X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
          if (A.constrained && (bcxy || (Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi))) s = __ldg(A.u + node);
          A.w[node] = s;
        }
      }
    }
    __syncthreads();
  }
}

// Reference-order fix-up of the ring nodes: lower-layer column partials in
// ascending column order, then (on z-shared planes) the upper layer's.
constexpr int FT = 256;
__global__ void __launch_bounds__(FT) lateral_fixup_exact_kernel(const __grid_constant__ ApplyArgs A, int P) {
  const long long rowpart = static_cast<long long>(A.ny + 1) * A.Nx;
  const long long colpart = static_cast<long long>(A.nx + 1) * (A.ny * (P - 1));
  const long long per_plane = rowpart + colpart;
  const long long total = per_plane * A.Nz;
  const long long lat_stride = static_cast<long long>(A.ncols) * (4 * P);
  for (long long l = blockIdx.x * static_cast<long long>(FT) + threadIdx.x; l < total;
       l += static_cast<long long>(gridDim.x) * FT) {
    const int Z = static_cast<int>(l / per_plane);
    const long long r = l - static_cast<long long>(Z) * per_plane;
    int X, Y;
    if (r < rowpart) {
      Y = static_cast<int>(r / A.Nx) * P;
      X = static_cast<int>(r % A.Nx);
    } else {
      const long long r2 = r - rowpart;
      const int yy = static_cast<int>(r2 / (A.nx + 1));
      X = static_cast<int>(r2 % (A.nx + 1)) * P;
      Y = (yy / (P - 1)) * P + 1 + yy % (P - 1);
    }
    const int ex_hi = X / P < A.nx ? X / P : A.nx - 1;
    const int ex_lo = (X % P == 0 && X > 0) ? X / P - 1 : ex_hi;
    const int ey_hi = Y / P < A.ny ? Y / P : A.ny - 1;
    const int ey_lo = (Y % P == 0 && Y > 0) ? Y / P - 1 : ey_hi;
    const double* latZ = A.lateral + Z * lat_stride;
    double s = 0.0;
    for (int cy = ey_lo; cy <= ey_hi; ++cy)
      for (int cx = ex_lo; cx <= ex_hi; ++cx)
        s = DA(s, latZ[static_cast<long long>(cy * A.nx + cx) * (4 * P) + ring_index(P, X - cx * P, Y - cy * P)]);
    if (Z % P == 0 && Z > 0 && Z < A.Nz - 1) {
      const double* up = A.zupper + static_cast<long long>(Z / P) * A.ncols * (4 * P);
      for (int cy = ey_lo; cy <= ey_hi; ++cy)
        for (int cx = ex_lo; cx <= ex_hi; ++cx)
          s = DA(s, up[static_cast<long long>(cy * A.nx + cx) * (4 * P) + ring_index(P, X - cx * P, Y - cy * P)]);
    }
    const long long node = X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
    if (A.constrained && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1 || (Z == 0 && A.bc_zlo) ||
                          (Z == A.Nz - 1 && A.bc_zhi)))
      s = A.u[node];
    A.w[node] = s;
  }
}

template <int P, int Q, int KIND>
cudaError_t launch_x(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  using K = XCfg<P, Q, KIND>;
  static std::atomic<uint64_t> configured{0};
  set_smem_attr_once(configured, reinterpret_cast<const void*>(&bp_apply_exact_kernel<P, Q, KIND>), K::SMEM_BYTES);
  if (s.gstride != K::GS) return cudaErrorInvalidValue;
  BasisX<P, Q> bs;
  for (int i = 0; i < Q; ++i)
    for (int j = 0; j <= P; ++j) {
      bs.B[i][j] = s.B[i * (P + 1) + j];
      bs.D[i][j] = s.D[i * (P + 1) + j];
    }
  bp_apply_exact_kernel<P, Q, KIND><<<a.ncols, K::NT, K::SMEM_BYTES, st>>>(a, bs);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_xk(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  constexpr int D = KIND == KIND_COLLOC ? 1 : 2;
  switch (s.p) {
    case 1: return launch_x<1, 1 + D, KIND>(s, a, st);
    case 2: return launch_x<2, 2 + D, KIND>(s, a, st);
    case 3: return launch_x<3, 3 + D, KIND>(s, a, st);
    case 4: return launch_x<4, 4 + D, KIND>(s, a, st);
    case 5: return launch_x<5, 5 + D, KIND>(s, a, st);
    case 6: return launch_x<6, 6 + D, KIND>(s, a, st);
    case 7: return launch_x<7, 7 + D, KIND>(s, a, st);
    case 8: return launch_x<8, 8 + D, KIND>(s, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_apply_exact(const Setup& s, const ApplyArgs& a, int fix_grid, cudaStream_t st) {
  cudaError_t e = cudaErrorInvalidValue;
  switch (s.kind) {
    case KIND_MASS: e = launch_xk<KIND_MASS>(s, a, st); break;
    case KIND_DIFF: e = launch_xk<KIND_DIFF>(s, a, st); break;
    case KIND_COLLOC: e = launch_xk<KIND_COLLOC>(s, a, st); break;
  }
  if (e != cudaSuccess) return e;
  lateral_fixup_exact_kernel<<<fix_grid, FT, 0, st>>>(a, s.p);
  return cudaGetLastError();
}

}  // namespace hxb
