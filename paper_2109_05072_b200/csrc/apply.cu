// Fused matrix-free BP operator apply for sm_100a: one kernel per apply.
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
// Work decomposition ("element columns"): a CTA owns one (ex, ey) column of
// elements and marches it along z. The structured-mesh gather is index
// arithmetic (mesh.hpp:81); no connectivity table is read.
//
// Deterministic, atomic-free transpose restriction (K4):
//  * z-shared node planes are summed in registers (carry of the previous
//    element's top plane), in element order;
//  * x/y-shared node lines are summed in global memory in COLUMN-TICKET
//    order: columns are claimed through an atomic ticket in row-major order,
//    a column publishes per-element progress with a release store, and a
//    column whose lateral nodes are shared with lower-ticket columns waits
//    (acquire) for those columns' progress before read-modify-writing them.
//    Every node's partial sums are therefore added in one fixed order, so
//    results are bitwise identical run to run (restriction.hpp:18-21), and
//    each L-vector entry is written to HBM once.
//
// Element pipeline (q x q threads per column, z-pencil -> y -> x pencils):
//   Z : thread (i,j) holds u(i,j,:) in registers; B_z u, D_z u        -> smem A
//   Y : thread (i,c) holds a y-pencil; B_y, D_y                         -> smem B
//   X : thread (b,c) holds x-pencils; gr, gs, gt at the q x 1 x 1 points,
//       G streamed from HBM straight to registers (coalesced, L2
//       evict-first, bulk-prefetched one element ahead), then D_x^T/B_x^T -> smem B
//   Y': B_y^T, D_y^T                                                     -> smem A
//   Z': B_z^T, D_z^T into the z-pencil registers = the element's result.
// The contraction order is the reference's (D,B,B),(B,D,B),(B,B,D) with the
// shared sweeps of tensor.hpp:193-202 / 226-234.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_util.cuh"
#include "internal.h"

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
struct BasisT {
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
  static constexpr int SMEM_BYTES = (SA_SIZE + SB_SIZE) * 8;
  static constexpr int MIN_BLOCKS = NT <= 64 ? 8 : (NT <= 96 ? 4 : 3);
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
  __shared__ unsigned int s_col;
  __shared__ int s_last;
  __shared__ double s_red[NT / 32];

  if (A.sc != nullptr && *(volatile int*)&A.sc->status != ST_RUNNING) return;  // CG already stopped

  const int t = threadIdx.x;
  const unsigned int epoch = *(volatile unsigned int*)&A.sync->epoch;
  const unsigned long long pbase = static_cast<unsigned long long>(epoch) * (A.nz + 1);
  const uint64_t pol = policy_evict_first();
  const bool do_dot = A.col_dot != nullptr;
  const bool zrole = t < N * N;
  const int zi = t % N, zj = t / N;

  for (;;) {
    if (t == 0) s_col = atomicAdd(&A.sync->ticket, 1u);
    __syncthreads();
    const int col = static_cast<int>(s_col);
    if (col >= A.ncols) break;
    const int ex = col % A.nx, ey = col / A.nx;
    const int X = ex * P + zi, Y = ey * P + zj;
    // Lateral sharing of this thread's node column (see header comment).
    const bool rmw = (zi == 0 && ex > 0) || (zj == 0 && ey > 0);
    const bool fin = !((zi == P && ex < A.nx - 1) || (zj == P && ey < A.ny - 1));
    const bool bcxy = A.constrained && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1);
    const bool need_wait = ex > 0 || ey > 0;
    double carry = 0.0, dot = 0.0;

    const double* Gcol = A.G + static_cast<long long>(col) * A.nz * A.gstride;
    const uint32_t gbytes = static_cast<uint32_t>(A.gstride * 8);
    if (t == 0) {
      prefetch_l2_bulk(Gcol, gbytes);
      if (A.nz > 1) prefetch_l2_bulk(Gcol + A.gstride, gbytes);
    }

    for (int ez = 0; ez < A.nz; ++ez) {
      if (t == 0 && ez + 2 < A.nz) prefetch_l2_bulk(Gcol + (ez + 2) * A.gstride, gbytes);
      const double* Ge = Gcol + ez * A.gstride;
      double out[N];

      // ---------------- phase Z: gather the z-pencil, contract along z
      if (zrole) {
        double uk[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const int Z = ez * P + k;
          const long long node = X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
          double v = __ldg(A.u + node);
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
            v[a] = s * ld_stream(Ge + a * QQ + t, pol);
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
            const double g0 = ld_stream(g + 0 * Q * QQ, pol), g1 = ld_stream(g + 1 * Q * QQ, pol);
            const double g2 = ld_stream(g + 2 * Q * QQ, pol), g3 = ld_stream(g + 3 * Q * QQ, pol);
            const double g4 = ld_stream(g + 4 * Q * QQ, pol), g5 = ld_stream(g + 5 * Q * QQ, pol);
            const double r = gr[a], s = gs[a], u = gt[a];
            gr[a] = g0 * r + g1 * s + g2 * u;
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
      }

      // ---------------- deterministic transpose restriction
      if (t == 0 && need_wait) {
        const unsigned long long target = pbase + ez + 1;
        const unsigned long long* pr = A.progress;
        if (ex > 0)
          while (ld_acquire_u64(pr + col - 1) < target) {
          }
        if (ey > 0) {
          if (ex > 0)
            while (ld_acquire_u64(pr + col - A.nx - 1) < target) {
            }
          while (ld_acquire_u64(pr + col - A.nx) < target) {
          }
          if (ex + 1 < A.nx)
            while (ld_acquire_u64(pr + col - A.nx + 1) < target) {
            }
        }
        __threadfence();
      }
      __syncthreads();
      if (zrole) {
        out[0] += carry;
        const int kend = (ez == A.nz - 1) ? N : P;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          if (k < kend) {
            const int Z = ez * P + k;
            const long long node = X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
            double v = out[k];
            if (A.constrained && (bcxy || (Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi)))
              v = __ldg(A.u + node);
            else if (rmw)
              v += __ldcg(A.w + node);
            A.w[node] = v;
            if (do_dot && fin) dot = fma(__ldg(A.u + node), v, dot);
          }
        }
        carry = out[P];
      }
      __syncthreads();
      if (t == 0) {
        __threadfence();
        st_release_u64(A.progress + col, pbase + ez + 1);
      }
    }
    if (do_dot) {
      const double s = block_sum<NT>(dot, s_red);
      if (t == 0) A.col_dot[col] = s;
    }
    __syncthreads();
  }

  // ---------------- last CTA: reset the ticket, bump the epoch, finish p.Ap
  __syncthreads();
  if (t == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(&A.sync->done, 1u);
    s_last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (do_dot) {
    double s = 0.0;
    for (int c = t; c < A.ncols; c += NT) s += __ldcg(A.col_dot + c);
    const double pAp = block_sum<NT>(s, s_red);
    if (t == 0) {
      if (A.dot_out) *A.dot_out = pAp;
      if (A.sc) {
        // solver.hpp:128-131
        if (!isfinite(pAp) || pAp <= 0.0) {
          A.sc->status = ST_DIVERGED;
        } else {
          A.sc->pAp = pAp;
          A.sc->alpha = A.sc->rz / pAp;
        }
      }
    }
  }
  if (t == 0) {
    A.sync->ticket = 0;
    A.sync->done = 0;
    A.sync->epoch = epoch + 1;
    __threadfence();
  }
}

template <int P, int Q, int KIND>
void* kernel_ptr() {
  return reinterpret_cast<void*>(&bp_apply_kernel<P, Q, KIND>);
}

template <int P, int Q, int KIND>
cudaError_t launch_t(const Setup& s, const ApplyArgs& a, int grid, cudaStream_t st) {
  using K = Cfg<P, Q, KIND>;
  BasisT<P, Q> bs;
  for (int i = 0; i < Q; ++i)
    for (int j = 0; j <= P; ++j) {
      bs.B[i][j] = s.B[i * (P + 1) + j];
      bs.D[i][j] = s.D[i * (P + 1) + j];
    }
  bp_apply_kernel<P, Q, KIND><<<grid, K::NT, K::SMEM_BYTES, st>>>(a, bs);
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
cudaError_t launch_k(const Setup& s, const ApplyArgs& a, int grid, cudaStream_t st) {
  constexpr int D = KIND == KIND_COLLOC ? 1 : 2;
  switch (s.p) {
    case 1: return launch_t<1, 1 + D, KIND>(s, a, grid, st);
    case 2: return launch_t<2, 2 + D, KIND>(s, a, grid, st);
    case 3: return launch_t<3, 3 + D, KIND>(s, a, grid, st);
    case 4: return launch_t<4, 4 + D, KIND>(s, a, grid, st);
    case 5: return launch_t<5, 5 + D, KIND>(s, a, grid, st);
    case 6: return launch_t<6, 6 + D, KIND>(s, a, grid, st);
    case 7: return launch_t<7, 7 + D, KIND>(s, a, grid, st);
    case 8: return launch_t<8, 8 + D, KIND>(s, a, grid, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int apply_occupancy_grid(const Setup& s) {
  const KInfo ki = info_for(s);
  if (!ki.fn) return 0;
  int per_sm = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ki.fn, ki.nt, ki.smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.device);
  if (per_sm < 1) per_sm = 1;
  const long long ncols = static_cast<long long>(s.dims[0]) * s.dims[1];
  long long g = static_cast<long long>(per_sm) * sms;
  if (g > ncols) g = ncols;
  return static_cast<int>(g < 1 ? 1 : g);
}

void apply_kernel_info(const Setup& s, int* regs, int* smem, int* threads, int* blocks_per_sm) {
  const KInfo ki = info_for(s);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, ki.fn);
  *regs = fa.numRegs;
  *smem = static_cast<int>(fa.sharedSizeBytes) + ki.smem;
  *threads = ki.nt;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, ki.fn, ki.nt, ki.smem);
}

cudaError_t launch_apply(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                         double* dot_out, DevScalars* sc, cudaStream_t st) {
  ApplyArgs a{};
  a.u = u;
  a.w = w;
  a.G = s.G;
  a.gstride = s.gstride;
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
  a.sync = ws.sync;
  a.progress = ws.progress;
  a.col_dot = (dot_out || sc) ? ws.col_dot : nullptr;
  a.sc = sc;
  a.dot_out = dot_out;
  switch (s.kind) {
    case KIND_MASS: return launch_k<KIND_MASS>(s, a, ws.apply_grid, st);
    case KIND_DIFF: return launch_k<KIND_DIFF>(s, a, ws.apply_grid, st);
    case KIND_COLLOC: return launch_k<KIND_COLLOC>(s, a, ws.apply_grid, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hxb
