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
// Work decomposition ("element columns"): a CTA owns KC element columns
// (ex, ey) and marches them along z (optionally one z-segment of them, see
// z_segments). The structured-mesh gather is index arithmetic (mesh.hpp:81);
// no connectivity table is read. BP1 at p = 1 uses one thread per column
// instead (tpc_mass_kernel).
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
// Element pipeline (one thread per pencil and column, z-pencil -> y -> x):
//   Z : thread (i,j) holds u(i,j,:) in registers; B_z u, D_z u        -> smem A
//   Y : thread (i,c) holds a y-pencil; B_y, D_y                         -> smem B
//   X : thread (b,c) holds x-pencils; gr, gs, gt at the q points of its x-line,
//       times the factors G_e (TMA-staged in shared memory, L2 evict-first,
//       bulk-prefetched two elements ahead), then D_x^T / B_x^T          -> smem B
//   Y': B_y^T, D_y^T                                                     -> smem A
//   Z': B_z^T, D_z^T into the z-pencil registers = the element's result.
// Every 1D contraction is either the plain product or its even-odd form
// (EOB, from p = 4); both round differently from the reference's loop order
// (fast mode; apply_exact.cu is the bit-exact path).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
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

// Even-odd form of a q x n basis matrix M on symmetric points,
// M[q-1-a][n-1-i] = sg M[a][i] (sg = +1 for B, -1 for D): with e_i = x_i +
// x_{n-1-i}, o_i = x_i - x_{n-1-i}, the pair (y_a, y_{q-1-a}) of y = M x is
// (A + B, sg (A - B)), A = sum_i P[a][i] e_i (+ M[a][n/2] x_mid), B = sum_i
// R[a][i] o_i -- half the multiply-adds and half the coefficients of the
// plain product (the transposed product likewise). Fast mode only: it
// rounds differently from the reference's loop order.
template <int N, int Q>
struct EOB {
  static constexpr int NH = N / 2, QH = Q / 2;
  double P[QH][NH];  // (M[a][i] + M[a][N-1-i]) / 2, a < q/2, i < n/2
  double R[QH][NH];  // (M[a][i] - M[a][N-1-i]) / 2
  double col[QH];    // M[a][n/2]      (n odd)
  double row[NH];    // M[q/2][i]      (q odd)
  double ctr;        // M[q/2][n/2]    (both odd)
};

template <int P, int Q>
struct alignas(16) BasisT {  // 16-byte aligned kernel parameter: paired constant loads (LDCU.128)
  double B[Q][P + 1];
  double D[Q][P + 1];
  EOB<P + 1, Q> eB, eD;
};

template <int N>
__device__ __forceinline__ void eo_split(const double (&x)[N], double (&e)[N / 2], double (&o)[N / 2]) {
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    e[i] = x[i] + x[N - 1 - i];
    o[i] = x[i] - x[N - 1 - i];
  }
}

// y = M x, y_a handed to st(a, y_a)
template <int SG, int N, int Q, class F>
__device__ __forceinline__ void eo_fwd(const EOB<N, Q>& m, const double (&e)[N / 2], const double (&o)[N / 2],
                                       const double (&x)[N], F&& st) {
  constexpr int NH = N / 2, QH = Q / 2;
#pragma unroll
  for (int a = 0; a < QH; ++a) {
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int i = 0; i < NH; ++i) {
      sa = fma(m.P[a][i], e[i], sa);
      sb = fma(m.R[a][i], o[i], sb);
    }
    if constexpr (N & 1) sa = fma(m.col[a], x[NH], sa);
    st(a, sa + sb);
    st(Q - 1 - a, SG > 0 ? sa - sb : sb - sa);
  }
  if constexpr (Q & 1) {
    double c = 0.0;
#pragma unroll
    for (int i = 0; i < NH; ++i) c = fma(m.row[i], SG > 0 ? e[i] : o[i], c);
    if constexpr (N & 1) c = fma(m.ctr, x[NH], c);
    st(QH, c);
  }
}

// y (+)= M^T v
template <int SG, bool ACC, int N, int Q>
__device__ __forceinline__ void eo_bwd(const EOB<N, Q>& m, const double (&v)[Q], double (&y)[N]) {
  constexpr int NH = N / 2, QH = Q / 2;
  double ve[QH], vo[QH];
#pragma unroll
  for (int a = 0; a < QH; ++a) {
    ve[a] = SG > 0 ? v[a] + v[Q - 1 - a] : v[a] - v[Q - 1 - a];
    vo[a] = SG > 0 ? v[a] - v[Q - 1 - a] : v[a] + v[Q - 1 - a];
  }
#pragma unroll
  for (int i = 0; i < NH; ++i) {
    double sp = 0.0, sq = 0.0;
#pragma unroll
    for (int a = 0; a < QH; ++a) {
      sp = fma(m.P[a][i], ve[a], sp);
      sq = fma(m.R[a][i], vo[a], sq);
    }
    double lo = sp + sq, hi = sp - sq;
    if constexpr (Q & 1) {
      lo = fma(m.row[i], v[QH], lo);
      hi = SG > 0 ? fma(m.row[i], v[QH], hi) : fma(-m.row[i], v[QH], hi);
    }
    y[i] = ACC ? y[i] + lo : lo;
    y[N - 1 - i] = ACC ? y[N - 1 - i] + hi : hi;
  }
  if constexpr (N & 1) {
    double c = 0.0;
#pragma unroll
    for (int a = 0; a < QH; ++a) c = fma(m.col[a], ve[a], c);
    if constexpr (Q & 1) c = fma(m.ctr, v[QH], c);
    y[NH] = ACC ? y[NH] + c : c;
  }
}

// Work split of the element kernel, per (P, KIND), as a code
// SK = TPC*1000000 + EO*100000 + R*100 + 10 + KC: KC element columns per CTA
// (fills the warps when q^2 is small), R*8 a register cap (R = 0: 255), EO the
// even-odd contractions (EOB above), TPC the thread-per-column kernels below
// (BP1 p = 1, 2 and BP5 p = 1; SK/10 % 10 is then the min CTAs per SM, SK/100 % 10
// the cp.async staging of the BP1 kernel). The tens digit is 1:
// one lane per pencil (splitting pencils over 2-4 lanes and double-buffered G
// staging lost every sweep and were removed). Values: measured per p on a B200
// (profiles/r1c_sk_sweep*.jsonl; with the column pads: r2t_sk_kc_sweep.jsonl).
constexpr int sk_default(int kind, int p) {
  // kind 0 = mass (Q = P+2), 1 = diffusion (Q = P+2), 2 = collocated (Q = P+1)
  constexpr int mass[9] = {0, 1000000, 1000100, 100014, 100015, 100013, 100012, 100011, 100012};
  // p = 7 BP3 / BP5 run the DMMA kernels; these entries serve HEXBP_NO_DMMA=1 setups
  constexpr int diff[9] = {0, 17, 12, 13, 101612, 102111, 100011, 102011, 100011};
  constexpr int coll[9] = {0, 1000020, 16, 12, 100013, 100012, 100012, 100011, 100011};
  return kind == 0 ? mass[p] : kind == 1 ? diff[p] : coll[p];
}
// Candidate codes compiled for (KIND, P); the first is the default. A sweep
// build (-DHX_SK_SWEEP='"header"', tools/build_variant.py) specialises this
// with more candidates, selected at run time by HEXBP_SK_<kind>_<p>=<code>.
template <int KIND, int P>
struct SkList {
  static constexpr int n = 1;
  static constexpr int v[1] = {sk_default(KIND, P)};
};
#ifdef HX_SK_SWEEP
#include HX_SK_SWEEP
#endif

// Column strides of the per-column scratch (CB) and of the staged G blocks
// (GSM) when a CTA packs KC > 1 element columns: best_stride above makes one
// column's pencil patterns conflict free, but the KC columns of a warp land
// on the same banks when CB / GS are multiples of 16 apart. Pads chosen per
// default (kind, p, KC) with an 8-byte-word bank model of all nine phase
// accesses, each half-warp a separate request (wavefronts = the largest number
// of distinct words on one bank; a whole-warp model mispredicted BP5 p = 2,
// measured 13% slower with its pads): 3-44% fewer modelled shared-memory
// wavefronts per element.
// Encoded cb_pad * 100 + gs_pad (gs_pad even: 16-byte TMA destinations), for
// every KC a work-split sweep may pick (p <= 6; KC = 1 needs none: the
// per-pencil strides of best_stride are already optimal under the model).
constexpr short kColPad[3][9][9] = {  // [kind][p][KC], generated by tools/bank_model.py --table
    {{0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, 700, 1314, 0, 1100, 1100, 1114, 1100},
     {0, 0, 500, 500, 500, 500, 500, 500, 500},
     {0, 0, 500, 500, 500, 512, 500, 500, 500},
     {0, 0, 1312, 1312, 1312, 1312, 1312, 1312, 1312},
     {0, 0, 400, 400, 400, 100, 100, 100, 100},
     {0, 0, 100, 100, 100, 100, 100, 100, 100},
     {0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, 0, 0, 0, 0, 0, 0, 0}},
    {{0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, 700, 1308, 4, 1108, 1104, 1108, 1108},
     {0, 0, 1500, 1500, 1500, 1500, 1500, 1500, 1500},
     {0, 0, 100, 100, 100, 112, 100, 100, 100},
     {0, 0, 4, 4, 4, 504, 4, 4, 4},
     {0, 0, 1100, 1100, 1100, 1100, 1100, 1100, 1100},
     {0, 0, 900, 1100, 1100, 1100, 1100, 1100, 1100},
     {0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, 0, 0, 0, 0, 0, 0, 0}},
    {{0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, 4, 204, 404, 404, 104, 404, 404},
     {0, 0, 1100, 1108, 1104, 1108, 1104, 1108, 1108},
     {0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, 700, 700, 700, 712, 700, 700, 700},
     {0, 0, 1004, 1004, 1004, 1004, 1004, 1004, 1004},
     {0, 0, 900, 900, 900, 900, 900, 900, 900},
     {0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, 0, 0, 0, 0, 0, 0, 0}}};
// Per-column stride pad of the u staging slabs (cp.async writes, phase-Z and
// epilogue reads: pencil pz of column kz at kz (2 n^3 + pad) + k n^2 + pz),
// the smallest pad minimising the same half-warp bank model.
constexpr int u_pad_cost(int N, int KC, int pad) {
  int total = 0;
  const int zi = KC * N * N;
  for (int h0 = 0; h0 < zi; h0 += 16)
    for (int k = 0; k < N; ++k) {
      int cnt[16] = {};
      int deg = 0;
      for (int t = h0; t < h0 + 16 && t < zi; ++t) {
        const int w = (t / (N * N)) * (2 * N * N * N + pad) + k * N * N + t % (N * N);
        const int b = ((w % 16) + 16) % 16;
        if (++cnt[b] > deg) deg = cnt[b];
      }
      total += deg;
    }
  return total;
}
constexpr int u_pad(int N, int KC) {
  int best = 0, bc = 1 << 30;
  for (int pad = 0; pad < 16; ++pad) {
    const int c = u_pad_cost(N, KC, pad);
    if (c < bc) {
      bc = c;
      best = pad;
    }
  }
  return best;
}
// Joint optimum of the pencil strides for BP5 p = 2 at six columns per CTA
// (tools/bank_model.py with the strides free: 468 -> 390 modelled wavefronts
// per element step) and BP3 p = 1 at seven; elsewhere best_stride's
// per-column choice is already jointly optimal. Encoded sa_cs * 100 + sb_is, 0 = best_stride.
constexpr int stride_override(int kind, int p, int kc) {
  return kind == 2 && p == 2 && kc == 6 ? 2217 : kind == 1 && p == 1 && kc == 7 ? 524 : 0;  // BP3 p = 1: 378 -> 324
}

constexpr int col_pad(int kind, int p, int kc) {
  if (kind == 0 && p == 8 && kc == 2) return 512;  // BP1 p = 8's default split (the table stops at p = 6)
  return kind >= 0 && kind < 3 && p >= 0 && p < 9 && kc >= 0 && kc < 9 ? kColPad[kind][p][kc] : 0;
}

template <int P, int Q, int KIND, int SK>
struct Cfg {
  static constexpr int N = P + 1;
  static constexpr int QQ = Q * Q;
  static constexpr bool EO = SK / 100000 % 10;   // even-odd contractions
  static constexpr int KC = SK % 10;      // element columns per CTA
  static constexpr int MAXREG = SK / 100 % 100 ? SK / 100 % 100 * 8 : 255;
  static constexpr int ZI = KC * N * N, YI = KC * N * Q, XI = KC * QQ;  // pencils per phase
  static constexpr int NT = ((XI + 31) / 32) * 32;
  static constexpr int FA = KIND == KIND_MASS ? 1 : 2;  // fields in smem A ([f][c][j][i])
  static constexpr int FB = KIND == KIND_MASS ? 1 : 3;  // fields in smem B ([f][i][c][b])
#ifdef HX_NO_COL_PAD
  static constexpr int SOV = 0;
#else
  static constexpr int SOV = stride_override(KIND, P, KC);
#endif
  static constexpr int SA_CS = SOV ? SOV / 100 : best_stride(N, Q, N * N, 0);
  static constexpr int SB_IS = SOV ? SOV % 100 : best_stride(N, Q, Q * Q, 1);
  static constexpr int SA_SIZE = FA * Q * SA_CS;
  static constexpr int SB_SIZE = FB * N * SB_IS;
#ifdef HX_NO_COL_PAD
  static constexpr int PADC = 0;
#else
  static constexpr int PADC = KC > 1 ? col_pad(KIND, P, KC) : 0;
#endif
  static constexpr int CB = (SA_SIZE + SB_SIZE + 1) / 2 * 2 + PADC / 100;  // per-column scratch (A then B)
  static constexpr int COMP = KIND == KIND_MASS ? 1 : 6;
  static constexpr int GS = (COMP * Q * Q * Q + 1) / 2 * 2;  // element block of G (== Setup::gstride)
  static constexpr int GSM = GS + PADC % 100;                // shared-memory stride of the staged G blocks
  static constexpr int G_OFF = (KC * CB + 1) / 2 * 2;        // 16-byte aligned TMA destinations
  static constexpr int U_OFF = G_OFF + KC * GSM;             // per column two u slabs (cp.async double buffer)
#ifdef HX_NO_COL_PAD
  static constexpr int USTR = 2 * N * N * N;
#else
  static constexpr int USTR = 2 * N * N * N + (KC > 1 ? u_pad(N, KC) : 0);  // per-column u staging stride
#endif
  static constexpr int BAR_OFF = U_OFF + KC * USTR;
  static constexpr int SMEM_BYTES = (BAR_OFF + 1) * 8;
};

// F: bit 0 = ConstrainedOperator semantics (ApplyArgs::constrained), bit 1 =
// the CG form with the fused p.Ap (ApplyArgs::col_dot), bit 2 = a sub-range
// launch with carry shares (the multi-GPU overlap) -- compile-time flags,
// so neither costs tests (or registers) in the phase bodies (+1-5% over the
// run-time flags across BP1/BP3/BP5 p = 2..8; BP1 p = 6, 8: -2%).
template <int P, int Q, int KIND, int SK, int F = 3, typename K_ = Cfg<P, Q, KIND, SK>>
__global__ void __launch_bounds__(K_::NT) __maxnreg__(K_::MAXREG)
    bp_apply_kernel(const __grid_constant__ ApplyArgs A, const __grid_constant__ BasisT<P, Q> bs, int nseg) {
  constexpr bool CON = (F & 1) != 0;
  constexpr bool RNG = (F & 4) != 0;  // carry shares of a sub-range launch (overlap.cu)
  using K = Cfg<P, Q, KIND, SK>;
  constexpr int N = K::N, QQ = K::QQ, NT = K::NT, KC = K::KC;
  constexpr int NH = N / 2;
  constexpr bool COLLOC = KIND == KIND_COLLOC;
  constexpr bool MASS = KIND == KIND_MASS;

  extern __shared__ double smem[];
  __shared__ double s_red[NT / 32];

  if (A.sc != nullptr && *(volatile int*)&A.sc->status != ST_RUNNING) return;  // CG already stopped

  const int t = threadIdx.x;
  const int item = t;               // pencil index (per phase)
  const int wfirst = t & ~31;       // first pencil of this warp: whole-warp phase skips
  const uint64_t pol = policy_evict_first();
  constexpr bool do_dot = (F & 2) != 0;
  // CTA = (column group, z-segment). A segment recomputes the element below
  // its first one without storing anything, so the carry hands it the full
  // bottom node plane and it owns that plane outright (no cross-CTA sum).
  // The segments split the launch's element range [zr0, zr1) (the whole
  // column, or a sub-range of the multi-GPU overlap, overlap.cu: a range that
  // starts / ends inside the slab leaves its bottom / top plane as a share in
  // carry_lo / carry_hi for launch_carry_combine -- no store, no dot).
  const int ncta = (A.ncols + KC - 1) / KC;
  const int seg = blockIdx.x / ncta;
  const int col0 = (blockIdx.x - seg * ncta) * KC;
  const int kv = A.ncols - col0 < KC ? A.ncols - col0 : KC;  // valid columns of this CTA
  const int zlen = A.zr1 - A.zr0;
  const int z_lo = A.zr0 + static_cast<int>(static_cast<long long>(seg) * zlen / nseg);
  const int z_hi = A.zr0 + static_cast<int>(static_cast<long long>(seg + 1) * zlen / nseg);
  const int e0 = seg > 0 ? z_lo - 1 : z_lo;

  // the basis (plain contractions): cB[a][i] = B(a, i), cD likewise
  double cB[Q][N], cD[Q][N];
#pragma unroll
  for (int r = 0; r < Q; ++r)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int c = r;
      cB[r][i] = c < Q ? bs.B[c][i] : 0.0;
      cD[r][i] = c < Q ? bs.D[c][i] : 0.0;
    }

  // z-pencil role: pencil (zi, zj) of column kz
  const bool zrole = item < K::ZI;
  const int zit = zrole ? item : K::ZI - 1;
  const int kz = zit / (N * N), pz = zit % (N * N);
  const int zi = pz % N, zj = pz / N;
  const int col = col0 + kz;
  const bool zvalid = zrole && kz < kv;
  const int ex = col % A.nx, ey = col / A.nx;
  const int X = ex * P + zi, Y = ey * P + zj;
  const bool bcxy = CON && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1);
  const bool ring = zi == 0 || zi == P || zj == 0 || zj == P;
  const bool owner = ring_owner(P, zi, zj, ex, ey, A.nx, A.ny);
  const LatLayout L(P, A.nx, A.ny);
  bool lat_is_y = false;
  const long long lat0 = (ring && zvalid) ? lat_store_index(L, P, A.nx, ex, ey, zi, zj, 0, lat_is_y) : 0;
  double* lat = (lat_is_y ? A.lateral : A.lat_x) + lat0;
  const long long lat_stride = lat_is_y ? L.y_zstride : L.x_zstride;
  double carry = 0.0, dot = 0.0;

  // Staging: each column's factor block G_e is copied global -> shared by the
  // TMA bulk engine (one elected thread, mbarrier completion), issued as soon
  // as the previous element's phase X has consumed the buffer; the z-pencils
  // of u for element ez+1 are fetched by LDGSTS (cp.async) into the other half
  // of a double buffer while element ez computes. Neither costs registers.
  constexpr uint32_t gbytes = K::GS * 8;
  const uint32_t bar = smem_u32(smem + K::BAR_OFF);
  const long long gcol = static_cast<long long>(A.nz) * K::GS;  // doubles per column of G
  const double* Gcta = A.G + static_cast<long long>(col0) * gcol;
  if (t == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue_g = [&](int ez) {  // thread 0
    mbar_arrive_expect_tx(bar, gbytes * kv);
    for (int kk = 0; kk < kv; ++kk)
      bulk_g2s(smem_u32(smem + K::G_OFF + kk * K::GSM), Gcta + kk * gcol + ez * K::GS, gbytes, bar, pol);
  };
  if (t == 0) {
    issue_g(e0);
    if (e0 + 1 < z_hi)
      for (int kk = 0; kk < kv; ++kk) prefetch_l2_bulk(Gcta + kk * gcol + (e0 + 1) * K::GS, gbytes);
  }
  double* Uz = smem + K::U_OFF + kz * K::USTR + pz;  // this z-pencil's u staging (buffer 0)
  auto fetch_u = [&](int ez, int buf) {
    if (zvalid) {
#pragma unroll
      for (int r = 0; r < N; ++r) {
        const int k = r;
        if (k < N) {
          const long long node =
              X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * (ez * P + k));
          cp_async8(smem_u32(Uz + buf * N * N * N + k * N * N), A.u + node);
        }
      }
    }
    cp_async_commit();
  };
  fetch_u(e0, 0);

  for (int ez = e0; ez < z_hi; ++ez) {
    const int le = ez - e0;  // element index within the CTA (buffer / barrier parity)
    if (t == 0 && ez + 2 < z_hi)
      for (int kk = 0; kk < kv; ++kk) prefetch_l2_bulk(Gcta + kk * gcol + (ez + 2) * K::GS, gbytes);
    if (ez + 1 < z_hi) {
      fetch_u(ez + 1, (le + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }

    // ---------------- phase Z: gather the z-pencil, contract along z
    if (wfirst < K::ZI) {
      double* SA = smem + kz * K::CB;
      double uk[N];
      const double* us = Uz + (le & 1) * N * N * N;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int Z = ez * P + k;
        double v = us[k * N * N];
        if (CON && (bcxy || (Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi))) v = 0.0;
        uk[k] = v;
      }
      if constexpr (K::EO) {
        double e[NH], o[NH];
        eo_split(uk, e, o);
        if constexpr (COLLOC) {
#pragma unroll
          for (int c = 0; c < Q; ++c)
            if (zrole) SA[c * K::SA_CS + pz] = uk[c];
        } else {
          eo_fwd<1>(bs.eB, e, o, uk, [&](int c, double v) {
            if (zrole) SA[c * K::SA_CS + pz] = v;
          });
        }
        if constexpr (!MASS)
          eo_fwd<-1>(bs.eD, e, o, uk, [&](int c, double v) {
            if (zrole) SA[(Q + c) * K::SA_CS + pz] = v;
          });
      } else
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        const int c = r;
        double s0, s1 = 0.0;
        if constexpr (COLLOC) {
          s0 = uk[r];
        } else {
          s0 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) s0 = fma(cB[r][k], uk[k], s0);
        }
        if constexpr (!MASS) {
#pragma unroll
          for (int k = 0; k < N; ++k) s1 = fma(cD[r][k], uk[k], s1);
        }
        if (zrole && c < Q) {
          SA[c * K::SA_CS + pz] = s0;
          if constexpr (!MASS) SA[(Q + c) * K::SA_CS + pz] = s1;
        }
      }
    }
    __syncthreads();

    // ---------------- phase Y: y-pencils
    if (wfirst < K::YI) {
      const bool act = item < K::YI;
      const int it = act ? item : K::YI - 1;
      const int ky = it / (N * Q), rem = it % (N * Q);
      const int i = rem % N, c = rem / N;
      const double* SA = smem + ky * K::CB;
      double* SB = smem + ky * K::CB + K::SA_SIZE;
      double y0[N], y1[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        y0[j] = SA[c * K::SA_CS + j * N + i];
        if constexpr (!MASS) y1[j] = SA[(Q + c) * K::SA_CS + j * N + i];
      }
      double* sb = SB + i * K::SB_IS + c * Q;
      if constexpr (K::EO) {
        double e0[NH], o0[NH];
        eo_split(y0, e0, o0);
        if constexpr (COLLOC) {
#pragma unroll
          for (int b = 0; b < Q; ++b)
            if (act) {
              sb[b] = y0[b];
              sb[2 * N * K::SB_IS + b] = y1[b];
            }
        } else {
          eo_fwd<1>(bs.eB, e0, o0, y0, [&](int b, double v) {
            if (act) sb[b] = v;
          });
          if constexpr (!MASS) {
            double e1[NH], o1[NH];
            eo_split(y1, e1, o1);
            eo_fwd<1>(bs.eB, e1, o1, y1, [&](int b, double v) {
              if (act) sb[2 * N * K::SB_IS + b] = v;
            });
          }
        }
        if constexpr (!MASS)
          eo_fwd<-1>(bs.eD, e0, o0, y0, [&](int b, double v) {
            if (act) sb[N * K::SB_IS + b] = v;
          });
      } else
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        const int b = r;
        double bb = 0.0, db = 0.0, bd = 0.0;
        if constexpr (COLLOC) {
          bb = y0[r];
          bd = y1[r];
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) bb = fma(cB[r][j], y0[j], bb);
          if constexpr (!MASS) {
#pragma unroll
            for (int j = 0; j < N; ++j) bd = fma(cB[r][j], y1[j], bd);
          }
        }
        if constexpr (!MASS) {
#pragma unroll
          for (int j = 0; j < N; ++j) db = fma(cD[r][j], y0[j], db);
        }
        if (act && b < Q) {
          sb[b] = bb;
          if constexpr (!MASS) {
            sb[N * K::SB_IS + b] = db;
            sb[2 * N * K::SB_IS + b] = bd;
          }
        }
      }
    }
    __syncthreads();

    // ---------------- phase X: x-pencils, pointwise factors, back along x
    mbar_wait_parity(bar, le & 1);  // the G blocks have landed in shared memory
    if (wfirst < K::XI) {
      const bool act = item < K::XI;
      const int it = act ? item : K::XI - 1;
      const int kx = it / QQ, pp = it % QQ;
      double* SB = smem + kx * K::CB + K::SA_SIZE;
      const double* Ge = smem + K::G_OFF + kx * K::GSM;
      if constexpr (MASS && K::EO) {
        double x0[N], v[Q], out[N];
#pragma unroll
        for (int i = 0; i < N; ++i) x0[i] = SB[i * K::SB_IS + pp];
        double e[NH], o[NH];
        eo_split(x0, e, o);
        eo_fwd<1>(bs.eB, e, o, x0, [&](int a, double val) { v[a] = val * Ge[a * QQ + pp]; });
        eo_bwd<1, false>(bs.eB, v, out);
#pragma unroll
        for (int i = 0; i < N; ++i)
          if (act) SB[i * K::SB_IS + pp] = out[i];
      } else if constexpr (MASS) {
        double x0[N], v[Q];
#pragma unroll
        for (int i = 0; i < N; ++i) x0[i] = SB[i * K::SB_IS + pp];
#pragma unroll
        for (int r = 0; r < Q; ++r) {
          const int a = r;
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) acc = fma(cB[r][i], x0[i], acc);
          v[r] = a < Q ? acc * Ge[a * QQ + pp] : 0.0;
        }
        double o[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int r = 0; r < Q; ++r) acc = fma(cB[r][i], v[r], acc);
          o[i] = acc;
        }
#pragma unroll
        for (int r = 0; r < N; ++r)
          if (act) SB[r * K::SB_IS + pp] = o[r];
      } else {
        double gr[Q], gs[Q], gt[Q];
        if constexpr (K::EO) {
          double x0[N], x1[N], x2[N];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            x0[i] = SB[i * K::SB_IS + pp];
            x1[i] = SB[(N + i) * K::SB_IS + pp];
            x2[i] = SB[(2 * N + i) * K::SB_IS + pp];
          }
          double e[NH], o[NH];
          eo_split(x0, e, o);
          eo_fwd<-1>(bs.eD, e, o, x0, [&](int a, double v) { gr[a] = v; });
          if constexpr (COLLOC) {
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              gs[a] = x1[a];
              gt[a] = x2[a];
            }
          } else {
            eo_split(x1, e, o);
            eo_fwd<1>(bs.eB, e, o, x1, [&](int a, double v) { gs[a] = v; });
            eo_split(x2, e, o);
            eo_fwd<1>(bs.eB, e, o, x2, [&](int a, double v) { gt[a] = v; });
          }
        } else {
          double x0[N], x1[N], x2[N];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            x0[i] = SB[i * K::SB_IS + pp];
            x1[i] = SB[(N + i) * K::SB_IS + pp];
            x2[i] = SB[(2 * N + i) * K::SB_IS + pp];
          }
#pragma unroll
          for (int r = 0; r < Q; ++r) {
            double rr = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) rr = fma(cD[r][i], x0[i], rr);
            gr[r] = rr;
            if constexpr (COLLOC) {
              gs[r] = x1[r];
              gt[r] = x2[r];
            } else {
              double ss = 0.0, uu = 0.0;
#pragma unroll
              for (int i = 0; i < N; ++i) {
                ss = fma(cB[r][i], x1[i], ss);
                uu = fma(cB[r][i], x2[i], uu);
              }
              gs[r] = ss;
              gt[r] = uu;
            }
          }
        }
#pragma unroll
        for (int r = 0; r < Q; ++r) {
          const int a = r;
          const int ac = a < Q ? a : Q - 1;
          const double* g = Ge + ac * QQ + pp;
          const double g0 = g[0 * Q * QQ], g1 = g[1 * Q * QQ], g2 = g[2 * Q * QQ];
          const double g3 = g[3 * Q * QQ], g4 = g[4 * Q * QQ], g5 = g[5 * Q * QQ];
          const double rr = gr[r], ss = gs[r], uu = gt[r];
          gr[r] = g0 * rr + g1 * ss + g2 * uu;  // operator.hpp:129-131
          gs[r] = g1 * rr + g3 * ss + g4 * uu;
          gt[r] = g2 * rr + g4 * ss + g5 * uu;
        }
        // back along x, field by field (partials reduce-scattered over the pencil's lanes)
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          double part[N];
          if constexpr (K::EO) {
            if (f == 0) {
              eo_bwd<-1, false>(bs.eD, gr, part);
            } else if constexpr (COLLOC) {
#pragma unroll
              for (int i = 0; i < N; ++i) part[i] = f == 1 ? gs[i] : gt[i];
            } else {
              if (f == 1)
                eo_bwd<1, false>(bs.eB, gs, part);
              else
                eo_bwd<1, false>(bs.eB, gt, part);
            }
          } else
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double acc = 0.0;
            if (f == 0) {
#pragma unroll
              for (int r = 0; r < Q; ++r) acc = fma(cD[r][i], gr[r], acc);
            } else if constexpr (COLLOC) {
              acc = f == 1 ? gs[i] : gt[i];
            } else {
#pragma unroll
              for (int r = 0; r < Q; ++r) acc = fma(cB[r][i], f == 1 ? gs[r] : gt[r], acc);
            }
            part[i] = acc;
          }
          const double (&o)[N] = part;
#pragma unroll
          for (int r = 0; r < N; ++r)
            if (act) SB[(f * N + r) * K::SB_IS + pp] = o[r];
        }
      }
    }
    __syncthreads();
    if (t == 0 && ez + 1 < z_hi) {  // G buffers consumed: stream the next element's blocks
      fence_proxy_async();
      issue_g(ez + 1);
    }

    // ---------------- phase Y': back along y
    if (wfirst < K::YI) {
      const bool act = item < K::YI;
      const int it = act ? item : K::YI - 1;
      const int ky = it / (N * Q), rem = it % (N * Q);
      const int i = rem % N, c = rem / N;
      double* SA = smem + ky * K::CB;
      const double* sb = smem + ky * K::CB + K::SA_SIZE + i * K::SB_IS + c * Q;
      double a0[Q], a1[Q], a2[Q];
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        const int b = r;
        const int bc = b < Q ? b : Q - 1;  // past-the-end rows carry zero coefficients
        a0[r] = sb[bc];
        if constexpr (!MASS) {
          a1[r] = sb[N * K::SB_IS + bc];
          a2[r] = sb[2 * N * K::SB_IS + bc];
        }
      }
      double p1[N], p2[N];
      if constexpr (K::EO) {
        if constexpr (MASS) {
          eo_bwd<1, false>(bs.eB, a0, p1);
        } else if constexpr (COLLOC) {
#pragma unroll
          for (int j = 0; j < N; ++j) {
            p1[j] = a0[j];
            p2[j] = a2[j];
          }
          eo_bwd<-1, true>(bs.eD, a1, p1);
        } else {
          eo_bwd<1, false>(bs.eB, a0, p1);
          eo_bwd<-1, true>(bs.eD, a1, p1);
          eo_bwd<1, false>(bs.eB, a2, p2);
        }
      } else
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double c1 = 0.0, c2 = 0.0;
        if constexpr (MASS) {
#pragma unroll
          for (int r = 0; r < Q; ++r) c1 = fma(cB[r][j], a0[r], c1);
        } else if constexpr (COLLOC) {
          c1 = a0[j];
#pragma unroll
          for (int r = 0; r < Q; ++r) c1 = fma(cD[r][j], a1[r], c1);
          c2 = a2[j];
        } else {
#pragma unroll
          for (int r = 0; r < Q; ++r) {
            c1 = fma(cB[r][j], a0[r], c1);
            c2 = fma(cB[r][j], a2[r], c2);
          }
#pragma unroll
          for (int r = 0; r < Q; ++r) c1 = fma(cD[r][j], a1[r], c1);
        }
        p1[j] = c1;
        p2[j] = c2;
      }
      const double (&o1)[N] = p1;
      const double (&o2)[N] = p2;
#pragma unroll
      for (int r = 0; r < N; ++r) {
        const int j = r;
        if (act && j < N) {
          SA[c * K::SA_CS + j * N + i] = o1[r];
          if constexpr (!MASS) SA[(Q + c) * K::SA_CS + j * N + i] = o2[r];
        }
      }
    }
    __syncthreads();

    // ---------------- phase Z': back along z into the z-pencil
    if (wfirst < K::ZI) {
      const double* SA = smem + kz * K::CB;
      double c1[Q], c2[Q];
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        const int c = r;
        const int cc = c < Q ? c : Q - 1;
        c1[r] = SA[cc * K::SA_CS + pz];
        if constexpr (!MASS) c2[r] = SA[(Q + cc) * K::SA_CS + pz];
      }
      double part[N];
      if constexpr (K::EO) {
        if constexpr (COLLOC) {
#pragma unroll
          for (int k = 0; k < N; ++k) part[k] = c1[k];
        } else {
          eo_bwd<1, false>(bs.eB, c1, part);
        }
        if constexpr (!MASS) eo_bwd<-1, true>(bs.eD, c2, part);
      } else
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double acc = 0.0;
        if constexpr (COLLOC) {
          acc = c1[k];
        } else {
#pragma unroll
          for (int r = 0; r < Q; ++r) acc = fma(cB[r][k], c1[r], acc);
        }
        if constexpr (!MASS) {
#pragma unroll
          for (int r = 0; r < Q; ++r) acc = fma(cD[r][k], c2[r], acc);
        }
        part[k] = acc;
      }
      double (&out)[N] = part;

      // ---------------- transpose restriction, part 1 (see header)
      out[0] += carry;
      carry = out[P];  // the top plane is the next element's bottom plane
      const bool lo_share = RNG && A.carry_lo != nullptr && ez == A.zr0;   // range starts inside the slab
      const bool hi_share = RNG && A.carry_hi != nullptr && ez == A.zr1 - 1;  // range ends inside the slab
      const int kend = (ez == A.nz - 1 || hi_share) ? N : P;
      const double* usz = Uz + (le & 1) * N * N * N;  // u of this element, still staged
      const int kbeg = lo_share ? 1 : 0;
      const int kstop = hi_share ? P : kend;
      if (zvalid && ez >= z_lo) {
        if (lo_share) A.carry_lo[static_cast<long long>(col) * N * N + pz] = out[0];
        if (hi_share) A.carry_hi[static_cast<long long>(col) * N * N + pz] = out[P];
        if (!do_dot) {  // plain apply: the lean epilogue
#pragma unroll
          for (int r = 0; r < N; ++r) {
            const int k = r;
            if (k >= kbeg && k < kstop) {
              const int Z = ez * P + k;
              if (ring) {
                lat[Z * lat_stride] = out[r];
              } else {
                const long long node =
                    X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
                double v = out[r];
                if (CON && ((Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi))) v = usz[k * N * N];
                A.w[node] = v;
              }
            }
          }
        } else {
#pragma unroll
          for (int r = 0; r < N; ++r) {
            const int k = r;
            if (k >= kbeg && k < kstop) {
              const int Z = ez * P + k;
              const double uv = usz[k * N * N];
              const bool zbc = CON && ((Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi));
              if (ring) {
                lat[Z * lat_stride] = out[r];
                // column-local share of p.Ap on the ring (ring.cuh); w = u rows counted once
                if (bcxy || zbc)
                  dot = (owner && !(A.zlo_shared && Z == 0)) ? fma(uv, uv, dot) : dot;
                else
                  dot = fma(uv, out[r], dot);
              } else {
                const long long node =
                    X + static_cast<long long>(A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
                const double v = zbc ? uv : out[r];
                A.w[node] = v;
                dot = fma(uv, v, dot);
              }
            }
          }
        }
      }
    }
    __syncthreads();  // smem A and the u buffer are rewritten next element
  }
  const double cdot = do_dot ? block_sum<NT>(dot, s_red) : 0.0;
  ring_dot_finish<NT>(A, blockIdx.x, cdot, s_red);
}

// Thread-per-column element kernel for BP1 at p = 1, 2 (n = 2, 3; q = 3, 4):
// one thread marches one element column in z with the element in registers
// and no barrier per element (the CTA-per-column kernel above pays five per
// element, which dominates at small p). The sum factorisation streams so that
// only one (p+1) q^2 stage is live: per node plane k, x then y interpolation
// (t[k][b][a]); per quadrature row (b, a), z interpolation, the mass factor
// and z back into the same registers (t becomes r2); per node plane k, y then
// x back, the z-carry and the stores. Every contraction sums in the plain
// loop order, as the CTA kernel's plain form. z-segments as in
// bp_apply_kernel; ring partials in the same lateral layout, so the consumers
// are unchanged.
//
// STG: the next element's factor block and u planes are fetched by cp.async
// into a per-thread shared-memory slot while this element computes (no
// registers held by the loads in flight; the row a of the factors is
// re-filled as soon as it has been read). Slot strides are odd in 16-byte
// (factors) / 8-byte (u) units, so the per-lane accesses are conflict free.
constexpr int TPC_T = 128;

template <int P, int Q>
struct TpcSmem {
  static constexpr int N2 = (P + 1) * (P + 1);
  static constexpr int GS = (Q * Q * Q + 1) / 2 * 2;
  static constexpr int GSP = (GS / 2) % 2 ? GS : GS + 2;  // doubles per thread: factor block
  static constexpr int USP = (P * N2) | 1;                // doubles per thread: u planes 1..P
  static constexpr int BYTES = TPC_T * (GSP + USP) * 8;
};

__device__ __forceinline__ void cp_async16_cg(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <int P, int Q, int MB, int STG>
__global__ void __launch_bounds__(TPC_T, MB)
    tpc_mass_kernel(const __grid_constant__ ApplyArgs A, const __grid_constant__ BasisT<P, Q> bs, int nseg) {
  constexpr int N = P + 1, N2 = N * N, QQ = Q * Q, Q3 = QQ * Q;
  constexpr int GS = (Q3 + 1) / 2 * 2;
  constexpr bool GROW = QQ % 2 == 0;  // a row g[a][.] of the factors is 16-byte aligned: stream it by rows
  using S = TpcSmem<P, Q>;
  __shared__ double s_red[TPC_T / 32];
  extern __shared__ double tsm[];
  if (A.sc != nullptr && *(volatile int*)&A.sc->status != ST_RUNNING) return;
  const int ncta = (A.ncols + TPC_T - 1) / TPC_T;
  const int seg = blockIdx.x / ncta;
  const int col_raw = (blockIdx.x - seg * ncta) * TPC_T + threadIdx.x;
  const bool valid = col_raw < A.ncols;
  const int col = valid ? col_raw : A.ncols - 1;
  const int ex = col % A.nx, ey = col / A.nx;
  const int z_lo = static_cast<int>(static_cast<long long>(seg) * A.nz / nseg);
  const int z_hi = static_cast<int>(static_cast<long long>(seg + 1) * A.nz / nseg);
  const int e0 = seg > 0 ? z_lo - 1 : z_lo;
  const bool do_dot = A.col_dot != nullptr;
  const long long plane = static_cast<long long>(A.Nx) * A.Ny;
  const long long base = ex * P + static_cast<long long>(A.Nx) * (ey * P);
  const LatLayout L(P, A.nx, A.ny);
  const double* Gcol = A.G + static_cast<long long>(col) * A.nz * GS;

  auto bcxy = [&](int i, int j) {
    const int X = ex * P + i, Y = ey * P + j;
    return A.constrained && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1);
  };
  auto zbc = [&](int Z) { return A.constrained && ((Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi)); };
  double uraw[N][N2];  // this element's u (unmasked), planes k = 0..P
  auto load_plane = [&](int k, int Z) {
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) uraw[k][j * N + i] = A.u[base + i + static_cast<long long>(A.Nx) * j + plane * Z];
  };
  double carry[N2];
#pragma unroll
  for (int l = 0; l < N2; ++l) carry[l] = 0.0;
  double dot = 0.0;
  double* gslot = tsm + threadIdx.x * S::GSP;
  double* uslot = tsm + TPC_T * S::GSP + threadIdx.x * S::USP;
  auto issue_u = [&](int ez) {  // planes 1..P of element ez
#pragma unroll
    for (int k = 1; k < N; ++k)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i)
          cp_async8(smem_u32(uslot + (k - 1) * N2 + j * N + i),
                    A.u + base + i + static_cast<long long>(A.Nx) * j + plane * (ez * P + k));
  };
  auto issue_g = [&](int ez, int a) {  // row a of element ez's factors (the whole block if !GROW)
    constexpr int n16 = GROW ? QQ / 2 : GS / 2;
    const double* src = Gcol + static_cast<long long>(ez) * GS + (GROW ? a * QQ : 0);
    double* dst = gslot + (GROW ? a * QQ : 0);
#pragma unroll
    for (int m = 0; m < n16; ++m) cp_async16_cg(smem_u32(dst + 2 * m), src + 2 * m);
  };
  load_plane(0, e0 * P);
  if constexpr (STG) {  // groups in flight, in order: U(ez), G(ez) at the top of element ez
    issue_u(e0);
    cp_async_commit();
#pragma unroll
    for (int a = 0; a < (GROW ? Q : 1); ++a) issue_g(e0, a);
    cp_async_commit();
  }
  for (int ez = e0; ez < z_hi; ++ez) {
    const bool nxt = ez + 1 < z_hi;
    if constexpr (STG) {
      cp_async_wait<1>();  // U(ez) has landed
#pragma unroll
      for (int k = 1; k < N; ++k)
#pragma unroll
        for (int l = 0; l < N2; ++l) uraw[k][l] = uslot[(k - 1) * N2 + l];
      if (nxt) issue_u(ez + 1);
      cp_async_commit();
    } else {
#pragma unroll
      for (int k = 1; k < N; ++k) load_plane(k, ez * P + k);
    }
    const double* ge = Gcol + static_cast<long long>(ez) * GS;
    double g[GROW ? 1 : GS];  // the whole block when its rows are not 16-byte aligned (p = 1)
    if constexpr (!GROW && !STG) {  // issued before the forward contractions, which cover its latency
#pragma unroll
      for (int m = 0; m < GS / 2; ++m) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(ge) + m);
        g[2 * m] = v.x;
        g[2 * m + 1] = v.y;
      }
    }
    // per node plane: masked input (ConstrainedOperator: P u), x then y interpolation
    double t[N][Q][Q];  // [k][b][a]
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double u[N2];
#pragma unroll
      for (int l = 0; l < N2; ++l) u[l] = (bcxy(l % N, l / N) || zbc(ez * P + k)) ? 0.0 : uraw[k][l];
      double t1[N][Q];  // [j][a]
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) s = fma(bs.B[a][i], u[j * N + i], s);
          t1[j][a] = s;
        }
#pragma unroll
      for (int b = 0; b < Q; ++b)
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) s = fma(bs.B[b][j], t1[j][a], s);
          t[k][b][a] = s;
        }
    }
    if constexpr (STG) cp_async_wait<1>();  // G(ez) has landed (U(ez + 1) may not have)
    if constexpr (!GROW && STG) {
#pragma unroll
      for (int m = 0; m < GS / 2; ++m) {
        const double2 v = reinterpret_cast<const double2*>(gslot)[m];
        g[2 * m] = v.x;
        g[2 * m + 1] = v.y;
      }
      if (nxt) issue_g(ez + 1, 0);
    }
    // per quadrature row (b, a): z interpolation, times the mass factor
    // (operator.hpp:139-142; device layout g[a][b + q c], setup.cu), z back
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      double gr[GROW ? QQ : 1];
      if constexpr (GROW) {
#pragma unroll
        for (int m = 0; m < QQ / 2; ++m) {
          const double2 v = STG ? reinterpret_cast<const double2*>(gslot + a * QQ)[m]
                                : __ldg(reinterpret_cast<const double2*>(ge + a * QQ) + m);
          gr[2 * m] = v.x;
          gr[2 * m + 1] = v.y;
        }
        if (STG && nxt) issue_g(ez + 1, a);  // the row has been read: refill it with the next element's
      }
#pragma unroll
      for (int b = 0; b < Q; ++b) {
        double v[Q];
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) s = fma(bs.B[c][k], t[k][b][a], s);
          v[c] = s * (GROW ? gr[b + Q * c] : g[a * QQ + b + Q * c]);
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < Q; ++c) s = fma(bs.B[c][k], v[c], s);
          t[k][b][a] = s;
        }
      }
    }
    if constexpr (STG) cp_async_commit();
    // per node plane: y then x back, z-carry, transpose restriction part 1
    // (every footprint node but the p = 2 centre is a ring node)
    const int kend = (ez == A.nz - 1) ? N : P;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double r1[N][Q];  // [j][a]
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < Q; ++b) s = fma(bs.B[b][j], t[k][b][a], s);
          r1[j][a] = s;
        }
      double o[N2];
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < Q; ++a) s = fma(bs.B[a][i], r1[j][a], s);
          o[j * N + i] = s;
        }
      if (k == 0) {
#pragma unroll
        for (int l = 0; l < N2; ++l) o[l] += carry[l];
      }
      if (k == P) {  // the top plane is the next element's bottom plane
#pragma unroll
        for (int l = 0; l < N2; ++l) carry[l] = o[l];
      }
      if (valid && ez >= z_lo && k < kend) {
        const int Z = ez * P + k;
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int i = 0; i < N; ++i) {
            const int l = j * N + i;
            const bool ring = i == 0 || i == P || j == 0 || j == P;
            const double val = o[l];
            if (ring) {
              bool is_y = false;
              const long long li = lat_store_index(L, P, A.nx, ex, ey, i, j, Z, is_y);
              (is_y ? A.lateral : A.lat_x)[li] = val;
              if (do_dot) {
                const double uv = uraw[k][l];
                if (bcxy(i, j) || zbc(Z)) {
                  if (ring_owner(P, i, j, ex, ey, A.nx, A.ny) && !(A.zlo_shared && Z == 0)) dot = fma(uv, uv, dot);
                } else {
                  dot = fma(uv, val, dot);
                }
              }
            } else {
              const long long node = base + i + static_cast<long long>(A.Nx) * j + plane * Z;
              const double w = zbc(Z) ? uraw[k][l] : val;
              A.w[node] = w;
              if (do_dot) dot = fma(uraw[k][l], w, dot);
            }
          }
      }
    }
    // the top input plane is the next element's bottom plane
#pragma unroll
    for (int l = 0; l < N2; ++l) uraw[0][l] = uraw[P][l];
  }
  const double cdot = do_dot ? block_sum<TPC_T>(dot, s_red) : 0.0;
  ring_dot_finish<TPC_T>(A, blockIdx.x, cdot, s_red);
}

// Thread-per-column kernel for BP5 at p = 1 (n = q = 2, GLL collocation:
// the interpolation is the identity, operator.hpp:55): one thread marches one
// element column; per element the 8 nodes, the three derivatives at the 8
// points (2-term sums), the factors (48 doubles, 16-byte loads issued before
// the derivatives), the fluxes and the transposed derivatives -- no shared
// memory, no barrier. Layout, z-carry, ring partials and p.Ap as
// tpc_mass_kernel.
template <int MB>
__global__ void __launch_bounds__(TPC_T, MB)
    tpc_colloc_p1_kernel(const __grid_constant__ ApplyArgs A, const __grid_constant__ BasisT<1, 2> bs, int nseg) {
  constexpr int P = 1, N = 2, N2 = 4, Q = 2, Q3 = 8, GS = 6 * Q3;
  __shared__ double s_red[TPC_T / 32];
  if (A.sc != nullptr && *(volatile int*)&A.sc->status != ST_RUNNING) return;
  const int ncta = (A.ncols + TPC_T - 1) / TPC_T;
  const int seg = blockIdx.x / ncta;
  const int col_raw = (blockIdx.x - seg * ncta) * TPC_T + threadIdx.x;
  const bool valid = col_raw < A.ncols;
  const int col = valid ? col_raw : A.ncols - 1;
  const int ex = col % A.nx, ey = col / A.nx;
  const int z_lo = static_cast<int>(static_cast<long long>(seg) * A.nz / nseg);
  const int z_hi = static_cast<int>(static_cast<long long>(seg + 1) * A.nz / nseg);
  const int e0 = seg > 0 ? z_lo - 1 : z_lo;
  const bool do_dot = A.col_dot != nullptr;
  const long long plane = static_cast<long long>(A.Nx) * A.Ny;
  const long long base = ex * P + static_cast<long long>(A.Nx) * (ey * P);
  const LatLayout L(P, A.nx, A.ny);
  const double* Gcol = A.G + static_cast<long long>(col) * A.nz * GS;
  const double D00 = bs.D[0][0], D01 = bs.D[0][1], D10 = bs.D[1][0], D11 = bs.D[1][1];
  auto d2 = [&](int a, double x0, double x1) { return a == 0 ? fma(D01, x1, D00 * x0) : fma(D11, x1, D10 * x0); };

  auto bcxy = [&](int i, int j) {
    const int X = ex * P + i, Y = ey * P + j;
    return A.constrained && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1);
  };
  auto zbc = [&](int Z) { return A.constrained && ((Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi)); };
  double uraw[N][N2];  // [k][j * 2 + i]
  auto load_plane = [&](int k, int Z) {
#pragma unroll
    for (int l = 0; l < N2; ++l) uraw[k][l] = A.u[base + (l & 1) + static_cast<long long>(A.Nx) * (l >> 1) + plane * Z];
  };
  double carry[N2] = {0.0, 0.0, 0.0, 0.0};
  double dot = 0.0;
  load_plane(0, e0 * P);
  for (int ez = e0; ez < z_hi; ++ez) {
    load_plane(1, ez * P + 1);
    double g[GS];
    const double2* gp = reinterpret_cast<const double2*>(Gcol + static_cast<long long>(ez) * GS);
#pragma unroll
    for (int m = 0; m < GS / 2; ++m) {
      const double2 v = __ldg(gp + m);
      g[2 * m] = v.x;
      g[2 * m + 1] = v.y;
    }
    double u[N][N2];  // ConstrainedOperator: P u
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int l = 0; l < N2; ++l) u[k][l] = (bcxy(l & 1, l >> 1) || zbc(ez * P + k)) ? 0.0 : uraw[k][l];
    // fluxes at the points (a, b, c) = nodes (i, j, k): G (gr, gs, gt), operator.hpp:129-131
    double fr[N][N2], fs[N][N2], ft[N][N2];
#pragma unroll
    for (int c = 0; c < Q; ++c)
#pragma unroll
      for (int b = 0; b < Q; ++b)
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          const double gr = d2(a, u[c][b * 2], u[c][b * 2 + 1]);
          const double gs = d2(b, u[c][a], u[c][2 + a]);
          const double gt = d2(c, u[0][b * 2 + a], u[1][b * 2 + a]);
          const double* ge = g + a * Q * Q + b + Q * c;  // component m at ge[m Q^3] (setup.cu)
          const double g0 = ge[0], g1 = ge[Q3], g2 = ge[2 * Q3], g3 = ge[3 * Q3], g4 = ge[4 * Q3], g5 = ge[5 * Q3];
          fr[c][b * 2 + a] = g0 * gr + g1 * gs + g2 * gt;
          fs[c][b * 2 + a] = g1 * gr + g3 * gs + g4 * gt;
          ft[c][b * 2 + a] = g2 * gr + g4 * gs + g5 * gt;
        }
    // transposed derivatives: out = Dx^T fr + Dy^T fs + Dz^T ft
    double o[N][N2];
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = fma(bs.D[1][i], fr[k][j * 2 + 1], bs.D[0][i] * fr[k][j * 2]);
          s = fma(bs.D[0][j], fs[k][i], s);
          s = fma(bs.D[1][j], fs[k][2 + i], s);
          s = fma(bs.D[0][k], ft[0][j * 2 + i], s);
          s = fma(bs.D[1][k], ft[1][j * 2 + i], s);
          o[k][j * 2 + i] = s;
        }
#pragma unroll
    for (int l = 0; l < N2; ++l) {
      o[0][l] += carry[l];
      carry[l] = o[P][l];
    }
    const int kend = (ez == A.nz - 1) ? N : P;
    if (valid && ez >= z_lo) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        if (k < kend) {
          const int Z = ez * P + k;
#pragma unroll
          for (int l = 0; l < N2; ++l) {  // every p = 1 footprint node is a ring node
            const int i = l & 1, j = l >> 1;
            bool is_y = false;
            const long long li = lat_store_index(L, P, A.nx, ex, ey, i, j, Z, is_y);
            (is_y ? A.lateral : A.lat_x)[li] = o[k][l];
            if (do_dot) {
              const double uv = uraw[k][l];
              if (bcxy(i, j) || zbc(Z)) {
                if (ring_owner(P, i, j, ex, ey, A.nx, A.ny) && !(A.zlo_shared && Z == 0)) dot = fma(uv, uv, dot);
              } else {
                dot = fma(uv, o[k][l], dot);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int l = 0; l < N2; ++l) uraw[0][l] = uraw[P][l];
  }
  const double cdot = do_dot ? block_sum<TPC_T>(dot, s_red) : 0.0;
  ring_dot_finish<TPC_T>(A, blockIdx.x, cdot, s_red);
}

// Transpose restriction, part 2, for plain applies: every ring node sums its
// 1-4 column partials in ascending column order (ring.cuh). (CG fuses this
// into its r-update, cg.cu; p.Ap is complete after part 1.)
constexpr int FT = 256;

__global__ void __launch_bounds__(FT) lateral_fixup_kernel(const __grid_constant__ ApplyArgs A, int P, int z_begin,
                                                          int z_end) {
  // one warp per node row (Y, Z): ring rows (Y % P == 0) finish every node,
  // other rows their x-face nodes X = fx*P
  const LatLayout L(P, A.nx, A.ny);
  const int lane = threadIdx.x & 31;
  const long long rows = static_cast<long long>(A.Ny) * (z_end - z_begin);
  for (long long rr = blockIdx.x * (FT / 32) + (threadIdx.x >> 5); rr < rows;
       rr += static_cast<long long>(gridDim.x) * (FT / 32)) {
    const long long row = rr + static_cast<long long>(A.Ny) * z_begin;
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

template <int P, int Q, int KIND, int SK>
void* kernel_ptr() {
  static std::atomic<uint64_t> configured{0};  // > 48 KB dynamic shared memory, per device
  set_smem_attr_once(configured, reinterpret_cast<const void*>(&bp_apply_kernel<P, Q, KIND, SK>),
                     Cfg<P, Q, KIND, SK>::SMEM_BYTES);
  return reinterpret_cast<void*>(&bp_apply_kernel<P, Q, KIND, SK>);
}

// the SK code in use for (kind, p): the default; sweep builds (tools/sk_sweep.py)
// read HEXBP_SK_<kind>_<p> at every launch to select one of their compiled candidates
int sk_select(int kind, int p, int dflt) {
#ifdef HX_SK_SWEEP
  char name[32];
  std::snprintf(name, sizeof(name), "HEXBP_SK_%d_%d", kind, p);
  if (const char* v = std::getenv(name)) return std::atoi(v);
#else
  (void)kind;
  (void)p;
#endif
  return dflt;
}

// z-segments per element column: enough CTAs for `waves` full waves of the
// resident slots (148 SMs x occupancy), segments of at least `min_len`
// elements (each segment recomputes one element). HEXBP_SEG_WAVES /
// HEXBP_SEG_MIN override (dev A/B).
int z_segments(int ncta, int occ, int nz) {
  static int sms = 0;
  static double waves = 2.0;
  static int min_len = 4;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
    if (const char* v = std::getenv("HEXBP_SEG_WAVES")) waves = std::atof(v);
    if (const char* v = std::getenv("HEXBP_SEG_MIN")) min_len = std::atoi(v) > 0 ? std::atoi(v) : 1;
  }
  const double want = waves * sms * occ;
  if (ncta >= want) return 1;
  int nseg = static_cast<int>((want + ncta - 1) / ncta);
  const int cap = nz / min_len > 1 ? nz / min_len : 1;
  return nseg < cap ? nseg : cap;
}

struct KInfo {
  void* fn;
  int nt;
  int smem;
  int cols;  // element columns per CTA
};

template <int P, int Q, int KIND, int I = 0>
KInfo info_sel(int sk) {
  using L = SkList<KIND, P>;
  if constexpr (I < L::n) {
    constexpr int c = L::v[I];
    if constexpr (c / 1000000 % 10 && KIND == KIND_COLLOC) {  // thread-per-column kernel, BP5 p = 1
      if (sk == c) return {reinterpret_cast<void*>(&tpc_colloc_p1_kernel<c / 10 % 10>), TPC_T, 0, TPC_T};
    } else if constexpr (c / 1000000 % 10) {  // thread-per-column kernel
      if (sk == c) return {reinterpret_cast<void*>(&tpc_mass_kernel<P, Q, c / 10 % 10, c / 100 % 10>), TPC_T,
                              c / 100 % 10 ? TpcSmem<P, Q>::BYTES : 0, TPC_T};
    } else {
      using K = Cfg<P, Q, KIND, c>;
      if (sk == c) return {kernel_ptr<P, Q, KIND, c>(), K::NT, K::SMEM_BYTES, K::KC};
    }
    return info_sel<P, Q, KIND, I + 1>(sk);
  } else {
    return {nullptr, 0, 0, 1};
  }
}

template <int P, int KIND>
KInfo info_t() {
  constexpr int Q = KIND == KIND_COLLOC ? P + 1 : P + 2;
  return info_sel<P, Q, KIND>(sk_select(KIND, P, SkList<KIND, P>::v[0]));
}

template <int N, int Q>
void fill_eo(const double (&M)[Q][N], EOB<N, Q>& e) {
  constexpr int NH = N / 2, QH = Q / 2;
  for (int a = 0; a < QH; ++a) {
    for (int i = 0; i < NH; ++i) {
      e.P[a][i] = 0.5 * (M[a][i] + M[a][N - 1 - i]);
      e.R[a][i] = 0.5 * (M[a][i] - M[a][N - 1 - i]);
    }
    e.col[a] = (N & 1) ? M[a][NH] : 0.0;
  }
  for (int i = 0; i < NH; ++i) e.row[i] = (Q & 1) ? M[QH][i] : 0.0;
  e.ctr = ((N & 1) && (Q & 1)) ? M[QH][NH] : 0.0;
}

template <int P, int Q, int KIND, int SK>
cudaError_t launch_tpc(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  static_assert((KIND == KIND_MASS && P <= 2) || (KIND == KIND_COLLOC && P == 1),
                "thread-per-column kernels: BP1 p = 1, 2; BP5 p = 1");
  BasisT<P, Q> bs;
  for (int i = 0; i < Q; ++i)
    for (int j = 0; j <= P; ++j) {
      bs.B[i][j] = s.B[i * (P + 1) + j];
      bs.D[i][j] = s.D[i * (P + 1) + j];
    }
  static int occ = 0;
  constexpr int MB = SK / 10 % 10;   // min CTAs per SM (register cap)
  if constexpr (KIND == KIND_COLLOC) {
    if (occ == 0 &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tpc_colloc_p1_kernel<MB>, TPC_T, 0) != cudaSuccess)
      occ = 1;
    const int ncta = (a.ncols + TPC_T - 1) / TPC_T;
    const int nseg = z_segments(ncta, occ, a.nz);
    tpc_colloc_p1_kernel<MB><<<ncta * nseg, TPC_T, 0, st>>>(a, bs, nseg);
    return cudaGetLastError();
  } else {
  constexpr int STG = SK / 100 % 10;  // cp.async staging of the next element (TpcSmem)
  constexpr int SMEM = STG ? TpcSmem<P, Q>::BYTES : 0;
  static std::atomic<uint64_t> configured{0};
  if (STG) set_smem_attr_once(configured, reinterpret_cast<const void*>(&tpc_mass_kernel<P, Q, MB, STG>), SMEM);
  if (occ == 0 &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tpc_mass_kernel<P, Q, MB, STG>, TPC_T, SMEM) != cudaSuccess)
    occ = 1;
  const int ncta = (a.ncols + TPC_T - 1) / TPC_T;
  const int nseg = z_segments(ncta, occ, a.nz);
  tpc_mass_kernel<P, Q, MB, STG><<<ncta * nseg, TPC_T, SMEM, st>>>(a, bs, nseg);
  return cudaGetLastError();
  }
}

template <int P, int Q, int KIND, int SK>
cudaError_t launch_t(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  if constexpr (SK / 1000000 % 10) return launch_tpc<P, Q, KIND, SK>(s, a, st);
  else {
  using K = Cfg<P, Q, KIND, SK>;
  kernel_ptr<P, Q, KIND, SK>();
  if (s.gstride != K::GS) return cudaErrorInvalidValue;
  BasisT<P, Q> bs;
  for (int i = 0; i < Q; ++i)
    for (int j = 0; j <= P; ++j) {
      bs.B[i][j] = s.B[i * (P + 1) + j];
      bs.D[i][j] = s.D[i * (P + 1) + j];
    }
  fill_eo(bs.B, bs.eB);
  fill_eo(bs.D, bs.eD);
  static int occ = 0;  // resident CTAs per SM, once per instantiation
  if (occ == 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bp_apply_kernel<P, Q, KIND, SK>, K::NT,
                                                                K::SMEM_BYTES) != cudaSuccess)
    occ = 1;
  const int ncta = (a.ncols + K::KC - 1) / K::KC;
  int nseg = z_segments(ncta, occ, a.zr1 - a.zr0);
  // a sub-range launch (overlap.cu) has ncols column-partial slots: at most KC segments
  if ((a.zr0 != 0 || a.zr1 != a.nz) && nseg > K::KC) nseg = K::KC;
  const int f = (a.constrained ? 1 : 0) + (a.col_dot != nullptr ? 2 : 0) +
                (a.carry_lo != nullptr || a.carry_hi != nullptr ? 4 : 0);
  switch (f) {
#define HXB_F(FF)                                                                                   \
  case FF: {                                                                                        \
    static std::atomic<uint64_t> cfg{0};                                                            \
    set_smem_attr_once(cfg, reinterpret_cast<const void*>(&bp_apply_kernel<P, Q, KIND, SK, FF>),    \
                       K::SMEM_BYTES);                                                              \
    bp_apply_kernel<P, Q, KIND, SK, FF><<<ncta * nseg, K::NT, K::SMEM_BYTES, st>>>(a, bs, nseg);    \
    break;                                                                                          \
  }
    HXB_F(0)
    HXB_F(1)
    HXB_F(2)
    HXB_F(3)
    HXB_F(4)
    HXB_F(5)
    HXB_F(6)
    HXB_F(7)
#undef HXB_F
  }
  return cudaGetLastError();
  }
}

template <int P, int Q, int KIND, int I = 0>
cudaError_t launch_sel(int sk, const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  using L = SkList<KIND, P>;
  if constexpr (I < L::n) {
    if (sk == L::v[I]) return launch_t<P, Q, KIND, L::v[I]>(s, a, st);
    return launch_sel<P, Q, KIND, I + 1>(sk, s, a, st);
  } else {
    return cudaErrorInvalidValue;  // code not compiled in
  }
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
  return {nullptr, 0, 0, 1};
}

KInfo info_for(const Setup& s) {
  switch (s.kind) {
    case KIND_MASS: return info_k<KIND_MASS>(s.p);
    case KIND_DIFF: return info_k<KIND_DIFF>(s.p);
    case KIND_COLLOC: return info_k<KIND_COLLOC>(s.p);
  }
  return {nullptr, 0, 0, 1};
}

template <int P, int KIND>
cudaError_t launch_p(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  constexpr int Q = KIND == KIND_COLLOC ? P + 1 : P + 2;
  return launch_sel<P, Q, KIND>(sk_select(KIND, P, SkList<KIND, P>::v[0]), s, a, st);
}

template <int KIND>
cudaError_t launch_k(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  switch (s.p) {
    case 1: return launch_p<1, KIND>(s, a, st);
    case 2: return launch_p<2, KIND>(s, a, st);
    case 3: return launch_p<3, KIND>(s, a, st);
    case 4: return launch_p<4, KIND>(s, a, st);
    case 5: return launch_p<5, KIND>(s, a, st);
    case 6: return launch_p<6, KIND>(s, a, st);
    case 7: return launch_p<7, KIND>(s, a, st);
    case 8: return launch_p<8, KIND>(s, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// Element ranges (ApplyArgs::zr0 / zr1, carry_lo / carry_hi) in the DFMA
// element kernel: every degree but the thread-per-column BP1 p = 1, 2, BP5 p = 1.
bool dfma_ranges_supported(const Setup& s) {
  const KInfo ki = info_for(s);
  return ki.fn != nullptr && ki.cols != TPC_T;
}

cudaError_t launch_apply_dfma(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  switch (s.kind) {
    case KIND_MASS: return launch_k<KIND_MASS>(s, a, st);
    case KIND_DIFF: return launch_k<KIND_DIFF>(s, a, st);
    case KIND_COLLOC: return launch_k<KIND_COLLOC>(s, a, st);
  }
  return cudaErrorInvalidValue;
}

int fixup_grid(const Setup& s) {
  const long long P = s.p;
  const long long nx = s.dims[0], ny = s.dims[1];
  const long long per_plane = (ny + 1) * (nx * P + 1) + (nx + 1) * ny * (P - 1);
  const long long total = per_plane * (s.dims[2] * P + 1);
  long long g = (total + FT - 1) / FT;
  if (g > 148 * 8) g = 148 * 8;
  return static_cast<int>(g < 1 ? 1 : g);
}

// DMMA kernels for the setups whose factors are laid out for them (Setup::g_aos,
// chosen at setup; HEXBP_NO_DMMA=1 there selects the DFMA layout for A/B runs).
bool use_mma(const Setup& s) {
  return (s.g_aos == 1 && mma_kernel_applies(s)) || (s.g_aos == 2 && mma5_kernel_applies(s));
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
  if (ki.fn == nullptr) {  // generic degree (multipass pipeline): no single element kernel
    *regs = *smem = *threads = *blocks_per_sm = 0;
    return;
  }
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, ki.fn);
  *regs = fa.numRegs;
  *smem = static_cast<int>(fa.sharedSizeBytes) + ki.smem;
  *threads = ki.nt;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, ki.fn, ki.nt, ki.smem);
}

ApplyArgs make_apply_args(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                          double* dot_out, DevScalars* sc) {
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
  a.zlo_shared = s.z0 > 0;
  a.zr0 = 0;
  a.zr1 = s.dims[2];
  if (ws.pt != nullptr && u == ws.pt) {  // the fast CG's row-pitched search direction (tma.cu)
    a.u_pitch = ws.pt_pitch;
    a.u_tmap = tma_u_staging_enabled() ? &ws.pt_map : nullptr;
  }
  if (ws.Apt != nullptr && w == ws.Apt) a.w_pitch = ws.pt_pitch;  // its row-pitched A p
  return a;
}

cudaError_t launch_apply(const Setup& s, const Workspace& ws, const double* u, double* w, int constrained,
                         double* dot_out, DevScalars* sc, cudaStream_t st, bool finish_ring) {
  const ApplyArgs a = make_apply_args(s, ws, u, w, constrained, dot_out, sc);
  if (ws.multipass) {  // Backend::Multipass analog (reference arithmetic; CG reduces in cg.cu)
    if (dot_out || sc) return cudaErrorInvalidValue;
    return launch_apply_multipass(s, ws.mp_buf, u, w, constrained, st);
  }
  if (ws.exact && !ws.fast_op) {
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
  lateral_fixup_kernel<<<ws.fixup_grid, FT, 0, st>>>(a, s.p, 0, a.Nz);
  return cudaGetLastError();
}

cudaError_t launch_lateral_fixup_planes(const Setup& s, const Workspace& ws, const double* u, double* w,
                                        int constrained, int z_begin, int z_end, cudaStream_t st) {
  ApplyArgs a{};
  a.u = u;
  a.w = w;
  a.nx = s.dims[0];
  a.ny = s.dims[1];
  a.nz = s.dims[2];
  a.Nx = s.dims[0] * s.p + 1;
  a.Ny = s.dims[1] * s.p + 1;
  a.Nz = s.dims[2] * s.p + 1;
  a.constrained = constrained;
  a.bc_zlo = s.bc_zlo;
  a.bc_zhi = s.bc_zhi;
  a.lateral = ws.lateral;
  a.lat_x = ws.lateral + LatLayout(s.p, s.dims[0], s.dims[1]).y_zstride * (s.dims[2] * s.p + 1);
  const long long rows = static_cast<long long>(a.Ny) * (z_end - z_begin);
  long long g = (rows + FT / 32 - 1) / (FT / 32);
  if (g > 148 * 8) g = 148 * 8;
  lateral_fixup_kernel<<<static_cast<int>(g < 1 ? 1 : g), FT, 0, st>>>(a, s.p, z_begin, z_end);
  return cudaGetLastError();
}

}  // namespace hxb
