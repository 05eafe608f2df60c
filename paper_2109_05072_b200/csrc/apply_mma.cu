// FP64 tensor-core (DMMA) operator kernel for the BP3 headline degree
// (p = 7: n = 8 nodes, q = 9 Gauss points per direction) -- fast mode.
//
// Why DMMA: the DFMA kernel (apply.cu) is issue-bound at p = 7 -- every
// warp-wide DFMA needs its basis coefficient staged through a uniform
// register (LDCU), so coefficient loads cost as many issue slots as the
// FMAs, and the kernel issues ~9000 warp instructions per element. An
// m8n8k4 f64 MMA does 256 FMAs per instruction with the basis fragment held
// in registers for the whole kernel: ~300 MMAs per element replace ~3300
// DFMAs and their ~2700 coefficient loads. B200's DMMA rate equals its DFMA
// rate (64 FMA/clk/SM measured, tools/micro/fp64_peak.cu), so the win is the
// instruction stream, not the FLOP rate.
//
// Shapes. Each 1D contraction Y[m][r] = sum_k M[m][k] X[k][r] runs as MMAs
// with A = basis tile (8 x 4, registers), B = 8 "pencils" of X (4 x 8,
// one LDS per lane), C = 8 x 8 outputs. The 9th Gauss point does not fit an
// 8-row tile: forward (q = 9 outputs) its row is a 2-term dot per lane plus
// a 4-lane butterfly; backward (q = 9 inputs) its column is one DFMA per
// output. Staging: G by a TMA bulk copy per element; u by one TMA tensor
// copy per element in the fast CG (row-pitched search direction, tma.cu) or
// cp.async on caller vectors. The phases and the atomic-free transpose
// restriction are those of apply.cu:
//   Z : 8 pencil groups (j)      u        -> B_z u, D_z u          (+ row 8)
//   Y : 9 groups (c)             -> B_y B_z u, D_y B_z u, B_y D_z u (+ row 8)
//   X : 11 groups of (b,c) lines -> gr, gs, gt; G; D_x^T, B_x^T   (+ row/col 8)
//       in the transposed MMA form (data as the A operand), so the forward
//       C fragment is directly the A fragment of the backward MMA (k-slot t
//       <-> a = 2t, 2t+1): no transpose between the two x contractions
//   Y': 9 groups (c)             -> C1 = B_y^T A1 + D_y^T A2, C2 = B_y^T A3
//   Z': 8 groups (j)             -> out = B_z^T C1 + D_z^T C2     -> scatter
// The phases of consecutive elements are software-pipelined into two barrier
// intervals per element (see the schedule at the end of the kernel).
// Shared-memory layouts are [field][k][pencil] with strides / XOR swizzles
// chosen so that the B-fragment loads (k = lane%4 (+4), pencil = lane/4) and
// the 16-byte C-fragment stores are bank-conflict free.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_util.cuh"
#include "internal.h"
#include "ring.cuh"

namespace hxb {
namespace {

constexpr int P = 7, N = 8, Q = 9, QQ = 81;
// Phase X (the heaviest, 11 pencil groups) runs one group per warp on warps
// 0..10; a 12th warp takes five of the eight Z items of interval A off them
// (12 warps x 80 registers still fit two CTAs per SM).
constexpr int NXW = 11;
constexpr int NW = 12, NT = NW * 32;
constexpr int GSE = (6 * Q * Q * Q + 1) / 2 * 2;  // element block of G (== Setup::gstride)
// shared-memory layout (doubles)
// u staging, [k][j][i]. cp.async path: rows of 8, k-stride 68 (conflict-free
// phase-Z loads). TMA path: the tensor copy's dense box in 128-byte aligned
// buffers. A box row must start 16-byte aligned in global memory, so the box
// is 10 wide from the even x at or below the element's first node and the
// element sits at x offset ex & 1 of every row (the pitch is even). (A box
// two rows deeper -- k-stride 100 = 4 mod 16, conflict-free phase-Z / Z'
// loads -- measured 1% slower: more staging traffic and spills.)
template <bool TMA> constexpr int us_rs() { return TMA ? N + 2 : N; }   // row stride
template <bool TMA> constexpr int us_ks() { return TMA ? N * (N + 2) : 68; }  // k stride
template <bool TMA> constexpr int us_sz() { return N * us_ks<TMA>(); }
// SA: [f][row][8c + i] with row stride 72 (= 8 mod 16 doubles) and the i-bit-2
// swizzle swa(row); used for Z->Y (row = j, c = a3) and X'->Y' (row = b = a2,
// c = a3). Both the 16-byte C-fragment stores (rows fixed per warp, pencil
// pairs i = 2t, 2t+1) and the 8-byte B-fragment loads (rows t, t+4, i = g) are
// bank-conflict free.
constexpr int SA_KS = 72;
constexpr int SA_F = Q * SA_KS;           // 648
__device__ __forceinline__ int swa(int row) { return (row & 2) << 1; }
// [f][i][b + 9c] (Y->X); stride = 12 (mod 16) plus an XOR-4 swizzle of the
// pencil index on rows i >= 4 keeps both the C-tile stores (rows 2t, 2t+1)
// and the B-fragment loads (rows t, t+4) conflict free.
constexpr int SB_KS = 92;
__device__ __forceinline__ int sbi(int k, int p) { return k * SB_KS + (p ^ (((k >> 2) & 1) << 2)); }
constexpr int SB_F = N * SB_KS;           // 736
constexpr int SC_KS = 68;                 // [f][c][i + 8j] (Y'->Z')
constexpr int SC_F = Q * SC_KS;           // 612
constexpr int NUB = 4;                    // u staging buffers: U(e-1) .. U(e+2) live at once
constexpr int US_REGION = NUB * us_sz<true>() + 16;  // >= NUB * us_sz<false>(), with the 128-byte alignment slack
static_assert(US_REGION >= NUB * us_sz<false>(), "staging region");
constexpr int OFF_SA = 0;                 // Z -> Y   : 2 fields, SA layout
constexpr int OFF_SP = OFF_SA + 2 * SA_F;  // X' -> Y' : 3 fields, SA layout
constexpr int OFF_SB = OFF_SP + 3 * SA_F;  // Y -> X   : 3 fields
constexpr int OFF_SC = OFF_SB + 3 * SB_F;  // Y' -> Z' : 2 fields
constexpr int OFF_G = OFF_SC + 2 * SC_F;   // 16-byte aligned (even)
constexpr int OFF_U = OFF_G + GSE;
constexpr int OFF_BAS = OFF_U + US_REGION;  // B, D (q x n each), resident
constexpr int OFF_R8 = OFF_BAS + 2 * Q * N;   // packed row-8 pairs (16-byte loads)
constexpr int OFF_BAR = OFF_R8 + 16 + 16;     // G mbarrier, then NUB u mbarriers (TMA path)
constexpr int SMEM_BYTES = (OFF_BAR + 1 + NUB) * 8;
static_assert(OFF_G % 2 == 0, "TMA destination must be 16-byte aligned");
static_assert(2 * (SMEM_BYTES + 1024) <= 228 * 1024, "two CTAs per SM");

struct MmaBasis {
  double B[Q][N];
  double D[Q][N];
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double lds_volatile(const double* p) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
  return v;
}

// sum over the 4 lanes of a quad (lanes sharing lane/4)
__device__ __forceinline__ double quad_sum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

// CON: ConstrainedOperator semantics (ApplyArgs::constrained), DOT: the CG
// form with the fused p.Ap (ApplyArgs::col_dot) -- compile-time, so neither
// adds tests to the phase bodies.
// LBC: the column touches the lateral (x/y) boundary of a constrained
// operator. Interior columns (94% at cfg3) run a copy of the body compiled
// without the lateral boundary tests.
template <bool CON, bool DOT, bool LBC, bool TMA>
__device__ __forceinline__ void mma_column(const ApplyArgs& A, const MmaBasis& bs, const CUtensorMap& tmu) {
  extern __shared__ double smem[];
  double* SA = smem + OFF_SA;
  double* SP = smem + OFF_SP;
  double* SB = smem + OFF_SB;
  double* SC = smem + OFF_SC;
  double* Gs = smem + OFF_G;
  double* Us = smem + OFF_U;
  if (TMA) Us += ((128 - (smem_u32(Us) & 127)) & 127) / 8;  // tensor copies land 128-byte aligned
  constexpr int UKS = us_ks<TMA>(), URS = us_rs<TMA>(), USZ = us_sz<TMA>();
  __shared__ double s_red[NW];

  if (A.sc != nullptr && *(volatile int*)&A.sc->status != ST_RUNNING) return;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const uint64_t pol = policy_evict_first();
  constexpr bool do_dot = DOT;
  const int col = blockIdx.x;
  const int ex = col % A.nx, ey = col / A.nx;
  const int nz = A.nz;              // elements per column of the slab (G column stride)
  const int e0 = A.zr0, e1 = A.zr1;  // elements this launch marches (dist.cu overlap: sub-ranges)
  const int ush = TMA ? (ex & 1) : 0;  // x offset of the element in a staged row (TMA box from an even x)
  const LatLayout Lat(P, A.nx, A.ny);

  // Basis: B and D stay in shared memory for the whole kernel. The 8 x 8
  // MMA fragments are read once into registers with volatile loads (read from
  // the parameter bank with a lane-dependent index, ptxas would re-issue
  // serialised LDCs inside the loop); the row-8 values (4-8 distinct
  // addresses per warp: broadcast loads) are read from shared memory at use.
  double* sB = smem + OFF_BAS;
  double* sD = sB + Q * N;
  if (tid < Q * N) {
    sB[tid] = (&bs.B[0][0])[tid];
    sD[tid] = (&bs.D[0][0])[tid];
  }
  __syncthreads();
  auto bas = [&](const double* m, int a, int i) { return lds_volatile(m + a * N + i); };
  const double aB0 = bas(sB, g, t), aB1 = bas(sB, g, t + 4);            // forward rows 0..7 (A = M[m][k])
  const double aD0 = bas(sD, g, t), aD1 = bas(sD, g, t + 4);
  const double tB0 = bas(sB, t, g), tB1 = bas(sB, t + 4, g);            // backward (A = M^T[i][a])
  const double tD0 = bas(sD, t, g), tD1 = bas(sD, t + 4, g);
  // phase X' (transposed form, k-slot t <-> a = 2t (+1)): B[k][n = i] = M[a][i]
  const double eB0 = bas(sB, 2 * t, g), eB1 = bas(sB, 2 * t + 1, g);
  const double eD0 = bas(sD, 2 * t, g), eD1 = bas(sD, 2 * t + 1, g);
  const double* rB = sB + 8 * N;  // row a = 8
  const double* rD = sD + 8 * N;
  // row 8 packed for 16-byte loads: R8[t] = (B8[t], B8[t+4], D8[t], D8[t+4]),
  // C8[g] = (B8[g], D8[g])
  double* R8 = smem + OFF_R8;
  if (tid < 4) {
    R8[4 * tid] = rB[tid];
    R8[4 * tid + 1] = rB[tid + 4];
    R8[4 * tid + 2] = rD[tid];
    R8[4 * tid + 3] = rD[tid + 4];
  } else if (tid < 12) {
    R8[16 + 2 * (tid - 4)] = rB[tid - 4];
    R8[16 + 2 * (tid - 4) + 1] = rD[tid - 4];
  }
  __syncthreads();
  // quad-sum partial of row 8 for fields M = B (0) or D (1) over k = t, t+4
  auto row8B = [&](double x0, double x1) {
    const double2 b = *reinterpret_cast<const double2*>(R8 + 4 * t);
    return fma(b.y, x1, b.x * x0);
  };
  auto row8D = [&](double x0, double x1) {
    const double2 d = *reinterpret_cast<const double2*>(R8 + 4 * t + 2);
    return fma(d.y, x1, d.x * x0);
  };
  auto c8 = [&]() { return *reinterpret_cast<const double2*>(R8 + 16 + 2 * g); };  // (B8[g], D8[g])
  auto f8B = [&]() { return *reinterpret_cast<const double2*>(rB + 2 * t); };     // (B8[2t], B8[2t+1])
  auto f8D = [&]() { return *reinterpret_cast<const double2*>(rD + 2 * t); };

  const double* Gcol = A.G + static_cast<long long>(col) * nz * GSE;
  constexpr uint32_t gbytes = GSE * 8;
  const uint32_t bar = smem_u32(smem + OFF_BAR);
  const uint32_t ubar0 = bar + 8;  // TMA path: u buffer b completes on ubar0 + 8 b
  if (tid == 0) {
    mbar_init(bar, 1);
    if (TMA)
      for (int b = 0; b < NUB; ++b) mbar_init(ubar0 + 8 * b, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(bar, gbytes);
    bulk_g2s(smem_u32(Gs), Gcol + e0 * GSE, gbytes, bar, pol);
    if (e1 - e0 > 1) prefetch_l2_bulk(Gcol + (e0 + 1) * GSE, gbytes);
  }
  // u staging of element e into buffer (e - e0) % NUB.
  // TMA path: one tensor copy of the 8^3 node block at (7 ex, 7 ey, 7 e),
  // issued by one thread, completing on the buffer's mbarrier (parity
  // ((e - e0) / NUB) & 1); readers wait on it (wait_u).
  // cp.async path: thread (i,j) of the footprint (tid < 64) copies its z-pencil.
  auto ubuf = [&](int e) { return Us + ((e - e0) & (NUB - 1)) * USZ; };
  auto wait_u = [&](int e) {
    if (TMA) mbar_wait_parity(ubar0 + 8 * ((e - e0) & (NUB - 1)), ((e - e0) / NUB) & 1);
  };
  auto fetch_u = [&](int e) {
    if (TMA) {
      if (e < e1 && tid == NXW * 32) {
        const uint32_t ub = ubar0 + 8 * ((e - e0) & (NUB - 1));
        fence_proxy_async();  // the buffer's previous contents were read through the generic proxy
        mbar_arrive_expect_tx(ub, USZ * 8);
        tma_load_3d(smem_u32(ubuf(e)), &tmu, ex * P - ush, ey * P, e * P, ub);
      }
    } else {
      if (e < e1 && tid < N * N) {
        const int i = tid & 7, j = tid >> 3;
        const uint32_t dst = smem_u32(ubuf(e) + tid);
        const long long upitch = A.u_pitch ? A.u_pitch : A.Nx;  // u may be row-pitched
        const long long base = (ex * P + i) + upitch * (ey * P + j);
        const long long plane = upitch * A.Ny;
#pragma unroll
        for (int k = 0; k < N; ++k) cp_async8(dst + k * UKS * 8, A.u + base + plane * (e * P + k));
      }
      cp_async_commit();
    }
  };

  // ------------------------------------------------ phase bodies
  // Z(e, j): z contraction of element e, pencil group j (i = g) -> SA
  auto phaseZ = [&](int e, int G) {
    wait_u(e);
    const double* us = ubuf(e);
    const int X = ex * P + g, Y = ey * P + G;
    const bool bcxy = LBC && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1);
    double b[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int k = t + 4 * s, Z = e * P + k;
      double v = us[k * UKS + G * URS + ush + g];
      if (CON && (bcxy || (Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi))) v = 0.0;
      b[s] = v;
    }
    double cb0 = 0, cb1 = 0, cd0 = 0, cd1 = 0;
    dmma(cb0, cb1, aB0, b[0]);
    dmma(cb0, cb1, aB1, b[1]);
    dmma(cd0, cd1, aD0, b[0]);
    dmma(cd0, cd1, aD1, b[1]);
    const double r8b = quad_sum(row8B(b[0], b[1]));
    const double r8d = quad_sum(row8D(b[0], b[1]));
    // SA[f][j = G][8 a3 + i]: rows a3 = g, cols i = 2t, 2t+1; row a3 = 8 at i = g
    double* sa = SA + G * SA_KS;
    const int h = swa(G);
    *reinterpret_cast<double2*>(sa + 8 * g + (2 * t ^ h)) = make_double2(cb0, cb1);
    *reinterpret_cast<double2*>(sa + SA_F + 8 * g + (2 * t ^ h)) = make_double2(cd0, cd1);
    if (t == 0) {
      sa[64 + (g ^ h)] = r8b;
      sa[SA_F + 64 + (g ^ h)] = r8d;
    }
  };

  // Y(c): y contraction, a3 group c (pencil i = g) -> SB
  auto phaseY = [&](int G) {
    const double* sa = SA + 8 * G + (g ^ swa(t));  // rows j = t, t+4 share the swizzle
    const double x00 = sa[t * SA_KS], x01 = sa[(t + 4) * SA_KS];
    const double x10 = sa[SA_F + t * SA_KS], x11 = sa[SA_F + (t + 4) * SA_KS];
    double bb0 = 0, bb1 = 0, db0 = 0, db1 = 0, bd0 = 0, bd1 = 0;
    dmma(bb0, bb1, aB0, x00);
    dmma(bb0, bb1, aB1, x01);
    dmma(db0, db1, aD0, x00);
    dmma(db0, db1, aD1, x01);
    dmma(bd0, bd1, aB0, x10);
    dmma(bd0, bd1, aB1, x11);
    const double r8bb = quad_sum(row8B(x00, x01));
    const double r8db = quad_sum(row8D(x00, x01));
    const double r8bd = quad_sum(row8B(x10, x11));
    // SB[f][k = i][p = b + 9c]; rows b = g, cols i = 2t, 2t+1
    const int i0 = sbi(2 * t, g + 9 * G), i1 = sbi(2 * t + 1, g + 9 * G);
    SB[i0] = bb0;
    SB[i1] = bb1;
    SB[SB_F + i0] = db0;
    SB[SB_F + i1] = db1;
    SB[2 * SB_F + i0] = bd0;
    SB[2 * SB_F + i1] = bd1;
    if (t == 0) {  // b = 8, k = i = g
      const int i8 = sbi(g, 8 + 9 * G);
      SB[i8] = r8bb;
      SB[SB_F + i8] = r8db;
      SB[2 * SB_F + i8] = r8bd;
    }
  };

  // X(G): x contraction forward, pointwise G, x contraction backward for the
  // pencils p = 8G + g over (b, c) (valid p < 81) -> SP.
  // Transposed MMA form: C^T[pencil][a] = sum_i X^T[pencil][i] M^T[i][a], so
  // lane (g, t) ends with pencil g at points a = 2t, 2t+1 -- exactly the
  // A-fragment (row g, k-slot t <-> a = 2t / 2t+1) of the backward MMA. No
  // transpose between the forward and backward x contractions.
  auto phaseX = [&](int G) {
    const int k0 = sbi(t, 8 * G + g), k1 = sbi(t + 4, 8 * G + g);
    const double x00 = SB[k0], x01 = SB[k1];
    const double x10 = SB[SB_F + k0], x11 = SB[SB_F + k1];
    const double x20 = SB[2 * SB_F + k0], x21 = SB[2 * SB_F + k1];
    double gr[2] = {0, 0}, gs[2] = {0, 0}, gt[2] = {0, 0};
    dmma(gr[0], gr[1], x00, aD0);
    dmma(gr[0], gr[1], x01, aD1);
    dmma(gs[0], gs[1], x10, aB0);
    dmma(gs[0], gs[1], x11, aB1);
    dmma(gt[0], gt[1], x20, aB0);
    dmma(gt[0], gt[1], x21, aB1);
    double r8r = quad_sum(row8D(x00, x01));  // a = 8 of pencil g (all 4 lanes)
    double r8s = quad_sum(row8B(x10, x11));
    double r8t = quad_sum(row8B(x20, x21));
    const int p = 8 * G + g;
    {
      // pointwise factors (operator.hpp:129-131); [qp][6] layout, qp = a + 9p:
      // points a = 2t, 2t+1 are 12 contiguous doubles (conflict-free 16-byte loads).
      // Pencils p >= 81 of the last group read pencil 80's factors (their
      // results are never stored), which keeps the phase branch-free.
      const int pc = p < QQ ? p : QQ - 1;
      const double2* gp = reinterpret_cast<const double2*>(Gs + (2 * t + Q * pc) * 6);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double2 ga = gp[3 * e], gb = gp[3 * e + 1], gc = gp[3 * e + 2];
        const double r = gr[e], s_ = gs[e], u = gt[e];
        gr[e] = ga.x * r + ga.y * s_ + gb.x * u;
        gs[e] = ga.y * r + gb.y * s_ + gc.x * u;
        gt[e] = gb.x * r + gc.x * s_ + gc.y * u;
      }
      const double2* g8 = reinterpret_cast<const double2*>(Gs + (8 + Q * pc) * 6);
      const double2 ga = g8[0], gb = g8[1], gc = g8[2];
      const double r = r8r, s_ = r8s, u = r8t;
      r8r = ga.x * r + ga.y * s_ + gb.x * u;
      r8s = ga.y * r + gb.y * s_ + gc.x * u;
      r8t = gb.x * r + gc.x * s_ + gc.y * u;
    }
    // backward: W[p][i] = sum_a A[p][a] M[a][i]; a = 8 term first
    double w1[2], w2[2], w3[2];
    const double2 fd = f8D(), fb = f8B();
    w1[0] = fd.x * r8r;
    w1[1] = fd.y * r8r;
    w2[0] = fb.x * r8s;
    w2[1] = fb.y * r8s;
    w3[0] = fb.x * r8t;
    w3[1] = fb.y * r8t;
    dmma(w1[0], w1[1], gr[0], eD0);
    dmma(w1[0], w1[1], gr[1], eD1);
    dmma(w2[0], w2[1], gs[0], eB0);
    dmma(w2[0], w2[1], gs[1], eB1);
    dmma(w3[0], w3[1], gt[0], eB0);
    dmma(w3[0], w3[1], gt[1], eB1);
    // pencil p = b + 9c, outputs i = 2t, 2t+1 -> SP[f][b][8c + i] (16-byte stores)
    if (p < QQ) {
      const int c = p / 9, bq = p - 9 * c;
      double* d = SP + bq * SA_KS + 8 * c + (2 * t ^ swa(bq));
      *reinterpret_cast<double2*>(d) = make_double2(w1[0], w1[1]);
      *reinterpret_cast<double2*>(d + SA_F) = make_double2(w2[0], w2[1]);
      *reinterpret_cast<double2*>(d + 2 * SA_F) = make_double2(w3[0], w3[1]);
    }
  };

  // Y'(c): y contraction backward, a3 group c (pencil i = g; over b) -> SC
  auto phaseYp = [&](int G) {
    const double* sa = SP + 8 * G + (g ^ swa(t));
    const double y00 = sa[t * SA_KS], y01 = sa[(t + 4) * SA_KS];
    const double y10 = sa[SA_F + t * SA_KS], y11 = sa[SA_F + (t + 4) * SA_KS];
    const double y20 = sa[2 * SA_F + t * SA_KS], y21 = sa[2 * SA_F + (t + 4) * SA_KS];
    const double* s8 = SP + 8 * SA_KS + 8 * G + 2 * t;  // b = 8, pencils i = 2t, 2t+1
    const double2 e1 = *reinterpret_cast<const double2*>(s8);
    const double2 e2 = *reinterpret_cast<const double2*>(s8 + SA_F);
    const double2 e3 = *reinterpret_cast<const double2*>(s8 + 2 * SA_F);
    double c1[2], c2[2];
    const double2 bd8 = c8();
    c1[0] = fma(bd8.y, e2.x, bd8.x * e1.x);
    c1[1] = fma(bd8.y, e2.y, bd8.x * e1.y);
    c2[0] = bd8.x * e3.x;
    c2[1] = bd8.x * e3.y;
    dmma(c1[0], c1[1], tB0, y00);
    dmma(c1[0], c1[1], tB1, y01);
    dmma(c1[0], c1[1], tD0, y10);
    dmma(c1[0], c1[1], tD1, y11);
    dmma(c2[0], c2[1], tB0, y20);
    dmma(c2[0], c2[1], tB1, y21);
    // rows j = g, cols i = 2t, 2t+1, c = G -> SC[f][c][i + 8j]
    double* sc = SC + G * SC_KS + 8 * g + 2 * t;
    *reinterpret_cast<double2*>(sc) = make_double2(c1[0], c1[1]);
    *reinterpret_cast<double2*>(sc + SC_F) = make_double2(c2[0], c2[1]);
  };

  // Z'(e, j) + transpose restriction part 1: z contraction backward of
  // element e, j group (pencil i = g); z-shared plane carried in registers
  // (this warp always owns group j).
  double carry[2] = {0.0, 0.0};
  double dot = 0.0;
  auto phaseZpMath = [&](int G, double* o) {
    const double* sc = SC + 8 * G + g;
    const double z00 = sc[t * SC_KS], z01 = sc[(t + 4) * SC_KS];
    const double z10 = sc[SC_F + t * SC_KS], z11 = sc[SC_F + (t + 4) * SC_KS];
    const double* s8 = SC + 8 * SC_KS + 8 * G + 2 * t;  // c = 8
    const double2 e1 = *reinterpret_cast<const double2*>(s8);
    const double2 e2 = *reinterpret_cast<const double2*>(s8 + SC_F);
    const double2 bd8 = c8();
    o[0] = fma(bd8.y, e2.x, bd8.x * e1.x);
    o[1] = fma(bd8.y, e2.y, bd8.x * e1.y);
    dmma(o[0], o[1], tB0, z00);
    dmma(o[0], o[1], tB1, z01);
    dmma(o[0], o[1], tD0, z10);
    dmma(o[0], o[1], tD1, z11);
  };
  auto phaseZpStore = [&](int e, int G, double* o) {
    // rows k = g (z node), cols i = 2t, 2t+1, j = G
    const double top0 = __shfl_sync(0xffffffffu, carry[0], 28 + t);
    const double top1 = __shfl_sync(0xffffffffu, carry[1], 28 + t);
    if (g == 0) {
      o[0] += top0;
      o[1] += top1;
    }
    if (g == P && e + 1 < e1) {
      carry[0] = o[0];
      carry[1] = o[1];
      return;
    }
    // range ends inside the slab (dist.cu overlap): leave this launch's share
    // of the plane for launch_carry_combine (no store, no dot)
    double* cplane = g == P ? A.carry_hi : (g == 0 && e == e0 ? A.carry_lo : nullptr);
    if (cplane != nullptr) {
      *reinterpret_cast<double2*>(cplane + col * (N * N) + G * N + 2 * t) = make_double2(o[0], o[1]);
      return;
    }
    const int Z = e * P + g, Y = ey * P + G;
    const bool zbc = CON && ((Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi));
    // u at these nodes: still staged in shared memory (z-plane k = g of element e)
    const double* ur = ubuf(e) + g * UKS + G * URS + ush + 2 * t;
    // 16-byte load unless the TMA box put the element at an odd x offset
    const double2 u2 = TMA && ush ? make_double2(ur[0], ur[1]) : *reinterpret_cast<const double2*>(ur);

    // ring partials -> lateral buffer (ring.cuh layout): a ring row (j = 0 or
    // P) stores all P+1 of its nodes as one 16-byte pair per lane
    const bool rowring = G == 0 || G == P;
    if (rowring)
      *reinterpret_cast<double2*>(A.lateral + Lat.y_index(P, A.nx, Z, ey + (G == P), G == 0, ex, 2 * t)) =
          make_double2(o[0], o[1]);
    if (!rowring) {
      // The row's P+1 nodes go to w, the two x-face nodes (i = 0, P) with
      // this column's partial: their w value is never read (the r-update /
      // lateral fix-up supplies them from latX; the neighbour column's store
      // of its own partial may win), but complete rows turn the L2's
      // evictions of this row's 32-byte sectors into full-sector writes
      // instead of DRAM read-modify-writes of ECC sectors (-0.38 GB of DRAM
      // reads per apply at cfg3), and the lanes' node pairs are 16-byte
      // stores whenever the row starts at an even node (parity uniform per row).
      const long long node0 =  // w may be row-pitched (ApplyArgs::w_pitch)
          ex * P + 2 * t + static_cast<long long>(A.w_pitch ? A.w_pitch : A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
      const double v0 = (zbc && t != 0) ? u2.x : o[0];      // i = 2t     (x-face at t = 0)
      const double v1 = (zbc && t != 3) ? u2.y : o[1];      // i = 2t + 1 (x-face at t = 3)
      if ((node0 & 1) == 0) {
        *reinterpret_cast<double2*>(A.w + node0) = make_double2(v0, v1);
      } else {
        A.w[node0] = v0;
        A.w[node0 + 1] = v1;
      }
      if (t == 0) A.lat_x[Lat.x_index(A.nx, Z, Y, ex, 1)] = o[0];
      if (t == 3) A.lat_x[Lat.x_index(A.nx, Z, Y, ex + 1, 0)] = o[1];
    }
    if (do_dot && !zbc && !LBC) {
      // interior column, no essential node in this row: every node -- ring or
      // not -- adds u * (its column value), the same FMAs as the general path
      dot = fma(u2.x, o[0], dot);
      dot = fma(u2.y, o[1], dot);
    } else if (do_dot) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double uv = q ? u2.y : u2.x;
        const int i = 2 * t + q, X = ex * P + i;
        const bool ring = rowring || i == 0 || i == P;
        if (ring) {  // column-local share of p.Ap on the ring (ring.cuh)
          if (zbc || (LBC && (X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1))) {
            if (ring_owner(P, i, G, ex, ey, A.nx, A.ny) && !(A.zlo_shared && Z == 0))
              dot = fma(uv, uv, dot);  // w = u, counted once
          } else {
            dot = fma(uv, o[q], dot);
          }
        } else {
          dot = fma(uv, zbc ? uv : o[q], dot);
        }
      }
    }
  };

  auto phaseZp = [&](int e, int G) {
    double o[2];
    phaseZpMath(G, o);
    phaseZpStore(e, G, o);
  };

  // ------------------------------------------------ skewed schedule
  // Two barrier intervals per element, each mixing independent work of
  // neighbouring elements so that no warp idles through a phase:
  //   A_e : X(e) [warp = pencil group], Z(e+1), Z'(e-1)      -> SP, SA, w
  //   B_e : Y'(e), Y(e+1)                                    -> SC, SB
  // Buffers: SA (Z->Y), SP (X'->Y'), SB (Y->X), SC (Y'->Z') are each written
  // and read in consecutive intervals; G(e+1) streams into the single G buffer
  // during B_e (TMA, mbarrier); u of element e+2 is staged (cp.async) during
  // A_e and B_e into one of NUB = 4 buffers (Z'(e-1) still reads u(e-1) for
  // the p.Ap dot).
  // Work map: Z'(j) on warp j (its carry registers), Z(0..4) on warp 11 and
  // Z(5..7) on warps 8..10, X(G) on warp G < 11, Y'(c) on warp c, Y(c) on
  // warp (c+9) % 12.
  fetch_u(e0);
  fetch_u(e0 + 1);
  if (!TMA) {
    cp_async_wait<0>();
    __syncthreads();
  }
  if (warp < N) phaseZ(e0, warp);
  __syncthreads();
  if (warp < Q) phaseY(warp);
  __syncthreads();
  for (int e = e0; e <= e1; ++e) {
    // ---- interval A_e
    fetch_u(e + 2);
    if (tid == 0 && e + 2 < e1) prefetch_l2_bulk(Gcol + (e + 2) * GSE, gbytes);
    // Z'(e-1) and Z(e+1) first: they do not read G, so the G(e) transfer
    // issued in B_{e-1} has the longest time to land before X(e) waits on it
    if (e > e0 && warp < N) phaseZp(e - 1, warp);
    if (e + 1 < e1) {
      // warp 11: Z(0..4); warps 8..10: Z(5..7) beside their X group
      if (warp == NXW) {
        for (int j = 0; j < 5; ++j) phaseZ(e + 1, j);
      } else if (warp >= 8) {
        phaseZ(e + 1, warp - 3);
      }
    }
    if (e < e1 && warp < NXW) {
      mbar_wait_parity(bar, (e - e0) & 1);
      phaseX(warp);
    }
    if (e == e1) break;
    __syncthreads();
    // ---- interval B_e
    if (tid == 0 && e + 1 < e1) {  // X(e) consumed the G buffer: stream G(e+1)
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, gbytes);
      bulk_g2s(smem_u32(Gs), Gcol + (e + 1) * GSE, gbytes, bar, pol);
    }
    if (warp < Q) phaseYp(warp);
    if (e + 1 < e1) {
      // Y(c) on warp (c + 9) % NW
      const int c = warp >= 9 ? warp - 9 : warp + NW - 9;
      if (c < Q) phaseY(c);
    }
    if (!TMA) cp_async_wait<0>();  // u(e+2), issued at the top of A_e, is read by Z(e+2) in A_{e+1}
    __syncthreads();
  }
  double cdot = 0.0;
  if (do_dot) {
    double v = dot;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int w = 0; w < NW; ++w) cdot += s_red[w];
    }
    __syncthreads();
  }
  ring_dot_finish<NT>(A, col, cdot, s_red);
}

template <bool CON, bool DOT, bool TMA>
__global__ void __launch_bounds__(NT, 2)
    bp3_p7_mma_kernel(const __grid_constant__ ApplyArgs A, const __grid_constant__ MmaBasis bs,
                      const __grid_constant__ CUtensorMap tmu) {
  if constexpr (CON) {
    const int ex = blockIdx.x % A.nx, ey = blockIdx.x / A.nx;
    if (ex > 0 && ex < A.nx - 1 && ey > 0 && ey < A.ny - 1)
      mma_column<true, DOT, false, TMA>(A, bs, tmu);
    else
      mma_column<true, DOT, true, TMA>(A, bs, tmu);
  } else {
    mma_column<false, DOT, false, TMA>(A, bs, tmu);
  }
}

}  // namespace

bool mma_kernel_applies(const Setup& s) { return s.kind == KIND_DIFF && s.p == P && s.gstride == GSE; }

cudaError_t launch_apply_mma(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  static std::atomic<uint64_t> configured[8] = {};
  const int v = (a.u_tmap ? 4 : 0) + (a.constrained ? 2 : 0) + (a.col_dot != nullptr ? 1 : 0);
  const void* fns[8] = {reinterpret_cast<const void*>(&bp3_p7_mma_kernel<false, false, false>),
                        reinterpret_cast<const void*>(&bp3_p7_mma_kernel<false, true, false>),
                        reinterpret_cast<const void*>(&bp3_p7_mma_kernel<true, false, false>),
                        reinterpret_cast<const void*>(&bp3_p7_mma_kernel<true, true, false>),
                        reinterpret_cast<const void*>(&bp3_p7_mma_kernel<false, false, true>),
                        reinterpret_cast<const void*>(&bp3_p7_mma_kernel<false, true, true>),
                        reinterpret_cast<const void*>(&bp3_p7_mma_kernel<true, false, true>),
                        reinterpret_cast<const void*>(&bp3_p7_mma_kernel<true, true, true>)};
  set_smem_attr_once(configured[v], fns[v], SMEM_BYTES);
  MmaBasis bs;
  for (int i = 0; i < Q; ++i)
    for (int j = 0; j < N; ++j) {
      bs.B[i][j] = s.B[i * N + j];
      bs.D[i][j] = s.D[i * N + j];
    }
  static const CUtensorMap none{};
  const CUtensorMap& tm = a.u_tmap ? *a.u_tmap : none;
  switch (v) {
#define HXB_MMA_CASE(V, CON, DOT, TMA) \
  case V: bp3_p7_mma_kernel<CON, DOT, TMA><<<a.ncols, NT, SMEM_BYTES, st>>>(a, bs, tm); break;
    HXB_MMA_CASE(0, false, false, false)
    HXB_MMA_CASE(1, false, true, false)
    HXB_MMA_CASE(2, true, false, false)
    HXB_MMA_CASE(3, true, true, false)
    HXB_MMA_CASE(4, false, false, true)
    HXB_MMA_CASE(5, false, true, true)
    HXB_MMA_CASE(6, true, false, true)
    default: bp3_p7_mma_kernel<true, true, true><<<a.ncols, NT, SMEM_BYTES, st>>>(a, bs, tm); break;
#undef HXB_MMA_CASE
  }
  return cudaGetLastError();
}

void mma_kernel_info(int* regs, int* smem, int* threads, int* blocks_per_sm) {
  cudaFuncSetAttribute(&bp3_p7_mma_kernel<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, bp3_p7_mma_kernel<true, true, false>);
  *regs = fa.numRegs;
  *smem = static_cast<int>(fa.sharedSizeBytes) + SMEM_BYTES;
  *threads = NT;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, bp3_p7_mma_kernel<true, true, false>, NT, SMEM_BYTES);
}

}  // namespace hxb
