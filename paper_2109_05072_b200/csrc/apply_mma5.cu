// FP64 tensor-core (DMMA) operator kernel for BP5 at p = 7 (collocated
// Gauss-Lobatto quadrature, n = q = 8, B = I exactly: basis.hpp:55-66) --
// fast mode. The collocated gradient is three D contractions
// (tensor.hpp:177-203 with B = I):
//   gr = D_x u,  gs = D_y u,  gt = D_z u     (A1,A2,A3) = G (gr,gs,gt)
//   w  = D_x^T A1 + D_y^T A2 + D_z^T A3
// Every contraction is an exact 8 x 8 tile (no ragged row as in BP3's q = 9):
// 96 m8n8k4 DMMAs per element.
//
// Phases (8 warps, 8 work items each):
//   Z (j group)  : gt = D_z u                                  -> GT
//   P (z plane c): gr = D_x u (transposed MMA form: rows j, cols a),
//                  gs = D_y u (standard form: rows j, cols i -- the same
//                  lane layout), gt from GT; G; W12 = D_x^T A1 (chained on
//                  the fragment) + D_y^T A2 (A2 through a warp-private 8x8
//                  transpose)                                   -> W, A3
//   Z' (j group) : out = W12 + D_z^T A3, then the transpose restriction
//                  (carry, ring partials to the lateral buffer: ring.cuh)
// skewed into ONE barrier interval per element: P(e) || Z(e+1) || Z'(e-1)
// (GT, A3, W double-buffered by element parity, u staged in 3 buffers).
// Factors: element block [c][comp][b][a] (Setup::g_aos = 2); each warp owns
// its plane c and streams that plane of the next element with its own TMA
// bulk copy + mbarrier as soon as it has read the current one.
// p.Ap (CG): the quadrature energy sum_q grad(Pu).G grad(Pu) in phase P plus
// u^2 on the owned ConstrainedOperator rows while masking the staged input
// = (Pu).A(Pu) + sum_bc u^2 = u.(P A P u + (I - P) u).
#include <cuda_runtime.h>

#include <cstdint>

#include "device_util.cuh"
#include "internal.h"
#include "ring.cuh"

namespace hxb {
namespace {

constexpr int P = 7, N = 8;
constexpr int NW = 8, NT = NW * 32;
constexpr int GPL = 6 * N * N;          // one z plane of all 6 components (doubles)
constexpr int GSE = 6 * N * N * N;      // element block of G (== Setup::gstride)
// u staging [k][j][i] (see apply_mma.cu): cp.async rows of 8, k-stride 68;
// TMA: 10-wide boxes from the even x at or below the element, 128-byte aligned
template <bool TMA> constexpr int us_rs() { return TMA ? N + 2 : N; }
template <bool TMA> constexpr int us_ks() { return TMA ? N * (N + 2) : 68; }
constexpr int NUB = 3;                  // U(e) (P), U(e+1) (Z), U(e+2) in flight
constexpr int US_REGION = NUB * N * us_ks<true>() + 16;
static_assert(US_REGION >= NUB * N * us_ks<false>(), "staging region");
constexpr int TS = 9 * 64;              // [c][j][i] tiles: c-stride 72 (+ i swizzle), 8 planes
__device__ __forceinline__ int tix(int c, int j, int i) { return c * 72 + j * 8 + (i ^ ((c & 2) << 1)); }
constexpr int OFF_GT = 0;                     // 2 x TS
constexpr int OFF_A3 = OFF_GT + 2 * TS;       // 2 x TS
constexpr int OFF_W = OFF_A3 + 2 * TS;        // 2 x TS
constexpr int OFF_U = OFF_W + 2 * TS;         // NUB x US_SZ
constexpr int OFF_G = OFF_U + US_REGION;      // NW x GPL (16-byte aligned)
constexpr int OFF_SCR = OFF_G + NW * GPL;     // NW x 64 (A2 transpose)
constexpr int OFF_D = OFF_SCR + NW * 64;      // D (8 x 8)
constexpr int OFF_BAR = OFF_D + 64;           // NW mbarriers (G planes), NUB (u buffers, TMA path)
constexpr int SMEM_BYTES = (OFF_BAR + NW + NUB) * 8;
static_assert(OFF_G % 2 == 0, "TMA destination must be 16-byte aligned");
static_assert(3 * (SMEM_BYTES + 1024) <= 228 * 1024, "three CTAs per SM");

struct Mma5Basis {
  double D[N][N];
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

// CON / DOT: constrained semantics and the fused p.Ap, compile-time (see apply_mma.cu)
template <bool CON, bool DOT, bool TMA>
__global__ void __launch_bounds__(NT, 3)
    bp5_p7_mma_kernel(const __grid_constant__ ApplyArgs A, const __grid_constant__ Mma5Basis bs,
                      const __grid_constant__ CUtensorMap tmu) {
  extern __shared__ double smem[];
  double* Us = smem + OFF_U;
  if (TMA) Us += ((128 - (smem_u32(Us) & 127)) & 127) / 8;  // tensor copies land 128-byte aligned
  constexpr int UKS = us_ks<TMA>(), URS = us_rs<TMA>(), USZ = N * UKS;
  __shared__ double s_red[NW];

  if (A.sc != nullptr && *(volatile int*)&A.sc->status != ST_RUNNING) return;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const uint64_t pol = policy_evict_first();
  constexpr bool do_dot = DOT;
  const int col = blockIdx.x;
  const int ex = col % A.nx, ey = col / A.nx;
  const int nz = A.nz;               // elements per column of the slab (G column stride)
  const int e0 = A.zr0, e1 = A.zr1;  // elements this launch marches (dist.cu overlap: sub-ranges)
  const int ush = TMA ? (ex & 1) : 0;  // x offset of the element in a staged row (TMA box from an even x)
  const LatLayout Lat(P, A.nx, A.ny);

  // basis fragments (registers for the whole kernel; see apply_mma.cu)
  double* sD = smem + OFF_D;
  if (tid < N * N) sD[tid] = (&bs.D[0][0])[tid];
  __syncthreads();
  const double aD0 = lds_volatile(sD + g * N + t), aD1 = lds_volatile(sD + g * N + t + 4);  // D[g][t]
  const double tD0 = lds_volatile(sD + t * N + g), tD1 = lds_volatile(sD + (t + 4) * N + g);  // D[t][g]
  const double eD0 = lds_volatile(sD + 2 * t * N + g), eD1 = lds_volatile(sD + (2 * t + 1) * N + g);

  // per-warp factor plane (plane c = warp) with its own mbarrier
  const double* Gcol = A.G + static_cast<long long>(col) * nz * GSE;
  double* Gp = smem + OFF_G + warp * GPL;
  const uint32_t bar = smem_u32(smem + OFF_BAR + warp);
  constexpr uint32_t pbytes = GPL * 8;
  const uint32_t ubar0 = smem_u32(smem + OFF_BAR + NW);  // TMA path: u buffer b completes on ubar0 + 8 b
  if (lane == 0) {
    mbar_init(bar, 1);
    if (TMA && warp == 0)
      for (int b = 0; b < NUB; ++b) mbar_init(ubar0 + 8 * b, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (lane == 0) {
    mbar_arrive_expect_tx(bar, pbytes);
    bulk_g2s(smem_u32(Gp), Gcol + e0 * GSE + warp * GPL, pbytes, bar, pol);
  }
  if (tid == 0 && e1 - e0 > 1) prefetch_l2_bulk(Gcol + (e0 + 1) * GSE, GSE * 8);

  // u staging of element e into buffer (e - e0) % NUB: one TMA tensor copy of
  // the 8^3 node block (TMA path, see apply_mma.cu) or thread (i,j) of the
  // footprint (tid < 64) copying its z-pencil by cp.async
  auto ubuf = [&](int e) { return Us + ((e - e0) % NUB) * USZ; };
  auto wait_u = [&](int e) {
    if (TMA) mbar_wait_parity(ubar0 + 8 * ((e - e0) % NUB), ((e - e0) / NUB) & 1);
  };
  auto fetch_u = [&](int e) {
    if (TMA) {
      if (e < e1 && tid == 32) {
        const uint32_t ub = ubar0 + 8 * ((e - e0) % NUB);
        fence_proxy_async();  // the buffer's previous contents were read / masked through the generic proxy
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
  // ConstrainedOperator input mask P u on the staged values (each thread its
  // own copies, after cp.async completion); u^2 of the owned constrained rows
  // goes to p.Ap
  double dot = 0.0;
  auto mask_u = [&](int e) {
    if (e >= e1 || tid >= N * N || !CON) return;
    wait_u(e);
    const int i = tid & 7, j = tid >> 3;
    const int X = ex * P + i, Y = ey * P + j;
    const bool bcxy = X == 0 || X == A.Nx - 1 || Y == 0 || Y == A.Ny - 1;
    const bool own_xy = (i < P || ex == A.nx - 1) && (j < P || ey == A.ny - 1);
    double* us = ubuf(e) + j * URS + ush + i;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int Z = e * P + k;
      if (bcxy || (Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi)) {
        if (do_dot && own_xy && (k < P || e == nz - 1) && !(A.zlo_shared && Z == 0))
          dot = fma(us[k * UKS], us[k * UKS], dot);
        us[k * UKS] = 0.0;
      }
    }
  };

  // ------------------------------------------------ phase bodies
  auto phaseZ = [&](int e, int G) {  // gt = D_z u, j group G -> GT
    wait_u(e);
    const double* us = ubuf(e);
    const double b0 = us[t * UKS + G * URS + ush + g], b1 = us[(t + 4) * UKS + G * URS + ush + g];
    double c0 = 0.0, c1 = 0.0;
    dmma(c0, c1, aD0, b0);
    dmma(c0, c1, aD1, b1);
    *reinterpret_cast<double2*>(smem + OFF_GT + (e & 1) * TS + tix(g, G, 2 * t)) = make_double2(c0, c1);
  };

  auto phaseP = [&](int e, int c) {  // z plane c of element e
    const double* us = ubuf(e) + c * UKS + ush;
    // gr (transposed form, rows j = g, cols a = 2t, 2t+1); gs (standard form, same layout)
    const double ua0 = us[g * URS + t], ua1 = us[g * URS + t + 4];
    const double ub0 = us[t * URS + g], ub1 = us[(t + 4) * URS + g];
    double gr[2] = {0.0, 0.0}, gs[2] = {0.0, 0.0};
    dmma(gr[0], gr[1], ua0, aD0);
    dmma(gr[0], gr[1], ua1, aD1);
    dmma(gs[0], gs[1], aD0, ub0);
    dmma(gs[0], gs[1], aD1, ub1);
    const double2 gt2 = *reinterpret_cast<const double2*>(smem + OFF_GT + (e & 1) * TS + tix(c, g, 2 * t));
    const double gt[2] = {gt2.x, gt2.y};
    // factors at (a = 2t+q, b = g, c): [c][m][b][a] -> this warp's plane buffer
    mbar_wait_parity(bar, (e - e0) & 1);
    double2 gm[6];
#pragma unroll
    for (int m = 0; m < 6; ++m) gm[m] = *reinterpret_cast<const double2*>(Gp + m * 64 + g * 8 + 2 * t);
    __syncwarp();
    if (lane == 0 && e + 1 < e1) {  // plane consumed: stream the next element's plane
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, pbytes);
      bulk_g2s(smem_u32(Gp), Gcol + (e + 1) * GSE + c * GPL, pbytes, bar, pol);
    }
    double a1[2], a2[2], a3[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double g0 = q ? gm[0].y : gm[0].x, g1 = q ? gm[1].y : gm[1].x, g2 = q ? gm[2].y : gm[2].x;
      const double g3 = q ? gm[3].y : gm[3].x, g4 = q ? gm[4].y : gm[4].x, g5 = q ? gm[5].y : gm[5].x;
      const double r = gr[q], s = gs[q], u = gt[q];
      a1[q] = g0 * r + g1 * s + g2 * u;  // apply_diffusion_factors (operator.hpp:129-131)
      a2[q] = g1 * r + g3 * s + g4 * u;
      a3[q] = g2 * r + g4 * s + g5 * u;
      if (do_dot) dot = fma(u, a3[q], fma(s, a2[q], fma(r, a1[q], dot)));  // quadrature energy
    }
    // W12 = D_x^T A1 (chained, k-slot t <-> a = 2t, 2t+1) + D_y^T A2 (via the warp scratch)
    double* scr = smem + OFF_SCR + warp * 64;
    *reinterpret_cast<double2*>(scr + g * 8 + ((2 * t) ^ ((g & 2) << 1))) = make_double2(a2[0], a2[1]);
    double w0 = 0.0, w1 = 0.0;
    dmma(w0, w1, a1[0], eD0);
    dmma(w0, w1, a1[1], eD1);
    __syncwarp();
    const double x0 = scr[t * 8 + (g ^ ((t & 2) << 1))], x1 = scr[(t + 4) * 8 + (g ^ ((t & 2) << 1))];
    dmma(w0, w1, tD0, x0);
    dmma(w0, w1, tD1, x1);
    __syncwarp();  // scratch reused by the next element
    *reinterpret_cast<double2*>(smem + OFF_W + (e & 1) * TS + tix(c, g, 2 * t)) = make_double2(w0, w1);
    *reinterpret_cast<double2*>(smem + OFF_A3 + (e & 1) * TS + tix(c, g, 2 * t)) = make_double2(a3[0], a3[1]);
  };

  double carry[2] = {0.0, 0.0};
  auto phaseZp = [&](int e, int G) {  // out = W12 + D_z^T A3, j group G; restriction part 1
    const double* a3s = smem + OFF_A3 + (e & 1) * TS;
    const double2 w = *reinterpret_cast<const double2*>(smem + OFF_W + (e & 1) * TS + tix(g, G, 2 * t));
    double o[2] = {w.x, w.y};
    dmma(o[0], o[1], tD0, a3s[tix(t, G, g)]);
    dmma(o[0], o[1], tD1, a3s[tix(t + 4, G, g)]);
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
    // of the plane for launch_carry_combine (the p.Ap energy form needs no node values)
    double* cplane = g == P ? A.carry_hi : (g == 0 && e == e0 ? A.carry_lo : nullptr);
    if (cplane != nullptr) {
      *reinterpret_cast<double2*>(cplane + col * (N * N) + G * N + 2 * t) = make_double2(o[0], o[1]);
      return;
    }
    const int Z = e * P + g, Y = ey * P + G;
    const bool zbc = CON && ((Z == 0 && A.bc_zlo) || (Z == A.Nz - 1 && A.bc_zhi));
    const bool rowring = G == 0 || G == P;
    if (rowring) {
      *reinterpret_cast<double2*>(A.lateral + Lat.y_index(P, A.nx, Z, ey + (G == P), G == 0, ex, 2 * t)) =
          make_double2(o[0], o[1]);
      return;
    }
    // the row's P+1 nodes go to w, the x-face nodes (i = 0, P) with this
    // column's partial (never read; full-sector L2 evictions instead of DRAM
    // read-modify-writes, see apply_mma.cu), and their partials to latX
    const long long node0 =  // w may be row-pitched (ApplyArgs::w_pitch)
        ex * P + 2 * t + static_cast<long long>(A.w_pitch ? A.w_pitch : A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
    double v[2] = {o[0], o[1]};
    if (zbc) {  // ConstrainedOperator rows: w = u (u may be row-pitched, ApplyArgs::u_pitch)
      const long long unode0 =
          ex * P + 2 * t + static_cast<long long>(A.u_pitch ? A.u_pitch : A.Nx) * (Y + static_cast<long long>(A.Ny) * Z);
      if (t != 0) v[0] = __ldg(A.u + unode0);
      if (t != 3) v[1] = __ldg(A.u + unode0 + 1);
    }
    if ((node0 & 1) == 0) {  // parity uniform per row
      *reinterpret_cast<double2*>(A.w + node0) = make_double2(v[0], v[1]);
    } else {
      A.w[node0] = v[0];
      A.w[node0 + 1] = v[1];
    }
    if (t == 0) A.lat_x[Lat.x_index(A.nx, Z, Y, ex, 1)] = o[0];
    if (t == 3) A.lat_x[Lat.x_index(A.nx, Z, Y, ex + 1, 0)] = o[1];
  };

  // ------------------------------------------------ schedule: A_e = P(e) || Z(e+1) || Z'(e-1)
  fetch_u(e0);
  fetch_u(e0 + 1);
  if (!TMA) cp_async_wait<0>();
  mask_u(e0);
  mask_u(e0 + 1);
  __syncthreads();
  phaseZ(e0, warp);
  __syncthreads();
  for (int e = e0; e <= e1; ++e) {
    fetch_u(e + 2);
    if (tid == 0 && e + 2 < e1) prefetch_l2_bulk(Gcol + (e + 2) * GSE, GSE * 8);
    if (e < e1) phaseP(e, warp);
    if (e > e0) phaseZp(e - 1, warp);
    if (e + 1 < e1) phaseZ(e + 1, warp);
    if (e == e1) break;
    if (!TMA) cp_async_wait<0>();
    mask_u(e + 2);
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

}  // namespace

bool mma5_kernel_applies(const Setup& s) { return s.kind == KIND_COLLOC && s.p == P && s.g_aos == 2; }

cudaError_t launch_apply_mma5(const Setup& s, const ApplyArgs& a, cudaStream_t st) {
  if (s.gstride != GSE) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> configured[8] = {};
  const int v = (a.u_tmap ? 4 : 0) + (a.constrained ? 2 : 0) + (a.col_dot != nullptr ? 1 : 0);
  const void* fns[8] = {reinterpret_cast<const void*>(&bp5_p7_mma_kernel<false, false, false>),
                        reinterpret_cast<const void*>(&bp5_p7_mma_kernel<false, true, false>),
                        reinterpret_cast<const void*>(&bp5_p7_mma_kernel<true, false, false>),
                        reinterpret_cast<const void*>(&bp5_p7_mma_kernel<true, true, false>),
                        reinterpret_cast<const void*>(&bp5_p7_mma_kernel<false, false, true>),
                        reinterpret_cast<const void*>(&bp5_p7_mma_kernel<false, true, true>),
                        reinterpret_cast<const void*>(&bp5_p7_mma_kernel<true, false, true>),
                        reinterpret_cast<const void*>(&bp5_p7_mma_kernel<true, true, true>)};
  set_smem_attr_once(configured[v], fns[v], SMEM_BYTES);
  Mma5Basis bs;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) bs.D[i][j] = s.D[i * N + j];
  static const CUtensorMap none{};
  const CUtensorMap& tm = a.u_tmap ? *a.u_tmap : none;
  switch (v) {
#define HXB_MMA5_CASE(V, CON, DOT, TMA) \
  case V: bp5_p7_mma_kernel<CON, DOT, TMA><<<a.ncols, NT, SMEM_BYTES, st>>>(a, bs, tm); break;
    HXB_MMA5_CASE(0, false, false, false)
    HXB_MMA5_CASE(1, false, true, false)
    HXB_MMA5_CASE(2, true, false, false)
    HXB_MMA5_CASE(3, true, true, false)
    HXB_MMA5_CASE(4, false, false, true)
    HXB_MMA5_CASE(5, false, true, true)
    HXB_MMA5_CASE(6, true, false, true)
    default: bp5_p7_mma_kernel<true, true, true><<<a.ncols, NT, SMEM_BYTES, st>>>(a, bs, tm); break;
#undef HXB_MMA5_CASE
  }
  return cudaGetLastError();
}

void mma5_kernel_info(int* regs, int* smem, int* threads, int* blocks_per_sm) {
  cudaFuncSetAttribute(&bp5_p7_mma_kernel<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, bp5_p7_mma_kernel<true, true, false>);
  *regs = fa.numRegs;
  *smem = static_cast<int>(fa.sharedSizeBytes) + SMEM_BYTES;
  *threads = NT;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, bp5_p7_mma_kernel<true, true, false>, NT, SMEM_BYTES);
}

}  // namespace hxb
