/* oracle/hexbp_oracle.c -- TEST INFRASTRUCTURE ONLY (see hexbp_oracle.h).
 *
 * Plain-C restatement of the reference CPU algorithm, used as the parity
 * checker for the CUDA product path. Citations are to
 * /root/reference/proj/include/hexbp/<file>:<line>. Operation order follows
 * the reference so that, compiled with -ffp-contract=off, outputs match the
 * reference bit for bit (tests/test_oracle.py).
 */
#define _GNU_SOURCE
#include "hexbp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.141592653589793; /* std::numbers::pi */
static __thread char g_err[256];

/* ------------------------------------------------------------------ */
/* quadrature.hpp                                                      */
/* ------------------------------------------------------------------ */

/* legendre_eval, quadrature.hpp:28-41 */
static void legendre(int n, double x, double* P, double* dP) {
  if (n == 0) {
    *P = 1.0;
    *dP = 0.0;
    return;
  }
  double pm1 = 1.0, dm1 = 0.0, p = x, d = 1.0;
  for (int k = 1; k < n; ++k) {
    const double pk1 = ((2 * k + 1) * x * p - k * pm1) / (k + 1);
    const double dk1 = dm1 + (2 * k + 1) * p;
    pm1 = p;
    dm1 = d;
    p = pk1;
    d = dk1;
  }
  *P = p;
  *dP = d;
}

typedef void (*fn2)(double x, int n, double* f, double* df);

static void f_legendre(double x, int n, double* f, double* df) { legendre(n, x, f, df); }

/* (P'_{n-1}, P''_{n-1}) via the Legendre ODE, quadrature.hpp:236-241 */
static void f_legendre_prime(double x, int n, double* f, double* df) {
  double p, dp;
  legendre(n - 1, x, &p, &dp);
  const double d2p = (2.0 * x * dp - (double)(n - 1) * n * p) / (1.0 - x * x);
  *f = dp;
  *df = d2p;
}

/* bracketed_newton, quadrature.hpp:51-69 (kNodeNewtonMaxIter=100, tol 1e-15) */
static double bracketed_newton(fn2 f, int n, double guess, double lo, double hi) {
  double flo, dummy;
  f(lo, n, &flo, &dummy);
  double x = (guess > lo && guess < hi) ? guess : 0.5 * (lo + hi);
  for (int it = 0; it < 100; ++it) {
    double fx, dfx;
    f(x, n, &fx, &dfx);
    if (fx == 0.0) return x;
    if ((fx > 0.0) == (flo > 0.0))
      lo = x;
    else
      hi = x;
    double xn = x - fx / dfx;
    if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
    const int done = fabs(xn - x) <= 1e-15 && fabs(fx) <= 1e-15;
    x = xn;
    if (done) break;
  }
  return x;
}

/* gl_rule, quadrature.hpp:75-106 */
int or_gl_rule(int n, double* pts, double* wts) {
  if (n < 1) return 1;
  for (int i = 0; i < n; ++i) pts[i] = wts[i] = 0.0;
  const double spacing = kPi / (n + 0.5);
  for (int i = 0; i < n / 2; ++i) {
    const double theta = spacing * (i + 0.75);
    const double guess = -cos(theta);
    const double lo = -cos(theta - 0.5 * spacing);
    const double hi = -cos(theta + 0.5 * spacing);
    const double x = bracketed_newton(f_legendre, n, guess, lo, hi);
    pts[i] = x;
    pts[n - 1 - i] = -x;
  }
  if (n % 2 == 1) pts[n / 2] = 0.0;
  for (int i = 0; i <= (n - 1) / 2; ++i) {
    const double x = pts[i];
    double P, dp;
    legendre(n, x, &P, &dp);
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    wts[i] = w;
    wts[n - 1 - i] = w;
  }
  return 0;
}

/* gll_rule, quadrature.hpp:110-148 */
int or_gll_rule(int n, double* pts, double* wts) {
  if (n < 2) return 1;
  for (int i = 0; i < n; ++i) pts[i] = wts[i] = 0.0;
  pts[0] = -1.0;
  pts[n - 1] = 1.0;
  const int m = n - 2;
  if (m > 0) {
    double* ip = malloc(sizeof(double) * (n - 1));
    double* iw = malloc(sizeof(double) * (n - 1));
    or_gl_rule(n - 1, ip, iw);
    for (int i = 0; i < m / 2; ++i) {
      const double lo = ip[i], hi = ip[i + 1];
      const double guess = -cos(kPi * (i + 1) / (n - 1));
      const double x = bracketed_newton(f_legendre_prime, n, guess, lo, hi);
      pts[1 + i] = x;
      pts[n - 2 - i] = -x;
    }
    if (m % 2 == 1) pts[1 + m / 2] = 0.0;
    free(ip);
    free(iw);
  }
  for (int i = 0; i <= (n - 1) / 2; ++i) {
    const double x = pts[i];
    double P, dp;
    legendre(n - 1, x, &P, &dp);
    const double w = 2.0 / ((double)n * (n - 1) * P * P);
    wts[i] = w;
    wts[n - 1 - i] = w;
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* basis.hpp                                                           */
/* ------------------------------------------------------------------ */

typedef struct {
  int p, n, q, collocated;
  double *npts, *nwts, *qpts, *qwts;
  double *B, *D, *Bt, *Dt; /* B,D: q x n row-major; Bt,Dt: n x q */
} Basis;

/* lagrange_eval, basis.hpp:48-81 */
static void lagrange_eval(const double* x, const double* w, int n, double y, double* values, double* derivs) {
  int at_node = -1;
  for (int j = 0; j < n; ++j)
    if (y == x[j]) at_node = j;
  if (at_node >= 0) {
    const int m = at_node;
    double diag = 0.0;
    for (int j = 0; j < n; ++j) {
      values[j] = (j == m) ? 1.0 : 0.0;
      if (j != m) {
        derivs[j] = (w[j] / w[m]) / (x[m] - x[j]);
        diag -= derivs[j];
      }
    }
    derivs[m] = diag;
    return;
  }
  double s = 0.0, t = 0.0;
  for (int k = 0; k < n; ++k) {
    const double d = y - x[k];
    s += w[k] / d;
    t += w[k] / (d * d);
  }
  for (int j = 0; j < n; ++j) {
    const double d = y - x[j];
    const double lj = (w[j] / d) / s;
    values[j] = lj;
    derivs[j] = lj * (t / s - 1.0 / d);
  }
}

/* build_basis, basis.hpp:86-111 (barycentric weights :34-42) */
static void build_basis(Basis* b, int p, int q, int gll) {
  const int n = p + 1;
  b->p = p;
  b->n = n;
  b->q = q;
  b->collocated = gll && q == p + 1;
  b->npts = malloc(sizeof(double) * n);
  b->nwts = malloc(sizeof(double) * n);
  b->qpts = malloc(sizeof(double) * q);
  b->qwts = malloc(sizeof(double) * q);
  or_gll_rule(n, b->npts, b->nwts);
  if (gll)
    or_gll_rule(q, b->qpts, b->qwts);
  else
    or_gl_rule(q, b->qpts, b->qwts);
  double* bw = malloc(sizeof(double) * n);
  for (int j = 0; j < n; ++j) {
    bw[j] = 1.0;
    for (int k = 0; k < n; ++k)
      if (k != j) bw[j] *= b->npts[j] - b->npts[k];
  }
  for (int j = 0; j < n; ++j) bw[j] = 1.0 / bw[j];
  b->B = malloc(sizeof(double) * q * n);
  b->D = malloc(sizeof(double) * q * n);
  b->Bt = malloc(sizeof(double) * q * n);
  b->Dt = malloc(sizeof(double) * q * n);
  for (int a = 0; a < q; ++a) lagrange_eval(b->npts, bw, n, b->qpts[a], b->B + a * n, b->D + a * n);
  for (int a = 0; a < q; ++a)
    for (int j = 0; j < n; ++j) {
      b->Bt[j * q + a] = b->B[a * n + j];
      b->Dt[j * q + a] = b->D[a * n + j];
    }
  free(bw);
}

static void free_basis(Basis* b) {
  free(b->npts);
  free(b->nwts);
  free(b->qpts);
  free(b->qwts);
  free(b->B);
  free(b->D);
  free(b->Bt);
  free(b->Dt);
}

/* ------------------------------------------------------------------ */
/* tensor.hpp                                                          */
/* ------------------------------------------------------------------ */

/* contract_dim, tensor.hpp:50-114. A is rows x cols row-major. */
static void contract_dim(const double* A, int rows, int cols, int axis, const double* x, const int* xd, double* y,
                         int accumulate) {
  const int m = rows, n = cols;
  const int n0 = xd[0], n1 = xd[1], n2 = xd[2];
  if (axis == 0) {
    const int rest = n1 * n2;
    for (int c = 0; c < rest; ++c) {
      const double* xc = x + (size_t)c * n0;
      double* yc = y + (size_t)c * m;
      for (int a = 0; a < m; ++a) {
        const double* Ar = A + (size_t)a * n;
        double sum = 0.0;
        for (int i = 0; i < n; ++i) sum += Ar[i] * xc[i];
        yc[a] = accumulate ? yc[a] + sum : sum;
      }
    }
  } else if (axis == 1) {
    for (int k = 0; k < n2; ++k) {
      const double* xk = x + (size_t)k * n0 * n1;
      double* yk = y + (size_t)k * n0 * m;
      for (int a = 0; a < m; ++a) {
        double* yrow = yk + (size_t)a * n0;
        if (!accumulate) memset(yrow, 0, sizeof(double) * n0);
        const double* Ar = A + (size_t)a * n;
        for (int j = 0; j < n; ++j) {
          const double c = Ar[j];
          const double* xrow = xk + (size_t)j * n0;
          for (int i = 0; i < n0; ++i) yrow[i] += c * xrow[i];
        }
      }
    }
  } else {
    const int plane = n0 * n1;
    for (int a = 0; a < m; ++a) {
      double* yplane = y + (size_t)a * plane;
      if (!accumulate) memset(yplane, 0, sizeof(double) * plane);
      const double* Ar = A + (size_t)a * n;
      for (int k = 0; k < n; ++k) {
        const double c = Ar[k];
        const double* xplane = x + (size_t)k * plane;
        for (int i = 0; i < plane; ++i) yplane[i] += c * xplane[i];
      }
    }
  }
}

typedef struct {
  double *a, *b, *c, *nodal, *qf[3];
} Scratch; /* ElemScratch, tensor.hpp:118-137 */

static void scratch_init(Scratch* s, int n, int q) {
  const int big = n > q ? n : q;
  const size_t cap = (size_t)big * big * big;
  s->a = malloc(sizeof(double) * cap);
  s->b = malloc(sizeof(double) * cap);
  s->c = malloc(sizeof(double) * cap);
  s->nodal = malloc(sizeof(double) * n * n * n);
  for (int i = 0; i < 3; ++i) s->qf[i] = malloc(sizeof(double) * q * q * q);
}

static void scratch_free(Scratch* s) {
  free(s->a);
  free(s->b);
  free(s->c);
  free(s->nodal);
  for (int i = 0; i < 3; ++i) free(s->qf[i]);
}

/* elem_interp, tensor.hpp:141-152 */
static void elem_interp(const Basis* bs, const double* u, double* out, double* t0, double* t1) {
  const int n = bs->n, q = bs->q;
  if (bs->collocated) {
    memcpy(out, u, sizeof(double) * n * n * n);
    return;
  }
  int d0[3] = {n, n, n}, d1[3] = {q, n, n}, d2[3] = {q, q, n};
  contract_dim(bs->B, q, n, 0, u, d0, t0, 0);
  contract_dim(bs->B, q, n, 1, t0, d1, t1, 0);
  contract_dim(bs->B, q, n, 2, t1, d2, out, 0);
}

/* elem_interp_transpose, tensor.hpp:155-172 */
static void elem_interp_transpose(const Basis* bs, const double* v, double* out, double* t0, double* t1) {
  const int n = bs->n, q = bs->q;
  if (bs->collocated) {
    memcpy(out, v, sizeof(double) * n * n * n);
    return;
  }
  int d0[3] = {q, q, q}, d1[3] = {q, q, n}, d2[3] = {q, n, n};
  contract_dim(bs->Bt, n, q, 2, v, d0, t0, 0);
  contract_dim(bs->Bt, n, q, 1, t0, d1, t1, 0);
  contract_dim(bs->Bt, n, q, 0, t1, d2, out, 0);
}

/* elem_grad, tensor.hpp:177-203 */
static void elem_grad(const Basis* bs, const double* u, double* gr, double* gs, double* gt, Scratch* ws) {
  const int n = bs->n, q = bs->q;
  int nd[3] = {n, n, n};
  if (bs->collocated) {
    contract_dim(bs->D, q, n, 0, u, nd, gr, 0);
    contract_dim(bs->D, q, n, 1, u, nd, gs, 0);
    contract_dim(bs->D, q, n, 2, u, nd, gt, 0);
    return;
  }
  int d1[3] = {q, n, n}, d2[3] = {q, q, n};
  contract_dim(bs->D, q, n, 0, u, nd, ws->a, 0);
  contract_dim(bs->B, q, n, 1, ws->a, d1, ws->b, 0);
  contract_dim(bs->B, q, n, 2, ws->b, d2, gr, 0);
  contract_dim(bs->B, q, n, 0, u, nd, ws->a, 0);
  contract_dim(bs->D, q, n, 1, ws->a, d1, ws->b, 0);
  contract_dim(bs->B, q, n, 2, ws->b, d2, gs, 0);
  contract_dim(bs->B, q, n, 1, ws->a, d1, ws->b, 0);
  contract_dim(bs->D, q, n, 2, ws->b, d2, gt, 0);
}

/* elem_grad_transpose, tensor.hpp:207-235 */
static void elem_grad_transpose(const Basis* bs, const double* gr, const double* gs, const double* gt, double* out,
                                Scratch* ws) {
  const int n = bs->n, q = bs->q;
  int qd[3] = {q, q, q};
  if (bs->collocated) {
    contract_dim(bs->Dt, n, q, 0, gr, qd, out, 0);
    contract_dim(bs->Dt, n, q, 1, gs, qd, out, 1);
    contract_dim(bs->Dt, n, q, 2, gt, qd, out, 1);
    return;
  }
  int d1[3] = {q, q, n}, d2[3] = {q, n, n};
  contract_dim(bs->Bt, n, q, 2, gs, qd, ws->a, 0);
  contract_dim(bs->Dt, n, q, 1, ws->a, d1, ws->b, 0);
  contract_dim(bs->Dt, n, q, 2, gt, qd, ws->c, 0);
  contract_dim(bs->Bt, n, q, 1, ws->c, d1, ws->b, 1);
  contract_dim(bs->Bt, n, q, 0, ws->b, d2, out, 0);
  contract_dim(bs->Bt, n, q, 2, gr, qd, ws->a, 0);
  contract_dim(bs->Bt, n, q, 1, ws->a, d1, ws->b, 0);
  contract_dim(bs->Dt, n, q, 0, ws->b, d2, out, 1);
}

/* ------------------------------------------------------------------ */
/* mesh.hpp / geometry.hpp / operator.hpp                               */
/* ------------------------------------------------------------------ */

typedef struct {
  int bp, p, dims[3], grid[3];
  double amplitude;
  int64_t nL;
  int E, nen, q3, comp;
  Basis basis;
  double* coords; /* 3 per node */
  int* elem_nodes;
  double* factors; /* AoS (e*q3+qp)*comp+c */
  unsigned char* essential;
  int32_t* bdofs;
  int64_t nb;
} Problem;

/* axis_node_coords, mesh.hpp:59-67 */
static void axis_coords(int elems, int p, double length, double* x) {
  double pts[64], wts[64];
  or_gll_rule(p + 1, pts, wts);
  const double h = length / elems;
  for (int e = 0; e < elems; ++e)
    for (int k = 0; k < p; ++k) x[(size_t)e * p + k] = (e + 0.5 * (pts[k] + 1.0)) * h;
  x[(size_t)elems * p] = length;
}

void or_destroy(void* hv) {
  Problem* h = (Problem*)hv;
  if (!h) return;
  free_basis(&h->basis);
  free(h->coords);
  free(h->elem_nodes);
  free(h->factors);
  free(h->essential);
  free(h->bdofs);
  free(h);
}

const char* or_last_error(void) { return g_err; }

/* Element layers [z0, z1) of the (ex, ey, gez) box -- the multi-GPU slab
 * partition's local problem (coordinates from the global box, essential
 * nodes = global box surface only). or_create is the z0 = 0, z1 = gez case. */
void* or_create_slab(int bp, int p, int ex, int ey, int gez, int z0, int z1, double amplitude) {
  const int ez = z1 - z0;
  if (!(bp == 1 || bp == 3 || bp == 5) || p < 1 || p > 16 || ex < 1 || ey < 1 || gez < 1 || z0 < 0 || z1 > gez ||
      ez < 1 || !(amplitude >= 0.0 && amplitude <= 0.15)) {
    snprintf(g_err, sizeof g_err, "or_create: invalid arguments");
    return NULL;
  }
  Problem* h = calloc(1, sizeof(Problem));
  h->bp = bp;
  h->p = p;
  h->dims[0] = ex;
  h->dims[1] = ey;
  h->dims[2] = ez;
  h->amplitude = amplitude;
  for (int d = 0; d < 3; ++d) h->grid[d] = h->dims[d] * p + 1;
  h->nL = (int64_t)h->grid[0] * h->grid[1] * h->grid[2];
  h->E = ex * ey * ez;
  const int n = p + 1;
  h->nen = n * n * n;
  /* default_quad_points / quad_kind_for, operator.hpp:55-56 */
  const int q = bp == 5 ? p + 1 : p + 2;
  build_basis(&h->basis, p, q, bp == 5);
  h->q3 = q * q * q;
  h->comp = bp == 1 ? 1 : 6;

  /* build_box_mesh, mesh.hpp:86-123 */
  double* axis[3];
  const int gdim[3] = {ex, ey, gez};
  for (int d = 0; d < 3; ++d) {
    axis[d] = malloc(sizeof(double) * (gdim[d] * p + 1));
    axis_coords(gdim[d], p, 1.0, axis[d]);
  }
  h->coords = malloc(sizeof(double) * 3 * h->nL);
  for (int kz = 0; kz < h->grid[2]; ++kz)
    for (int ky = 0; ky < h->grid[1]; ++ky)
      for (int kx = 0; kx < h->grid[0]; ++kx) {
        const double x = axis[0][kx], y = axis[1][ky], z = axis[2][kz + z0 * p];
        double disp = 0.0;
        if (amplitude > 0.0)
          disp = amplitude * sin(2.0 * kPi * x / 1.0) * sin(2.0 * kPi * y / 1.0) * sin(2.0 * kPi * z / 1.0);
        const size_t g = (size_t)kx + (size_t)h->grid[0] * (ky + (size_t)h->grid[1] * kz);
        h->coords[3 * g + 0] = x + 1.0 * disp;
        h->coords[3 * g + 1] = y + 1.0 * disp;
        h->coords[3 * g + 2] = z + 1.0 * disp;
      }
  for (int d = 0; d < 3; ++d) free(axis[d]);
  /* fill_elem_nodes, mesh.hpp:71-82 */
  h->elem_nodes = malloc(sizeof(int) * (size_t)h->E * h->nen);
  size_t pos = 0;
  for (int ez_ = 0; ez_ < ez; ++ez_)
    for (int ey_ = 0; ey_ < ey; ++ey_)
      for (int ex_ = 0; ex_ < ex; ++ex_)
        for (int k = 0; k <= p; ++k)
          for (int j = 0; j <= p; ++j)
            for (int i = 0; i <= p; ++i)
              h->elem_nodes[pos++] = (ex_ * p + i) + h->grid[0] * ((ey_ * p + j) + h->grid[1] * (ez_ * p + k));

  /* boundary_nodes, mesh.hpp:126-135 */
  h->essential = calloc((size_t)h->nL, 1);
  int64_t nb = 0;
  for (int kz = 0; kz < h->grid[2]; ++kz)
    for (int ky = 0; ky < h->grid[1]; ++ky)
      for (int kx = 0; kx < h->grid[0]; ++kx)
        if (kx == 0 || kx == h->grid[0] - 1 || ky == 0 || ky == h->grid[1] - 1 || kz + z0 * p == 0 ||
            kz + z0 * p == gez * p) {
          h->essential[kx + (size_t)h->grid[0] * (ky + (size_t)h->grid[1] * kz)] = 1;
          ++nb;
        }
  h->nb = nb;
  h->bdofs = malloc(sizeof(int32_t) * (nb ? nb : 1));
  nb = 0;
  for (int64_t g = 0; g < h->nL; ++g)
    if (h->essential[g]) h->bdofs[nb++] = (int32_t)g;

  /* compute_jacobians + mass_factors/diffusion_factors, geometry.hpp:78-193 */
  const int q3 = h->q3;
  h->factors = malloc(sizeof(double) * (size_t)h->E * q3 * h->comp);
  int bad_elem = -1, bad_qpt = -1;
  double bad_det = 0.0;
#pragma omp parallel
  {
    Scratch ws;
    scratch_init(&ws, n, q);
    double* J = malloc(sizeof(double) * q3 * 9);
#pragma omp for schedule(static)
    for (int e = 0; e < h->E; ++e) {
      const int* nodes = h->elem_nodes + (size_t)e * h->nen;
      for (int c = 0; c < 3; ++c) {
        for (int i = 0; i < h->nen; ++i) ws.nodal[i] = h->coords[3 * (size_t)nodes[i] + c];
        elem_grad(&h->basis, ws.nodal, ws.qf[0], ws.qf[1], ws.qf[2], &ws);
        for (int qp = 0; qp < q3; ++qp)
          for (int d = 0; d < 3; ++d) J[qp * 9 + c * 3 + d] = ws.qf[d][qp];
      }
      for (int qp = 0; qp < q3; ++qp) {
        const double* j = J + qp * 9;
        const double det =
            j[0] * (j[4] * j[8] - j[5] * j[7]) - j[1] * (j[3] * j[8] - j[5] * j[6]) + j[2] * (j[3] * j[7] - j[4] * j[6]);
        if (!(det > 0.0)) {
#pragma omp critical
          {
            if (bad_elem < 0 || e < bad_elem) {
              bad_elem = e;
              bad_qpt = qp;
              bad_det = det;
            }
          }
        }
        const int a = qp % q, b = (qp / q) % q, cc = qp / (q * q);
        const double w = h->basis.qwts[a] * h->basis.qwts[b] * h->basis.qwts[cc]; /* tensor_weight :139-143 */
        const size_t idx = (size_t)e * q3 + qp;
        if (h->comp == 1) {
          h->factors[idx] = w * det;
        } else {
          const double inv[9] = {(j[4] * j[8] - j[5] * j[7]) / det, (j[2] * j[7] - j[1] * j[8]) / det,
                                 (j[1] * j[5] - j[2] * j[4]) / det, (j[5] * j[6] - j[3] * j[8]) / det,
                                 (j[0] * j[8] - j[2] * j[6]) / det, (j[2] * j[3] - j[0] * j[5]) / det,
                                 (j[3] * j[7] - j[4] * j[6]) / det, (j[1] * j[6] - j[0] * j[7]) / det,
                                 (j[0] * j[4] - j[1] * j[3]) / det};
          double* g = h->factors + idx * 6;
          int c = 0;
          for (int r = 0; r < 3; ++r)
            for (int s = r; s < 3; ++s) {
              double dot = 0.0;
              for (int k = 0; k < 3; ++k) dot += inv[r * 3 + k] * inv[s * 3 + k];
              g[c++] = w * det * dot;
            }
        }
      }
    }
    free(J);
    scratch_free(&ws);
  }
  if (bad_elem >= 0) {
    snprintf(g_err, sizeof g_err,
             "non-positive Jacobian determinant %f at element %d, quadrature point %d", bad_det, bad_elem, bad_qpt);
    or_destroy(h);
    return NULL;
  }
  return h;
}

void* or_create(int bp, int p, int ex, int ey, int ez, double amplitude) {
  return or_create_slab(bp, p, ex, ey, ez, 0, ez, amplitude);
}

int64_t or_size(void* h) { return ((Problem*)h)->nL; }
int or_num_elements(void* h) { return ((Problem*)h)->E; }
int or_q(void* h) { return ((Problem*)h)->basis.q; }
int or_components(void* h) { return ((Problem*)h)->comp; }
int64_t or_num_boundary(void* h) { return ((Problem*)h)->nb; }
void or_boundary(void* hv, int32_t* out) {
  Problem* h = hv;
  memcpy(out, h->bdofs, sizeof(int32_t) * h->nb);
}
void or_basis(void* hv, double* B, double* D) {
  Problem* h = hv;
  memcpy(B, h->basis.B, sizeof(double) * h->basis.q * h->basis.n);
  memcpy(D, h->basis.D, sizeof(double) * h->basis.q * h->basis.n);
}
void or_rules(void* hv, double* qp, double* qw, double* np, double* nw) {
  Problem* h = hv;
  memcpy(qp, h->basis.qpts, sizeof(double) * h->basis.q);
  memcpy(qw, h->basis.qwts, sizeof(double) * h->basis.q);
  memcpy(np, h->basis.npts, sizeof(double) * h->basis.n);
  memcpy(nw, h->basis.nwts, sizeof(double) * h->basis.n);
}
void or_factors(void* hv, double* out) {
  Problem* h = hv;
  memcpy(out, h->factors, sizeof(double) * (size_t)h->E * h->q3 * h->comp);
}
void or_coords(void* hv, double* out) {
  Problem* h = hv;
  memcpy(out, h->coords, sizeof(double) * 3 * h->nL);
}

/* Fused apply: element_apply (operator.hpp:217-236) per element into an
 * E-vector, then scatter_add (restriction.hpp:67-80). Summing E-vector
 * slots in ascending order per dof equals accumulating elements in
 * ascending order from 0.0, which is what the second loop does. */
static void apply_raw(Problem* h, const double* u, double* w) {
  const int n = h->basis.n, q3 = h->q3, nen = h->nen;
  double* ev = malloc(sizeof(double) * (size_t)h->E * nen);
#pragma omp parallel
  {
    Scratch ws;
    scratch_init(&ws, n, h->basis.q);
#pragma omp for schedule(static)
    for (int e = 0; e < h->E; ++e) {
      const int* gids = h->elem_nodes + (size_t)e * nen;
      for (int i = 0; i < nen; ++i) ws.nodal[i] = u[gids[i]];
      const double* f = h->factors + (size_t)e * q3 * h->comp;
      if (h->comp == 6) {
        elem_grad(&h->basis, ws.nodal, ws.qf[0], ws.qf[1], ws.qf[2], &ws);
        /* apply_diffusion_factors, operator.hpp:124-137 */
        for (int qp = 0; qp < q3; ++qp) {
          const double* g = f + (size_t)qp * 6;
          const double r = ws.qf[0][qp], s = ws.qf[1][qp], t = ws.qf[2][qp];
          ws.qf[0][qp] = g[0] * r + g[1] * s + g[2] * t;
          ws.qf[1][qp] = g[1] * r + g[3] * s + g[4] * t;
          ws.qf[2][qp] = g[2] * r + g[4] * s + g[5] * t;
        }
        elem_grad_transpose(&h->basis, ws.qf[0], ws.qf[1], ws.qf[2], ws.nodal, &ws);
      } else {
        elem_interp(&h->basis, ws.nodal, ws.qf[0], ws.a, ws.b);
        for (int qp = 0; qp < q3; ++qp) ws.qf[0][qp] *= f[qp]; /* apply_mass_factors :139-142 */
        elem_interp_transpose(&h->basis, ws.qf[0], ws.nodal, ws.a, ws.b);
      }
      memcpy(ev + (size_t)e * nen, ws.nodal, sizeof(double) * nen);
    }
    scratch_free(&ws);
  }
  memset(w, 0, sizeof(double) * h->nL);
  for (int e = 0; e < h->E; ++e) {
    const int* gids = h->elem_nodes + (size_t)e * nen;
    const double* ve = ev + (size_t)e * nen;
    for (int i = 0; i < nen; ++i) w[gids[i]] += ve[i];
  }
  free(ev);
}

/* ConstrainedOperator::apply, solver.hpp:60-65 */
int or_apply(void* hv, int constrained, const double* u, double* w) {
  Problem* h = hv;
  if (!constrained) {
    apply_raw(h, u, w);
    return 0;
  }
  double* s = malloc(sizeof(double) * h->nL);
  memcpy(s, u, sizeof(double) * h->nL);
  for (int64_t i = 0; i < h->nb; ++i) s[h->bdofs[i]] = 0.0;
  apply_raw(h, s, w);
  for (int64_t i = 0; i < h->nb; ++i) w[h->bdofs[i]] = u[h->bdofs[i]];
  free(s);
  return 0;
}

/* deterministic_dot, dense.hpp:52-81 (kReductionBlock = 4096) */
double or_dot(const double* a, const double* b, int64_t n) {
  const int64_t nb = (n + 4095) / 4096;
  double sum = 0.0;
  for (int64_t blk = 0; blk < nb; ++blk) {
    const int64_t lo = blk * 4096, hi = lo + 4096 < n ? lo + 4096 : n;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i) s += a[i] * b[i];
    sum += s;
  }
  return sum;
}

/* cg without preconditioner, solver.hpp:91-153 */
int or_cg(void* hv, int constrained, const double* b, double* x, double rel_tol, int max_iter, int* iterations,
          int* converged, double* final_rel, double* history) {
  Problem* h = hv;
  const int64_t n = h->nL;
  double* r = malloc(sizeof(double) * n);
  double* p = malloc(sizeof(double) * n);
  double* Ap = malloc(sizeof(double) * n);
  int status = 0;
  *iterations = 0;
  *converged = 0;
  or_apply(h, constrained, x, Ap);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - Ap[i];
  const double r0 = sqrt(or_dot(r, r, n));
  int hl = 0;
  history[hl++] = r0;
  if (!isfinite(r0)) {
    status = 2;
    goto done;
  }
  if (r0 == 0.0) {
    *converged = 1;
    *final_rel = 0.0;
    goto done;
  }
  memcpy(p, r, sizeof(double) * n);
  double rz = or_dot(r, r, n);
  for (int k = 1; k <= max_iter; ++k) {
    or_apply(h, constrained, p, Ap);
    const double pAp = or_dot(p, Ap, n);
    if (!isfinite(pAp) || pAp <= 0.0) {
      status = 2;
      goto done;
    }
    const double alpha = rz / pAp;
    for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
    for (int64_t i = 0; i < n; ++i) r[i] -= alpha * Ap[i];
    const double rnorm = sqrt(or_dot(r, r, n));
    if (!isfinite(rnorm)) {
      status = 2;
      goto done;
    }
    history[hl++] = rnorm;
    *iterations = k;
    if (rnorm / r0 <= rel_tol) {
      *converged = 1;
      break;
    }
    const double rz_next = or_dot(r, r, n);
    const double beta = rz_next / rz;
    rz = rz_next;
    for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
  }
  *final_rel = history[hl - 1] / r0;
done:
  free(r);
  free(p);
  free(Ap);
  return status;
}

/* jacobi_diagonal, solver.hpp:155-205: element diagonals (loops k, j, i over
 * nodes, c, b, a over quadrature points, the reference's expression order)
 * scattered with scatter_add's ascending-slot order; constrained: 1 on the
 * essential dofs (solver.hpp:200-205). */
void or_jacobi_diagonal(void* hv, int constrained, double* out) {
  Problem* h = hv;
  const Basis* bs = &h->basis;
  const int n = bs->n, q = bs->q, nen = h->nen;
  const int diff = h->bp != 1;
  double* de = malloc(sizeof(double) * nen);
  memset(out, 0, sizeof(double) * h->nL);
#define BB(a, i) bs->B[(a) * n + (i)]
#define DD(a, i) bs->D[(a) * n + (i)]
  for (int e = 0; e < h->E; ++e) {
    const double* f = h->factors + (size_t)e * h->q3 * h->comp;
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          double sum = 0.0;
          for (int c = 0; c < q; ++c)
            for (int b = 0; b < q; ++b)
              for (int a = 0; a < q; ++a) {
                const int qp = a + q * (b + q * c);
                if (diff) {
                  const double* g = f + (size_t)qp * 6;
                  const double dr = DD(a, i) * BB(b, j) * BB(c, k);
                  const double ds = BB(a, i) * DD(b, j) * BB(c, k);
                  const double dt = BB(a, i) * BB(b, j) * DD(c, k);
                  sum += g[0] * dr * dr + g[3] * ds * ds + g[5] * dt * dt +
                         2.0 * (g[1] * dr * ds + g[2] * dr * dt + g[4] * ds * dt);
                } else {
                  const double phi = BB(a, i) * BB(b, j) * BB(c, k);
                  sum += f[qp] * phi * phi;
                }
              }
          de[i + n * (j + n * k)] = sum;
        }
    /* scatter_add (restriction.hpp:67-80): ascending slots = ascending e */
    const int* nodes = h->elem_nodes + (size_t)e * nen;
    for (int l = 0; l < nen; ++l) out[nodes[l]] += de[l];
  }
#undef BB
#undef DD
  free(de);
  if (constrained)
    for (int64_t i = 0; i < h->nb; ++i) out[h->bdofs[i]] = 1.0;
}

/* cg with the optional Jacobi preconditioner z = r / diag (solver.hpp:91-153);
 * diag == NULL is or_cg. */
int or_pcg(void* hv, int constrained, const double* b, double* x, const double* diag, double rel_tol, int max_iter,
           int* iterations, int* converged, double* final_rel, double* history) {
  Problem* h = hv;
  const int64_t n = h->nL;
  double* r = malloc(sizeof(double) * n);
  double* z = malloc(sizeof(double) * n);
  double* p = malloc(sizeof(double) * n);
  double* Ap = malloc(sizeof(double) * n);
  int status = 0;
  *iterations = 0;
  *converged = 0;
  or_apply(h, constrained, x, Ap);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - Ap[i];
  const double r0 = sqrt(or_dot(r, r, n));
  int hl = 0;
  history[hl++] = r0;
  if (!isfinite(r0)) {
    status = 2;
    goto done;
  }
  if (r0 == 0.0) {
    *converged = 1;
    *final_rel = 0.0;
    goto done;
  }
  for (int64_t i = 0; i < n; ++i) z[i] = diag ? r[i] / diag[i] : r[i];
  memcpy(p, z, sizeof(double) * n);
  double rz = or_dot(r, z, n);
  for (int k = 1; k <= max_iter; ++k) {
    or_apply(h, constrained, p, Ap);
    const double pAp = or_dot(p, Ap, n);
    if (!isfinite(pAp) || pAp <= 0.0) {
      status = 2;
      goto done;
    }
    const double alpha = rz / pAp;
    for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
    for (int64_t i = 0; i < n; ++i) r[i] -= alpha * Ap[i];
    const double rnorm = sqrt(or_dot(r, r, n));
    if (!isfinite(rnorm)) {
      status = 2;
      goto done;
    }
    history[hl++] = rnorm;
    *iterations = k;
    if (rnorm / r0 <= rel_tol) {
      *converged = 1;
      break;
    }
    for (int64_t i = 0; i < n; ++i) z[i] = diag ? r[i] / diag[i] : r[i];
    const double rz_next = or_dot(r, z, n);
    const double beta = rz_next / rz;
    rz = rz_next;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  *final_rel = history[hl - 1] / r0;
done:
  free(r);
  free(z);
  free(p);
  free(Ap);
  return status;
}

/* ------------------------------------------------------------------ */
/* seeded inputs: std::mt19937_64 + uniform_real_distribution(-1,1)    */
/* (libstdc++ generate_canonical with one 64-bit draw)                 */
/* ------------------------------------------------------------------ */

typedef struct {
  uint64_t mt[312];
  int mti;
} Mt64;

static void mt_seed(Mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

static uint64_t mt_next(Mt64* s) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i - 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    s->mti = 0;
  }
  uint64_t y = s->mt[s->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

static double uniform_m1_1(Mt64* s) {
  double c = (double)mt_next(s) * 1.0 / 18446744073709551616.0;
  if (c >= 1.0) c = nextafter(1.0, 0.0);
  return c * (1.0 - -1.0) + -1.0;
}

void or_random_vector(uint64_t seed, int64_t n, double* out) {
  Mt64 s;
  mt_seed(&s, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = uniform_m1_1(&s);
}

/* detail::mix_seed, bench.hpp:193-204 (BPKind enum values 0,1,2) */
uint64_t or_mix_seed(uint64_t seed, int bp, int p, int ex, int ey, int ez) {
  uint64_t h = seed ^ 0x9e3779b97f4a7c15ULL;
  const uint64_t vals[5] = {(uint64_t)(bp == 1 ? 0 : (bp == 3 ? 1 : 2)), (uint64_t)p, (uint64_t)ex, (uint64_t)ey,
                            (uint64_t)ez};
  for (int i = 0; i < 5; ++i) {
    h ^= vals[i] + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdULL;
    h ^= h >> 33;
  }
  return h;
}

/* bench RHS, bench.hpp:234-243 */
void or_bench_rhs(void* hv, uint64_t seed, double* b) {
  Problem* h = hv;
  or_random_vector(or_mix_seed(seed, h->bp, h->p, h->dims[0], h->dims[1], h->dims[2]), h->nL, b);
  if (h->bp != 1)
    for (int64_t i = 0; i < h->nb; ++i) b[h->bdofs[i]] = 0.0;
}
