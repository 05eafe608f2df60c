// Host-side 1D tables for the device setup: Gauss / Gauss-Lobatto rules and
// the Lagrange interpolation/differentiation tables on GLL nodes. These feed
// the kernels as a few hundred bytes of kernel parameters.
//
// The algorithms are the ones the reference uses (quadrature.hpp:28-148,
// basis.hpp:34-111, mesh.hpp:59-67), evaluated in the same operation order
// so the device setup reproduces the reference's factors bit for bit.
#include <cmath>
#include <stdexcept>
#include <utility>
#include <vector>

#include "internal.h"

namespace hxb {
namespace {

constexpr double kPi = 3.141592653589793;

std::pair<double, double> legendre(int n, double x) {  // quadrature.hpp:28-41
  if (n == 0) return {1.0, 0.0};
  double pm1 = 1.0, dm1 = 0.0, p = x, d = 1.0;
  for (int k = 1; k < n; ++k) {
    const double pk1 = ((2 * k + 1) * x * p - k * pm1) / (k + 1);
    const double dk1 = dm1 + (2 * k + 1) * p;
    pm1 = p;
    dm1 = d;
    p = pk1;
    d = dk1;
  }
  return {p, d};
}

template <class F>
double newton_bracketed(F&& f, double guess, double lo, double hi) {  // quadrature.hpp:51-69
  const double flo = f(lo).first;
  double x = (guess > lo && guess < hi) ? guess : 0.5 * (lo + hi);
  for (int it = 0; it < 100; ++it) {
    const auto [fx, dfx] = f(x);
    if (fx == 0.0) return x;
    if ((fx > 0.0) == (flo > 0.0))
      lo = x;
    else
      hi = x;
    double xn = x - fx / dfx;
    if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
    const bool done = std::abs(xn - x) <= 1e-15 && std::abs(fx) <= 1e-15;
    x = xn;
    if (done) break;
  }
  return x;
}

}  // namespace

void gl_rule(int n, double* pts, double* wts) {  // quadrature.hpp:75-106
  if (n < 1) throw std::invalid_argument("gl_rule: need at least 1 point");
  for (int i = 0; i < n; ++i) pts[i] = wts[i] = 0.0;
  const double spacing = kPi / (n + 0.5);
  auto f = [n](double x) { return legendre(n, x); };
  for (int i = 0; i < n / 2; ++i) {
    const double theta = spacing * (i + 0.75);
    const double x = newton_bracketed(f, -std::cos(theta), -std::cos(theta - 0.5 * spacing),
                                      -std::cos(theta + 0.5 * spacing));
    pts[i] = x;
    pts[n - 1 - i] = -x;
  }
  if (n % 2 == 1) pts[n / 2] = 0.0;
  for (int i = 0; i <= (n - 1) / 2; ++i) {
    const double x = pts[i];
    const double dp = legendre(n, x).second;
    wts[i] = wts[n - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
}

void gll_rule(int n, double* pts, double* wts) {  // quadrature.hpp:110-148
  if (n < 2) throw std::invalid_argument("gll_rule: need at least 2 points");
  for (int i = 0; i < n; ++i) pts[i] = wts[i] = 0.0;
  pts[0] = -1.0;
  pts[n - 1] = 1.0;
  const int m = n - 2;
  if (m > 0) {
    std::vector<double> ip(n - 1), iw(n - 1);
    gl_rule(n - 1, ip.data(), iw.data());
    auto fprime = [n](double x) {
      const auto [p, dp] = legendre(n - 1, x);
      const double d2p = (2.0 * x * dp - static_cast<double>(n - 1) * n * p) / (1.0 - x * x);
      return std::pair<double, double>{dp, d2p};
    };
    for (int i = 0; i < m / 2; ++i) {
      const double x = newton_bracketed(fprime, -std::cos(kPi * (i + 1) / (n - 1)), ip[i], ip[i + 1]);
      pts[1 + i] = x;
      pts[n - 2 - i] = -x;
    }
    if (m % 2 == 1) pts[1 + m / 2] = 0.0;
  }
  for (int i = 0; i <= (n - 1) / 2; ++i) {
    const double p = legendre(n - 1, pts[i]).first;
    wts[i] = wts[n - 1 - i] = 2.0 / (static_cast<double>(n) * (n - 1) * p * p);
  }
}

void build_basis(int p, int q, bool gll, double* B, double* D, double* qpts, double* qwts, double* npts,
                 double* nwts) {  // basis.hpp:86-111
  const int n = p + 1;
  gll_rule(n, npts, nwts);
  if (gll)
    gll_rule(q, qpts, qwts);
  else
    gl_rule(q, qpts, qwts);
  std::vector<double> bw(n, 1.0);  // barycentric weights, basis.hpp:34-42
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      if (k != j) bw[j] *= npts[j] - npts[k];
  for (double& v : bw) v = 1.0 / v;
  for (int a = 0; a < q; ++a) {  // lagrange_eval, basis.hpp:48-81
    double* vals = B + a * n;
    double* ders = D + a * n;
    const double y = qpts[a];
    int at = -1;
    for (int j = 0; j < n; ++j)
      if (y == npts[j]) at = j;
    if (at >= 0) {
      double diag = 0.0;
      for (int j = 0; j < n; ++j) {
        vals[j] = (j == at) ? 1.0 : 0.0;
        if (j != at) {
          ders[j] = (bw[j] / bw[at]) / (npts[at] - npts[j]);
          diag -= ders[j];
        }
      }
      ders[at] = diag;
      continue;
    }
    double s = 0.0, t = 0.0;
    for (int k = 0; k < n; ++k) {
      const double d = y - npts[k];
      s += bw[k] / d;
      t += bw[k] / (d * d);
    }
    for (int j = 0; j < n; ++j) {
      const double d = y - npts[j];
      const double lj = (bw[j] / d) / s;
      vals[j] = lj;
      ders[j] = lj * (t / s - 1.0 / d);
    }
  }
}

std::vector<double> axis_node_coords(int elems, int p, double length) {  // mesh.hpp:59-67
  std::vector<double> pts(p + 1), wts(p + 1);
  gll_rule(p + 1, pts.data(), wts.data());
  const double h = length / elems;
  std::vector<double> x(static_cast<std::size_t>(elems) * p + 1);
  for (int e = 0; e < elems; ++e)
    for (int k = 0; k < p; ++k) x[static_cast<std::size_t>(e) * p + k] = (e + 0.5 * (pts[k] + 1.0)) * h;
  x.back() = length;
  return x;
}

}  // namespace hxb

// ---------------------------------------------------------------------------
// Benchmark right-hand side (bench.hpp:193-204, 234-243).
#include <random>

extern "C" int hexbp_bench_rhs(int bp, int p, const int dims[3], uint64_t seed, int64_t offset, int64_t count,
                               double* out) {
  if (!dims || !out || p < 1 || !(bp == 1 || bp == 3 || bp == 5)) {
    hxb::set_error("bench_rhs: invalid argument");
    return HEXBP_INVALID_ARGUMENT;
  }
  const int64_t g[3] = {static_cast<int64_t>(dims[0]) * p + 1, static_cast<int64_t>(dims[1]) * p + 1,
                        static_cast<int64_t>(dims[2]) * p + 1};
  const int64_t n = g[0] * g[1] * g[2];
  if (offset < 0 || count < 0 || offset + count > n) {
    hxb::set_error("bench_rhs: range outside the L-vector");
    return HEXBP_INVALID_ARGUMENT;
  }
  // detail::mix_seed with BPKind values BP1=0, BP3=1, BP5=2.
  uint64_t h = seed ^ 0x9e3779b97f4a7c15ull;
  auto mix = [&h](uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
  };
  mix(static_cast<uint64_t>(bp == 1 ? 0 : (bp == 3 ? 1 : 2)));
  mix(static_cast<uint64_t>(p));
  for (int d = 0; d < 3; ++d) mix(static_cast<uint64_t>(dims[d]));
  std::mt19937_64 rng(h);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int64_t i = 0; i < offset; ++i) (void)dist(rng);
  for (int64_t i = 0; i < count; ++i) out[i] = dist(rng);
  if (bp != 1) {  // homogeneous essential BCs on the box surface (mesh.hpp:126-135)
    for (int64_t i = 0; i < count; ++i) {
      const int64_t gi = offset + i;
      const int64_t kx = gi % g[0], ky = (gi / g[0]) % g[1], kz = gi / (g[0] * g[1]);
      if (kx == 0 || kx == g[0] - 1 || ky == 0 || ky == g[1] - 1 || kz == 0 || kz == g[2] - 1) out[i] = 0.0;
    }
  }
  return HEXBP_OK;
}

// std::mt19937_64(seed) + uniform_real_distribution<double>(lo, hi): the
// probe vectors of check_equivalence (verify.hpp:64-70), same libstdc++ draws.
extern "C" int hexbp_uniform_stream(uint64_t seed, double lo, double hi, int64_t count, double* out) {
  if (!out || count < 0 || !(lo < hi)) {
    hxb::set_error("uniform_stream: invalid argument");
    return HEXBP_INVALID_ARGUMENT;
  }
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (int64_t i = 0; i < count; ++i) out[i] = dist(rng);
  return HEXBP_OK;
}

