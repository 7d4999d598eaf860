// window.cu -- plan-time fit of the per-tap window polynomials (host code).
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "window.cuh"

namespace sfb {

namespace {

typedef long double ld;

// the reference's stable sinh form (windows.py:111-115), in 80-bit precision
ld omega_ld(ld x, ld beta) {
  if (!(fabsl(x) < 1.0L)) return 0.0L;
  ld s = sqrtl(fmaxl(0.0L, 1.0L - x * x));
  return expl(beta * (s - 1.0L)) * (-expm1l(-2.0L * beta * s)) / (-expm1l(-2.0L * beta));
}

// Chebyshev interpolation of f on [-1,1] at p+1 first-kind nodes, returned as
// monomial coefficients a[0..p] (long double).
template <class F>
std::vector<ld> fit_monomial(F f, int p) {
  const ld pi = 3.141592653589793238462643383279502884L;
  const int n = p + 1;
  std::vector<ld> fx(n), c(n, 0.0L);
  for (int k = 0; k < n; ++k) fx[k] = f(cosl(pi * (k + 0.5L) / n));
  for (int j = 0; j < n; ++j) {
    ld s = 0;
    for (int k = 0; k < n; ++k) s += fx[k] * cosl(pi * j * (k + 0.5L) / n);
    c[j] = s * 2.0L / n;
  }
  c[0] *= 0.5L;
  // Chebyshev -> monomial via T_{j+1} = 2u T_j - T_{j-1}
  std::vector<ld> a(n, 0.0L), tm(n, 0.0L), t0(n, 0.0L), t1(n, 0.0L);
  t0[0] = 1.0L;
  if (n > 1) t1[1] = 1.0L;
  for (int i = 0; i < n; ++i) a[i] += c[0] * t0[i];
  if (n > 1)
    for (int i = 0; i < n; ++i) a[i] += c[1] * t1[i];
  for (int j = 2; j < n; ++j) {
    for (int i = 0; i < n; ++i) tm[i] = -t0[i] + (i > 0 ? 2.0L * t1[i - 1] : 0.0L);
    for (int i = 0; i < n; ++i) a[i] += c[j] * tm[i];
    t0 = t1;
    t1 = tm;
  }
  return a;
}

template <int M>
double validate(const WinCoef& C, ld beta) {
  double w[2 * M];
  double worst = 0.0;
  const int G = 4096;
  for (int i = 0; i <= G; ++i) {
    double d = (double)i / G;
    if (d >= 1.0) d = 0.99999999999999989;  // d lies in [0, 1)
    window_taps<M>(C, d, w);
    for (int t = 1 - M; t <= M; ++t) {
      ld ref = omega_ld(((ld)t - (ld)d) / (ld)M, beta);
      double err = fabs((double)((ld)w[t + M - 1] - ref));
      if (err > worst) worst = err;
    }
  }
  return worst;
}

template <int M>
double validate_dispatch(const WinCoef& C, ld beta) {
  return validate<M>(C, beta);
}

double validate_m(int m, const WinCoef& C, ld beta) {
  switch (m) {
#define SF_V(MM) \
  case MM:       \
    return validate_dispatch<MM>(C, beta);
    SF_V(2) SF_V(3) SF_V(4) SF_V(5) SF_V(6) SF_V(7) SF_V(8) SF_V(9) SF_V(10) SF_V(11) SF_V(12)
    SF_V(13) SF_V(14) SF_V(15) SF_V(16)
#undef SF_V
  }
  return 1.0;
}

}  // namespace

namespace {
WinCoef fit_window_uncached(int m, double beta_d, double* max_err_out);
struct FitCache {
  std::mutex mu;
  std::map<std::pair<int, double>, std::pair<WinCoef, double>> fits;
};
FitCache& fit_cache() {
  static FitCache c;
  return c;
}
}  // namespace

// The fit and its long-double validation (~10 ms) depend only on (m, beta):
// memoised per process, so plans that repeat a window (the CLI's thousands of
// small plans, sinc plans, adjoint sub-plans) pay for it once.
WinCoef fit_window(int m, double beta_d, double* max_err_out) {
  FitCache& c = fit_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.fits.find({m, beta_d});
    if (it != c.fits.end()) {
      if (max_err_out) *max_err_out = it->second.second;
      return it->second.first;
    }
  }
  double err = 0.0;
  const WinCoef w = fit_window_uncached(m, beta_d, &err);  // throws on bad m
  std::lock_guard<std::mutex> lk(c.mu);
  c.fits.emplace(std::make_pair(m, beta_d), std::make_pair(w, err));
  if (max_err_out) *max_err_out = err;
  return w;
}

namespace {
WinCoef fit_window_uncached(int m, double beta_d, double* max_err_out) {
  if (m < 2 || m > kMaxM)
    fail(5, "window cut-off m=" + std::to_string(m) + " outside the supported range [2, 16]");
  WinCoef C;
  std::memset(&C, 0, sizeof(C));
  const int P = window_degree(m);
  const int NE = P / 2 + 1, NO = (P + 1) / 2;
  const ld beta = (ld)beta_d;
  const ld M = (ld)m;
  for (int q = 0; q < m; ++q) {
    std::vector<ld> a;
    if (q < m - 1) {
      const ld t = (ld)(q + 1);
      a = fit_monomial([&](ld u) { return omega_ld((t - 0.5L * (u + 1.0L)) / M, beta); }, P);
    } else {
      // edge: g_m(d) = sqrt(d) H(u); H = g_m / sqrt(d), analytic on [-1, 1]
      a = fit_monomial(
          [&](ld u) {
            ld d = 0.5L * (u + 1.0L);
            return omega_ld((M - d) / M, beta) / sqrtl(d);
          },
          P);
    }
    for (int k = 0; k < NE; ++k) C.e[q][k] = (double)a[2 * k];
    for (int k = 0; k < NO; ++k) C.o[q][k] = (double)a[2 * k + 1];
  }
  const double err = validate_m(m, C, beta);
  if (max_err_out) *max_err_out = err;
  if (!(err <= 5e-15))
    fail(5, "window polynomial validation failed for m=" + std::to_string(m) +
                " (max error " + std::to_string(err) + ")");
  return C;
}
}  // namespace

}  // namespace sfb

// ---------------------------------------------------------------------------
// Public window evaluation (drop-in for windows.py's omega_eval, omega_hat_eval,
// phi_eval, phi_hat_eval, sinh kind): the reference's closed forms evaluated
// elementwise on the device -- not the per-tap polynomials of the hot path.
namespace sfb {

// omega(x) = e^{beta(s-1)} (1 - e^{-2 beta s}) / (1 - e^{-2 beta}),
// s = sqrt(max(0, 1 - x^2)), zero unless |x| < 1   (windows.py:106-125)
__device__ inline double omega_sinh(double beta, double x) {
  if (!(fabs(x) < 1.0)) return 0.0;
  // x*x rounded on its own (no fused 1 - x*x): the reference's numpy rounding,
  // which matters near |x| = 1 where 1 - x^2 cancels
  const double s = sqrt(fmax(0.0, 1.0 - __dmul_rn(x, x)));
  return exp(beta * (s - 1.0)) * (-expm1(-2.0 * beta * s)) / (-expm1(-2.0 * beta));
}

__global__ void k_window_eval(int func, double beta, double scale, const double* __restrict__ x,
                              int64_t n, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double xi = x[i];
  double r;
  switch (func) {
    case 0: r = omega_sinh(beta, xi); break;               // omega_eval
    case 1: r = omega_hat_sinh(beta, xi); break;           // omega_hat_eval
    case 2: r = omega_sinh(beta, xi * scale); break;       // phi_eval: scale = n_grid/m
    default: r = scale * omega_hat_sinh(beta, xi * scale); // phi_hat_eval: scale = m/n_grid
  }
  out[i] = r;
}

void run_window_eval(int func, double beta, int m, int64_t n_grid, const double* x, int64_t n,
                     double* out, cudaStream_t s) {
  // the quotients are formed first, as in windows.py:212-220
  const double scale = func == 2 ? (double)n_grid / (double)m
                     : func == 3 ? (double)m / (double)n_grid : 1.0;
  if (n <= 0) return;
  const int T = 256;
  k_window_eval<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(func, beta, scale, x, n, out);
  SF_LAUNCH_CHECK();
}

}  // namespace sfb
