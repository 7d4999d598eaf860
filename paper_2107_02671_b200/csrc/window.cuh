// window.cuh -- the sinh-type window of arXiv 2107.02671 on the device.
//
// Reference: omega(x) = sinh(beta sqrt(1-x^2)) / sinh(beta) on |x| < 1, zero
// outside, beta = 2 pi m (1 - 1/(2 sigma)) (pkg/src/sincfft/windows.py:94-95,
// 109-124), applied on a grid as phi(t) = omega(n_grid t / m) (windows.py:
// 212-214); its Fourier transform through I1 (windows.py:143-160, 217-220).
//
// On the NNFFT path every window value has the form
//     g_t(d) = omega((t - d)/m),   t in [1-m, m],  d in [0, 1)
// where d is the fractional grid offset of a node (spread: d = N1 v -
// floor(N1 v), nnfft.py:188-191; gather: d = N2 xs - floor(N2 xs),
// nnfft.py:200-204; omega is even so the sign of the argument is irrelevant).
//
// Instead of sqrt + exp + expm1 per tap (the reference's form; ~40 fp64 ops)
// each tap is a degree-P polynomial in u = 2d - 1, fitted at plan time in
// 80-bit long double and validated against the exact window to <= 5e-15
// absolute (|omega| <= 1).  Two symmetries halve the work:
//   * g_{1-t}(u) = g_t(-u): tap pair (t, 1-t) shares the even part E(u^2) and
//     the odd part u*O(u^2) of one polynomial: g_t = E + uO, g_{1-t} = E - uO;
//   * the two edge taps t = m, 1-m carry the sqrt branch point of omega at
//     |x| = 1: g_m(d) = sqrt(d) H(u), g_{1-m}(d) = sqrt(1-d) H(-u) with H
//     analytic, so they are exactly zero where the reference's are (d = 0).
// Cost: about m*(P+1) DFMA + 2 sqrt per node for all 2m taps.
#pragma once

#include <cmath>

#include "common.cuh"

namespace sfb {

constexpr int kMaxM = 16;   // largest supported window cut-off m
constexpr int kMaxNE = 9;   // even coefficients for P <= 16
constexpr int kMaxNO = 8;   // odd coefficients for P <= 16

// polynomial degree per cut-off, chosen from a long-double fit study so the
// worst tap error is <= 1e-15 for every sigma in [5/4, 2]
__host__ __device__ constexpr int window_degree(int m) {
  return m <= 2 ? 16 : m <= 3 ? 15 : m <= 6 ? 14 : m <= 9 ? 13 : 12;
}

// Coefficients for the m tap pairs; pair q < m-1 is the inner pair
// (t = q+1, 1-t), pair m-1 the edge pair.  Passed to kernels by value, so the
// coefficients live in the constant bank and feed DFMA operands directly.
struct WinCoef {
  double e[kMaxM][kMaxNE];
  double o[kMaxM][kMaxNO];
};

// Polynomial in v = u^2 with compile-time coefficient offsets: Horner, or
// Estrin's scheme (SFB_ESTRIN=1: the same number of FMAs with a dependency
// depth of ~log2(N), the powers v^2, v^4, v^8 formed once per node).  Estrin
// measured slower in both spread and gather (the extra live powers push the
// spread past 124 registers into spills: 0.373 -> 0.385 ms, gather 0.297 ->
// 0.321 ms), so Horner is the default.
#ifndef SFB_ESTRIN
#define SFB_ESTRIN 0  // Horner: Estrin measured slower (spills; gather 0.297 -> 0.321 ms)
#endif
struct VPow {
  double p[4];  // v, v^2, v^4, v^8
};
__host__ __device__ __forceinline__ VPow vpowers(double v) {
  VPow w;
  w.p[0] = v;
  w.p[1] = v * v;
  w.p[2] = w.p[1] * w.p[1];
  w.p[3] = w.p[2] * w.p[2];
  return w;
}
template <int N, int OFF = 0>
__host__ __device__ __forceinline__ double poly(const double* c, const VPow& w) {
#if SFB_ESTRIN
  if constexpr (N == 1) {
    return c[OFF];
  } else if constexpr (N == 2) {
    return fma(c[OFF + 1], w.p[0], c[OFF]);
  } else {
    constexpr int H = N > 8 ? 8 : N > 4 ? 4 : 2;  // largest power of two below N
    constexpr int L = H == 8 ? 3 : H == 4 ? 2 : 1;
    return fma(poly<N - H, OFF + H>(c, w), w.p[L], poly<H, OFF>(c, w));
  }
#else
  double r = c[OFF + N - 1];
#pragma unroll
  for (int k = N - 2; k >= 0; --k) r = fma(r, w.p[0], c[OFF + k]);
  return r;
#endif
}

// sqrt(d), d in [0, 1], for the two edge taps of the moment spread.  For m >= 4
// the edge taps are small (|g| <= sinh(beta sqrt(2/m)) / sinh(beta) < 7e-3 at
// m = 4, < 7e-9 at m = 8), so the square root needs far less than full
// precision: the hardware reciprocal-square-root seed (MUFU.RSQ64H, relative
// error 2^-22) and ONE Goldschmidt step (1.5 eps^2 ~ 9e-14 relative, < 6e-16
// absolute on the tap) instead of the IEEE routine's seed + 2 steps + fix-up +
// slow-path branch.  d = 0 gives exactly 0 (the clamped seed is finite).
// Measured and NOT used in the per-node window passes below: freed of the
// IEEE routine's slow-path call, ptxas interleaves many more tap pairs there
// and spills (config-3 spread 385 -> 650 us, gather 256 -> 263 us).
template <int M, bool FAST>
__device__ __forceinline__ double edge_sqrt(double d) {
  if constexpr (M >= 4 && FAST) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(fmax(d, 1e-300)));
    const double g = d * y, h = 0.5 * y;
    return fma(g, fma(-g, h, 0.5), g);
  }
  return sqrt(d);
}

// All 2M tap values w[i] = g_{i+1-M}(d) for one node.  Host and device use
// the same instruction sequence (host validation emulates the kernel).
template <int M>
__host__ __device__ __forceinline__ void window_taps(const WinCoef& C, double d, double* w) {
  constexpr int P = window_degree(M);
  constexpr int NE = P / 2 + 1;
  constexpr int NO = (P + 1) / 2;
  const double u = 2.0 * d - 1.0;
  const VPow vw = vpowers(u * u);
#pragma unroll
  for (int q = 0; q < M; ++q) {
    const double E = poly<NE>(C.e[q], vw);
    const double O = poly<NO>(C.o[q], vw);
    const double hi = fma(u, O, E);
    const double lo = fma(-u, O, E);
    if (q < M - 1) {
      w[M + q] = hi;
      w[M - 1 - q] = lo;
    } else {
      w[2 * M - 1] = sqrt(d) * hi;
      w[0] = sqrt(1.0 - d) * lo;
    }
  }
}

// Accumulate f * g_t(d) into r[t + M - 1] for all 2M taps, consuming each tap
// pair as soon as it is formed (keeps the live register set small).
template <int M, bool REAL>
__device__ __forceinline__ void window_accumulate(const WinCoef& C, double d, double2 fv,
                                                  double2* r) {
  constexpr int P = window_degree(M);
  constexpr int NE = P / 2 + 1;
  constexpr int NO = (P + 1) / 2;
  const double u = 2.0 * d - 1.0;
  const VPow vw = vpowers(u * u);
  const double sq_hi = sqrt(d), sq_lo = sqrt(1.0 - d);
#pragma unroll
  for (int q = 0; q < M; ++q) {
    const double E = poly<NE>(C.e[q], vw);
    const double O = poly<NO>(C.o[q], vw);
    double hi = fma(u, O, E);
    double lo = fma(-u, O, E);
    const int ih = (q < M - 1) ? M + q : 2 * M - 1;
    const int il = (q < M - 1) ? M - 1 - q : 0;
    if (q == M - 1) {
      hi *= sq_hi;
      lo *= sq_lo;
    }
    r[ih].x = fma(fv.x, hi, r[ih].x);
    r[il].x = fma(fv.x, lo, r[il].x);
    if (!REAL) {
      r[ih].y = fma(fv.y, hi, r[ih].y);
      r[il].y = fma(fv.y, lo, r[il].y);
    }
  }
}

// window_taps for two nodes at once (shared coefficient loads)
template <int M>
__device__ __forceinline__ void window_taps2(const WinCoef& C, double d0, double d1, double* w0,
                                             double* w1) {
  constexpr int P = window_degree(M);
  constexpr int NE = P / 2 + 1;
  constexpr int NO = (P + 1) / 2;
  const double u0 = 2.0 * d0 - 1.0, u1 = 2.0 * d1 - 1.0;
  const VPow vw0 = vpowers(u0 * u0), vw1 = vpowers(u1 * u1);
#pragma unroll
  for (int q = 0; q < M; ++q) {
    const double E0 = poly<NE>(C.e[q], vw0), E1 = poly<NE>(C.e[q], vw1);
    const double O0 = poly<NO>(C.o[q], vw0), O1 = poly<NO>(C.o[q], vw1);
    const double hi0 = fma(u0, O0, E0), lo0 = fma(-u0, O0, E0);
    const double hi1 = fma(u1, O1, E1), lo1 = fma(-u1, O1, E1);
    if (q < M - 1) {
      w0[M + q] = hi0, w0[M - 1 - q] = lo0;
      w1[M + q] = hi1, w1[M - 1 - q] = lo1;
    } else {
      w0[2 * M - 1] = sqrt(d0) * hi0, w0[0] = sqrt(1.0 - d0) * lo0;
      w1[2 * M - 1] = sqrt(d1) * hi1, w1[0] = sqrt(1.0 - d1) * lo1;
    }
  }
}

// Two nodes (d0, f0) and (d1, f1) of ONE cell accumulated into the same taps:
// every coefficient (a uniform constant-bank load) feeds two independent
// Horner chains, halving the constant loads per node and doubling the ILP.
template <int M, bool REAL>
__device__ __forceinline__ void window_accumulate2(const WinCoef& C, double d0, double2 f0,
                                                   double d1, double2 f1, double2* r) {
  constexpr int P = window_degree(M);
  constexpr int NE = P / 2 + 1;
  constexpr int NO = (P + 1) / 2;
  const double u0 = 2.0 * d0 - 1.0, u1 = 2.0 * d1 - 1.0;
  const VPow vw0 = vpowers(u0 * u0), vw1 = vpowers(u1 * u1);
  const double sh0 = sqrt(d0), sl0 = sqrt(1.0 - d0), sh1 = sqrt(d1), sl1 = sqrt(1.0 - d1);
#pragma unroll
  for (int q = 0; q < M; ++q) {
    const double E0 = poly<NE>(C.e[q], vw0), E1 = poly<NE>(C.e[q], vw1);
    const double O0 = poly<NO>(C.o[q], vw0), O1 = poly<NO>(C.o[q], vw1);
    double hi0 = fma(u0, O0, E0), lo0 = fma(-u0, O0, E0);
    double hi1 = fma(u1, O1, E1), lo1 = fma(-u1, O1, E1);
    const int ih = (q < M - 1) ? M + q : 2 * M - 1;
    const int il = (q < M - 1) ? M - 1 - q : 0;
    if (q == M - 1) {
      hi0 *= sh0, lo0 *= sl0, hi1 *= sh1, lo1 *= sl1;
    }
    r[ih].x = fma(f1.x, hi1, fma(f0.x, hi0, r[ih].x));
    r[il].x = fma(f1.x, lo1, fma(f0.x, lo0, r[il].x));
    if (!REAL) {
      r[ih].y = fma(f1.y, hi1, fma(f0.y, hi0, r[ih].y));
      r[il].y = fma(f1.y, lo1, fma(f0.y, lo0, r[il].y));
    }
  }
}

// Gather form of window_accumulate2: two targets (d0 over h0[0..2M), d1 over
// h1[0..2M)) interpolated together, every coefficient feeding both Horner
// chains and each tap pair consumed as soon as it is formed (no tap arrays).
// ALLSAME: every lane of the warp has both targets on one window (h1 == h0,
// checked with a warp vote by the caller): the second target reuses the first
// one's loaded values with no second loads and no register copies.
template <int M, bool ALLSAME = false>
__device__ __forceinline__ void window_dot2(const WinCoef& C, double d0, double d1,
                                            const double2* h0, const double2* h1, double2& s0,
                                            double2& s1, bool same = false) {
  constexpr int P = window_degree(M);
  constexpr int NE = P / 2 + 1;
  constexpr int NO = (P + 1) / 2;
  const double u0 = 2.0 * d0 - 1.0, u1 = 2.0 * d1 - 1.0;
  const VPow vw0 = vpowers(u0 * u0), vw1 = vpowers(u1 * u1);
  const double sh0 = sqrt(d0), sl0 = sqrt(1.0 - d0), sh1 = sqrt(d1), sl1 = sqrt(1.0 - d1);
#pragma unroll
  for (int q = 0; q < M; ++q) {
    const double E0 = poly<NE>(C.e[q], vw0), E1 = poly<NE>(C.e[q], vw1);
    const double O0 = poly<NO>(C.o[q], vw0), O1 = poly<NO>(C.o[q], vw1);
    double hi0 = fma(u0, O0, E0), lo0 = fma(-u0, O0, E0);
    double hi1 = fma(u1, O1, E1), lo1 = fma(-u1, O1, E1);
    const int ih = (q < M - 1) ? M + q : 2 * M - 1;
    const int il = (q < M - 1) ? M - 1 - q : 0;
    if (q == M - 1) {
      hi0 *= sh0, lo0 *= sl0, hi1 *= sh1, lo1 *= sl1;
    }
    // same: both targets read one window (h1 == h0) -- the second pair of
    // loads is predicated off, so a quarter-warp of such threads costs no
    // shared-memory wavefront for it
    const double2 a0 = h0[ih], b0 = h0[il];
    if constexpr (ALLSAME) {
      s0.x = fma(a0.x, hi0, fma(b0.x, lo0, s0.x));
      s0.y = fma(a0.y, hi0, fma(b0.y, lo0, s0.y));
      s1.x = fma(a0.x, hi1, fma(b0.x, lo1, s1.x));
      s1.y = fma(a0.y, hi1, fma(b0.y, lo1, s1.y));
    } else {
      const double2 a1 = same ? a0 : h1[ih], b1 = same ? b0 : h1[il];
      s0.x = fma(a0.x, hi0, fma(b0.x, lo0, s0.x));
      s0.y = fma(a0.y, hi0, fma(b0.y, lo0, s0.y));
      s1.x = fma(a1.x, hi1, fma(b1.x, lo1, s1.x));
      s1.y = fma(a1.y, hi1, fma(b1.y, lo1, s1.y));
    }
  }
}

// window_dot2 for NT targets at once: every coefficient feeds NT Horner
// chains (the uniform coefficient loads amortised over NT targets).
template <int M, int NT>
__device__ __forceinline__ void window_dotn(const WinCoef& C, const double* d,
                                            const double2* const* h, double2* s) {
  constexpr int P = window_degree(M);
  constexpr int NE = P / 2 + 1;
  constexpr int NO = (P + 1) / 2;
  double u[NT];
  VPow vw[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    u[t] = 2.0 * d[t] - 1.0;
    vw[t] = vpowers(u[t] * u[t]);
  }
#pragma unroll
  for (int q = 0; q < M; ++q) {
    const int ih = (q < M - 1) ? M + q : 2 * M - 1;
    const int il = (q < M - 1) ? M - 1 - q : 0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const double E = poly<NE>(C.e[q], vw[t]);
      const double O = poly<NO>(C.o[q], vw[t]);
      double hi = fma(u[t], O, E), lo = fma(-u[t], O, E);
      if (q == M - 1) {
        hi *= sqrt(d[t]);
        lo *= sqrt(1.0 - d[t]);
      }
      const double2 a = h[t][ih], b = h[t][il];
      s[t].x = fma(a.x, hi, fma(b.x, lo, s[t].x));
      s[t].y = fma(a.y, hi, fma(b.y, lo, s[t].y));
    }
  }
}

// Fourier transform of the sinh shape function, omega_hat(v)
// (windows.py:143-160), all three branches; on the NNFFT path only the
// w > 1e-3 branch is reachable.
__device__ inline double omega_hat_sinh(double beta, double v) {
  const double pi = 3.141592653589793238462643383279502884;
  const double one_m = -expm1(-2.0 * beta);
  const double w = beta * beta - 4.0 * pi * pi * v * v;
  if (w > 1e-3) {
    const double z = sqrt(w);
    return 2.0 * pi * beta * cyl_bessel_i1(z) * exp(-beta) / (one_m * z);
  }
  const double pref = 2.0 * pi * beta * exp(-beta) / one_m;
  if (w >= -1e-3) return pref * (0.5 + w / 16.0 + w * w / 384.0 + w * w * w / 18432.0);
  const double zn = sqrt(-w);
  return pref * j1(zn) / zn;
}

// phi_hat(v) = (m/n_grid) omega_hat(v m / n_grid)   (windows.py:217-220)
__device__ inline double phi_hat_sinh(double beta, int m, int64_t n_grid, double v) {
  const double sc = (double)m / (double)n_grid;
  return sc * omega_hat_sinh(beta, v * sc);
}

// Host: fit + validate the coefficients for cut-off m and shape beta.
// Throws Error(SINCFFT_EUNSUPPORTED) if m is outside [2, kMaxM] or the
// validation bound fails.  Defined in window.cu.
WinCoef fit_window(int m, double beta, double* max_err_out = nullptr);

}  // namespace sfb
