// direct.cu -- the quadratic-cost exact sums of the reference's direct.py on
// the GPU: the oracles the fast transforms are checked
// against, affordable at configs 3 and 5 only on the device.
//
// Reference (pkg/src/sincfft/direct.py):
//   nndft_direct          :28-64   out_j = sum_k f_k e^{-2 pi i N v_k x_j}
//   ndft_direct           :67-90   out_j = sum_{k in I_N} c_k e^{2 pi i k x_j}
//   sinc_transform_direct :93-112  out_j = sum_k c_k sinc(N pi (b_j - a_k))
// The reference forms the phase 2 pi N v x in fp64 (absolute phase error
// ~ulp(2 pi N v x), i.e. ~1e-10 at N = 2^20) and sums pairwise.  Here the
// phase is carried in two doubles (TwoProduct by fma) and reduced modulo the
// period before sincospi, and the sums are compensated (TwoSum), so these
// are at least as accurate as the reference's; the parity tests compare at
// the reference's own determinism tolerance (1e-13 sum|f|, test_direct.py).
//
// Layout: one thread per target (kDirectTPT targets per thread for ILP);
// sources stream through shared memory in tiles shared by the CTA.
#include "nnfft_impl.cuh"

namespace sfb {

constexpr int kDirectThreads = 256;
constexpr int kDirectTile = 256;  // sources per shared-memory tile
constexpr int kDirectTPT = 2;     // targets per thread

struct Comp {  // compensated (Neumaier) accumulator
  double s = 0.0, c = 0.0;
  __device__ __forceinline__ void add(double x) {
    const double t = s + x;
    c += fabs(s) >= fabs(x) ? (s - t) + x : (x - t) + s;
    s = t;
  }
  __device__ __forceinline__ double value() const { return s + c; }
};

// e^{-2 pi i t} for t = N * (v * x) carried as hi + lo, hi reduced mod 1
__device__ __forceinline__ void phase_turns(double a, double b, double N, double* sn,
                                            double* cs) {
  const double p = a * b;
  const double pe = fma(a, b, -p);
  const double t = N * p;
  const double te = fma(N, p, -t) + N * pe;
  const double r = t - rint(t);  // exact
  sincospi(2.0 * (r + te), sn, cs);
}

template <int KIND>  // 0: nndft (e^{-2 pi i N v x}), 1: ndft (e^{+2 pi i k x})
__global__ void __launch_bounds__(kDirectThreads) k_exp_direct(const double2* __restrict__ f,
                                                               const double* __restrict__ v,
                                                               int64_t M1,
                                                               const double* __restrict__ x,
                                                               int64_t M2, double N,
                                                               double2* __restrict__ out) {
  __shared__ double2 fs[kDirectTile];
  __shared__ double vs[kDirectTile];
  const int64_t j0 = ((int64_t)blockIdx.x * kDirectThreads) * kDirectTPT + threadIdx.x;
  double xj[kDirectTPT];
  Comp re[kDirectTPT], im[kDirectTPT];
#pragma unroll
  for (int u = 0; u < kDirectTPT; ++u) {
    const int64_t j = j0 + u * kDirectThreads;
    xj[u] = j < M2 ? x[j] : 0.0;
  }
  for (int64_t k0 = 0; k0 < M1; k0 += kDirectTile) {
    __syncthreads();
    for (int i = threadIdx.x; i < kDirectTile; i += kDirectThreads) {
      const int64_t k = k0 + i;
      fs[i] = k < M1 ? f[k] : make_double2(0.0, 0.0);
      // ndft: frequency index k - N/2 of I_N (exact integer)
      vs[i] = k < M1 ? (KIND == 0 ? v[k] : (double)(k - M1 / 2)) : 0.0;
    }
    __syncthreads();
    const int n = M1 - k0 < kDirectTile ? (int)(M1 - k0) : kDirectTile;
    for (int i = 0; i < n; ++i) {
      const double2 fk = fs[i];
      const double vk = vs[i];
#pragma unroll
      for (int u = 0; u < kDirectTPT; ++u) {
        double sn, cs;
        phase_turns(vk, xj[u], KIND == 0 ? N : 1.0, &sn, &cs);
        if (KIND == 0) sn = -sn;  // e^{-i theta}
        re[u].add(fk.x * cs);
        re[u].add(-fk.y * sn);
        im[u].add(fk.x * sn);
        im[u].add(fk.y * cs);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kDirectTPT; ++u) {
    const int64_t j = j0 + u * kDirectThreads;
    if (j < M2) out[j] = make_double2(re[u].value(), im[u].value());
  }
}

// sinc(N pi d), d = b - a carried as hi + lo; value 1 at d == 0 exactly
// (special.py:86-93 tests the rounded argument for 0; so does this)
__device__ __forceinline__ double sinc_term(double b, double a, double N) {
  const double y = -a;
  const double d = b + y;
  if (d == 0.0) return 1.0;
  const double z = d - b;
  const double de = (b - (d - z)) + (y - z);  // TwoSum error of b + (-a)
  const double s = N * d;
  const double se = fma(N, d, -s) + N * de;
  const double k = rint(s);
  const double r = (s - k) + se;  // |r| <= 1/2 + tiny
  double sp = sinpi(r);
  if (fmod(k, 2.0) != 0.0) sp = -sp;
  return sp / (3.141592653589793238462643383279502884 * (s + se));
}

__global__ void __launch_bounds__(kDirectThreads) k_sinc_direct(const double2* __restrict__ c,
                                                                const double* __restrict__ a,
                                                                int64_t L1,
                                                                const double* __restrict__ b,
                                                                int64_t L2, double N,
                                                                double2* __restrict__ out) {
  __shared__ double2 cs_[kDirectTile];
  __shared__ double as[kDirectTile];
  const int64_t j0 = ((int64_t)blockIdx.x * kDirectThreads) * kDirectTPT + threadIdx.x;
  double bj[kDirectTPT];
  Comp re[kDirectTPT], im[kDirectTPT];
#pragma unroll
  for (int u = 0; u < kDirectTPT; ++u) {
    const int64_t j = j0 + u * kDirectThreads;
    bj[u] = j < L2 ? b[j] : 0.0;
  }
  for (int64_t k0 = 0; k0 < L1; k0 += kDirectTile) {
    __syncthreads();
    for (int i = threadIdx.x; i < kDirectTile; i += kDirectThreads) {
      const int64_t k = k0 + i;
      cs_[i] = k < L1 ? c[k] : make_double2(0.0, 0.0);
      as[i] = k < L1 ? a[k] : 0.0;
    }
    __syncthreads();
    const int n = L1 - k0 < kDirectTile ? (int)(L1 - k0) : kDirectTile;
    for (int i = 0; i < n; ++i) {
      const double2 ck = cs_[i];
      const double ak = as[i];
#pragma unroll
      for (int u = 0; u < kDirectTPT; ++u) {
        const double kern = sinc_term(bj[u], ak, N);
        re[u].add(ck.x * kern);
        im[u].add(ck.y * kern);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kDirectTPT; ++u) {
    const int64_t j = j0 + u * kDirectThreads;
    if (j < L2) out[j] = make_double2(re[u].value(), im[u].value());
  }
}

static unsigned direct_grid(int64_t M2) {
  return (unsigned)std::max<int64_t>(1, ceil_div(M2, (int64_t)kDirectThreads * kDirectTPT));
}

void run_nndft_direct(const double2* f, const double* v, int64_t M1, const double* x,
                      int64_t M2, double N, double2* out, cudaStream_t s) {
  k_exp_direct<0><<<direct_grid(M2), kDirectThreads, 0, s>>>(f, v, M1, x, M2, N, out);
  SF_LAUNCH_CHECK();
}

void run_ndft_direct(const double2* c, int64_t Nc, const double* x, int64_t M, double2* out,
                     cudaStream_t s) {
  k_exp_direct<1><<<direct_grid(M), kDirectThreads, 0, s>>>(c, nullptr, Nc, x, M, 1.0, out);
  SF_LAUNCH_CHECK();
}

void run_sinc_direct(const double2* c, const double* a, int64_t L1, const double* b, int64_t L2,
                     double N, double2* out, cudaStream_t s) {
  k_sinc_direct<<<direct_grid(L2), kDirectThreads, 0, s>>>(c, a, L1, b, L2, N, out);
  SF_LAUNCH_CHECK();
}

}  // namespace sfb
