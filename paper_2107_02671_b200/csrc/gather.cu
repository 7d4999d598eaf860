// gather.cu -- step 4 of Algorithm 2.1: interpolate the fine-grid values at
// the M2 spatial nodes with the second window and divide by phi_hat_1.
//
// Reference (pkg/src/sincfft/nnfft.py:198-205, 241-243):
//     out_j = sum_{t=1-m2}^{m2} h[(c_j + t) mod N2] phi_2(xs_j - (c_j+t)/N2)
//             / phi_hat_1(N x_j),   xs_j = x_j N/N1, c_j = floor(N2 xs_j).
// Targets are sorted by position at plan time, so a warp reads one short,
// contiguous window of h (L1-resident); the 2m2 window values come from the
// per-tap polynomials (window.cuh); the scale 1/phi_hat_1 (times the
// Clenshaw-Curtis weight for fast-sinc stage 1) is one sorted fp64 stream;
// the result is stored to the target's original index.
#include "nnfft_impl.cuh"

namespace sfb {

struct GatherArgs {
  const double* pos;
  const int* perm;
  const double* scale;
  const double2* h;  // [batch][Kout], h[k'] = h_{s_lo + k'}
  double2* out;      // (M2, batch) row-major
  int64_t M2, Kout, N2, s_lo;
  int batch;
};

template <int M>
__global__ void __launch_bounds__(256) k_gather(GatherArgs a, WinCoef C) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= a.M2) return;
  const int col = blockIdx.y;
  const double pos = a.pos[j];
  const double c = floor(pos);
  const double d = pos - c;
  double w[2 * M];
  window_taps<M>(C, d, w);
  const double2* h = a.h + (int64_t)col * a.Kout;
  int64_t k0 = (int64_t)c + (1 - M) - a.s_lo;
  double2 s = make_double2(0.0, 0.0);
  if (k0 >= 0 && k0 + 2 * M <= a.Kout) {
    const double2* hp = h + k0;
#pragma unroll
    for (int i = 0; i < 2 * M; ++i) {
      const double2 v = __ldg(hp + i);
      s.x = fma(v.x, w[i], s.x);
      s.y = fma(v.y, w[i], s.y);
    }
  } else {  // periodic wrap (only when Kout == N2 covers every residue)
#pragma unroll
    for (int i = 0; i < 2 * M; ++i) {
      int64_t k = (k0 + i) % a.N2;
      if (k < 0) k += a.N2;
      const double2 v = __ldg(h + k);
      s.x = fma(v.x, w[i], s.x);
      s.y = fma(v.y, w[i], s.y);
    }
  }
  const double sc = a.scale[j];
  a.out[(int64_t)a.perm[j] * a.batch + col] = make_double2(s.x * sc, s.y * sc);
}

void run_gather(const NnfftPlanImpl& p, const double2* h, double2* out, int batch,
                cudaStream_t s) {
  GatherArgs a{p.gp.pos.p, p.gp.perm.p, p.gp.scale.p, h,          out,
               p.g.M2,     p.fft.Kout,  p.g.N2,        p.fft.s_lo, batch};
  const dim3 grid((unsigned)ceil_div(p.g.M2, 256), batch);
  switch (p.g.m2) {
#define SF_CASE(MM)                                          \
  case MM:                                                   \
    k_gather<MM><<<grid, 256, 0, s>>>(a, p.c2);              \
    SF_LAUNCH_CHECK();                                       \
    return;
    SF_CASE(2) SF_CASE(3) SF_CASE(4) SF_CASE(5) SF_CASE(6) SF_CASE(7) SF_CASE(8) SF_CASE(9)
    SF_CASE(10) SF_CASE(11) SF_CASE(12) SF_CASE(13) SF_CASE(14) SF_CASE(15) SF_CASE(16)
#undef SF_CASE
  }
  fail(5, "unsupported m2");
}

}  // namespace sfb
