// adjoint.cu -- the adjoint NNFFT (BASELINE north star
// "NNFFT, adjoint-NNFFT and fast-sinc entry points"): the exact conjugate
// transpose of nnfft_trafo (nnfft.py:210-243), stage by stage.  The
// reference has no adjoint NNFFT, so its parity is pinned by the
// inner-product identity <A f, y> = <f, A^H y> to rounding and by the exact
// sum out_k = sum_j y_j e^{+2 pi i N v_k x_j} within the NNFFT's bound.
//
// Forward:  A = diag(1/phi_hat_1(N x)) G_x (1/N2) F diag(1/phi_hat_2) (1/N1) S_v
//   (S_v: spread, window 1; F: pruned length-N2 DFT; G_x: gather, window 2)
// Adjoint:  A^H = S_v^T (1/N1) diag(1/phi_hat_2) (1/N2) F^H G_x^T diag(1/phi_hat_1)
// realised with the forward's own kernels:
//   1. y_j / phi_hat_1(N x_j)                       (k_scale_rows, original order)
//   2. G_x^T = spread of those values at N2 xs_j with window 2 onto the
//      N2-periodic grid (N2 + 2h points, halo folded: k_fold_copy)
//   3. F^H = conj(F conj(.)): the pruned DFT with inputs at the N2 residues
//      and outputs at l - K/2, l in [0, K) (conj on load, conj on k_post)
//   4. times 1/(N1 N2 phi_hat_2(l - K/2))           (k_post)
//   5. S_v^T = gather over the K-grid at N1 v_k with window 1
// The sub-plans are built lazily on the first adjoint call (capi.cu).
#include "nnfft_impl.cuh"

namespace sfb {

namespace {
unsigned nb(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, 256)); }
}  // namespace

__global__ void k_adj_scale_init(const double* x, int64_t n, double Nd, double beta1, int m1,
                                 int64_t N1, double* s1) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) s1[i] = 1.0 / phi_hat_sinh(beta1, m1, N1, Nd * x[i]);
}

__global__ void k_scale_xs(const double* x, int64_t n, double ratio, double* xs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) xs[i] = x[i] * ratio;
}

// rows of a (n, B) row-major complex array times s[row]
__global__ void k_scale_rows(const double2* y, const double* s, int64_t n, int B, double2* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * B) return;
  const double d = s[e / B];
  const double2 v = y[e];
  out[e] = make_double2(v.x * d, v.y * d);
}

// periodic fold of a [B][N2 + 2h] grid (position i - N2/2 - h) to [B][N2]
// (position l - N2/2), l in [0, N2)
__global__ void k_fold_copy(const double2* grid, int64_t Ka, int64_t n2, int64_t h, int B,
                            double2* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n2 * B) return;
  const int64_t b = e / n2, l = e % n2;
  const double2* g = grid + b * Ka;
  double2 v = g[l + h];
  if (l >= n2 - h) {
    const double2 t = g[l + h - n2];
    v.x += t.x, v.y += t.y;
  }
  if (l < h) {
    const double2 t = g[l + h + n2];
    v.x += t.x, v.y += t.y;
  }
  out[e] = v;
}

// g[b][l] = conj(h[b][l]) / (N1 phi_hat_2(l - K/2))   (1/N2 is in the pre-chirp)
__global__ void k_adj_post(const double2* h, const double* hat2, int64_t K, int B, double inv_n1,
                           double2* g) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= K * B) return;
  const double d = inv_n1 / hat2[e % K];
  const double2 v = h[e];
  g[e] = make_double2(v.x * d, -v.y * d);
}

void build_adjoint(const NnfftPlanImpl& p, NnfftAdjoint& a, cudaStream_t s) {
  const Geometry& g = p.g;
  a.halo = g.m2 + 1;
  const int64_t Ka = g.N2 + 2 * a.halo;
  // 1. 1/phi_hat_1(N x_j) in original order (nnfft.py:175)
  a.s1.alloc(g.M2);
  k_adj_scale_init<<<nb(g.M2), 256, 0, s>>>(p.x_clip.p, g.M2, (double)g.N, g.beta1, g.m1, g.N1,
                                           a.s1.p);
  SF_LAUNCH_CHECK();
  // 2. spread at N2 xs, xs = x N/N1 (the gather's positions, nnfft.py:200)
  DevArray<double> xs(g.M2);
  k_scale_xs<<<nb(g.M2), 256, 0, s>>>(p.x_clip.p, g.M2, (double)g.N / (double)g.N1, xs.p);
  SF_LAUNCH_CHECK();
  NnfftPlanImpl& sx = a.spread_x;
  sx.device = p.device;
  sx.g.K = Ka;
  sx.g.M1 = g.M2;
  sx.g.m1 = g.m2;
  sx.c1 = p.c2;
  build_sources(sx, xs.p, g.M2, (double)g.N2, Ka, s);
  // 3. pruned DFT: N2 folded inputs -> K outputs at l - K/2
  NnfftPlanImpl& q = a.fft;
  q.device = p.device;
  q.g.K = g.N2;
  q.g.N2 = g.N2;
  q.fft.s_lo = -g.K / 2;
  q.fft.Kout = g.K;
  q.fft.conj_in = true;
  q.fft.in_scale = 1.0 / (double)g.N2;
  build_fft(q, s);
  // 5. gather over the K-grid at N1 v_k (positions exactly as the spread's)
  NnfftPlanImpl& gv = a.gather_v;
  gv.device = p.device;
  gv.g.M2 = g.M1;
  gv.g.m2 = g.m1;
  gv.g.N2 = g.K;
  gv.c2 = p.c1;
  build_targets(gv, p.v_clip.p, g.M1, 1.0, (double)g.N1, g.K, g.m1, TargetScale{}, s, -g.K / 2,
                g.K);
  SF_CUDA(cudaStreamSynchronize(s));
}

void run_adjoint(const NnfftPlanImpl& p, const NnfftAdjoint& a, const double2* y, double2* out,
                 int batch, cudaStream_t s) {
  const Geometry& g = p.g;
  const int64_t Ka = g.N2 + 2 * a.halo;
  Scratch ys(sizeof(double2) * (size_t)g.M2 * batch, s);
  k_scale_rows<<<nb(g.M2 * batch), 256, 0, s>>>(y, a.s1.p, g.M2, batch, ys.as<double2>());
  SF_LAUNCH_CHECK();
  Scratch grid(sizeof(double2) * (size_t)Ka * batch, s);
  run_spread(a.spread_x, ys.as<double2>(), grid.as<double2>(), batch, s);
  Scratch folded(sizeof(double2) * (size_t)g.N2 * batch, s);
  k_fold_copy<<<nb(g.N2 * batch), 256, 0, s>>>(grid.as<double2>(), Ka, g.N2, a.halo, batch,
                                              folded.as<double2>());
  SF_LAUNCH_CHECK();
  Scratch work(sizeof(double2) * (size_t)a.fft.fft.work_elems() * batch, s);
  Scratch h(sizeof(double2) * (size_t)g.K * batch, s);
  run_fft(a.fft, folded.as<double2>(), h.as<double2>(), work.as<double2>(), batch, s);
  k_adj_post<<<nb(g.K * batch), 256, 0, s>>>(h.as<double2>(), p.hat2.p, g.K, batch,
                                             1.0 / (double)g.N1, grid.as<double2>());
  SF_LAUNCH_CHECK();
  run_gather(a.gather_v, grid.as<double2>(), out, batch, s);
}

}  // namespace sfb
