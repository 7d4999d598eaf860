// nfft.cu -- the classical NFFT and its adjoint (reference pkg/src/sincfft/
// nfft.py), built from the NNFFT's kernels.
//
// Reference (nfft.py:53-123), sigma N = n_over even, I_N = {-N/2 .. N/2-1}:
//   plan    hat_k = phi_hat(k), stencil l = floor(n_over x_j) + t (t = 1-m..m),
//           idx = l mod n_over, val = phi(x_j - l/n_over)            (:74-96)
//   trafo   buf[k mod n_over] = c_k / hat_k;  g = IFFT(buf)/n_over;
//           out_j = sum_t g[idx_jt] val_jt                             (:99-109)
//   adjoint G = bincount(idx, y val);  T = FFT(G)/n_over;
//           out_k = T[k mod n_over] / hat_k                             (:112-123)
//
// B200 realisation -- no new kernels on the hot part:
//   * trafo = the NNFFT's steps 2-4 with K = N inputs at l - N/2, DFT length
//     n_over, input factor 1/(n_over hat_l) folded into the Bluestein
//     pre-chirp (or the direct path's D), and the inverse DFT taken as
//     conj(F(conj c)): the FFT's first load conjugates, the gather (whose
//     window values are real) stores conj(out).  The gather is the NNFFT
//     gather with xs = x, grid n_over, scale 1 (targets sorted by (slice,
//     cell), periodic wrap at +-1/2 as in the reference's `mod`).
//   * adjoint = the NNFFT spread with N1 = n_over onto a grid of n_over + 2h
//     points (h = m + 1 halo cells each side, cell = floor(n_over x) + K/2),
//     a fold of the 2h halo points onto their residues mod n_over (in place,
//     2h threads), then the forward pruned DFT of the n_over folded points
//     at outputs k in I_N (s_lo = -N/2, Kout = N) and a divide by hat_k.
#include "nfft_impl.cuh"

#include <cstring>
#include <string>

namespace sfb {

// fold the halos of a grid of n_over + 2h points (position l - n_over/2 - h)
// onto residues mod n_over: [0, h) -> +n_over, [h + n_over, K) -> -n_over
__global__ void k_fold_halo(double2* grid, int64_t n_over, int64_t h) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 2 * h) return;
  const int64_t src = i < h ? i : n_over + i;  // left halo, then right halo
  const int64_t dst = i < h ? i + n_over : i;  // (n_over + i) - n_over = i, i in [h, 2h)
  const double2 v = grid[src];
  grid[dst].x += v.x;
  grid[dst].y += v.y;
}

__global__ void k_div_hat(const double2* in, const double* hat, double2* out, int64_t n) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double2 v = in[k];
  const double d = hat[k];
  out[k] = make_double2(v.x / d, v.y / d);
}

// phi_hat(k - N/2) on I_N (nfft.py:81) -- the NNFFT's phi_hat_2 with K = N
__global__ void k_hat_band(double* hat, int64_t N, double beta, int m, int64_t n_over,
                           unsigned long long* bad) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= N) return;
  const double v = phi_hat_sinh(beta, m, n_over, (double)(k - N / 2));
  hat[k] = v;
  if (!(v > 0.0)) atomicAdd(bad, 1ull);
}

__global__ void k_clip_nodes(const double* in, double* out, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = fmin(fmax(in[i], -0.5), 0.5);
}

__global__ void k_absmax_nodes(const double* a, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = fabs(a[i]);
    m = (v > m || v != v) ? v : m;
  }
  for (int o = 16; o; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, m, o);
    m = (t > m || t != t) ? t : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

template <int M>
__global__ void k_export_nfft(const double* x, int64_t n, int64_t n_over, WinCoef C,
                              int64_t* idx, double* val) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double pos = (double)n_over * x[j];
  const double c = floor(pos);
  double w[2 * M];
  window_taps<M>(C, pos - c, w);
  for (int t = 0; t < 2 * M; ++t) {
    int64_t l = ((int64_t)c + (t + 1 - M)) % n_over;
    if (l < 0) l += n_over;
    idx[j * 2 * M + t] = l;
    val[j * 2 * M + t] = w[t];
  }
}

namespace {
unsigned nblk(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, 256)); }
}  // namespace

void build_nfft(NfftPlanImpl& p, int64_t N, int64_t M, double sigma, int m, const double* x_dev,
                int device, cudaStream_t s) {
  // validation in the reference's order (nfft.py:60-89)
  if (N <= 0 || N % 2) fail(1, "nfft_plan: N must be a positive even integer");
  const double n_over_f = sigma * (double)N;
  const int64_t n_over = (int64_t)std::llround(n_over_f);
  if (std::fabs(n_over_f - (double)n_over) > 1e-9 || n_over % 2)
    fail(1, "nfft_plan: sigma*N must be an even integer, got " + std::to_string(n_over_f));
  if (2 * m > n_over / 2)
    fail(1, "nfft_plan: need 2*m <= sigma*N/2, got 2*" + std::to_string(m) + " > " +
                std::to_string(n_over / 2));
  if (M <= 0) fail(1, "nfft_plan: nodes must be a nonempty 1-d array");
  if (m < 2) fail(1, "m must be an integer >= 2");
  // windows.py:77-80: the sinh window needs 5/4 <= sigma <= 2
  if (!(1.25 - 1e-9 <= sigma && sigma <= 2.0 + 1e-9))
    fail(1, "sinh window requires 5/4 <= sigma <= 2, got sigma=" + std::to_string(sigma));
  if (m > kMaxM) fail(5, "window cut-offs above 16 are not supported by the B200 kernels");
  if (n_over >= ((int64_t)1 << 30) || M >= ((int64_t)1 << 31))
    fail(5, "problem size exceeds the 2^30-point grid / 2^31-node envelope");
  p.N = N;
  p.M = M;
  p.n_over = n_over;
  p.m = m;
  p.sigma = sigma;
  p.device = device;
  const double pi = 3.141592653589793238462643383279502884;
  p.beta = 2.0 * pi * m * (1.0 - 1.0 / (2.0 * sigma));  // windows.py:94-95
  {
    Scratch r(sizeof(unsigned long long), s);
    SF_CUDA(cudaMemsetAsync(r.p, 0, sizeof(unsigned long long), s));
    k_absmax_nodes<<<std::min<unsigned>(nblk(M), 1024), 256, 0, s>>>(x_dev, M,
                                                                    r.as<unsigned long long>());
    SF_LAUNCH_CHECK();
    unsigned long long bits = 0;
    SF_CUDA(cudaMemcpyAsync(&bits, r.p, sizeof(bits), cudaMemcpyDeviceToHost, s));
    SF_CUDA(cudaStreamSynchronize(s));
    double xmax;
    std::memcpy(&xmax, &bits, sizeof xmax);
    if (!(xmax <= 0.5 + 1e-12)) fail(1, "nfft_plan: nodes must lie in [-1/2, 1/2]");
  }
  p.x_clip.alloc(M);
  k_clip_nodes<<<nblk(M), 256, 0, s>>>(x_dev, p.x_clip.p, M);
  SF_LAUNCH_CHECK();
  p.hat.alloc(N);
  {
    Scratch bad(sizeof(unsigned long long), s);
    SF_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), s));
    k_hat_band<<<nblk(N), 256, 0, s>>>(p.hat.p, N, p.beta, m, n_over,
                                       bad.as<unsigned long long>());
    SF_LAUNCH_CHECK();
    unsigned long long nbad = 0;
    SF_CUDA(cudaMemcpyAsync(&nbad, bad.p, sizeof nbad, cudaMemcpyDeviceToHost, s));
    SF_CUDA(cudaStreamSynchronize(s));
    if (nbad)
      fail(2, "nfft_plan: window transform must be strictly positive on the frequency band; "
              "choose a larger sigma or a different window");
  }
  const WinCoef c = fit_window(m, p.beta);

  // trafo: FFT over the N coefficients (deconvolved in the pre-chirp), gather
  NnfftPlanImpl& t = p.tr;
  t.device = device;
  t.g.K = N;
  t.g.N2 = n_over;
  t.g.M2 = M;
  t.g.m2 = m;
  t.g.beta2 = p.beta;
  t.c2 = c;
  t.hat2.alloc(N);
  SF_CUDA(cudaMemcpyAsync(t.hat2.p, p.hat.p, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
  t.sp.n_sms = 148;
  SF_CUDA(cudaDeviceGetAttribute(&t.sp.n_sms, cudaDevAttrMultiProcessorCount, device));
  build_targets(t, p.x_clip.p, M, 1.0, (double)n_over, n_over, m, TargetScale{}, s);
  t.gp.conj_out = true;
  t.fft.conj_in = true;
  t.fft.in_scale = 1.0 / (double)n_over;
  build_fft(t, s);

  // adjoint: spread onto n_over + 2h points, fold, FFT to I_N
  p.halo = m + 1;
  NnfftPlanImpl& a = p.ad_spread;
  a.device = device;
  a.g.K = n_over + 2 * p.halo;
  a.g.M1 = M;
  a.g.m1 = m;
  a.g.beta1 = p.beta;
  a.c1 = c;
  build_sources(a, p.x_clip.p, M, (double)n_over, a.g.K, s);
  NnfftPlanImpl& q = p.ad_fft;
  q.device = device;
  q.g.K = n_over;
  q.g.N2 = n_over;
  q.fft.s_lo = -N / 2;
  q.fft.Kout = N;
  q.fft.in_scale = 1.0 / (double)n_over;  // no deconvolution before the FFT
  build_fft(q, s);
  SF_CUDA(cudaStreamSynchronize(s));
}

void run_nfft_trafo(const NfftPlanImpl& p, const double2* c, double2* out, cudaStream_t s) {
  const NnfftPlanImpl& t = p.tr;
  Scratch work(sizeof(double2) * (size_t)t.fft.work_elems(), s);
  Scratch h(sizeof(double2) * (size_t)t.fft.Kout, s);
  run_fft(t, c, h.as<double2>(), work.as<double2>(), 1, s);
  run_gather(t, h.as<double2>(), out, 1, s);
}

void run_nfft_adjoint(const NfftPlanImpl& p, const double2* y, double2* out, cudaStream_t s) {
  const NnfftPlanImpl& a = p.ad_spread;
  const NnfftPlanImpl& q = p.ad_fft;
  Scratch grid(sizeof(double2) * (size_t)a.g.K, s);
  Scratch work(sizeof(double2) * (size_t)q.fft.work_elems(), s);
  Scratch h(sizeof(double2) * (size_t)q.fft.Kout, s);
  run_spread(a, y, grid.as<double2>(), 1, s);
  k_fold_halo<<<nblk(2 * p.halo), 256, 0, s>>>(grid.as<double2>(), p.n_over, p.halo);
  SF_LAUNCH_CHECK();
  run_fft(q, grid.as<double2>() + p.halo, h.as<double2>(), work.as<double2>(), 1, s);
  k_div_hat<<<nblk(p.N), 256, 0, s>>>(h.as<double2>(), p.hat.p, out, p.N);
  SF_LAUNCH_CHECK();
}

template <int M>
static void export_nfft_m(const NfftPlanImpl& p, int64_t* idx, double* val, cudaStream_t s) {
  k_export_nfft<M><<<nblk(p.M), 256, 0, s>>>(p.x_clip.p, p.M, p.n_over, p.tr.c2, idx, val);
  SF_LAUNCH_CHECK();
}

void export_nfft(const NfftPlanImpl& p, int64_t* idx, double* val, double* hat, cudaStream_t s) {
  if (idx && val) {
    switch (p.m) {
#define SF_CASE(MM) \
  case MM:          \
    export_nfft_m<MM>(p, idx, val, s); break;
      SF_CASE(2) SF_CASE(3) SF_CASE(4) SF_CASE(5) SF_CASE(6) SF_CASE(7) SF_CASE(8) SF_CASE(9)
      SF_CASE(10) SF_CASE(11) SF_CASE(12) SF_CASE(13) SF_CASE(14) SF_CASE(15) SF_CASE(16)
#undef SF_CASE
      default:
        fail(5, "unsupported window cut-off");
    }
  }
  if (hat)
    SF_CUDA(cudaMemcpyAsync(hat, p.hat.p, sizeof(double) * p.N, cudaMemcpyDeviceToDevice, s));
}

}  // namespace sfb
