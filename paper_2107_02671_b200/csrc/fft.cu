// fft.cu -- step 2 (deconvolution + embedding) and step 3 (length-N2 DFT) of
// Algorithm 2.1 as one pruned Bluestein chirp-z transform.
//
// Reference (pkg/src/sincfft/nnfft.py:235-239):
//     buf[(l - K/2) mod N2] = g_l / (N1 phi_hat_2(l - K/2)),  l in [0, K)
//     h = fft(buf) / N2                                    (fft_core.py:24-25)
// and the gather then reads h_s only for s in [s_lo, s_lo + Kout)
// (nnfft.py:200-205, 242).  With W = exp(-2 pi i/N2) and s = s_lo + k':
//     h_{s_lo+k'} = Q_k' sum_l (g_l P_l) b_{k'-l}
//     P_l  = W^{l s_lo + l^2/2} / (N1 N2 phi_hat_2(l - K/2))
//     b_j  = W^{-j^2/2},  j in [-(K-1), Kout-1]
//     Q_k' = W^{-(K/2) k' - (K/2) s_lo + k'^2/2}
// The sum is a linear convolution evaluated exactly as a cyclic one of any
// length L >= K + Kout - 1; L is picked 7-smooth so the two FFTs of length L
// use radices 2,3,4,5,7,8 only.  This keeps the reference's exact N2 (parity
// at m <= 6 depends on it) whatever its prime factors are,
// reads only the K nonzero inputs and writes only the Kout outputs in use.
//
// Kernels (L = L1 * L2, four-step; natural index n = n1 + L1 n2):
//   k_single   L <= kSingleMax: one CTA per column does everything in smem.
//   k_colfwd   C columns n1 per CTA: DFT over n2 (DIF, reversed order p),
//              times W_L^{n1 k2}, store Y[n1 + L1 p].
//   k_rowmul   row p per CTA: DIF over n1, times Bhat, inverse DIT over k1.
//   k_colinv   C columns per CTA: times conj twiddle, inverse DIT over k2,
//              output k' = n1 + L1 n2 < Kout times Q.
// Bhat is produced at plan time by k_colfwd + k_rowmul(spectrum mode) (or
// k_single) on b, so it is in exactly the layout the forward pass produces.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "nnfft_impl.cuh"
#include "fft_reg.cuh"

#ifndef SFB_FFT_ROW_TMA
#define SFB_FFT_ROW_TMA 0  // 1: the config-3 row staged by one TMA bulk copy (measured
                           // 0.174 -> 0.176 ms: the extra barrier; kept off)
#endif

namespace sfb {

constexpr int kSingleMax = 8192;      // largest L done by one CTA
constexpr int kRowMax = 8192;         // largest row length L1
#ifndef SFB_FFT_COLELEMS
#define SFB_FFT_COLELEMS 2048
#endif
constexpr int kColElems = SFB_FFT_COLELEMS;  // C * L2 per single-column column-kernel CTA
constexpr int kColElemsB = 4096;             // per point-major (batched) CTA
constexpr int kTwSplit = 4096;        // two-level W_L table split
#ifndef SFB_FFT_BATCHLD
#define SFB_FFT_BATCHLD 0  // register passes: all loads of a phase issued before first use
#endif
#ifndef SFB_FFT_ABL
#define SFB_FFT_ABL 0  // timing ablations of k_colfwd_r1 (wrong results): 1 no loads, 2 no stores
#endif
#ifndef SFB_FFT_L2HINT
#define SFB_FFT_L2HINT 1  // register passes: tables evict-first, intermediates evict-last
#endif
#if SFB_FFT_L2HINT
#define FFT_LD_TABLE(p) ld_hint((p), l2_policy_first())
#define FFT_LD_ONCE(p) ld_hint((p), l2_policy_first())
#define FFT_ST_KEEP(p, v) st_hint((p), (v), l2_policy_last())
#else
#define FFT_LD_TABLE(p) __ldg(p)
#define FFT_LD_ONCE(p) (*(p))
#define FFT_ST_KEEP(p, v) (*(p) = (v))
#endif
#ifndef SFB_FFT_ROWHINT
#define SFB_FFT_ROWHINT 2  // row pass hint bits: 1 row load, 2 B-hat load, 4 row store
#endif
#if SFB_FFT_L2HINT && (SFB_FFT_ROWHINT & 1)
#define FFT_ROW_LD(p) FFT_LD_ONCE(p)
#else
#define FFT_ROW_LD(p) (*(p))
#endif
#if SFB_FFT_L2HINT && (SFB_FFT_ROWHINT & 2)
#define FFT_ROW_TAB(p) FFT_LD_TABLE(p)
#else
#define FFT_ROW_TAB(p) __ldg(p)
#endif
#if SFB_FFT_L2HINT && (SFB_FFT_ROWHINT & 4)
#define FFT_ROW_ST(p, v) FFT_ST_KEEP(p, v)
#else
#define FFT_ROW_ST(p, v) (*(p) = (v))
#endif
#ifndef SFB_DIRECT_PARMIN
#define SFB_DIRECT_PARMIN 32
#endif
#ifndef SFB_FFT_CPL
#define SFB_FFT_CPL 0  // register column passes: exchange layout padded every 8 slots
#endif
#ifndef SFB_FFT_RPL
#define SFB_FFT_RPL 0  // register row pass: padded every 16 slots
#endif
constexpr int kColPL = SFB_FFT_CPL, kRowPL = SFB_FFT_RPL;
#ifndef SFB_FFT_CMINB
#define SFB_FFT_CMINB 2
#endif
constexpr int64_t kFixMax = 2048;     // largest shortfall D of a short Bluestein length

enum { IN_GP = 0, IN_PLAIN = 1 };     // input mode: g*P (execute) or plain array (plan)

// W^{e2/2} for W = exp(-2 pi i / N2), e2 an exact integer
__device__ __forceinline__ double2 wpow_half(int64_t e2, int64_t N2) {
  const int64_t m = 2 * N2;
  int64_t r = e2 % m;
  if (r < 0) r += m;
  if (r >= N2) r -= m;  // r in [-N2, N2): angle -pi r / N2 in (-pi, pi]
  double sn, cs;
  sincospi(-(double)r / (double)N2, &sn, &cs);
  return make_double2(cs, sn);
}

__device__ __forceinline__ double2 wbig(const double2* __restrict__ lo,
                                        const double2* __restrict__ hi, int64_t q) {
  return cmul(__ldg(hi + (q / kTwSplit)), __ldg(lo + (q % kTwSplit)));
}

// ------------------------------------------------------------ table kernels
// inverse of revr: the position holding frequency k after the DIF of length N
template <int N, int R>
__device__ __forceinline__ int posr(int k) {
  using Sh = RegShape<N, R>;
  int p = 0;
#pragma unroll
  for (int q = 0; q < Sh::A; ++q)
    p |= ((k >> (Sh::LOGR * q)) & (R - 1)) << (Sh::LOG2N - Sh::LOGR * (q + 1));
  if (Sh::R0 > 1) p |= (k >> (Sh::LOGR * Sh::A)) & (Sh::R0 - 1);
  return p;
}

// B-hat (4096-point rows, 1024 rows; produced in the radix-8 DIF orders of
// the plan-time kernels) permuted to the radix-16 output orders of the
// register passes: rows always, the row index (column DIF position) too when
// the column passes run radix 16
__global__ void k_bhat_x16(const double2* __restrict__ in, double2* __restrict__ out,
                           int64_t L, int cols16) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= L) return;
  const int q = (int)(i & 4095), p = (int)(i >> 12);
  const int q8 = posr<4096, 8>(revr<4096, 16>(q));
  const int p8 = cols16 ? posr<1024, 8>(revr<1024, 16>(p)) : p;
  out[i] = in[((int64_t)p8 << 12) + q8];
}

__global__ void k_twiddle(double2* tw, int64_t n, int64_t count, int64_t step) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  // W_n^{i*step} = exp(-2 pi i (i*step mod n) / n)
  const int64_t e = (i * step) % n;
  double sn, cs;
  sincospi(-2.0 * (double)e / (double)n, &sn, &cs);
  tw[i] = make_double2(cs, sn);
}

__global__ void k_prechirp(double2* P, const double* hat2, int64_t K, int64_t N2, int64_t s_lo,
                           double inv_n1n2) {
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l >= K) return;
  // exponent 2e = 2 l s_lo + l^2, reduced exactly (|.| < 2^62 for K, N2 < 2^30)
  const int64_t e2 = (2 * l * (s_lo % (2 * N2))) % (2 * N2) + (l * l) % (2 * N2);
  const double d = hat2 ? inv_n1n2 / hat2[l] : inv_n1n2;  // no deconvolution: NFFT adjoint
  P[l] = cscale(wpow_half(e2, N2), d);
}

__global__ void k_postchirp(double2* Q, int64_t Kout, int64_t K, int64_t N2, int64_t s_lo) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= Kout) return;
  const int64_t m = 2 * N2;
  const int64_t e2 = (-(K % m) * k) % m - ((K % m) * (s_lo % m)) % m + (k * k) % m;
  Q[k] = wpow_half(e2, N2);
}

__global__ void k_chirp_kernel(double2* b, int64_t L, int64_t K, int64_t Kout, int64_t N2) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= L) return;
  // cyclic slot i holds j = i (i < Kout) or j = i - L (i > L - K), else 0
  int64_t j;
  if (i < Kout) j = i;
  else if (i > L - K) j = i - L;
  else {
    b[i] = make_double2(0.0, 0.0);
    return;
  }
  const int64_t m = 2 * N2;
  b[i] = wpow_half(-((j * j) % m), N2);
}

// Short cyclic length (L = K + Kout - 1 - D, 0 < D <= kFixMax): the chirp
// slots i in [L - K + 1, Kout - 1] are claimed by both j = i and j = i - L;
// k_chirp_kernel keeps j = i, so for k' < D the terms l >= K - D + k' used
// b_{k'-l+L} instead of b_{k'-l}.  The fix adds, after the inverse pass,
//   Q_k' * sum_{t=k'}^{D-1} a_{K-D+t} c_{t-k'},  a_l = g_l P_l,
//   c_u = b_{-(K-D)-u} - b_{-(K-D)-u+L}   (a D-point correlation, D^2/2 MACs)
// which lets the planner take a much smoother L (config 3: 2^22 instead of
// 4096 * 1029 at D = 79).
__global__ void k_fix_table(double2* c, int64_t D, int64_t K, int64_t L, int64_t N2) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= D) return;
  const int64_t m = 2 * N2;
  const int64_t j1 = -(K - D) - u, j2 = j1 + L;
  const double2 b1 = wpow_half(-((j1 % m) * (j1 % m) % m), N2);
  const double2 b2 = wpow_half(-((j2 % m) * (j2 % m) % m), N2);
  c[u] = make_double2(b1.x - b2.x, b1.y - b2.y);
}

// one warp per (k' < D, column); grid/h column-major ([B][K], [B][Kout]) or
// point-major ([K][B], [Kout][B])
__global__ void k_bluestein_fix(const double2* __restrict__ g, const double2* __restrict__ P,
                                const double2* __restrict__ c, const double2* __restrict__ Q,
                                double2* h, int64_t K, int64_t D, int64_t Kout, int conj_in,
                                int B, int point_major) {
  pdl_trigger();
  pdl_wait();  // reads the previous kernel's output
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int col = blockIdx.y;
  if (k >= D) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t t = k + lane; t < D; t += 32) {
    const int64_t l = K - D + t;
    double2 gv = point_major ? g[l * B + col] : g[(int64_t)col * K + l];
    if (conj_in) gv.y = -gv.y;
    const double2 av = cmul(gv, P[l]);
    const double2 cv = c[t - k];
    acc.x += av.x * cv.x - av.y * cv.y;
    acc.y += av.x * cv.y + av.y * cv.x;
  }
  for (int o = 16; o; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if (lane == 0) {
    const double2 d = cmul(Q[k], acc);
    double2* hp = point_major ? h + k * B + col : h + (int64_t)col * Kout + k;
    hp->x += d.x;
    hp->y += d.y;
  }
}

// ------------------------------------------------------------ FFT kernels
struct FftArgs {
  const double2* g;    // IN_GP: grid[batch][K]; IN_PLAIN: x[L]
  const double2* P;
  const double2* Q;
  const double2* Bhat;
  double2* Y;          // work [batch][L]
  double2* h;          // out [batch][Kout]
  const double2* tw1;
  const double2* tw2;
  const double2* tw_lo;
  const double2* tw_hi;
  const int* rev2;
  int64_t K, L, L1, L2, Kout;
  int C_log2;
  int conj_in;         // conjugate the input (inverse DFT via conj(F(conj x)))
  FftStages st1, st2;
  // radix-16 row transforms (register row passes of the config-3 shape):
  // their per-stage twiddles and B-hat permuted to their output order
  FftStages st1x, st2x;
  const double2* tw1x;
  const double2* tw2x;
  const double2* Bhatx;
};

// Global <-> shared copies are issued kU elements per thread at a time so
// that kU independent loads are in flight before the first dependent store
// (a plain strided loop serialises one DRAM latency per element).
#ifndef SFB_FFT_KU
#define SFB_FFT_KU 8
#endif
constexpr int kU = SFB_FFT_KU;
// the single-column column kernels (k_colfwd / k_colinv) run 4 CTAs per SM
// with C = 2 columns; fewer loads in flight keep them under 64 registers
#ifndef SFB_FFT_KU_COL
#define SFB_FFT_KU_COL 4
#endif
constexpr int kUc = SFB_FFT_KU_COL;

template <int MODE>
__global__ void __launch_bounds__(512) k_single(FftArgs a, int spectrum) {
  extern __shared__ double2 sm[];
  const int col = blockIdx.y;
  const int L = (int)a.L;
  const int T = blockDim.x;
  const double2* g = a.g + (int64_t)col * (MODE == IN_GP ? a.K : 0);
  for (int i0 = threadIdx.x; i0 < L; i0 += kU * T) {
    double2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * T;
      v[u] = make_double2(0.0, 0.0);
      if (MODE == IN_GP) {
        if (i < a.K) {
          double2 gv = __ldg(g + i);
          if (a.conj_in) gv.y = -gv.y;
          v[u] = cmul(gv, __ldg(a.P + i));
        }
      } else if (i < L) {
        v[u] = __ldg(g + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * T < L) sm[spad(i0 + u * T)] = v[u];
  }
  __syncthreads();
  fft_dif(sm, 0, a.st1, a.tw1);
  if (spectrum) {
    const double inv = 1.0 / (double)L;
    for (int i = threadIdx.x; i < L; i += T) a.Y[i] = cscale(sm[spad(i)], inv);
    return;
  }
  for (int i0 = threadIdx.x; i0 < L; i0 += kU * T) {
    double2 bv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * T < L) bv[u] = __ldg(a.Bhat + i0 + u * T);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * T;
      if (i < L) sm[spad(i)] = cconj(cmul(sm[spad(i)], bv[u]));
    }
  }
  __syncthreads();
  fft_dit(sm, 0, a.st1, a.tw1);
  double2* h = a.h + (int64_t)col * a.Kout;
  for (int k0 = threadIdx.x; k0 < a.Kout; k0 += kU * T) {
    double2 qv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (k0 + u * T < a.Kout) qv[u] = __ldg(a.Q + k0 + u * T);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int k = k0 + u * T;
      if (k < a.Kout) h[k] = cmul(cconj(sm[spad(k)]), qv[u]);
    }
  }
}

#ifndef SFB_FFT_COL_MINB
#define SFB_FFT_COL_MINB 4  // 32 KiB + <= 64 registers: 4 CTAs per SM
#endif
template <int MODE, int NCT = 0, int NBL = 0>
__global__ void __launch_bounds__(256, SFB_FFT_COL_MINB) k_colfwd(FftArgs a) {
  extern __shared__ double2 sm[];
  const int col = blockIdx.y;
  const int C = 1 << a.C_log2;
  const int64_t c0 = (int64_t)blockIdx.x * C;
  const int L2 = (int)a.L2;
  const int n_el = L2 << a.C_log2;
  const int T = blockDim.x;
  const double2* g = a.g + (int64_t)col * (MODE == IN_GP ? a.K : 0);
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kUc * T) {
    double2 v[kUc];
#pragma unroll
    for (int u = 0; u < kUc; ++u) {
      const int e = e0 + u * T;
      const int64_t n1 = c0 + (e & (C - 1));
      const int64_t n = n1 + a.L1 * (e >> a.C_log2);
      v[u] = make_double2(0.0, 0.0);
      if (e < n_el && n1 < a.L1) {
        if (MODE == IN_GP) {
          if (n < a.K) {
            double2 gv = __ldg(g + n);
            if (a.conj_in) gv.y = -gv.y;
            v[u] = cmul(gv, __ldg(a.P + n));
          }
        } else {
          v[u] = __ldg(g + n);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUc; ++u)
      if (e0 + u * T < n_el) sm[spad(e0 + u * T)] = v[u];
  }
  __syncthreads();
  if constexpr (NCT > 0) fft_dif_ct<NCT, NBL, 256>(sm, a.st2, a.tw2);
  else fft_dif(sm, a.C_log2, a.st2, a.tw2);
  double2* Y = a.Y + (int64_t)col * a.L;
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kUc * T) {
    double2 w[kUc];
#pragma unroll
    for (int u = 0; u < kUc; ++u) {
      const int e = e0 + u * T;
      const int64_t n1 = c0 + (e & (C - 1));
      w[u] = make_double2(1.0, 0.0);
      if (e < n_el && n1 < a.L1) w[u] = wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)__ldg(a.rev2 + (e >> a.C_log2)));
    }
#pragma unroll
    for (int u = 0; u < kUc; ++u) {
      const int e = e0 + u * T;
      const int64_t n1 = c0 + (e & (C - 1));
      if (e < n_el && n1 < a.L1) Y[n1 + a.L1 * (e >> a.C_log2)] = cmul(sm[spad(e)], w[u]);
    }
  }
}

template <int NCT = 0>
__global__ void __launch_bounds__(256, SFB_FFT_MINB) k_rowmul(FftArgs a, int spectrum) {
  extern __shared__ double2 sm[];
  const int col = blockIdx.y;
  const int64_t p = blockIdx.x;
  const int L1 = (int)a.L1;
  const int T = blockDim.x;
  double2* row = a.Y + (int64_t)col * a.L + p * a.L1;
  for (int i0 = threadIdx.x; i0 < L1; i0 += kU * T) {
    double2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * T < L1) v[u] = row[i0 + u * T];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * T < L1) sm[spad(i0 + u * T)] = v[u];
  }
  __syncthreads();
  if constexpr (NCT > 0) fft_dif_ct<NCT, 0, 256>(sm, a.st1, a.tw1);
  else fft_dif(sm, 0, a.st1, a.tw1);
  const double2* B = a.Bhat + p * a.L1;
  if (spectrum) {
    const double inv = 1.0 / (double)a.L;
    for (int i = threadIdx.x; i < L1; i += T) row[i] = cscale(sm[spad(i)], inv);
    return;
  }
  for (int i0 = threadIdx.x; i0 < L1; i0 += kU * T) {
    double2 bv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * T < L1) bv[u] = __ldg(B + i0 + u * T);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * T;
      if (i < L1) sm[spad(i)] = cconj(cmul(sm[spad(i)], bv[u]));
    }
  }
  __syncthreads();
  if constexpr (NCT > 0) fft_dit_ct<NCT, 0, 256>(sm, a.st1, a.tw1);
  else fft_dit(sm, 0, a.st1, a.tw1);
  for (int i = threadIdx.x; i < L1; i += T) row[i] = cconj(sm[spad(i)]);
}

template <int NCT = 0, int NBL = 0>
__global__ void __launch_bounds__(256, SFB_FFT_COL_MINB) k_colinv(FftArgs a) {
  extern __shared__ double2 sm[];
  const int col = blockIdx.y;
  const int C = 1 << a.C_log2;
  const int64_t c0 = (int64_t)blockIdx.x * C;
  const int L2 = (int)a.L2;
  const int n_el = L2 << a.C_log2;
  const int T = blockDim.x;
  const double2* Y = a.Y + (int64_t)col * a.L;
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kUc * T) {
    double2 v[kUc], w[kUc];
#pragma unroll
    for (int u = 0; u < kUc; ++u) {
      const int e = e0 + u * T;
      const int64_t n1 = c0 + (e & (C - 1));
      const int p = e >> a.C_log2;
      v[u] = make_double2(0.0, 0.0);
      w[u] = make_double2(1.0, 0.0);
      if (e < n_el && n1 < a.L1) {
        v[u] = Y[n1 + a.L1 * p];
        w[u] = wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)__ldg(a.rev2 + p));
      }
    }
#pragma unroll
    for (int u = 0; u < kUc; ++u)
      if (e0 + u * T < n_el) sm[spad(e0 + u * T)] = cmul(cconj(v[u]), w[u]);
  }
  __syncthreads();
  if constexpr (NCT > 0) fft_dit_ct<NCT, NBL, 256>(sm, a.st2, a.tw2);
  else fft_dit(sm, a.C_log2, a.st2, a.tw2);
  double2* h = a.h + (int64_t)col * a.Kout;
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kUc * T) {
    double2 qv[kUc];
#pragma unroll
    for (int u = 0; u < kUc; ++u) {
      const int e = e0 + u * T;
      const int64_t k = c0 + (e & (C - 1)) + a.L1 * (e >> a.C_log2);
      qv[u] = make_double2(0.0, 0.0);
      if (e < n_el && c0 + (e & (C - 1)) < a.L1 && k < a.Kout) qv[u] = __ldg(a.Q + k);
    }
#pragma unroll
    for (int u = 0; u < kUc; ++u) {
      const int e = e0 + u * T;
      const int64_t n1 = c0 + (e & (C - 1));
      const int64_t k = n1 + a.L1 * (e >> a.C_log2);
      if (e < n_el && n1 < a.L1 && k < a.Kout) h[k] = cmul(cconj(sm[spad(e)]), qv[u]);
    }
  }
}

// ------------------------------------------- batch-minor (point-major) I/O
// Same three Bluestein passes for B columns stored point-major: element
// (n, b) at n*B + b (the layout of the column-vectorised spread/gather,
// batched.cu).  A CTA interleaves CB consecutive COLUMNS in shared memory
// (instead of CB consecutive n1), so every global row access is CB*16
// contiguous bytes and no transposes are needed around the FFT.
struct FftBArgs {
  FftArgs a;
  int B;      // columns in this launch (a column group)
  int ldg;    // row stride of grid / h (the full batch)
  int ldy;    // row stride of the work array Y (the group)
  int cb_log2_col, cb_log2_row;
};

template <int NCT = 0, int NBL = 0>
__global__ void __launch_bounds__(256, SFB_FFT_MINB) k_colfwd_b(FftBArgs x) {
  extern __shared__ double2 sm[];
  const FftArgs& a = x.a;
  const int CB = 1 << x.cb_log2_col;
  const int64_t n1 = blockIdx.x;
  const int b0 = blockIdx.y * CB;
  const int L2 = (int)a.L2;
  const int n_el = L2 << x.cb_log2_col;
  const int T = blockDim.x;
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kU * T) {
    double2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int b = b0 + (e & (CB - 1));
      const int64_t n = n1 + a.L1 * (int64_t)(e >> x.cb_log2_col);
      v[u] = make_double2(0.0, 0.0);
      if (e < n_el && b < x.B && n < a.K) v[u] = cmul(__ldg(a.g + n * x.ldg + b), __ldg(a.P + n));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (e0 + u * T < n_el) sm[spad(e0 + u * T)] = v[u];
  }
  __syncthreads();
  if constexpr (NCT > 0) fft_dif_ct<NCT, NBL, 256>(sm, a.st2, a.tw2);
  else fft_dif(sm, x.cb_log2_col, a.st2, a.tw2);
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kU * T) {
    double2 w[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      w[u] = make_double2(1.0, 0.0);
      if (e < n_el) w[u] = wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)__ldg(a.rev2 + (e >> x.cb_log2_col)));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int b = b0 + (e & (CB - 1));
      if (e < n_el && b < x.B)
        a.Y[(n1 + a.L1 * (int64_t)(e >> x.cb_log2_col)) * x.ldy + b] = cmul(sm[spad(e)], w[u]);
    }
  }
}

template <int NCT = 0, int NBL = 0>
__global__ void __launch_bounds__(256, SFB_FFT_MINB) k_rowmul_b(FftBArgs x) {
  extern __shared__ double2 sm[];
  const FftArgs& a = x.a;
  const int CB = 1 << x.cb_log2_row;
  const int64_t p = blockIdx.x;
  const int b0 = blockIdx.y * CB;
  const int L1 = (int)a.L1;
  const int n_el = L1 << x.cb_log2_row;
  const int T = blockDim.x;
  double2* Y = a.Y + p * a.L1 * x.ldy;
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kU * T) {
    double2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int b = b0 + (e & (CB - 1));
      v[u] = make_double2(0.0, 0.0);
      if (e < n_el && b < x.B) v[u] = Y[(int64_t)(e >> x.cb_log2_row) * x.ldy + b];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (e0 + u * T < n_el) sm[spad(e0 + u * T)] = v[u];
  }
  __syncthreads();
  if constexpr (NCT > 0) fft_dif_ct<NCT, NBL, 256>(sm, a.st1, a.tw1);
  else fft_dif(sm, x.cb_log2_row, a.st1, a.tw1);
  const double2* Bh = a.Bhat + p * a.L1;
  for (int e = threadIdx.x; e < n_el; e += T)
    sm[spad(e)] = cconj(cmul(sm[spad(e)], __ldg(Bh + (e >> x.cb_log2_row))));
  __syncthreads();
  if constexpr (NCT > 0) fft_dit_ct<NCT, NBL, 256>(sm, a.st1, a.tw1);
  else fft_dit(sm, x.cb_log2_row, a.st1, a.tw1);
  for (int e = threadIdx.x; e < n_el; e += T) {
    const int b = b0 + (e & (CB - 1));
    if (b < x.B) Y[(int64_t)(e >> x.cb_log2_row) * x.ldy + b] = cconj(sm[spad(e)]);
  }
}

template <int NCT = 0, int NBL = 0>
__global__ void __launch_bounds__(256, SFB_FFT_MINB) k_colinv_b(FftBArgs x) {
  extern __shared__ double2 sm[];
  const FftArgs& a = x.a;
  const int CB = 1 << x.cb_log2_col;
  const int64_t n1 = blockIdx.x;
  const int b0 = blockIdx.y * CB;
  const int L2 = (int)a.L2;
  const int n_el = L2 << x.cb_log2_col;
  const int T = blockDim.x;
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kU * T) {
    double2 v[kU], w[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int b = b0 + (e & (CB - 1));
      const int pp = e >> x.cb_log2_col;
      v[u] = make_double2(0.0, 0.0);
      w[u] = make_double2(1.0, 0.0);
      if (e < n_el && b < x.B) {
        v[u] = a.Y[(n1 + a.L1 * (int64_t)pp) * x.ldy + b];
        w[u] = wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)__ldg(a.rev2 + pp));
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (e0 + u * T < n_el) sm[spad(e0 + u * T)] = cmul(cconj(v[u]), w[u]);
  }
  __syncthreads();
  if constexpr (NCT > 0) fft_dit_ct<NCT, NBL, 256>(sm, a.st2, a.tw2);
  else fft_dit(sm, x.cb_log2_col, a.st2, a.tw2);
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kU * T) {
    double2 qv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int64_t k = n1 + a.L1 * (int64_t)(e >> x.cb_log2_col);
      qv[u] = make_double2(0.0, 0.0);
      if (e < n_el && k < a.Kout) qv[u] = __ldg(a.Q + k);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int b = b0 + (e & (CB - 1));
      const int64_t k = n1 + a.L1 * (int64_t)(e >> x.cb_log2_col);
      if (e < n_el && b < x.B && k < a.Kout) a.h[k * x.ldg + b] = cmul(cconj(sm[spad(e)]), qv[u]);
    }
  }
}

// ------------------------------ register-resident batched passes (fft_reg.cuh)
// Same three passes and layouts as k_colfwd_b / k_rowmul_b / k_colinv_b, with
// the butterflies held in registers: global loads feed the first stage, the
// last stage stores to global, and only the exchanges between stages go
// through shared memory.
template <int N, int NBL, int T, int MINB>
__global__ void __launch_bounds__(T, MINB) k_colfwd_rb(FftBArgs x) {
  using F = RegFft<N, NBL, T>;
  constexpr int S0 = N / 8;
  extern __shared__ double2 sm[];
  const FftArgs& a = x.a;
  const int64_t n1 = blockIdx.y;
  const int b0 = blockIdx.x * F::NB;  // column groups fastest: whole point rows
  F f;
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k), b = b0 + F::vec(k);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int64_t n = n1 + a.L1 * (int64_t)F::template pos<S0>(u, r);
      f.x[k][r] = make_double2(0.0, 0.0);
      if (b < x.B && n < a.K) f.x[k][r] = cmul(__ldg(a.g + n * x.ldg + b), __ldg(a.P + n));
    }
  }
  f.dif(sm, a.st2, a.tw2);
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k), b = b0 + F::vec(k);
    if (b >= x.B) continue;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int p = 8 * u + r;  // position p holds frequency rev8(p)
      const double2 w = wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)rev8<N>(p));
      a.Y[(n1 + a.L1 * (int64_t)p) * x.ldy + b] = cmul(f.x[k][r], w);
    }
  }
}

template <int N, int NBL, int T, int MINB>
__global__ void __launch_bounds__(T, MINB) k_rowmul_rb(FftBArgs x) {
  using F = RegFft<N, NBL, T>;
  constexpr int S0 = N / 8;
  extern __shared__ double2 sm[];
  const FftArgs& a = x.a;
  const int64_t p = blockIdx.y;
  const int b0 = blockIdx.x * F::NB;
  double2* Y = a.Y + p * a.L1 * x.ldy;
  F f;
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k), b = b0 + F::vec(k);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      f.x[k][r] = make_double2(0.0, 0.0);
      if (b < x.B) f.x[k][r] = Y[(int64_t)F::template pos<S0>(u, r) * x.ldy + b];
    }
  }
  f.dif(sm, a.st1, a.tw1);
  const double2* Bh = a.Bhat + p * a.L1;
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
#pragma unroll
    for (int r = 0; r < 8; ++r) f.x[k][r] = cconj(cmul(f.x[k][r], __ldg(Bh + 8 * u + r)));
  }
  f.dit(sm, a.st1, a.tw1);
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k), b = b0 + F::vec(k);
    if (b >= x.B) continue;
#pragma unroll
    for (int r = 0; r < 8; ++r)
      Y[(int64_t)F::template pos<S0>(u, r) * x.ldy + b] = cconj(f.x[k][r]);
  }
}

template <int N, int NBL, int T, int MINB>
__global__ void __launch_bounds__(T, MINB) k_colinv_rb(FftBArgs x) {
  using F = RegFft<N, NBL, T>;
  constexpr int S0 = N / 8;
  extern __shared__ double2 sm[];
  const FftArgs& a = x.a;
  const int64_t n1 = blockIdx.y;
  const int b0 = blockIdx.x * F::NB;  // column groups fastest: whole point rows
  F f;
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k), b = b0 + F::vec(k);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int p = 8 * u + r;
      f.x[k][r] = make_double2(0.0, 0.0);
      if (b < x.B) {
        const double2 v = a.Y[(n1 + a.L1 * (int64_t)p) * x.ldy + b];
        f.x[k][r] = cmul(cconj(v), wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)rev8<N>(p)));
      }
    }
  }
  f.dit(sm, a.st2, a.tw2);
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k), b = b0 + F::vec(k);
    if (b >= x.B) continue;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int64_t kk = n1 + a.L1 * (int64_t)F::template pos<S0>(u, r);
      if (kk < a.Kout) a.h[kk * x.ldg + b] = cmul(cconj(f.x[k][r]), __ldg(a.Q + kk));
    }
  }
}

// Single-column (column-major [batch][*]) register-resident passes: the NB
// vectors of a column CTA are NB consecutive n1 (as k_colfwd's C columns);
// the row CTA holds one row (NB = 1).
template <int N, int NBL, int T, int MINB, int R = 8, int PL = 0>
__global__ void __launch_bounds__(T, MINB) k_colfwd_r1(FftArgs a) {
  pdl_trigger();
  pdl_wait();  // reads the previous kernel's output
  using F = RegFft<N, NBL, T, R, PL>;
  constexpr int S0 = N / R;
  extern __shared__ double2 sm[];
  const int col = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * F::NB;
  const double2* g = a.g + (int64_t)col * a.K;
  F f;
#if SFB_FFT_BATCHLD
  // every load of the pass issued before the first use (no branch around a
  // load: out-of-range elements read index 0 and are zeroed after), so the
  // thread's 2R loads are in flight together instead of one pair at a time
  {
    int64_t idx[F::BPT][R];
    bool ok[F::BPT][R];
#pragma unroll
    for (int k = 0; k < F::BPT; ++k) {
      const int u = F::but(k);
      const int64_t n1 = c0 + F::vec(k);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t n = n1 + a.L1 * (int64_t)F::template pos<S0>(u, r);
        ok[k][r] = n1 < a.L1 && n < a.K;
        idx[k][r] = ok[k][r] ? n : 0;
      }
    }
    double2 pv[F::BPT][R];
#if SFB_FFT_ABL & 1  // timing ablation: no input loads
#pragma unroll
    for (int k = 0; k < F::BPT; ++k)
#pragma unroll
      for (int r = 0; r < R; ++r) f.x[k][r] = pv[k][r] = make_double2((double)idx[k][r], 1.0);
    if (false)
#endif
#pragma unroll
    for (int k = 0; k < F::BPT; ++k)
#pragma unroll
      for (int r = 0; r < R; ++r) f.x[k][r] = __ldg(g + idx[k][r]);
#if SFB_FFT_ABL & 1
    if (false)
#endif
#pragma unroll
    for (int k = 0; k < F::BPT; ++k)
#pragma unroll
      for (int r = 0; r < R; ++r) pv[k][r] = __ldg(a.P + idx[k][r]);
#pragma unroll
    for (int k = 0; k < F::BPT; ++k)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double2 gv = f.x[k][r];
        if (a.conj_in) gv.y = -gv.y;
        f.x[k][r] = ok[k][r] ? cmul(gv, pv[k][r]) : make_double2(0.0, 0.0);
      }
  }
#else
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
    const int64_t n1 = c0 + F::vec(k);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t n = n1 + a.L1 * (int64_t)F::template pos<S0>(u, r);
      f.x[k][r] = make_double2(0.0, 0.0);
      if (n1 < a.L1 && n < a.K) {
        double2 gv = __ldg(g + n);
        if (a.conj_in) gv.y = -gv.y;
        f.x[k][r] = cmul(gv, FFT_LD_TABLE(a.P + n));
      }
    }
  }
#endif
  f.dif(sm, R == 16 ? a.st2x : a.st2, R == 16 ? a.tw2x : a.tw2);
  double2* Y = a.Y + (int64_t)col * a.L;
#if SFB_FFT_BATCHLD
  {
    double2 tw[F::BPT][R];
#pragma unroll
    for (int k = 0; k < F::BPT; ++k) {
      const int u = F::but(k);
      const int64_t n1 = min(c0 + F::vec(k), a.L1 - 1);
#pragma unroll
      for (int r = 0; r < R; ++r)
        tw[k][r] = wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)revr<N, R>(R * u + r));
    }
#pragma unroll
    for (int k = 0; k < F::BPT; ++k) {
      const int u = F::but(k);
      const int64_t n1 = c0 + F::vec(k);
      if (n1 >= a.L1) continue;
#pragma unroll
      for (int r = 0; r < R; ++r) {
#if SFB_FFT_ABL & 2  // timing ablation: stores only for a NaN
        if (f.x[k][r].x != f.x[k][r].x)
#endif
        Y[n1 + a.L1 * (int64_t)(R * u + r)] = cmul(f.x[k][r], tw[k][r]);
      }
    }
  }
#else
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
    const int64_t n1 = c0 + F::vec(k);
    if (n1 >= a.L1) continue;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int p = R * u + r;
      FFT_ST_KEEP(Y + n1 + a.L1 * (int64_t)p, cmul(f.x[k][r], wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)revr<N, R>(p))));
    }
  }
#endif
}

// ------------------------------------- TMA-pipelined persistent column pass
// k_colfwd_r1 as a persistent kernel (one 512-thread CTA per SM, all 148
// resident) whose tiles (NB = 4 adjacent columns x 1024 rows = 64 KB) move
// with 2D TMA tensor copies through a 3-stage shared-memory ring: the tile
// two ahead is loaded (cp.async.bulk.tensor.2d, UTMALDG) and the previous
// tile is stored (cp.async.bulk.tensor.2d global <- shared, UTMASTG) while
// the current one is transformed in registers.  The stage buffer that
// received a tile serves as that tile's exchange buffer and then stages its
// output.  The prechirp P of the next tile is prefetched into registers.
// Single column (batch 1) with a grid padded to whole rows of L1.
struct TmaMaps {
  CUtensorMap in;   // grid g viewed as [rows][2 * L1] float64
  CUtensorMap out;  // work Y viewed as [L2][2 * L1] float64
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            unsigned long long* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(mbar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int c0, int c1,
                                             const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
          reinterpret_cast<uint64_t>(tm)),
      "r"(c0), "r"(c1), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

constexpr int kTmaStages = 3;
constexpr int kTmaBox = 256;  // rows per TMA box (box dims <= 256)

template <int N, int T>
__global__ void __launch_bounds__(T, 1) k_colfwd_tma(FftArgs a, const __grid_constant__ TmaMaps tm,
                                                     int ntiles) {
  using F = RegFft<N, 2, T, 8>;
  constexpr int R = 8, NB = F::NB, S0 = N / R;
  constexpr int TILE = N * NB;  // double2 per tile
  static_assert(F::BPT == 1, "one radix-8 butterfly per thread");
  extern __shared__ __align__(128) double2 smt[];
  __shared__ __align__(8) unsigned long long full[kTmaStages];
  const int tid = threadIdx.x;
  const int u = F::but(0), b = F::vec(0);
  pdl_trigger();
  if (tid == 0) {
    for (int i = 0; i < kTmaStages; ++i) mbar_init(&full[i], 1);
  }
  __syncthreads();
  pdl_wait();  // the grid is the previous kernel's output
  // rows of the input that can hold nonzeros: the rest is zero (pruned)
  const int in_rows = (int)((a.K + a.L1 - 1) / a.L1);
  const int in_boxes = (in_rows + kTmaBox - 1) / kTmaBox;
  auto issue_load = [&](int t, int st) {
    double2* buf = smt + (size_t)st * TILE;
    const int c0 = 2 * NB * t;  // float64 column of the tile
    mbar_expect_tx(&full[st], (unsigned)(in_boxes * kTmaBox * NB * sizeof(double2)));
    for (int q = 0; q < in_boxes; ++q)
      tma_load_2d(buf + q * kTmaBox * NB, &tm.in, c0, q * kTmaBox, &full[st]);
  };
  int t = blockIdx.x;
  if (tid == 0) {
    if (t < ntiles) issue_load(t, 0);
    if (t + (int)gridDim.x < ntiles) issue_load(t + gridDim.x, 1);
  }
  // P of this thread's 8 inputs, one tile ahead
  auto load_p = [&](int tt, double2* pv) {
    const int64_t n1 = (int64_t)tt * NB + b;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t n = n1 + a.L1 * (int64_t)(u + r * S0);
      pv[r] = __ldg(a.P + (n < a.K ? n : 0));
    }
  };
  double2 pv[R];
  if (t < ntiles) load_p(t, pv);
  F f;
  for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
    const int st = i % kTmaStages;
    double2* buf = smt + (size_t)st * TILE;
    const int64_t n1 = (int64_t)t * NB + b;
    mbar_wait(&full[st], (i / kTmaStages) & 1);
    // rows >= in_boxes * kTmaBox were not loaded: they are zero
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = u + r * S0;
      const int64_t n = n1 + a.L1 * (int64_t)row;
      double2 gv = row < in_boxes * kTmaBox ? buf[row * NB + b] : make_double2(0.0, 0.0);
      if (a.conj_in) gv.y = -gv.y;
      f.x[0][r] = n < a.K ? cmul(gv, pv[r]) : make_double2(0.0, 0.0);
    }
    // the output twiddles W_L^{n1 rev(p)} (L2-resident tables) and the next
    // tile's P are in flight during the transform
    double2 tw[R];
#pragma unroll
    for (int r = 0; r < R; ++r) tw[r] = wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)revr<N, R>(R * u + r));
    if (t + (int)gridDim.x < ntiles) load_p(t + gridDim.x, pv);
    __syncthreads();  // every input read: the stage becomes the exchange buffer
    f.dif(buf, a.st2, a.tw2);
    __syncthreads();  // exchanges done: the stage now stages the output tile
#pragma unroll
    for (int r = 0; r < R; ++r) buf[(R * u + r) * NB + b] = cmul(f.x[0][r], tw[r]);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const int c0 = 2 * NB * t;
      for (int q = 0; q < N / kTmaBox; ++q)
        tma_store_2d(&tm.out, c0, q * kTmaBox, buf + q * kTmaBox * NB);
      bulk_commit();
      // the load two tiles ahead reuses the stage of the PREVIOUS tile's
      // output: its store (one group back) must have finished reading
      const int t2 = t + 2 * gridDim.x;
      if (t2 < ntiles) {
        bulk_wait_read<1>();
        issue_load(t2, (i + 2) % kTmaStages);
      }
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // stores complete
}

template <int N, int T, int MINB, int R = 8, int PL = 0>
__global__ void __launch_bounds__(T, MINB) k_rowmul_r1(FftArgs a) {
  pdl_trigger();
  pdl_wait();  // reads the previous kernel's output
  using F = RegFft<N, 0, T, R, PL>;
  constexpr int S0 = N / R;
  extern __shared__ double2 sm[];
  const int col = blockIdx.y;
  const int64_t p = blockIdx.x;
  double2* row = a.Y + (int64_t)col * a.L + p * a.L1;
  F f;
#if SFB_FFT_ROW_TMA
  // the row is one contiguous 64 KB range: one TMA bulk copy into the
  // exchange buffer (linear layout), stage-0 legs read from it, one barrier
  // before the first (swizzled) exchange reuses the buffer
  __shared__ __align__(8) unsigned long long mbar;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    bulk_g2s(sm, row, (unsigned)(sizeof(double2) * N), &mbar);
  }
  __syncthreads();
  mbar_wait(&mbar, 0);
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
#pragma unroll
    for (int r = 0; r < R; ++r) f.x[k][r] = sm[F::template pos<S0>(u, r)];
  }
  __syncthreads();
#else
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
#pragma unroll
    for (int r = 0; r < R; ++r) f.x[k][r] = FFT_ROW_LD(row + F::template pos<S0>(u, r));
  }
#endif
  f.dif(sm, R == 16 ? a.st1x : a.st1, R == 16 ? a.tw1x : a.tw1);
  const double2* Bh = (R == 16 ? a.Bhatx : a.Bhat) + p * a.L1;
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
#pragma unroll
    for (int r = 0; r < R; ++r) f.x[k][r] = cconj(cmul(f.x[k][r], FFT_ROW_TAB(Bh + R * u + r)));
  }
  f.dit(sm, R == 16 ? a.st1x : a.st1, R == 16 ? a.tw1x : a.tw1);
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
#pragma unroll
    for (int r = 0; r < R; ++r) FFT_ROW_ST(row + F::template pos<S0>(u, r), cconj(f.x[k][r]));
  }
}

template <int N, int NBL, int T, int MINB, int R = 8, int PL = 0>
__global__ void __launch_bounds__(T, MINB) k_colinv_r1(FftArgs a) {
  pdl_trigger();
  pdl_wait();  // reads the previous kernel's output
  using F = RegFft<N, NBL, T, R, PL>;
  constexpr int S0 = N / R;
  extern __shared__ double2 sm[];
  const int col = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * F::NB;
  const double2* Y = a.Y + (int64_t)col * a.L;
  F f;
#if SFB_FFT_BATCHLD
  {
    double2 tw[F::BPT][R];
#pragma unroll
    for (int k = 0; k < F::BPT; ++k) {
      const int u = F::but(k);
      const int64_t n1 = min(c0 + F::vec(k), a.L1 - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        f.x[k][r] = Y[n1 + a.L1 * (int64_t)(R * u + r)];
        tw[k][r] = wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)revr<N, R>(R * u + r));
      }
    }
#pragma unroll
    for (int k = 0; k < F::BPT; ++k) {
      const bool ok = c0 + F::vec(k) < a.L1;
#pragma unroll
      for (int r = 0; r < R; ++r)
        f.x[k][r] = ok ? cmul(cconj(f.x[k][r]), tw[k][r]) : make_double2(0.0, 0.0);
    }
  }
#else
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
    const int64_t n1 = c0 + F::vec(k);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int p = R * u + r;
      f.x[k][r] = make_double2(0.0, 0.0);
      if (n1 < a.L1)
        f.x[k][r] = cmul(cconj(FFT_LD_ONCE(Y + n1 + a.L1 * (int64_t)p)),
                         wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)revr<N, R>(p)));
    }
  }
#endif
  f.dit(sm, R == 16 ? a.st2x : a.st2, R == 16 ? a.tw2x : a.tw2);
  double2* h = a.h + (int64_t)col * a.Kout;
#if SFB_FFT_BATCHLD
  {
    double2 qv[F::BPT][R];
#pragma unroll
    for (int k = 0; k < F::BPT; ++k) {
      const int u = F::but(k);
      const int64_t n1 = c0 + F::vec(k);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t kk = n1 + a.L1 * (int64_t)F::template pos<S0>(u, r);
        qv[k][r] = __ldg(a.Q + ((kk < a.Kout && n1 < a.L1) ? kk : 0));
      }
    }
#pragma unroll
    for (int k = 0; k < F::BPT; ++k) {
      const int u = F::but(k);
      const int64_t n1 = c0 + F::vec(k);
      if (n1 >= a.L1) continue;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t kk = n1 + a.L1 * (int64_t)F::template pos<S0>(u, r);
        if (kk < a.Kout) h[kk] = cmul(cconj(f.x[k][r]), qv[k][r]);
      }
    }
  }
#else
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
    const int64_t n1 = c0 + F::vec(k);
    if (n1 >= a.L1) continue;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t kk = n1 + a.L1 * (int64_t)F::template pos<S0>(u, r);
      if (kk < a.Kout) FFT_ST_KEEP(h + kk, cmul(cconj(f.x[k][r]), FFT_LD_TABLE(a.Q + kk)));
    }
  }
#endif
}

// ------------------------------------------- distributed (column-split) FFT
// The three Bluestein passes split over P ranks: rank r
// owns the Bc = L1/P columns n1 in [r Bc, (r+1) Bc) for the column passes and
// the Br = L2/P rows p in [r Br, (r+1) Br) for the row pass.  Host-side
// collectives (sharding.py) move the data between the layouts below:
//   pack      partial grid g[K] -> S[P][Sb], S[q] = columns of rank q as
//             [i][c] (g[q Bc + c + L1 i], i < I = ceil(K/L1)), plus the
//             Bluestein tail fix of THIS rank's partial grid in rank 0's block
//             (linear, so the reduce-scatter sums it too)      -> reduce-scatter
//   colfwd    own block [i][c] -> Yc[p][c] (p in [0, L2): rank-major rows
//             for the all-to-all)                              -> all-to-all
//   rowmul    rows [q][p_local][c] in place (q = source rank)  -> all-to-all
//   colinv    [p][c] -> H[k2][c] = h[r Bc + c + L1 k2], k2 < K2 = ceil(Kout/L1)
//             (rank 0 adds the summed tail fix)                -> all-gather
//   unpack    [P][K2][Bc] -> h[Kout] natural, then the ordinary gather.
// Instantiated for the config-3 shape (L1 = 4096 rows, L2 = 1024 columns); a
// plan without it keeps the replicated FFT after an all-reduce.
struct DistArgs {
  FftArgs a;
  int rank, world;
  int64_t Bc, Br, I, K2, Sb;
  int bc_log2, br_log2;
  // fused transposes over peer memory (NVLink P2P / CUDA IPC): when set, the
  // column pass and the row pass store every element straight into the
  // receive buffer of the rank that owns it (the layout the all-to-all would
  // have delivered), so no collective runs between the passes
  int use_peers;
  double2* peer[kDistMaxRanks];
  // fused first / last exchanges: this sender's chunk offset in each
  // receiver's grid-row buffer; every receiver's h-row range; rank 0's fix
  int64_t poff[kDistMaxRanks];
  int64_t hlo[kDistMaxRanks], hcnt[kDistMaxRanks];
  const double2* fixp;
  int64_t fixD;
};

__global__ void k_dpack(const double2* __restrict__ g, double2* __restrict__ S, DistArgs d) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= d.world * d.Sb) return;
  const int64_t q = o / d.Sb, e = o - q * d.Sb;
  double2 v = make_double2(0.0, 0.0);
  if (e < d.I * d.Bc) {
    const int64_t i = e >> d.bc_log2, c = e & (d.Bc - 1);
    const int64_t n = q * d.Bc + c + d.a.L1 * i;
    if (n < d.a.K) v = g[n];
  }
  S[o] = v;
}

template <int N, int NBL, int T, int MINB, int R = 8>
__global__ void __launch_bounds__(T, MINB) k_dcolfwd(DistArgs d, const double2* __restrict__ Rb,
                                                    double2* __restrict__ Yc) {
  using F = RegFft<N, NBL, T, R>;
  constexpr int S0 = N / R;
  extern __shared__ double2 sm[];
  const FftArgs& a = d.a;
  const int64_t c0 = (int64_t)blockIdx.x * F::NB;
  F f;
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
    const int64_t c = c0 + F::vec(k), n1 = d.rank * d.Bc + c;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = F::template pos<S0>(u, r);
      const int64_t n = n1 + a.L1 * i;
      f.x[k][r] = make_double2(0.0, 0.0);
      if (i < d.I && n < a.K) f.x[k][r] = cmul(__ldg(Rb + (i << d.bc_log2) + c), __ldg(a.P + n));
    }
  }
  f.dif(sm, R == 16 ? a.st2x : a.st2, R == 16 ? a.tw2x : a.tw2);
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
    const int64_t c = c0 + F::vec(k), n1 = d.rank * d.Bc + c;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int p = R * u + r;
      const double2 v = cmul(f.x[k][r], wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)revr<N, R>(p)));
      if (d.use_peers)  // row p belongs to rank p / Br: its block from this rank
        d.peer[p >> d.br_log2][((((int64_t)d.rank << d.br_log2) + (p & (d.Br - 1))) << d.bc_log2) + c] = v;
      else
        Yc[((int64_t)p << d.bc_log2) + c] = v;
    }
  }
}

template <int N, int T, int MINB, int R = 8>
__global__ void __launch_bounds__(T, MINB) k_drowmul(DistArgs d, double2* __restrict__ Rr) {
  using F = RegFft<N, 0, T, R>;
  constexpr int S0 = N / R;
  extern __shared__ double2 sm[];
  const FftArgs& a = d.a;
  const int64_t pl = blockIdx.x, p = d.rank * d.Br + pl;
  // element n1 of local row pl: block (n1 / Bc) of the all-to-all, [pl][n1 % Bc]
  auto at = [&](int n1) -> int64_t {
    return ((((int64_t)(n1 >> d.bc_log2)) * d.Br + pl) << d.bc_log2) + (n1 & (d.Bc - 1));
  };
  F f;
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
#pragma unroll
    for (int r = 0; r < R; ++r) f.x[k][r] = Rr[at(F::template pos<S0>(u, r))];
  }
  f.dif(sm, R == 16 ? a.st1x : a.st1, R == 16 ? a.tw1x : a.tw1);
  const double2* Bh = (R == 16 ? a.Bhatx : a.Bhat) + p * a.L1;
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
#pragma unroll
    for (int r = 0; r < R; ++r) f.x[k][r] = cconj(cmul(f.x[k][r], __ldg(Bh + R * u + r)));
  }
  f.dit(sm, R == 16 ? a.st1x : a.st1, R == 16 ? a.tw1x : a.tw1);
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int n1 = F::template pos<S0>(u, r);
      if (d.use_peers)  // column n1 belongs to rank n1 / Bc: block [this rank][pl][c]
        d.peer[n1 >> d.bc_log2][((((int64_t)d.rank << d.br_log2) + pl) << d.bc_log2) +
                                (n1 & (d.Bc - 1))] = cconj(f.x[k][r]);
      else
        Rr[at(n1)] = cconj(f.x[k][r]);
    }
  }
}

template <int N, int NBL, int T, int MINB, int R = 8>
__global__ void __launch_bounds__(T, MINB) k_dcolinv(DistArgs d, const double2* __restrict__ Y2,
                                                    double2* __restrict__ H) {
  using F = RegFft<N, NBL, T, R>;
  constexpr int S0 = N / R;
  extern __shared__ double2 sm[];
  const FftArgs& a = d.a;
  const int64_t c0 = (int64_t)blockIdx.x * F::NB;
  F f;
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
    const int64_t c = c0 + F::vec(k), n1 = d.rank * d.Bc + c;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int p = R * u + r;
      f.x[k][r] = cmul(cconj(__ldg(Y2 + ((int64_t)p << d.bc_log2) + c)),
                       wbig(a.tw_lo, a.tw_hi, n1 * (int64_t)revr<N, R>(p)));
    }
  }
  f.dit(sm, R == 16 ? a.st2x : a.st2, R == 16 ? a.tw2x : a.tw2);
#pragma unroll
  for (int k = 0; k < F::BPT; ++k) {
    const int u = F::but(k);
    const int64_t c = c0 + F::vec(k), n1 = d.rank * d.Bc + c;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t k2 = F::template pos<S0>(u, r);
      const int64_t kk = n1 + a.L1 * k2;
      if (k2 < d.K2 && kk < a.Kout) {
        double2 v = cmul(cconj(f.x[k][r]), __ldg(a.Q + kk));
        if (d.use_peers) {  // straight into every rank whose targets read h row k2
          if (d.fixp && kk < d.fixD) v = cadd(v, d.fixp[kk]);  // rank 0: the Bluestein tail fix
          for (int q = 0; q < d.world; ++q) {
            const int64_t lk = k2 - d.hlo[q];
            if (lk >= 0 && lk < d.hcnt[q])
              d.peer[q][((d.rank * d.hcnt[q] + lk) << d.bc_log2) + c] = v;
          }
        } else {
          H[(k2 << d.bc_log2) + c] = v;
        }
      }
    }
  }
}

__global__ void k_dfix_add(double2* H, const double2* __restrict__ fix, int64_t D) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < D) {  // k' < D <= Bc: column k', k2 = 0 of rank 0's block
    H[k].x += fix[k].x;
    H[k].y += fix[k].y;
  }
}

__global__ void k_dunpack(const double2* __restrict__ Hall, double2* __restrict__ h, DistArgs d) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= d.a.Kout) return;
  const int64_t n1 = k % d.a.L1, k2 = k / d.a.L1;
  const int64_t q = n1 >> d.bc_log2, c = n1 & (d.Bc - 1);
  h[k] = Hall[((q * d.K2 + k2) << d.bc_log2) + c];
}

// Sparse exchange for position partitions: a rank's partial grid is nonzero
// only on rows [ilo, ilo + nrow) (row i = grid indices [i L1, (i+1) L1)), and
// its targets read only h rows [k2lo, k2lo + cnt); so the reduce-scatter and
// the all-gather become all-to-alls of those rows (per rank ~K/P and
// ~Kout/P complex instead of K and Kout).  Chunks destined to rank 0 carry
// the sender's partial tail fix (Dpad extra elements).
__global__ void k_dpack_rows(const double2* __restrict__ g, double2* __restrict__ S, DistArgs d,
                             int64_t ilo, int64_t nrow, int64_t dpad) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t seg = nrow * d.Bc;
  const int64_t total = d.world * seg + dpad;
  if (o >= total) return;
  // chunk 0 = [rows of column block 0][fix], then chunks 1.. of seg elements
  int64_t q, e;
  if (o < seg + dpad) {
    q = 0, e = o;
  } else {
    q = 1 + (o - seg - dpad) / seg, e = (o - seg - dpad) % seg;
  }
  double2 v = make_double2(0.0, 0.0);
  if (e < seg) {
    const int64_t i = ilo + (e >> d.bc_log2), c = e & (d.Bc - 1);
    const int64_t n = q * d.Bc + c + d.a.L1 * i;
    if (n < d.a.K) v = g[n];
  }
  if (d.use_peers) d.peer[q][d.poff[q] + e] = v;  // straight into receiver q's buffer
  else S[o] = v;
}

__global__ void k_dunpack_rows(const double2* __restrict__ recv, double2* __restrict__ R,
                               DistArgs d, RowSplit rs, int64_t dfix) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nblk = d.I * d.Bc;
  if (o >= nblk + dfix) return;
  double2 acc = make_double2(0.0, 0.0);
  if (o < nblk) {
    const int64_t i = o >> d.bc_log2, c = o & (d.Bc - 1);
    for (int s = 0; s < rs.n; ++s) {
      const int64_t li = i - rs.lo[s];
      if (li >= 0 && li < rs.cnt[s]) {
        const double2 v = recv[rs.off[s] + (li << d.bc_log2) + c];
        acc.x += v.x;
        acc.y += v.y;
      }
    }
  } else {  // rank 0: the senders' tail-fix partials follow their rows
    const int64_t k = o - nblk;
    for (int s = 0; s < rs.n; ++s) {
      const double2 v = recv[rs.off[s] + (rs.cnt[s] << d.bc_log2) + k];
      acc.x += v.x;
      acc.y += v.y;
    }
  }
  R[o] = acc;
}

__global__ void k_dpack_hrows(const double2* __restrict__ H, double2* __restrict__ S, DistArgs d,
                              RowSplit rs, int64_t total) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= total) return;
  int r = 0;
  while (r + 1 < rs.n && o >= rs.off[r + 1]) ++r;
  const int64_t e = o - rs.off[r];
  const int64_t k2 = rs.lo[r] + (e >> d.bc_log2), c = e & (d.Bc - 1);
  S[o] = k2 < d.K2 ? H[(k2 << d.bc_log2) + c] : make_double2(0.0, 0.0);
}

__global__ void k_dunpack_hrows(const double2* __restrict__ recv, double2* __restrict__ h,
                                DistArgs d, int64_t k2lo, int64_t cnt) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t seg = cnt * d.Bc;
  if (o >= d.world * seg) return;
  const int64_t q = o / seg, e = o - q * seg;
  const int64_t k2 = k2lo + (e >> d.bc_log2), c = e & (d.Bc - 1);
  const int64_t k = q * d.Bc + c + d.a.L1 * k2;
  if (k < d.a.Kout) h[k] = recv[o];
}

// ------------------------------------------------------ direct four-step
// n = P n1 + n2 (n1 < A, n2 < P),  k = k1 + A k2:
//   X[k1 + A k2] = sum_n2 W_P^{n2 k2} [ W_N2^{n2 k1} sum_n1 x[P n1 + n2] W_A^{n1 k1} ]
// x[n] = g[l] D[l] for n = (l - K/2) mod N2, l in [0, K) (the embedded,
// deconvolved grid of nnfft.py:236-238 with the 1/N1, 1/N2 factors in D).
struct DirectArgs {
  const double2* g;   // [batch][K]
  const double* D;
  double2* Y;         // [batch][A][P]
  double2* h;         // [batch][Kout]
  const double2* twA;
  const double2* twP;
  const double2* w_lo;  // W_N2 two-level table
  const double2* w_hi;
  const double2* cp;    // omega_P^{n^2/2}, n < P
  const double2* bhat;  // FFT_LP(b)/LP, reversed layout
  const int* revA;
  const int* revP;
  int64_t K, N2, A, P, LP, Kout, s_lo;
  int C_log2, R_log2;
  int p_smooth;
  int conj_in;
  FftStages stA, stP;
  // Rader rows (P prime, P - 1 smooth): input gather g^q, output scatter g^-q
  int rader;
  const int* rin;
  const int* rout;
};

__global__ void __launch_bounds__(256, SFB_FFT_MINB) k_dstep1(DirectArgs a) {
  extern __shared__ double2 sm[];
  const int col = blockIdx.y;
  const int C = 1 << a.C_log2;
  const int64_t c0 = (int64_t)blockIdx.x * C;
  const int A = (int)a.A;
  const int n_el = A << a.C_log2;
  const int T = blockDim.x;
  const double2* g = a.g + (int64_t)col * a.K;
  const int64_t halfK = a.K / 2;
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kU * T) {
    double2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int64_t n2 = c0 + (e & (C - 1));
      const int64_t n = a.P * (int64_t)(e >> a.C_log2) + n2;
      v[u] = make_double2(0.0, 0.0);
      if (e < n_el && n2 < a.P) {
        int64_t l = -1;
        if (n < a.K - halfK) l = n + halfK;                     // n in [0, K/2)
        else if (n >= a.N2 - halfK) l = n - a.N2 + halfK;       // n in [N2 - K/2, N2)
        if (l >= 0) {
          double2 gv = __ldg(g + l);
          if (a.conj_in) gv.y = -gv.y;
          v[u] = cscale(gv, __ldg(a.D + l));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (e0 + u * T < n_el) sm[spad(e0 + u * T)] = v[u];
  }
  __syncthreads();
  fft_dif(sm, a.C_log2, a.stA, a.twA);
  double2* Y = a.Y + (int64_t)col * a.A * a.P;
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kU * T) {
    double2 w[kU];
    int64_t k1v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int64_t n2 = c0 + (e & (C - 1));
      w[u] = make_double2(1.0, 0.0);
      k1v[u] = 0;
      if (e < n_el && n2 < a.P) {
        k1v[u] = __ldg(a.revA + (e >> a.C_log2));
        w[u] = wbig(a.w_lo, a.w_hi, n2 * k1v[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int64_t n2 = c0 + (e & (C - 1));
      if (e < n_el && n2 < a.P) Y[k1v[u] * a.P + n2] = cmul(sm[spad(e)], w[u]);
    }
  }
}

__global__ void __launch_bounds__(256, SFB_FFT_MINB) k_dstep2(DirectArgs a) {
  extern __shared__ double2 sm[];
  __shared__ double2 y0s[64], a0s[64];  // Rader: y[0] and sum_{n>0} y[n] per row
  const int col = blockIdx.y;
  const int R = 1 << a.R_log2;
  const int64_t r0 = (int64_t)blockIdx.x * R;
  const int n = a.p_smooth ? (int)a.P : (int)a.LP;
  const int n_el = n << a.R_log2;
  const int T = blockDim.x;
  const double2* Y = a.Y + (int64_t)col * a.A * a.P;
  // load rows r0.. (element (n2, row b) at e = n2 * R + b): Bluestein
  // pre-chirp, or the Rader gather a_q = y[g^q mod P], q < P - 1
  for (int e0 = threadIdx.x; e0 < n_el; e0 += kU * T) {
    double2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * T;
      const int64_t k1 = r0 + (e & (R - 1));
      const int n2 = e >> a.R_log2;
      v[u] = make_double2(0.0, 0.0);
      if (a.rader) {
        if (e < n_el && k1 < a.A) v[u] = Y[k1 * a.P + __ldg(a.rin + n2)];
      } else if (e < n_el && k1 < a.A && n2 < a.P) {
        v[u] = Y[k1 * a.P + n2];
        if (!a.p_smooth) v[u] = cmul(v[u], __ldg(a.cp + n2));
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (e0 + u * T < n_el) sm[spad(e0 + u * T)] = v[u];
  }
  if (a.rader && threadIdx.x < R) {
    const int64_t k1 = r0 + threadIdx.x;
    y0s[threadIdx.x] = k1 < a.A ? Y[k1 * a.P] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_dif(sm, a.R_log2, a.stP, a.twP);
  if (!a.p_smooth) {
    if (a.rader && threadIdx.x < R) a0s[threadIdx.x] = sm[spad(threadIdx.x)];  // DFT bin 0
    __syncthreads();
    for (int e = threadIdx.x; e < n_el; e += T)
      sm[spad(e)] = cconj(cmul(sm[spad(e)], __ldg(a.bhat + (e >> a.R_log2))));
    __syncthreads();
    fft_dit(sm, a.R_log2, a.stP, a.twP);
  }
  double2* h = a.h + (int64_t)col * a.Kout;
  const int nout = (int)(a.rader ? a.P - 1 : a.P) << a.R_log2;  // positions of each row
  for (int e = threadIdx.x; e < nout; e += T) {
    const int b = e & (R - 1);
    const int64_t k1 = r0 + b;
    if (k1 >= a.A) continue;
    const int q = e >> a.R_log2;
    int64_t k2;
    double2 X;
    if (a.rader) {  // X[g^-q] = y[0] + (a conv w)[q]
      k2 = __ldg(a.rout + q);
      X = cadd(y0s[b], cconj(sm[spad(e)]));
    } else if (a.p_smooth) {
      k2 = __ldg(a.revP + q);
      X = sm[spad(e)];
    } else {
      k2 = q;
      X = cmul(cconj(sm[spad(e)]), __ldg(a.cp + q));
    }
    int64_t kk = (k1 + a.A * k2 - a.s_lo) % a.N2;
    if (kk < 0) kk += a.N2;
    if (kk < a.Kout) h[kk] = X;
  }
  if (a.rader && threadIdx.x < R && r0 + threadIdx.x < a.A) {  // X[0] = y[0] + sum_{n>0} y[n]
    int64_t kk = (r0 + threadIdx.x - a.s_lo) % a.N2;
    if (kk < 0) kk += a.N2;
    if (kk < a.Kout) h[kk] = cadd(y0s[threadIdx.x], a0s[threadIdx.x]);
  }
}

// b_j = conj(cp_|j|) on the cyclic length LP: j in [0, P) and LP - j, j in [1, P)
__global__ void k_bluestein_b(double2* b, const double2* cp, int64_t P, int64_t LP) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= LP) return;
  int64_t j = -1;
  if (i < P) j = i;
  else if (i > LP - P) j = LP - i;
  b[i] = j >= 0 ? cconj(cp[j]) : make_double2(0.0, 0.0);
}

__global__ void k_chirp_p(double2* cp, int64_t P) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= P) return;
  // omega_P^{n^2/2} = exp(-pi i (n^2 mod 2P) / P)
  const int64_t r = (n * n) % (2 * P);
  double sn, cs;
  sincospi(-(double)r / (double)P, &sn, &cs);
  cp[n] = make_double2(cs, sn);
}

__global__ void k_deconv(double* D, const double* hat2, int64_t K, double inv_n1n2) {
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l < K) D[l] = hat2 ? inv_n1n2 / hat2[l] : inv_n1n2;
}

// ------------------------------------------------------------ host planning
namespace {

bool smooth7(int64_t x) {
  for (int p : {2, 3, 5, 7})
    while (x % p == 0) x /= p;
  return x == 1;
}

int64_t next_smooth(int64_t x) {
  while (!smooth7(x)) ++x;
  return x;
}

FftStages make_stages(int64_t n) {
  FftStages st{};
  st.n = (int)n;
  int64_t r = n;
  std::vector<int> rad;
#if SFB_FFT_MAXR >= 16
  while (r % 16 == 0) rad.push_back(16), r /= 16;
#endif
  while (r % 8 == 0) rad.push_back(8), r /= 8;
  if (r % 4 == 0) rad.push_back(4), r /= 4;
  if (r % 2 == 0) rad.push_back(2), r /= 2;
  for (int p : {7, 5, 3})
    while (r % p == 0) rad.push_back(p), r /= p;
  if (r != 1) fail(3, "internal: non-smooth FFT length");
  if ((int)rad.size() > kMaxStages) fail(3, "internal: too many FFT stages");
  st.nst = (int)rad.size();
  int off = 0, S = (int)n;
  for (int i = 0; i < st.nst; ++i) {
    st.rad[i] = rad[i];
    S /= rad[i];
    st.toff[i] = off;
    off += S;
  }
  if (st.nst == 0) {  // n == 1: no stages
    st.nst = 0;
  }
  return st;
}

// the radix-16 decomposition of a power-of-two n (16s first, then one 8/4/2)
FftStages make_stages16(int64_t n) {
  FftStages st{};
  st.n = (int)n;
  int64_t r = n;
  std::vector<int> rad;
  while (r % 16 == 0) rad.push_back(16), r /= 16;
  if (r % 8 == 0) rad.push_back(8), r /= 8;
  if (r % 4 == 0) rad.push_back(4), r /= 4;
  if (r % 2 == 0) rad.push_back(2), r /= 2;
  if (r != 1) fail(3, "internal: make_stages16 needs a power of two");
  st.nst = (int)rad.size();
  int off = 0, S = (int)n;
  for (int i = 0; i < st.nst; ++i) {
    st.rad[i] = rad[i];
    S /= rad[i];
    st.toff[i] = off;
    off += S;
  }
  return st;
}

// position p after DIF holds frequency rev[p]
std::vector<int> digit_reverse(const FftStages& st) {
  std::vector<int> rev(st.n);
  for (int p = 0; p < st.n; ++p) {
    int rem = p, S = st.n, G = 1, k = 0;
    for (int q = 0; q < st.nst; ++q) {
      S /= st.rad[q];
      const int d = rem / S;
      rem %= S;
      k += d * G;
      G *= st.rad[q];
    }
    rev[p] = k;
  }
  return rev;
}

// Relative cost of one length-n smem FFT per point: every stage is one
// shared-memory round trip (~4 DFMA-equivalents per point) plus its
// butterfly arithmetic per point (radix 16/8/4/2 are cheap, odd radices not).
double stage_cost(int64_t n) {
  double c = 0;
  const FftStages st = make_stages(n);
  for (int i = 0; i < st.nst; ++i) {
    switch (st.rad[i]) {
      case 16: c += 4 + 6.5; break;
      case 8: c += 4 + 5.5; break;
      case 4: c += 4 + 4.5; break;
      case 2: c += 4 + 3.0; break;
      case 3: c += 4 + 7.0; break;
      case 5: c += 4 + 10.0; break;
      case 7: c += 4 + 14.0; break;
    }
  }
  return c;
}

// Model cost of the four-step L1 x L2 (smem stage costs per point), with
// factors calibrated on B200 (config 3: 4096 x 1024 best, 8192-point rows
// 16 % slower; config 4 point-major: 512 x 512 best, 4096 x 64 1.8x slower).
double cost(int64_t L1, int64_t L2) {
  double c = (double)(L1 * L2) * (2.0 * stage_cost(L1) + 2.0 * stage_cost(L2) + 12.0);
  if (L1 > 4096) c *= 1.25;       // rows above 64 KiB: one CTA per SM
  if (L1 > 16 * L2) c *= 1.3;     // very short columns starve the column kernels
  // column kernels move C contiguous elements (16*C bytes) per row
  int C = 8;
  while (C > 1 && C * L2 > kColElems) C >>= 1;
  if (C < 8) c *= 1.0 + 0.04 * (C == 4 ? 1 : C == 2 ? 2 : 3);
  return c;
}

// compact per-stage twiddles of an n-point FFT: stage q holds W_n^{j*G_q}, j < S_q
void launch_stage_twiddles(DevArray<double2>& t, const FftStages& st, cudaStream_t s) {
  int64_t total = 0, S = st.n, G = 1;
  for (int q = 0; q < st.nst; ++q) S /= st.rad[q], total += S;
  t.alloc(std::max<int64_t>(total, 1));
  S = st.n;
  for (int q = 0; q < st.nst; ++q) {
    S /= st.rad[q];
    k_twiddle<<<(unsigned)ceil_div(S, 256), 256, 0, s>>>(t.p + st.toff[q], st.n, S, G);
    SF_LAUNCH_CHECK();
    G *= st.rad[q];
  }
}

void launch_twiddle(DevArray<double2>& t, int64_t n, int64_t count, int64_t step,
                    cudaStream_t s) {
  t.alloc(std::max<int64_t>(count, 1));
  k_twiddle<<<(unsigned)ceil_div(count, 256), 256, 0, s>>>(t.p, n, count, step);
  SF_LAUNCH_CHECK();
}

size_t smem_bytes(int64_t elems) { return sizeof(double2) * (size_t)((elems + 7) / 8 * 8); }

template <class Kern>
void set_smem(Kern k, size_t bytes) {
  SF_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

FftArgs make_args(const NnfftPlanImpl& p) {
  const FftPlan& f = p.fft;
  FftArgs a{};
  a.P = f.P.p;
  a.Q = f.Q.p;
  a.Bhat = f.Bhat.p;
  a.tw1 = f.tw1.p;
  a.tw2 = f.tw2.p;
  a.tw_lo = f.tw_lo.p;
  a.tw_hi = f.tw_hi.p;
  a.rev2 = f.rev2.p;
  a.K = p.g.K;
  a.L = f.L;
  a.L1 = f.L1;
  a.L2 = f.L2;
  a.Kout = f.Kout;
  a.C_log2 = f.C_log2;
  a.conj_in = f.conj_in ? 1 : 0;
  a.st1 = f.st1;
  a.st2 = f.st2;
  a.st1x = f.st1x;
  a.st2x = f.st2x;
  a.tw1x = f.tw1x.p;
  a.tw2x = f.tw2x.p;
  a.Bhatx = f.Bhatx.p;
  return a;
}

}  // namespace

namespace {

constexpr int kDirectSmem = 4096;   // elements per CTA in step 1 (and step 2 target)
constexpr int kDirectSmem2 = 8192;  // hard cap for one step-2 row (R = 1)

bool is_prime(int64_t n) {
  if (n < 2) return false;
  for (int64_t q = 2; q * q <= n; ++q)
    if (n % q == 0) return false;
  return true;
}

int64_t powmod(int64_t b, int64_t e, int64_t m) {
  int64_t r = 1;
  b %= m;
  while (e) {
    if (e & 1) r = r * b % m;
    b = b * b % m;
    e >>= 1;
  }
  return r;
}

// smallest generator of the multiplicative group mod the prime P
int64_t primitive_root(int64_t P) {
  std::vector<int64_t> fac;
  int64_t m = P - 1;
  for (int64_t q = 2; q * q <= m; ++q)
    if (m % q == 0) {
      fac.push_back(q);
      while (m % q == 0) m /= q;
    }
  if (m > 1) fac.push_back(m);
  for (int64_t g = 2; g < P; ++g) {
    bool ok = true;
    for (int64_t q : fac) ok = ok && powmod(g, (P - 1) / q, P) != 1;
    if (ok) return g;
  }
  fail(3, "internal: no primitive root");
  return 0;
}

static double direct_par_min() {
  static const double v = [] {
    const char* e = getenv("SFB_DIRECT_PARMIN");
    return e ? atof(e) : (double)SFB_DIRECT_PARMIN;
  }();
  return v;
}
// pick N2 = A * P for the direct path; false if no split fits.  best_out is
// the model cost per point (stage costs + ~1 unit per byte of HBM traffic)
bool choose_direct(int64_t N2, DirectFft& d, double* best_out = nullptr) {
  double best = 1e300;
  bool found = false;
  for (int64_t A = 2; A <= 2048 && A <= N2; ++A) {
    if (N2 % A || !smooth7(A)) continue;
    const int64_t P = N2 / A;
    const bool ps = smooth7(P);
    // a prime P with P - 1 smooth takes Rader's cyclic convolution of length
    // P - 1 instead of Bluestein's of length >= 2P - 1
    const bool rader = !ps && P > 2 && is_prime(P) && smooth7(P - 1) && !getenv("SFB_NO_RADER");
    const int64_t LP = ps ? P : rader ? P - 1 : next_smooth(2 * P - 1);
    if (LP > kDirectSmem2) continue;
    int C = 8;
    while (C > 1 && C * A > kDirectSmem) C >>= 1;
    if (C < 2) continue;
    // these sizes are launch/latency bound: a split with few step-2 rows (A)
    // or few step-1 CTAs (P / C) leaves most SMs idle (N2 = 16464 split as
    // 3 x 5488 took 43 us, twice its neighbours)
    const double par = std::min((double)A, (double)P / C);
    const double cst = (stage_cost(A) + (ps ? stage_cost(P)
                                          : 2.0 * stage_cost(LP) * (double)LP / (double)P) +
                        48.0) *
                       (C < 4 ? 1.15 : 1.0) * (par < direct_par_min() ? direct_par_min() / par : 1.0);
    if (cst < best) {
      best = cst, found = true;
      d.A = A, d.P = P, d.LP = LP, d.p_smooth = ps, d.C = C, d.rader = rader;
    }
  }
  if (best_out) *best_out = best;
  return found;
}

int log2i(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}

void build_direct(NnfftPlanImpl& p, cudaStream_t s) {
  DirectFft& d = p.fft.d;
  const Geometry& g = p.g;
  const int n2len = (int)(d.p_smooth ? d.P : d.LP);
  d.R = 1;
  while (2 * d.R * n2len <= kDirectSmem && d.R < 64) d.R *= 2;
  // these lengths are launch/latency bound (N2 ~ 16K at configs 2 and 5):
  // fewer columns/rows per CTA until the grids cover the SMs
  const int64_t want = 2 * (int64_t)p.sp.n_sms;
  while (d.R > 1 && ceil_div(d.A, (int64_t)d.R) < want) d.R >>= 1;
  while (d.C > 2 && ceil_div(d.P, (int64_t)d.C) < want) d.C >>= 1;
  // tuning overrides, clamped to what the kernels' shared memory holds: R rows
  // of n2len in step 2 (and the 64-entry Rader row tables), C columns of A in
  // step 1; both powers of two
  auto pow2_floor = [](int x) { int r = 1; while (2 * r <= x) r *= 2; return r; };
  if (const char* e = getenv("SFB_DIRECT_R"))
    d.R = pow2_floor(std::min(std::max(1, atoi(e)), std::min(64, kDirectSmem2 / n2len)));
  if (const char* e = getenv("SFB_DIRECT_C"))
    d.C = pow2_floor(std::min(std::max(2, atoi(e)), std::max(2, kDirectSmem / (int)d.A)));
  d.C_log2 = log2i(d.C);
  d.R_log2 = log2i(d.R);
  d.stA = make_stages(d.A);
  d.stP = make_stages(n2len);
  launch_stage_twiddles(d.twA, d.stA, s);
  launch_stage_twiddles(d.twP, d.stP, s);
  launch_twiddle(d.w_lo, g.N2, kTwSplit, 1, s);
  launch_twiddle(d.w_hi, g.N2, ceil_div(g.N2, kTwSplit) + 1, kTwSplit, s);
  auto upload = [&](DevArray<int>& dst, const std::vector<int>& v) {
    dst.alloc((int64_t)v.size());
    SF_CUDA(cudaMemcpyAsync(dst.p, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice, s));
    SF_CUDA(cudaStreamSynchronize(s));
  };
  upload(d.revA, digit_reverse(d.stA));
  if (d.p_smooth) upload(d.revP, digit_reverse(d.stP));
  d.D.alloc(g.K);
  k_deconv<<<(unsigned)ceil_div(g.K, 256), 256, 0, s>>>(d.D.p, p.hat2.p, g.K, p.fft.in_scale);
  SF_LAUNCH_CHECK();
  if (d.rader) {
    // Rader: X[g^-q] - y[0] = sum_p y[g^p] W^(g^(p-q)), a cyclic convolution
    // of a_p = y[g^p] with w_m = W^(g^-m), m, p, q < P - 1
    const int64_t g0 = primitive_root(d.P), LR = d.P - 1;
    std::vector<int> rin(LR), rout(LR);
    const int64_t ginv = powmod(g0, d.P - 2, d.P);
    int64_t x = 1, y = 1;
    for (int64_t q = 0; q < LR; ++q, x = x * g0 % d.P, y = y * ginv % d.P) {
      rin[q] = (int)x;
      rout[q] = (int)y;
    }
    upload(d.rin, rin);
    upload(d.rout, rout);
    std::vector<double2> w(LR);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int64_t m = 0; m < LR; ++m) {
      const long double ang = -2.0L * pi * (long double)rout[m] / (long double)d.P;
      w[m] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    DevArray<double2> b(LR);
    SF_CUDA(cudaMemcpyAsync(b.p, w.data(), sizeof(double2) * LR, cudaMemcpyHostToDevice, s));
    d.bhat.alloc(LR);
    FftArgs fa{};
    fa.g = b.p;
    fa.Y = d.bhat.p;
    fa.L = LR;
    fa.st1 = d.stP;
    fa.tw1 = d.twP.p;
    k_single<IN_PLAIN><<<dim3(1, 1), 512, smem_bytes(LR), s>>>(fa, 1);
    SF_LAUNCH_CHECK();
    SF_CUDA(cudaStreamSynchronize(s));
  } else if (!d.p_smooth) {
    d.cp.alloc(d.P);
    k_chirp_p<<<(unsigned)ceil_div(d.P, 256), 256, 0, s>>>(d.cp.p, d.P);
    SF_LAUNCH_CHECK();
    DevArray<double2> b(d.LP);
    k_bluestein_b<<<(unsigned)ceil_div(d.LP, 256), 256, 0, s>>>(b.p, d.cp.p, d.P, d.LP);
    SF_LAUNCH_CHECK();
    d.bhat.alloc(d.LP);
    FftArgs fa{};
    fa.g = b.p;
    fa.Y = d.bhat.p;
    fa.L = d.LP;
    fa.st1 = d.stP;
    fa.tw1 = d.twP.p;
    k_single<IN_PLAIN><<<dim3(1, 1), 512, smem_bytes(d.LP), s>>>(fa, 1);
    SF_LAUNCH_CHECK();
    SF_CUDA(cudaStreamSynchronize(s));
  }
}

DirectArgs make_direct_args(const NnfftPlanImpl& p) {
  const DirectFft& d = p.fft.d;
  DirectArgs a{};
  a.D = d.D.p;
  a.twA = d.twA.p;
  a.twP = d.twP.p;
  a.w_lo = d.w_lo.p;
  a.w_hi = d.w_hi.p;
  a.cp = d.cp.p;
  a.bhat = d.bhat.p;
  a.revA = d.revA.p;
  a.revP = d.revP.p;
  a.K = p.g.K;
  a.N2 = p.g.N2;
  a.A = d.A;
  a.P = d.P;
  a.LP = d.LP;
  a.Kout = p.fft.Kout;
  a.s_lo = p.fft.s_lo;
  a.C_log2 = d.C_log2;
  a.R_log2 = d.R_log2;
  a.p_smooth = d.p_smooth ? 1 : 0;
  a.rader = d.rader ? 1 : 0;
  a.rin = d.rin.p;
  a.rout = d.rout.p;
  a.conj_in = p.fft.conj_in ? 1 : 0;
  a.stA = d.stA;
  a.stP = d.stP;
  return a;
}

}  // namespace

template <int NBL, int T, int MINB>
void set_reg_smem() {
  const size_t sm = sizeof(double2) * ((size_t)512 << NBL);
  set_smem(k_colfwd_rb<512, NBL, T, MINB>, sm);
  set_smem(k_rowmul_rb<512, NBL, T, MINB>, sm);
  set_smem(k_colinv_rb<512, NBL, T, MINB>, sm);
}

void build_fft(NnfftPlanImpl& p, cudaStream_t s) {
  set_smem(k_dstep1, smem_bytes(kDirectSmem));
  set_smem(k_dstep2, smem_bytes(kDirectSmem2));
  // dynamic shared memory limits (per device; the plan's device is current)
  set_smem(k_single<IN_GP>, smem_bytes(kSingleMax));
  set_smem(k_single<IN_PLAIN>, smem_bytes(kSingleMax));
  set_smem(k_colfwd<IN_GP>, smem_bytes(kColElems));
  set_smem(k_colfwd<IN_PLAIN>, smem_bytes(kColElems));
  set_smem(k_rowmul<0>, smem_bytes(kRowMax));
  set_smem(k_colinv<0, 0>, smem_bytes(kColElems));
  set_smem(k_colfwd<IN_GP, 1024, 2>, smem_bytes(kColElems));
  set_smem(k_colinv<1024, 2>, smem_bytes(kColElems));
  set_smem(k_colfwd<IN_GP, 1024, 1>, smem_bytes(kColElems));
  set_smem(k_colinv<1024, 1>, smem_bytes(kColElems));
  set_smem(k_rowmul<4096>, smem_bytes(kRowMax));
  set_smem(k_colfwd_b<0, 0>, smem_bytes(kColElemsB));
  set_smem(k_rowmul_b<0, 0>, smem_bytes(kColElemsB));
  set_smem(k_colinv_b<0, 0>, smem_bytes(kColElemsB));
  set_smem(k_colfwd_b<512, 3>, smem_bytes(kColElemsB));
  set_smem(k_rowmul_b<512, 3>, smem_bytes(kColElemsB));
  set_smem(k_colinv_b<512, 3>, smem_bytes(kColElemsB));
  set_reg_smem<2, 256, 4>();
  set_reg_smem<2, 128, 4>();
  set_smem(k_colfwd_r1<1024, 2, 512, SFB_FFT_CMINB, 8, kColPL>,
           sizeof(double2) * RegFft<1024, 2, 512, 8, kColPL>::SMEM_ELEMS);
  set_smem(k_colinv_r1<1024, 2, 512, SFB_FFT_CMINB, 8, kColPL>,
           sizeof(double2) * RegFft<1024, 2, 512, 8, kColPL>::SMEM_ELEMS);
  set_smem(k_colfwd_r1<1024, 2, 256, 2, 16>, sizeof(double2) * 4096);
  set_smem(k_colinv_r1<1024, 2, 256, 2, 16>, sizeof(double2) * 4096);
  set_smem(k_rowmul_r1<4096, 256, 2>, sizeof(double2) * 4096);
  set_smem(k_drowmul<4096, 256, 2>, sizeof(double2) * 4096);
  set_smem(k_rowmul_r1<4096, 256, 2, 16, kRowPL>,
           sizeof(double2) * RegFft<4096, 0, 256, 16, kRowPL>::SMEM_ELEMS);
  set_smem(k_drowmul<4096, 256, 2, 16>, sizeof(double2) * 4096);
  FftPlan& f = p.fft;
  const Geometry& g = p.g;
  const int64_t Lmin = g.K + f.Kout - 1;
  // direct four-step when it is cheaper than the Bluestein over L (model:
  // stage costs per point + ~1 unit per byte moved; Bluestein moves ~144
  // bytes per point of L, the direct path ~48 per point of N2), and always for
  // launch-bound sizes (2 kernels instead of 3)
  double dcost = 0.0;
  const bool can_direct = Lmin > kSingleMax && !getenv("SFB_NO_DIRECT_FFT") &&
                          choose_direct(g.N2, f.d, &dcost);
  bool use_direct = false;
  if (can_direct) {
    double gbest = 1e300;
    for (int64_t L2 = 2; L2 <= 2048; ++L2) {
      if (!smooth7(L2)) continue;
      const int64_t L1 = next_smooth(ceil_div(Lmin, L2));
      if (L1 > kRowMax || L1 < 2) continue;
      gbest = std::min(gbest, (double)(L1 * L2) / (double)g.N2 *
                                  (2.0 * stage_cost(L1) + 2.0 * stage_cost(L2) + 144.0));
    }
    // (a direct split left with little parallelism competes on cost)
    const bool par_ok = std::min((double)f.d.A, (double)f.d.P / f.d.C) >= direct_par_min() / 2;
    use_direct = (g.N2 <= 65536 && par_ok) || dcost < gbest;
  }
  if (use_direct) {
    f.direct = true;
    f.single = false;
    f.L = f.d.A * f.d.P;
    f.L1 = f.d.A;
    f.L2 = f.d.P;
    build_direct(p, s);
    return;
  }
  if (Lmin <= kSingleMax) {
    f.single = true;
    f.L = next_smooth(Lmin);
    f.L1 = f.L;
    f.L2 = 1;
  } else {
    f.single = false;
    double best = 1e300;
    // L may fall short of K + Kout - 1 by D <= Dmax slots (fixed afterwards
    // by k_bluestein_fix at ~D^2 cost), which admits much smoother lengths
    // (D <= Kout - 1 keeps L >= K: the K inputs themselves must not wrap -- a
    // plan whose targets sit in a few cells has Kout of a few dozen)
    const int64_t Dmax = getenv("SFB_FFT_NO_SHORT_L")
                             ? 0
                             : std::max<int64_t>(
                                   0, std::min<int64_t>({kFixMax, Lmin / 8, f.Kout - 1}));
    for (int64_t L2 = 2; L2 <= 2048; ++L2) {
      if (!smooth7(L2)) continue;
      for (int pass = 0; pass < 2; ++pass) {
        const int64_t L1 = next_smooth(ceil_div(pass ? Lmin - Dmax : Lmin, L2));
        if (L1 > kRowMax || L1 < 2) continue;
        const int64_t D = std::max<int64_t>(0, Lmin - L1 * L2);
        const double c = cost(L1, L2) + (double)D * (double)D;
        if (c < best) best = c, f.L1 = L1, f.L2 = L2;
      }
    }
    if (const char* e = getenv("SFB_FFT_L1L2")) {  // tuning override "L1xL2"
      long long a1 = 0, a2 = 0;
      if (sscanf(e, "%lldx%lld", &a1, &a2) == 2 && a1 * a2 >= Lmin - Dmax && smooth7(a1) &&
          smooth7(a2) && a1 <= kRowMax && a2 <= 2048)
        f.L1 = a1, f.L2 = a2, best = 0;
    }
    if (best >= 1e300)
      fail(5, "FFT length " + std::to_string(Lmin) + " exceeds the supported four-step range");
    f.L = f.L1 * f.L2;
    f.fixD = std::max<int64_t>(0, Lmin - f.L);
    int C = 8;
    while (C > 1 && C * f.L2 > kColElems) C >>= 1;
    f.C = C;
    f.C_log2 = 0;
    while ((1 << f.C_log2) < C) ++f.C_log2;
  }
  f.st1 = make_stages(f.L1);
  f.st2 = make_stages(f.L2);
  launch_stage_twiddles(f.tw1, f.st1, s);
  if (!f.single) {
    launch_stage_twiddles(f.tw2, f.st2, s);
    launch_twiddle(f.tw_lo, f.L, kTwSplit, 1, s);
    launch_twiddle(f.tw_hi, f.L, ceil_div(f.L, kTwSplit) + 1, kTwSplit, s);
    std::vector<int> rev = digit_reverse(f.st2);
    f.rev2.alloc(f.L2);
    SF_CUDA(cudaMemcpyAsync(f.rev2.p, rev.data(), sizeof(int) * rev.size(),
                            cudaMemcpyHostToDevice, s));
    SF_CUDA(cudaStreamSynchronize(s));  // rev is a host temporary
  }
  // chirp tables
  f.P.alloc(g.K);
  f.Q.alloc(f.Kout);
  k_prechirp<<<(unsigned)ceil_div(g.K, 256), 256, 0, s>>>(
      f.P.p, p.hat2.p, g.K, g.N2, f.s_lo, f.in_scale);
  SF_LAUNCH_CHECK();
  k_postchirp<<<(unsigned)ceil_div(f.Kout, 256), 256, 0, s>>>(f.Q.p, f.Kout, g.K, g.N2, f.s_lo);
  SF_LAUNCH_CHECK();
  // Bhat = FFT_L(b) / L in the forward layout
  f.Bhat.alloc(f.L);
  DevArray<double2> b(f.L);
  k_chirp_kernel<<<(unsigned)ceil_div(f.L, 256), 256, 0, s>>>(b.p, f.L, g.K, f.Kout, g.N2);
  SF_LAUNCH_CHECK();
  if (f.fixD > 0) {
    f.fixc.alloc(f.fixD);
    k_fix_table<<<(unsigned)ceil_div(f.fixD, 256), 256, 0, s>>>(f.fixc.p, f.fixD, g.K, f.L, g.N2);
    SF_LAUNCH_CHECK();
  }
  FftArgs a = make_args(p);
  a.g = b.p;
  if (f.single) {
    const size_t sm = smem_bytes(f.L);
    a.Y = f.Bhat.p;
    k_single<IN_PLAIN><<<dim3(1, 1), 512, sm, s>>>(a, 1);
    SF_LAUNCH_CHECK();
  } else {
    const size_t smc = smem_bytes(f.L2 * f.C), smr = smem_bytes(f.L1);
    a.Y = f.Bhat.p;
    k_colfwd<IN_PLAIN><<<dim3((unsigned)ceil_div(f.L1, f.C), 1), 256, smc, s>>>(a);
    SF_LAUNCH_CHECK();
    k_rowmul<0><<<dim3((unsigned)f.L2, 1), 256, smr, s>>>(a, 1);
    SF_LAUNCH_CHECK();
    f.x16 = 0;
    if (f.L1 == 4096 && f.L2 == 1024 && f.st1.n == 4096 && f.st2.n == 1024) {
      // radix-16 register passes (rows; columns too at x16 = 2): their
      // stages, twiddles and B-hat in their output order
      // rows only: 0.188 -> 0.179 ms; radix-16 columns (x16 = 2: 16 double2
      // per thread, 128 registers, 16 warps/SM) measured 0.207 ms
      f.x16 = 1;
      if (const char* e = getenv("SFB_FFT_X16")) f.x16 = std::max(0, std::min(2, atoi(e)));
    }
    if (f.x16 > 0) {
      f.st1x = make_stages16(4096);
      launch_stage_twiddles(f.tw1x, f.st1x, s);
      f.st2x = make_stages16(1024);
      launch_stage_twiddles(f.tw2x, f.st2x, s);
      f.Bhatx.alloc(f.L);
      k_bhat_x16<<<(unsigned)ceil_div(f.L, (int64_t)256), 256, 0, s>>>(f.Bhat.p, f.Bhatx.p, f.L,
                                                                      f.x16 == 2 ? 1 : 0);
      SF_LAUNCH_CHECK();
    }
  }
  SF_CUDA(cudaStreamSynchronize(s));  // b is released at scope exit
}

static void launch_fix(const NnfftPlanImpl& p, const double2* grid, double2* h, int batch,
                       int point_major, cudaStream_t s) {
  const FftPlan& f = p.fft;
  if (f.fixD <= 0) return;
  launch_pdl(k_bluestein_fix, dim3((unsigned)ceil_div(f.fixD * 32, 256), batch), dim3(256), 0, s,
             grid, (const double2*)f.P.p, (const double2*)f.fixc.p, (const double2*)f.Q.p, h,
             p.g.K, f.fixD, f.Kout, f.conj_in ? 1 : 0, batch, point_major);
}

bool fft_supports_point_major(const NnfftPlanImpl& p) {
  return !p.fft.direct && !p.fft.single;
}

// Register-resident passes for this plan's point-major shape (512 x 512,
// config 4): 4 columns x 256 threads, 64 registers, 4 CTAs/SM (the row pass:
// 4 columns x 128 threads x 2 butterflies, see launch_reg_point_major).  Measured
// alternatives: 8 columns x 256 (2 butterflies per thread: spills), 8 x 512,
// 4 x 256 at 3 CTAs/SM -- 1.89-2.75 ms against 1.77 ms; the shared-memory
// kernels k_*_b (SFB_FFT_REG=0) 2.20 ms.
static bool reg_point_major(const FftPlan& f) {
  if (!(f.L1 == 512 && f.L2 == 512 && f.st1.n == 512 && f.st2.n == 512)) return false;
  const char* e = getenv("SFB_FFT_REG");
  return !(e && atoi(e) == 0);
}

template <int NBL, int T, int MINB>
static void launch_reg_point_major_t(const FftBArgs& x, int64_t L1, int64_t L2, cudaStream_t s,
                                     int which) {
  const size_t sm = sizeof(double2) * ((size_t)512 << NBL);
  const dim3 gc((unsigned)ceil_div(x.B, 1 << NBL), (unsigned)L1);  // column groups fastest
  const dim3 gr((unsigned)ceil_div(x.B, 1 << NBL), (unsigned)L2);
  if (which == 0) k_colfwd_rb<512, NBL, T, MINB><<<gc, T, sm, s>>>(x);
  if (which == 1) k_rowmul_rb<512, NBL, T, MINB><<<gr, T, sm, s>>>(x);
  if (which == 2) k_colinv_rb<512, NBL, T, MINB><<<gc, T, sm, s>>>(x);
  SF_LAUNCH_CHECK();
}

static void launch_reg_point_major(const FftBArgs& x, int64_t L1, int64_t L2, cudaStream_t s) {
  // SFB_FFT_RB_T128: bit p set -> pass p (0 colfwd, 1 rowmul, 2 colinv) runs
  // with 128 threads and TWO butterflies per thread (128 registers, 4 CTAs per
  // SM) instead of 256 threads and one.  Measured at config 4: rowmul 616 ->
  // 585 us (the fused forward-multiply-inverse pass has the longest dependent
  // chain per thread and gains from the second butterfly's ILP); colfwd 524 ->
  // 612, colinv 625 -> 967 (spills).  Default: rowmul only.
  static const int t128 = [] {
    const char* e = getenv("SFB_FFT_RB_T128");
    return e ? atoi(e) : 2;
  }();
  for (int w = 0; w < 3; ++w) {
    if (t128 >> w & 1) launch_reg_point_major_t<2, 128, 4>(x, L1, L2, s, w);
    else launch_reg_point_major_t<2, 256, 4>(x, L1, L2, s, w);
  }
}

// Columns can be transformed in groups of G (SFB_FFT_GROUP): the group's work array Y (L x G
// complex) stays L2-resident across the three passes, so only the grid reads
// and the h writes go to DRAM (all 256 columns at once: 3 x 2 x 1.1 GB).
int fft_point_major_group(int batch) {
  int G = 0;  // all columns at once (16-64 column groups measured 7-48 % slower)
  if (const char* e = getenv("SFB_FFT_GROUP")) G = atoi(e);
  if (G <= 0 || G > batch) G = batch;
  return G;
}

void run_fft_point_major(const NnfftPlanImpl& p, const double2* grid, double2* h, double2* work,
                         int batch, cudaStream_t s) {
  const FftPlan& f = p.fft;
  const int G = fft_point_major_group(batch);
  int cc = 8, cr = 8;
  while (cc > 1 && cc * f.L2 > kColElemsB) cc >>= 1;
  while (cr > 1 && cr * f.L1 > kColElemsB) cr >>= 1;
  const size_t smc = smem_bytes(f.L2 * cc), smr = smem_bytes(f.L1 * cr);
  const bool reg = reg_point_major(f);
  for (int b0 = 0; b0 < batch; b0 += G) {
    FftBArgs x{};
    x.a = make_args(p);
    x.a.g = grid + b0;
    x.a.h = h + b0;
    x.a.Y = work;
    x.B = std::min(G, batch - b0);
    x.ldg = batch;
    x.ldy = G;
    x.cb_log2_col = log2i(cc);
    x.cb_log2_row = log2i(cr);
    const dim3 gc((unsigned)f.L1, (unsigned)ceil_div(x.B, cc));
    const dim3 gr((unsigned)f.L2, (unsigned)ceil_div(x.B, cr));
    if (reg) {  // register-resident passes (512 x 512, the config-4 shape)
      launch_reg_point_major(x, f.L1, f.L2, s);
      continue;
    }
    // compile-time specialisation of the config-4 shape (512 x 512, 8 columns)
    const bool ctc = f.L2 == 512 && x.cb_log2_col == 3 && f.st2.n == 512;
    const bool ctr = f.L1 == 512 && x.cb_log2_row == 3 && f.st1.n == 512;
    if (ctc) k_colfwd_b<512, 3><<<gc, 256, smc, s>>>(x);
    else k_colfwd_b<0, 0><<<gc, 256, smc, s>>>(x);
    SF_LAUNCH_CHECK();
    if (ctr) k_rowmul_b<512, 3><<<gr, 256, smr, s>>>(x);
    else k_rowmul_b<0, 0><<<gr, 256, smr, s>>>(x);
    SF_LAUNCH_CHECK();
    if (ctc) k_colinv_b<512, 3><<<gc, 256, smc, s>>>(x);
    else k_colinv_b<0, 0><<<gc, 256, smc, s>>>(x);
    SF_LAUNCH_CHECK();
  }
  launch_fix(p, grid, h, batch, 1, s);
}

// Register-resident single-column passes for the config-3 shape (4096 x
// 1024): columns 4 x 512 threads (2 CTAs/SM), rows 256 threads with 2
// butterflies each.  Measured alternatives (FFT per step): shared-memory
// kernels (SFB_FFT_REG1=0) 0.217 ms; columns 2 x 256 with rows of 512 threads
// 0.214; columns 4 x 512 with rows of 512 0.238; columns 2 x 256 at 3 or 4
// CTAs/SM 0.199 / 0.192; columns 4 x 256 0.219; columns 8 x 1024 0.206; this
// one 0.188 ms.  A persistent cp.async-pipelined version measured 9 % slower.
// radix-16 register passes (plan-time SFB_FFT_X16: 0 off, 1 rows, 2 rows and
// columns): 4096 = 16^3 and 1024 = 16^2 * 4 take 2 shared-memory exchanges per
// transform instead of 3 with radix 8
static bool row16(const FftPlan& f) { return f.x16 >= 1; }
static bool col16(const FftPlan& f) { return f.x16 >= 2; }

static bool reg_single(const FftPlan& f) {
  if (!(f.L1 == 4096 && f.L2 == 1024 && f.st1.n == 4096 && f.st2.n == 1024)) return false;
  const char* e = getenv("SFB_FFT_REG1");
  return !(e && atoi(e) == 0);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    SF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) fail(3, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
// [rows][2 * row_len] float64 (rows of row_len complex), boxes of
// {2 * NB, kTmaBox}; out-of-range rows read as zero
static void encode_rows(CUtensorMap* m, const void* base, int64_t row_len, int64_t rows, int nb) {
  const cuuint64_t dims[2] = {(cuuint64_t)(2 * row_len), (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(2 * row_len * sizeof(double))};
  const cuuint32_t box[2] = {(cuuint32_t)(2 * nb), (cuuint32_t)kTmaBox};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(
      m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(3, "cuTensorMapEncodeTiled failed");
}
#ifndef SFB_FFT_TMA
#define SFB_FFT_TMA 0  // TMA-pipelined persistent forward column pass (padded single column)
#endif
static bool fft_tma_enabled() {
  static const int v = [] {
    const char* e = getenv("SFB_FFT_TMA");
    return e ? atoi(e) : SFB_FFT_TMA;
  }();
  return v != 0;
}

static void launch_reg_single(const FftArgs& a, const FftPlan& f, int batch, cudaStream_t s,
                              bool padded, int n_sms) {
  constexpr int CBL = 2, CT = 512, CMINB = SFB_FFT_CMINB, RT = 256, RMINB = 2;
  const size_t smc = sizeof(double2) * ((size_t)1024 << CBL), smr = sizeof(double2) * 4096;
  const size_t smcp = sizeof(double2) * RegFft<1024, CBL, CT, 8, kColPL>::SMEM_ELEMS;
  const size_t smrp = sizeof(double2) * RegFft<4096, 0, RT, 16, kRowPL>::SMEM_ELEMS;
  const dim3 gc((unsigned)ceil_div(f.L1, (int64_t)1 << CBL), batch);
  // programmatic dependent launches: each pass is scheduled during the
  // previous one's last wave and waits (griddepcontrol.wait) for its output
  if (padded && batch == 1 && !col16(f) && fft_tma_enabled()) {
    TmaMaps tm;
    encode_rows(&tm.in, a.g, f.L1, ceil_div(a.K, f.L1), 1 << CBL);
    encode_rows(&tm.out, a.Y, f.L1, f.L2, 1 << CBL);
    const int ntiles = (int)(f.L1 >> CBL);
    const size_t smt = sizeof(double2) * ((size_t)1024 << CBL) * kTmaStages;
    static bool attr = false;
    if (!attr) {
      SF_CUDA(cudaFuncSetAttribute(k_colfwd_tma<1024, CT>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smt));
      attr = true;
    }
    launch_pdl(k_colfwd_tma<1024, CT>, dim3((unsigned)std::min(ntiles, n_sms)), dim3(CT), smt, s,
               a, tm, ntiles);
  } else if (col16(f)) {
    launch_pdl(k_colfwd_r1<1024, CBL, 256, 2, 16>, gc, dim3(256), smc, s, a);
  } else {
    launch_pdl(k_colfwd_r1<1024, CBL, CT, CMINB, 8, kColPL>, gc, dim3(CT), smcp, s, a);
  }
  const dim3 gr((unsigned)f.L2, batch);
  if (row16(f)) launch_pdl(k_rowmul_r1<4096, RT, RMINB, 16, kRowPL>, gr, dim3(RT), smrp, s, a);
  else launch_pdl(k_rowmul_r1<4096, RT, RMINB>, gr, dim3(RT), smr, s, a);
  if (col16(f)) launch_pdl(k_colinv_r1<1024, CBL, 256, 2, 16>, gc, dim3(256), smc, s, a);
  else launch_pdl(k_colinv_r1<1024, CBL, CT, CMINB, 8, kColPL>, gc, dim3(CT), smcp, s, a);
}

void run_fft(const NnfftPlanImpl& p, const double2* grid, double2* h, double2* work, int batch,
             cudaStream_t s, bool grid_padded) {
  const FftPlan& f = p.fft;
  if (f.direct) {
    DirectArgs a = make_direct_args(p);
    a.g = grid;
    a.Y = work;
    a.h = h;
    const DirectFft& d = f.d;
    k_dstep1<<<dim3((unsigned)ceil_div(d.P, d.C), batch), 256, smem_bytes(d.A * d.C), s>>>(a);
    SF_LAUNCH_CHECK();
    const int64_t n2len = d.p_smooth ? d.P : d.LP;
    k_dstep2<<<dim3((unsigned)ceil_div(d.A, d.R), batch), 256, smem_bytes(n2len * d.R), s>>>(a);
    SF_LAUNCH_CHECK();
    return;
  }
  FftArgs a = make_args(p);
  a.g = grid;
  a.h = h;
  a.Y = work;
  if (f.single) {
    const size_t sm = smem_bytes(f.L);
    k_single<IN_GP><<<dim3(1, batch), 512, sm, s>>>(a, 0);
    SF_LAUNCH_CHECK();
    return;
  }
  if (reg_single(f)) {
    grid_padded = grid_padded && batch == 1 && !col16(f) && fft_tma_enabled();
    if (grid_padded)  // zero the row padding the TMA path reads past K
      SF_CUDA(cudaMemsetAsync(const_cast<double2*>(grid) + p.g.K, 0,
                              sizeof(double2) * (size_t)(ceil_div(p.g.K, f.L1) * f.L1 - p.g.K), s));
    launch_reg_single(a, f, batch, s, grid_padded, p.sp.n_sms);
    launch_fix(p, grid, h, batch, 0, s);
    return;
  }
  const size_t smc = smem_bytes(f.L2 * f.C), smr = smem_bytes(f.L1);
  const dim3 gc((unsigned)ceil_div(f.L1, f.C), batch);
  // compile-time specialisations of the shapes in use (config 3: 4096 x 1024)
  const bool ct_col = f.L2 == 1024 && f.C_log2 == 2 && f.st2.n == 1024;
  const bool ct_col1 = f.L2 == 1024 && f.C_log2 == 1 && f.st2.n == 1024;
  const bool ct_row = f.L1 == 4096 && f.st1.n == 4096;
  if (ct_col) k_colfwd<IN_GP, 1024, 2><<<gc, 256, smc, s>>>(a);
  else if (ct_col1) k_colfwd<IN_GP, 1024, 1><<<gc, 256, smc, s>>>(a);
  else k_colfwd<IN_GP><<<gc, 256, smc, s>>>(a);
  SF_LAUNCH_CHECK();
  if (ct_row) k_rowmul<4096><<<dim3((unsigned)f.L2, batch), 256, smr, s>>>(a, 0);
  else k_rowmul<0><<<dim3((unsigned)f.L2, batch), 256, smr, s>>>(a, 0);
  SF_LAUNCH_CHECK();
  if (ct_col) k_colinv<1024, 2><<<gc, 256, smc, s>>>(a);
  else if (ct_col1) k_colinv<1024, 1><<<gc, 256, smc, s>>>(a);
  else k_colinv<0, 0><<<gc, 256, smc, s>>>(a);
  SF_LAUNCH_CHECK();
  launch_fix(p, grid, h, batch, 0, s);
}


// ---------------------------------------------------- distributed FFT (host)
static bool dist_shape(const FftPlan& f) {
  return !f.direct && !f.single && !f.conj_in && f.L1 == 4096 && f.L2 == 1024 &&
         f.st1.n == 4096 && f.st2.n == 1024;
}

bool dist_layout(const NnfftPlanImpl& p, int world, DistLayout* out) {
  const FftPlan& f = p.fft;
  DistLayout d{};
  d.ok = false;
  if (world >= 1 && (world & (world - 1)) == 0 && dist_shape(f) && f.L1 % world == 0 &&
      f.L2 % world == 0 && f.L1 / world >= 2 && f.fixD <= f.L1 / world) {
    d.Bc = f.L1 / world;
    d.Br = f.L2 / world;
    d.I = ceil_div(p.g.K, f.L1);
    d.K2 = ceil_div(f.Kout, f.L1);
    d.Sb = d.I * d.Bc + (f.fixD + 7) / 8 * 8;
    d.ok = true;
  }
  *out = d;
  return d.ok;
}

static DistArgs dist_args(const NnfftPlanImpl& p, int world, int rank) {
  DistLayout l;
  if (!dist_layout(p, world, &l)) fail(1, "distributed FFT: unsupported plan shape or world size");
  if (rank < 0 || rank >= world) fail(1, "distributed FFT: rank out of range");
  DistArgs d{};
  d.a = make_args(p);
  d.rank = rank;
  d.world = world;
  d.Bc = l.Bc;
  d.Br = l.Br;
  d.I = l.I;
  d.K2 = l.K2;
  d.Sb = l.Sb;
  d.bc_log2 = log2i((int)l.Bc);
  d.br_log2 = log2i((int)l.Br);
  d.use_peers = 0;
  d.fixp = nullptr;
  d.fixD = p.fft.fixD;
  return d;
}

void run_dist_pack(const NnfftPlanImpl& p, int world, const double2* grid, double2* S,
                   cudaStream_t s) {
  const DistArgs d = dist_args(p, world, 0);
  const int64_t n = (int64_t)world * d.Sb;
  k_dpack<<<(unsigned)ceil_div(n, (int64_t)256), 256, 0, s>>>(grid, S, d);
  SF_LAUNCH_CHECK();
  const FftPlan& f = p.fft;
  if (f.fixD > 0) {  // this rank's share of the tail fix, into rank 0's block
    k_bluestein_fix<<<dim3((unsigned)ceil_div(f.fixD * 32, 256), 1), 256, 0, s>>>(
        grid, f.P.p, f.fixc.p, f.Q.p, S + d.I * d.Bc, p.g.K, f.fixD, f.Kout, 0, 1, 0);
    SF_LAUNCH_CHECK();
  }
}

void run_dist_colfwd(const NnfftPlanImpl& p, int world, int rank, const double2* R, double2* Yc,
                     cudaStream_t s) {
  const DistArgs d = dist_args(p, world, rank);
  if (col16(p.fft))
    k_dcolfwd<1024, 1, 128, 4, 16><<<(unsigned)(d.Bc / 2), 128, sizeof(double2) * 2048, s>>>(d, R, Yc);
  else
    k_dcolfwd<1024, 1, 256, 4><<<(unsigned)(d.Bc / 2), 256, sizeof(double2) * 2048, s>>>(d, R, Yc);
  SF_LAUNCH_CHECK();
}

void run_dist_rowmul(const NnfftPlanImpl& p, int world, int rank, double2* Rr, cudaStream_t s) {
  const DistArgs d = dist_args(p, world, rank);
  if (row16(p.fft)) k_drowmul<4096, 256, 2, 16><<<(unsigned)d.Br, 256, sizeof(double2) * 4096, s>>>(d, Rr);
  else k_drowmul<4096, 256, 2><<<(unsigned)d.Br, 256, sizeof(double2) * 4096, s>>>(d, Rr);
  SF_LAUNCH_CHECK();
}

void run_dist_colinv(const NnfftPlanImpl& p, int world, int rank, const double2* Y2,
                     const double2* R, double2* H, cudaStream_t s) {
  const DistArgs d = dist_args(p, world, rank);
  if (col16(p.fft))
    k_dcolinv<1024, 1, 128, 4, 16><<<(unsigned)(d.Bc / 2), 128, sizeof(double2) * 2048, s>>>(d, Y2, H);
  else
    k_dcolinv<1024, 1, 256, 4><<<(unsigned)(d.Bc / 2), 256, sizeof(double2) * 2048, s>>>(d, Y2, H);
  SF_LAUNCH_CHECK();
  if (rank == 0 && p.fft.fixD > 0) {
    k_dfix_add<<<(unsigned)ceil_div(p.fft.fixD, (int64_t)256), 256, 0, s>>>(H, R + d.I * d.Bc,
                                                                          p.fft.fixD);
    SF_LAUNCH_CHECK();
  }
}

void run_dist_unpack(const NnfftPlanImpl& p, int world, const double2* Hall, double2* h,
                     cudaStream_t s) {
  const DistArgs d = dist_args(p, world, 0);
  k_dunpack<<<(unsigned)ceil_div(p.fft.Kout, (int64_t)256), 256, 0, s>>>(Hall, h, d);
  SF_LAUNCH_CHECK();
}


static int64_t dist_dpad(const NnfftPlanImpl& p) { return (p.fft.fixD + 7) / 8 * 8; }

void run_dist_pack_rows(const NnfftPlanImpl& p, int world, const double2* grid, int64_t ilo,
                        int64_t nrow, double2* send, cudaStream_t s) {
  const DistArgs d = dist_args(p, world, 0);
  if (world > kDistMaxRanks) fail(1, "sparse exchange: at most 16 ranks");
  const int64_t dpad = dist_dpad(p);
  const int64_t total = world * nrow * d.Bc + dpad;
  k_dpack_rows<<<(unsigned)ceil_div(total, (int64_t)256), 256, 0, s>>>(grid, send, d, ilo, nrow,
                                                                    dpad);
  SF_LAUNCH_CHECK();
  const FftPlan& f = p.fft;
  if (f.fixD > 0) {
    k_bluestein_fix<<<dim3((unsigned)ceil_div(f.fixD * 32, 256), 1), 256, 0, s>>>(
        grid, f.P.p, f.fixc.p, f.Q.p, send + nrow * d.Bc, p.g.K, f.fixD, f.Kout, 0, 1, 0);
    SF_LAUNCH_CHECK();
  }
}

void run_dist_unpack_rows(const NnfftPlanImpl& p, int world, int rank, const double2* recv,
                          const int64_t* ilo, const int64_t* nrow, double2* block,
                          cudaStream_t s) {
  const DistArgs d = dist_args(p, world, rank);
  if (world > kDistMaxRanks) fail(1, "sparse exchange: at most 16 ranks");
  RowSplit rs{};
  rs.n = world;
  const int64_t extra = rank == 0 ? dist_dpad(p) : 0;
  int64_t off = 0;
  for (int q = 0; q < world; ++q) {
    rs.lo[q] = ilo[q];
    rs.cnt[q] = nrow[q];
    rs.off[q] = off;
    off += nrow[q] * d.Bc + extra;
  }
  const int64_t dfix = rank == 0 ? p.fft.fixD : 0;
  const int64_t n = d.I * d.Bc + dfix;
  k_dunpack_rows<<<(unsigned)ceil_div(n, (int64_t)256), 256, 0, s>>>(recv, block, d, rs, dfix);
  SF_LAUNCH_CHECK();
}

void run_dist_pack_hrows(const NnfftPlanImpl& p, int world, const double2* hblk,
                         const int64_t* k2lo, const int64_t* cnt, double2* send, cudaStream_t s) {
  const DistArgs d = dist_args(p, world, 0);
  if (world > kDistMaxRanks) fail(1, "sparse exchange: at most 16 ranks");
  RowSplit rs{};
  rs.n = world;
  int64_t off = 0;
  for (int r = 0; r < world; ++r) {
    rs.lo[r] = k2lo[r];
    rs.cnt[r] = cnt[r];
    rs.off[r] = off;
    off += cnt[r] * d.Bc;
  }
  k_dpack_hrows<<<(unsigned)ceil_div(off, (int64_t)256), 256, 0, s>>>(hblk, send, d, rs, off);
  SF_LAUNCH_CHECK();
}

void run_dist_unpack_hrows(const NnfftPlanImpl& p, int world, const double2* recv, int64_t k2lo,
                           int64_t cnt, double2* h, cudaStream_t s) {
  const DistArgs d = dist_args(p, world, 0);
  const int64_t n = world * cnt * d.Bc;
  k_dunpack_hrows<<<(unsigned)ceil_div(n, (int64_t)256), 256, 0, s>>>(recv, h, d, k2lo, cnt);
  SF_LAUNCH_CHECK();
}


void run_dist_colfwd_peer(const NnfftPlanImpl& p, int world, int rank, const double2* R,
                          double2* const* peers, cudaStream_t s) {
  DistArgs d = dist_args(p, world, rank);
  if (world > kDistMaxRanks) fail(1, "peer transposes: at most 16 ranks");
  d.use_peers = 1;
  for (int q = 0; q < world; ++q) d.peer[q] = peers[q];
  if (col16(p.fft))
    k_dcolfwd<1024, 1, 128, 4, 16><<<(unsigned)(d.Bc / 2), 128, sizeof(double2) * 2048, s>>>(d, R, nullptr);
  else
    k_dcolfwd<1024, 1, 256, 4><<<(unsigned)(d.Bc / 2), 256, sizeof(double2) * 2048, s>>>(d, R, nullptr);
  SF_LAUNCH_CHECK();
}

void run_dist_rowmul_peer(const NnfftPlanImpl& p, int world, int rank, double2* Rr,
                          double2* const* peers, cudaStream_t s) {
  DistArgs d = dist_args(p, world, rank);
  if (world > kDistMaxRanks) fail(1, "peer transposes: at most 16 ranks");
  d.use_peers = 1;
  for (int q = 0; q < world; ++q) d.peer[q] = peers[q];
  if (row16(p.fft)) k_drowmul<4096, 256, 2, 16><<<(unsigned)d.Br, 256, sizeof(double2) * 4096, s>>>(d, Rr);
  else k_drowmul<4096, 256, 2><<<(unsigned)d.Br, 256, sizeof(double2) * 4096, s>>>(d, Rr);
  SF_LAUNCH_CHECK();
}


void run_dist_pack_rows_peer(const NnfftPlanImpl& p, int world, int rank, const double2* grid,
                             int64_t ilo, int64_t nrow, double2* const* peers,
                             const int64_t* poff, cudaStream_t s) {
  DistArgs d = dist_args(p, world, rank);
  if (world > kDistMaxRanks) fail(1, "peer exchange: at most 16 ranks");
  d.use_peers = 1;
  for (int q = 0; q < world; ++q) d.peer[q] = peers[q], d.poff[q] = poff[q];
  const int64_t dpad = dist_dpad(p);
  const int64_t total = world * nrow * d.Bc + dpad;
  k_dpack_rows<<<(unsigned)ceil_div(total, (int64_t)256), 256, 0, s>>>(grid, nullptr, d, ilo,
                                                                    nrow, dpad);
  SF_LAUNCH_CHECK();
  const FftPlan& f = p.fft;
  if (f.fixD > 0) {  // this rank's tail-fix partial, into rank 0's buffer after its rows
    k_bluestein_fix<<<dim3((unsigned)ceil_div(f.fixD * 32, 256), 1), 256, 0, s>>>(
        grid, f.P.p, f.fixc.p, f.Q.p, peers[0] + poff[0] + nrow * d.Bc, p.g.K, f.fixD, f.Kout, 0,
        1, 0);
    SF_LAUNCH_CHECK();
  }
}

void run_dist_colinv_peer(const NnfftPlanImpl& p, int world, int rank, const double2* Y2,
                          const double2* R, double2* const* peers, const int64_t* k2lo,
                          const int64_t* cnt, cudaStream_t s) {
  DistArgs d = dist_args(p, world, rank);
  if (world > kDistMaxRanks) fail(1, "peer exchange: at most 16 ranks");
  d.use_peers = 1;
  for (int q = 0; q < world; ++q) d.peer[q] = peers[q], d.hlo[q] = k2lo[q], d.hcnt[q] = cnt[q];
  d.fixp = (rank == 0 && p.fft.fixD > 0) ? R + d.I * d.Bc : nullptr;
  if (col16(p.fft))
    k_dcolinv<1024, 1, 128, 4, 16><<<(unsigned)(d.Bc / 2), 128, sizeof(double2) * 2048, s>>>(d, Y2, nullptr);
  else
    k_dcolinv<1024, 1, 256, 4><<<(unsigned)(d.Bc / 2), 256, sizeof(double2) * 2048, s>>>(d, Y2, nullptr);
  SF_LAUNCH_CHECK();
}

}  // namespace sfb
