// fft.cuh -- fp64 complex FFT building blocks in shared memory (sm_100a).
//
// Step 3 of Algorithm 2.1 is one forward DFT of length N2 (ref:
// pkg/src/sincfft/nnfft.py:239 -> fft_core.py:24-25, scipy/pocketfft).  N2 is
// dictated by the reference's geometry and is never a power of two (its
// factors include the primes 11, 19, 41, 79, 257, 2341, 65537),
// and parity needs that exact N2.  Only K = N1 + 2 m1 inputs are nonzero and
// the gather reads only the Kout ~ N2/sigma1 outputs around s = 0, so the
// DFT is realised as a PRUNED Bluestein chirp-z transform over a 7-smooth
// length L >= K + Kout - 1 ~ N2 (fft.cu), whose two FFTs of length L are
// built from the in-place mixed-radix (2,3,4,5,7,8,16) routines below.
//
// Layout conventions
//   * a transform of length n in shared memory occupies elements e in
//     [0, n*nb): element i of batch b is e = i*nb + b (nb interleaved
//     transforms, b fastest so consecutive lanes touch consecutive words);
//   * physical slot spad(e) permutes slots within aligned groups of 8 (XOR
//     swizzle) to break the power-of-two strides of the late stages;
//   * DIF maps natural order -> digit-reversed order, DIT maps digit-reversed
//     order -> natural order, both in place and with forward sign
//     exp(-2 pi i/n); inverse transforms use conj(FFT(conj(x))).
#pragma once

#include "common.cuh"
#include "fft_consts.cuh"

namespace sfb {

// largest butterfly radix (16: fewer shared-memory passes; 8: fewer registers,
// measured faster: 3 resident CTAs/SM beat one fewer smem pass --
// more resident CTAs) and the matching minimum CTAs/SM for __launch_bounds__
#ifndef SFB_FFT_MAXR
#define SFB_FFT_MAXR 8
#endif
#if SFB_FFT_MAXR >= 16
#define SFB_FFT_MINB 2
#else
#define SFB_FFT_MINB 3
#endif

constexpr int kMaxStages = 24;

struct FftStages {
  int n;
  int nst;
  int rad[kMaxStages];   // DIF order; product == n
  int toff[kMaxStages];  // offset of stage q's twiddles W_n^{j*G_q}, j < S_q, in the table
};

// XOR swizzle within each aligned group of 8 16-byte slots: maps the strided
// butterfly accesses of every stage shape used here to distinct bank groups
// within a quarter-warp (simulated: 1.0x for radix-16 rows, <= 1.33x for the
// odd-radix column stages; plain +1-per-8 padding gave 2x on radix-16 S=1)
__device__ __forceinline__ int spad(int e) { return e ^ (((e >> 3) ^ (e >> 6)) & 7); }

// ------------------------------------------------------------ radix kernels
template <int R>
struct Dft;

template <>
struct Dft<2> {
  static __device__ __forceinline__ void run(double2* x) {
    const double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  }
};

template <>
struct Dft<4> {
  static __device__ __forceinline__ void run(double2* x) {
    const double2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
    const double2 t2 = cadd(x[1], x[3]), t3 = cmul_mi(csub(x[1], x[3]));
    x[0] = cadd(t0, t2);
    x[2] = csub(t0, t2);
    x[1] = cadd(t1, t3);
    x[3] = csub(t1, t3);
  }
};

template <>
struct Dft<8> {
  static __device__ __forceinline__ void run(double2* x) {
    const double h = 0.70710678118654752440;  // sqrt(1/2)
    double2 a[4], b[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      a[r] = cadd(x[r], x[r + 4]);
      b[r] = csub(x[r], x[r + 4]);
    }
    // b_r *= W8^r : W8 = (1 - i)/sqrt2, W8^2 = -i, W8^3 = -(1 + i)/sqrt2
    b[1] = make_double2(h * (b[1].x + b[1].y), h * (b[1].y - b[1].x));
    b[2] = cmul_mi(b[2]);
    b[3] = make_double2(h * (b[3].y - b[3].x), -h * (b[3].x + b[3].y));
    Dft<4>::run(a);
    Dft<4>::run(b);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      x[2 * r] = a[r];
      x[2 * r + 1] = b[r];
    }
  }
};

// 16 = 4 x 4: X[k1 + 4 k2] = DFT4_{n2}( W16^{n2 k1} DFT4_{n1}(x[4 n1 + n2]) )
template <>
struct Dft<16> {
  static __device__ __forceinline__ void run(double2* x) {
    const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;  // cos, sin(pi/8)
    const double h = 0.70710678118654752440;
    double2 y[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
      double2 t[4] = {x[n2], x[4 + n2], x[8 + n2], x[12 + n2]};
      Dft<4>::run(t);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) y[n2][k1] = t[k1];
    }
    // W16^e = exp(-2 pi i e / 16) for e = n2*k1 in {1,2,3,4,6,9}
    y[1][1] = cmul(y[1][1], make_double2(c1, -s1));
    y[1][2] = cmul(y[1][2], make_double2(h, -h));
    y[1][3] = cmul(y[1][3], make_double2(s1, -c1));
    y[2][1] = cmul(y[2][1], make_double2(h, -h));
    y[2][2] = cmul_mi(y[2][2]);
    y[2][3] = cmul(y[2][3], make_double2(-h, -h));
    y[3][1] = cmul(y[3][1], make_double2(s1, -c1));
    y[3][2] = cmul(y[3][2], make_double2(-h, -h));
    y[3][3] = cmul(y[3][3], make_double2(-c1, s1));
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      double2 t[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
      Dft<4>::run(t);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) x[k1 + 4 * k2] = t[k2];
    }
  }
};

// generic odd radix via the symmetric real-pair formulation
template <int R>
struct DftOdd {
  static __device__ __forceinline__ void run(double2* x) {
    constexpr int H = (R - 1) / 2;
    double2 s[H + 1], d[H + 1];
    double2 x0 = x[0];
    double2 sum = x0;
#pragma unroll
    for (int r = 1; r <= H; ++r) {
      s[r] = cadd(x[r], x[R - r]);
      d[r] = csub(x[r], x[R - r]);
      sum = cadd(sum, s[r]);
    }
    double2 out[R];
    out[0] = sum;
#pragma unroll
    for (int k = 1; k <= H; ++k) {
      double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 1; r <= H; ++r) {
        const double c = RadixConst<R>::c((r * k) % R);
        const double sn = RadixConst<R>::s((r * k) % R);
        A.x = fma(s[r].x, c, A.x);
        A.y = fma(s[r].y, c, A.y);
        B.x = fma(d[r].x, sn, B.x);
        B.y = fma(d[r].y, sn, B.y);
      }
      // X_k = A - i B, X_{R-k} = A + i B
      out[k] = make_double2(A.x + B.y, A.y - B.x);
      out[R - k] = make_double2(A.x - B.y, A.y + B.x);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = out[r];
  }
};
template <>
struct Dft<3> : DftOdd<3> {};
template <>
struct Dft<5> : DftOdd<5> {};
template <>
struct Dft<7> : DftOdd<7> {};

// -------------------------------------------------------------- one stage
// DIF stage (natural -> reversed): twiddle after the butterfly.
// DIT stage (reversed -> natural): twiddle before the butterfly.
// Butterfly q = g*S + j touches elements g*R*S + j + r*S, r < R; its twiddle
// for leg r is W_n^{r*j*G} with G = n/(R*S).  One load per butterfly from a
// compact per-stage table (w = W_n^{j*G} at tw[j]; all stages of an n-point
// FFT need only ~n/15 distinct values, so the table stays L1-resident); leg r
// uses w^r formed by a multiply tree (<= 4 roundings, ~1e-15 relative -- far
// inside the 1e-12 parity budget).
// x[r] *= w^r, r = 1..R-1, with powers formed as a tree (dependency depth
// <= 4 complex multiplies instead of a 15-deep running product)
template <int R>
__device__ __forceinline__ void apply_twiddles(double2* x, double2 w) {
  if (R == 2) {
    x[1] = cmul(x[1], w);
    return;
  }
  const double2 w2 = cmul(w, w);
  x[1] = cmul(x[1], w);
  x[2] = cmul(x[2], w2);
  if (R == 3) return;
  const double2 w3 = cmul(w2, w);
  x[3] = cmul(x[3], w3);
  if (R == 4) return;
  const double2 w4 = cmul(w2, w2);
  x[4] = cmul(x[4], w4);
  if (R == 5) return;
  x[5] = cmul(x[5], cmul(w4, w));
  x[6] = cmul(x[6], cmul(w4, w2));
  if (R == 7) return;
  x[7] = cmul(x[7], cmul(w4, w3));
  if (R == 8) return;
  const double2 w8 = cmul(w4, w4);
  x[8] = cmul(x[8], w8);
  x[9] = cmul(x[9], cmul(w8, w));
  x[10] = cmul(x[10], cmul(w8, w2));
  x[11] = cmul(x[11], cmul(w8, w3));
  const double2 w12 = cmul(w8, w4);
  x[12] = cmul(x[12], w12);
  x[13] = cmul(x[13], cmul(w12, w));
  x[14] = cmul(x[14], cmul(w12, w2));
  x[15] = cmul(x[15], cmul(w12, w3));
}

template <int R, bool DIT>
__device__ __forceinline__ void fft_stage(double2* s, int nb_log2, int S, int G,
                                          const double2* __restrict__ tw, int tid, int nthr) {
  const int nb = 1 << nb_log2;
  const int nbf = (G * S) << nb_log2;
  if (tid >= nbf) return;
  // nthr is a multiple of nb, so the batch lane b is fixed per thread and the
  // butterfly index q advances by dq = nthr/nb: update (g, j) incrementally
  const int b = tid & (nb - 1);
  int q = tid >> nb_log2;
  const int dq = nthr >> nb_log2;
  int g = q / S;
  int j = q - g * S;
  const int dg = dq / S, dj = dq - dg * S;
  for (; q < (nbf >> nb_log2); q += dq) {
    const int base = g * R * S + j;
    double2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = s[spad(((base + r * S) << nb_log2) + b)];
    const bool twid = j != 0;
    double2 w1 = make_double2(1.0, 0.0);
    if (twid) w1 = __ldg(tw + j);
    if (DIT && twid) apply_twiddles<R>(x, w1);
    Dft<R>::run(x);
    if (!DIT && twid) apply_twiddles<R>(x, w1);
#pragma unroll
    for (int r = 0; r < R; ++r) s[spad(((base + r * S) << nb_log2) + b)] = x[r];
    j += dj;
    g += dg;
    if (j >= S) {
      j -= S;
      ++g;
    }
  }
}

template <bool DIT>
__device__ __forceinline__ void fft_stage_dispatch(int R, double2* s, int nb_log2, int S, int G,
                                                   const double2* __restrict__ tw, int tid,
                                                   int nthr) {
  switch (R) {
    case 2: fft_stage<2, DIT>(s, nb_log2, S, G, tw, tid, nthr); break;
    case 3: fft_stage<3, DIT>(s, nb_log2, S, G, tw, tid, nthr); break;
    case 4: fft_stage<4, DIT>(s, nb_log2, S, G, tw, tid, nthr); break;
    case 5: fft_stage<5, DIT>(s, nb_log2, S, G, tw, tid, nthr); break;
    case 7: fft_stage<7, DIT>(s, nb_log2, S, G, tw, tid, nthr); break;
    case 8: fft_stage<8, DIT>(s, nb_log2, S, G, tw, tid, nthr); break;
#if SFB_FFT_MAXR >= 16
    case 16: fft_stage<16, DIT>(s, nb_log2, S, G, tw, tid, nthr); break;
#endif
    default: break;
  }
}

// Full in-place transforms of nb interleaved length-n vectors in smem.
// Caller must __syncthreads() before (data loaded); these end synchronized.
__device__ __forceinline__ void fft_dif(double2* s, int nb_log2, const FftStages& st,
                                        const double2* __restrict__ tw) {
  int G = 1, S = st.n;
  for (int q = 0; q < st.nst; ++q) {
    const int R = st.rad[q];
    S /= R;
    fft_stage_dispatch<false>(R, s, nb_log2, S, G, tw + st.toff[q], threadIdx.x, blockDim.x);
    __syncthreads();
    G *= R;
  }
}

__device__ __forceinline__ void fft_dit(double2* s, int nb_log2, const FftStages& st,
                                        const double2* __restrict__ tw) {
  int S = 1, G = st.n;
  for (int q = st.nst - 1; q >= 0; --q) {
    const int R = st.rad[q];
    G /= R;
    fft_stage_dispatch<true>(R, s, nb_log2, S, G, tw + st.toff[q], threadIdx.x, blockDim.x);
    __syncthreads();
    S *= R;
  }
}

// ------------------------------------------- compile-time specialisations
// The same stages with n, the batch width NB = 2^NBL and the thread count
// known at compile time (power-of-two n, radix 8 then 4 or 2, exactly the
// decomposition make_stages() produces): every index, the butterfly loop and
// -- for strides that are multiples of 512 slots, where the XOR swizzle
// reduces to an offset -- the swizzled addresses fold into constants.
__host__ __device__ constexpr int ct_nst(int n) {
  int k = 0;
  while (n % 8 == 0) n /= 8, ++k;
  if (n % 4 == 0) n /= 4, ++k;
  if (n % 2 == 0) n /= 2, ++k;
  return n == 1 ? k : -1;
}
__host__ __device__ constexpr int ct_rad(int n, int q) {
  int k = 0;
  while (n % 8 == 0) {
    if (k == q) return 8;
    n /= 8, ++k;
  }
  if (n % 4 == 0) {
    if (k == q) return 4;
    n /= 4, ++k;
  }
  if (n % 2 == 0 && k == q) return 2;
  return 0;
}
__host__ __device__ constexpr int ct_prod(int n, int a, int b) {  // rad[a..b)
  int p = 1;
  for (int q = a; q < b; ++q) p *= ct_rad(n, q);
  return p;
}

template <int R, bool DIT, int S, int G, int NBL, int NTHR>
__device__ __forceinline__ void fft_stage_ct(double2* s, const double2* __restrict__ tw,
                                             int tid) {
  constexpr int NB = 1 << NBL;
  constexpr int NQ = G * S;        // butterflies per vector
  constexpr int DQ = NTHR >> NBL;  // butterflies a thread advances by
  constexpr int STRIDE = S << NBL; // slot distance between legs
  const int b = tid & (NB - 1);
  const int q0 = tid >> NBL;
#pragma unroll
  for (int it = 0; it < (NQ + DQ - 1) / DQ; ++it) {
    const int q = q0 + it * DQ;
    if ((NQ % DQ) != 0 && q >= NQ) break;
    const int g = q / S, j = q % S;
    const int e0 = (((g * R * S) + j) << NBL) + b;
    double2 x[R];
    if constexpr (STRIDE % 512 == 0) {
      const int p0 = spad(e0);
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = s[p0 + r * STRIDE];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = s[spad(e0 + r * STRIDE)];
    }
    const bool twid = j != 0;
    double2 w1 = make_double2(1.0, 0.0);
    if (twid) w1 = __ldg(tw + j);
    if (DIT && twid) apply_twiddles<R>(x, w1);
    Dft<R>::run(x);
    if (!DIT && twid) apply_twiddles<R>(x, w1);
    if constexpr (STRIDE % 512 == 0) {
      const int p0 = spad(e0);
#pragma unroll
      for (int r = 0; r < R; ++r) s[p0 + r * STRIDE] = x[r];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) s[spad(e0 + r * STRIDE)] = x[r];
    }
  }
}

template <int N, int NBL, int NTHR, bool DIT, int Q>
__device__ __forceinline__ void fft_ct_from(double2* s, const FftStages& st,
                                            const double2* __restrict__ tw) {
  constexpr int NST = ct_nst(N);
  static_assert(NST > 0, "compile-time FFT needs a power-of-two length");
  if constexpr (Q >= 0 && Q < NST) {
    constexpr int R = ct_rad(N, Q);
    constexpr int S = ct_prod(N, Q + 1, NST);
    constexpr int G = ct_prod(N, 0, Q);
    fft_stage_ct<R, DIT, S, G, NBL, NTHR>(s, tw + st.toff[Q], threadIdx.x);
    __syncthreads();
    fft_ct_from<N, NBL, NTHR, DIT, DIT ? Q - 1 : Q + 1>(s, st, tw);
  }
}

template <int N, int NBL, int NTHR>
__device__ __forceinline__ void fft_dif_ct(double2* s, const FftStages& st,
                                           const double2* __restrict__ tw) {
  fft_ct_from<N, NBL, NTHR, false, 0>(s, st, tw);
}

template <int N, int NBL, int NTHR>
__device__ __forceinline__ void fft_dit_ct(double2* s, const FftStages& st,
                                           const double2* __restrict__ tw) {
  fft_ct_from<N, NBL, NTHR, true, ct_nst(N) - 1>(s, st, tw);
}

}  // namespace sfb
