// fft_reg.cuh -- register-resident radix-8 FFT stages (sm_100a, fp64).
//
// The shared-memory routines of fft.cuh make every stage a shared-memory
// round trip (load R legs, butterfly, store R legs) plus one more round trip
// for each global load and store: 8 x 16 bytes of shared-memory traffic per
// element for a 512-point transform, 16 x 16 for the fused forward-multiply-
// inverse row pass.  At fp64 complex (8 elements per SM clock) that traffic,
// not the arithmetic or HBM, bounded the batched config-4 FFT.
//
// Here each thread owns BPT radix-8 butterflies (8 elements each) in
// registers for a whole transform: stage 0 is fed straight from global
// memory, the last stage stores straight to global memory, and consecutive
// stages exchange through shared memory once (write own outputs, barrier,
// read own next inputs: 2 x 16 bytes per element per exchange).  The fused
// row pass keeps the last DIF stage and the first DIT stage (both stride 1,
// same thread, same 8 positions) in registers with the B-hat multiply between
// them.  Length N = 8^a * R0 with R0 in {1, 2, 4} (config 4: 512 x 512,
// config 3: 4096 x 1024), NB = 2^NBL interleaved vectors per CTA, T threads.
//
// Position conventions are exactly those of fft_stage<8, DIT> (fft.cuh):
// butterfly u of a stage with stride S = N / 8^(q+1) has legs
// g*8S + j + r*S (u = g*S + j), DIF applies W^{r j G} after the DFT, DIT
// before it, both from the same compact per-stage table tw + st.toff[q]; the
// smem slot of (position i, vector b) is spad(i * NB + b).  So the outputs
// (digit-reversed after DIF) are bit-identical in layout to the smem kernels'.
#pragma once

#include "fft.cuh"

namespace sfb {

__host__ __device__ constexpr int ilog8(int n) { return n < 8 ? 0 : 1 + ilog8(n / 8); }
__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int ilogr(int n, int r) { return n < r ? 0 : 1 + ilogr(n / r, r); }

// N = R^a * R0 with the main radix R in {8, 16} and R0 in {1, 2, 4, 8} (< R):
// a radix-R stages first, then one radix-R0 stage of stride 1 -- make_stages()
// order for R = 8 (and its radix-16 counterpart make_stages16)
template <int N, int R = 8>
struct RegShape {
  static constexpr int LOGR = ilog2c(R);
  static constexpr int A = ilogr(N, R);        // radix-R stages
  static constexpr int R0 = N >> (LOGR * A);   // final radix (1: none)
  static constexpr int LOG2N = ilog2c(N);
  static_assert(R == 8 || R == 16, "main radix 8 or 16");
  static_assert(R0 == 1 || R0 == 2 || R0 == 4 || R0 == 8, "N must be R^a * {1,2,4,8}");
  static_assert((1 << LOG2N) == N, "N must be a power of two");
};

// frequency held by position p after the DIF of length N (the digit reversal
// of fft.cu's digit_reverse(), without a load): p = sum_q d_q S_q,
// k = sum_q d_q R^q with S_q = N / R^(q+1) and the radix-R0 digit last
template <int N, int R = 8>
__device__ __forceinline__ int revr(int p) {
  using Sh = RegShape<N, R>;
  int k = 0;
#pragma unroll
  for (int q = 0; q < Sh::A; ++q)
    k |= ((p >> (Sh::LOG2N - Sh::LOGR * (q + 1))) & (R - 1)) << (Sh::LOGR * q);
  if (Sh::R0 > 1) k |= (p & (Sh::R0 - 1)) << (Sh::LOGR * Sh::A);
  return k;
}
template <int N>
__device__ __forceinline__ int rev8(int p) {
  return revr<N, 8>(p);
}

// Shared-memory slot of exchange element e: the XOR swizzle spad(e) (PL = 0)
// or one pad slot every 2^PL elements (PL > 0): phys = e + (e >> PL).  With
// padding, the R legs of a butterfly (elements eb + r S NB) sit at
// base + off(r), base = eb + (eb >> PL) computed once per exchange and off(r)
// a compile-time constant, so an exchange costs one address computation per
// thread instead of R swizzles.  off(r) = r S NB + (r S NB >> PL) holds when
// (eb mod 2^PL) + (r S NB mod 2^PL) < 2^PL for every leg: for S NB >= 2^PL
// always; for the column passes (NB = 4, PL = 3) and S = 1, eb mod 8 = b < 4
// and r S NB mod 8 <= 4; for the row pass (NB = 1, PL = 4), eb = 16 u.
// Both layouts keep every quarter-warp's 16-byte accesses on distinct bank
// groups for the shapes instantiated (fft.cu).
template <int N_, int NBL, int T, int R_ = 8, int PL = 0>
struct RegFft {
  using Sh = RegShape<N_, R_>;
  static constexpr int R = R_;
  static constexpr int R0 = Sh::R0;
  static constexpr int N = N_;
  static constexpr int NBLOG = NBL;
  static constexpr int NB = 1 << NBL;
  static constexpr int NQ = (N / R) << NBL;  // R-element groups per stage (all vectors)
  static constexpr int BPT = NQ / T;
  static_assert(NQ % T == 0 && BPT >= 1, "threads must divide the butterflies");

  double2 x[BPT][R];

  // vector (column) of this thread's k-th group, and the group index u
  static __device__ __forceinline__ int vec(int k) { return (threadIdx.x + k * T) & (NB - 1); }
  static __device__ __forceinline__ int but(int k) { return (threadIdx.x + k * T) >> NBL; }
  // position of leg r of radix-R butterfly u in a stage of stride S; S = 1
  // is also the layout of the final radix-R0 stage (positions R u + r)
  template <int S>
  static __device__ __forceinline__ int pos(int u, int r) {
    return (u / S) * R * S + (u % S) + r * S;
  }
  // DIF/DIT stage index of radix-R stride S (S = N / R^(q+1))
  template <int S>
  static constexpr int stage() { return ilogr(N / S, R) - 1; }

  // smem elements per exchange buffer (the padded layout is 2^-PL larger)
  static constexpr int SMEM_ELEMS = PL ? ((N << NBL) + ((N << NBL) >> PL)) : (N << NBL);
  template <int S>
  static constexpr int off(int r) {
    return r * S * NB + ((r * S * NB) >> (PL ? PL : 0));
  }
  template <int S>
  static __device__ __forceinline__ int pbase(int k) {
    const int eb = (pos<S>(but(k), 0) << NBL) + vec(k);
    return eb + (eb >> PL);
  }
  template <int S>
  __device__ __forceinline__ void to_smem(double2* sm) const {
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      if constexpr (PL > 0) {
        double2* p = sm + pbase<S>(k);
#pragma unroll
        for (int r = 0; r < R; ++r) p[off<S>(r)] = x[k][r];
      } else {
        const int u = but(k), b = vec(k);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          SF_BOUNDS(spad((pos<S>(u, r) << NBL) + b) < SMEM_ELEMS);
          sm[spad((pos<S>(u, r) << NBL) + b)] = x[k][r];
        }
      }
    }
  }
  template <int S>
  __device__ __forceinline__ void from_smem(const double2* sm) {
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      if constexpr (PL > 0) {
        const double2* p = sm + pbase<S>(k);
#pragma unroll
        for (int r = 0; r < R; ++r) x[k][r] = p[off<S>(r)];
      } else {
        const int u = but(k), b = vec(k);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          SF_BOUNDS(spad((pos<S>(u, r) << NBL) + b) < SMEM_ELEMS);
          x[k][r] = sm[spad((pos<S>(u, r) << NBL) + b)];
        }
      }
    }
  }
  // write own stride-S outputs, barrier, read own stride-S2 inputs (the
  // positions a thread reads are the ones it writes next: no second barrier)
  template <int S, int S2>
  __device__ __forceinline__ void exchange(double2* sm) {
    to_smem<S>(sm);
    __syncthreads();
    from_smem<S2>(sm);
  }
  template <int S, bool DIT>
  __device__ __forceinline__ void butterflies(const FftStages& st, const double2* __restrict__ tw) {
    const double2* t = tw + st.toff[stage<S>()];
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int j = but(k) % S;
      const bool twid = S > 1 && j != 0;
      double2 w1 = make_double2(1.0, 0.0);
      if (twid) w1 = __ldg(t + j);
      if (DIT && twid) apply_twiddles<R>(x[k], w1);
      Dft<R>::run(x[k]);
      if (!DIT && twid) apply_twiddles<R>(x[k], w1);
    }
  }
  // the stride-1 radix-R0 stage: R/R0 butterflies on positions R u + r (no twiddles)
  __device__ __forceinline__ void radix_r0() {
#pragma unroll
    for (int k = 0; k < BPT; ++k)
#pragma unroll
      for (int c = 0; c < R / R0; ++c) Dft<R0>::run(&x[k][c * R0]);
  }

  // DIF from the radix-R stage of stride S (its inputs in x); ends with the
  // final-stage outputs (positions R u + r) in registers, no barrier after
  template <int S>
  __device__ __forceinline__ void dif_from(double2* sm, const FftStages& st,
                                           const double2* __restrict__ tw) {
    butterflies<S, false>(st, tw);
    if constexpr (S > R0) {
      exchange<S, S / R>(sm);
      dif_from<S / R>(sm, st, tw);
    } else if constexpr (R0 > 1) {
      exchange<S, 1>(sm);
      radix_r0();
    }
  }
  __device__ __forceinline__ void dif(double2* sm, const FftStages& st,
                                      const double2* __restrict__ tw) {
    dif_from<N / R>(sm, st, tw);
  }
  // DIT from the radix-8 stage of stride S; ends with the stride-N/8
  // (natural-order) outputs in registers
  template <int S>
  __device__ __forceinline__ void dit_from(double2* sm, const FftStages& st,
                                           const double2* __restrict__ tw) {
    butterflies<S, true>(st, tw);
    if constexpr (S < N / R) {
      exchange<S, S * R>(sm);
      dit_from<S * R>(sm, st, tw);
    }
  }
  // full DIT from the final-stage layout (positions 8u + r, digit-reversed)
  __device__ __forceinline__ void dit(double2* sm, const FftStages& st,
                                      const double2* __restrict__ tw) {
    if constexpr (R0 > 1) {
      radix_r0();
      exchange<1, R0>(sm);
      dit_from<R0>(sm, st, tw);
    } else {
      dit_from<1>(sm, st, tw);
    }
  }
};

}  // namespace sfb
