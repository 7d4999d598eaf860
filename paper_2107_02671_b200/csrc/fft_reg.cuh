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
// them.  Length N = 8^a (the shapes the planner picks for the batched path:
// 512 x 512), NB = 2^NBL interleaved vectors (columns) per CTA, T threads.
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

__host__ __device__ constexpr int ilog8(int n) { return n <= 1 ? 0 : 1 + ilog8(n / 8); }

// frequency held by position p after a radix-8 DIF of length N = 8^a: the
// base-8 digits of p reversed (= digit_reverse() of fft.cu, without a load)
template <int N>
__device__ __forceinline__ int rev8(int p) {
  int k = 0;
#pragma unroll
  for (int q = 0; q < ilog8(N); ++q) k = (k << 3) | ((p >> (3 * q)) & 7);
  return k;
}

template <int N, int NBL, int T>
struct RegFft {
  static constexpr int NB = 1 << NBL;
  static constexpr int NQ = (N / 8) << NBL;  // butterflies per stage (all vectors)
  static constexpr int BPT = NQ / T;
  static constexpr int NST = ilog8(N);
  static_assert(NQ % T == 0 && BPT >= 1, "threads must divide the butterflies");
  static_assert((1 << (3 * NST)) == N, "N must be a power of 8");

  double2 x[BPT][8];

  // vector (column) of this thread's k-th butterfly, and its index u
  static __device__ __forceinline__ int vec(int k) { return (threadIdx.x + k * T) & (NB - 1); }
  static __device__ __forceinline__ int but(int k) { return (threadIdx.x + k * T) >> NBL; }
  // position of leg r of butterfly u in a stage of stride S
  template <int S>
  static __device__ __forceinline__ int pos(int u, int r) {
    return (u / S) * 8 * S + (u % S) + r * S;
  }
  // DIF/DIT stage index of stride S (S = N / 8^(q+1))
  template <int S>
  static constexpr int stage() { return NST - 1 - ilog8(S); }

  template <int S>
  __device__ __forceinline__ void to_smem(double2* sm) const {
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int u = but(k), b = vec(k);
#pragma unroll
      for (int r = 0; r < 8; ++r) sm[spad((pos<S>(u, r) << NBL) + b)] = x[k][r];
    }
  }
  template <int S>
  __device__ __forceinline__ void from_smem(const double2* sm) {
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int u = but(k), b = vec(k);
#pragma unroll
      for (int r = 0; r < 8; ++r) x[k][r] = sm[spad((pos<S>(u, r) << NBL) + b)];
    }
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
      if (DIT && twid) apply_twiddles<8>(x[k], w1);
      Dft<8>::run(x[k]);
      if (!DIT && twid) apply_twiddles<8>(x[k], w1);
    }
  }

  // DIF stages of strides S, S/8, ..., 1 (data of stride S already in x);
  // ends with the stride-1 outputs in registers (no barrier after)
  template <int S>
  __device__ __forceinline__ void dif_from(double2* sm, const FftStages& st,
                                           const double2* __restrict__ tw) {
    butterflies<S, false>(st, tw);
    if constexpr (S > 1) {
      to_smem<S>(sm);
      __syncthreads();
      from_smem<S / 8>(sm);
      dif_from<S / 8>(sm, st, tw);
    }
  }
  // DIT stages of strides S, 8S, ..., N/8 (data of stride S in x); ends with
  // the stride-N/8 (natural-order) outputs in registers
  template <int S>
  __device__ __forceinline__ void dit_from(double2* sm, const FftStages& st,
                                           const double2* __restrict__ tw) {
    butterflies<S, true>(st, tw);
    if constexpr (S < N / 8) {
      to_smem<S>(sm);
      __syncthreads();
      from_smem<S * 8>(sm);
      dit_from<S * 8>(sm, st, tw);
    }
  }
};

}  // namespace sfb
