// gather.cu -- step 4 of Algorithm 2.1: interpolate the fine-grid values at
// the M2 spatial nodes with the second window and divide by phi_hat_1.
//
// Reference (pkg/src/sincfft/nnfft.py:198-205, 241-243):
//     out_j = sum_{t=1-m2}^{m2} h[(c_j + t) mod N2] phi_2(xs_j - (c_j+t)/N2)
//             / phi_hat_1(N x_j),   xs_j = x_j N/N1, c_j = floor(N2 xs_j).
// Targets are sorted at plan time by (slice of the original index, position):
// within a slice a CTA's targets read one short contiguous window of h (staged
// in shared memory), and its outputs -- stored to the targets' original
// indices -- all fall in the slice's window of `out`, small enough to stay
// L2-resident so the scattered 16-byte stores merge into full sectors.  The
// 2m2 window values come from the per-tap polynomials (window.cuh); the scale
// 1/phi_hat_1 (times the Clenshaw-Curtis weight for fast-sinc stage 1) is one
// sorted fp64 stream.
#include "nnfft_impl.cuh"

namespace sfb {

struct GatherArgs {
  const double* pos;
  const int* perm;
  const double* scale;
  const int2* span;  // per CTA block: {klo, khi} h range read (plan time)
  const double2* h;  // [batch][Kout], h[k'] = h_{s_lo + k'}
  double2* out;      // (M2, batch) row-major
  int64_t M2, Kout, N2, s_lo;
  int batch;
  int conj_out;
};



template <int M>
__device__ __forceinline__ double2 gather_dot(const double2* hp, const double* w) {
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < 2 * M; ++i) {
    const double2 v = hp[i];
    s.x = fma(v.x, w[i], s.x);
    s.y = fma(v.y, w[i], s.y);
  }
  return s;
}

// One CTA = 256 consecutive sorted targets of one slice.  Their 2m-tap windows
// cover one short contiguous range of h; the CTA stages that range
// in shared memory with coalesced loads, so each tap is an LDS (broadcast for
// coincident targets) instead of a dependent global load.  CTAs whose range
// exceeds kGatherSpan (sparse regions) or wraps around N2 read h directly.
template <int M>
__global__ void __launch_bounds__(kGatherThreads) k_gather(GatherArgs a, WinCoef C) {
  __shared__ double2 hs[kGatherSpan];
  const int64_t j0 = (int64_t)blockIdx.x * kGatherThreads;
  const int64_t j = j0 + threadIdx.x;
  const int col = blockIdx.y;
  const bool act = j < a.M2;
  double pos = 0.0, sc = 0.0;
  int dst = 0;
  if (act) {
    pos = __ldg(a.pos + j);
    sc = __ldg(a.scale + j);
    dst = __ldg(a.perm + j);
  }
  const double2* h = a.h + (int64_t)col * a.Kout;
  // the block's h range is precomputed at plan time, so its asynchronous copy
  // into shared memory starts at once and overlaps the window evaluation
  const int2 sp = __ldg(a.span + blockIdx.x);
  const int64_t klo = sp.x, khi = sp.y;
  const bool staged = klo >= 0 && khi < a.Kout && khi - klo + 1 <= kGatherSpan;
  if (staged) {
    for (int64_t i = threadIdx.x; i <= khi - klo; i += kGatherThreads)
      cp_async16(hs + i, h + klo + i);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  const double c = floor(pos);
  double w[2 * M];
  window_taps<M>(C, pos - c, w);
  if (staged) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  }
  if (!act) return;
  const int64_t k0 = (int64_t)c + (1 - M) - a.s_lo;
  double2 s;
  if (staged) {
    s = gather_dot<M>(hs + (k0 - klo), w);
  } else if (k0 >= 0 && k0 + 2 * M <= a.Kout) {
    s = gather_dot<M>(h + k0, w);
  } else {  // periodic wrap (only when Kout == N2 covers every residue)
    s = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < 2 * M; ++i) {
      int64_t k = (k0 + i) % a.N2;
      if (k < 0) k += a.N2;
      const double2 v = __ldg(h + k);
      s.x = fma(v.x, w[i], s.x);
      s.y = fma(v.y, w[i], s.y);
    }
  }
  // scattered store, but inside this slice's window of `out` (the plan sorts
  // targets by (original-index slice, position)), which stays L2-resident, so
  // both 16-byte halves of each 32-byte sector merge in L2 before eviction
  a.out[(int64_t)dst * a.batch + col] = make_double2(s.x * sc, a.conj_out ? -(s.y * sc) : s.y * sc);
}

// kGatherTPT = 2: each thread interpolates targets j0 + t and j0 + 256 + t
// of a 512-target group together (window_dot2: one coefficient load per two
// Horner steps, no tap arrays).  The staged h range must be complete before
// the first tap pair is consumed, so the copy is awaited first.
template <int M>
__device__ __forceinline__ double2 gather_one(const GatherArgs& a, const double2* h, double pos,
                                              const WinCoef& C) {
  const double c = floor(pos);
  double w[2 * M];
  window_taps<M>(C, pos - c, w);
  const int64_t k0 = (int64_t)c + (1 - M) - a.s_lo;
  if (k0 >= 0 && k0 + 2 * M <= a.Kout) return gather_dot<M>(h + k0, w);
  double2 s = make_double2(0.0, 0.0);  // periodic wrap (Kout == N2)
#pragma unroll
  for (int i = 0; i < 2 * M; ++i) {
    int64_t k = (k0 + i) % a.N2;
    if (k < 0) k += a.N2;
    const double2 v = __ldg(h + k);
    s.x = fma(v.x, w[i], s.x);
    s.y = fma(v.y, w[i], s.y);
  }
  return s;
}

#ifndef SFB_GATHER_ABL
#define SFB_GATHER_ABL 0  // timing ablations (wrong results): 1 sorted stores, 2 no windows
#endif
#ifndef SFB_GATHER_RECTMA
#define SFB_GATHER_RECTMA 0  // plan records by bulk copies (needs group-padded tables)
#endif
#ifndef SFB_GATHER_OCTET
#define SFB_GATHER_OCTET 1  // k_gather2 on the octet-ordered records
#endif
#ifndef SFB_GATHER_HINT
#define SFB_GATHER_HINT 0  // L2 hints: 1 streaming record loads, 2 span copy evict-last
#endif
#ifndef SFB_GATHER_PF
#define SFB_GATHER_PF 0  // L2 prefetch distance in CTAs (0: off)
#endif
#ifndef SFB_GATHER_ALLSAME
#define SFB_GATHER_ALLSAME 1  // warps whose 32 threads all hold a same-window pair: no second loads
#endif
#ifndef SFB_GATHER_TMA
#define SFB_GATHER_TMA 1  // the h span staged by one TMA bulk copy
#endif
#ifndef SFB_GATHER2_MINB
#define SFB_GATHER2_MINB (8 * 128 / SFB_GATHER_THREADS)  // 64 registers (0.381 -> 0.299 ms at config 3)
#endif
// kGatherTPT = 2 * NP: each thread interpolates NP pairs of targets (j, j +
// kGatherThreads) of its group, one window_dot2 per pair, after ONE staged
// copy of the group's h span -- more targets per CTA amortise the copy
// latency every CTA exposes at its start.
template <int M>
__global__ void __launch_bounds__(kGatherThreads, SFB_GATHER2_MINB) k_gather2(GatherArgs a,
                                                                            WinCoef C) {
  constexpr int NP = kGatherTPT / 2;
  __shared__ __align__(128) double2 hs[kGatherSpan];  // bank group of hs[i] = i mod 8
  const int64_t jb = (int64_t)blockIdx.x * kGatherGroup + threadIdx.x;
  const int col = blockIdx.y;
  const double2* h = a.h + (int64_t)col * a.Kout;
  pdl_trigger();
#if SFB_GATHER_TMA
  __shared__ __align__(8) unsigned long long mbar;
  if (threadIdx.x == 0) mbar_init(&mbar, 1);
#endif
#if SFB_GATHER_RECTMA
  // the group's plan records (positions, scales, destinations: contiguous,
  // padded to whole groups at plan time) arrive by three bulk copies issued
  // at once -- no per-thread loads in front of the span copy
  __shared__ __align__(16) double rpos[kGatherGroup], rsc[kGatherGroup];
  __shared__ __align__(16) int rdst[kGatherGroup];
  __shared__ __align__(8) unsigned long long mbar_r;
  if (threadIdx.x == 0) {
    mbar_init(&mbar_r, 1);
    const int64_t j0 = (int64_t)blockIdx.x * kGatherGroup;
    mbar_expect_tx(&mbar_r, kGatherGroup * (2 * sizeof(double) + sizeof(int)));
    bulk_g2s_tx(rpos, a.pos + j0, kGatherGroup * sizeof(double), &mbar_r);
    bulk_g2s_tx(rsc, a.scale + j0, kGatherGroup * sizeof(double), &mbar_r);
    bulk_g2s_tx(rdst, a.perm + j0, kGatherGroup * sizeof(int), &mbar_r);
  }
#endif
  const int2 sp = __ldg(a.span + blockIdx.x);
  const int64_t klo = sp.x, khi = sp.y;
  const bool staged = klo >= 0 && khi < a.Kout && khi - klo + 1 <= kGatherSpan;
  // the plan's target tables are independent of the previous kernel: their
  // loads are in flight while this CTA waits for h
  double pos[2 * NP], sc[2 * NP];
  int dst[2 * NP];
#if SFB_GATHER_RECTMA
  __syncthreads();  // mbar_r initialised before anyone polls it
  mbar_wait(&mbar_r, 0);
#endif
#pragma unroll
  for (int t = 0; t < 2 * NP; ++t) {
    const int64_t j = jb + (int64_t)t * kGatherThreads;
    pos[t] = t > 0 ? pos[0] : 0.0;  // inactive targets keep a window in range
    sc[t] = 0.0;
    dst[t] = -1;
    if (j < a.M2) {
#if SFB_GATHER_ABL & 8  // ablation: no record loads (positions inside the span)
      pos[t] = (double)(klo + a.s_lo + 8) + 0.001 * (threadIdx.x & 255);
      sc[t] = 1.0;
      dst[t] = (int)j;
#elif SFB_GATHER_RECTMA
      pos[t] = rpos[threadIdx.x + t * kGatherThreads];
      sc[t] = rsc[threadIdx.x + t * kGatherThreads];
      dst[t] = rdst[threadIdx.x + t * kGatherThreads];
#elif SFB_GATHER_HINT & 1  // streaming record loads (evict-first in L2)
      pos[t] = __ldcs(a.pos + j);
      sc[t] = __ldcs(a.scale + j);
      dst[t] = __ldcs(a.perm + j);
#else
      pos[t] = __ldg(a.pos + j);
      sc[t] = __ldg(a.scale + j);
      dst[t] = __ldg(a.perm + j);
#endif
    }
  }
  pdl_wait();  // h is the previous kernel's output
#if SFB_GATHER_ABL & 4  // ablation: no span copy (smem left as is)
  if (false) {
#elif SFB_GATHER_TMA
  if (true) {
#endif
#if SFB_GATHER_TMA
  // the span is one contiguous range: one bulk copy on the TMA engine,
  // completing on an mbarrier (no per-thread copy instructions)
  if (staged && threadIdx.x == 0) {
#if SFB_GATHER_HINT & 2  // the span copy marks h evict-last in L2
    bulk_g2s_hint<true>(hs, h + klo, (unsigned)((khi - klo + 1) * sizeof(double2)), &mbar);
#else
    bulk_g2s(hs, h + klo, (unsigned)((khi - klo + 1) * sizeof(double2)), &mbar);
#endif
  }
#if SFB_GATHER_PF
  // L2 prefetch for the group SFB_GATHER_PF CTAs ahead (about one resident
  // wave: the CTA that will start when this one ends) -- its plan records and
  // its h span -- so CTA start waits on L2, not DRAM
  if (threadIdx.x == 32) {
    const int64_t gf = (int64_t)blockIdx.x + SFB_GATHER_PF;
    if (gf * kGatherGroup + kGatherGroup <= a.M2) {
      bulk_prefetch_l2(a.pos + gf * kGatherGroup, kGatherGroup * sizeof(double));
      bulk_prefetch_l2(a.scale + gf * kGatherGroup, kGatherGroup * sizeof(double));
      bulk_prefetch_l2(a.perm + gf * kGatherGroup, kGatherGroup * sizeof(int));
      const int2 spf = __ldg(a.span + gf);
      if (spf.x >= 0 && spf.y < a.Kout && spf.y - spf.x + 1 <= kGatherSpan)
        bulk_prefetch_l2(h + spf.x, (unsigned)((spf.y - spf.x + 1) * sizeof(double2)));
    }
  }
#endif
  if (staged) {
    __syncthreads();  // the barrier is initialised before anyone polls it
    mbar_wait(&mbar, 0);
  }
#if SFB_GATHER_TMA
  }
#endif
#else
  if (staged) {
    for (int64_t i = threadIdx.x; i <= khi - klo; i += kGatherThreads)
      cp_async16(hs + i, h + klo + i);
    cp_async_commit();
  }
  if (staged) {
    cp_async_wait<0>();
    __syncthreads();
  }
#endif
  if (dst[0] < 0) return;
  const double sg = a.conj_out ? -1.0 : 1.0;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const double p0 = pos[2 * q], p1 = dst[2 * q + 1] >= 0 ? pos[2 * q + 1] : p0;
    double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
    if (dst[2 * q] < 0) break;
    if (staged) {
      const double c0 = floor(p0), c1 = floor(p1);
      const int64_t k0 = (int64_t)c0 + (1 - M) - a.s_lo, k1 = (int64_t)c1 + (1 - M) - a.s_lo;
#if SFB_GATHER_ABL & 2  // ablation (timing only): taps read, no window polynomials
      const double2* h0 = hs + (k0 - klo);
      const double2* h1 = hs + (k1 - klo);
#pragma unroll
      for (int t = 0; t < 2 * M; ++t) {
        s0.x += h0[t].x * p0, s0.y += h0[t].y * p0;
        s1.x += h1[t].x * p1, s1.y += h1[t].y * p1;
      }
#else
      SF_BOUNDS(k0 >= klo && k0 + 2 * M - 1 <= khi && k1 >= klo && k1 + 2 * M - 1 <= khi);
#if SFB_GATHER_ALLSAME
      if (__all_sync(__activemask(), k0 == k1))  // (lanes past M2 have left)
        window_dot2<M, true>(C, p0 - c0, p1 - c1, hs + (k0 - klo), hs + (k1 - klo), s0, s1, true);
      else
#endif
      window_dot2<M>(C, p0 - c0, p1 - c1, hs + (k0 - klo), hs + (k1 - klo), s0, s1, k0 == k1);
#endif
    } else {
      s0 = gather_one<M>(a, h, p0, C);
      if (dst[2 * q + 1] >= 0) s1 = gather_one<M>(a, h, p1, C);
    }
#if SFB_GATHER_ABL & 1  // ablation (timing only): sorted-order stores instead of scattered
    a.out[(jb + 2 * q * kGatherThreads) * a.batch + col] =
        make_double2(s0.x * sc[2 * q], sg * (s0.y * sc[2 * q]));
    if (dst[2 * q + 1] >= 0)
      a.out[(jb + (2 * q + 1) * kGatherThreads) * a.batch + col] =
          make_double2(s1.x * sc[2 * q + 1], sg * (s1.y * sc[2 * q + 1]));
#else
    a.out[(int64_t)dst[2 * q] * a.batch + col] =
        make_double2(s0.x * sc[2 * q], sg * (s0.y * sc[2 * q]));
    if (dst[2 * q + 1] >= 0)
      a.out[(int64_t)dst[2 * q + 1] * a.batch + col] =
          make_double2(s1.x * sc[2 * q + 1], sg * (s1.y * sc[2 * q + 1]));
#endif
  }
}

// SFB_GATHER_NT = 4: k_gather2 with each thread interpolating 4 targets
// (j0 + t + i * T, i < 4) through one window_dotn -- every coefficient load
// feeds 4 Horner chains -- over kGatherThreads / 2 threads per CTA, so a CTA
// still covers kGatherGroup targets and one staged span.
#ifndef SFB_GATHER_NT
#define SFB_GATHER_NT 2
#endif
#ifndef SFB_GATHER4_MINB
#define SFB_GATHER4_MINB 12
#endif
template <int M>
__global__ void __launch_bounds__(kGatherGroup / 4, SFB_GATHER4_MINB) k_gather4(GatherArgs a,
                                                                             WinCoef C) {
  constexpr int T = kGatherGroup / 4, NT = 4;
  __shared__ __align__(16) double2 hs[kGatherSpan];
  __shared__ __align__(8) unsigned long long mbar;
  const int64_t jb = (int64_t)blockIdx.x * kGatherGroup + threadIdx.x;
  const int col = blockIdx.y;
  const double2* h = a.h + (int64_t)col * a.Kout;
  pdl_trigger();
  const int2 sp = __ldg(a.span + blockIdx.x);
  const int64_t klo = sp.x, khi = sp.y;
  const bool staged = klo >= 0 && khi < a.Kout && khi - klo + 1 <= kGatherSpan;
  double pos[NT], sc[NT];
  int dst[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int64_t j = jb + (int64_t)t * T;
    pos[t] = t > 0 ? pos[0] : 0.0;
    sc[t] = 0.0;
    dst[t] = -1;
    if (j < a.M2) {
      pos[t] = __ldg(a.pos + j);
      sc[t] = __ldg(a.scale + j);
      dst[t] = __ldg(a.perm + j);
    }
  }
  pdl_wait();
  if (staged && threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    bulk_g2s(hs, h + klo, (unsigned)((khi - klo + 1) * sizeof(double2)), &mbar);
  }
  if (staged) {
    __syncthreads();
    mbar_wait(&mbar, 0);
  }
  if (dst[0] < 0) return;
  const double sg = a.conj_out ? -1.0 : 1.0;
  double2 s[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) s[t] = make_double2(0.0, 0.0);
  if (staged) {
    double d[NT];
    const double2* hp[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const double c = floor(pos[t]);
      d[t] = pos[t] - c;
      hp[t] = hs + ((int64_t)c + (1 - M) - a.s_lo - klo);
    }
    window_dotn<M, NT>(C, d, hp, s);
  } else {
#pragma unroll
    for (int t = 0; t < NT; ++t)
      if (dst[t] >= 0) s[t] = gather_one<M>(a, h, pos[t], C);
  }
#pragma unroll
  for (int t = 0; t < NT; ++t)
    if (dst[t] >= 0)
      a.out[(int64_t)dst[t] * a.batch + col] =
          make_double2(s[t].x * sc[t], sg * (s[t].y * sc[t]));
}

void run_gather(const NnfftPlanImpl& p, const double2* h, double2* out, int batch,
                cudaStream_t s) {
  // k_gather2 reads the octet-ordered records (bank-conflict-free span loads)
  const bool oct = kGatherTPT == 2 && p.gp.opos.p != nullptr && SFB_GATHER_OCTET;
  GatherArgs a{oct ? p.gp.opos.p : p.gp.pos.p, oct ? p.gp.operm.p : p.gp.perm.p,
               oct ? p.gp.oscale.p : p.gp.scale.p, p.gp.span.p, h, out,
               p.g.M2,     p.fft.Kout,  p.g.N2,        p.fft.s_lo,  batch, p.gp.conj_out ? 1 : 0};
  const dim3 grid((unsigned)ceil_div(p.g.M2, (int64_t)kGatherGroup), batch);
  switch (p.g.m2) {
#define SF_CASE(MM)                                                                            \
  case MM:                                                                                     \
    if (SFB_GATHER_NT == 4 && kGatherTPT == 2)                                                 \
      launch_pdl(k_gather4<MM>, grid, dim3(kGatherGroup / 4), 0, s, a, p.c2);                  \
    else if (kGatherTPT >= 2) launch_pdl(k_gather2<MM>, grid, dim3(kGatherThreads), 0, s, a, p.c2); \
    else k_gather<MM><<<grid, kGatherThreads, 0, s>>>(a, p.c2);                                \
    break;
    SF_CASE(2) SF_CASE(3) SF_CASE(4) SF_CASE(5) SF_CASE(6) SF_CASE(7) SF_CASE(8) SF_CASE(9)
    SF_CASE(10) SF_CASE(11) SF_CASE(12) SF_CASE(13) SF_CASE(14) SF_CASE(15) SF_CASE(16)
#undef SF_CASE
    default:
      fail(5, "unsupported m2");
  }
  SF_LAUNCH_CHECK();
}

}  // namespace sfb
