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
  __shared__ double2 hs[kGatherSpan];
  const int64_t jb = (int64_t)blockIdx.x * kGatherGroup + threadIdx.x;
  const int col = blockIdx.y;
  const double2* h = a.h + (int64_t)col * a.Kout;
  pdl_trigger();
  const int2 sp = __ldg(a.span + blockIdx.x);
  const int64_t klo = sp.x, khi = sp.y;
  const bool staged = klo >= 0 && khi < a.Kout && khi - klo + 1 <= kGatherSpan;
  // the plan's target tables are independent of the previous kernel: their
  // loads are in flight while this CTA waits for h
  double pos[2 * NP], sc[2 * NP];
  int dst[2 * NP];
#pragma unroll
  for (int t = 0; t < 2 * NP; ++t) {
    const int64_t j = jb + (int64_t)t * kGatherThreads;
    pos[t] = t > 0 ? pos[0] : 0.0;  // inactive targets keep a window in range
    sc[t] = 0.0;
    dst[t] = -1;
    if (j < a.M2) {
      pos[t] = __ldg(a.pos + j);
      sc[t] = __ldg(a.scale + j);
      dst[t] = __ldg(a.perm + j);
    }
  }
  pdl_wait();  // h is the previous kernel's output
#if SFB_GATHER_TMA
  // the span is one contiguous range: one bulk copy on the TMA engine,
  // completing on an mbarrier (no per-thread copy instructions)
  __shared__ __align__(8) unsigned long long mbar;
  if (staged && threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    bulk_g2s(hs, h + klo, (unsigned)((khi - klo + 1) * sizeof(double2)), &mbar);
  }
  if (staged) {
    __syncthreads();  // the barrier is initialised before anyone polls it
    mbar_wait(&mbar, 0);
  }
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
      window_dot2<M>(C, p0 - c0, p1 - c1, hs + (k0 - klo), hs + (k1 - klo), s0, s1);
    } else {
      s0 = gather_one<M>(a, h, p0, C);
      if (dst[2 * q + 1] >= 0) s1 = gather_one<M>(a, h, p1, C);
    }
    a.out[(int64_t)dst[2 * q] * a.batch + col] =
        make_double2(s0.x * sc[2 * q], sg * (s0.y * sc[2 * q]));
    if (dst[2 * q + 1] >= 0)
      a.out[(int64_t)dst[2 * q + 1] * a.batch + col] =
          make_double2(s1.x * sc[2 * q + 1], sg * (s1.y * sc[2 * q + 1]));
  }
}

// Persistent form of k_gather2 (SFB_GATHER_PERSIST): every CTA walks the
// 256-target groups g = blockIdx.x, blockIdx.x + gridDim.x, ... -- round-robin,
// so at any moment all CTAs work on one band of consecutive groups (one index
// slice: the scattered output stores still merge in L2) -- and the next
// group's h span is on its way (TMA bulk copy into the other half of a
// double buffer) and its plan records in registers while the current group is
// interpolated: no CTA-start latency after the first group.
#ifndef SFB_GATHER3_MINB
#define SFB_GATHER3_MINB 4
#endif
#ifndef SFB_GATHER_PERSIST_DEFAULT
#define SFB_GATHER_PERSIST_DEFAULT 0
#endif
__device__ __forceinline__ bool span_fits(const GatherArgs& a, int2 sp) {
  return sp.x >= 0 && sp.y < a.Kout && sp.y - sp.x + 1 <= kGatherSpan;
}
// the plan records (position, scale, destination) of this thread's two
// targets of group g into stage st of the record buffers (cp.async, no
// registers held); out-of-range targets are zero-filled
__device__ __forceinline__ void issue_grec(const GatherArgs& a, int64_t g, double (*rp)[2][kGatherThreads],
                                          double (*rs)[2][kGatherThreads],
                                          int (*rd)[2][kGatherThreads], int st) {
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int64_t j = g * kGatherGroup + threadIdx.x + (int64_t)t * kGatherThreads;
    const bool ok = j < a.M2;
    const int64_t jj = ok ? j : 0;
    cp_async8z(&rp[st][t][threadIdx.x], a.pos + jj, ok ? 8 : 0);
    cp_async8z(&rs[st][t][threadIdx.x], a.scale + jj, ok ? 8 : 0);
    cp_async4z(&rd[st][t][threadIdx.x], a.perm + jj, ok ? 4 : 0);
  }
  cp_async_commit();
}
template <int M>
__global__ void __launch_bounds__(kGatherThreads, SFB_GATHER3_MINB)
    k_gather3(GatherArgs a, WinCoef C, int64_t n_groups) {
  static_assert(kGatherTPT == 2, "two targets per thread");
  __shared__ __align__(16) double2 hs[2][kGatherSpan];
  __shared__ double rp[2][2][kGatherThreads], rs[2][2][kGatherThreads];
  __shared__ int rd[2][2][kGatherThreads];
  __shared__ __align__(8) unsigned long long mbar[2];
  const int col = blockIdx.y;
  const double2* h = a.h + (int64_t)col * a.Kout;
  const int64_t stride = gridDim.x;
  int64_t g = blockIdx.x;
  if (g >= n_groups) return;
  issue_grec(a, g, rp, rs, rd, 0);
  int2 sp_cur = __ldg(a.span + g);
  int2 sp_nxt = g + stride < n_groups ? __ldg(a.span + g + stride) : make_int2(-1, -1);
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
  }
  __syncthreads();
  pdl_wait();  // h is the previous kernel's output
  if (threadIdx.x == 0) {
    if (span_fits(a, sp_cur))
      bulk_g2s(hs[0], h + sp_cur.x, (unsigned)((sp_cur.y - sp_cur.x + 1) * sizeof(double2)),
               &mbar[0]);
    else
      mbar_arrive(&mbar[0]);
  }
  const double sg = a.conj_out ? -1.0 : 1.0;
  for (int i = 0; g < n_groups; ++i, g += stride) {
    const int b = i & 1;
    const int64_t gn = g + stride;
    // the other buffers were released by the barrier that ended iteration i-1
    if (gn < n_groups) {
      if (threadIdx.x == 0) {
        if (span_fits(a, sp_nxt))
          bulk_g2s(hs[b ^ 1], h + sp_nxt.x,
                   (unsigned)((sp_nxt.y - sp_nxt.x + 1) * sizeof(double2)), &mbar[b ^ 1]);
        else
          mbar_arrive(&mbar[b ^ 1]);
      }
      issue_grec(a, gn, rp, rs, rd, b ^ 1);
    } else {
      cp_async_commit();  // keep the group count: wait<1> below covers stage b
    }
    const int2 sp = sp_cur;
    sp_cur = sp_nxt;
    if (gn + stride < n_groups) sp_nxt = __ldg(a.span + gn + stride);
    cp_async_wait<1>();  // this thread's records of group g
    const int64_t j0 = g * kGatherGroup + threadIdx.x;
    const bool act0 = j0 < a.M2, act1 = j0 + kGatherThreads < a.M2;
    const double p0 = act0 ? rp[b][0][threadIdx.x] : 0.0;
    const double p1 = act1 ? rp[b][1][threadIdx.x] : p0;  // inactive: a window in range
    mbar_wait(&mbar[b], (i >> 1) & 1);
    if (act0) {
      double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
      if (span_fits(a, sp)) {
        const double c0 = floor(p0), c1 = floor(p1);
        const int64_t k0 = (int64_t)c0 + (1 - M) - a.s_lo, k1 = (int64_t)c1 + (1 - M) - a.s_lo;
        window_dot2<M>(C, p0 - c0, p1 - c1, hs[b] + (k0 - sp.x), hs[b] + (k1 - sp.x), s0, s1);
      } else {
        s0 = gather_one<M>(a, h, p0, C);
        if (act1) s1 = gather_one<M>(a, h, p1, C);
      }
      const double sc0 = rs[b][0][threadIdx.x];
      a.out[(int64_t)rd[b][0][threadIdx.x] * a.batch + col] =
          make_double2(s0.x * sc0, sg * (s0.y * sc0));
      if (act1) {
        const double sc1 = rs[b][1][threadIdx.x];
        a.out[(int64_t)rd[b][1][threadIdx.x] * a.batch + col] =
            make_double2(s1.x * sc1, sg * (s1.y * sc1));
      }
    }
    __syncthreads();  // every read of hs[b] is done before it is refilled
  }
}

bool gather_persistent() {
  static const int v = [] {
    const char* e = getenv("SFB_GATHER_PERSIST");
    return e ? atoi(e) : SFB_GATHER_PERSIST_DEFAULT;
  }();
  return v != 0;
}

void run_gather(const NnfftPlanImpl& p, const double2* h, double2* out, int batch,
                cudaStream_t s) {
  GatherArgs a{p.gp.pos.p, p.gp.perm.p, p.gp.scale.p, p.gp.span.p, h, out,
               p.g.M2,     p.fft.Kout,  p.g.N2,        p.fft.s_lo,  batch, p.gp.conj_out ? 1 : 0};
  const dim3 grid((unsigned)ceil_div(p.g.M2, (int64_t)kGatherGroup), batch);
  const int64_t n_groups = ceil_div(p.g.M2, (int64_t)kGatherGroup);
  // persistent: resident CTAs x SMs, fewer when there are fewer groups
  auto pgrid = [&](auto kern) {
    static int per_sm = -1;
    if (per_sm < 0) SF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                                          kGatherThreads, 0));
    return dim3((unsigned)std::min<int64_t>(n_groups, (int64_t)std::max(per_sm, 1) * p.sp.n_sms),
                batch);
  };
  switch (p.g.m2) {
#define SF_CASE(MM)                                                                            \
  case MM:                                                                                     \
    if (kGatherTPT == 2 && gather_persistent())                                                \
      launch_pdl(k_gather3<MM>, pgrid(k_gather3<MM>), dim3(kGatherThreads), 0, s, a, p.c2,     \
                 n_groups);                                                                    \
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
