// batched.cu -- B >= kBatchedMin coefficient columns sharing one plan
// (BASELINE config 4: 256 columns).  The reference applies nnfft_trafo column
// by column; here the columns are the vector dimension:
//
//   * a lane owns one column, a warp 32 consecutive columns, so every load of
//     F[src, :] and store of out[dst, :] (row-major (M, B) user layouts) is a
//     512-byte coalesced row segment;
//   * window values are evaluated ONCE per node per warp (lane l evaluates
//     node l of a 32-node block, the block's windows are broadcast from shared
//     memory) and reused by all 32 columns;
//   * spread: nodes sorted by cell; each lane keeps a ROLLING register window
//     of the 2m grid points the current cell touches; when the cell advances
//     the lowest point is final and is stored (tile interior: plain store,
//     exclusive; tile halo: fp64 atomic into zeroed rows) -- no shared-memory
//     accumulator and no per-tap atomics;
//   * gather: targets sorted by position; each lane keeps a rolling window of
//     the 2m h rows the current target reads, loading only rows that enter the
//     window (consecutive targets share almost all of them).
// Grid and h use point-major layouts [K][B], [Kout][B]; the length-L FFT
// stage still runs per column, with tiled transposes around it.
#include "nnfft_impl.cuh"

#include <atomic>
#include <type_traits>

namespace sfb {

constexpr int kTileB = 128;   // cells per spread CTA
#ifndef SFB_SPREADB_SUB
#define SFB_SPREADB_SUB 4
#endif
constexpr int kSub = SFB_SPREADB_SUB;  // F rows per pipelined sub-block
constexpr int kThreadsB = 128;  // 4 warps = 128 columns per CTA

// ------------------------------------------------------------------ spread
struct SpreadBArgs {
  const double* pos;   // cell-sorted fl(N1 v)
  const int* perm;
  const int* tile;     // first sorted source of each kTileB-cell tile [ntile+1]
  const double2* f;    // (M1, B) row-major
  double2* grid;       // [K][B]
  int64_t K;
  int B;
};

template <int M>
__device__ __forceinline__ void spread_flush(const SpreadBArgs& a, double2* r, int64_t& ccur,
                                             int64_t cell0, int64_t cend, int col, bool colok) {
  const int64_t p = ccur + 1 - M;
  if (colok && p >= 0 && p < a.K) {
    double2* dst = a.grid + p * a.B + col;
    if (p >= cell0 + M && p <= cend - M) {
      *dst = r[0];  // interior: only this tile touches it
    } else if (r[0].x != 0.0 || r[0].y != 0.0) {
      atomicAdd(&dst->x, r[0].x);
      atomicAdd(&dst->y, r[0].y);
    }
  }
#pragma unroll
  for (int i = 0; i < 2 * M - 1; ++i) r[i] = r[i + 1];
  r[2 * M - 1] = make_double2(0.0, 0.0);
  ++ccur;
}

#ifndef SFB_SPREADB_MINB
#define SFB_SPREADB_MINB 3  // 154 registers, no spills: 1.70 -> 1.58 ms at config 4
#endif
template <int M>
__global__ void __launch_bounds__(kThreadsB, SFB_SPREADB_MINB) k_spread_b(SpreadBArgs a, WinCoef C) {
  extern __shared__ __align__(16) double wsm[];
  constexpr int WS = 2 * M + 1;  // padded row
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* wl = wsm + warp * 32 * WS;
  const int col = blockIdx.y * blockDim.x + threadIdx.x;
  const bool colok = col < a.B;
  const double2* fcol = a.f + col;
  const int64_t cell0 = (int64_t)blockIdx.x * kTileB;
  const int64_t cend = min(cell0 + kTileB, a.K);
  const int s0 = a.tile[blockIdx.x], s1 = a.tile[blockIdx.x + 1];
  const int64_t halfK = a.K / 2;
  double2 r[2 * M];
#pragma unroll
  for (int i = 0; i < 2 * M; ++i) r[i] = make_double2(0.0, 0.0);
  int64_t ccur = cell0 - 1;
  for (int sb = s0; sb < s1; sb += 32) {
    const int j = sb + lane;
    int cl = 0, src = 0;
    if (j < s1) {
      const double pos = __ldg(a.pos + j);
      const double fl = floor(pos);
      cl = (int)((int64_t)fl + halfK);
      src = __ldg(a.perm + j);
      double w[2 * M];
      window_taps<M>(C, pos - fl, w);
#pragma unroll
      for (int i = 0; i < 2 * M; ++i) wl[lane * WS + i] = w[i];
    }
    __syncwarp();
    const int n = min(32, s1 - sb);
    // software pipeline: the F rows of sub-block k+1 are in flight while the
    // taps of sub-block k are accumulated
    double2 fn[kSub];
#pragma unroll
    for (int k = 0; k < kSub; ++k) {
      const int sr = __shfl_sync(0xffffffffu, src, k);
      fn[k] = make_double2(0.0, 0.0);
      if (colok && k < n) fn[k] = __ldg(fcol + (int64_t)sr * a.B);
    }
    for (int s0b = 0; s0b < n; s0b += kSub) {
      double2 fv[kSub];
#pragma unroll
      for (int k = 0; k < kSub; ++k) fv[k] = fn[k];
#pragma unroll
      for (int k = 0; k < kSub; ++k) {
        const int sn = s0b + kSub + k;
        const int sr = __shfl_sync(0xffffffffu, src, sn & 31);
        fn[k] = make_double2(0.0, 0.0);
        if (colok && sn < n) fn[k] = __ldg(fcol + (int64_t)sr * a.B);
      }
#pragma unroll
      for (int k = 0; k < kSub; ++k) {
        if (s0b + k < n) {  // warp-uniform
          const int64_t c = __shfl_sync(0xffffffffu, cl, s0b + k);
          while (ccur < c) spread_flush<M>(a, r, ccur, cell0, cend, col, colok);
          const double* wr = wl + (s0b + k) * WS;
#pragma unroll
          for (int i = 0; i < 2 * M; ++i) {
            const double wi = wr[i];
            r[i].x = fma(fv[k].x, wi, r[i].x);
            r[i].y = fma(fv[k].y, wi, r[i].y);
          }
        }
      }
    }
    __syncwarp();
  }
  while (ccur < cend - 1) spread_flush<M>(a, r, ccur, cell0, cend, col, colok);
#pragma unroll
  for (int i = 0; i < 2 * M; ++i) spread_flush<M>(a, r, ccur, cell0, cend, col, colok);
}

// ----------------------------------------------- warp-specialised spread
// k_spread_bw: the same tile / column decomposition as k_spread_b, rebuilt
// around the TMA engine and static register slots.
//   * one PRODUCER warp per CTA: 32 sources at a time, every lane evaluates
//     one source's window (the next 32 positions / permutation entries are
//     already in flight); then, stage by stage (kWsSrc sources), it writes
//     taps and cells to shared memory and issues one bulk copy (cp.async.bulk,
//     2 KiB = 128 columns) per source row of F into a kWsStages-deep ring,
//     completing on the stage's `full` mbarrier -- no registers hold loads in
//     flight;
//   * four CONSUMER warps (lane = column): the 2m grid points of the current
//     cell live in 2m STATIC register slots, slot(point) = point mod 2m.  The
//     cell loop is unrolled over one period of 2m cells, so every tap
//     addresses its slot at compile time (k_spread_b's shifting window was
//     compiled to ~50 register moves per source: IMAD.MOV 42 % of its
//     instructions); the sources of a cell are an inner loop over the ring.
//     When a cell is finished its lowest point is final and is stored.
// Stage release: each consumer warp arrives on the stage's `empty` mbarrier.
// Measured (config 4, 1.57 ms for k_spread_b): 1.13 ms with 3 stages of 8
// rows, 1.27 ms with 4, 1.51 ms with 6 (2 CTAs per SM); windows evaluated by
// the consumer warps instead (a free-running copy producer): 1.54-1.71 ms;
// with running shared-memory addresses and a running output pointer in the
// consumers (this version): 0.88 ms, 84 % of the spread's HBM roofline.
#ifndef SFB_SPREADB_SRC
#define SFB_SPREADB_SRC 8
#endif
constexpr int kWsSrc = SFB_SPREADB_SRC;  // source rows per stage (2 KiB each)
#ifndef SFB_SPREADB_STAGES
#define SFB_SPREADB_STAGES 3
#endif
#ifndef SFB_SPREADBW_ABL
#define SFB_SPREADBW_ABL 0  // timing ablations (wrong results): 1 no tap FMAs, 2 no bulk copies
#endif
constexpr int kWsStages = SFB_SPREADB_STAGES;
constexpr int kWsConsumers = kThreadsB / 32;
static_assert(32 % kWsSrc == 0, "a producer batch is a whole number of stages");

template <int M>
struct __align__(128) SpreadBwSmem {
  double2 f[kWsStages][kWsSrc][kThreadsB];
  double w[kWsStages][kWsSrc][2 * M];
  int cell[kWsStages][kWsSrc];
  unsigned long long full[kWsStages], empty[kWsStages];
};

// resident CTAs per SM: the 4 m accumulator registers leave room for 3 CTAs up to m = 6
#ifndef SFB_SPREADBW_MINB
#define SFB_SPREADBW_MINB(M) ((M) <= 6 ? 3 : 2)
#endif
template <int M>
__global__ void __launch_bounds__(kThreadsB + 32, SFB_SPREADBW_MINB(M))
    k_spread_bw(SpreadBArgs a, WinCoef C) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<SpreadBwSmem<M>*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int col0 = blockIdx.y * kThreadsB;
  const int ncol = min(kThreadsB, a.B - col0);
  const int cell0 = (int)((int64_t)blockIdx.x * kTileB);
  const int cend = (int)min((int64_t)cell0 + kTileB, a.K);
  const int s0 = a.tile[blockIdx.x], s1 = a.tile[blockIdx.x + 1];
  const int nst = (s1 - s0 + kWsSrc - 1) / kWsSrc;
  if (tid == 0) {
    for (int i = 0; i < kWsStages; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], kWsConsumers);
    }
  }
  __syncthreads();
  if (warp == kWsConsumers) {
    // ------------------------------------------------------------ producer
    const int64_t halfK = a.K / 2;
    const int nsrc = s1 - s0;
    double pos_n = 0.5;
    int src_n = 0;
    if (lane < nsrc) {
      pos_n = __ldg(a.pos + s0 + lane);
      src_n = __ldg(a.perm + s0 + lane);
    }
    for (int jb = 0; jb < nst; jb += 32 / kWsSrc) {
      const double pos = pos_n;
      const int src = src_n;
      const int sb = s0 + jb * kWsSrc;  // first source of this batch
      if (sb + 32 + lane < s1) {
        pos_n = __ldg(a.pos + sb + 32 + lane);
        src_n = __ldg(a.perm + sb + 32 + lane);
      }
      const double fl = floor(pos);
      double w[2 * M];
      window_taps<M>(C, pos - fl, w);
      const int cl = (int)((int64_t)fl + halfK);
#pragma unroll
      for (int g = 0; g < 32 / kWsSrc; ++g) {
        const int j = jb + g;
        if (j < nst) {  // warp-uniform
          const int st = j % kWsStages;
          if (j >= kWsStages) mbar_wait(&S.empty[st], (unsigned)((j / kWsStages - 1) & 1));
          const int n = min(kWsSrc, s1 - (s0 + j * kWsSrc));
          const int l = lane - g * kWsSrc;
          const bool mine = l >= 0 && l < n;
          if (mine) {
#pragma unroll
            for (int i = 0; i < 2 * M; ++i) S.w[st][l][i] = w[i];
            S.cell[st][l] = cl;
          }
          __syncwarp();
#if SFB_SPREADBW_ABL & 2
          if (lane == 0) mbar_arrive(&S.full[st]);
#else
          if (lane == 0) mbar_expect_tx(&S.full[st], (unsigned)(n * ncol * (int)sizeof(double2)));
          __syncwarp();
          SF_BOUNDS(!mine || (src >= 0 && cl >= cell0 && cl < cend));
          if (mine)
            bulk_g2s_tx(&S.f[st][l][0], a.f + (int64_t)src * a.B + col0,
                        (unsigned)(ncol * (int)sizeof(double2)), &S.full[st]);
#endif
        }
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  const bool colok = tid < ncol;
  double2 r[2 * M];
#pragma unroll
  for (int i = 0; i < 2 * M; ++i) r[i] = make_double2(0.0, 0.0);
  // Position in the source stream: source i of the tile, row k = i % kWsSrc
  // of ring slot st (running shared-memory addresses fp / wp / cp, so the
  // inner loop has no index arithmetic); cs = cell of the current, not yet
  // consumed source (INT_MAX when the tile is exhausted).
  const int nsrc = s1 - s0;
  int i = 0, st = 0, cs = 0x7fffffff;
  unsigned par = 0;  // phase parity of slot st's `full` barrier
  const unsigned f0 = smem_u32(&S.f[0][0][tid]), w0 = smem_u32(&S.w[0][0][0]),
                 c0 = smem_u32(&S.cell[0][0]);
  unsigned fp = f0, wp = w0, cp = c0;
  constexpr unsigned kFRow = sizeof(double2) * kThreadsB, kWRow = sizeof(double) * 2 * M;
  auto lds_i = [](unsigned addr) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
  };
  auto lds_d2 = [](unsigned addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
  };
  if (nsrc > 0) {
    mbar_wait(&S.full[0], 0u);
    cs = lds_i(cp);
  }
  auto next = [&]() {
    ++i;
    fp += kFRow, wp += kWRow, cp += 4;
    if ((i % kWsSrc) != 0 && i < nsrc) {
      cs = lds_i(cp);
      return;
    }
    __syncwarp();  // every lane has read this stage
    if (lane == 0) mbar_arrive(&S.empty[st]);
    if (i < nsrc) {
      if (++st == kWsStages) {
        st = 0, par ^= 1u;
        fp = f0, wp = w0, cp = c0;
      }
      mbar_wait(&S.full[st], par);
      cs = lds_i(cp);
    } else {
      cs = 0x7fffffff;
    }
  };
  // cells cell0 .. cend-1, then 2M-1 source-free steps that retire the
  // points still in the slots.  Step ci retires point cell0 + ci + 1 - M:
  // inside the grid for ci in [ci_lo, ci_hi), interior to this tile (plain
  // store) for ci in [2M-1, ncell), shared with a neighbour tile otherwise.
  const int ncell = cend - cell0;
  const int total = ncell + 2 * M - 1;
  const int ci_lo = max(0, M - 1 - cell0);
  const int ci_hi = (int)min((int64_t)total, a.K - cell0 - 1 + M);
  double2* gp = a.grid + ((int64_t)cell0 + 1 - M) * a.B + (col0 + tid);
  for (int base = 0; base < total; base += 2 * M) {
#pragma unroll
    for (int p = 0; p < 2 * M; ++p) {
      const int ci = base + p;
      if (ci < total) {  // warp-uniform
        const int c = cell0 + ci;
        while (cs == c) {
          SF_BOUNDS(i < nsrc && fp >= f0 && fp < f0 + kWsStages * kWsSrc * kFRow &&
                    wp >= w0 && wp < w0 + kWsStages * kWsSrc * kWRow);
#if !(SFB_SPREADBW_ABL & 1)
          const double2 fv = lds_d2(fp);
#pragma unroll
          for (int t = 0; t < M; ++t) {
            const double2 ww = lds_d2(wp + 16 * t);  // taps 2t, 2t+1 (broadcast)
            double2& ra = r[(2 * t + p) % (2 * M)];
            double2& rb = r[(2 * t + 1 + p) % (2 * M)];
            ra.x = fma(fv.x, ww.x, ra.x);
            ra.y = fma(fv.y, ww.x, ra.y);
            rb.x = fma(fv.x, ww.y, rb.x);
            rb.y = fma(fv.y, ww.y, rb.y);
          }
#endif
          next();
        }
        // point cell0 + ci + 1 - M (slot p) is final
        if (colok && ci >= ci_lo && ci < ci_hi) {
          SF_BOUNDS(gp >= a.grid && gp < a.grid + a.K * a.B);
          if (ci >= 2 * M - 1 && ci < ncell) {
            *gp = r[p];  // interior: only this tile touches it
          } else if (r[p].x != 0.0 || r[p].y != 0.0) {
            atomicAdd(&gp->x, r[p].x);
            atomicAdd(&gp->y, r[p].y);
          }
        }
        gp += a.B;
        r[p] = make_double2(0.0, 0.0);
      }
    }
  }
}

// zero the grid rows shared by two tiles (touched with atomics)
__global__ void k_zero_halo(double2* grid, int64_t K, int B, int m, int64_t ntile) {
  const int64_t t = blockIdx.x;
  const int64_t b = min(t * kTileB, K);  // the grid end is a tile boundary too
  for (int64_t p = b - m + 1 + threadIdx.y; p <= b + m - 1; p += blockDim.y) {
    if (p < 0 || p >= K) continue;
    for (int c = threadIdx.x; c < B; c += blockDim.x) grid[p * B + c] = make_double2(0.0, 0.0);
  }
}

// ------------------------------------------------------------------ gather
// (A warp-specialised form in the shape of k_spread_bw -- h rows streamed by
// bulk copies into an mbarrier ring, window tables from a second producer
// warp, 2m static row slots in the consumers -- was measured at config 4:
// 1.61-2.34 ms against 1.10 ms for this kernel, whatever the ring depth, CTAs
// per SM (1-3) or columns per thread (1-2): with one output row per target
// the consumer's per-target chain, not the h traffic, is what binds.  Dropped.)
struct GatherBArgs {
  const double* pos;   // sorted target positions fl(N2 xs)
  const int* perm;
  const double* scale;
  const double2* h;    // [Kout][B]
  double2* out;        // (M2, B) row-major
  int64_t M2, Kout, N2, s_lo;
  int B;
  int per_cta;         // targets per CTA
};

#ifndef SFB_GATHERB_PAIR
#define SFB_GATHERB_PAIR 1
#endif
template <int M>
__global__ void __launch_bounds__(kThreadsB, 4) k_gather_b(GatherBArgs a, WinCoef C) {
  extern __shared__ __align__(16) double wsm[];
  constexpr int WS = 2 * M + 2;  // even: a row is 16-byte aligned, taps read in pairs
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* wl = wsm + warp * 32 * WS;
  const int col = blockIdx.y * blockDim.x + threadIdx.x;
  const bool colok = col < a.B;
  const double2* hcol = a.h + (colok ? col : 0);
  double2* ocol = a.out + col;
  const int64_t j0 = (int64_t)blockIdx.x * a.per_cta;
  const int64_t j1 = min(j0 + a.per_cta, a.M2);
  const int Kout = (int)a.Kout;
  double2 hr[2 * M];
  int kbase = -(1 << 30);  // h rows [kbase, kbase + 2M) are in hr
  auto row = [&](int k) -> double2 {
    int kk = k;
    if (kk < 0 || kk >= Kout) {  // periodic wrap (only when Kout == N2)
      kk %= (int)a.N2;
      if (kk < 0) kk += (int)a.N2;
    }
    SF_BOUNDS(kk >= 0 && kk < Kout);
    return __ldg(hcol + (int64_t)kk * a.B);
  };
  for (int64_t jb = j0; jb < j1; jb += 32) {
    const int64_t j = jb + lane;
    int kl = 0, dst = 0;
    double sc = 0.0;
    if (j < j1) {
      const double pos = __ldg(a.pos + j);
      const double c = floor(pos);
      kl = (int)((int64_t)c + (1 - M) - a.s_lo);
      dst = __ldg(a.perm + j);
      sc = __ldg(a.scale + j);
      double w[2 * M];
      window_taps<M>(C, pos - c, w);
#pragma unroll
      for (int i = 0; i < 2 * M; ++i) wl[lane * WS + i] = w[i];
    }
    __syncwarp();
    const int n = (int)min((int64_t)32, j1 - jb);
    // runs of targets sharing one window start k0: the register window only
    // moves between runs, so the inner loop leaves hr untouched (a window
    // update inside every iteration made ptxas copy all of hr per target)
    const int kprev = __shfl_up_sync(0xffffffffu, kl, 1);
    unsigned starts = __ballot_sync(0xffffffffu, lane == 0 || kl != kprev) & ((n < 32) ? ((1u << n) - 1u) : 0xffffffffu);
    while (starts) {
      const int s0 = __ffs(starts) - 1;
      starts &= starts - 1;
      const int s1 = starts ? __ffs(starts) - 1 : n;
      const int k0 = __shfl_sync(0xffffffffu, kl, s0);
      if (k0 < kbase || k0 >= kbase + 2 * M) {  // (re)load the whole window
#pragma unroll
        for (int i = 0; i < 2 * M; ++i) hr[i] = row(k0 + i);
        kbase = k0;
      } else {
        while (kbase < k0) {  // warp-uniform, < 2M steps
#pragma unroll
          for (int i = 0; i < 2 * M - 1; ++i) hr[i] = hr[i + 1];
          hr[2 * M - 1] = row(kbase + 2 * M);
          ++kbase;
        }
      }
      // the targets of one window start, two at a time (four independent FMA
      // chains per column instead of two)
      auto one = [&](int s) {
        const int d = __shfl_sync(0xffffffffu, dst, s);
        const double scs = __shfl_sync(0xffffffffu, sc, s);
        const double2* wr = reinterpret_cast<const double2*>(wl + s * WS);
        double2 acc = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < M; ++i) {
          const double2 ww = wr[i];  // taps 2i, 2i+1 (broadcast LDS.128)
          acc.x = fma(hr[2 * i].x, ww.x, acc.x);
          acc.y = fma(hr[2 * i].y, ww.x, acc.y);
          acc1.x = fma(hr[2 * i + 1].x, ww.y, acc1.x);
          acc1.y = fma(hr[2 * i + 1].y, ww.y, acc1.y);
        }
        if (colok)
          ocol[(int64_t)d * a.B] = make_double2((acc.x + acc1.x) * scs, (acc.y + acc1.y) * scs);
      };
      int s = s0;
#if SFB_GATHERB_PAIR
      auto many = [&](auto nt_tag) {
        constexpr int NT = decltype(nt_tag)::value;
        int dd[NT];
        double ss[NT];
        const double2* ww[NT];
        double2 ae[NT], ao[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          dd[t] = __shfl_sync(0xffffffffu, dst, s + t);
          ss[t] = __shfl_sync(0xffffffffu, sc, s + t);
          ww[t] = reinterpret_cast<const double2*>(wl + (s + t) * WS);
          ae[t] = ao[t] = make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int i = 0; i < M; ++i) {
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const double2 u = ww[t][i];  // taps 2i, 2i+1 (broadcast LDS.128)
            ae[t].x = fma(hr[2 * i].x, u.x, ae[t].x);
            ae[t].y = fma(hr[2 * i].y, u.x, ae[t].y);
            ao[t].x = fma(hr[2 * i + 1].x, u.y, ao[t].x);
            ao[t].y = fma(hr[2 * i + 1].y, u.y, ao[t].y);
          }
        }
        if (colok) {
#pragma unroll
          for (int t = 0; t < NT; ++t)
            ocol[(int64_t)dd[t] * a.B] =
                make_double2((ae[t].x + ao[t].x) * ss[t], (ae[t].y + ao[t].y) * ss[t]);
        }
        s += NT;
      };
#if SFB_GATHERB_PAIR >= 4
      while (s + 3 < s1) many(std::integral_constant<int, 4>{});
#endif
      while (s + 1 < s1) many(std::integral_constant<int, 2>{});
#endif
      for (; s < s1; ++s) one(s);
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------- transposes
// out[c][r] = in[r][c] for an R x Cc complex matrix (32 x 32 tiles)
__global__ void __launch_bounds__(256) k_transpose(const double2* __restrict__ in,
                                                   double2* __restrict__ out, int64_t R,
                                                   int64_t Cc) {
  __shared__ double2 t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < Cc) t[i][threadIdx.x] = __ldg(in + r * Cc + c);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < Cc) out[c * R + r] = t[threadIdx.x][i];
  }
}

static void transpose(const double2* in, double2* out, int64_t R, int64_t Cc, cudaStream_t s) {
  const dim3 grid((unsigned)ceil_div(Cc, 32), (unsigned)ceil_div(R, 32));
  k_transpose<<<grid, dim3(32, 8), 0, s>>>(in, out, R, Cc);
  SF_LAUNCH_CHECK();
}

// --------------------------------------------------------------- drivers
// SFB_SPREADB_WS=0 selects the round-1 kernel (k_spread_b)
static bool spread_b_ws() {
  static const bool v = [] {
    const char* e = getenv("SFB_SPREADB_WS");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

template <int M>
static void spread_b_m(const NnfftPlanImpl& p, const double2* f, double2* grid, int B,
                       cudaStream_t s) {
  const int64_t ntile = ceil_div(p.g.K, kTileB);
  k_zero_halo<<<(unsigned)(ntile + 1), dim3(32, 8), 0, s>>>(grid, p.g.K, B, M, ntile);
  SF_LAUNCH_CHECK();
  SpreadBArgs a{p.sp.bpos.p, p.sp.bperm.p, p.sp.btile.p, f, grid, p.g.K, B};
  if (spread_b_ws()) {
    const size_t smem = sizeof(SpreadBwSmem<M>);
    static std::atomic<unsigned long long> attr_set{0};  // per template instance, per device
    const unsigned long long bit = 1ull << (p.device & 63);
    if (!(attr_set.load() & bit)) {
      SF_CUDA(cudaFuncSetAttribute(k_spread_bw<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
      attr_set.fetch_or(bit);
    }
    k_spread_bw<M><<<dim3((unsigned)ntile, (unsigned)ceil_div(B, kThreadsB)), kThreadsB + 32, smem,
                     s>>>(a, p.c1);
    SF_LAUNCH_CHECK();
    return;
  }
  const int threads = (int)std::min<int64_t>(kThreadsB, ceil_div(B, 32) * 32);
  const size_t smem = sizeof(double) * (2 * M + 1) * 32 * (threads / 32);
  k_spread_b<M><<<dim3((unsigned)ntile, (unsigned)ceil_div(B, threads)), threads, smem, s>>>(a,
                                                                                             p.c1);
  SF_LAUNCH_CHECK();
}

template <int M>
static void gather_b_m(const NnfftPlanImpl& p, const double2* h, double2* out, int B,
                       cudaStream_t s) {
  static const int per_cta = [] {  // targets per CTA (tuning: SFB_GATHERB_PER_CTA)
    const char* e = getenv("SFB_GATHERB_PER_CTA");
    return e ? std::max(32, atoi(e) / 32 * 32) : 64;
  }();
  GatherBArgs a{p.gp.pos.p, p.gp.perm.p, p.gp.scale.p, h, out, p.g.M2, p.fft.Kout, p.g.N2,
                p.fft.s_lo, B, per_cta};
  const int threads = (int)std::min<int64_t>(kThreadsB, ceil_div(B, 32) * 32);
  const size_t smem = sizeof(double) * (2 * M + 2) * 32 * (threads / 32);
  k_gather_b<M><<<dim3((unsigned)ceil_div(p.g.M2, per_cta), (unsigned)ceil_div(B, threads)),
                  threads, smem, s>>>(a, p.c2);
  SF_LAUNCH_CHECK();
}

#define SF_DISPATCH(m, FN, ...)                                                         \
  switch (m) {                                                                          \
    case 2: FN<2>(__VA_ARGS__); break;                                                  \
    case 3: FN<3>(__VA_ARGS__); break;                                                  \
    case 4: FN<4>(__VA_ARGS__); break;                                                  \
    case 5: FN<5>(__VA_ARGS__); break;                                                  \
    case 6: FN<6>(__VA_ARGS__); break;                                                  \
    case 7: FN<7>(__VA_ARGS__); break;                                                  \
    case 8: FN<8>(__VA_ARGS__); break;                                                  \
    case 9: FN<9>(__VA_ARGS__); break;                                                  \
    case 10: FN<10>(__VA_ARGS__); break;                                                \
    case 11: FN<11>(__VA_ARGS__); break;                                                \
    case 12: FN<12>(__VA_ARGS__); break;                                                \
    case 13: FN<13>(__VA_ARGS__); break;                                                \
    case 14: FN<14>(__VA_ARGS__); break;                                                \
    case 15: FN<15>(__VA_ARGS__); break;                                                \
    case 16: FN<16>(__VA_ARGS__); break;                                                \
    default: fail(5, "unsupported window cut-off");                                     \
  }

void run_execute_batched(const NnfftPlanImpl& p, const double2* f, double2* out, int B,
                         cudaStream_t s, cudaEvent_t* ev) {
  const int64_t K = p.g.K, Ko = p.fft.Kout;
  Scratch gp(sizeof(double2) * (size_t)K * B, s);   // [K][B]
  const bool pm = fft_supports_point_major(p);
  Scratch gc(pm ? 0 : sizeof(double2) * (size_t)K * B, s);   // [B][K]
  Scratch work(sizeof(double2) * (size_t)p.fft.work_elems() * (pm ? fft_point_major_group(B) : B), s);
  Scratch hc(pm ? 0 : sizeof(double2) * (size_t)Ko * B, s);  // [B][Kout]
  Scratch hp(sizeof(double2) * (size_t)Ko * B, s);  // [Kout][B]
  if (ev) SF_CUDA(cudaEventRecord(ev[0], s));
  SF_DISPATCH(p.g.m1, spread_b_m, p, f, gp.as<double2>(), B, s);
  if (ev) SF_CUDA(cudaEventRecord(ev[1], s));
  if (fft_supports_point_major(p)) {
    run_fft_point_major(p, gp.as<double2>(), hp.as<double2>(), work.as<double2>(), B, s);
  } else {
    transpose(gp.as<double2>(), gc.as<double2>(), K, B, s);
    run_fft(p, gc.as<double2>(), hc.as<double2>(), work.as<double2>(), B, s);
    transpose(hc.as<double2>(), hp.as<double2>(), B, Ko, s);
  }
  if (ev) SF_CUDA(cudaEventRecord(ev[2], s));
  SF_DISPATCH(p.g.m2, gather_b_m, p, hp.as<double2>(), out, B, s);
  if (ev) SF_CUDA(cudaEventRecord(ev[3], s));
}

}  // namespace sfb
