// spread.cu -- step 1 of Algorithm 2.1: spread the M1 frequency nodes onto the
// K = N1 + 2 m1 point grid with the first window.
//
// Reference (pkg/src/sincfft/nnfft.py:188-196, 229-233):
//     g[c_k + t + K/2] += f_k phi_1((c_k + t)/N1 - v_k),  c_k = floor(N1 v_k),
//     t = 1-m1 .. m1, then g /= N1 (folded into the Bluestein pre-chirp).
// The reference scatters with two np.bincount passes over an M1 x 2m1 table.
//
// B200 design (no global atomics per tap, no shared-memory fp64 atomics --
// those are CAS loops on sm_100a):
//   * sources are sorted by cell at plan time and cut into chunks of <= 4
//     sources of ONE cell; a lane owns a chunk and accumulates its 2m taps in
//     registers (window from the per-tap polynomials, window.cuh);
//   * chunks come in blocks of 32 (one per lane) of one 256-cell tile; the
//     kernel is persistent and every warp is an independent worker over a
//     contiguous range of blocks, with a private shared-memory accumulator
//     for its current tile (plus halo) that it flushes with one fp64 RED per
//     touched grid point (REDG.ADD.F64, native on sm_100a) when the tile
//     changes -- a tile is flushed by the one or two warps that cover it;
//   * lanes with equal cells in one block (rare by the rank-major chunk
//     order) are serialised by __match_any_sync rounds;
//   * the loads are a cp.async pipeline into per-warp shared-memory rings:
//     block descriptors (positions, permutation, counts) two blocks ahead and
//     the random 16-byte f gather one block ahead, so the f latency (the
//     spread's floor: ~97 DRAM bytes per 16-byte read at config 3, see
//     tools/randread.cu) overlaps a whole block of window arithmetic and no
//     registers are held for prefetching.
#include "nnfft_impl.cuh"

#include <atomic>
#include <type_traits>

namespace sfb {

struct SpreadArgs {
  const double* pos;     // slot order, [n_blocks * 32 * 4]
  const int* perm;       // slot order
  const int* info;       // per chunk
  const int* blk_tile;   // per block
  const int64_t* wstart; // first block of each warp
  const void* f;         // complex (M1, batch) row-major, or real (M1)
  double2* grid;         // [batch][K]
  int64_t K, n_blocks;
  int batch;
};

static_assert(kChunk == 4, "slot records assume 4 sources per chunk");
static_assert(kBlockChunks == 32, "one chunk per lane");

#ifndef SFB_SPREAD_HINT
#define SFB_SPREAD_HINT 0  // L2 hint bits: 1 descriptors evict-first, 2 f evict-last, 4 f evict-first
#endif
#ifndef SFB_SPREAD_F64B
#define SFB_SPREAD_F64B 1  // f gather with the .L2::64B fill size
#endif
constexpr int kDescStages = 3;  // descriptor ring depth (blocks)
constexpr int kFStages = 2;     // f ring depth (blocks)

// per-warp shared-memory state; slot-major so every lane access is a
// conflict-free consecutive 16-byte (or 8/4-byte) record
template <int M, bool REAL>
struct WarpSmem {
  using FT = typename std::conditional<REAL, double, double2>::type;
  static constexpr int SPAN = kTile + 2 * M - 1;
  double2 acc[SPAN];
  double2 pos[kDescStages][2][32];  // slots {0,1}, {2,3}
  int4 perm[kDescStages][32];
  int info[kDescStages][32];
  FT f[kFStages][kChunk][32];
};

template <bool REAL, class W>
__device__ __forceinline__ void issue_desc(const SpreadArgs& a, W& S, int64_t b, int64_t b1,
                                           int st, int lane) {
  if (b < b1) {
    const int64_t ci = b * kBlockChunks + lane;
#if SFB_SPREAD_HINT & 1  // streaming descriptors: evict-first
    const unsigned long long pol = l2_policy_first();
    cp_async16_pol(&S.pos[st][0][lane], a.pos + ci * kChunk, pol);
    cp_async16_pol(&S.pos[st][1][lane], a.pos + ci * kChunk + 2, pol);
    cp_async16_pol(&S.perm[st][lane], a.perm + ci * kChunk, pol);
#else
    cp_async16(&S.pos[st][0][lane], a.pos + ci * kChunk);
    cp_async16(&S.pos[st][1][lane], a.pos + ci * kChunk + 2);
    cp_async16(&S.perm[st][lane], a.perm + ci * kChunk);
#endif
    cp_async4(&S.info[st][lane], a.info + ci);
  }
  cp_async_commit();
}

template <bool REAL, class W>
__device__ __forceinline__ void issue_f(const SpreadArgs& a, W& S, bool live, int st_d, int st_f,
                                        int col, int lane) {
  if (live) {
    const int cnt = S.info[st_d][lane] & 255;
    const int4 pm = S.perm[st_d][lane];
    SF_BOUNDS(cnt <= kChunk && pm.x >= 0 && pm.y >= 0 && pm.z >= 0 && pm.w >= 0);
    const int src[kChunk] = {pm.x, pm.y, pm.z, pm.w};
#pragma unroll
    for (int s = 0; s < kChunk; ++s) {
      if (REAL) {
        const double* fp = static_cast<const double*>(a.f) + (s < cnt ? src[s] : 0);
        cp_async8z(&S.f[st_f][s][lane], fp, s < cnt ? 8 : 0);
      } else {
        const double2* fp =
            static_cast<const double2*>(a.f) + (s < cnt ? (int64_t)src[s] * a.batch + col : 0);
#if SFB_SPREAD_HINT & 2  // f: evict-last (its 64-byte neighbours are other sources)
        cp_async16z_pol(&S.f[st_f][s][lane], fp, s < cnt ? 16 : 0, l2_policy_last());
#elif SFB_SPREAD_HINT & 4
        cp_async16z_pol(&S.f[st_f][s][lane], fp, s < cnt ? 16 : 0, l2_policy_first());
#elif SFB_SPREAD_F64B
        cp_async16z_l2_64(&S.f[st_f][s][lane], fp, s < cnt ? 16 : 0);
#else
        cp_async16z(&S.f[st_f][s][lane], fp, s < cnt ? 16 : 0);
#endif
      }
    }
  }
  cp_async_commit();
}

template <int M, class W>
__device__ __forceinline__ void flush_tile(const SpreadArgs& a, W& S, int tile, int col,
                                           int lane) {
  constexpr int SPAN = W::SPAN;
  double2* grid = a.grid + (int64_t)col * a.K;
  const int64_t base = (int64_t)tile * kTile - (M - 1);  // grid index of slot 0
  __syncwarp();
  for (int p = lane; p < SPAN; p += 32) {
    const double2 t = S.acc[p];
    const int64_t gi = base + p;
    if (gi >= 0 && gi < a.K && (t.x != 0.0 || t.y != 0.0)) {
      atomicAdd(&grid[gi].x, t.x);
      atomicAdd(&grid[gi].y, t.y);
    }
    S.acc[p] = make_double2(0.0, 0.0);
  }
  __syncwarp();
}

#ifndef SFB_SPREAD_PM
#define SFB_SPREAD_PM 0
#endif
#ifndef SFB_SPREAD_ABL
#define SFB_SPREAD_ABL 0  // timing ablations (wrong results): 1 no accumulate rounds, 2 no window polynomials
#endif
// Pair-major form of one block (SFB_SPREAD_PM): a lane's NS (2 or 4) sources
// are evaluated together, tap pair by tap pair -- every coefficient (a
// uniform constant-bank load) feeds NS Horner chains instead of 2 -- and each
// pair's two taps are added into the tile accumulator as soon as they are
// formed, so no 2m-tap register array is held (~40 fewer registers).  Lanes
// of one cell are serialised by rounds computed once per block (rank among
// the lanes with that cell); the hi and lo taps of one pair are added in two
// steps, so lanes of different cells never touch one slot in the same step.
__device__ __forceinline__ double2 as_c(double2 v) { return v; }
__device__ __forceinline__ double2 as_c(double v) { return make_double2(v, 0.0); }
template <int M, bool REAL, int NS, class FT>
__device__ __forceinline__ void pm_block(const WinCoef& C, const double* pp, const FT* fs,
                                         int lane, int cnt, int lcell, double2* acc) {
  constexpr int P = window_degree(M);
  constexpr int NE = P / 2 + 1;
  constexpr int NO = (P + 1) / 2;
  double u[NS];
  double2 fv[NS];
  VPow vw[NS];
#pragma unroll
  for (int t = 0; t < NS; ++t) {
    const double d = pp[t] - floor(pp[t]);
    u[t] = 2.0 * d - 1.0;
    vw[t] = vpowers(u[t] * u[t]);
    fv[t] = as_c(fs[32 * t + lane]);
  }
  int same = 0;
  __match_all_sync(0xffffffffu, cnt > 0 ? lcell : -1 - lane, &same);
  const unsigned peers = __match_any_sync(0xffffffffu, cnt > 0 ? lcell : (0x40000000 | lane));
  const int myround = cnt > 0 ? __popc(peers & ((1u << lane) - 1u)) : -1;
  const int nrounds = same ? 1 : __reduce_max_sync(0xffffffffu, (unsigned)(myround + 1));
#pragma unroll
  for (int q = 0; q < M; ++q) {
    double hr = 0.0, hm = 0.0, lr = 0.0, lm = 0.0;
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const double E = poly<NE>(C.e[q], vw[t]);
      const double O = poly<NO>(C.o[q], vw[t]);
      double hi = fma(u[t], O, E), lo = fma(-u[t], O, E);
      if (q == M - 1) {
        const double d = pp[t] - floor(pp[t]);
        hi *= sqrt(d);
        lo *= sqrt(1.0 - d);
      }
      hr = fma(fv[t].x, hi, hr);
      lr = fma(fv[t].x, lo, lr);
      if (!REAL) {
        hm = fma(fv[t].y, hi, hm);
        lm = fma(fv[t].y, lo, lm);
      }
    }
    const int ih = (q < M - 1) ? M + q : 2 * M - 1;
    const int il = (q < M - 1) ? M - 1 - q : 0;
    if (same) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        hr += __shfl_xor_sync(0xffffffffu, hr, o);
        lr += __shfl_xor_sync(0xffffffffu, lr, o);
        if (!REAL) {
          hm += __shfl_xor_sync(0xffffffffu, hm, o);
          lm += __shfl_xor_sync(0xffffffffu, lm, o);
        }
      }
      if (lane == 0) {
        double2 t = acc[lcell + ih];
        t.x += hr, t.y += hm;
        acc[lcell + ih] = t;
        t = acc[lcell + il];
        t.x += lr, t.y += lm;
        acc[lcell + il] = t;
      }
      continue;
    }
    for (int r = 0; r < nrounds; ++r) {
      if (myround == r) {
        double2 t = acc[lcell + ih];
        t.x += hr, t.y += hm;
        acc[lcell + ih] = t;
      }
      __syncwarp();
      if (myround == r) {
        double2 t = acc[lcell + il];
        t.x += lr, t.y += lm;
        acc[lcell + il] = t;
      }
      __syncwarp();
    }
  }
  __syncwarp();
}

template <int M, bool REAL>
#ifndef SFB_SPREAD_MINB
#define SFB_SPREAD_MINB 2  // resident CTAs per SM (registers <= 65536 / (32 warps * MINB))
#endif
__global__ void __launch_bounds__(kSpreadWarps * 32, SFB_SPREAD_MINB) k_spread(SpreadArgs a,
                                                                             WinCoef C) {
  using W = WarpSmem<M, REAL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  W& S = reinterpret_cast<W*>(smem_raw)[warp];
  const int col = blockIdx.y;
  // contiguous, cost-balanced block range of this warp (plan time)
  const int64_t gw = (int64_t)blockIdx.x * kSpreadWarps + warp;
  const int64_t b0 = a.wstart[gw], b1 = a.wstart[gw + 1];
  if (b0 >= b1) return;
  for (int p = lane; p < W::SPAN; p += 32) S.acc[p] = make_double2(0.0, 0.0);

  // prologue: descriptors of blocks b0, b0+1; f of block b0
  issue_desc<REAL>(a, S, b0, b1, 0, lane);
  issue_desc<REAL>(a, S, b0 + 1, b1, 1, lane);
  cp_async_wait<1>();
  issue_f<REAL>(a, S, true, 0, 0, col, lane);
  int tile = -1;
  int next_tile = __ldg(a.blk_tile + b0);
  for (int64_t b = b0; b < b1; ++b) {
    const int i = (int)(b - b0);
    const int sd = i % kDescStages, sf = i & 1;
    issue_desc<REAL>(a, S, b + 2, b1, (i + 2) % kDescStages, lane);
    cp_async_wait<2>();  // descriptors of b+1 have landed
    issue_f<REAL>(a, S, b + 1 < b1, (i + 1) % kDescStages, (i + 1) & 1, col, lane);
    const int btile = next_tile;
    if (b + 1 < b1) next_tile = __ldg(a.blk_tile + b + 1);
    SF_BOUNDS(btile >= 0 && (int64_t)btile * kTile < a.K + kTile);
    if (btile != tile) {
      if (tile >= 0) flush_tile<M>(a, S, tile, col, lane);
      tile = btile;
    }
    cp_async_wait<2>();  // f of b has landed
    const int info = S.info[sd][lane];
    const int cnt = info & 255;
    const int lcell = info >> 8;
    const double2 p01 = S.pos[sd][0][lane], p23 = S.pos[sd][1][lane];
#if SFB_SPREAD_PM
    {
      // padding slots have f = 0 and a harmless position; a block where no
      // lane holds more than 2 sources runs the 2-source form
      const double pp[4] = {p01.x, p01.y, p23.x, p23.y};
      const auto* fs = &S.f[sf][0][0];
      if (__any_sync(0xffffffffu, cnt > 2))
        pm_block<M, REAL, 4>(C, pp, fs, lane, cnt, lcell, S.acc);
      else
        pm_block<M, REAL, 2>(C, pp, fs, lane, cnt, lcell, S.acc);
      continue;
    }
#endif
    double2 r[2 * M];
#pragma unroll
    for (int k = 0; k < 2 * M; ++k) r[k] = make_double2(0.0, 0.0);
#if SFB_SPREAD_ABL & 2  // timing ablation: f values as taps, no polynomials
    if (cnt > 0 && !REAL) {
      const double2* fs = reinterpret_cast<const double2*>(&S.f[sf][0][0]);
#pragma unroll
      for (int k = 0; k < 2 * M; ++k) {
        r[k].x = fs[lane + 32 * (k & 3)].x * p01.x;
        r[k].y = fs[lane + 32 * (k & 3)].y * p23.y;
      }
    } else
#endif
    if (cnt > 0) {
      if (REAL) {
        const double* fs = reinterpret_cast<const double*>(&S.f[sf][0][0]);
        window_accumulate2<M, true>(C, p01.x - floor(p01.x), make_double2(fs[lane], 0.0),
                                    p01.y - floor(p01.y), make_double2(fs[32 + lane], 0.0), r);
        if (cnt > 2)
          window_accumulate2<M, true>(C, p23.x - floor(p23.x), make_double2(fs[64 + lane], 0.0),
                                      p23.y - floor(p23.y), make_double2(fs[96 + lane], 0.0), r);
      } else {
        const double2* fs = reinterpret_cast<const double2*>(&S.f[sf][0][0]);
        // a padding slot has f = 0 (zero-filled) and a harmless position, so
        // pairs may run with a dead second node
        window_accumulate2<M, false>(C, p01.x - floor(p01.x), fs[lane], p01.y - floor(p01.y),
                                     fs[32 + lane], r);
        if (cnt > 2)
          window_accumulate2<M, false>(C, p23.x - floor(p23.x), fs[64 + lane],
                                       p23.y - floor(p23.y), fs[96 + lane], r);
      }
    }
    // add into the warp-private tile accumulator.  A block whose 32 chunks
    // all share one cell (the densest cells of clustered inputs: thousands of
    // sources in one cell) is summed across lanes first (butterfly) and added
    // once; otherwise equal cells in one block would race, so leaders of each
    // cell group go first, round by round (rarely more than one round)
#if SFB_SPREAD_ABL & 1  // timing ablation (wrong results): plain stores, no rounds
    if (cnt > 0) {
#pragma unroll
      for (int k = 0; k < 2 * M; ++k) S.acc[lcell + k] = r[k];
    }
    __syncwarp();
    continue;
#endif
    int same = 0;
    __match_all_sync(0xffffffffu, cnt > 0 ? lcell : -1 - lane, &same);
    if (same) {
#pragma unroll
      for (int k = 0; k < 2 * M; ++k) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          r[k].x += __shfl_xor_sync(0xffffffffu, r[k].x, o);
          r[k].y += __shfl_xor_sync(0xffffffffu, r[k].y, o);
        }
      }
      if (lane == 0) {
        SF_BOUNDS(lcell >= 0 && lcell + 2 * M - 1 < W::SPAN);
#pragma unroll
        for (int k = 0; k < 2 * M; ++k) {
          double2 t = S.acc[lcell + k];
          t.x += r[k].x;
          t.y += r[k].y;
          S.acc[lcell + k] = t;
        }
      }
      __syncwarp();
      continue;
    }
    unsigned pending = __ballot_sync(0xffffffffu, cnt > 0);
    while (pending) {
      const bool mine = (pending >> lane) & 1u;
      const unsigned peers = __match_any_sync(0xffffffffu, mine ? lcell : (0x40000000 | lane));
      const bool leader = mine && ((__ffs(peers) - 1) == lane);
#pragma unroll
      for (int k = 0; k < 2 * M; ++k) {
        if (leader) {
          SF_BOUNDS(lcell >= 0 && lcell + k < W::SPAN);
          double2 t = S.acc[lcell + k];
          t.x += r[k].x;
          t.y += r[k].y;
          S.acc[lcell + k] = t;
        }
        __syncwarp();
      }
      pending &= ~__ballot_sync(0xffffffffu, leader);
    }
  }
  cp_async_wait<0>();
  flush_tile<M>(a, S, tile, col, lane);
}

// Small inputs (a few hundred blocks: configs 1 and 2, the 16,385 Chebyshev
// sources of fast-sinc stage 3): the persistent pipeline leaves most SMs idle
// and each warp pays its full load-latency chain for one block.  Here one
// thread per source slot evaluates its 2m taps and adds them to the grid with
// fp64 REDs (L2-resident grid; contention only at the densest cells).
template <int M, bool REAL>
__global__ void __launch_bounds__(256) k_spread_small(SpreadArgs a, WinCoef C) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // slot
  const int col = blockIdx.y;
  // whole warps only (the slot count is a multiple of 128): the 4 slots of a
  // chunk are 4 consecutive lanes and take part in the shuffles below
  if (s >= a.n_blocks * kBlockChunks * kChunk) return;
  const int64_t ci = s / kChunk;
  const int info = __ldg(a.info + ci);
  const int cnt = info & 255;
  const bool act = (int)(s % kChunk) < cnt;
  double2 r[2 * M];
#pragma unroll
  for (int k = 0; k < 2 * M; ++k) r[k] = make_double2(0.0, 0.0);
  if (act) {
    const double pos = __ldg(a.pos + s);
    const int src = __ldg(a.perm + s);
    double2 fv;
    if (REAL) fv = make_double2(__ldg(static_cast<const double*>(a.f) + src), 0.0);
    else fv = __ldg(static_cast<const double2*>(a.f) + (int64_t)src * a.batch + col);
    window_accumulate<M, REAL>(C, pos - floor(pos), fv, r);
  }
  // a chunk's sources share one cell: sum its 4 lanes' taps first, so only
  // one lane per chunk issues the fp64 REDs (the Chebyshev sources of
  // fast-sinc stage 3 pile hundreds into the end cells)
#pragma unroll
  for (int k = 0; k < 2 * M; ++k) {
    r[k].x += __shfl_xor_sync(0xffffffffu, r[k].x, 1);
    r[k].x += __shfl_xor_sync(0xffffffffu, r[k].x, 2);
    if (!REAL) {
      r[k].y += __shfl_xor_sync(0xffffffffu, r[k].y, 1);
      r[k].y += __shfl_xor_sync(0xffffffffu, r[k].y, 2);
    }
  }
  if ((s % kChunk) != 0 || cnt == 0) return;
  const int lcell = info >> 8;
  const int tile = __ldg(a.blk_tile + ci / kBlockChunks);
  double2* grid = a.grid + (int64_t)col * a.K;
  const int64_t base = (int64_t)tile * kTile - (M - 1) + lcell;  // as flush_tile
#pragma unroll
  for (int k = 0; k < 2 * M; ++k) {
    const int64_t gi = base + k;
    if (gi >= 0 && gi < a.K) {
      atomicAdd(&grid[gi].x, r[k].x);
      if (!REAL) atomicAdd(&grid[gi].y, r[k].y);
    }
  }
}

// Dense sources (hundreds per cell: fast-sinc stage 1 puts 2^22 sources on
// 8,224 cells).  Every tap is a polynomial in u = 2d - 1 (window.cuh), so the
// sum over a cell's sources of f * g_t(d) is a fixed combination of the
// cell's moments  S_j = sum f u^j,  S'_j = sum f sqrt(d) u^j,
// S''_j = sum f sqrt(1-d) u^j  (j <= P; the primed sets feed the two edge
// taps): 1 multiply + 3 FMAs per power and source instead of ~160 fp64 ops
// per source for the 2m tap polynomials.  Cells are cut into plan-time units
// of <= kDenseUnit sources (heavy cells of clustered inputs spread over many
// units); a group of kDenseLanes lanes owns a unit, sums its moments over the
// group by shuffles, forms the 2m taps from the uniform coefficients and adds
// them to the grid with one fp64 RED per tap.  Complex f runs the moments
// once per component.  Fast-sinc stage 1 (config 5, ~510 sources per cell):
// 82 us for the per-source spread, 79 us for a warp per cell (the 42-moment
// butterflies cost as much as the sources), 50 us with 2 lanes x 64 sources
// per unit and the next batch's loads in flight (measured over lanes 1-16 and
// units 16-512).
struct DenseArgs {
  const double* pos;   // fl(N1 v), cell-sorted
  const int* perm;     // cell-sorted
  const int4* units;   // {cell, first, end, 0}
  const void* f;
  double2* grid;
  int64_t K, n_units;
  int batch;
};

#ifndef SFB_DENSE_LANES
#define SFB_DENSE_LANES 2
#endif
constexpr int kDenseLanes = SFB_DENSE_LANES;  // lanes per unit
#ifndef SFB_DENSE_G
#define SFB_DENSE_G 2
#endif
#ifndef SFB_DENSE_FAST_SQRT
#define SFB_DENSE_FAST_SQRT 1  // edge-tap square roots from the rsqrt seed + one step (window.cuh)
#endif

template <int M, bool REAL>
#ifndef SFB_DENSE_MINB
#define SFB_DENSE_MINB 2
#endif
__global__ void __launch_bounds__(256, SFB_DENSE_MINB) k_spread_dense(DenseArgs a, WinCoef C) {
  constexpr int P = window_degree(M);
  constexpr int NE = P / 2 + 1;
  constexpr int NO = (P + 1) / 2;
  constexpr int L = kDenseLanes, G = SFB_DENSE_G;  // G sources per lane per load batch
  const int lane = threadIdx.x & 31;
  const int gl = lane % L;
  const int64_t un_i = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * (32 / L) + lane / L;
  const int col = blockIdx.y;
  if (((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * (32 / L) >= a.n_units) return;
  int4 un = make_int4(0, 0, 0, 0);  // inactive groups: empty unit
  if (un_i < a.n_units) un = __ldg(a.units + un_i);
  const int64_t cell = un.x;
  const int s0 = un.y, s1 = un.z;
  double2* grid = a.grid + (int64_t)col * a.K;
#pragma unroll 1
  for (int comp = 0; comp < (REAL ? 1 : 2); ++comp) {
    double m0[P + 1], m1[P + 1], m2[P + 1];
#pragma unroll
    for (int j = 0; j <= P; ++j) m0[j] = m1[j] = m2[j] = 0.0;
    // G sources per lane at a time, software-pipelined: the f loads of batch
    // g and the position / permutation loads of batch g + 1 are in flight
    // together, then batch g's arithmetic
    double pv[G];
    int src[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int s = s0 + gl + L * i;
      pv[i] = s < s1 ? __ldg(a.pos + s) : 0.5;
      src[i] = s < s1 ? __ldg(a.perm + s) : -1;
    }
#pragma unroll 1
    for (int g = 0;; g += G) {
      if (__all_sync(0xffffffffu, s0 + L * g >= s1)) break;
      double fr[G];
#pragma unroll
      for (int i = 0; i < G; ++i) {
        fr[i] = 0.0;
        if (src[i] >= 0) {
          if (REAL) {
            fr[i] = __ldg(static_cast<const double*>(a.f) + src[i]);
          } else {
            const double* fp = reinterpret_cast<const double*>(static_cast<const double2*>(a.f) +
                                                               (int64_t)src[i] * a.batch + col);
            fr[i] = __ldg(fp + comp);
          }
        }
      }
      double pn[G];
      int sn[G];
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int s = s0 + gl + L * (g + G + i);
        pn[i] = s < s1 ? __ldg(a.pos + s) : 0.5;
        sn[i] = s < s1 ? __ldg(a.perm + s) : -1;
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const double pos = pv[i], fv = fr[i];
        const double d = pos - floor(pos);
        const double u = 2.0 * d - 1.0;
        const double fb = fv * edge_sqrt<M, SFB_DENSE_FAST_SQRT != 0>(d),
                     fc = fv * edge_sqrt<M, SFB_DENSE_FAST_SQRT != 0>(1.0 - d);
        double pw = 1.0;
#pragma unroll
        for (int j = 0; j <= P; ++j) {
          m0[j] = fma(fv, pw, m0[j]);
          m1[j] = fma(fb, pw, m1[j]);
          m2[j] = fma(fc, pw, m2[j]);
          pw *= u;
        }
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        pv[i] = pn[i];
        src[i] = sn[i];
      }
    }
#pragma unroll
    for (int j = 0; j <= P; ++j) {
#pragma unroll
      for (int o = 1; o < L; o <<= 1) {
        m0[j] += __shfl_xor_sync(0xffffffffu, m0[j], o);
        m1[j] += __shfl_xor_sync(0xffffffffu, m1[j], o);
        m2[j] += __shfl_xor_sync(0xffffffffu, m2[j], o);
      }
    }
    // tap pair q: g_{q+1} = E + uO and g_{-q} = E - uO (edge pair: times
    // sqrt(d), sqrt(1-d)), so sum f g = sum_k e_k S_2k +- o_k S_2k+1; lane gl
    // of the group adds taps gl, gl + L, ...
#pragma unroll
    for (int q = 0; q < M; ++q) {
      const double* ma = q < M - 1 ? m0 : m1;
      const double* mb = q < M - 1 ? m0 : m2;
      double ea = 0.0, oa = 0.0, eb = 0.0, ob = 0.0;
#pragma unroll
      for (int k = 0; k < NE; ++k) {
        ea = fma(C.e[q][k], ma[2 * k], ea);
        eb = fma(C.e[q][k], mb[2 * k], eb);
      }
#pragma unroll
      for (int k = 0; k < NO; ++k) {
        oa = fma(C.o[q][k], ma[2 * k + 1], oa);
        ob = fma(C.o[q][k], mb[2 * k + 1], ob);
      }
      const int ih = (q < M - 1) ? M + q : 2 * M - 1;
      const int il = (q < M - 1) ? M - 1 - q : 0;
      const double th = ea + oa, tl = eb - ob;
      if (s0 < s1 && (ih % L) == gl) {
        const int64_t gi = cell - (M - 1) + ih;
        if (gi >= 0 && gi < a.K && th != 0.0) atomicAdd(reinterpret_cast<double*>(grid + gi) + comp, th);
      }
      if (s0 < s1 && (il % L) == gl) {
        const int64_t gi = cell - (M - 1) + il;
        if (gi >= 0 && gi < a.K && tl != 0.0) atomicAdd(reinterpret_cast<double*>(grid + gi) + comp, tl);
      }
    }
  }
}

static int64_t small_spread_blocks() {
  static const int64_t v = [] {
    const char* e = getenv("SFB_SPREAD_SMALL_MAX");
    return e ? (int64_t)atoll(e) : (int64_t)512;
  }();
  return v;
}

template <int M, bool REAL>
static void launch_spread_m(const NnfftPlanImpl& p, const void* f, double2* grid, int batch,
                            cudaStream_t s) {
  if (p.sp.n_blocks == 0) return;
  const size_t smem = sizeof(WarpSmem<M, REAL>) * kSpreadWarps;
  static std::atomic<unsigned long long> attr_set{0};  // per template instance, per device
  const unsigned long long bit = 1ull << (p.device & 63);
  if (!(attr_set.load() & bit)) {
    SF_CUDA(cudaFuncSetAttribute(k_spread<M, REAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr_set.fetch_or(bit);
  }
  if (p.sp.dense) {
    DenseArgs d{p.sp.bpos.p, p.sp.bperm.p, p.sp.units.p, f, grid, p.g.K, p.sp.n_units, batch};
    if (p.sp.n_units == 0) return;
    k_spread_dense<M, REAL>
        <<<dim3((unsigned)ceil_div(ceil_div(p.sp.n_units, (int64_t)(32 / kDenseLanes)) * 32,
                                   (int64_t)256),
                batch),
           256, 0, s>>>(d, p.c1);
    SF_LAUNCH_CHECK();
    return;
  }
  SpreadArgs a{p.sp.pos.p, p.sp.perm.p, p.sp.info.p, p.sp.blk_tile.p, p.sp.wstart.p, f, grid,
               p.g.K, p.sp.n_blocks, batch};
  if (p.sp.n_blocks <= small_spread_blocks()) {
    const int64_t slots = p.sp.n_blocks * kBlockChunks * kChunk;
    k_spread_small<M, REAL><<<dim3((unsigned)ceil_div(slots, (int64_t)256), batch), 256, 0, s>>>(
        a, p.c1);
    SF_LAUNCH_CHECK();
    return;
  }
  // persistent: n_ctas = min(2 per SM, blocks / 32) CTAs, warp ranges from the plan
  k_spread<M, REAL><<<dim3((unsigned)p.sp.n_ctas, batch), kSpreadWarps * 32, smem, s>>>(a, p.c1);
  SF_LAUNCH_CHECK();
}

template <bool REAL>
static void launch_spread(const NnfftPlanImpl& p, const void* f, double2* grid, int batch,
                          cudaStream_t s, bool zero = true) {
  if (zero) SF_CUDA(cudaMemsetAsync(grid, 0, sizeof(double2) * (size_t)p.g.K * batch, s));
  switch (p.g.m1) {
#define SF_CASE(MM) \
  case MM:          \
    return launch_spread_m<MM, REAL>(p, f, grid, batch, s);
    SF_CASE(2) SF_CASE(3) SF_CASE(4) SF_CASE(5) SF_CASE(6) SF_CASE(7) SF_CASE(8) SF_CASE(9)
    SF_CASE(10) SF_CASE(11) SF_CASE(12) SF_CASE(13) SF_CASE(14) SF_CASE(15) SF_CASE(16)
#undef SF_CASE
  }
  fail(5, "unsupported m1");
}

void run_spread(const NnfftPlanImpl& p, const double2* f, double2* grid, int batch,
                cudaStream_t s) {
  launch_spread<false>(p, f, grid, batch, s);
}

// the two halves of run_spread, for per-kernel timing (capi.cu: the profiled
// execute records its first event between them)
void run_spread_zero(const NnfftPlanImpl& p, double2* grid, int batch, cudaStream_t s) {
  SF_CUDA(cudaMemsetAsync(grid, 0, sizeof(double2) * (size_t)p.g.K * batch, s));
}
void run_spread_kernel(const NnfftPlanImpl& p, const double2* f, double2* grid, int batch,
                       cudaStream_t s) {
  launch_spread<false>(p, f, grid, batch, s, false);
}

void run_spread_real(const NnfftPlanImpl& p, const double* f, double2* grid, cudaStream_t s) {
  launch_spread<true>(p, f, grid, 1, s);
}

}  // namespace sfb
