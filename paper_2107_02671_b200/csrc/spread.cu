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
//   * a CTA owns a work unit (<= 1024 chunks of one 256-cell tile); each warp
//     has a private shared-memory accumulator for the tile plus halo and adds
//     its lanes' registers there; lanes with equal cells (rare by the
//     rank-major chunk order) are serialised by __match_any_sync rounds;
//   * warps' accumulators are summed and flushed with one fp64 RED per grid
//     point (REDG.ADD.F64, native on sm_100a) into the zeroed K-grid.
#include "nnfft_impl.cuh"

#ifndef SFB_SPREAD_WARP_FLUSH
#define SFB_SPREAD_WARP_FLUSH 1  // measured: 0.479 -> 0.472 ms at config 3
#endif

namespace sfb {

struct SpreadArgs {
  const double* pos;    // slot order
  const int* perm;      // slot order
  const int* info;      // per chunk
  const int4* units;
  const void* f;        // complex (M1, batch) row-major, or real (M1)
  double2* grid;        // [batch][K]
  int64_t K;
  int batch;
};

static_assert(kChunk == 4, "slot loads assume 4 sources per chunk");

struct ChunkLoad {
  int info;
  double2 p01, p23;  // positions of slots 0..3
  int4 perm;
};

__device__ __forceinline__ ChunkLoad load_chunk(const SpreadArgs& a, int ci, bool valid) {
  ChunkLoad c;
  c.info = 0;
  c.p01 = c.p23 = make_double2(0.5, 0.5);
  c.perm = make_int4(0, 0, 0, 0);
  if (valid) {
    c.info = __ldg(a.info + ci);
    const double2* pp = reinterpret_cast<const double2*>(a.pos) + 2 * (int64_t)ci;
    c.p01 = __ldg(pp);
    c.p23 = __ldg(pp + 1);
    c.perm = __ldg(reinterpret_cast<const int4*>(a.perm) + ci);
  }
  return c;
}

template <int M, bool REAL>
__global__ void __launch_bounds__(kSpreadThreads, 2) k_spread(SpreadArgs a, WinCoef C) {
  constexpr int SPAN = kTile + 2 * M - 1;
  extern __shared__ double2 acc[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarp = blockDim.x >> 5;
  const int col = blockIdx.y;
  double2* my = acc + warp * SPAN;
#if SFB_SPREAD_WARP_FLUSH
  // warps are independent: each zeroes and flushes its own accumulator, so a
  // warp that runs out of blocks never waits for the slowest one of the CTA
  for (int i = lane; i < SPAN; i += 32) my[i] = make_double2(0.0, 0.0);
  __syncwarp();
#else
  for (int i = threadIdx.x; i < SPAN * nwarp; i += blockDim.x) acc[i] = make_double2(0.0, 0.0);
  __syncthreads();
#endif
  const int4 u = a.units[blockIdx.x];
  const int stride = nwarp * 32;
  int cb = u.y + warp * 32;
  ChunkLoad nxt = load_chunk(a, cb + lane, cb + lane < u.z);
  for (; cb < u.z; cb += stride) {
    const ChunkLoad cur = nxt;
    const bool valid = cb + lane < u.z;
    const int cnt = cur.info & 255;
    const int lcell = cur.info >> 8;
    // the random f gather of this block (all four issued back to back) ...
    double2 fv[kChunk];
    const int src[kChunk] = {cur.perm.x, cur.perm.y, cur.perm.z, cur.perm.w};
#pragma unroll
    for (int s = 0; s < kChunk; ++s) {
      fv[s] = make_double2(0.0, 0.0);
      if (s < cnt) {
        if (REAL) {
          fv[s].x = __ldg(static_cast<const double*>(a.f) + src[s]);
        } else {
          fv[s] = __ldg(static_cast<const double2*>(a.f) + (int64_t)src[s] * a.batch + col);
        }
      }
    }
    // ... and the next block's descriptors, in flight during this block's math
    nxt = load_chunk(a, cb + stride + lane, cb + stride + lane < u.z);
    const double pos[kChunk] = {cur.p01.x, cur.p01.y, cur.p23.x, cur.p23.y};
    double2 r[2 * M];
#pragma unroll
    for (int i = 0; i < 2 * M; ++i) r[i] = make_double2(0.0, 0.0);
#pragma unroll
    for (int s = 0; s < kChunk; s += 2) {
      // a padding slot has f = 0 and a harmless position, so pairs may run
      // with a dead second node; skip only fully empty pairs
      if (s < cnt)
        window_accumulate2<M, REAL>(C, pos[s] - floor(pos[s]), fv[s], pos[s + 1] - floor(pos[s + 1]),
                                    fv[s + 1], r);
    }
    // add into the warp-private tile accumulator; equal cells in one warp
    // would race, so leaders of each cell group go first, round by round
    unsigned pending = __ballot_sync(0xffffffffu, valid && cnt > 0);
    while (pending) {
      const bool mine = (pending >> lane) & 1u;
      const unsigned peers = __match_any_sync(0xffffffffu, mine ? lcell : (0x40000000 | lane));
      const bool leader = mine && ((__ffs(peers) - 1) == lane);
#pragma unroll
      for (int i = 0; i < 2 * M; ++i) {
        if (leader) {
          double2 t = my[lcell + i];
          t.x += r[i].x;
          t.y += r[i].y;
          my[lcell + i] = t;
        }
        __syncwarp();
      }
      pending &= ~__ballot_sync(0xffffffffu, leader);
    }
  }
  // flush: grid index of accumulator slot p is tile*kTile - (M-1) + p
  double2* grid = a.grid + (int64_t)col * a.K;
  const int64_t base = (int64_t)u.x * kTile - (M - 1);
#if SFB_SPREAD_WARP_FLUSH
  __syncwarp();
  for (int p = lane; p < SPAN; p += 32) {
    const double2 t = my[p];
    const int64_t gi = base + p;
    if (gi >= 0 && gi < a.K && (t.x != 0.0 || t.y != 0.0)) {
      atomicAdd(&grid[gi].x, t.x);
      atomicAdd(&grid[gi].y, t.y);
    }
  }
  return;
#endif
  __syncthreads();
  for (int p = threadIdx.x; p < SPAN; p += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int w = 0; w < nwarp; ++w) {
      const double2 t = acc[w * SPAN + p];
      s.x += t.x;
      s.y += t.y;
    }
    const int64_t gi = base + p;
    if (gi >= 0 && gi < a.K && (s.x != 0.0 || s.y != 0.0)) {
      atomicAdd(&grid[gi].x, s.x);
      atomicAdd(&grid[gi].y, s.y);
    }
  }
}

template <int M, bool REAL>
static void launch_spread_m(const NnfftPlanImpl& p, const void* f, double2* grid, int batch,
                            cudaStream_t s) {
  const size_t smem = sizeof(double2) * (kTile + 2 * M - 1) * (kSpreadThreads / 32);
  SpreadArgs a{p.sp.pos.p, p.sp.perm.p, p.sp.info.p, p.sp.units.p, f, grid, p.g.K, batch};
  if (p.sp.n_units == 0) return;
  k_spread<M, REAL><<<dim3((unsigned)p.sp.n_units, batch), kSpreadThreads, smem, s>>>(a, p.c1);
  SF_LAUNCH_CHECK();
}

template <bool REAL>
static void launch_spread(const NnfftPlanImpl& p, const void* f, double2* grid, int batch,
                          cudaStream_t s) {
  SF_CUDA(cudaMemsetAsync(grid, 0, sizeof(double2) * (size_t)p.g.K * batch, s));
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

void run_spread_real(const NnfftPlanImpl& p, const double* f, double2* grid, cudaStream_t s) {
  launch_spread<true>(p, f, grid, 1, s);
}

}  // namespace sfb
