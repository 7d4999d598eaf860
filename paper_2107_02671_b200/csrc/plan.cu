// plan.cu -- step 0 of Algorithm 2.1 on the device (ref: pkg/src/sincfft/
// nnfft.py:131-207): validation, clipping, node binning/sorting, the phi_hat
// tables and the FFT tables.  Window values are not tabulated (the reference
// stores M x 2m tables, nnfft.py:188-205); kernels evaluate them from the
// per-tap polynomials instead, so a plan holds O(M1 + M2 + K + L) data.
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>
#include <cstdlib>
#include <string>

#include "nnfft_impl.cuh"

#include <chrono>

#include <cstdio>

#ifndef SFB_SPREAD_CTAS
#define SFB_SPREAD_CTAS 2  // persistent spread CTAs per SM (matches SFB_SPREAD_MINB)
#endif

namespace sfb {

// --------------------------------------------------------------- geometry
// ref: NnfftGeometry.from_parameters, nnfft.py:51-89 (same rules & order)
Geometry make_geometry(int64_t N, int64_t M1, int64_t M2, double sigma1, double sigma2, int m1,
                       int m2) {
  if (N <= 0) fail(1, "N must be a positive integer");
  if (M1 <= 0) fail(1, "M1 must be a positive integer");
  if (M2 <= 0) fail(1, "M2 must be a positive integer");
  if (m1 < 2) fail(1, "m1 must be an integer >= 2");
  if (m2 < 2) fail(1, "m2 must be an integer >= 2");
  if (!(sigma1 > 1.0) || !(sigma2 > 1.0)) fail(1, "sigma1 and sigma2 must be > 1");
  const double n1f = sigma1 * (double)N;
  const int64_t N1 = (int64_t)std::llround(n1f);
  if (std::fabs(n1f - (double)N1) > 1e-9 || (N1 % 2) != 0)
    fail(1, "sigma1*N must be an even integer, got " + std::to_string(n1f));
  if (2 * m1 > N1 / 2)
    fail(1, "need 2*m1 <= N1/2, got 2*" + std::to_string(m1) + " > " + std::to_string(N1 / 2));
  const int64_t K = N1 + 2 * m1;
  const double n2f = sigma2 * (double)K;
  // Python round() is round-half-even; n2f is never a half-integer tie that
  // matters here, but mirror it exactly anyway
  double r = std::nearbyint(n2f);
  int64_t N2 = (int64_t)r;
  if (std::fabs(n2f - (double)N2) > 1e-9) N2 = (int64_t)std::ceil(n2f);
  if (N2 % 2) N2 += 1;
  const double sigma2_eff = (double)N2 / (double)K;
  if ((double)(2 * m2) > (1.0 - (double)N / (double)N1) * (double)N2 + 1e-9)
    fail(1, "need 2*m2 <= (1 - 1/sigma1)*N2, got 2*" + std::to_string(m2) + " > " +
                std::to_string((1.0 - (double)N / (double)N1) * (double)N2));
  if (m1 > kMaxM || m2 > kMaxM)
    fail(5, "window cut-offs above 16 are not supported by the B200 kernels");
  if (K >= (int64_t)1 << 30 || N2 >= (int64_t)1 << 30 || M1 >= (int64_t)1 << 31 ||
      M2 >= (int64_t)1 << 31)
    fail(5, "problem size exceeds the 2^30-point grid / 2^31-node envelope");
  Geometry g{};
  g.N = N;
  g.M1 = M1;
  g.M2 = M2;
  g.N1 = N1;
  g.K = K;
  g.N2 = N2;
  g.m1 = m1;
  g.m2 = m2;
  g.sigma1 = (double)N1 / (double)N;
  g.sigma2 = sigma2_eff;
  g.a = (double)K / (double)N1;
  const double pi = 3.141592653589793238462643383279502884;
  // ref: windows.py:77-80 -- sinh requires 5/4 <= sigma <= 2 (+-1e-9)
  if (!(1.25 - 1e-9 <= g.sigma1 && g.sigma1 <= 2.0 + 1e-9))
    fail(1, "sinh window requires 5/4 <= sigma <= 2, got sigma=" + std::to_string(g.sigma1));
  if (!(1.25 - 1e-9 <= g.sigma2 && g.sigma2 <= 2.0 + 1e-9))
    fail(1, "sinh window requires 5/4 <= sigma <= 2, got sigma=" + std::to_string(g.sigma2));
  g.beta1 = 2.0 * pi * m1 * (1.0 - 1.0 / (2.0 * g.sigma1));  // windows.py:94-95
  g.beta2 = 2.0 * pi * m2 * (1.0 - 1.0 / (2.0 * g.sigma2));
  return g;
}

// ---------------------------------------------------------------- kernels
__global__ void k_absmax(const double* a, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = fabs(a[i]);
    m = (v > m || v != v) ? v : m;  // NaN propagates
  }
  for (int o = 16; o; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, m, o);
    m = (t > m || t != t) ? t : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_clip(const double* in, double* out, int64_t n, double lim) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = fmin(fmax(in[i], -lim), lim);
}

// source keys: cell index floor(N1 v) + K/2 (nnfft.py:188-190)
__global__ void k_src_keys(const double* v, int64_t n, double N1, int64_t halfK, unsigned* key,
                           int* idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double pos = N1 * v[i];
  key[i] = (unsigned)((int64_t)floor(pos) + halfK);
  idx[i] = (int)i;
}

__global__ void k_take_scaled(const double* v, const int* perm, int64_t n, double scale,
                              double* out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) out[j] = scale * v[perm[j]];
}

// first index with key >= c, for c in [0, ncell]
__global__ void k_lower_bound(const unsigned* key, int64_t n, int64_t ncell, int* start) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > ncell) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)key[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  start[c] = (int)lo;
}

__global__ void k_chunk_counts(const int* start, int64_t ncell, int* nch) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  nch[c] = (start[c + 1] - start[c] + kChunk - 1) / kChunk;
}

// moment-spread work units: cells cut into runs of <= kDenseUnit sources
__global__ void k_dense_counts(const int* start, int64_t ncell, int* nu) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  nu[c] = (start[c + 1] - start[c] + kDenseUnit - 1) / kDenseUnit;
}

__global__ void k_dense_emit(const int* start, const int* nu, const int* off, int64_t ncell,
                             int4* units) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  for (int r = 0; r < nu[c]; ++r) {
    const int s0 = start[c] + r * kDenseUnit;
    units[off[c] + r] = make_int4((int)c, s0, min(s0 + kDenseUnit, start[c + 1]), 0);
  }
}

// chunk sort key: (tile, rank within cell, local cell)
constexpr int kLcBits = 12;                   // local cell < kTile <= 4096
constexpr int kTileKeyShift = kLcBits + 30;  // rank < 2^30
static_assert(kTile <= (1 << kLcBits), "local cell field too small");

__global__ void k_chunk_emit(const int* start, const int* nch, const int* off, int64_t ncell,
                             unsigned long long* key, int2* desc) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  const int n = start[c + 1] - start[c];
  const int k = nch[c];
  const int o = off[c];
  const unsigned long long tile = (unsigned long long)(c / kTile);
  const int lc = (int)(c % kTile);
  for (int r = 0; r < k; ++r) {
    key[o + r] = (tile << kTileKeyShift) | ((unsigned long long)r << kLcBits) | (unsigned long long)lc;
    const int cnt = min(kChunk, n - r * kChunk);
    desc[o + r] = make_int2(start[c] + r * kChunk, (lc << 8) | cnt);
  }
}

// chunk c (sorted order, tile t = key >> kTileKeyShift) goes to padded chunk
// boff[t] * 32 + (c - tstart[t]); padding chunks stay zero (count 0)
__global__ void k_chunk_slots(const int2* chunks, const unsigned long long* key, int64_t n,
                              const int* tstart, const int* boff, const double* pos,
                              const int* perm, double* spos, int* sperm, int* info) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int t = (int)(key[c] >> kTileKeyShift);
  const int64_t q = (int64_t)boff[t] * kBlockChunks + (c - tstart[t]);
  const int2 d = chunks[c];
  const int cnt = d.y & 255;
  info[q] = d.y;
  for (int s = 0; s < kChunk; ++s) {
    spos[q * kChunk + s] = s < cnt ? pos[d.x + s] : 0.5;
    sperm[q * kChunk + s] = s < cnt ? perm[d.x + s] : 0;
  }
}

__global__ void k_tile_starts(const int* cstart, int64_t K, int T, int64_t ntile, int* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t <= ntile) out[t] = cstart[min(t * T, K)];
}

__global__ void k_tile_bounds(const unsigned long long* key, int64_t n, int64_t ntile,
                              int* tstart) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > ntile) return;
  const unsigned long long target = (unsigned long long)t << kTileKeyShift;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  tstart[t] = (int)lo;
}

__global__ void k_block_counts(const int* tstart, int64_t ntile, int* nb) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ntile) return;
  nb[t] = (tstart[t + 1] - tstart[t] + kBlockChunks - 1) / kBlockChunks;
}

__global__ void k_block_emit(const int* nb, const int* boff, int64_t ntile, int* blk_tile) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ntile) return;
  for (int j = 0; j < nb[t]; ++j) blk_tile[boff[t] + j] = (int)t;
}

// Estimated cost of each 32-chunk block for the spread's static warp ranges
// (spread.cu): window pairs (4 units each for the lane that needs the most)
// plus accumulator rounds (1 unit each; a single-cell block is one butterfly).
// One warp per block.
struct CostW {
  int pair, round, base, same;
};
__global__ void k_block_cost(const int* info, int64_t nblk, long long* cost, CostW cw) {
  const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= nblk) return;
  const int in = info[b * kBlockChunks + lane];
  const int cnt = in & 255, lc = in >> 8;
  const int pairs = __reduce_max_sync(0xffffffffu, cnt > 2 ? 2 : cnt > 0 ? 1 : 0);
  int same = 0;
  __match_all_sync(0xffffffffu, cnt > 0 ? lc : -1 - lane, &same);
  const unsigned peers = __match_any_sync(0xffffffffu, cnt > 0 ? lc : -1 - lane);
  const int rounds = same ? cw.same : __reduce_max_sync(0xffffffffu, __popc(peers));
  if (lane == 0) cost[b] = cw.pair * pairs + cw.round * rounds + cw.base;
}

// first block of warp w: the first b with prefix cost[0..b] > w * total / W
__global__ void k_warp_starts(const long long* incl, int64_t nblk, int64_t W, int64_t* wstart) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w > W) return;
  if (w == W) {
    wstart[w] = nblk;
    return;
  }
  const long long total = incl[nblk - 1];
  const long long target = (long long)((double)total * (double)w / (double)W);
  int64_t lo = 0, hi = nblk;  // first b with incl[b] > target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (incl[mid] <= target) lo = mid + 1;
    else hi = mid;
  }
  wstart[w] = w == 0 ? 0 : lo;
}

// target keys: (original-index slice, floor(N2 * xs) + N2), xs = x * (N/N1)
// (nnfft.py:200-201)
int64_t gather_slice() {
  const char* e = getenv("SFB_GATHER_SLICE_LOG2");
  if (e && atoi(e) >= 9 && atoi(e) <= 30) return (int64_t)1 << atoi(e);
  return kGatherSliceDefault;
}

__global__ void k_tgt_keys(const double* x, int64_t n, double ratio, double N2d, int64_t N2,
                           int cell_bits, int64_t slice, unsigned long long* key, int* idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double xs = x[i] * ratio;
  const unsigned long long cell = (unsigned long long)((int64_t)floor(N2d * xs) + N2);
  key[i] = ((unsigned long long)(i / slice) << cell_bits) | cell;
  idx[i] = (int)i;
}

// sorted target positions and 1/phi_hat_1(N x) (nnfft.py:175, 243)
__global__ void k_tgt_tables(const double* x, const int* perm, int64_t n, double ratio, double N2d,
                             int with_hat, double Nd, double beta1, int m1, int64_t N1,
                             double* pos, double* scale, unsigned long long* min_hat_bits) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double xv = x[perm[j]];
  pos[j] = N2d * (xv * ratio);
  if (!with_hat) {
    scale[j] = 1.0;
    return;
  }
  const double hat = phi_hat_sinh(beta1, m1, N1, Nd * xv);
  scale[j] = 1.0 / hat;
  if (!(hat > 0.0)) atomicAdd(min_hat_bits, 1ull);
}

// h range [klo, khi] (k' = s - s_lo) read by each gather CTA of kGatherGroup
// sorted targets; {-1, -1} (never staged) if it does not fit in int
__global__ void k_pad_targets(double* pos, double* scale, int* perm, int64_t n, int64_t npad) {
  for (int64_t j = n + threadIdx.x; j < npad; j += blockDim.x) {
    pos[j] = pos[n - 1];
    scale[j] = 0.0;
    perm[j] = -1;
  }
}

// Octet order of one full gather group (one CTA of kGatherGroup threads per
// group): the group's targets (position-sorted) are stably sorted by the
// residue r = (floor(pos) - floor(pos_first)) mod 8 of their window start in
// the staged span, and the element at rank p of that order goes to lane
// q = p / 32 of octet o = p % 32, i.e. record n = (o / 16) * T + (o % 16) * 8 + q
// (thread t of k_gather2 takes records t and t + T; its quarter-warp is the 8
// consecutive t).  Balanced residues give every octet one target per residue;
// dense groups (few distinct cells) give octets whose equal residues share a
// cell, i.e. one broadcast address.  A partial last group is left sorted.
#ifndef SFB_GATHER_PAIRS
#define SFB_GATHER_PAIRS 1  // k_octet_pairs (same-cell pairs per thread) instead of k_octet_order
#endif
__global__ void k_octet_order(const double* pos, const double* scale, const int* perm,
                              int64_t M2, double* opos, double* oscale, int* operm) {
  constexpr int G = kGatherGroup, T = kGatherThreads;
  __shared__ int res[G];
  const int64_t j0 = (int64_t)blockIdx.x * G;
  const int i = threadIdx.x;
  const int64_t j = j0 + i;
  if (j0 + G > M2) {  // partial group: copy
    if (j < M2) opos[j] = pos[j], oscale[j] = scale[j], operm[j] = perm[j];
    return;
  }
  const double base = floor(pos[j0]);
  const int r = (int)((int64_t)(floor(pos[j]) - base) & 7);
  res[i] = r;
  __syncthreads();
  int rank = 0;
  for (int k = 0; k < G; ++k) {
    const int rk = res[k];
    rank += (rk < r) || (rk == r && k < i);
  }
  const int o = rank % 32, q = rank / 32;
  const int64_t n = j0 + (o / 16) * T + (o % 16) * 8 + q;
  opos[n] = pos[j];
  oscale[n] = scale[j];
  operm[n] = perm[j];
}

// Pair-and-octet order of one full gather group (one thread per group):
// targets of one cell are paired (consecutive in the sorted group) and a pair
// goes to ONE thread as its two targets, which then read one h window (the
// second target's loads are predicated off, window_dot2 `same`).  Octets
// (quarter-warps: 8 consecutive threads) are filled first with 8 pairs of
// pairwise distinct window residues mod 8 -- no bank conflict and no second
// load in the whole octet -- then lane l of every other octet takes a
// leftover pair of residue l or two single targets of residue l (one per
// target set), falling back to the fullest residue bucket.  Thread t takes
// records t (set 0) and t + T (set 1).
__global__ void k_octet_pairs(const double* pos, const double* scale, const int* perm, int64_t M2,
                              int64_t ngroups, double* opos, double* oscale, int* operm) {
  constexpr int G = kGatherGroup, T = kGatherThreads, NOCT = T / 8;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  const int64_t j0 = g * G;
  if (j0 + G > M2) {  // partial group: copy
    for (int64_t j = j0; j < M2; ++j) opos[j] = pos[j], oscale[j] = scale[j], operm[j] = perm[j];
    return;
  }
  const double base = floor(pos[j0]);
  // units: (set-0 index, set-1 index); a pair has equal cells
  short ua[2 * T], ub[2 * T];
  unsigned char ures[2 * T], upair[2 * T];
  int nu = 0;
  short singles[G];
  int ns = 0;
  for (int i = 0; i < G;) {
    const double ci = floor(pos[j0 + i]);
    if (i + 1 < G && floor(pos[j0 + i + 1]) == ci) {
      ua[nu] = (short)i, ub[nu] = (short)(i + 1);
      ures[nu] = (unsigned char)((int64_t)(ci - base) & 7), upair[nu] = 1;
      ++nu;
      i += 2;
    } else {
      singles[ns++] = (short)i;
      ++i;
    }
  }
  // residue buckets of the single targets (position order inside a bucket)
  short sb_[8][G];
  int sn[8] = {0, 0, 0, 0, 0, 0, 0, 0}, shead[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < ns; ++k) {
    const int r = (int)((int64_t)(floor(pos[j0 + singles[k]]) - base) & 7);
    sb_[r][sn[r]++] = singles[k];
  }
  short slot_of[T];   // unit placed at thread slot
  bool used[T];
  for (int k = 0; k < T; ++k) used[k] = false;
  int oct = 0;
  // pure pair octets: one pair of each residue
  while (oct < NOCT) {
    int pick[8];
    bool ok = true;
    for (int r = 0; r < 8 && ok; ++r) {
      pick[r] = -1;
      for (int k = 0; k < nu; ++k)
        if (!used[k] && upair[k] && ures[k] == r) { pick[r] = k; break; }
      ok = pick[r] >= 0;
    }
    if (!ok) break;
    for (int r = 0; r < 8; ++r) slot_of[oct * 8 + r] = (short)pick[r], used[pick[r]] = true;
    ++oct;
  }
  // mixed octets: lane l prefers residue l in both target sets -- a leftover
  // pair of residue l, else two singles of residue l -- and falls back to the
  // fullest bucket, so a quarter-warp repeats a residue only when a bucket
  // runs dry
  auto take_single = [&](int r) -> int {
    if (shead[r] >= sn[r]) {
      int best = -1;
      for (int q = 0; q < 8; ++q)
        if (shead[q] < sn[q] && (best < 0 || sn[q] - shead[q] > sn[best] - shead[best])) best = q;
      if (best < 0) return -1;
      r = best;
    }
    return sb_[r][shead[r]++];
  };
  int nu2 = nu;
  for (int t = oct * 8; t < T; ++t) {
    const int l = t & 7;
    int pk = -1;
    for (int k = 0; k < nu && pk < 0; ++k)
      if (!used[k] && upair[k] && ures[k] == l) pk = k;
    int sa = -1, sbb = -1;
    if (pk < 0) {
      sa = take_single(l);
      if (sa >= 0) sbb = take_single(l);
    }
    if (pk < 0 && (sa < 0 || sbb < 0)) {  // no singles left: any leftover pair
      for (int k = 0; k < nu && pk < 0; ++k)
        if (!used[k] && upair[k]) pk = k;
    }
    if (pk >= 0) {
      used[pk] = true;
      slot_of[t] = (short)pk;
    } else {  // a new unit of two singles
      ua[nu2] = (short)sa, ub[nu2] = (short)sbb;
      slot_of[t] = (short)nu2++;
    }
  }
  for (int t = 0; t < T; ++t) {
    const int a = ua[slot_of[t]], b = ub[slot_of[t]];
    opos[j0 + t] = pos[j0 + a], oscale[j0 + t] = scale[j0 + a], operm[j0 + t] = perm[j0 + a];
    opos[j0 + T + t] = pos[j0 + b], oscale[j0 + T + t] = scale[j0 + b],
                  operm[j0 + T + t] = perm[j0 + b];
  }
}

__global__ void k_gather_spans(const double* pos, int64_t n, int64_t nblk, int m2, int64_t s_lo,
                               int2* span) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const int64_t j0 = b * kGatherGroup, jl = min(j0 + kGatherGroup, n) - 1;
  const int64_t lo = (int64_t)floor(pos[j0]) + 1 - m2 - s_lo;
  const int64_t hi = (int64_t)floor(pos[jl]) + m2 - s_lo;
  span[b] = (lo >= 0 && hi < (1ll << 31) && lo <= hi) ? make_int2((int)lo, (int)hi)
                                                       : make_int2(-1, -1);
}

__global__ void k_hat2(double* hat2, int64_t K, double beta2, int m2, int64_t N2,
                       unsigned long long* bad) {
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l >= K) return;
  const double h = phi_hat_sinh(beta2, m2, N2, (double)(l - K / 2));
  hat2[l] = h;
  if (!(h > 0.0)) atomicAdd(bad, 1ull);
}

__global__ void k_mul_scale(double* scale, const int* perm, const double* w, int64_t n) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) scale[j] *= w[perm[j]];
}

// ------------------------------------------------------------ host helpers
namespace {

inline unsigned blocks(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, ceil_div(n, t)); }

double device_absmax(const double* a, int64_t n, cudaStream_t s) {
  Scratch r(sizeof(unsigned long long), s);
  SF_CUDA(cudaMemsetAsync(r.p, 0, sizeof(unsigned long long), s));
  k_absmax<<<std::min<unsigned>(blocks(n), 1024), 256, 0, s>>>(a, n, r.as<unsigned long long>());
  SF_LAUNCH_CHECK();
  unsigned long long bits = 0;
  SF_CUDA(cudaMemcpyAsync(&bits, r.p, sizeof(bits), cudaMemcpyDeviceToHost, s));
  SF_CUDA(cudaStreamSynchronize(s));
  double m;
  std::memcpy(&m, &bits, sizeof(m));
  return m;
}

// min / max of a device array (order-preserving integer keys for doubles)
__device__ __forceinline__ unsigned long long order_key(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_minmax(const double* a, int64_t n, unsigned long long* mn,
                         unsigned long long* mx) {
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    lo = fmin(lo, a[i]);
    hi = fmax(hi, a[i]);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mn, order_key(lo));
    atomicMax(mx, order_key(hi));
  }
}

double from_order_key(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
}

void device_minmax(const double* a, int64_t n, cudaStream_t s, double* lo, double* hi) {
  Scratch r(2 * sizeof(unsigned long long), s);
  const unsigned long long init[2] = {~0ull, 0ull};
  SF_CUDA(cudaMemcpyAsync(r.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_minmax<<<std::min<unsigned>(blocks(n), 1024), 256, 0, s>>>(
      a, n, r.as<unsigned long long>(), r.as<unsigned long long>() + 1);
  SF_LAUNCH_CHECK();
  unsigned long long out[2];
  SF_CUDA(cudaMemcpyAsync(out, r.p, sizeof(out), cudaMemcpyDeviceToHost, s));
  SF_CUDA(cudaStreamSynchronize(s));
  *lo = from_order_key(out[0]);
  *hi = from_order_key(out[1]);
}

int key_bits(uint64_t maxkey) {
  int b = 1;
  while (b < 64 && (maxkey >> b) != 0) ++b;
  return b;
}

template <class T>
T read1(const T* dev, cudaStream_t s) {
  T v;
  SF_CUDA(cudaMemcpyAsync(&v, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
  SF_CUDA(cudaStreamSynchronize(s));
  return v;
}

// exclusive scan of n ints into off[0..n], returns total
int64_t exclusive_scan(const int* in, int* off, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, off, (int)n + 1, s));
  Scratch t(tb, s);
  // in has n entries; scan n+1 using a padded copy so off[n] is the total
  Scratch pad(sizeof(int) * (n + 1), s);
  SF_CUDA(cudaMemsetAsync(pad.p, 0, sizeof(int) * (n + 1), s));
  SF_CUDA(cudaMemcpyAsync(pad.p, in, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
  SF_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, pad.as<int>(), off, (int)n + 1, s));
  return (int64_t)read1(off + n, s);
}

}  // namespace

// Spread structure (SpreadPlan) for M1 sources at positions N1 * v (v clipped,
// device, original order) on a K-point grid, cell floor(N1 v) + K/2:
// cell-sorted sources cut into chunks, blocks and cost-balanced warp ranges
// (spread.cu), plus the cell-sorted copies the batched path reads.
void build_sources(NnfftPlanImpl& p, const double* v, int64_t M1, double N1, int64_t K,
                   cudaStream_t s) {
    Scratch kin(sizeof(unsigned) * M1, s), kout(sizeof(unsigned) * M1, s);
    Scratch iin(sizeof(int) * M1, s);
    p.sp.perm.alloc(M1);
    k_src_keys<<<blocks(M1), 256, 0, s>>>(v, M1, N1, K / 2, kin.as<unsigned>(),
                                          iin.as<int>());
    SF_LAUNCH_CHECK();
    size_t tb = 0;
    const int bits = key_bits((uint64_t)K);
    SF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.as<unsigned>(), kout.as<unsigned>(),
                                            iin.as<int>(), p.sp.perm.p, (int)M1, 0, bits, s));
    {
      Scratch t(tb, s);
      SF_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, kin.as<unsigned>(), kout.as<unsigned>(),
                                              iin.as<int>(), p.sp.perm.p, (int)M1, 0, bits, s));
    }
    p.sp.pos.alloc(M1);
    k_take_scaled<<<blocks(M1), 256, 0, s>>>(v, p.sp.perm.p, M1, N1,
                                             p.sp.pos.p);
    SF_LAUNCH_CHECK();
    Scratch cstart(sizeof(int) * (K + 1), s), nch(sizeof(int) * K, s),
        coff(sizeof(int) * (K + 1), s);
    k_lower_bound<<<blocks(K + 1), 256, 0, s>>>(kout.as<unsigned>(), M1, K, cstart.as<int>());
    k_chunk_counts<<<blocks(K), 256, 0, s>>>(cstart.as<int>(), K, nch.as<int>());
    SF_LAUNCH_CHECK();
    const int64_t nchunks = exclusive_scan(nch.as<int>(), coff.as<int>(), K, s);
    p.sp.n_chunks = nchunks;
    Scratch ckey(sizeof(unsigned long long) * nchunks, s), cdesc(sizeof(int2) * nchunks, s);
    Scratch ckey2(sizeof(unsigned long long) * nchunks, s);
    p.sp.chunks.alloc(nchunks);
    k_chunk_emit<<<blocks(K), 256, 0, s>>>(cstart.as<int>(), nch.as<int>(), coff.as<int>(), K,
                                           ckey.as<unsigned long long>(), cdesc.as<int2>());
    SF_LAUNCH_CHECK();
    const int64_t ntile = ceil_div(K, kTile);
    const int kb = kTileKeyShift + key_bits((uint64_t)ntile);
    tb = 0;
    SF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ckey.as<unsigned long long>(),
                                            ckey2.as<unsigned long long>(), cdesc.as<int2>(),
                                            p.sp.chunks.p, (int)nchunks, 0, kb, s));
    {
      Scratch t(tb, s);
      SF_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, ckey.as<unsigned long long>(),
                                              ckey2.as<unsigned long long>(), cdesc.as<int2>(),
                                              p.sp.chunks.p, (int)nchunks, 0, kb, s));
    }
    Scratch tstart(sizeof(int) * (ntile + 1), s), nb(sizeof(int) * ntile, s),
        boff(sizeof(int) * (ntile + 1), s);
    k_tile_bounds<<<blocks(ntile + 1), 256, 0, s>>>(ckey2.as<unsigned long long>(), nchunks, ntile,
                                                    tstart.as<int>());
    k_block_counts<<<blocks(ntile), 256, 0, s>>>(tstart.as<int>(), ntile, nb.as<int>());
    SF_LAUNCH_CHECK();
    p.sp.n_blocks = exclusive_scan(nb.as<int>(), boff.as<int>(), ntile, s);
    p.sp.blk_tile.alloc(std::max<int64_t>(p.sp.n_blocks, 1));
    k_block_emit<<<blocks(ntile), 256, 0, s>>>(nb.as<int>(), boff.as<int>(), ntile,
                                               p.sp.blk_tile.p);
    SF_LAUNCH_CHECK();
    SF_CUDA(cudaDeviceGetAttribute(&p.sp.n_sms, cudaDevAttrMultiProcessorCount, p.device));
    // dense sources: keep the per-cell starts for the moment spread
    // (SFB_SPREAD_DENSE: 0 never, 1 always, default by average cell load)
    {
      const char* e = getenv("SFB_SPREAD_DENSE");
      p.sp.dense = e ? atoi(e) != 0 : M1 >= kDenseMin * K;
      if (p.sp.dense) {
        Scratch nu(sizeof(int) * K, s), uoff(sizeof(int) * (K + 1), s);
        k_dense_counts<<<blocks(K), 256, 0, s>>>(cstart.as<int>(), K, nu.as<int>());
        SF_LAUNCH_CHECK();
        p.sp.n_units = exclusive_scan(nu.as<int>(), uoff.as<int>(), K, s);
        p.sp.units.alloc(std::max<int64_t>(p.sp.n_units, 1));
        k_dense_emit<<<blocks(K), 256, 0, s>>>(cstart.as<int>(), nu.as<int>(), uoff.as<int>(), K,
                                              p.sp.units.p);
        SF_LAUNCH_CHECK();
      }
    }
    // batched path: keep the cell-sorted arrays and the 128-cell tile starts
    {
      const int64_t ntb = ceil_div(K, 128);
      p.sp.btile.alloc(ntb + 1);
      k_tile_starts<<<blocks(ntb + 1), 256, 0, s>>>(cstart.as<int>(), K, 128, ntb, p.sp.btile.p);
      SF_LAUNCH_CHECK();
    }
    // re-lay the sorted sources out in chunk-slot order (kChunk slots per
    // chunk, 32 chunks per block, blocks padded with empty chunks)
    const int64_t npad = std::max<int64_t>(p.sp.n_blocks, 1) * kBlockChunks;
    DevArray<double> spos(npad * kChunk);
    DevArray<int> sperm(npad * kChunk);
    p.sp.info.alloc(npad);
    SF_CUDA(cudaMemsetAsync(spos.p, 0, sizeof(double) * npad * kChunk, s));
    SF_CUDA(cudaMemsetAsync(sperm.p, 0, sizeof(int) * npad * kChunk, s));
    SF_CUDA(cudaMemsetAsync(p.sp.info.p, 0, sizeof(int) * npad, s));
    k_chunk_slots<<<blocks(nchunks), 256, 0, s>>>(p.sp.chunks.p, ckey2.as<unsigned long long>(),
                                                  nchunks, tstart.as<int>(), boff.as<int>(),
                                                  p.sp.pos.p, p.sp.perm.p, spos.p, sperm.p,
                                                  p.sp.info.p);
    SF_LAUNCH_CHECK();
    // static cost-balanced warp ranges of the persistent spread kernel
    {
      const int64_t nblk = p.sp.n_blocks;
      const char* e1 = getenv("SFB_SPREAD_CTAS_PER_SM");
      const char* e2 = getenv("SFB_SPREAD_BLOCKS_PER_WARP");
      const int cps = e1 ? std::max(1, atoi(e1)) : SFB_SPREAD_CTAS;
      const int bpw = e2 ? std::max(1, atoi(e2)) : 1;  // 1 measured best (configs 1-3, 5)
      p.sp.n_ctas = (int)std::max<int64_t>(
          1, std::min<int64_t>(cps * (int64_t)p.sp.n_sms, ceil_div(nblk, bpw * kSpreadWarps)));
      const int64_t W = (int64_t)p.sp.n_ctas * kSpreadWarps;
      p.sp.wstart.alloc(W + 1);
      if (nblk > 0) {
        Scratch cost(sizeof(long long) * nblk, s), incl(sizeof(long long) * nblk, s);
        CostW cw{4, 1, 0, 2};  // tuning: SFB_SPREAD_COST="pair,round,base,same"
        if (const char* e = getenv("SFB_SPREAD_COST"))
          sscanf(e, "%d,%d,%d,%d", &cw.pair, &cw.round, &cw.base, &cw.same);
        k_block_cost<<<blocks(nblk * 32), 256, 0, s>>>(p.sp.info.p, nblk, cost.as<long long>(),
                                                       cw);
        SF_LAUNCH_CHECK();
        size_t tb3 = 0;
        SF_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb3, cost.as<long long>(),
                                              incl.as<long long>(), (int)nblk, s));
        Scratch t(tb3, s);
        SF_CUDA(cub::DeviceScan::InclusiveSum(t.p, tb3, cost.as<long long>(),
                                              incl.as<long long>(), (int)nblk, s));
        k_warp_starts<<<blocks(W + 1), 256, 0, s>>>(incl.as<long long>(), nblk, W,
                                                    p.sp.wstart.p);
        SF_LAUNCH_CHECK();
      } else {
        SF_CUDA(cudaMemsetAsync(p.sp.wstart.p, 0, sizeof(int64_t) * (W + 1), s));
      }
    }
    SF_CUDA(cudaStreamSynchronize(s));
    p.sp.bpos = std::move(p.sp.pos);
    p.sp.bperm = std::move(p.sp.perm);
    p.sp.pos = std::move(spos);
    p.sp.perm = std::move(sperm);
    p.sp.chunks.release();
}

// Gather structure (GatherPlan) for M2 targets at positions N2 * xs,
// xs = ratio * x (x clipped, device, original order): targets sorted by
// (original-index slice, cell), the per-target scale (1/phi_hat_1(N x) for
// the NNFFT, 1 for the NFFT), the per-CTA h spans and the output window
// [s_lo, s_lo + Kout) the gather reads (Kout <= N2; wider windows wrap).
void build_targets(NnfftPlanImpl& p, const double* x, int64_t M2, double ratio, double pos_scale,
                   int64_t N2, int m2, const TargetScale& ts, cudaStream_t s,
                   int64_t force_s_lo, int64_t force_kout) {
    Scratch kin(sizeof(unsigned long long) * M2, s), kout(sizeof(unsigned long long) * M2, s);
    Scratch iin(sizeof(int) * M2, s);
    // pos / scale / perm are padded to whole gather groups (a group's records
    // are fetched by fixed-size bulk copies): pos repeats the last position,
    // scale 0, perm -1
    const int64_t m2pad = ceil_div(M2, (int64_t)kGatherGroup) * kGatherGroup;
    p.gp.perm.alloc(m2pad);
    const int cbits = key_bits((uint64_t)(2 * N2 + 2));
    const int64_t slice = gather_slice();
    k_tgt_keys<<<blocks(M2), 256, 0, s>>>(x, M2, ratio, pos_scale, N2, cbits, slice,
                                          kin.as<unsigned long long>(), iin.as<int>());
    SF_LAUNCH_CHECK();
    size_t tb = 0;
    const int bits = cbits + key_bits((uint64_t)((M2 - 1) / slice));
    SF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.as<unsigned long long>(),
                                            kout.as<unsigned long long>(), iin.as<int>(),
                                            p.gp.perm.p, (int)M2, 0, bits, s));
    {
      Scratch t(tb, s);
      SF_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, kin.as<unsigned long long>(),
                                              kout.as<unsigned long long>(), iin.as<int>(),
                                              p.gp.perm.p, (int)M2, 0, bits, s));
    }
    p.gp.pos.alloc(m2pad);
    p.gp.scale.alloc(m2pad);
    Scratch bad(sizeof(unsigned long long), s);
    SF_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), s));
    k_tgt_tables<<<blocks(M2), 256, 0, s>>>(x, p.gp.perm.p, M2, ratio, pos_scale, ts.hat1 ? 1 : 0,
                                            ts.N, ts.beta1, ts.m1, ts.N1, p.gp.pos.p,
                                            p.gp.scale.p, bad.as<unsigned long long>());
    SF_LAUNCH_CHECK();
    if (read1(bad.as<unsigned long long>(), s))
      fail(2, "nnfft_plan: phi_hat_1(N x_j) must be strictly positive at every node");
    if (m2pad > M2) {
      k_pad_targets<<<1, 256, 0, s>>>(p.gp.pos.p, p.gp.scale.p, p.gp.perm.p, M2, m2pad);
      SF_LAUNCH_CHECK();
    }
    double plo, phi;
    device_minmax(p.gp.pos.p, M2, s, &plo, &phi);
    int64_t s_lo = (int64_t)std::floor(plo) + 1 - m2;
    const int64_t s_hi = (int64_t)std::floor(phi) + m2;
    p.fft.Kout = std::min<int64_t>(s_hi - s_lo + 1, N2);
    if (force_kout > 0) {  // the caller's h window (adjoint gather over a whole K-grid)
      if (s_lo < force_s_lo || s_hi >= force_s_lo + force_kout)
        fail(1, "internal: target window outside the forced h range");
      s_lo = force_s_lo;
      p.fft.Kout = force_kout;
    }
    p.fft.s_lo = s_lo;
    const int64_t nblk = ceil_div(M2, kGatherGroup);
    p.gp.span.alloc(nblk);
    k_gather_spans<<<blocks(nblk), 256, 0, s>>>(p.gp.pos.p, M2, nblk, m2, s_lo, p.gp.span.p);
    SF_LAUNCH_CHECK();
    octet_order(p, M2, s);
}

void octet_order(NnfftPlanImpl& p, int64_t M2, cudaStream_t s) {
  static_assert(kGatherGroup == 2 * kGatherThreads && kGatherThreads % 8 == 0,
                "octet order assumes two targets per thread");
  const int64_t m2pad = p.gp.pos.n;
  if (p.gp.opos.n != m2pad) {
    p.gp.opos.alloc(m2pad);
    p.gp.oscale.alloc(m2pad);
    p.gp.operm.alloc(m2pad);
  }
  if (m2pad > M2) {  // padding records as in pos / scale / perm
    SF_CUDA(cudaMemcpyAsync(p.gp.opos.p + M2, p.gp.pos.p + M2, sizeof(double) * (m2pad - M2),
                            cudaMemcpyDeviceToDevice, s));
    SF_CUDA(cudaMemcpyAsync(p.gp.oscale.p + M2, p.gp.scale.p + M2,
                            sizeof(double) * (m2pad - M2), cudaMemcpyDeviceToDevice, s));
    SF_CUDA(cudaMemcpyAsync(p.gp.operm.p + M2, p.gp.perm.p + M2, sizeof(int) * (m2pad - M2),
                            cudaMemcpyDeviceToDevice, s));
  }
  const int64_t ngroups = ceil_div(M2, (int64_t)kGatherGroup);
  if (ngroups > 0 && SFB_GATHER_PAIRS)
    k_octet_pairs<<<(unsigned)ceil_div(ngroups, (int64_t)64), 64, 0, s>>>(
        p.gp.pos.p, p.gp.scale.p, p.gp.perm.p, M2, ngroups, p.gp.opos.p, p.gp.oscale.p,
        p.gp.operm.p);
  else if (ngroups > 0)
    k_octet_order<<<(unsigned)ngroups, kGatherGroup, 0, s>>>(p.gp.pos.p, p.gp.scale.p, p.gp.perm.p,
                                                            M2, p.gp.opos.p, p.gp.oscale.p,
                                                            p.gp.operm.p);
  SF_LAUNCH_CHECK();
}

// SFB_PLAN_TIMING=1: wall time of every plan stage (stream synchronised), on stderr
struct PlanLaps {
  cudaStream_t s;
  bool on;
  std::chrono::steady_clock::time_point t0;
  explicit PlanLaps(cudaStream_t st) : s(st), on(getenv("SFB_PLAN_TIMING") != nullptr) {
    if (on) cudaStreamSynchronize(s);
    t0 = std::chrono::steady_clock::now();
  }
  void lap(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[plan] %-28s %8.2f ms\n", what,
            std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

void build_plan(NnfftPlanImpl& p, const double* v_dev, const double* x_dev, cudaStream_t s) {
  const Geometry& g = p.g;
  PlanLaps laps(s);
  // --- domain checks and clipping (nnfft.py:162-170)
  const double vlim = 0.5 / g.a;
  const double vmax = device_absmax(v_dev, g.M1, s);
  if (!(vmax <= vlim + 1e-12)) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "nnfft_plan: frequencies exceed 1/(2a) = %.6g; apply rescale_frequencies to map "
             "[-1/2, 1/2] data into the band",
             vlim);
    fail(1, buf);
  }
  const double xmax = device_absmax(x_dev, g.M2, s);
  if (!(xmax <= 0.5 + 1e-12)) fail(1, "nnfft_plan: spatial nodes must lie in [-1/2, 1/2]");
  p.v_clip.alloc(g.M1);
  p.x_clip.alloc(g.M2);
  k_clip<<<blocks(g.M1), 256, 0, s>>>(v_dev, p.v_clip.p, g.M1, vlim);
  k_clip<<<blocks(g.M2), 256, 0, s>>>(x_dev, p.x_clip.p, g.M2, 0.5);
  SF_LAUNCH_CHECK();
  laps.lap("domain checks + clip");

  // --- window polynomials (window.cu); sigma of window 2 is N2/K (nnfft.py:173)
  p.c1 = fit_window(g.m1, g.beta1);
  p.c2 = fit_window(g.m2, g.beta2);
  laps.lap("window polynomial fits");

  // --- phi_hat_2 at l - K/2 (nnfft.py:180-183)
  p.hat2.alloc(g.K);
  {
    Scratch bad(sizeof(unsigned long long), s);
    SF_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), s));
    k_hat2<<<blocks(g.K), 256, 0, s>>>(p.hat2.p, g.K, g.beta2, g.m2, g.N2,
                                       bad.as<unsigned long long>());
    SF_LAUNCH_CHECK();
    if (read1(bad.as<unsigned long long>(), s))
      fail(2, "nnfft_plan: phi_hat_2 must be strictly positive on the coarse grid");
  }

  laps.lap("phi_hat_2 table");
  // --- sources: sort by cell, chunk, tile into blocks
  build_sources(p, p.v_clip.p, g.M1, (double)g.N1, g.K, s);
  laps.lap("build_sources");

  // --- targets: sort by (original-index slice, fine-grid cell), 1/phi_hat_1,
  //     and the output window [s_lo, s_hi] the gather reads
  TargetScale ts;
  ts.hat1 = true;
  ts.N = (double)g.N;
  ts.beta1 = g.beta1;
  ts.m1 = g.m1;
  ts.N1 = g.N1;
  int64_t fs_lo = 0, fkout = 0;
  if (p.full_window) {  // every |x| <= 1/2, one slot of slack each side
    const double pmax = (double)g.N2 * ((double)g.N / (double)g.N1) * 0.5;
    fs_lo = (int64_t)std::floor(-pmax) - g.m2;
    const int64_t s_hi = (int64_t)std::floor(pmax) + g.m2 + 1;
    fkout = std::min<int64_t>(s_hi - fs_lo + 1, g.N2);
  }
  build_targets(p, p.x_clip.p, g.M2, (double)g.N / (double)g.N1, (double)g.N2, g.N2, g.m2, ts, s,
                fs_lo, fkout);
  laps.lap("build_targets");

  p.fft.in_scale = 1.0 / ((double)g.N1 * (double)g.N2);
  build_fft(p, s);
  SF_CUDA(cudaStreamSynchronize(s));
  laps.lap("build_fft");
}

// Grid indices the spread can touch, [c + K/2 + 1 - m1, c + K/2 + m1] for the
// cells c = floor(N1 v) of the plan's sources, and h indices k' = s - s_lo the
// gather reads (one slot of margin each side for the rounding of N1 v).
void dist_support(const NnfftPlanImpl& p, cudaStream_t s, int64_t out[4]) {
  const Geometry& g = p.g;
  double vlo, vhi, plo, phi;
  device_minmax(p.v_clip.p, g.M1, s, &vlo, &vhi);
  device_minmax(p.gp.pos.p, g.M2, s, &plo, &phi);
  const int64_t h = g.K / 2;
  out[0] = std::max<int64_t>(0, (int64_t)std::floor((double)g.N1 * vlo) + h + 1 - g.m1 - 1);
  out[1] = std::min<int64_t>(g.K - 1, (int64_t)std::floor((double)g.N1 * vhi) + h + g.m1 + 1);
  out[2] = std::max<int64_t>(0, (int64_t)std::floor(plo) + 1 - g.m2 - p.fft.s_lo);
  out[3] = std::min<int64_t>(p.fft.Kout - 1, (int64_t)std::floor(phi) + g.m2 - p.fft.s_lo);
}

void fuse_target_weights(NnfftPlanImpl& p, const double* w_dev, cudaStream_t s) {
  k_mul_scale<<<blocks(p.g.M2), 256, 0, s>>>(p.gp.scale.p, p.gp.perm.p, w_dev, p.g.M2);
  SF_LAUNCH_CHECK();
  k_mul_scale<<<blocks(p.g.M2), 256, 0, s>>>(p.gp.oscale.p, p.gp.operm.p, w_dev, p.g.M2);
  SF_LAUNCH_CHECK();
}

}  // namespace sfb
