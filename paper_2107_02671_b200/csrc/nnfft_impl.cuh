// nnfft_impl.cuh -- device-resident NNFFT plan (Algorithm 2.1) and its stages.
//
// Reference mapping (pkg/src/sincfft/nnfft.py):
//   geometry            :51-89   -> Geometry (computed on the host, plan.cu)
//   step 0 tables       :131-207 -> SpreadPlan / GatherPlan / FftPlan: nodes are
//                                   binned & sorted on the device; window values
//                                   are NOT tabulated but evaluated per node from
//                                   per-tap polynomials (window.cuh)
//   step 1 spread       :229-233 -> spread.cu  (k_spread)
//   step 2 deconv+embed :235-238 -> folded into the Bluestein pre-chirp table P
//   step 3 FFT          :239     -> fft.cu     (pruned Bluestein, 1 or 3 kernels)
//   step 4 gather       :241-243 -> gather.cu  (k_gather, 1/phi_hat_1 fused)
#pragma once

#include <mutex>

#include "common.cuh"
#include "fft.cuh"
#include "window.cuh"

namespace sfb {

struct Geometry {
  int64_t N, M1, M2, N1, K, N2;
  int m1, m2;
  double sigma1, sigma2, a, beta1, beta2;
};

// Sources, sorted by cell c = floor(N1 v) + K/2 and grouped into "chunks" of
// at most kChunk sources of one cell.  Chunks of a tile of kTile cells are
// ordered rank-major (chunk rank within its cell, then cell), so a warp's 32
// consecutive chunks almost always have pairwise distinct cells, and padded
// with empty chunks to whole "blocks" of 32 (one chunk per lane), so a block
// belongs to one tile.  The sources are stored in chunk-slot order (chunk c
// owns slots [4c, 4c+4)), so a lane's positions and permutation are two
// contiguous 16-byte records.  The spread kernel is persistent: each warp
// walks a contiguous range of blocks (spread.cu).
#ifndef SFB_SPREAD_TILE
#define SFB_SPREAD_TILE 256
#endif
constexpr int kTile = SFB_SPREAD_TILE;
constexpr int kChunk = 4;
constexpr int kBlockChunks = 32;  // chunks per block = lanes per warp
#ifndef SFB_SPREAD_WARPS
#define SFB_SPREAD_WARPS 8
#endif
constexpr int kSpreadWarps = SFB_SPREAD_WARPS;  // warps per spread CTA (independent workers)

struct SpreadPlan {
  DevArray<double> pos;    // fl(N1 * v) in chunk-slot order    [n_blocks * 32 * kChunk]
  DevArray<int> perm;      // original source index, slot order [n_blocks * 32 * kChunk]
  DevArray<int> info;      // (local cell << 8) | count, 0 = empty [n_blocks * 32]
  DevArray<int> blk_tile;  // tile of each block                  [n_blocks]
  DevArray<int2> chunks;   // plan-time only: {first sorted index, info}
  DevArray<int64_t> wstart; // first block of each spread warp         [n_ctas * 8 + 1]
  int64_t n_chunks = 0, n_blocks = 0;
  int n_sms = 148, n_ctas = 1;
  // batched path (batched.cu): cell-sorted sources and per-128-cell tile starts
  DevArray<double> bpos;
  DevArray<int> bperm;
  DevArray<int> btile;
  // dense sources (>= kDenseMin per cell on average, e.g. fast-sinc stage 1):
  // per-cell window moments instead of per-source windows (spread.cu)
  DevArray<int4> units;    // {cell, first, end, 0}: <= kDenseUnit sources of one cell
  int64_t n_units = 0;
  bool dense = false;
};

constexpr int64_t kDenseMin = 64;   // average sources per cell from which the moment spread is used
#ifndef SFB_DENSE_UNIT
#define SFB_DENSE_UNIT 128
#endif
constexpr int kDenseUnit = SFB_DENSE_UNIT;  // sources per moment-spread unit (heavy cells are split)

constexpr int kBatchedMin = 16;  // columns from which the column-vectorised path is used

// Targets sorted by fl(N2 * xs); scale = 1/phi_hat_1(N x_j) in sorted order
// (optionally times an external per-target weight, used by the fast sinc
// transform to fuse alpha = w * g into stage 1).
// Targets are sorted by (j / kGatherSlice, fine-grid cell): slices of
// kGatherSlice original indices keep each CTA's scattered output stores inside
// a 16 MiB window of `out` (L2-resident; 2^20 measured best of 2^18..2^23).  kGatherSlice is a multiple of the
// gather CTA size, so no CTA straddles two slices.
constexpr int64_t kGatherSliceDefault = (int64_t)1 << 20;
int64_t gather_slice();  // kGatherSliceDefault unless SFB_GATHER_SLICE_LOG2 is set (tuning)

#ifndef SFB_GATHER_THREADS
#define SFB_GATHER_THREADS 128  // 128 x 8 CTAs/SM measured 3 % faster than 256 x 4
#endif
#ifndef SFB_GATHER_SPAN
#define SFB_GATHER_SPAN 1024
#endif
constexpr int kGatherThreads = SFB_GATHER_THREADS;  // threads per gather CTA
#ifndef SFB_GATHER_TPT
#define SFB_GATHER_TPT 2
#endif
constexpr int kGatherTPT = SFB_GATHER_TPT;                 // targets per thread
constexpr int kGatherGroup = kGatherThreads * kGatherTPT;  // targets per CTA
constexpr int kGatherSpan = SFB_GATHER_SPAN;  // h values staged per CTA (16 KiB)

struct GatherPlan {
  bool conj_out = false;  // store conj(out) (pairs with FftPlan::conj_in)
  DevArray<double> pos;
  DevArray<int> perm;
  DevArray<double> scale;
  DevArray<int2> span;  // per gather CTA: {klo, khi} h range (h index k' = s - s_lo)
  // the same records in "octet order" for the single-column gather (k_gather2):
  // inside every full group of kGatherGroup targets, the targets are dealt
  // to threads so that the 8 lanes of each quarter-warp have pairwise distinct
  // window starts mod 8 (or equal starts) -- their 16-byte shared-memory loads
  // of the staged h span are then free of bank conflicts (plan.cu
  // k_octet_order).  pos / scale / perm above stay position-sorted for the
  // batched gather's rolling windows.
  DevArray<double> opos, oscale;
  DevArray<int> operm;
};

// Pruned Bluestein: h_{s_lo + k'} = Q[k'] * sum_l (g_l P_l) b_{k'-l},
// k' in [0, Kout), l in [0, K), realised as a cyclic convolution of length
// L = L1 * L2 (7-smooth) via FFT.  Bhat = FFT_L(b)/L stored in the four-step
// "digit-reversed" layout the forward kernels produce.
// Direct four-step DFT of length N2 = A * P (used when it fits): step 1 does
// the A-point DFTs of the P columns x[P n1 + n2] in shared memory (A 7-smooth)
// reading only the K nonzero inputs; step 2 does the P-point DFTs of the A rows
// in shared memory -- directly when P is 7-smooth, else by an in-smem
// Bluestein of smooth length LP >= 2P-1 -- writing only the Kout outputs the
// gather reads.  Traffic ~16(K + 2 N2 + Kout) bytes instead of ~3 passes over L.
struct DirectFft {
  int64_t A = 0, P = 0, LP = 0;
  int C = 1, C_log2 = 0;  // step-1 columns per CTA
  int R = 1, R_log2 = 0;  // step-2 rows per CTA
  bool p_smooth = false;
  bool rader = false;      // P prime, P - 1 smooth: Rader rows of length LP = P - 1
  FftStages stA{}, stP{};  // stP: P (smooth), LP (Bluestein) or P - 1 (Rader)
  DevArray<double2> twA, twP, w_lo, w_hi, cp, bhat;
  DevArray<int> revA, revP, rin, rout;
  DevArray<double> D;      // 1 / (N1 N2 phi_hat_2(l - K/2)), l in [0, K)
};

struct FftPlan {
  int64_t L = 0, L1 = 0, L2 = 0, Kout = 0, s_lo = 0;
  double in_scale = 0.0;  // input factor: 1/(N1 N2) (NNFFT, with 1/phi_hat_2), 1/n_over (NFFT)
  int64_t fixD = 0;       // L = K + Kout - 1 - fixD: outputs k' < fixD corrected (fft.cu)
  DevArray<double2> fixc; // the correction's correlation kernel [fixD]
  bool conj_in = false;   // inverse DFT as conj(F(conj x)) (NFFT trafo; gather conjugates)
  int C = 1, C_log2 = 0;  // columns per CTA in the column kernels
  bool single = true;     // L fits one CTA
  bool direct = false;    // DirectFft path instead of the Bluestein over L
  FftStages st1{}, st2{}; // L1 (rows / single) and L2 (columns)
  DevArray<double2> tw1, tw2, tw_lo, tw_hi;
  DevArray<int> rev2;
  DevArray<double2> P, Q, Bhat;
  // radix-16 register passes of the config-3 shape: x16 = 1 rows, 2 rows and
  // columns; their stages, twiddles, and Bhat permuted to their output order
  int x16 = 0;
  FftStages st1x{}, st2x{};
  DevArray<double2> tw1x, tw2x, Bhatx;
  DirectFft d;
  // scratch elements per column for run_fft's `work`
  int64_t work_elems() const { return single ? 0 : direct ? d.A * d.P : L; }
};

struct NnfftPlanImpl {
  Geometry g{};
  int device = 0;
  // h window [s_lo, s_lo + Kout) from the geometry (|x| <= 1/2) instead of
  // the targets' extent, so plans over different target shards share one FFT
  // (the distributed FFT needs identical L, Kout, chirps on every rank)
  bool full_window = false;
  WinCoef c1{}, c2{};
  SpreadPlan sp;
  GatherPlan gp;
  FftPlan fft;
  DevArray<double> v_clip, x_clip;  // original order, for export_tables
  DevArray<double> hat2;            // phi_hat_2 at l - K/2          [K]
};

// Adjoint NNFFT sub-plans (adjoint.cu), built lazily from a forward plan
struct NnfftAdjoint {
  int64_t halo = 0;
  DevArray<double> s1;      // 1/phi_hat_1(N x_j), original order
  NnfftPlanImpl spread_x;   // spread at N2 xs onto N2 + 2 halo points (window 2)
  NnfftPlanImpl fft;        // N2 folded inputs -> K outputs at l - K/2 (conjugated)
  NnfftPlanImpl gather_v;   // gather over the K-grid at N1 v (window 1)
};
void build_adjoint(const NnfftPlanImpl& p, NnfftAdjoint& a, cudaStream_t stream);
// y: (M2, batch) row-major -> out: (M1, batch) row-major, device pointers
void run_adjoint(const NnfftPlanImpl& p, const NnfftAdjoint& a, const double2* y, double2* out,
                 int batch, cudaStream_t stream);

// ----- plan.cu
Geometry make_geometry(int64_t N, int64_t M1, int64_t M2, double sigma1, double sigma2, int m1,
                       int m2);
// v, x are device pointers (original order, unclipped) on `stream`.
void build_plan(NnfftPlanImpl& p, const double* v_dev, const double* x_dev, cudaStream_t stream);
// the two halves of build_plan, reused by the classical NFFT (nfft.cu)
struct TargetScale {
  bool hat1 = false;  // scale = 1/phi_hat_1(N x) (NNFFT) or 1 (NFFT)
  double N = 0.0, beta1 = 0.0;
  int m1 = 0;
  int64_t N1 = 0;
};
void build_sources(NnfftPlanImpl& p, const double* v, int64_t M1, double N1, int64_t K,
                   cudaStream_t stream);
// positions pos_scale * (ratio * x); N2 = the periodic length the gather
// wraps at (and the clamp of Kout)
void build_targets(NnfftPlanImpl& p, const double* x, int64_t M2, double ratio, double pos_scale,
                   int64_t N2, int m2, const TargetScale& ts, cudaStream_t stream,
                   int64_t force_s_lo = 0, int64_t force_kout = 0);
// multiply the gather scale by per-target weights (device, original order)
void fuse_target_weights(NnfftPlanImpl& p, const double* w_dev, cudaStream_t stream);

// ----- fft.cu
void octet_order(NnfftPlanImpl& p, int64_t M2, cudaStream_t stream);  // GatherPlan::opos/oscale/operm
void build_fft(NnfftPlanImpl& p, cudaStream_t stream);
// grid[batch][K] -> h[batch][Kout] (work: batch*L complex scratch)
// grid_padded: grid holds whole rows of L1 (ceil(K / L1) * L1 elements per
// column) -- the TMA column pass reads rows past K (zeroed by run_fft)
void run_fft(const NnfftPlanImpl& p, const double2* grid, double2* h, double2* work, int batch,
             cudaStream_t stream, bool grid_padded = false);
// point-major variant: grid[K][batch] -> h[Kout][batch] (Bluestein path only)
bool fft_supports_point_major(const NnfftPlanImpl& p);
// Distributed (column-split) FFT over `world` ranks (fft.cu; layouts there).
struct DistLayout {
  bool ok;
  int64_t Bc, Br;  // columns / rows per rank
  int64_t I, K2;   // grid rows ceil(K/L1), output rows ceil(Kout/L1)
  int64_t Sb;      // elements per rank block of the reduce-scatter buffer
};
bool dist_layout(const NnfftPlanImpl& p, int world, DistLayout* out);
// plan.cu: [n_lo, n_hi] grid indices of the plan's spread, [k_lo, k_hi] h
// indices of its gather (for the sparse exchange of position partitions)
void dist_support(const NnfftPlanImpl& p, cudaStream_t s, int64_t out[4]);
// Sparse (position-partitioned) exchange: row ranges per rank
constexpr int kDistMaxRanks = 16;
struct RowSplit {
  int n;
  int64_t lo[kDistMaxRanks], cnt[kDistMaxRanks], off[kDistMaxRanks];
};
void run_dist_pack_rows(const NnfftPlanImpl& p, int world, const double2* grid, int64_t ilo,
                        int64_t nrow, double2* send, cudaStream_t s);
void run_dist_unpack_rows(const NnfftPlanImpl& p, int world, int rank, const double2* recv,
                          const int64_t* ilo, const int64_t* nrow, double2* block,
                          cudaStream_t s);
void run_dist_pack_hrows(const NnfftPlanImpl& p, int world, const double2* hblk,
                         const int64_t* k2lo, const int64_t* cnt, double2* send, cudaStream_t s);
void run_dist_unpack_hrows(const NnfftPlanImpl& p, int world, const double2* recv, int64_t k2lo,
                           int64_t cnt, double2* h, cudaStream_t s);
void run_dist_pack(const NnfftPlanImpl& p, int world, const double2* grid, double2* S,
                   cudaStream_t s);
void run_dist_colfwd(const NnfftPlanImpl& p, int world, int rank, const double2* R, double2* Yc,
                     cudaStream_t s);
void run_dist_rowmul(const NnfftPlanImpl& p, int world, int rank, double2* Rr, cudaStream_t s);
// the same two passes storing straight into the owners' receive buffers
// (peers[q]: rank q's buffer, this process's view; the all-to-all layouts)
void run_dist_colfwd_peer(const NnfftPlanImpl& p, int world, int rank, const double2* R,
                          double2* const* peers, cudaStream_t s);
void run_dist_rowmul_peer(const NnfftPlanImpl& p, int world, int rank, double2* Rr,
                          double2* const* peers, cudaStream_t s);
// fused first / last exchanges: pack the grid rows into every receiver's
// buffer at this sender's offsets; the inverse column pass stores h rows into
// every rank whose targets read them (rank 0 adds the summed tail fix)
void run_dist_pack_rows_peer(const NnfftPlanImpl& p, int world, int rank, const double2* grid,
                             int64_t ilo, int64_t nrow, double2* const* peers,
                             const int64_t* poff, cudaStream_t s);
void run_dist_colinv_peer(const NnfftPlanImpl& p, int world, int rank, const double2* Y2,
                          const double2* R, double2* const* peers, const int64_t* k2lo,
                          const int64_t* cnt, cudaStream_t s);
void run_dist_colinv(const NnfftPlanImpl& p, int world, int rank, const double2* Y2,
                     const double2* R, double2* H, cudaStream_t s);
void run_dist_unpack(const NnfftPlanImpl& p, int world, const double2* Hall, double2* h,
                     cudaStream_t s);
// columns per group of the point-major FFT (its work array holds L x group)
int fft_point_major_group(int batch);
void run_fft_point_major(const NnfftPlanImpl& p, const double2* grid, double2* h, double2* work,
                         int batch, cudaStream_t stream);

// ----- spread.cu / gather.cu
// f: (M1, batch) row-major; grid[batch][K] is zeroed and accumulated.
void run_spread(const NnfftPlanImpl& p, const double2* f, double2* grid, int batch,
                cudaStream_t stream);
void run_spread_zero(const NnfftPlanImpl& p, double2* grid, int batch, cudaStream_t s);
void run_spread_kernel(const NnfftPlanImpl& p, const double2* f, double2* grid, int batch,
                       cudaStream_t s);
// real-valued coefficients (fast sinc input), batch 1
void run_spread_real(const NnfftPlanImpl& p, const double* f, double2* grid, cudaStream_t stream);
// out: (M2, batch) row-major, original target order.
void run_gather(const NnfftPlanImpl& p, const double2* h, double2* out, int batch,
                cudaStream_t stream);

// whole transform with device pointers (scratch allocated stream-ordered)
void run_execute(const NnfftPlanImpl& p, const double2* f, double2* out, int batch,
                 cudaStream_t stream);
// ----- direct.cu: exact O(M1 M2) sums (reference direct.py), device pointers
void run_nndft_direct(const double2* f, const double* v, int64_t M1, const double* x,
                      int64_t M2, double N, double2* out, cudaStream_t stream);
void run_ndft_direct(const double2* c, int64_t Nc, const double* x, int64_t M, double2* out,
                     cudaStream_t stream);
// public window evaluation (window.cu): func 0 omega, 1 omega_hat, 2 phi, 3 phi_hat
void run_window_eval(int func, double beta, int m, int64_t n_grid, const double* x, int64_t n,
                     double* out, cudaStream_t s);
void run_sinc_direct(const double2* c, const double* a, int64_t L1, const double* b, int64_t L2,
                     double N, double2* out, cudaStream_t stream);
// ----- batched.cu: batch >= kBatchedMin columns, columns across lanes
// ev (optional): 4 events recorded around spread | transpose+FFT+transpose | gather
void run_execute_batched(const NnfftPlanImpl& p, const double2* f, double2* out, int batch,
                         cudaStream_t stream, cudaEvent_t* ev = nullptr);

}  // namespace sfb
