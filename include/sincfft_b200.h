/*
 * sincfft_b200.h -- C ABI of the B200-native NNFFT / fast sinc transform.
 *
 * This is the drop-in boundary for the hot path named by BASELINE.json's
 * north star.  The reference (arXiv 2107.02671, package `sincfft`) is pure
 * Python and has no FFI; its "operator API" is a handful of Python
 * functions.  Every entry point below replaces one of them and is bound from
 * Python through ctypes (paper_2107_02671_b200/_lib.py); INTEGRATION.md shows
 * the binding a maintainer of the reference would add.
 *
 * Conventions
 *   - complex arrays are interleaved (re, im) doubles, i.e. numpy complex128;
 *   - a batch of B coefficient vectors is an (M1, B) row-major array
 *     (column b of F is F[:, b]); outputs are (M2, B) row-major;
 *   - `ptr_kind` says whether user pointers are host (SINCFFT_PTR_HOST,
 *     copied inside the call; SINCFFT_PTR_HOST_ASYNC: same, without the final
 *     synchronisation) or device (SINCFFT_PTR_DEVICE) memory;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); all work of
 *     one call is ordered on it, and host-pointer calls synchronize it before
 *     returning;
 *   - every function returns a status code; on failure
 *     sincfft_last_error() returns a thread-local message.
 *   - plans are immutable after creation; concurrent execute calls on one
 *     plan are allowed (scratch memory is stream-ordered per call), matching
 *     the reference contract.
 */
#ifndef SINCFFT_B200_H
#define SINCFFT_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define SINCFFT_API __attribute__((visibility("default")))
#else
#define SINCFFT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python shim maps them to the reference's exception
 * classes (ref: pkg/src/sincfft/errors.py:4-13) */
#define SINCFFT_OK 0
#define SINCFFT_EPARAM 1       /* -> sincfft.errors.ParameterError        */
#define SINCFFT_EPOSITIVITY 2  /* -> sincfft.errors.PositivityError       */
#define SINCFFT_ECUDA 3        /* CUDA runtime failure (RuntimeError)     */
#define SINCFFT_ENOMEM 4       /* device allocation failed (MemoryError)  */
#define SINCFFT_EUNSUPPORTED 5 /* outside the implemented envelope        */

#define SINCFFT_PTR_HOST 0       /* host memory; the call returns when done   */
#define SINCFFT_PTR_DEVICE 1     /* device memory, stream-ordered             */
#define SINCFFT_PTR_HOST_ASYNC 2 /* host memory (page-locked for overlap): the
                                  * copies and kernels are enqueued on `stream`
                                  * and the call returns at once; the caller
                                  * synchronizes `stream` before reading `out`
                                  * or reusing `f` (pipelined batches)        */

typedef struct sincfft_nnfft_plan_s *sincfft_nnfft_plan;
typedef struct sincfft_sinc_plan_s *sincfft_sinc_plan;
typedef struct sincfft_nfft_plan_s *sincfft_nfft_plan;

/* fast sinc layouts (sincfft.fast_sinc.SincMode, fast_sinc.py:32-38) */
#define SINCFFT_SINC_GENERAL 0
#define SINCFFT_SINC_EQUISPACED_SOURCES 1
#define SINCFFT_SINC_EQUISPACED_TARGETS 2
#define SINCFFT_SINC_EQUISPACED_BOTH 3

/* Geometry of a plan (ref: NnfftGeometry, pkg/src/sincfft/nnfft.py:30-89). */
typedef struct {
  int64_t N, M1, M2, N1, K, N2;
  int32_t m1, m2;
  double sigma1, sigma2, a, beta1, beta2;
  /* FFT realisation: pruned Bluestein of length L = L1*L2 over the
   * Kout = s_hi - s_lo + 1 outputs the gather reads */
  int64_t L, L1, L2, Kout, s_lo;
} sincfft_geometry;

/* Thread-local description of the last failure ("" if none). */
SINCFFT_API const char *sincfft_last_error(void);

/* ABI version (major*10000 + minor*100 + patch). */
SINCFFT_API int sincfft_version(void);

/* Number of visible CUDA devices (0 if none / no driver). */
SINCFFT_API int sincfft_device_count(void);

/* --- NNFFT (Algorithm 2.1) ---------------------------------------------
 * Replaces sincfft.nnfft.nnfft_plan (pkg/src/sincfft/nnfft.py:131-207).
 * N is the (already rescaled) bandwidth N*, v[M1] frequencies with
 * |v| <= 1/(2a) (+1e-12; clipped), x[M2] nodes in [-1/2, 1/2] (+1e-12;
 * clipped).  Only the sinh window is implemented (north star); m1, m2 in
 * [2, 16].  Validation follows nnfft.py:51-89,152-183 and fails with
 * SINCFFT_EPARAM / SINCFFT_EPOSITIVITY. */
SINCFFT_API int sincfft_nnfft_plan_create(sincfft_nnfft_plan *plan, int64_t N, int64_t M1, int64_t M2,
                              double sigma1, double sigma2, int32_t m1, int32_t m2,
                              const double *v, const double *x, int32_t ptr_kind,
                              int32_t device, void *stream);

/* As sincfft_nnfft_plan_create, with flags.  SINCFFT_PLAN_FULL_WINDOW: size
 * the gather's h window [s_lo, s_lo + Kout) from the geometry (every
 * |x| <= 1/2) instead of this plan's target extent, so plans built over
 * different target shards of one problem share an identical FFT (required by
 * the distributed FFT below; outputs equal the default plan's to rounding). */
#define SINCFFT_PLAN_FULL_WINDOW 1
SINCFFT_API int sincfft_nnfft_plan_create_ex(sincfft_nnfft_plan *plan, int64_t N, int64_t M1,
                                             int64_t M2, double sigma1, double sigma2, int32_t m1,
                                             int32_t m2, const double *v, const double *x,
                                             int32_t ptr_kind, int32_t device, int32_t flags,
                                             void *stream);

SINCFFT_API int sincfft_nnfft_plan_destroy(sincfft_nnfft_plan plan);

SINCFFT_API int sincfft_nnfft_plan_geometry(sincfft_nnfft_plan plan, sincfft_geometry *geo);

/* Replaces sincfft.nnfft.nnfft_trafo (nnfft.py:210-243), extended to B
 * columns sharing one plan (the reference applied column by column).
 * f: (M1, batch) complex, out: (M2, batch) complex. */
SINCFFT_API int sincfft_nnfft_execute(sincfft_nnfft_plan plan, const double *f, double *out,
                          int64_t batch, int32_t ptr_kind, void *stream);

/* Split execute for source-sharded multi-GPU runs: step 1 only (spread onto
 * the K-grid, device buffer grid[batch][K] complex, overwritten), and steps
 * 2-4 (deconvolution + FFT + gather) from a caller-supplied (e.g. all-reduced)
 * device grid.  execute == spread followed by finish. */
SINCFFT_API int sincfft_nnfft_spread(sincfft_nnfft_plan plan, const double *f, double *grid_dev,
                         int64_t batch, int32_t ptr_kind, void *stream);
SINCFFT_API int sincfft_nnfft_finish(sincfft_nnfft_plan plan, const double *grid_dev, double *out,
                         int64_t batch, int32_t ptr_kind, void *stream);

/* Distributed FFT for source- and target-sharded runs (
 * additive, no reference counterpart).  Instead of all-reducing the K-grid
 * and replicating the FFT, the three Bluestein passes are split over the
 * `world` ranks (rank r: columns [r Bc, (r+1) Bc) and rows [r Br, (r+1) Br))
 * and the caller runs four collectives between five steps (all device
 * pointers, complex doubles, single column, stream-ordered):
 *   dist_pack(grid)            -> send[world * Sb]   ; reduce-scatter(sum) -> block[Sb]
 *   dist_colfwd(block)         -> cols[L2 * Bc]      ; all-to-all (equal splits) -> rows
 *   dist_rowmul(rows)             in place           ; all-to-all -> cols2[L2 * Bc]
 *   dist_colinv(cols2, block)  -> hblk[K2 * Bc]      ; all-gather -> hall[world * K2 * Bc]
 *   dist_gather(hall)          -> out[M2] for this plan's targets
 * Plans of all ranks must be built with SINCFFT_PLAN_FULL_WINDOW over the
 * same N, sigma, m.  dist_layout: sizes[0] = 1 if the plan and world size are
 * supported (the config-3 shape 4096 x 1024, world a power of two dividing
 * both), sizes[1] = Sb, sizes[2] = L2 * Bc, sizes[3] = K2 * Bc, sizes[4] = Bc,
 * sizes[5] = Br (element counts of complex doubles). */
SINCFFT_API int sincfft_nnfft_dist_layout(sincfft_nnfft_plan plan, int32_t world, int64_t *sizes);
SINCFFT_API int sincfft_nnfft_dist_pack(sincfft_nnfft_plan plan, int32_t world,
                                        const double *grid_dev, double *send_dev, void *stream);
SINCFFT_API int sincfft_nnfft_dist_colfwd(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                                          const double *block_dev, double *cols_dev, void *stream);
SINCFFT_API int sincfft_nnfft_dist_rowmul(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                                          double *rows_dev, void *stream);
SINCFFT_API int sincfft_nnfft_dist_colinv(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                                          const double *cols_dev, const double *block_dev,
                                          double *hblk_dev, void *stream);
SINCFFT_API int sincfft_nnfft_dist_gather(sincfft_nnfft_plan plan, int32_t world,
                                          const double *hall_dev, double *out_dev, void *stream);

/* Sparse exchange variant of the distributed FFT for POSITION partitions
 * (each rank's sources cover a contiguous grid range, its targets a
 * contiguous h range): the reduce-scatter and the all-gather above become
 * all-to-alls of only the rows a rank touches.  grid row i = grid indices
 * [i L1, (i+1) L1), h row k2 = h indices [k2 L1, (k2+1) L1).
 *   dist_support(out4)   -> [n_lo, n_hi] grid indices spread, [k_lo, k_hi] h
 *                           indices gathered by this plan (host values)
 *   dist_pack_rows(grid, ilo, nrow) -> send: world chunks, chunk q = rows
 *                           [ilo, ilo + nrow) of column block q ([i][c]);
 *                           chunk 0 carries Dpad = ceil8(D) more elements (this
 *                           rank's Bluestein tail fix)         ; all-to-all(v)
 *   dist_unpack_rows(recv, ilo[world], nrow[world]) -> block[Sb] (rows of
 *                           every sender summed; rank 0 also sums the fixes)
 *   ... dist_colfwd / all-to-all / dist_rowmul / all-to-all / dist_colinv ...
 *   dist_pack_hrows(hblk, k2lo[world], cnt[world]) -> send: chunk r = rows
 *                           [k2lo_r, k2lo_r + cnt_r) of this rank's h block
 *                                                              ; all-to-all(v)
 *   dist_gather_rows(recv, k2lo, cnt) -> out[M2] (own h rows, then the gather) */
SINCFFT_API int sincfft_nnfft_dist_support(sincfft_nnfft_plan plan, int64_t *out4, void *stream);
SINCFFT_API int sincfft_nnfft_dist_pack_rows(sincfft_nnfft_plan plan, int32_t world,
                                             const double *grid_dev, int64_t ilo, int64_t nrow,
                                             double *send_dev, void *stream);
SINCFFT_API int sincfft_nnfft_dist_unpack_rows(sincfft_nnfft_plan plan, int32_t world,
                                               int32_t rank, const double *recv_dev,
                                               const int64_t *ilo, const int64_t *nrow,
                                               double *block_dev, void *stream);
SINCFFT_API int sincfft_nnfft_dist_pack_hrows(sincfft_nnfft_plan plan, int32_t world,
                                              const double *hblk_dev, const int64_t *k2lo,
                                              const int64_t *cnt, double *send_dev, void *stream);
SINCFFT_API int sincfft_nnfft_dist_gather_rows(sincfft_nnfft_plan plan, int32_t world,
                                               const double *recv_dev, int64_t k2lo, int64_t cnt,
                                               double *out_dev, void *stream);

/* Fused transposes over peer memory (additive): the two middle all-to-alls
 * of the distributed FFT replaced by stores into the owners' receive buffers.
 * Every rank allocates its rows buffer (L2 * Bc complex) and cols2 buffer
 * with sincfft_ipc_alloc, exchanges sincfft_ipc_handle()s (64 bytes) through
 * the process group and maps the peers' buffers with sincfft_ipc_open (NVLink
 * P2P between the GPUs of a node).  Per transform:
 *   dist_colfwd_peer(block, peers = rows buffers of all ranks)  ; barrier
 *   dist_rowmul_peer(own rows, peers = cols2 buffers of all ranks) ; barrier
 *   dist_colinv(own cols2, ...) as before.
 * peers[q] is rank q's buffer as mapped in this process (its own for q == rank). */
SINCFFT_API int sincfft_ipc_alloc(int32_t device, int64_t bytes, void **ptr);
SINCFFT_API int sincfft_ipc_free(void *ptr);
SINCFFT_API int sincfft_ipc_handle(void *ptr, uint8_t *handle64);
SINCFFT_API int sincfft_ipc_open(int32_t device, const uint8_t *handle64, void **ptr);
SINCFFT_API int sincfft_ipc_close(void *ptr);
SINCFFT_API int sincfft_nnfft_dist_colfwd_peer(sincfft_nnfft_plan plan, int32_t world,
                                               int32_t rank, const double *block_dev,
                                               const uint64_t *peers, void *stream);
SINCFFT_API int sincfft_nnfft_dist_rowmul_peer(sincfft_nnfft_plan plan, int32_t world,
                                               int32_t rank, double *rows_dev,
                                               const uint64_t *peers, void *stream);
/* The first and last exchanges fused the same way: pack_rows_peer writes
 * chunk q straight into receiver q's grid-row buffer at poff[q] (this
 * sender's offset there; chunks to rank 0 carry the tail fix), and
 * colinv_peer stores each h row into every rank r whose targets read it
 * (rows [k2lo[r], k2lo[r] + cnt[r]), receiver layout [sender][row][c]);
 * rank 0 adds the summed tail fix from its block.  Barrier after each. */
SINCFFT_API int sincfft_nnfft_dist_pack_rows_peer(sincfft_nnfft_plan plan, int32_t world,
                                                  int32_t rank, const double *grid_dev,
                                                  int64_t ilo, int64_t nrow,
                                                  const uint64_t *peers, const int64_t *poff,
                                                  void *stream);
SINCFFT_API int sincfft_nnfft_dist_colinv_peer(sincfft_nnfft_plan plan, int32_t world,
                                               int32_t rank, const double *cols_dev,
                                               const double *block_dev, const uint64_t *peers,
                                               const int64_t *k2lo, const int64_t *cnt,
                                               void *stream);

/* Observability: one execute with DEVICE pointers and CUDA events recorded
 * on `stream` between the stages; returns after synchronizing the stream
 * with stage_ms[0..3] = spread kernel (single column: the grid memset runs
 * before the first event; batched: the halo-row zeroing is included), FFT
 * (deconvolution + pruned Bluestein), gather, whole call (grid zeroing
 * included), in milliseconds. */
SINCFFT_API int sincfft_nnfft_execute_profiled(sincfft_nnfft_plan plan, const double *f,
                                               double *out, int64_t batch, void *stream,
                                               double *stage_ms);

/* Number of kernel launches one execute of `batch` columns issues. */
SINCFFT_API int sincfft_nnfft_launches_per_execute(sincfft_nnfft_plan plan, int64_t batch);

/* Materialise the reference's step-0 tables (NnfftPlan.spread_idx/_val,
 * gather_idx/_val, hat1, hat2; nnfft.py:92-107,175-205) into HOST buffers,
 * in the reference's layout, from the device-side plan.  Any pointer may be
 * NULL to skip that table.  Used by drop-in callers that inspect plans and by
 * the parity tests of the window evaluation. */
SINCFFT_API int sincfft_nnfft_export_tables(sincfft_nnfft_plan plan, int64_t *spread_idx, double *spread_val,
                                int64_t *gather_idx, double *gather_val, double *hat1,
                                double *hat2);

/* Adjoint NNFFT (BASELINE north star "adjoint-NNFFT entry point"; SURVEY.md
 * 8f row f4; not in the reference): the exact conjugate transpose of
 * sincfft_nnfft_execute on the same plan, out_k ~ sum_j y_j e^{+2 pi i N v_k x_j}.
 * y: (M2, batch) row-major complex, out: (M1, batch).  The adjoint's
 * sub-plans are built on the first call (thread-safe) and kept with the plan. */
SINCFFT_API int sincfft_nnfft_adjoint(sincfft_nnfft_plan plan, const double *y, double *out,
                                      int64_t batch, int32_t ptr_kind, void *stream);

/* --- fast sinc transform (Algorithm 6.3, all four layouts) ---------------
 * Replaces sincfft.fast_sinc.sinc_plan (fast_sinc.py:123-223).  The caller
 * supplies the Clenshaw-Curtis points z[n+1] and weights w[n+1] (host
 * plan-time data, sinc_approx.py:97-106), the rescaled bandwidth n_star
 * (fast_sinc.py:97-107) and the layout `mode` (SINCFFT_SINC_*, detected or
 * forced by the caller exactly as fast_sinc.py:171-192).  Stage 1 is the
 * NNFFT (n_star, a*N/n_star, z/2) (fast_sinc.py:205-209) or, for equispaced
 * sources, the NFFT trafo (L1, wrap(-(N/(2 L1)) z)) (:200-203); stage 3 is
 * the NNFFT (n_star, -(N/n_star) z/2, b) (:216-220) or, for equispaced
 * targets (L2 = N), the NFFT adjoint (N, -z/2) (:211-214). */
SINCFFT_API int sincfft_sinc_plan_create(sincfft_sinc_plan *plan, int64_t N, int64_t n_star, int64_t L1,
                             int64_t L2, int64_t n, const double *z, const double *w,
                             const double *a, const double *b, double sigma1, double sigma2,
                             int32_t m1, int32_t m2, int32_t mode, int32_t ptr_kind,
                             int32_t device, void *stream);

SINCFFT_API int sincfft_sinc_plan_destroy(sincfft_sinc_plan plan);

/* Geometry of the two inner plans (stage 1: sources -> Chebyshev nodes,
 * stage 3: Chebyshev nodes -> targets). */
SINCFFT_API int sincfft_sinc_plan_geometry(sincfft_sinc_plan plan, sincfft_geometry *stage1,
                               sincfft_geometry *stage3);

/* Replaces sincfft.fast_sinc.fast_sinc_transform (fast_sinc.py:226-249).
 * c: L1 coefficients, complex (c_is_real = 0) or real fp64 (c_is_real = 1,
 * the reference promotes real input to complex128); out: L2 complex. */
SINCFFT_API int sincfft_sinc_execute(sincfft_sinc_plan plan, const double *c, int32_t c_is_real,
                         double *out, int32_t ptr_kind, void *stream);

/* The two stages of sincfft_sinc_execute, for source/target-sharded runs
 * (additive): stage1 writes alpha = w .* (stage-1 transform of c) at the n+1
 * Clenshaw-Curtis nodes into a caller device buffer (linear in c, so partial
 * alphas of source shards sum -- one all-reduce of (n+1) complex); stage3
 * evaluates this plan's targets from alpha.  Device pointers, stream-ordered. */
SINCFFT_API int sincfft_sinc_stage1(sincfft_sinc_plan plan, const double *c, int32_t c_is_real,
                                    double *alpha_dev, void *stream);
SINCFFT_API int sincfft_sinc_stage3(sincfft_sinc_plan plan, const double *alpha_dev,
                                    double *out_dev, void *stream);

/* --- classical NFFT ---------------------------------
 * Replaces sincfft.nfft (nfft.py:53-123), sinh window: nfft_plan(N, x,
 * sigma, m) -> sincfft_nfft_plan_create (N even, sigma N an even integer,
 * 2m <= sigma N / 2, |x| <= 1/2 + 1e-12, same messages and status classes);
 * nfft_trafo: c[N] (I_N = -N/2 .. N/2-1) -> out[M]; nfft_adjoint: y[M] ->
 * out[N].  export_tables fills the reference plan's spread_idx / spread_val
 * ([M x 2m], host) and hat ([N], host); NULL skips a table. */
SINCFFT_API int sincfft_nfft_plan_create(sincfft_nfft_plan *plan, int64_t N, int64_t M, double sigma,
                                         int32_t m, const double *x, int32_t ptr_kind,
                                         int32_t device, void *stream);
SINCFFT_API int sincfft_nfft_plan_destroy(sincfft_nfft_plan plan);
SINCFFT_API int sincfft_nfft_plan_geometry(sincfft_nfft_plan plan, int64_t *n_over,
                                           sincfft_geometry *trafo, sincfft_geometry *adjoint);
SINCFFT_API int sincfft_nfft_trafo(sincfft_nfft_plan plan, const double *c, double *out,
                                   int32_t ptr_kind, void *stream);
SINCFFT_API int sincfft_nfft_adjoint(sincfft_nfft_plan plan, const double *y, double *out,
                                     int32_t ptr_kind, void *stream);
SINCFFT_API int sincfft_nfft_export_tables(sincfft_nfft_plan plan, int64_t *spread_idx,
                                           double *spread_val, double *hat);

/* --- exact quadratic-cost sums ---------------------
 * The reference's oracles (pkg/src/sincfft/direct.py), fp64 on the GPU, with
 * the phase carried in two doubles and compensated sums (at least as
 * accurate as the reference's).  Inputs/outputs follow `ptr_kind`; the call
 * synchronizes `stream` for host pointers.  Replace, in order:
 *   nndft_direct          direct.py:28-64   out_j = sum_k f_k e^{-2 pi i N v_k x_j}
 *   ndft_direct           direct.py:67-90   out_j = sum_{k in I_Nc} c_k e^{2 pi i k x_j}
 *                                           (Nc even, k = -Nc/2 .. Nc/2-1)
 *   sinc_transform_direct direct.py:93-112  out_j = sum_k c_k sinc(N pi (b_j - a_k)) */
SINCFFT_API int sincfft_nndft_direct(const double *f, const double *v, int64_t M1, const double *x,
                                     int64_t M2, int64_t N, double *out, int32_t ptr_kind,
                                     int32_t device, void *stream);
SINCFFT_API int sincfft_ndft_direct(const double *c, int64_t Nc, const double *x, int64_t M,
                                    double *out, int32_t ptr_kind, int32_t device, void *stream);
SINCFFT_API int sincfft_sinc_direct(const double *c, const double *a, int64_t L1, const double *b,
                                    int64_t L2, int64_t N, double *out, int32_t ptr_kind,
                                    int32_t device, void *stream);

/* ---- public window functions (sinh kind) ------------------------------------
 * Replaces windows.py:106-125 (omega_eval), :135-160 (omega_hat_eval),
 * :212-214 (phi_eval), :217-220 (phi_hat_eval) of the reference for
 * kind = "sinh": out[i] = F(x[i]) with the reference's closed forms, evaluated
 * on the device.  func: SINCFFT_WIN_OMEGA, _OMEGA_HAT, _PHI, _PHI_HAT; beta is
 * the window shape 2 pi m (1 - 1/(2 sigma)); m and n_grid dilate phi / phi_hat
 * (phi(t) = omega(t n_grid/m), phi_hat(v) = (m/n_grid) omega_hat(v m/n_grid)).
 * n == 0 is a no-op. */
#define SINCFFT_WIN_OMEGA 0
#define SINCFFT_WIN_OMEGA_HAT 1
#define SINCFFT_WIN_PHI 2
#define SINCFFT_WIN_PHI_HAT 3
SINCFFT_API int sincfft_window_eval(int32_t func, double beta, int32_t m, int64_t n_grid,
                                    const double *x, int64_t n, double *out, int32_t ptr_kind,
                                    int32_t device, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SINCFFT_B200_H */
