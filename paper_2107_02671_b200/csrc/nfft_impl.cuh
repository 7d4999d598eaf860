// nfft_impl.cuh -- device-resident classical NFFT plan (reference nfft.py,
// SURVEY.md 8f row f1): three NNFFT sub-plans sharing the NNFFT kernels.
#pragma once

#include "nnfft_impl.cuh"

namespace sfb {

struct NfftPlanImpl {
  int64_t N = 0, M = 0, n_over = 0;  // degree, nodes, oversampled grid sigma N
  int m = 0;
  double sigma = 0.0, beta = 0.0;
  int device = 0;
  int64_t halo = 0;                  // adjoint grid halo h = m + 1 per side
  DevArray<double> x_clip, hat;      // nodes (original order), phi_hat on I_N
  NnfftPlanImpl tr;                  // trafo: FFT (K = N, conj) + gather (grid n_over)
  NnfftPlanImpl ad_spread;           // adjoint: spread on n_over + 2h points
  NnfftPlanImpl ad_fft;              // adjoint: FFT of the folded n_over points -> I_N
};

// x_dev: device nodes (original order, unclipped) on `stream`
void build_nfft(NfftPlanImpl& p, int64_t N, int64_t M, double sigma, int m, const double* x_dev,
                int device, cudaStream_t stream);
// c[N] -> out[M]  (nfft.py:99-109);  y[M] -> out[N]  (nfft.py:112-123); device pointers
void run_nfft_trafo(const NfftPlanImpl& p, const double2* c, double2* out, cudaStream_t stream);
void run_nfft_adjoint(const NfftPlanImpl& p, const double2* y, double2* out, cudaStream_t stream);
// reference-layout plan tables: spread_idx/val [M x 2m] (device), hat [N] (device)
void export_nfft(const NfftPlanImpl& p, int64_t* idx, double* val, double* hat,
                 cudaStream_t stream);

}  // namespace sfb
