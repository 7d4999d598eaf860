// randread.cu -- microbenchmark: cost of the spread's random f gather.
// Reads n double2 from a 256 MiB array through an index vector that is
// (a) a full random permutation, (b) random inside windows of W elements
// (the "slice" orderings), (c) sequential; and fp64 RED throughput into a
// 33.5 MB grid.  Prints ms per pass; run under ncu for dram bytes.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <numeric>
#include <random>
#include <cuda_runtime.h>

__global__ void k_read(const double2* __restrict__ f, const int* __restrict__ idx, int n,
                       double2* out) {
  double2 acc = make_double2(0, 0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double2 v = __ldg(f + idx[i]);
    acc.x += v.x;
    acc.y += v.y;
  }
  if (acc.x == 12345.0) out[0] = acc;
}

// variants of the same random 16-byte read: 0 ld.global.nc, 1 ld.global.cg
// (L2 only), 2 ld.global.nc.L2::64B, 3 ld.global.nc.L2::128B,
// 4 ld.global.nc.L1::no_allocate, 5 8-byte reads of .x only
template <int V>
__global__ void k_read_v(const double2* __restrict__ f, const int* __restrict__ idx, int n,
                         double2* out) {
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double2* p = f + idx[i];
    double a = 0.0, b = 0.0;
    if (V == 0) asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
    if (V == 1) asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
    if (V == 2) asm volatile("ld.global.nc.L2::64B.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
    if (V == 3) asm volatile("ld.global.nc.L2::128B.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
    if (V == 4)
      asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                   : "=d"(a), "=d"(b) : "l"(p));
    if (V == 5) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(a) : "l"(p));
    acc += a + b;
  }
  if (acc == 12345.0) out[0] = make_double2(acc, 0);
}

__global__ void k_red(double* g, const int* __restrict__ idx, int n, int K) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int p = idx[i] % K;
    atomicAdd(g + 2 * (size_t)p, 1.0);
    atomicAdd(g + 2 * (size_t)p + 1, 1.0);
  }
}

int main() {
  // L2G=32|64|128: cudaLimitMaxL2FetchGranularity before the context does any work
  if (const char* e = getenv("L2G")) {
    cudaError_t rc = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(e));
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    printf("L2 fetch granularity: asked %s, rc %d, now %zu\n", e, (int)rc, got);
  }
  const int n = 1 << 24;
  std::vector<int> h(n);
  double2* f;
  int* idx;
  double2* out;
  double* g;
  const int K = 2097184;
  cudaMalloc(&f, sizeof(double2) * n);
  cudaMalloc(&idx, sizeof(int) * n);
  cudaMalloc(&out, 16);
  cudaMalloc(&g, 16 * (size_t)K);
  cudaMemset(f, 0, sizeof(double2) * n);
  cudaMemset(g, 0, 16 * (size_t)K);
  std::mt19937 rng(1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long windows[] = {0, 1L << 24, 1L << 23, 1L << 22, 1L << 21, 1L << 20, 1L << 16};
  for (long W : windows) {
    std::iota(h.begin(), h.end(), 0);
    if (W > 0)
      for (long s = 0; s < n; s += W) std::shuffle(h.begin() + s, h.begin() + std::min<long>(n, s + W), rng);
    cudaMemcpy(idx, h.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      k_read<<<148 * 8, 256>>>(f, idx, n, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    printf("read window=%ld ms=%.4f  (%.1f GB/s useful)\n", W, best, 16.0 * n / best / 1e6);
  }
  {
    std::iota(h.begin(), h.end(), 0);
    std::shuffle(h.begin(), h.end(), rng);
    cudaMemcpy(idx, h.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
    auto run = [&](auto kern, const char* name) {
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        kern<<<148 * 8, 256>>>(f, idx, n, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
      }
      printf("variant %-28s random 16B reads: ms=%.4f\n", name, best);
    };
    run(k_read_v<0>, "ld.global.nc");
    run(k_read_v<1>, "ld.global.cg");
    run(k_read_v<2>, "ld.global.nc.L2::64B");
    run(k_read_v<3>, "ld.global.nc.L2::128B");
    run(k_read_v<4>, "nc.L1::no_allocate");
    run(k_read_v<5>, "8-byte .x only");
  }
  // RED: coalesced-ish (index i) vs random over the grid
  for (int mode = 0; mode < 2; ++mode) {
    std::iota(h.begin(), h.end(), 0);
    if (mode) std::shuffle(h.begin(), h.end(), rng);
    cudaMemcpy(idx, h.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      k_red<<<148 * 8, 256>>>(g, idx, n, K);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    printf("red mode=%s n=%d x2 ms=%.4f  (%.1f G red/s)\n", mode ? "random" : "sequential", n, best,
           2.0 * n / best / 1e6);
  }
  return 0;
}
