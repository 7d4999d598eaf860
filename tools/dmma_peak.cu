// dmma_peak.cu -- does the FP64 tensor-core path (DMMA, mma.sync .f64) add
// throughput on top of the DFMA pipe on this B200?  Three kernels, each
// warp running independent chains: DFMA only, DMMA only (m8n8k4 and
// m16n8k16), and both interleaved in the same warp.  Prints TFLOP/s of each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void dmma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int MODE>  // 0 DFMA, 1 DMMA 884, 2 DMMA 16816, 3 DFMA + DMMA 884, 4 DFMA + DMMA 16816
__global__ void k_mix(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  double d[4][2];
  double e[2][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i][0] = d[i][1] = i;
#pragma unroll
  for (int i = 0; i < 2; ++i) e[i][0] = e[i][1] = e[i][2] = e[i][3] = i;
  double aa[8], bb[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) aa[i] = a + i * 1e-3;
#pragma unroll
  for (int i = 0; i < 4; ++i) bb[i] = b + i * 1e-3;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE >= 3) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    if (MODE == 1 || MODE == 3) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma884(d[i], a, b);
    }
    if (MODE == 2 || MODE == 4) {
#pragma unroll
      for (int i = 0; i < 2; ++i) dmma16816(e[i], aa, bb);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
#pragma unroll
  for (int i = 0; i < 2; ++i) s += e[i][0] + e[i][1] + e[i][2] + e[i][3];
  if (s == 42.0) out[0] = s;
}

template <int MODE>
void run(const char* name, int sms, double* out) {
  const int threads = 256, blocks = sms * 4, iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mix<MODE><<<blocks, threads>>>(out, 10, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_mix<MODE><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double warps = (double)blocks * threads / 32.0;
  double dfma = 0, dmma = 0;
  if (MODE == 0 || MODE >= 3) dfma = 2.0 * 8 * iters * warps * 32;
  if (MODE == 1 || MODE == 3) dmma = 2.0 * 8 * 8 * 4 * 4 * iters * warps;
  if (MODE == 2 || MODE == 4) dmma = 2.0 * 16 * 8 * 16 * 2 * iters * warps;
  const double t = best * 1e-3;
  printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, "
         "\"total_tflops\": %.2f}\n",
         name, best, dfma / t / 1e12, dmma / t / 1e12, (dfma + dmma) / t / 1e12);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  run<0>("dfma", sms, out);
  run<1>("dmma_m8n8k4", sms, out);
  run<2>("dmma_m16n8k16", sms, out);
  run<3>("dfma+dmma_m8n8k4", sms, out);
  run<4>("dfma+dmma_m16n8k16", sms, out);
  return 0;
}
