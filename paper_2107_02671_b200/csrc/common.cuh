// common.cuh -- shared helpers for the B200 NNFFT library (sm_100a, fp64).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

// Bounds-checked build (make EXTRA=-DSFB_BOUNDS=1): device-side asserts on the
// indices of every shared-memory accumulator / staging buffer and of the
// table-driven global accesses of the hot kernels.  compute-sanitizer is
// closed on this project's GPU pool, so this build, run over the GPU test
// suite and tools/sanitize_cases.py, is the memcheck substitute
// (profiles/r02/r02x_bounds_checked.log).  Off in the shipped library.
#ifndef SFB_BOUNDS
#define SFB_BOUNDS 0
#endif
#if SFB_BOUNDS
#include <cassert>
#define SF_BOUNDS(cond) assert(cond)
#else
#define SF_BOUNDS(cond) ((void)0)
#endif

namespace sfb {

// Error carrying one of the SINCFFT_* status codes (see include/sincfft_b200.h).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define SF_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      if (e_ == cudaErrorMemoryAllocation)                                              \
        ::sfb::fail(4, std::string("CUDA out of memory at " #call ": ") +               \
                           cudaGetErrorString(e_));                                     \
      ::sfb::fail(3, std::string("CUDA error at " #call ": ") + cudaGetErrorString(e_)); \
    }                                                                                   \
  } while (0)

#define SF_LAUNCH_CHECK() SF_CUDA(cudaGetLastError())

// ---------------------------------------------------------------- complex fp64
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(a.x * s, a.y * s);
}
// a * (-i)
__host__ __device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Stream-ordered scratch buffer (cudaMallocAsync pool); freed on the stream.
struct Scratch {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  Scratch() = default;
  Scratch(size_t bytes, cudaStream_t st) : s(st) {
    if (bytes) SF_CUDA(cudaMallocAsync(&p, bytes, st));
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Owning device allocation (plan-lifetime tables).
template <class T>
struct DevArray {
  T* p = nullptr;
  int64_t n = 0;
  DevArray() = default;
  explicit DevArray(int64_t count) { alloc(count); }
  void alloc(int64_t count) {
    release();
    n = count;
    if (count > 0) SF_CUDA(cudaMalloc(&p, sizeof(T) * (size_t)count));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevArray() { release(); }
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  DevArray(DevArray&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DevArray& operator=(DevArray&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p, n = o.n;
      o.p = nullptr, o.n = 0;
    }
    return *this;
  }
};

// ---- programmatic dependent launch (PDL): a kernel launched with
// launch_pdl() may be scheduled while the previous kernel in the stream is
// still running its last wave; it runs its independent prologue, then
// pdl_wait() blocks until that kernel has completed and its writes are
// visible.  pdl_trigger() lets the NEXT kernel be scheduled.  Both are no-ops
// for kernels launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
bool pdl_enabled();  // capi.cu: SFB_PDL (default on)
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args... args) {
  if (!pdl_enabled()) {
    kernel<<<grid, block, smem, s>>>(args...);
    SF_LAUNCH_CHECK();
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SF_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
}

// ---- bulk async copy (the TMA engine, non-tensor form) completing on an
// mbarrier: one thread issues the whole contiguous copy; bytes % 16 == 0,
// both addresses 16-byte aligned
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* mbar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mbar))
      : "memory");
}
// TMA prefetch of a contiguous global range into L2 (no destination, no
// completion): bytes % 16 == 0, 16-byte aligned
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}
// one arrival that also expects `bytes` of transaction count, then bulk
// copies that only complete bytes (bulk_g2s_tx): several copies, one phase
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_tx(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mbar))
      : "memory");
}
// bulk copy with an L2 eviction-priority hint (createpolicy: evict_last keeps
// the source resident against streaming traffic, evict_first streams it)
template <bool LAST>
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes,
                                              unsigned long long* mbar) {
  unsigned long long pol;
  if (LAST)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mbar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

// ---- L2 eviction-priority hints on plain loads / stores (createpolicy):
// tables read once per pass stream through (evict_first), intermediates the
// next kernel reads stay (evict_last)
__device__ __forceinline__ unsigned long long l2_policy_first() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_last() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_hint(const double2* p, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
               "l"(pol)
               : "memory");
}

// ---- cp.async (global -> shared without registers); src_bytes < size zero-fills
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(src_bytes));
}
// the random gathers (spread f reads): 64-byte L2 fill instead of the default
// (tools/randread.cu under ncu: 97 -> 59 DRAM bytes per random 16-byte read)
__device__ __forceinline__ void cp_async16z_l2_64(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(src_bytes));
}
// cp.async with an L2 cache-policy operand (createpolicy) and the 64-byte fill
__device__ __forceinline__ void cp_async16z_pol(void* smem, const void* gmem, int src_bytes,
                                                unsigned long long pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint.L2::64B [%0], [%1], 16, %2, %3;\n" ::"r"(sa),
               "l"(gmem), "r"(src_bytes), "l"(pol));
}
__device__ __forceinline__ void cp_async16_pol(void* smem, const void* gmem,
                                               unsigned long long pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa),
               "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void cp_async8z(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4z(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

}  // namespace sfb
