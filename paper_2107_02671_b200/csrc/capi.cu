// capi.cu -- the extern "C" drop-in boundary (include/sincfft_b200.h).
//
// Each entry point replaces one function of the reference's Python API
// (pkg/src/sincfft/nnfft.py, fast_sinc.py); the ctypes shim in
// paper_2107_02671_b200/_lib.py binds them and maps status codes to the
// reference's exception classes (errors.py:4-13).
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>
#include <new>
#include <string>

#include "../../include/sincfft_b200.h"
#include "nfft_impl.cuh"

// Small transforms are launch-bound (configs 1-2: microseconds of GPU work
// behind ~10 runtime calls), so device-pointer executes of small plans are
// captured once per (f, out, batch) into a CUDA graph and replayed.
struct GraphCache {
  struct Entry {
    const void* f;
    void* out;
    int64_t batch;
    cudaGraphExec_t exec;
  };
  struct Key {
    const void* f;
    void* out;
    int64_t batch;
  };
  std::mutex mu;
  std::vector<Entry> entries;  // least recently used first, at most kMax
  std::vector<Key> seen;       // keys executed once without a graph, at most kMax
  static constexpr size_t kMax = 8;
  ~GraphCache() {
    for (auto& e : entries) cudaGraphExecDestroy(e.exec);
  }
};

struct sincfft_nnfft_plan_s {
  sfb::NnfftPlanImpl impl;
  GraphCache graphs;
  std::mutex adj_mu;                       // adjoint sub-plans, built on first use
  std::unique_ptr<sfb::NnfftAdjoint> adj;
};

struct sincfft_sinc_plan_s {
  sfb::NnfftPlanImpl st1, st3;                  // NNFFT stages (non-grid node sets)
  std::unique_ptr<sfb::NfftPlanImpl> nf1, nf3;  // NFFT trafo / adjoint stages (grid sets)
  int64_t N = 0, n_star = 0, L1 = 0, L2 = 0, n = 0;
  int device = 0, mode = 0;
  GraphCache graphs;  // device-pointer executes, keyed on (c, out, c_is_real)
};

struct sincfft_nfft_plan_s {
  sfb::NfftPlanImpl impl;
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    g_last_error.clear();
    f();
    return SINCFFT_OK;
  } catch (const sfb::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return SINCFFT_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SINCFFT_ECUDA;
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

void check_ptr_kind(int32_t k) {
  if (k != SINCFFT_PTR_HOST && k != SINCFFT_PTR_DEVICE && k != SINCFFT_PTR_HOST_ASYNC)
    sfb::fail(1, "ptr_kind must be 0 (host), 1 (device) or 2 (host, asynchronous)");
}

// device copy of caller data (host -> device, or device alias)
struct InBuf {
  std::unique_ptr<sfb::Scratch> tmp;
  const void* ptr = nullptr;
  InBuf(const void* user, size_t bytes, int32_t kind, cudaStream_t s) {
    if (kind == SINCFFT_PTR_DEVICE) {
      ptr = user;
    } else {
      tmp.reset(new sfb::Scratch(bytes, s));
      if (bytes) SF_CUDA(cudaMemcpyAsync(tmp->p, user, bytes, cudaMemcpyHostToDevice, s));
      ptr = tmp->p;
    }
  }
};

struct OutBuf {  // device output, copied back to a host `out` at finish()
  std::unique_ptr<sfb::Scratch> tmp;
  void* user;
  size_t bytes;
  int32_t kind;
  void* ptr;
  OutBuf(void* u, size_t b, int32_t k, cudaStream_t s) : user(u), bytes(b), kind(k) {
    if (kind == SINCFFT_PTR_DEVICE) {
      ptr = user;
    } else {
      tmp.reset(new sfb::Scratch(bytes, s));
      ptr = tmp->p;
    }
  }
  void finish(cudaStream_t s) {
    if (kind == SINCFFT_PTR_DEVICE) return;
    if (bytes) SF_CUDA(cudaMemcpyAsync(user, ptr, bytes, cudaMemcpyDeviceToHost, s));
    if (kind == SINCFFT_PTR_HOST) SF_CUDA(cudaStreamSynchronize(s));
  }
};

void set_device(int dev) {
  int cur = -1;
  SF_CUDA(cudaGetDevice(&cur));
  if (cur != dev) SF_CUDA(cudaSetDevice(dev));
  // keep freed stream-ordered scratch cached in the device pool (the default
  // release threshold 0 would hand it back to the driver at every sync and
  // turn each execute's scratch into fresh cudaMalloc calls)
  static bool configured[64] = {};
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaMemPool_t pool;
    SF_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    SF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    configured[dev] = true;
  }
}

__global__ void k_scale_copy(const double* in, double* out, int64_t n, double s) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = s * in[i];
}

// t = np.mod(q z + 0.5, 1.0) - 0.5 with numpy's float mod (fast_sinc.py:118-120)
__global__ void k_wrap_half(const double* z, double* out, int64_t n, double q) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = q * z[i] + 0.5;
  double r = fmod(a, 1.0);
  if (r != 0.0) {
    if (r < 0.0) r += 1.0;
  } else {
    r = 0.0;
  }
  out[i] = r - 0.5;
}

__global__ void k_real_to_complex(const double* in, double2* out, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_double2(in[i], 0.0);
}

void fill_geometry(const sfb::NnfftPlanImpl& p, sincfft_geometry* g) {
  g->N = p.g.N;
  g->M1 = p.g.M1;
  g->M2 = p.g.M2;
  g->N1 = p.g.N1;
  g->K = p.g.K;
  g->N2 = p.g.N2;
  g->m1 = p.g.m1;
  g->m2 = p.g.m2;
  g->sigma1 = p.g.sigma1;
  g->sigma2 = p.g.sigma2;
  g->a = p.g.a;
  g->beta1 = p.g.beta1;
  g->beta2 = p.g.beta2;
  g->L = p.fft.L;
  g->L1 = p.fft.L1;
  g->L2 = p.fft.L2;
  g->Kout = p.fft.Kout;
  g->s_lo = p.fft.s_lo;
}

// reference-layout step-0 tables (nnfft.py:185-205) from the device plan
template <int M>
__global__ void k_export_spread(const double* v, int64_t n, double N1, int64_t K, sfb::WinCoef C,
                                int64_t* idx, double* val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double pos = N1 * v[i];
  const double c = floor(pos);
  double w[2 * M];
  sfb::window_taps<M>(C, pos - c, w);
  for (int t = 0; t < 2 * M; ++t) {
    int64_t sp = (int64_t)c + (t + 1 - M) + K / 2;
    double vv = w[t];
    if (sp < 0 || sp >= K) {
      vv = 0.0;
      sp = sp < 0 ? 0 : K - 1;
    }
    idx[i * 2 * M + t] = sp;
    val[i * 2 * M + t] = vv;
  }
}

template <int M>
__global__ void k_export_gather(const double* x, int64_t n, double ratio, double N2d, int64_t N2,
                                double Nd, double beta1, int m1, int64_t N1, sfb::WinCoef C,
                                int64_t* idx, double* val, double* hat1) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double pos = N2d * (x[j] * ratio);
  const double c = floor(pos);
  double w[2 * M];
  sfb::window_taps<M>(C, pos - c, w);
  for (int t = 0; t < 2 * M; ++t) {
    int64_t sp = ((int64_t)c + (t + 1 - M)) % N2;
    if (sp < 0) sp += N2;
    idx[j * 2 * M + t] = sp;
    val[j * 2 * M + t] = w[t];
  }
  hat1[j] = sfb::phi_hat_sinh(beta1, m1, N1, Nd * x[j]);
}

template <int M>
void export_spread_m(const sfb::NnfftPlanImpl& p, int64_t* idx, double* val, cudaStream_t s) {
  k_export_spread<M><<<(unsigned)sfb::ceil_div(p.g.M1, 256), 256, 0, s>>>(
      p.v_clip.p, p.g.M1, (double)p.g.N1, p.g.K, p.c1, idx, val);
  SF_LAUNCH_CHECK();
}

template <int M>
void export_gather_m(const sfb::NnfftPlanImpl& p, int64_t* idx, double* val, double* hat1,
                     cudaStream_t s) {
  k_export_gather<M><<<(unsigned)sfb::ceil_div(p.g.M2, 256), 256, 0, s>>>(
      p.x_clip.p, p.g.M2, (double)p.g.N / (double)p.g.N1, (double)p.g.N2, p.g.N2, (double)p.g.N,
      p.g.beta1, p.g.m1, p.g.N1, p.c2, idx, val, hat1);
  SF_LAUNCH_CHECK();
}

#define SF_DISPATCH_M(m, CALL)                                                        \
  switch (m) {                                                                        \
    case 2: CALL(2); break;                                                           \
    case 3: CALL(3); break;                                                           \
    case 4: CALL(4); break;                                                           \
    case 5: CALL(5); break;                                                           \
    case 6: CALL(6); break;                                                           \
    case 7: CALL(7); break;                                                           \
    case 8: CALL(8); break;                                                           \
    case 9: CALL(9); break;                                                           \
    case 10: CALL(10); break;                                                         \
    case 11: CALL(11); break;                                                         \
    case 12: CALL(12); break;                                                         \
    case 13: CALL(13); break;                                                         \
    case 14: CALL(14); break;                                                         \
    case 15: CALL(15); break;                                                         \
    case 16: CALL(16); break;                                                         \
    default: sfb::fail(5, "unsupported window cut-off");                              \
  }

void build_nnfft(sfb::NnfftPlanImpl& p, int64_t N, int64_t M1, int64_t M2, double sigma1,
                 double sigma2, int m1, int m2, const double* v_dev, const double* x_dev,
                 int device, cudaStream_t s) {
  p.g = sfb::make_geometry(N, M1, M2, sigma1, sigma2, m1, m2);
  p.device = device;
  sfb::build_plan(p, v_dev, x_dev, s);
}

}  // namespace

namespace sfb {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SFB_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}
}  // namespace sfb

namespace {

bool use_graph(const sfb::NnfftPlanImpl& p, int64_t batch) {
  static const bool off = getenv("SINCFFT_NO_GRAPHS") != nullptr;
  static const int64_t lim = [] {
    const char* e = getenv("SINCFFT_GRAPH_MAX_NODES");
    return e ? (int64_t)atoll(e) : ((int64_t)1 << 19);
  }();
  // single columns of any size: replaying the captured spread/FFT/gather
  // sequence saves the inter-launch gaps (config 3: 0.851 -> 0.840 ms); large
  // batches stay uncaptured (their scratch would be pinned per cached graph)
  return !off && (batch == 1 || (p.g.M1 + p.g.M2) * batch <= lim);
}

// Replays the spread/FFT/gather sequence of (f, out, batch) as a CUDA graph.
// A key is captured on its SECOND execute (a caller that allocates a fresh
// output every call never pays capture + instantiate); hits move to the back
// (LRU); a new key reuses the least recently used exec through
// cudaGraphExecUpdate (same topology, new pointers) instead of instantiating.
// Returns false when the caller should launch directly (first sighting).
template <class Capture>
bool launch_graph(GraphCache& gc, const void* f, void* out, int64_t batch, cudaStream_t s,
                  Capture&& capture) {
  std::lock_guard<std::mutex> lk(gc.mu);
  cudaGraphExec_t exec = nullptr;
  for (size_t i = 0; i < gc.entries.size(); ++i) {
    const GraphCache::Entry e = gc.entries[i];
    if (e.f == f && e.out == out && e.batch == batch) {
      gc.entries.erase(gc.entries.begin() + i);
      gc.entries.push_back(e);
      exec = e.exec;
      break;
    }
  }
  if (!exec) {
    bool seen = false;
    for (size_t i = 0; i < gc.seen.size(); ++i) {
      if (gc.seen[i].f == f && gc.seen[i].out == out && gc.seen[i].batch == batch) {
        gc.seen.erase(gc.seen.begin() + i);
        seen = true;
        break;
      }
    }
    if (!seen) {
      if (gc.seen.size() == GraphCache::kMax) gc.seen.erase(gc.seen.begin());
      gc.seen.push_back({f, out, batch});
      return false;
    }
    cudaStream_t cs;
    SF_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    try {
      SF_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      capture(cs);
      SF_CUDA(cudaStreamEndCapture(cs, &graph));
      if (gc.entries.size() == GraphCache::kMax) {
        cudaGraphExec_t lru = gc.entries.front().exec;
        gc.entries.erase(gc.entries.begin());
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(lru, graph, &info) == cudaSuccess) {
          exec = lru;
        } else {
          cudaGetLastError();  // clear the update failure
          cudaGraphExecDestroy(lru);
        }
      }
      if (!exec) SF_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    } catch (...) {
      cudaStreamEndCapture(cs, &graph);
      if (graph) cudaGraphDestroy(graph);
      cudaStreamDestroy(cs);
      throw;
    }
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    gc.entries.push_back({f, out, batch, exec});
  }
  // launched under the lock: another thread's eviction may update or destroy exec
  SF_CUDA(cudaGraphLaunch(exec, s));
  return true;
}

}  // namespace

namespace sfb {

void run_execute(const NnfftPlanImpl& p, const double2* f, double2* out, int batch,
                 cudaStream_t s) {
  if (batch >= kBatchedMin) return run_execute_batched(p, f, out, batch, s);
  // a single column's grid is padded to whole FFT rows (TMA column pass)
  const bool pad = batch == 1 && p.fft.L1 > 0 && !p.fft.direct && !p.fft.single;
  const int64_t kg = pad ? ceil_div(p.g.K, p.fft.L1) * p.fft.L1 : p.g.K;
  Scratch grid(sizeof(double2) * (size_t)kg * batch, s);
  Scratch work(sizeof(double2) * (size_t)p.fft.work_elems() * batch, s);
  Scratch h(sizeof(double2) * (size_t)p.fft.Kout * batch, s);
  run_spread(p, f, grid.as<double2>(), batch, s);
  run_fft(p, grid.as<double2>(), h.as<double2>(), work.as<double2>(), batch, s, pad);
  run_gather(p, h.as<double2>(), out, batch, s);
}

}  // namespace sfb

extern "C" {

const char* sincfft_last_error(void) { return g_last_error.c_str(); }

int sincfft_version(void) { return 100; }

int sincfft_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int sincfft_nnfft_plan_create(sincfft_nnfft_plan* plan, int64_t N, int64_t M1, int64_t M2,
                              double sigma1, double sigma2, int32_t m1, int32_t m2,
                              const double* v, const double* x, int32_t ptr_kind, int32_t device,
                              void* stream) {
  return sincfft_nnfft_plan_create_ex(plan, N, M1, M2, sigma1, sigma2, m1, m2, v, x, ptr_kind,
                                      device, 0, stream);
}

int sincfft_nnfft_plan_create_ex(sincfft_nnfft_plan* plan, int64_t N, int64_t M1, int64_t M2,
                                 double sigma1, double sigma2, int32_t m1, int32_t m2,
                                 const double* v, const double* x, int32_t ptr_kind,
                                 int32_t device, int32_t flags, void* stream) {
  return guarded([&] {
    if (flags & ~SINCFFT_PLAN_FULL_WINDOW) sfb::fail(1, "nnfft_plan: unknown flags");
    if (!plan) sfb::fail(1, "plan pointer is NULL");
    *plan = nullptr;
    check_ptr_kind(ptr_kind);
    if (!v || !x) sfb::fail(1, "nnfft_plan: v and x must be non-NULL");
    // geometry first: its errors must not depend on the data or the device
    (void)sfb::make_geometry(N, M1, M2, sigma1, sigma2, m1, m2);
    set_device(device);
    cudaStream_t s = as_stream(stream);
    auto* h = new sincfft_nnfft_plan_s();
    try {
      InBuf vb(v, sizeof(double) * M1, ptr_kind, s), xb(x, sizeof(double) * M2, ptr_kind, s);
      h->impl.full_window = (flags & SINCFFT_PLAN_FULL_WINDOW) != 0;
      build_nnfft(h->impl, N, M1, M2, sigma1, sigma2, m1, m2, (const double*)vb.ptr,
                  (const double*)xb.ptr, device, s);
      SF_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      delete h;
      throw;
    }
    *plan = h;
  });
}

int sincfft_nnfft_plan_destroy(sincfft_nnfft_plan plan) {
  return guarded([&] {
    if (!plan) return;
    set_device(plan->impl.device);
    delete plan;
  });
}

int sincfft_nnfft_plan_geometry(sincfft_nnfft_plan plan, sincfft_geometry* geo) {
  return guarded([&] {
    if (!plan || !geo) sfb::fail(1, "NULL argument");
    fill_geometry(plan->impl, geo);
  });
}

int sincfft_nnfft_execute(sincfft_nnfft_plan plan, const double* f, double* out, int64_t batch,
                          int32_t ptr_kind, void* stream) {
  return guarded([&] {
    if (!plan || !f || !out) sfb::fail(1, "NULL argument");
    check_ptr_kind(ptr_kind);
    if (batch < 1 || batch > 65535) sfb::fail(1, "batch must be in [1, 65535]");
    const sfb::NnfftPlanImpl& p = plan->impl;
    set_device(p.device);
    cudaStream_t s = as_stream(stream);
    const size_t fb = sizeof(double2) * (size_t)p.g.M1 * batch;
    const size_t ob = sizeof(double2) * (size_t)p.g.M2 * batch;
    InBuf fin(f, fb, ptr_kind, s);
    if (ptr_kind == SINCFFT_PTR_DEVICE && use_graph(p, batch) &&
        launch_graph(plan->graphs, f, out, batch, s, [&](cudaStream_t cs) {
          sfb::run_execute(plan->impl, (const double2*)f, (double2*)out, (int)batch, cs);
        })) {
    } else if (ptr_kind == SINCFFT_PTR_DEVICE) {
      sfb::run_execute(p, (const double2*)fin.ptr, (double2*)out, (int)batch, s);
    } else {
      sfb::Scratch o(ob, s);
      sfb::run_execute(p, (const double2*)fin.ptr, o.as<double2>(), (int)batch, s);
      SF_CUDA(cudaMemcpyAsync(out, o.p, ob, cudaMemcpyDeviceToHost, s));
      if (ptr_kind == SINCFFT_PTR_HOST) SF_CUDA(cudaStreamSynchronize(s));
    }
  });
}

int sincfft_nnfft_spread(sincfft_nnfft_plan plan, const double* f, double* grid_dev,
                         int64_t batch, int32_t ptr_kind, void* stream) {
  return guarded([&] {
    if (!plan || !f || !grid_dev) sfb::fail(1, "NULL argument");
    check_ptr_kind(ptr_kind);
    if (batch < 1 || batch > 65535) sfb::fail(1, "batch must be in [1, 65535]");
    const sfb::NnfftPlanImpl& p = plan->impl;
    set_device(p.device);
    cudaStream_t s = as_stream(stream);
    InBuf fin(f, sizeof(double2) * (size_t)p.g.M1 * batch, ptr_kind, s);
    sfb::run_spread(p, (const double2*)fin.ptr, (double2*)grid_dev, (int)batch, s);
    if (ptr_kind == SINCFFT_PTR_HOST) SF_CUDA(cudaStreamSynchronize(s));
  });
}

int sincfft_nnfft_finish(sincfft_nnfft_plan plan, const double* grid_dev, double* out,
                         int64_t batch, int32_t ptr_kind, void* stream) {
  return guarded([&] {
    if (!plan || !grid_dev || !out) sfb::fail(1, "NULL argument");
    check_ptr_kind(ptr_kind);
    if (batch < 1 || batch > 65535) sfb::fail(1, "batch must be in [1, 65535]");
    const sfb::NnfftPlanImpl& p = plan->impl;
    set_device(p.device);
    cudaStream_t s = as_stream(stream);
    sfb::Scratch work(sizeof(double2) * (size_t)p.fft.work_elems() * batch, s);
    sfb::Scratch h(sizeof(double2) * (size_t)p.fft.Kout * batch, s);
    sfb::run_fft(p, (const double2*)grid_dev, h.as<double2>(), work.as<double2>(), (int)batch, s);
    const size_t ob = sizeof(double2) * (size_t)p.g.M2 * batch;
    if (ptr_kind == SINCFFT_PTR_DEVICE) {
      sfb::run_gather(p, h.as<double2>(), (double2*)out, (int)batch, s);
    } else {
      sfb::Scratch o(ob, s);
      sfb::run_gather(p, h.as<double2>(), o.as<double2>(), (int)batch, s);
      SF_CUDA(cudaMemcpyAsync(out, o.p, ob, cudaMemcpyDeviceToHost, s));
      if (ptr_kind == SINCFFT_PTR_HOST) SF_CUDA(cudaStreamSynchronize(s));
    }
  });
}

int sincfft_nnfft_dist_layout(sincfft_nnfft_plan plan, int32_t world, int64_t* sizes) {
  return guarded([&] {
    if (!plan || !sizes) sfb::fail(1, "NULL argument");
    sfb::DistLayout l;
    const bool ok = sfb::dist_layout(plan->impl, world, &l);
    sizes[0] = ok ? 1 : 0;
    sizes[1] = ok ? l.Sb : 0;                    // reduce-scatter block (per rank)
    sizes[2] = ok ? plan->impl.fft.L2 * l.Bc : 0;  // column-pass output = all-to-all buffer
    sizes[3] = ok ? l.K2 * l.Bc : 0;              // h block (per rank, all-gather)
    sizes[4] = ok ? l.Bc : 0;
    sizes[5] = ok ? l.Br : 0;
  });
}

#define SF_DIST_PROLOGUE(...)                                      \
  if (!plan || __VA_ARGS__) sfb::fail(1, "NULL argument");        \
  const sfb::NnfftPlanImpl& p = plan->impl;                       \
  set_device(p.device);                                           \
  cudaStream_t s = as_stream(stream)

int sincfft_nnfft_dist_pack(sincfft_nnfft_plan plan, int32_t world, const double* grid_dev,
                            double* send_dev, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!grid_dev || !send_dev);
    sfb::run_dist_pack(p, world, (const double2*)grid_dev, (double2*)send_dev, s);
  });
}

int sincfft_nnfft_dist_colfwd(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                              const double* block_dev, double* cols_dev, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!block_dev || !cols_dev);
    sfb::run_dist_colfwd(p, world, rank, (const double2*)block_dev, (double2*)cols_dev, s);
  });
}

int sincfft_nnfft_dist_rowmul(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                              double* rows_dev, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!rows_dev);
    sfb::run_dist_rowmul(p, world, rank, (double2*)rows_dev, s);
  });
}

int sincfft_nnfft_dist_colinv(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                              const double* cols_dev, const double* block_dev, double* hblk_dev,
                              void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!cols_dev || !block_dev || !hblk_dev);
    sfb::run_dist_colinv(p, world, rank, (const double2*)cols_dev, (const double2*)block_dev,
                         (double2*)hblk_dev, s);
  });
}

int sincfft_nnfft_dist_gather(sincfft_nnfft_plan plan, int32_t world, const double* hall_dev,
                              double* out_dev, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!hall_dev || !out_dev);
    sfb::Scratch h(sizeof(double2) * (size_t)p.fft.Kout, s);
    sfb::run_dist_unpack(p, world, (const double2*)hall_dev, h.as<double2>(), s);
    sfb::run_gather(p, h.as<double2>(), (double2*)out_dev, 1, s);
  });
}

// ---- peer-memory buffers (CUDA IPC; NVLink P2P between the GPUs of a node)
int sincfft_ipc_alloc(int32_t device, int64_t bytes, void** ptr) {
  return guarded([&] {
    if (!ptr || bytes <= 0) sfb::fail(1, "ipc_alloc: bad arguments");
    set_device(device);
    SF_CUDA(cudaMalloc(ptr, (size_t)bytes));  // its own allocation: the handle covers it exactly
  });
}

int sincfft_ipc_free(void* ptr) {
  return guarded([&] { SF_CUDA(cudaFree(ptr)); });
}

int sincfft_ipc_handle(void* ptr, uint8_t* handle64) {
  return guarded([&] {
    if (!ptr || !handle64) sfb::fail(1, "NULL argument");
    cudaIpcMemHandle_t h;
    SF_CUDA(cudaIpcGetMemHandle(&h, ptr));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(handle64, &h, sizeof(h));
  });
}

int sincfft_ipc_open(int32_t device, const uint8_t* handle64, void** ptr) {
  return guarded([&] {
    if (!handle64 || !ptr) sfb::fail(1, "NULL argument");
    set_device(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    SF_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int sincfft_ipc_close(void* ptr) {
  return guarded([&] { SF_CUDA(cudaIpcCloseMemHandle(ptr)); });
}

int sincfft_nnfft_dist_colfwd_peer(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                                   const double* block_dev, const uint64_t* peers,
                                   void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!block_dev || !peers);
    double2* pp[sfb::kDistMaxRanks] = {};
    for (int q = 0; q < world && q < sfb::kDistMaxRanks; ++q) pp[q] = (double2*)peers[q];
    sfb::run_dist_colfwd_peer(p, world, rank, (const double2*)block_dev, pp, s);
  });
}

int sincfft_nnfft_dist_rowmul_peer(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                                   double* rows_dev, const uint64_t* peers, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!rows_dev || !peers);
    double2* pp[sfb::kDistMaxRanks] = {};
    for (int q = 0; q < world && q < sfb::kDistMaxRanks; ++q) pp[q] = (double2*)peers[q];
    sfb::run_dist_rowmul_peer(p, world, rank, (double2*)rows_dev, pp, s);
  });
}

int sincfft_nnfft_dist_pack_rows_peer(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                                      const double* grid_dev, int64_t ilo, int64_t nrow,
                                      const uint64_t* peers, const int64_t* poff, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!grid_dev || !peers || !poff);
    double2* pp[sfb::kDistMaxRanks] = {};
    for (int q = 0; q < world && q < sfb::kDistMaxRanks; ++q) pp[q] = (double2*)peers[q];
    sfb::run_dist_pack_rows_peer(p, world, rank, (const double2*)grid_dev, ilo, nrow, pp, poff, s);
  });
}

int sincfft_nnfft_dist_colinv_peer(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                                   const double* cols_dev, const double* block_dev,
                                   const uint64_t* peers, const int64_t* k2lo,
                                   const int64_t* cnt, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!cols_dev || !block_dev || !peers || !k2lo || !cnt);
    double2* pp[sfb::kDistMaxRanks] = {};
    for (int q = 0; q < world && q < sfb::kDistMaxRanks; ++q) pp[q] = (double2*)peers[q];
    sfb::run_dist_colinv_peer(p, world, rank, (const double2*)cols_dev,
                              (const double2*)block_dev, pp, k2lo, cnt, s);
  });
}

int sincfft_nnfft_dist_support(sincfft_nnfft_plan plan, int64_t* out4, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!out4);
    sfb::dist_support(p, s, out4);
  });
}

int sincfft_nnfft_dist_pack_rows(sincfft_nnfft_plan plan, int32_t world, const double* grid_dev,
                                 int64_t ilo, int64_t nrow, double* send_dev, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!grid_dev || !send_dev);
    sfb::run_dist_pack_rows(p, world, (const double2*)grid_dev, ilo, nrow, (double2*)send_dev, s);
  });
}

int sincfft_nnfft_dist_unpack_rows(sincfft_nnfft_plan plan, int32_t world, int32_t rank,
                                   const double* recv_dev, const int64_t* ilo,
                                   const int64_t* nrow, double* block_dev, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!recv_dev || !ilo || !nrow || !block_dev);
    sfb::run_dist_unpack_rows(p, world, rank, (const double2*)recv_dev, ilo, nrow,
                              (double2*)block_dev, s);
  });
}

int sincfft_nnfft_dist_pack_hrows(sincfft_nnfft_plan plan, int32_t world, const double* hblk_dev,
                                  const int64_t* k2lo, const int64_t* cnt, double* send_dev,
                                  void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!hblk_dev || !k2lo || !cnt || !send_dev);
    sfb::run_dist_pack_hrows(p, world, (const double2*)hblk_dev, k2lo, cnt, (double2*)send_dev,
                             s);
  });
}

int sincfft_nnfft_dist_gather_rows(sincfft_nnfft_plan plan, int32_t world, const double* recv_dev,
                                   int64_t k2lo, int64_t cnt, double* out_dev, void* stream) {
  return guarded([&] {
    SF_DIST_PROLOGUE(!recv_dev || !out_dev);
    sfb::Scratch h(sizeof(double2) * (size_t)p.fft.Kout, s);
    sfb::run_dist_unpack_hrows(p, world, (const double2*)recv_dev, k2lo, cnt, h.as<double2>(), s);
    sfb::run_gather(p, h.as<double2>(), (double2*)out_dev, 1, s);
  });
}

int sincfft_nnfft_execute_profiled(sincfft_nnfft_plan plan, const double* f, double* out,
                                   int64_t batch, void* stream, double* stage_ms) {
  return guarded([&] {
    if (!plan || !f || !out || !stage_ms) sfb::fail(1, "NULL argument");
    if (batch < 1 || batch > 65535) sfb::fail(1, "batch must be in [1, 65535]");
    const sfb::NnfftPlanImpl& p = plan->impl;
    set_device(p.device);
    cudaStream_t s = as_stream(stream);
    const bool batched = batch >= sfb::kBatchedMin;
    sfb::Scratch grid(batched ? 0 : sizeof(double2) * (size_t)p.g.K * batch, s);
    sfb::Scratch work(batched ? 0 : sizeof(double2) * (size_t)p.fft.work_elems() * batch, s);
    sfb::Scratch h(batched ? 0 : sizeof(double2) * (size_t)p.fft.Kout * batch, s);
    cudaEvent_t ev[4], evz = nullptr;
    for (auto& e : ev) SF_CUDA(cudaEventCreate(&e));
    if (!batched) SF_CUDA(cudaEventCreate(&evz));
    if (batch >= sfb::kBatchedMin) {
      sfb::run_execute_batched(p, (const double2*)f, (double2*)out, (int)batch, s, ev);
    } else {
      // the grid memset (a ~7 us copy-engine fill at config 3) runs before the
      // first event: stage 0 is the spread KERNEL's duration
      SF_CUDA(cudaEventRecord(evz, s));
      sfb::run_spread_zero(p, grid.as<double2>(), (int)batch, s);
      SF_CUDA(cudaEventRecord(ev[0], s));
      sfb::run_spread_kernel(p, (const double2*)f, grid.as<double2>(), (int)batch, s);
      SF_CUDA(cudaEventRecord(ev[1], s));
      sfb::run_fft(p, grid.as<double2>(), h.as<double2>(), work.as<double2>(), (int)batch, s);
      SF_CUDA(cudaEventRecord(ev[2], s));
      sfb::run_gather(p, h.as<double2>(), (double2*)out, (int)batch, s);
      SF_CUDA(cudaEventRecord(ev[3], s));
    }
    SF_CUDA(cudaEventSynchronize(ev[3]));
    float t;
    for (int i = 0; i < 3; ++i) {
      SF_CUDA(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
      stage_ms[i] = t;
    }
    SF_CUDA(cudaEventElapsedTime(&t, evz ? evz : ev[0], ev[3]));
    stage_ms[3] = t;
    for (auto& e : ev) cudaEventDestroy(e);
    if (evz) cudaEventDestroy(evz);
  });
}

int sincfft_nnfft_launches_per_execute(sincfft_nnfft_plan plan, int64_t batch) {
  if (!plan) return -1;
  const int fft = plan->impl.fft.single ? 1 : plan->impl.fft.direct ? 2
                                            : 3 + (plan->impl.fft.fixD > 0 ? 1 : 0);
  // column-vectorised batch: halo zeroing + spread + [2 transposes] + FFT + gather
  if (batch >= sfb::kBatchedMin) {
    if (!sfb::fft_supports_point_major(plan->impl)) return 1 + 1 + 2 + fft + 1;
    const int64_t G = sfb::fft_point_major_group((int)batch);
    return 1 + 1 + 3 * ((batch + G - 1) / G) + (plan->impl.fft.fixD > 0 ? 1 : 0) + 1;
  }
  // grid memset (a launch on the stream) + spread + FFT + gather
  return 1 + 1 + fft + 1;
}

int sincfft_nnfft_export_tables(sincfft_nnfft_plan plan, int64_t* spread_idx, double* spread_val,
                                int64_t* gather_idx, double* gather_val, double* hat1,
                                double* hat2) {
  return guarded([&] {
    if (!plan) sfb::fail(1, "NULL plan");
    const sfb::NnfftPlanImpl& p = plan->impl;
    set_device(p.device);
    cudaStream_t s = nullptr;
    const int64_t n1 = p.g.M1 * 2 * p.g.m1, n2 = p.g.M2 * 2 * p.g.m2;
    {
      sfb::Scratch di(sizeof(int64_t) * n1, s), dv(sizeof(double) * n1, s);
#define SF_EXP_S(MM) export_spread_m<MM>(p, di.as<int64_t>(), dv.as<double>(), s)
      SF_DISPATCH_M(p.g.m1, SF_EXP_S);
#undef SF_EXP_S
      if (spread_idx)
        SF_CUDA(cudaMemcpyAsync(spread_idx, di.p, sizeof(int64_t) * n1, cudaMemcpyDeviceToHost, s));
      if (spread_val)
        SF_CUDA(cudaMemcpyAsync(spread_val, dv.p, sizeof(double) * n1, cudaMemcpyDeviceToHost, s));
      SF_CUDA(cudaStreamSynchronize(s));
    }
    {
      sfb::Scratch di(sizeof(int64_t) * n2, s), dv(sizeof(double) * n2, s),
          dh(sizeof(double) * p.g.M2, s);
#define SF_EXP_G(MM) export_gather_m<MM>(p, di.as<int64_t>(), dv.as<double>(), dh.as<double>(), s)
      SF_DISPATCH_M(p.g.m2, SF_EXP_G);
#undef SF_EXP_G
      if (gather_idx)
        SF_CUDA(cudaMemcpyAsync(gather_idx, di.p, sizeof(int64_t) * n2, cudaMemcpyDeviceToHost, s));
      if (gather_val)
        SF_CUDA(cudaMemcpyAsync(gather_val, dv.p, sizeof(double) * n2, cudaMemcpyDeviceToHost, s));
      if (hat1)
        SF_CUDA(cudaMemcpyAsync(hat1, dh.p, sizeof(double) * p.g.M2, cudaMemcpyDeviceToHost, s));
      SF_CUDA(cudaStreamSynchronize(s));
    }
    if (hat2)
      SF_CUDA(cudaMemcpy(hat2, p.hat2.p, sizeof(double) * p.g.K, cudaMemcpyDeviceToHost));
  });
}

// ------------------------------------------------------------- adjoint NNFFT
int sincfft_nnfft_adjoint(sincfft_nnfft_plan plan, const double* y, double* out, int64_t batch,
                          int32_t ptr_kind, void* stream) {
  return guarded([&] {
    if (!plan || !y || !out) sfb::fail(1, "NULL argument");
    if (batch < 1) sfb::fail(1, "batch must be >= 1");
    check_ptr_kind(ptr_kind);
    const sfb::NnfftPlanImpl& p = plan->impl;
    set_device(p.device);
    cudaStream_t s = as_stream(stream);
    {
      std::lock_guard<std::mutex> lk(plan->adj_mu);
      if (!plan->adj) {
        std::unique_ptr<sfb::NnfftAdjoint> a(new sfb::NnfftAdjoint());
        cudaStream_t bs;
        SF_CUDA(cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking));
        try {
          sfb::build_adjoint(p, *a, bs);
        } catch (...) {
          cudaStreamDestroy(bs);
          throw;
        }
        SF_CUDA(cudaStreamDestroy(bs));
        plan->adj = std::move(a);
      }
    }
    InBuf yb(y, sizeof(double2) * (size_t)p.g.M2 * batch, ptr_kind, s);
    OutBuf ob(out, sizeof(double2) * (size_t)p.g.M1 * batch, ptr_kind, s);
    sfb::run_adjoint(p, *plan->adj, (const double2*)yb.ptr, (double2*)ob.ptr, (int)batch, s);
    ob.finish(s);
  });
}

// ------------------------------------------------------------- fast sinc
int sincfft_sinc_plan_create(sincfft_sinc_plan* plan, int64_t N, int64_t n_star, int64_t L1,
                             int64_t L2, int64_t n, const double* z, const double* w,
                             const double* a, const double* b, double sigma1, double sigma2,
                             int32_t m1, int32_t m2, int32_t mode, int32_t ptr_kind,
                             int32_t device, void* stream) {
  return guarded([&] {
    if (!plan) sfb::fail(1, "plan pointer is NULL");
    *plan = nullptr;
    check_ptr_kind(ptr_kind);
    if (!z || !w || !a || !b) sfb::fail(1, "sinc_plan: NULL node/weight array");
    if (N <= 0 || n_star < N || n < 2 || L1 <= 0 || L2 <= 0)
      sfb::fail(1, "sinc_plan: invalid sizes");
    if (mode < SINCFFT_SINC_GENERAL || mode > SINCFFT_SINC_EQUISPACED_BOTH)
      sfb::fail(1, "sinc_plan: unknown mode");
    const bool nfft1 = mode == SINCFFT_SINC_EQUISPACED_SOURCES || mode == SINCFFT_SINC_EQUISPACED_BOTH;
    const bool nfft3 = mode == SINCFFT_SINC_EQUISPACED_TARGETS || mode == SINCFFT_SINC_EQUISPACED_BOTH;
    if (nfft3 && L2 != N) sfb::fail(1, "sinc_plan: equispaced-targets mode requires L2 = N");
    set_device(device);
    cudaStream_t s = as_stream(stream);
    auto* h = new sincfft_sinc_plan_s();
    try {
      h->N = N, h->n_star = n_star, h->L1 = L1, h->L2 = L2, h->n = n, h->device = device;
      h->mode = mode;
      const int64_t nz = n + 1;
      InBuf zb(z, sizeof(double) * nz, ptr_kind, s), wb(w, sizeof(double) * nz, ptr_kind, s),
          ab(a, sizeof(double) * L1, ptr_kind, s), bb(b, sizeof(double) * L2, ptr_kind, s);
      const double scale = (double)N / (double)n_star;  // fast_sinc.py:198
      sfb::Scratch v1(sizeof(double) * L1, s), x1(sizeof(double) * nz, s),
          v3(sizeof(double) * nz, s);
      const unsigned g1 = (unsigned)sfb::ceil_div(L1, 256), gz = (unsigned)sfb::ceil_div(nz, 256);
      k_scale_copy<<<g1, 256, 0, s>>>((const double*)ab.ptr, v1.as<double>(), L1, scale);
      k_scale_copy<<<gz, 256, 0, s>>>((const double*)zb.ptr, x1.as<double>(), nz, 0.5);
      k_scale_copy<<<gz, 256, 0, s>>>((const double*)zb.ptr, v3.as<double>(), nz, -0.5 * scale);
      SF_LAUNCH_CHECK();
      if (nfft1) {
        // plan1 = nfft_plan(L1, wrap(-(N/(2 L1)) z), sigma1, m1)  (fast_sinc.py:200-203)
        sfb::Scratch t1(sizeof(double) * nz, s);
        k_wrap_half<<<gz, 256, 0, s>>>((const double*)zb.ptr, t1.as<double>(), nz,
                                       -((double)N / (2.0 * (double)L1)));
        SF_LAUNCH_CHECK();
        h->nf1.reset(new sfb::NfftPlanImpl());
        sfb::build_nfft(*h->nf1, L1, nz, sigma1, m1, t1.as<double>(), device, s);
        // alpha = w * g fused into the NFFT gather's scale (fast_sinc.py:246)
        sfb::fuse_target_weights(h->nf1->tr, (const double*)wb.ptr, s);
      } else {
        // plan1 = nnfft_plan(n_star, a*scale, z/2)      (fast_sinc.py:205-209)
        build_nnfft(h->st1, n_star, L1, nz, sigma1, sigma2, m1, m2, v1.as<double>(),
                    x1.as<double>(), device, s);
        // alpha = w * g fused into stage-1's gather scale (fast_sinc.py:246)
        sfb::fuse_target_weights(h->st1, (const double*)wb.ptr, s);
      }
      if (nfft3) {
        // plan3 = nfft_plan(N, -z/2, sigma1, m1), applied as the adjoint (fast_sinc.py:211-214)
        sfb::Scratch t3(sizeof(double) * nz, s);
        k_scale_copy<<<gz, 256, 0, s>>>((const double*)zb.ptr, t3.as<double>(), nz, -0.5);
        SF_LAUNCH_CHECK();
        h->nf3.reset(new sfb::NfftPlanImpl());
        sfb::build_nfft(*h->nf3, N, nz, sigma1, m1, t3.as<double>(), device, s);
      } else {
        // plan3 = nnfft_plan(n_star, -(scale/2) z, b)   (fast_sinc.py:216-220)
        build_nnfft(h->st3, n_star, nz, L2, sigma1, sigma2, m1, m2, v3.as<double>(),
                    (const double*)bb.ptr, device, s);
      }
      SF_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      delete h;
      throw;
    }
    *plan = h;
  });
}

int sincfft_sinc_plan_destroy(sincfft_sinc_plan plan) {
  return guarded([&] {
    if (!plan) return;
    set_device(plan->device);
    delete plan;
  });
}

int sincfft_sinc_plan_geometry(sincfft_sinc_plan plan, sincfft_geometry* stage1,
                               sincfft_geometry* stage3) {
  return guarded([&] {
    if (!plan) sfb::fail(1, "NULL plan");
    if (stage1) fill_geometry(plan->nf1 ? plan->nf1->tr : plan->st1, stage1);
    if (stage3) fill_geometry(plan->nf3 ? plan->nf3->ad_fft : plan->st3, stage3);
  });
}

// stage 1 (NNFFT or NFFT trafo of c at the Chebyshev nodes, times the
// Clenshaw-Curtis weights folded into its gather scale) and stage 3 (from the
// weighted alpha to the targets) of the fast sinc transform
static void sinc_stage1(sincfft_sinc_plan plan, const void* cdev, int c_is_real, double2* alpha,
                        cudaStream_t s) {
  if (plan->nf1) {
    // stage 1 = NFFT trafo of c (complex; real input promoted like the reference)
    const double2* cc = (const double2*)cdev;
    sfb::Scratch cz(c_is_real ? sizeof(double2) * (size_t)plan->L1 : 1, s);
    if (c_is_real) {
      k_real_to_complex<<<(unsigned)sfb::ceil_div(plan->L1, 256), 256, 0, s>>>(
          (const double*)cdev, cz.as<double2>(), plan->L1);
      SF_LAUNCH_CHECK();
      cc = cz.as<double2>();
    }
    sfb::run_nfft_trafo(*plan->nf1, cc, alpha, s);
  } else {
    const sfb::NnfftPlanImpl& p1 = plan->st1;
    sfb::Scratch g1(sizeof(double2) * (size_t)p1.g.K, s);
    sfb::Scratch w1(sizeof(double2) * (size_t)p1.fft.work_elems(), s);
    sfb::Scratch h1(sizeof(double2) * (size_t)p1.fft.Kout, s);
    if (c_is_real) sfb::run_spread_real(p1, (const double*)cdev, g1.as<double2>(), s);
    else sfb::run_spread(p1, (const double2*)cdev, g1.as<double2>(), 1, s);
    sfb::run_fft(p1, g1.as<double2>(), h1.as<double2>(), w1.as<double2>(), 1, s);
    sfb::run_gather(p1, h1.as<double2>(), alpha, 1, s);
  }
}

static void sinc_stage3(sincfft_sinc_plan plan, const double2* alpha, double* out,
                        int32_t ptr_kind, cudaStream_t s) {
  const size_t ob = sizeof(double2) * (size_t)plan->L2;
  auto stage3 = [&](double2* dst) {
    if (plan->nf3) sfb::run_nfft_adjoint(*plan->nf3, alpha, dst, s);
    else sfb::run_execute(plan->st3, alpha, dst, 1, s);
  };
  if (ptr_kind == SINCFFT_PTR_DEVICE) {
    stage3((double2*)out);
  } else {
    sfb::Scratch o(ob, s);
    stage3(o.as<double2>());
    SF_CUDA(cudaMemcpyAsync(out, o.p, ob, cudaMemcpyDeviceToHost, s));
    if (ptr_kind == SINCFFT_PTR_HOST) SF_CUDA(cudaStreamSynchronize(s));
  }
}

int sincfft_sinc_execute(sincfft_sinc_plan plan, const double* c, int32_t c_is_real, double* out,
                         int32_t ptr_kind, void* stream) {
  return guarded([&] {
    if (!plan || !c || !out) sfb::fail(1, "NULL argument");
    check_ptr_kind(ptr_kind);
    set_device(plan->device);
    cudaStream_t s = as_stream(stream);
    const size_t cb = (c_is_real ? sizeof(double) : sizeof(double2)) * (size_t)plan->L1;
    // device pointers: the ~13 launches of the two stages replayed as one CUDA
    // graph (captured on the second execute with the same buffers)
    static const bool no_graphs = getenv("SINCFFT_NO_GRAPHS") != nullptr;
    if (ptr_kind == SINCFFT_PTR_DEVICE && !no_graphs &&
        launch_graph(plan->graphs, c, out, c_is_real ? 1 : 0, s, [&](cudaStream_t cs) {
          sfb::Scratch a2(sizeof(double2) * (size_t)(plan->n + 1), cs);
          sinc_stage1(plan, c, c_is_real, a2.as<double2>(), cs);
          sinc_stage3(plan, a2.as<double2>(), out, SINCFFT_PTR_DEVICE, cs);
        }))
      return;
    InBuf cin(c, cb, ptr_kind, s);
    sfb::Scratch alpha(sizeof(double2) * (size_t)(plan->n + 1), s);
    sinc_stage1(plan, cin.ptr, c_is_real, alpha.as<double2>(), s);
    sinc_stage3(plan, alpha.as<double2>(), out, ptr_kind, s);
  });
}

int sincfft_sinc_stage1(sincfft_sinc_plan plan, const double* c, int32_t c_is_real,
                        double* alpha_dev, void* stream) {
  return guarded([&] {
    if (!plan || !c || !alpha_dev) sfb::fail(1, "NULL argument");
    set_device(plan->device);
    sinc_stage1(plan, c, c_is_real, (double2*)alpha_dev, as_stream(stream));
  });
}

int sincfft_sinc_stage3(sincfft_sinc_plan plan, const double* alpha_dev, double* out_dev,
                        void* stream) {
  return guarded([&] {
    if (!plan || !alpha_dev || !out_dev) sfb::fail(1, "NULL argument");
    set_device(plan->device);
    sinc_stage3(plan, (const double2*)alpha_dev, out_dev, SINCFFT_PTR_DEVICE, as_stream(stream));
  });
}

// ------------------------------------------------------------- classical NFFT
int sincfft_nfft_plan_create(sincfft_nfft_plan* plan, int64_t N, int64_t M, double sigma,
                             int32_t m, const double* x, int32_t ptr_kind, int32_t device,
                             void* stream) {
  return guarded([&] {
    if (!plan) sfb::fail(1, "plan pointer is NULL");
    *plan = nullptr;
    check_ptr_kind(ptr_kind);
    if (!x) sfb::fail(1, "nfft_plan: NULL nodes");
    if (N <= 0 || N % 2) sfb::fail(1, "nfft_plan: N must be a positive even integer");
    if (M <= 0) sfb::fail(1, "nfft_plan: nodes must be a nonempty 1-d array");
    set_device(device);
    cudaStream_t s = as_stream(stream);
    auto* h = new sincfft_nfft_plan_s();
    try {
      InBuf xb(x, sizeof(double) * M, ptr_kind, s);
      sfb::build_nfft(h->impl, N, M, sigma, m, (const double*)xb.ptr, device, s);
      SF_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      delete h;
      throw;
    }
    *plan = h;
  });
}

int sincfft_nfft_plan_destroy(sincfft_nfft_plan plan) {
  return guarded([&] {
    if (!plan) return;
    set_device(plan->impl.device);
    delete plan;
  });
}

int sincfft_nfft_plan_geometry(sincfft_nfft_plan plan, int64_t* n_over, sincfft_geometry* trafo,
                               sincfft_geometry* adjoint) {
  return guarded([&] {
    if (!plan) sfb::fail(1, "NULL plan");
    if (n_over) *n_over = plan->impl.n_over;
    if (trafo) fill_geometry(plan->impl.tr, trafo);
    if (adjoint) fill_geometry(plan->impl.ad_fft, adjoint);
  });
}

int sincfft_nfft_trafo(sincfft_nfft_plan plan, const double* c, double* out, int32_t ptr_kind,
                       void* stream) {
  return guarded([&] {
    if (!plan || !c || !out) sfb::fail(1, "NULL argument");
    check_ptr_kind(ptr_kind);
    const sfb::NfftPlanImpl& p = plan->impl;
    set_device(p.device);
    cudaStream_t s = as_stream(stream);
    InBuf cb(c, sizeof(double2) * (size_t)p.N, ptr_kind, s);
    OutBuf ob(out, sizeof(double2) * (size_t)p.M, ptr_kind, s);
    sfb::run_nfft_trafo(p, (const double2*)cb.ptr, (double2*)ob.ptr, s);
    ob.finish(s);
  });
}

int sincfft_nfft_adjoint(sincfft_nfft_plan plan, const double* y, double* out, int32_t ptr_kind,
                         void* stream) {
  return guarded([&] {
    if (!plan || !y || !out) sfb::fail(1, "NULL argument");
    check_ptr_kind(ptr_kind);
    const sfb::NfftPlanImpl& p = plan->impl;
    set_device(p.device);
    cudaStream_t s = as_stream(stream);
    InBuf yb(y, sizeof(double2) * (size_t)p.M, ptr_kind, s);
    OutBuf ob(out, sizeof(double2) * (size_t)p.N, ptr_kind, s);
    sfb::run_nfft_adjoint(p, (const double2*)yb.ptr, (double2*)ob.ptr, s);
    ob.finish(s);
  });
}

int sincfft_nfft_export_tables(sincfft_nfft_plan plan, int64_t* spread_idx, double* spread_val,
                               double* hat) {
  return guarded([&] {
    if (!plan) sfb::fail(1, "NULL plan");
    const sfb::NfftPlanImpl& p = plan->impl;
    set_device(p.device);
    cudaStream_t s = 0;
    const int64_t n = p.M * 2 * p.m;
    sfb::Scratch di(sizeof(int64_t) * n, s), dv(sizeof(double) * n, s), dh(sizeof(double) * p.N, s);
    sfb::export_nfft(p, di.as<int64_t>(), dv.as<double>(), dh.as<double>(), s);
    if (spread_idx)
      SF_CUDA(cudaMemcpyAsync(spread_idx, di.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    if (spread_val)
      SF_CUDA(cudaMemcpyAsync(spread_val, dv.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    if (hat) SF_CUDA(cudaMemcpyAsync(hat, dh.p, sizeof(double) * p.N, cudaMemcpyDeviceToHost, s));
    SF_CUDA(cudaStreamSynchronize(s));
  });
}

// ---------------------------------------------------------------- direct sums

int sincfft_nndft_direct(const double* f, const double* v, int64_t M1, const double* x,
                         int64_t M2, int64_t N, double* out, int32_t ptr_kind, int32_t device,
                         void* stream) {
  return guarded([&] {
    if (!f || !v || !x || !out) sfb::fail(1, "NULL argument");
    if (M1 <= 0 || M2 <= 0) sfb::fail(1, "f and x must be nonempty 1-d arrays");
    check_ptr_kind(ptr_kind);
    set_device(device);
    cudaStream_t s = as_stream(stream);
    InBuf fb(f, sizeof(double2) * M1, ptr_kind, s), vb(v, sizeof(double) * M1, ptr_kind, s),
        xb(x, sizeof(double) * M2, ptr_kind, s);
    OutBuf ob(out, sizeof(double2) * M2, ptr_kind, s);
    sfb::run_nndft_direct((const double2*)fb.ptr, (const double*)vb.ptr, M1,
                          (const double*)xb.ptr, M2, (double)N, (double2*)ob.ptr, s);
    ob.finish(s);
  });
}

int sincfft_ndft_direct(const double* c, int64_t Nc, const double* x, int64_t M, double* out,
                        int32_t ptr_kind, int32_t device, void* stream) {
  return guarded([&] {
    if (!c || !x || !out) sfb::fail(1, "NULL argument");
    if (Nc <= 0 || M <= 0) sfb::fail(1, "c and x must be nonempty 1-d arrays");
    if (Nc % 2) sfb::fail(1, "ndft_direct: len(c) must be even");
    check_ptr_kind(ptr_kind);
    set_device(device);
    cudaStream_t s = as_stream(stream);
    InBuf cb(c, sizeof(double2) * Nc, ptr_kind, s), xb(x, sizeof(double) * M, ptr_kind, s);
    OutBuf ob(out, sizeof(double2) * M, ptr_kind, s);
    sfb::run_ndft_direct((const double2*)cb.ptr, Nc, (const double*)xb.ptr, M, (double2*)ob.ptr,
                         s);
    ob.finish(s);
  });
}

int sincfft_sinc_direct(const double* c, const double* a, int64_t L1, const double* b,
                        int64_t L2, int64_t N, double* out, int32_t ptr_kind, int32_t device,
                        void* stream) {
  return guarded([&] {
    if (!c || !a || !b || !out) sfb::fail(1, "NULL argument");
    if (L1 <= 0 || L2 <= 0) sfb::fail(1, "c and b must be nonempty 1-d arrays");
    check_ptr_kind(ptr_kind);
    set_device(device);
    cudaStream_t s = as_stream(stream);
    InBuf cb(c, sizeof(double2) * L1, ptr_kind, s), ab(a, sizeof(double) * L1, ptr_kind, s),
        bb(b, sizeof(double) * L2, ptr_kind, s);
    OutBuf ob(out, sizeof(double2) * L2, ptr_kind, s);
    sfb::run_sinc_direct((const double2*)cb.ptr, (const double*)ab.ptr, L1,
                         (const double*)bb.ptr, L2, (double)N, (double2*)ob.ptr, s);
    ob.finish(s);
  });
}


int sincfft_window_eval(int32_t func, double beta, int32_t m, int64_t n_grid, const double* x,
                        int64_t n, double* out, int32_t ptr_kind, int32_t device, void* stream) {
  return guarded([&] {
    if (func < SINCFFT_WIN_OMEGA || func > SINCFFT_WIN_PHI_HAT)
      sfb::fail(1, "window_eval: unknown window function");
    if (n < 0) sfb::fail(1, "window_eval: negative length");
    if (n == 0) return;
    if (!x || !out) sfb::fail(1, "NULL argument");
    if ((func == SINCFFT_WIN_PHI || func == SINCFFT_WIN_PHI_HAT) && (m <= 0 || n_grid <= 0))
      sfb::fail(1, "window_eval: m and n_grid must be positive");
    check_ptr_kind(ptr_kind);
    set_device(device);
    cudaStream_t s = as_stream(stream);
    InBuf xb(x, sizeof(double) * n, ptr_kind, s);
    OutBuf ob(out, sizeof(double) * n, ptr_kind, s);
    sfb::run_window_eval(func, beta, m, n_grid, (const double*)xb.ptr, n, (double*)ob.ptr, s);
    ob.finish(s);
  });
}

}  // extern "C"
