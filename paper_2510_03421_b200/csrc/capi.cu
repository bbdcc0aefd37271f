// extern "C" entry points of libpermanent_b200.so (include/permanent_b200.h).
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <dlfcn.h>
#include <functional>
#include <map>
#include <mutex>
#include <thread>

#include <nccl.h>  // types only: the library is dlopen'ed (no link-time NCCL)

#include "engine.cuh"

using namespace permb200;

namespace permb200 {
const char* last_error();
int int_permanent(int alg, int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, int64_t* out,
                  int* fits_int64, void* stream);
int comb_permanent(bool ryser, int mode, int m, int n, const void* a, int64_t lda, int dev_ptr,
                   uint64_t step_budget, double* out, int64_t* ivalue, void* stream);
int batch_permanent(int alg, bool cplx, int64_t B, int m, int n, const double* a, double* out, int dev_ptr,
                    void* stream);
int batch_select(int m, int n);
int tiny_permanent(int alg, bool cplx, int m, int n, const double* a, double* out);
static int tiny_glynn_max_n() {
  static const int v = [] {
    const char* e = std::getenv("PERM_TINY_GLYNN_MAX_N");
    // 0 (off): since the walk path went zero-copy (setup as kernel
    // parameters, mapped result; one warp below 256 steps) it beats the
    // warp-per-matrix batch kernel at every n (profiles/r2_tiny_glynn_threshold.txt,
    // r2_dispatch_fit.txt); PERM_TINY_GLYNN_MAX_N=12 restores the old route
    return (e && *e) ? std::atoi(e) : 0;
  }();
  return v;
}
int dd_permanent(int alg, bool cplx, int m, int n, const double* a, int64_t lda, int dev_ptr, double* out4,
                 void* stream);
int int_walk_partial(int alg, int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, uint64_t k0,
                     uint64_t k1, int64_t* partial, void* stream);
int int_walk_finish(int alg, int m, int n, const int64_t* a, int64_t lda, int width, const int64_t* partials, int G,
                    int64_t* out, int* fits_int64);
int int_walk_plan(int alg, int m, int n, const int64_t* a, int64_t lda, int* kind, int* groups);
}

namespace {

int check_shape(int alg, int m, int n) {
  if (m < 1 || n < 1) {
    set_error("matrix must have m >= 1 and n >= 1");
    return PERM_BAD_SHAPE;
  }
  if (m > n) {
    set_error("need m <= n; transpose first");
    return PERM_BAD_SHAPE;
  }
  // src/algorithms.py:47 caps subset / sign walks at 62 columns; the device
  // kernels hold the state vector in registers, up to 64 entries.
  if (n > 62) {
    set_error("walk over more than 62 columns");
    return PERM_BAD_SHAPE;
  }
  (void)alg;
  return PERM_OK;
}

// Rectangular Ryser: the all-subsets weighted Gray walk (2^n steps) or the
// reference's combination order (sum_{s<=m} C(n, s) subsets), whichever the
// B200 cost model measured faster (tools/ryser_rect_probe.py,
// profiles/r2_ryser_rect.txt; per-call microseconds through the public API):
//   walk ~ 27 + 2^n (0.4 + 0.11 m) 1e-3   (zero-copy walk: latency floor 27 us)
//   comb ~ 36 + C (10 + 12 m) 1e-3        (combination kernels: floor 36 us)
bool ryser_rect_use_comb(int m, int n) {
  if (m >= n) return false;
  if (n > 62) return true;
  static const int force = [] {  // PERM_RYSER_RECT = "walk" / "comb" (experiments)
    const char* e = std::getenv("PERM_RYSER_RECT");
    if (!e || !*e) return 0;
    return std::string(e) == "comb" ? 1 : std::string(e) == "walk" ? 2 : 0;
  }();
  if (force) return force == 1;
  long double c = 0, b = 1;  // running C(n, s)
  for (int s = 1; s <= m; ++s) {
    b = b * (n - s + 1) / s;
    c += b;
  }
  const long double walk_us = 27.0L + std::ldexp(1.0L, n) * (0.4L + 0.11L * m) * 1e-3L;
  const long double comb_us = 36.0L + c * (10.0L + 12.0L * m) * 1e-3L;
  return comb_us < walk_us;
}

// Every float kernel of the reference starts its sum at zero = a[0,0] -
// a[0,0] (src/_kernels.py:30, 117, 228, 375, 533), so a non-finite a[0,0]
// turns the real (imaginary) part of the result into NaN even where the
// algebra would give +-inf (e.g. combinatoric of [[inf, 1], [1, 1]]).
// Applied to every float single-permanent result; finite a[0,0] changes
// nothing (not even the sign of a zero).
int ref_zero_quirk(bool cplx, const double* a, int dev_ptr, void* stream_, double* out) {
  double a00[2] = {0.0, 0.0};
  if (dev_ptr) {
    cudaStream_t stream = pick_stream(stream_);
    PERM_CUDA_TRY(cudaMemcpyAsync(a00, a, (cplx ? 2 : 1) * sizeof(double), cudaMemcpyDeviceToHost, stream));
    PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  } else {
    a00[0] = a[0];
    if (cplx) a00[1] = a[1];
  }
  if (!std::isfinite(a00[0])) out[0] += a00[0] - a00[0];
  if (cplx && !std::isfinite(a00[1])) out[1] += a00[1] - a00[1];
  return PERM_OK;
}

int walk_single_impl(int alg, bool cplx, int m, int n, const double* a, int64_t lda, int dev_ptr, double* out,
                     double* magsum, void* stream_);

// Single permanent through the walk engine; returns normalized value.
int walk_single(int alg, bool cplx, int m, int n, const double* a, int64_t lda, int dev_ptr, double* out,
                double* magsum, void* stream_) {
  const int st = walk_single_impl(alg, cplx, m, n, a, lda, dev_ptr, out, magsum, stream_);
  return st ? st : ref_zero_quirk(cplx, a, dev_ptr, stream_, out);
}

int walk_single_impl(int alg, bool cplx, int m, int n, const double* a, int64_t lda, int dev_ptr, double* out,
                     double* magsum, void* stream_) {
  clear_error();
  // very rectangular Ryser (and any width past the walks' 62 columns, where
  // the reference's ryser_rect has no cap): the reference's combination order
  if (alg == PERM_ALG_RYSER && magsum == nullptr && m >= 1 && m < n && ryser_rect_use_comb(m, n))
    return comb_permanent(true, cplx ? 1 : 0, m, n, a, lda, dev_ptr, UINT64_MAX, out, nullptr, stream_);
  int st = check_shape(alg, m, n);
  if (st) return st;
  // walks shorter than one warp-group of chunks (Glynn n <= 8, Ryser n <= 7)
  // on a caller's stream: the register-resident thread-per-matrix batch
  // kernels, batch of one (the default stream takes the zero-copy one-warp
  // walk below, which measured faster: profiles/r2_dispatch_fit.txt)
  if (magsum == nullptr && !dev_ptr && lda == n && walk_steps(alg, m, n) < 256 && stream_ != nullptr)
    return batch_permanent(alg, cplx, 1, m, n, a, out, 0, stream_);
  // Glynn n = 9..TINY_GLYNN_MAX_N (rectangles ones-padded and pre-scaled on the
  // host): one warp walks the matrix (the
  // warp-per-matrix batch kernel) on the zero-copy path, cheaper than a
  // device-wide walk launch at these sizes
  if (magsum == nullptr && !dev_ptr && lda == n && stream_ == nullptr && alg == PERM_ALG_GLYNN &&
      n <= tiny_glynn_max_n()) {
    const int tst = tiny_permanent(alg, cplx, m, n, a, out);
    if (tst >= 0) return tst;
  }
  cudaStream_t stream = pick_stream(stream_);
  HostMat A;
  st = load_matrix(m, n, a, lda, dev_ptr, cplx, &A, stream);
  if (st) return st;
  WalkSetup ws;
  st = build_walk(alg, A, &ws, /*exact_state=*/true);
  if (st) return st;
  // default stream: the zero-copy path (setup as kernel parameters, result
  // through mapped memory); a caller's stream keeps stream-ordered copies
  double r8[8];
  st = run_walk_host(ws, 0, walk_steps(alg, m, n), magsum != nullptr, r8, stream, stream_ == nullptr);
  if (st) return st;
  double re = r8[0] + r8[1], im = r8[2] + r8[3], mg = r8[4];
  normalize(alg, m, n, ws.scale_log2, &re, &im, &mg);
  out[0] = re;
  if (cplx) out[1] = im;
  if (magsum) *magsum = mg;
  return PERM_OK;
}

int walk_partial(int alg, bool cplx, int m, int n, const double* a, int64_t lda, int dev_ptr, uint64_t k_begin,
                 uint64_t k_end, int mag, double* partial, int partial_on_device, void* stream_) {
  clear_error();
  int st = check_shape(alg, m, n);
  if (st) return st;
  const uint64_t steps = walk_steps(alg, m, n);
  if (k_begin > k_end || k_end > steps) {
    set_error("Gray range outside the walk");
    return PERM_BAD_ARG;
  }
  cudaStream_t stream = pick_stream(stream_);
  HostMat A;
  st = load_matrix(m, n, a, lda, dev_ptr, cplx, &A, stream);
  if (st) return st;
  WalkSetup ws;
  st = build_walk(alg, A, &ws, /*exact_state=*/true);
  if (st) return st;
  Scratch* s = scratch();
  if (!s) return cuda_fail(cudaErrorNoDevice, "scratch");
  const size_t part_bytes = (size_t)kMaxPartials * kPartialStride * sizeof(double);
  st = ensure_dev(s, part_bytes + ws.buf.size() * sizeof(double) + 64 * sizeof(double) + 256);
  if (st) return st;
  if (k_begin == k_end) {  // empty shard
    if (partial_on_device) {
      PERM_CUDA_TRY(cudaMemsetAsync(partial, 0, 8 * sizeof(double), stream));
    } else {
      std::fill(partial, partial + 8, 0.0);
    }
    return PERM_OK;
  }
  if (!partial_on_device) return run_walk_host(ws, k_begin, k_end, mag, partial, stream, stream_ == nullptr);
  st = run_walk(ws, k_begin, k_end, mag, partial, stream);
  if (st) return st;
  s->async_pending = true;
  return PERM_OK;
}

int walk_finish(int alg, bool cplx, int m, int n, const double* a, int64_t lda, const double* partials, int G,
                double* out, double* magsum) {
  clear_error();
  int st = check_shape(alg, m, n);
  if (st) return st;
  int s = 0;
  if (alg == PERM_ALG_GLYNN && m < n) {
    HostMat A;
    st = load_matrix(m, n, a, lda, 0, cplx, &A, nullptr);
    if (st) return st;
    s = prescale_log2(A);
  }
  double h = 0, l = 0, h2 = 0, l2 = 0, mg = 0;
  for (int g = 0; g < G; ++g) {
    const double* p = partials + 8 * (size_t)g;
    dd_add(h, l, p[0], p[1]);
    dd_add(h2, l2, p[2], p[3]);
    mg += p[4];
  }
  double re = h + l, im = h2 + l2;
  normalize(alg, m, n, s, &re, &im, &mg);
  out[0] = re;
  if (cplx) out[1] = im;
  if (magsum) *magsum = mg;
  return ref_zero_quirk(cplx, a, 0, nullptr, out);
}

// ---- single-process multi-device driver (perm_sharded_*) ------------------
// One persistent host worker per shard slot: slot i binds devices[i] and
// walks shard i of `ngpu` with the single-device code path (its own
// thread-local scratch and the per-thread default stream of that device);
// the caller's thread combines the partials in shard order.  The exchange is
// 64 bytes per device once per permanent, so it goes through pinned host
// memory; nothing on the data path is collective.
class ShardPool {
 public:
  // run fns[i] on worker i, wait for all
  void run(const std::vector<std::function<void()>>& fns) {
    std::unique_lock<std::mutex> call(call_mu_);  // one sharded call at a time
    while (workers_.size() < fns.size()) workers_.emplace_back(new Worker());
    for (size_t i = 0; i < fns.size(); ++i) workers_[i]->post(fns[i]);
    for (size_t i = 0; i < fns.size(); ++i) workers_[i]->wait();
  }

 private:
  struct Worker {
    std::mutex mu;
    std::condition_variable cv;
    std::function<void()> job;
    bool busy = false;
    Worker() {
      std::thread([this] {
        for (;;) {
          std::function<void()> f;
          {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [this] { return (bool)job; });
            f = std::move(job);
          }
          f();
          {
            std::lock_guard<std::mutex> lk(mu);
            busy = false;
          }
          cv.notify_all();
        }
      }).detach();  // workers live for the process (their scratch is thread-local)
    }
    void post(std::function<void()> f) {
      {
        std::lock_guard<std::mutex> lk(mu);
        busy = true;
        job = std::move(f);
      }
      cv.notify_all();
    }
    void wait() {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [this] { return !busy; });
    }
  };
  std::mutex call_mu_;
  std::vector<Worker*> workers_;  // never freed: detached threads reference them
};

ShardPool& shard_pool() {
  static ShardPool* p = new ShardPool();
  return *p;
}

struct ShardStatus {
  int st = PERM_OK;
  std::string err;
};

// Run `body(i, k0, k1)` for every shard i on devices[i]; first failure wins.
int run_shards(int alg, int m, int n, int ngpu, const int* devices,
               const std::function<int(int, uint64_t, uint64_t)>& body) {
  if (ngpu < 1 || ngpu > 64 || devices == nullptr) {
    set_error("ngpu must be 1..64 with a device list");
    return PERM_BAD_ARG;
  }
  std::vector<ShardStatus> res(ngpu);
  std::vector<std::function<void()>> fns;
  for (int i = 0; i < ngpu; ++i) {
    fns.push_back([&, i] {
      uint64_t k0 = 0, k1 = 0;
      int st = perm_walk_shard(alg, m, n, i, ngpu, &k0, &k1);
      if (!st) {
        const cudaError_t e = cudaSetDevice(devices[i]);
        st = e == cudaSuccess ? body(i, k0, k1) : cuda_fail(e, "cudaSetDevice");
      }
      res[i].st = st;
      if (st) res[i].err = last_error();
    });
  }
  shard_pool().run(fns);
  for (int i = 0; i < ngpu; ++i)
    if (res[i].st) {
      set_error("shard " + std::to_string(i) + " (device " + std::to_string(devices[i]) + "): " + res[i].err);
      return res[i].st;
    }
  return PERM_OK;
}

// ---- NCCL exchange for the multi-device driver ----------------------------
// libnccl.so.2 is opened at first use (RTLD_NOLOAD first: reuse the copy a
// host framework such as torch already loaded), so the engine has no hard
// NCCL dependency.  One communicator clique per distinct device list.
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!api.tried) {
    api.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (h) {
      api.commInitAll = reinterpret_cast<decltype(api.commInitAll)>(dlsym(h, "ncclCommInitAll"));
      api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
      api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
      api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
      api.errStr = reinterpret_cast<decltype(api.errStr)>(dlsym(h, "ncclGetErrorString"));
      api.ok = api.commInitAll && api.allGather && api.groupStart && api.groupEnd && api.errStr;
    }
  }
  return api;
}

struct NcclClique {
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;
  std::vector<double*> part, gathered;  // per device: 8 doubles, G x 8 doubles
};

int nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string("NCCL error '") + nccl_api().errStr(r) + "' in " + what);
  return PERM_CUDA;
}

// communicators, streams and buffers for `devs`, created once (never freed:
// they live as long as the process, like the engine's other scratch)
int nccl_clique(const std::vector<int>& devs, NcclClique** out) {
  static std::map<std::vector<int>, NcclClique*> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(devs);
  if (it != cache.end()) {
    *out = it->second;
    return PERM_OK;
  }
  NcclApi& api = nccl_api();
  const int G = (int)devs.size();
  NcclClique* c = new NcclClique();
  c->comms.resize(G);
  ncclResult_t r = api.commInitAll(c->comms.data(), G, devs.data());
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitAll");
  }
  for (int i = 0; i < G; ++i) {
    PERM_CUDA_TRY(cudaSetDevice(devs[i]));
    cudaStream_t st;
    PERM_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    c->streams.push_back(st);
    double *p = nullptr, *g = nullptr;
    PERM_CUDA_TRY(cudaMalloc(&p, 8 * sizeof(double)));
    PERM_CUDA_TRY(cudaMalloc(&g, (size_t)G * 8 * sizeof(double)));
    c->part.push_back(p);
    c->gathered.push_back(g);
  }
  cache[devs] = c;
  *out = c;
  return PERM_OK;
}

// Every device walks its shard asynchronously (device-resident partial, one
// launch per device from this thread), one ncclAllGather of 8 doubles per
// device inside a group, one read-back from the first device.
int sharded_float_nccl(int alg, bool cplx, int m, int n, const double* a, int64_t lda, int ngpu,
                       const int* devices, double* parts) {
  int cur = 0;
  cudaGetDevice(&cur);
  std::vector<int> devs(devices, devices + ngpu);
  NcclClique* c = nullptr;
  int st = nccl_clique(devs, &c);
  if (st) return st;
  for (int i = 0; i < ngpu && !st; ++i) {
    uint64_t k0 = 0, k1 = 0;
    st = perm_walk_shard(alg, m, n, i, ngpu, &k0, &k1);
    if (st) break;
    PERM_CUDA_TRY(cudaSetDevice(devs[i]));
    st = walk_partial(alg, cplx, m, n, a, lda, 0, k0, k1, 0, c->part[i], 1, c->streams[i]);
  }
  if (st) {
    cudaSetDevice(cur);
    return st;
  }
  NcclApi& api = nccl_api();
  ncclResult_t r = api.groupStart();
  for (int i = 0; i < ngpu && r == ncclSuccess; ++i)
    r = api.allGather(c->part[i], c->gathered[i], 8, ncclFloat64, c->comms[i], c->streams[i]);
  const ncclResult_t r2 = api.groupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess) {
    cudaSetDevice(cur);
    return nccl_fail(r != ncclSuccess ? r : r2, "ncclAllGather");
  }
  PERM_CUDA_TRY(cudaSetDevice(devs[0]));
  PERM_CUDA_TRY(cudaMemcpyAsync(parts, c->gathered[0], (size_t)ngpu * 8 * sizeof(double), cudaMemcpyDeviceToHost,
                                c->streams[0]));
  for (int i = 0; i < ngpu; ++i) {
    PERM_CUDA_TRY(cudaSetDevice(devs[i]));
    PERM_CUDA_TRY(cudaStreamSynchronize(c->streams[i]));
  }
  PERM_CUDA_TRY(cudaSetDevice(cur));
  return PERM_OK;
}

// Exchange for perm_sharded_{f64,c128}: NCCL when the devices are distinct
// and libnccl is present, else the host-worker path.  PERM_SHARDED_EXCHANGE
// = "nccl" / "host" forces one.
bool use_nccl_exchange(int ngpu, const int* devices) {
  const char* e = std::getenv("PERM_SHARDED_EXCHANGE");
  const std::string mode = e ? e : "";
  if (mode == "host") return false;
  std::vector<int> d(devices, devices + ngpu);
  std::sort(d.begin(), d.end());
  if (std::adjacent_find(d.begin(), d.end()) != d.end()) return false;  // a device listed twice
  if (mode != "nccl" && ngpu < 2) return false;
  return nccl_api().ok;
}

int sharded_float(int alg, bool cplx, int m, int n, const double* a, int64_t lda, int ngpu, const int* devices,
                  double* out, double* magsum) {
  clear_error();
  int st = check_shape(alg, m, n);
  if (st) return st;
  if (alg != PERM_ALG_GLYNN && alg != PERM_ALG_RYSER) {
    set_error("sharded walks are Glynn or Ryser");
    return PERM_BAD_ARG;
  }
  std::vector<double> parts((size_t)std::max(ngpu, 1) * 8, 0.0);
  if (ngpu >= 1 && ngpu <= 64 && devices && magsum == nullptr && use_nccl_exchange(ngpu, devices)) {
    st = sharded_float_nccl(alg, cplx, m, n, a, lda, ngpu, devices, parts.data());
    if (st) return st;
    return walk_finish(alg, cplx, m, n, a, lda, parts.data(), ngpu, out, magsum);
  }
  st = run_shards(alg, m, n, ngpu, devices, [&](int i, uint64_t k0, uint64_t k1) {
    return walk_partial(alg, cplx, m, n, a, lda, 0, k0, k1, magsum != nullptr, &parts[(size_t)i * 8], 0, nullptr);
  });
  if (st) return st;
  return walk_finish(alg, cplx, m, n, a, lda, parts.data(), ngpu, out, magsum);
}

}  // namespace

extern "C" {

int perm_version(void) { return 100; }
const char* perm_last_error(void) { return permb200::last_error(); }

int perm_set_device(int device) {
  clear_error();
  PERM_CUDA_TRY(cudaSetDevice(device));
  return PERM_OK;
}

double perm_last_kernel_ms(void) {
  KernelTimer& t = kernel_timer();
  if (!t.ok || !t.pending) return -1.0;
  if (cudaEventSynchronize(t.stop) != cudaSuccess) return -1.0;
  float ms = 0.0f;
  if (cudaEventElapsedTime(&ms, t.start, t.stop) != cudaSuccess) return -1.0;
  return (double)ms;
}

int perm_set_timing(int on) {
  set_timing(on != 0);
  return PERM_OK;
}

int perm_last_kernel_plan(int* grid, int* log2L) {
  KernelTimer& t = kernel_timer();
  *grid = t.last_grid;
  *log2L = t.last_log2L;
  return PERM_OK;
}

int perm_fp64_peak_probe(double seconds, double* dfma_per_s) {
  clear_error();
  return fp64_peak_probe(seconds, 0, dfma_per_s);
}

int perm_fp64_pipe_probe(int op, double seconds, double* ops_per_s) {
  clear_error();
  return fp64_peak_probe(seconds, op, ops_per_s);
}

int perm_walk_repeat_ms(int alg, int cplx, int m, int n, const double* a, int64_t lda, int reps,
                        double* ms_per_launch) {
  clear_error();
  if ((alg != PERM_ALG_GLYNN && alg != PERM_ALG_RYSER) || reps < 1 || !ms_per_launch) {
    set_error("alg must be GLYNN or RYSER, reps >= 1");
    return PERM_BAD_ARG;
  }
  int st = check_shape(alg, m, n);
  if (st) return st;
  HostMat A;
  st = load_matrix(m, n, a, lda, 0, cplx != 0, &A, nullptr);
  if (st) return st;
  WalkSetup ws;
  st = build_walk(alg, A, &ws, /*exact_state=*/true);
  if (st) return st;
  Scratch* s = scratch();
  if (!s) return cuda_fail(cudaErrorNoDevice, "scratch");
  cudaStream_t stream;
  PERM_CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  const size_t part_bytes = (size_t)kMaxPartials * kPartialStride * sizeof(double);
  st = ensure_dev(s, part_bytes + ws.buf.size() * sizeof(double) + 64 * sizeof(double) + 256);
  if (st) return st;
  double* dst = reinterpret_cast<double*>(static_cast<char*>(s->dev) + s->dev_cap) - 8;
  const uint64_t steps = walk_steps(alg, m, n);
  st = run_walk(ws, 0, steps, 0, dst, stream);  // warm-up (and the setup's first upload)
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (!st) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, stream);
    for (int r = 0; r < reps && !st; ++r) st = run_walk_resident(ws, 0, steps, 0, dst, stream);
    cudaEventRecord(e1, stream);
  }
  const cudaError_t se = cudaStreamSynchronize(stream);
  float ms = 0.0f;
  if (!st && se == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaStreamDestroy(stream);
  if (st) return st;
  if (se != cudaSuccess) return cuda_fail(se, "walk repeat");
  *ms_per_launch = (double)ms / reps;
  return PERM_OK;
}

int perm_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int perm_glynn_f64(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, double* magsum,
                   void* stream) {
  return walk_single(PERM_ALG_GLYNN, false, m, n, a, lda, dev_ptr, out, magsum, stream);
}
int perm_glynn_c128(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, double* magsum,
                    void* stream) {
  return walk_single(PERM_ALG_GLYNN, true, m, n, a, lda, dev_ptr, out, magsum, stream);
}
int perm_ryser_f64(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, double* magsum,
                   void* stream) {
  return walk_single(PERM_ALG_RYSER, false, m, n, a, lda, dev_ptr, out, magsum, stream);
}
int perm_ryser_c128(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, double* magsum,
                    void* stream) {
  return walk_single(PERM_ALG_RYSER, true, m, n, a, lda, dev_ptr, out, magsum, stream);
}

}  // extern "C"

namespace {
// Small integer matrices whose every intermediate -- of the reference's
// checked int64 kernel and of the float engine alike -- is an integer below
// 2^52: the state / row sums are bounded by the column (Glynn, ones pad
// included) or row (Ryser, combinatoric) sums of |a|, the products by their
// product, the running sums by 2^(steps) times that.  On these the float
// path is exact and the reference cannot flag an overflow, so its value and
// flag are the float engine's, at the zero-copy path's latency (the exact
// integer path stages summaries and certificates: ~2x slower per call).
bool int_small_certified(int alg, int m, int n, const int64_t* a, int64_t lda) {
  if (m < 1 || m > n || n > 30) return false;
  long double prod_r = 1.0L, prod_c = 1.0L;
  for (int i = 0; i < m; ++i) {
    long double r = 0;
    for (int j = 0; j < n; ++j) {
      const int64_t x = a[(size_t)i * lda + j];
      if (x > (1LL << 31) || x < -(1LL << 31)) return false;
      r += std::fabs((long double)x);
    }
    prod_r *= std::max(r, 1.0L);
  }
  for (int j = 0; j < n; ++j) {
    long double c = (long double)(n - m);
    for (int i = 0; i < m; ++i) c += std::fabs((long double)a[(size_t)i * lda + j]);
    prod_c *= std::max(c, 1.0L);
  }
  long double bound;
  // Glynn: square only.  The rectangular float walk runs on the pre-scaled
  // matrix 2^s A (build_walk); with s < 0 its state entries are multiples of
  // 2^s and the n-factor products need up to n |s| more mantissa bits, so
  // they are not exact (found by the int128 fuzz: a 7x9 matrix with one
  // column of 674s came back 84 off).
  if (alg == PERM_ALG_GLYNN) bound = (m == n) ? std::ldexp(prod_c, n) : 1e300L;
  else if (alg == PERM_ALG_RYSER) bound = (m == n) ? std::ldexp(prod_r, n + 1) : 1e300L;
  else bound = prod_r;
  return bound < std::ldexp(1.0L, 52);
}

// -1: not taken (not certified, or a host-side refusal); else the status
int int_via_float(int alg, int m, int n, const int64_t* a, int64_t lda, int dev_ptr, uint64_t step_budget,
                  int64_t* out, int* fits_int64, void* stream) {
  if (dev_ptr || stream != nullptr || !int_small_certified(alg, m, n, a, lda)) return -1;
  std::vector<double> d((size_t)m * n);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) d[(size_t)i * n + j] = (double)a[(size_t)i * lda + j];
  double v = 0.0;
  const int st = (alg == PERM_ALG_COMBINATORIC)
                     ? comb_permanent(false, 0, m, n, d.data(), n, 0, step_budget, &v, nullptr, nullptr)
                     : walk_single(alg, false, m, n, d.data(), n, 0, &v, nullptr, nullptr);
  if (st) return st;
  const double r = std::nearbyint(v);
  if (!(std::fabs(v - r) <= 1e-6) || !(std::fabs(r) < 4503599627370496.0)) return -1;  // not exact: exact path
  const int64_t iv = (int64_t)r;
  out[0] = iv;
  out[1] = iv < 0 ? -1 : 0;
  if (fits_int64) *fits_int64 = 1;
  return PERM_OK;
}
}  // namespace

extern "C" {

int perm_glynn_i64(int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, int64_t* out,
                   int* fits_int64, void* stream) {
  if (width == 64 || width == 128) {
    const int fst = int_via_float(PERM_ALG_GLYNN, m, n, a, lda, dev_ptr, UINT64_MAX, out, fits_int64, stream);
    if (fst >= 0) return fst;
  }
  return int_permanent(PERM_ALG_GLYNN, m, n, a, lda, dev_ptr, width, out, fits_int64, stream);
}
int perm_ryser_i64(int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, int64_t* out,
                   int* fits_int64, void* stream) {
  if (width == 64 && m < n && m >= 1) {
    // the reference's rectangular int kernel walks combinations
    // lexicographically (src/_kernels.py:265-365); its overflow flag depends
    // on that order, so replay it
    int64_t v = 0;
    int st = comb_permanent(true, 2, m, n, a, lda, dev_ptr, UINT64_MAX, nullptr, &v, stream);
    if (st) return st;
    out[0] = v;
    out[1] = v < 0 ? -1 : 0;
    if (fits_int64) *fits_int64 = 1;
    return PERM_OK;
  }
  if (m == n && (width == 64 || width == 128)) {
    const int fst = int_via_float(PERM_ALG_RYSER, m, n, a, lda, dev_ptr, UINT64_MAX, out, fits_int64, stream);
    if (fst >= 0) return fst;
  }
  return int_permanent(PERM_ALG_RYSER, m, n, a, lda, dev_ptr, width, out, fits_int64, stream);
}

// The reference's ryser_rect kernels for any m <= n, square included
// (src/algorithms.py:118-137 accepts m == n; src/_kernels.py:226-365): the
// lexicographic combination order, so the checked-int64 overflow flag of
// ryser_rectangular(square) is the reference's (the square Gray walk checks
// other intermediates).
int perm_ryser_rect_f64(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, void* stream) {
  const int st = comb_permanent(true, 0, m, n, a, lda, dev_ptr, UINT64_MAX, out, nullptr, stream);
  return st ? st : ref_zero_quirk(false, a, dev_ptr, stream, out);
}
int perm_ryser_rect_c128(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, void* stream) {
  const int st = comb_permanent(true, 1, m, n, a, lda, dev_ptr, UINT64_MAX, out, nullptr, stream);
  return st ? st : ref_zero_quirk(true, a, dev_ptr, stream, out);
}
int perm_ryser_rect_i64(int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int64_t* out, void* stream) {
  int64_t v = 0;
  int st = comb_permanent(true, 2, m, n, a, lda, dev_ptr, UINT64_MAX, nullptr, &v, stream);
  if (st) return st;
  out[0] = v;
  out[1] = v < 0 ? -1 : 0;
  return PERM_OK;
}

int perm_comb_f64(int m, int n, const double* a, int64_t lda, int dev_ptr, uint64_t step_budget, double* out,
                  void* stream) {
  const int st = comb_permanent(false, 0, m, n, a, lda, dev_ptr, step_budget, out, nullptr, stream);
  return st ? st : ref_zero_quirk(false, a, dev_ptr, stream, out);
}
int perm_comb_c128(int m, int n, const double* a, int64_t lda, int dev_ptr, uint64_t step_budget, double* out,
                   void* stream) {
  const int st = comb_permanent(false, 1, m, n, a, lda, dev_ptr, step_budget, out, nullptr, stream);
  return st ? st : ref_zero_quirk(true, a, dev_ptr, stream, out);
}
int perm_comb_i64(int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, uint64_t step_budget,
                  int64_t* out, int* fits_int64, void* stream) {
  if (width != 64 && width != 128) {
    clear_error();
    set_error("width must be 64 or 128");
    return PERM_BAD_ARG;
  }
  const int fst = int_via_float(PERM_ALG_COMBINATORIC, m, n, a, lda, dev_ptr, step_budget, out, fits_int64, stream);
  if (fst >= 0) return fst;
  int st = comb_permanent(false, width == 64 ? 2 : 3, m, n, a, lda, dev_ptr, step_budget, nullptr, out, stream);
  if (st) return st;
  if (width == 64) out[1] = out[0] < 0 ? -1 : 0;
  if (fits_int64) *fits_int64 = (out[1] == (out[0] < 0 ? -1 : 0)) ? 1 : 0;
  return PERM_OK;
}

int perm_batch_f64(int alg, int64_t B, int m, int n, const double* a, double* out, int dev_ptr, void* stream) {
  return batch_permanent(alg, false, B, m, n, a, out, dev_ptr, stream);
}
int perm_batch_c128(int alg, int64_t B, int m, int n, const double* a, double* out, int dev_ptr, void* stream) {
  return batch_permanent(alg, true, B, m, n, a, out, dev_ptr, stream);
}
int perm_batch_select(int m, int n) { return batch_select(m, n); }

int perm_permanent_dd(int alg, int cplx, int m, int n, const double* a, int64_t lda, int dev_ptr, double* out4,
                      void* stream) {
  return dd_permanent(alg, cplx != 0, m, n, a, lda, dev_ptr, out4, stream);
}

uint64_t perm_walk_steps(int alg, int m, int n) {
  if (check_shape(alg, m, n)) return 0;
  return walk_steps(alg, m, n);
}

int perm_walk_shard(int alg, int m, int n, int rank, int world, uint64_t* k_begin, uint64_t* k_end) {
  clear_error();
  int st = check_shape(alg, m, n);
  if (st) return st;
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("bad rank/world");
    return PERM_BAD_ARG;
  }
  const uint64_t steps = walk_steps(alg, m, n);
  // split in units of 2^u with >= 64 units per rank where possible, so each
  // shard boundary is aligned for the full-speed chunked kernel
  int lg = 0;
  while ((1 << lg) < world) ++lg;
  const int lsteps = __builtin_ctzll(steps);
  const int u = std::max(0, lsteps - lg - 6);
  const uint64_t units = steps >> u;
  const uint64_t b = (uint64_t)((unsigned __int128)units * (unsigned)rank / (unsigned)world);
  const uint64_t e = (uint64_t)((unsigned __int128)units * (unsigned)(rank + 1) / (unsigned)world);
  *k_begin = b << u;
  *k_end = e << u;
  return PERM_OK;
}

int perm_walk_partial_f64(int alg, int m, int n, const double* a, int64_t lda, int dev_ptr, uint64_t k_begin,
                          uint64_t k_end, int mag, double* partial, int partial_on_device, void* stream) {
  return walk_partial(alg, false, m, n, a, lda, dev_ptr, k_begin, k_end, mag, partial, partial_on_device, stream);
}
int perm_walk_partial_c128(int alg, int m, int n, const double* a, int64_t lda, int dev_ptr, uint64_t k_begin,
                           uint64_t k_end, int mag, double* partial, int partial_on_device, void* stream) {
  return walk_partial(alg, true, m, n, a, lda, dev_ptr, k_begin, k_end, mag, partial, partial_on_device, stream);
}
int perm_walk_finish_f64(int alg, int m, int n, const double* a, int64_t lda, const double* partials, int G,
                         double* out, double* magsum) {
  return walk_finish(alg, false, m, n, a, lda, partials, G, out, magsum);
}
int perm_walk_finish_c128(int alg, int m, int n, const double* a, int64_t lda, const double* partials, int G,
                          double* out, double* magsum) {
  return walk_finish(alg, true, m, n, a, lda, partials, G, out, magsum);
}

int perm_walk_partial_i64(int alg, int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width,
                          uint64_t k_begin, uint64_t k_end, int64_t* partial, void* stream) {
  return int_walk_partial(alg, m, n, a, lda, dev_ptr, width, k_begin, k_end, partial, stream);
}
int perm_walk_finish_i64(int alg, int m, int n, const int64_t* a, int64_t lda, int width, const int64_t* partials,
                         int G, int64_t* out, int* fits_int64) {
  return int_walk_finish(alg, m, n, a, lda, width, partials, G, out, fits_int64);
}

int perm_int_walk_plan(int alg, int m, int n, const int64_t* a, int64_t lda, int* kind, int* groups) {
  if (a == nullptr || kind == nullptr || groups == nullptr) return PERM_BAD_ARG;
  return int_walk_plan(alg, m, n, a, lda, kind, groups);
}

int perm_sharded_exchange(int ngpu, const int* devices) {
  if (ngpu < 1 || ngpu > 64 || devices == nullptr) return -1;
  return use_nccl_exchange(ngpu, devices) ? 1 : 0;
}

int perm_sharded_f64(int alg, int m, int n, const double* a, int64_t lda, int ngpu, const int* devices, double* out,
                     double* magsum) {
  return sharded_float(alg, false, m, n, a, lda, ngpu, devices, out, magsum);
}
int perm_sharded_c128(int alg, int m, int n, const double* a, int64_t lda, int ngpu, const int* devices,
                      double* out, double* magsum) {
  return sharded_float(alg, true, m, n, a, lda, ngpu, devices, out, magsum);
}
int perm_sharded_i64(int alg, int m, int n, const int64_t* a, int64_t lda, int width, int ngpu, const int* devices,
                     int64_t* out, int* fits_int64) {
  clear_error();
  int st = check_shape(alg, m, n);
  if (st) return st;
  std::vector<int64_t> parts((size_t)std::max(ngpu, 1) * 8, 0);
  st = run_shards(alg, m, n, ngpu, devices, [&](int i, uint64_t k0, uint64_t k1) {
    return int_walk_partial(alg, m, n, a, lda, 0, width, k0, k1, &parts[(size_t)i * 8], nullptr);
  });
  if (st) return st;
  return int_walk_finish(alg, m, n, a, lda, width, parts.data(), ngpu, out, fits_int64);
}

// src/dispatch.py:84-95 (strict '>' comparisons: ties take the else branch)
int perm_select(int m, int n, const double* p, int64_t batch, int ngpu) {
  (void)batch;
  (void)ngpu;
  if (m > n || m < 1) return -PERM_BAD_SHAPE;
  const double r = (double)m / (double)n;
  if ((double)n <= p[7]) {
    if (m == n && (double)n <= p[3]) return PERM_ALG_COMBINATORIC;
    const double h1 = p[0] * r + p[1] * n + p[2];
    return h1 > 0 ? PERM_ALG_COMBINATORIC : PERM_ALG_GLYNN;
  }
  const double h2 = p[4] * r + p[5] * n + p[6];
  return h2 > 0 ? PERM_ALG_GLYNN : PERM_ALG_RYSER;
}

}  // extern "C"
