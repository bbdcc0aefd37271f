// Host-side engine internals: error state, scratch, matrix staging, walk
// setup/normalization and the fixed-order finalize kernel.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>

#include "engine.cuh"

namespace permb200 {

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
void clear_error() { g_err.clear(); }
const char* last_error() { return g_err.c_str(); }
int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string("CUDA error '") + cudaGetErrorString(e) + "' in " + what);
  return PERM_CUDA;
}

// ---------------------------------------------------------------- scratch
static thread_local Scratch g_scratch[16];

Scratch* scratch() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  if (dev < 0 || dev >= 16) return nullptr;
  Scratch* s = &g_scratch[dev];
  if (s->device != dev) {
    s->device = dev;
    if (cudaMallocHost(&s->host, kHostResultDoubles * sizeof(double)) != cudaSuccess) return nullptr;
    if (cudaMalloc(&s->done, sizeof(unsigned int)) != cudaSuccess) return nullptr;
    if (cudaMemset(s->done, 0, sizeof(unsigned int)) != cudaSuccess) return nullptr;
    // keep stream-ordered allocations cached across synchronizations (the
    // default release threshold of 0 returns them to the driver at every
    // sync, which made each batch call pay ~2 ms of re-mapping)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  return s;
}

int ensure_dev(Scratch* s, size_t bytes) {
  if (s->dev_cap >= bytes) return PERM_OK;
  if (s->dev) {
    PERM_CUDA_TRY(cudaDeviceSynchronize());
    PERM_CUDA_TRY(cudaFree(s->dev));
    s->dev = nullptr;
    s->dev_cap = 0;
  }
  size_t cap = std::max<size_t>(bytes, 1 << 20);
  PERM_CUDA_TRY(cudaMalloc(&s->dev, cap));
  s->dev_cap = cap;
  return PERM_OK;
}

int stage_h2d(Scratch* s, void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (s->stage_cap < bytes) {
    if (s->stage) cudaFreeHost(s->stage);
    s->stage = nullptr;
    s->stage_cap = 0;
    const size_t cap = std::max<size_t>(bytes, 1 << 16);
    PERM_CUDA_TRY(cudaMallocHost(&s->stage, cap));
    s->stage_cap = cap;
  }
  // the staging buffer (and the scratch it feeds) may still be in use by an
  // asynchronous call (device-side partial) queued earlier on this thread
  if (s->async_pending) {
    PERM_CUDA_TRY(cudaDeviceSynchronize());
    s->async_pending = false;
  }
  std::memcpy(s->stage, src, bytes);
  PERM_CUDA_TRY(cudaMemcpyAsync(dst, s->stage, bytes, cudaMemcpyHostToDevice, stream));
  return PERM_OK;
}

cudaStream_t pick_stream(void* stream) {
  (void)scratch();  // per-device setup (pinned buffers, mem-pool threshold) on first use
  return stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
}

// ---------------------------------------------------------------- matrices
int load_matrix(int m, int n, const double* a, int64_t lda, int dev_ptr, bool cplx, HostMat* out,
                cudaStream_t stream) {
  if (m < 1 || n < 1) {
    set_error("matrix must have m >= 1 and n >= 1");
    return PERM_BAD_SHAPE;
  }
  if (lda < n) {
    set_error("lda < n");
    return PERM_BAD_ARG;
  }
  const int w = cplx ? 2 : 1;
  out->m = m;
  out->n = n;
  out->cplx = cplx;
  out->d.assign((size_t)m * n * w, 0.0);
  if (dev_ptr) {
    PERM_CUDA_TRY(cudaMemcpy2DAsync(out->d.data(), (size_t)n * w * sizeof(double), a,
                                    (size_t)lda * w * sizeof(double), (size_t)n * w * sizeof(double), m,
                                    cudaMemcpyDeviceToHost, stream));
    PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  } else {
    for (int i = 0; i < m; ++i)
      std::memcpy(&out->d[(size_t)i * n * w], a + (size_t)i * lda * w, (size_t)n * w * sizeof(double));
  }
  return PERM_OK;
}

// ---------------------------------------------------------------- setup
uint64_t walk_steps(int alg, int m, int n) {
  (void)m;
  if (alg == PERM_ALG_GLYNN) return 1ull << (n - 1);
  return (n >= 64) ? 0 : (1ull << n);
}

int prescale_log2(const HostMat& A) {
  // RMS over the nonzero entries: zeros carry no scale (a padded identity
  // keeps k = 1 and stays exact), dense rows get k ~ 1/|a_ij|
  long double ss = 0;
  long nz = 0;
  for (int i = 0; i < A.m; ++i)
    for (int j = 0; j < A.n; ++j) {
      long double r = A.re(i, j), im = A.im(i, j);
      const long double q = r * r + im * im;
      if (q != 0) {
        ss += q;
        ++nz;
      }
    }
  if (nz == 0) return 0;
  double rms = std::sqrt((double)(ss / (long double)nz));
  if (!std::isfinite(rms) || rms == 0.0) return 0;
  double e = -std::log2(rms);
  double r = std::nearbyint(e);  // ties-to-even, same as Python round()
  return (int)r;
}

static inline double binom_d(int a, int b) {
  if (b < 0 || b > a) return 0.0;
  unsigned __int128 r = 1;
  for (int i = 1; i <= b; ++i) r = r * (unsigned __int128)(a - b + i) / (unsigned __int128)i;
  return (double)(long double)r;
}

// Exact walk state (DESIGN 2.1 "Exact state"): every state component of a
// walk is a signed subset sum of one column (Glynn: sum_i d_i a_ij) or one
// row (Ryser: sum_{j in S} a_ij), bounded by c = sum |entries| of it.  Round
// each entry of that column / row to the grid q = 2^(e - 52), c <= 2^e: then
// every partial sum is an integer multiple of q below 2^52 q, so seeds and all
// 2^B in-place updates are exact and the state never drifts.  The matrix
// moves by <= q/2 per entry, the same size as one FP64 rounding of the column
// sums the walk already forms (<= c 2^-52); a CPU study
// (tools/chunk_drift_exp.c, profiles/r2_chunk_drift.txt) puts the drift
// of the unquantized walk at 30-100x the error this leaves.  Real and
// imaginary parts get their own grids.  Integer-valued matrices are already
// on every grid q <= 1 and stay bit-identical.
// x rounded to the nearest multiple of 2^qe (ties to even).  |x| < 2^(qe+51):
// one add and one subtract of C = 1.5 * 2^(qe+52), whose binade has ulp
// 2^qe (the walk's setup is on the per-call path: libm ldexp / nearbyint per
// entry cost ~6 us at n = 20); larger |x| (one entry carrying most of its
// line) and grids near the top of the range take the exact libm path.
static inline double round_to_grid(double x, int qe, double C, bool magic_ok) {
  if (magic_ok && std::fabs(x) < C * (1.0 / 3.0)) {
    const double t = x + C;  // IEEE semantics (no -ffast-math): not folded
    return t - C;
  }
  return std::ldexp(std::nearbyint(std::ldexp(x, -qe)), qe);
}

static void quantize_line(double* x, size_t count, size_t stride, const std::vector<size_t>& keep_exact) {
  long double c = 0;
  for (size_t k = 0; k < count; ++k) c += std::fabs((long double)x[k * stride]);
  if (!(c > 0) || !std::isfinite((double)c)) return;
  int e = 0;
  std::frexp((double)c * (1.0 + 4e-16), &e);  // c <= 2^e (margin for the long double -> double cast)
  const int qe = std::max(e - 52, -1074);
  const bool magic_ok = qe + 52 <= 1000;
  const double C = magic_ok ? std::ldexp(1.5, qe + 52) : 0.0;
  for (size_t k : keep_exact) {  // ones rows of rectangular Glynn must stay on the grid
    if (round_to_grid(x[k * stride], qe, C, magic_ok) != x[k * stride]) return;
  }
  for (size_t k = 0; k < count; ++k) x[k * stride] = round_to_grid(x[k * stride], qe, C, magic_ok);
}

int build_walk(int alg, const HostMat& A, WalkSetup* ws, bool exact_state) {
  const int m = A.m, n = A.n;
  const int w = A.cplx ? 2 : 1;
  ws->cplx = A.cplx;
  ws->exact = exact_state;
  ws->scale_log2 = 0;
  ws->weighted = false;
  ws->wlen = 0;
  if (alg == PERM_ALG_GLYNN) {
    // ones-padded n x n matrix, real rows scaled by k = 2^s
    const int s = (m < n) ? prescale_log2(A) : 0;
    const bool fast_scale = std::abs(s) <= 1000;  // x * 2^s == ldexp(x, s) while 2^s is finite
    const double ks = fast_scale ? std::ldexp(1.0, s) : 1.0;
    ws->scale_log2 = s;
    ws->P = n;
    ws->B = n - 1;
    ws->v0_off = 0;
    ws->U_off = (size_t)n * w;
    ws->buf.assign((size_t)n * w + (size_t)(n - 1) * n * w, 0.0);
    // the walked matrix: real rows scaled by 2^s, ones rows below
    std::vector<double> G((size_t)n * n * w);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        G[((size_t)i * n + j) * w] = i < m ? (fast_scale ? A.re(i, j) * ks : std::ldexp(A.re(i, j), s)) : 1.0;
        if (w == 2)
          G[((size_t)i * n + j) * w + 1] = i < m ? (fast_scale ? A.im(i, j) * ks : std::ldexp(A.im(i, j), s)) : 0.0;
      }
    if (exact_state) {
      std::vector<size_t> ones;
      for (int i = m; i < n; ++i) ones.push_back((size_t)i);
      for (int j = 0; j < n; ++j) {
        quantize_line(&G[(size_t)j * w], (size_t)n, (size_t)n * w, ones);
        if (w == 2) quantize_line(&G[(size_t)j * w + 1], (size_t)n, (size_t)n * w, {});
      }
    }
    auto row_re = [&](int i, int j) { return G[((size_t)i * n + j) * w]; };
    auto row_im = [&](int i, int j) { return G[((size_t)i * n + j) * w + 1]; };
    for (int j = 0; j < n; ++j) {
      // exactly-rounded column sums (long double accumulation)
      long double sr = 0, si = 0;
      for (int i = 0; i < n; ++i) { sr += row_re(i, j); si += row_im(i, j); }
      ws->buf[(size_t)j * w] = (double)sr;
      if (w == 2) ws->buf[(size_t)j * w + 1] = (double)si;
    }
    for (int t = 0; t < n - 1; ++t) {
      const int i = n - 1 - t;  // Gray bit t flips row n-1-t (src/_kernels.py:393)
      for (int j = 0; j < n; ++j) {
        ws->buf[ws->U_off + ((size_t)t * n + j) * w] = -2.0 * row_re(i, j);
        if (w == 2) ws->buf[ws->U_off + ((size_t)t * n + j) * w + 1] = -2.0 * row_im(i, j);
      }
    }
    return PERM_OK;
  }
  if (alg == PERM_ALG_RYSER) {
    // state = row sums over the chosen column subset; Gray bit t = column t
    ws->P = m;
    ws->B = n;
    ws->v0_off = 0;
    ws->U_off = (size_t)m * w;
    size_t nU = (size_t)n * m * w;
    if (m < n) {
      ws->weighted = true;
      ws->wlen = n + 1;
    }
    ws->w_off = ws->U_off + nU;
    ws->buf.assign(ws->w_off + ws->wlen, 0.0);
    for (int t = 0; t < n; ++t)
      for (int i = 0; i < m; ++i) {
        ws->buf[ws->U_off + ((size_t)t * m + i) * w] = A.re(i, t);
        if (w == 2) ws->buf[ws->U_off + ((size_t)t * m + i) * w + 1] = A.im(i, t);
      }
    if (ws->weighted)  // src/algorithms.py:110-115; zero above size m
      for (int s = 1; s <= m; ++s) {
        double c = binom_d(n - s, m - s);
        ws->buf[ws->w_off + s] = ((m - s) & 1) ? -c : c;
      }
    if (exact_state)  // state component i = row i's subset sum: U[t][i] over t
      for (int i = 0; i < m; ++i)
        for (int part = 0; part < w; ++part)
          quantize_line(&ws->buf[ws->U_off + (size_t)i * w + part], (size_t)n, (size_t)m * w, {});
    return PERM_OK;
  }
  set_error("unknown algorithm");
  return PERM_BAD_ARG;
}

void normalize(int alg, int m, int n, int scale_log2, double* re, double* im, double* mag) {
  if (alg == PERM_ALG_GLYNN) {
    // per = sum / (2^(n-1) * (n-m)! * k^m)   (src/algorithms.py:159-160, 182-184)
    const int e = -(n - 1) - m * scale_log2;
    double f = 1.0;
    for (int i = 2; i <= n - m; ++i) f *= (double)i;
    *re = std::ldexp(*re, e) / f;
    *im = std::ldexp(*im, e) / f;
    *mag = std::ldexp(*mag, e) / f;
  } else if (alg == PERM_ALG_RYSER) {
    if (m == n && (n & 1)) {  // src/_kernels.py:143-144
      *re = -*re;
      *im = -*im;
    }
  }
}

// ---------------------------------------------------------------- timing
static std::atomic<bool> g_timing{false};
bool timing_enabled() { return g_timing.load(std::memory_order_relaxed); }
void set_timing(bool on) { g_timing.store(on, std::memory_order_relaxed); }
// CUDA events bracketing the last walk kernel launched by this host thread
// (bench.py reads its duration for the live roofline figure).
static thread_local KernelTimer g_timer[16];
KernelTimer& kernel_timer() {
  int dev = 0;
  cudaGetDevice(&dev);
  KernelTimer& t = g_timer[dev & 15];
  if (!t.init) {
    t.init = true;
    t.ok = cudaEventCreate(&t.start) == cudaSuccess && cudaEventCreate(&t.stop) == cudaSuccess;
  }
  return t;
}

// FP64-pipe probes over a full grid, 8 independent chains per thread:
// OP 0 = DFMA (the metric's "FMA peak"), OP 1 = alternating DADD / DMUL (the
// walk's instruction mix).  On B200 the second runs at the nominal 64/clk/SM,
// the first ~8% lower (three-operand reads), so the walk's roofline
// denominator is the larger of the two.
template <int OP>
__global__ void fp64_probe_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if constexpr (OP == 0) x[i] = fma(x[i], a, b);
        else x[i] = (i & 1) ? x[i] * a : x[i] + b;
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

int fp64_peak_probe(double seconds, int op, double* ops_per_s) {
  if (op != 0 && op != 1) {
    set_error("probe op must be 0 (DFMA) or 1 (DADD/DMUL)");
    return PERM_BAD_ARG;
  }
  int dev = 0, nsm = 148;
  PERM_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  PERM_CUDA_TRY(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = nsm * 4, threads = 512, iters = 2048;
  const double per_launch = (double)blocks * threads * iters * 16 * 8;
  auto kern = op == 0 ? fp64_probe_kernel<0> : fp64_probe_kernel<1>;
  const double a = op == 0 ? 0.999 : 0.999999, b = op == 0 ? 1e-3 : 1e-9;
  kern<<<blocks, threads>>>(d, iters, a, b);  // warm-up
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(d, iters, a, b);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int reps = (int)std::max(1.0, seconds / std::max(1e-6, ms * 1e-3));
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) kern<<<blocks, threads>>>(d, iters, a, b);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  *ops_per_s = per_launch * reps / (ms * 1e-3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PERM_OK : cuda_fail(e, "fp64 probe");
}

// ---------------------------------------------------------------- kernels
walk_fn walk_lookup_f64_w0(int P);
walk_fn walk_lookup_f64_w1(int P);
walk_fn walk_lookup_c128_w0(int P);
walk_fn walk_lookup_c128_w1(int P);

walk_fn walk_lookup(int dtype, bool weighted, int P) {
  if (dtype == 0) return weighted ? walk_lookup_f64_w1(P) : walk_lookup_f64_w0(P);
  return weighted ? walk_lookup_c128_w1(P) : walk_lookup_c128_w0(P);
}

static bool walk_inline_fits(const WalkSetup& ws) {
  if (ws.weighted ? (ws.B > 62 || ws.wlen > 63) : ws.B > ws.P) return false;
  const size_t bytes = (size_t)walk_inline_doubles(ws.P, ws.cplx ? 2 : 1, ws.weighted) * sizeof(double);
  return bytes <= kWalkInlineMaxBytes;
}

static int launch_setup(const WalkSetup& ws, uint64_t k_begin, uint64_t k_end, int mag, double* dst,
                        unsigned int* flag, unsigned int seq, bool allow_inline, cudaStream_t stream,
                        bool upload = true) {
  if (ws.P < 1 || ws.P > 64) {
    set_error("state length out of range (1..64)");
    return PERM_BAD_SHAPE;
  }
  Scratch* s = scratch();
  if (!s) {
    set_error("no CUDA device");
    return PERM_CUDA;
  }
  const size_t part_bytes = (size_t)kMaxPartials * kPartialStride * sizeof(double);
  const size_t data_bytes = ws.buf.size() * sizeof(double);
  int st = ensure_dev(s, part_bytes + data_bytes + 256);
  if (st) return st;
  double* partials = static_cast<double*>(s->dev);
  double* data = partials + (size_t)kMaxPartials * kPartialStride;
  const uint64_t steps = k_end - k_begin;
  const bool inl = allow_inline && (walk_tiled(k_begin, steps) || (steps > 0 && steps < 256)) && walk_inline_fits(ws);
  if (!inl && upload) {
    st = stage_h2d(s, data, ws.buf.data(), data_bytes, stream);
    if (st) return st;
  }
  walk_fn fn = walk_lookup(ws.cplx ? 1 : 0, ws.weighted, ws.P);
  if (!fn) {
    set_error("no walk kernel for this state length");
    return PERM_BAD_SHAPE;
  }
  WalkJob job;
  job.dtype = ws.cplx ? 1 : 0;
  job.P = ws.P;
  job.B = ws.B;
  job.weighted = ws.weighted;
  job.v0 = data + ws.v0_off;
  job.U = data + ws.U_off;
  job.w = ws.weighted ? data + ws.w_off : nullptr;
  job.wlen = ws.wlen;
  job.mag = mag;
  job.k_begin = k_begin;
  job.k_end = k_end;
  job.partials = partials;
  job.final_out = dst;
  job.done = s->done;
  job.inline_host = inl ? ws.buf.data() : nullptr;
  job.flag = flag;
  job.seq = seq;
  WalkPlan plan;
  KernelTimer& tm = kernel_timer();
  const bool timed = tm.ok && timing_enabled();
  if (timed) cudaEventRecord(tm.start, stream);
  PERM_CUDA_TRY(fn(job, &plan, stream));
  if (timed) cudaEventRecord(tm.stop, stream);
  tm.pending = timed;
  tm.last_grid = plan.grid;
  tm.last_log2L = plan.log2L;
  return PERM_OK;
}

int run_walk(const WalkSetup& ws, uint64_t k_begin, uint64_t k_end, int mag, double* dst, cudaStream_t stream) {
  return launch_setup(ws, k_begin, k_end, mag, dst, nullptr, 0, true, stream);
}

int run_walk_resident(const WalkSetup& ws, uint64_t k_begin, uint64_t k_end, int mag, double* dst,
                      cudaStream_t stream) {
  return launch_setup(ws, k_begin, k_end, mag, dst, nullptr, 0, true, stream, /*upload=*/false);
}

static int mapped_slot(Scratch* s) {
  if (s->mres_host) return PERM_OK;
  PERM_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&s->mres_host), 8 * sizeof(double) + 64, cudaHostAllocMapped));
  PERM_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->mres_dev), s->mres_host, 0));
  s->mflag_host = reinterpret_cast<unsigned int*>(s->mres_host + 8);
  s->mflag_dev = reinterpret_cast<unsigned int*>(s->mres_dev + 8);
  *reinterpret_cast<volatile unsigned int*>(s->mflag_host) = 0;
  return PERM_OK;
}

int run_walk_host(const WalkSetup& ws, uint64_t k_begin, uint64_t k_end, int mag, double* host8,
                  cudaStream_t stream, bool zero_copy) {
  Scratch* s = scratch();
  if (!s) return cuda_fail(cudaErrorNoDevice, "scratch");
  const uint64_t steps = k_end - k_begin;
  if (zero_copy && (walk_tiled(k_begin, steps) || (steps > 0 && steps < 256)) && walk_inline_fits(ws)) {
    int st = mapped_slot(s);
    if (st) return st;
    if (s->async_pending) {  // an earlier device-output call may still use the scratch
      PERM_CUDA_TRY(cudaDeviceSynchronize());
      s->async_pending = false;
    }
    const unsigned int seq = ++s->mseq;
    st = launch_setup(ws, k_begin, k_end, mag, s->mres_dev, s->mflag_dev, seq, true, stream);
    if (st) return st;
    // spin on the flag; after 2 ms fall back to a blocking wait (which also
    // surfaces launch / execution errors)
    volatile unsigned int* f = s->mflag_host;
    const auto t0 = std::chrono::steady_clock::now();
    while (*f != seq) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(2)) {
        PERM_CUDA_TRY(cudaStreamSynchronize(stream));
        if (*f != seq) {
          set_error("walk finished without publishing its result");
          return PERM_CUDA;
        }
        break;
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const volatile double* r = s->mres_host;
    for (int i = 0; i < 8; ++i) host8[i] = r[i];
    return PERM_OK;
  }
  const size_t part_bytes = (size_t)kMaxPartials * kPartialStride * sizeof(double);
  int st = ensure_dev(s, part_bytes + ws.buf.size() * sizeof(double) + 64 * sizeof(double) + 256);
  if (st) return st;
  double* dst = reinterpret_cast<double*>(static_cast<char*>(s->dev) + s->dev_cap) - 8;
  st = run_walk(ws, k_begin, k_end, mag, dst, stream);
  if (st) return st;
  PERM_CUDA_TRY(cudaMemcpyAsync(s->host, dst, 8 * sizeof(double), cudaMemcpyDeviceToHost, stream));
  PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  std::copy(s->host, s->host + 8, host8);
  return PERM_OK;
}

}  // namespace permb200
