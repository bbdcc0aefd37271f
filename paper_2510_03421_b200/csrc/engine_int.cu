// Exact integer path (north_star item 3): host planning for the CHECKED
// (reference int64 semantics) and WRAP (certified int128) Gray walks.
#include <algorithm>
#include <cmath>
#include <utility>

#include "engine.cuh"
#include "int_walk.cuh"

namespace permb200 {

typedef __int128 s128;
static const s128 kI64Max = (s128)INT64_MAX;
static const s128 kI64Min = (s128)INT64_MIN;

struct IntMat {
  int m = 0, n = 0;
  std::vector<int64_t> d;
  int64_t at(int i, int j) const { return d[(size_t)i * n + j]; }
};

static int load_int_matrix(int m, int n, const int64_t* a, int64_t lda, int dev_ptr, IntMat* out,
                           cudaStream_t stream) {
  if (m < 1 || n < 1) {
    set_error("matrix must have m >= 1 and n >= 1");
    return PERM_BAD_SHAPE;
  }
  if (m > n || n > 62) {
    set_error(m > n ? "need m <= n; transpose first" : "walk over more than 62 columns");
    return PERM_BAD_SHAPE;
  }
  out->m = m;
  out->n = n;
  out->d.assign((size_t)m * n, 0);
  if (dev_ptr) {
    PERM_CUDA_TRY(cudaMemcpy2DAsync(out->d.data(), (size_t)n * 8, a, (size_t)lda * 8, (size_t)n * 8, m,
                                    cudaMemcpyDeviceToHost, stream));
    PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  } else {
    for (int i = 0; i < m; ++i) std::copy(a + (size_t)i * lda, a + (size_t)i * lda + n, &out->d[(size_t)i * n]);
  }
  return PERM_OK;
}

// Walk description in int64 (v0, U, w) -- SURVEY Appendix A, no pre-scale.
struct IntSetup {
  int P = 0, B = 0;
  bool weighted = false;
  std::vector<int64_t> v0, U, w;
  // raw update rows (Glynn: row n-1-t; Ryser: column t) and the factor that
  // turns them into U (-2 for Glynn, +1 for Ryser): the 128-bit-state kernel
  // forms u * factor in 128 bits, where -2 * a_ij may not fit int64
  std::vector<int64_t> R;
  int64_t rscale = 1;
  std::vector<int64_t> v0w;  // exact initial state as (lo, hi) pairs

  bool pre_overflow = false;  // reference flags before/independently of the walk
  s128 bound = 0;             // max |state entry| along the walk
};

static void setup_int(int alg, const IntMat& A, IntSetup* s) {
  const int m = A.m, n = A.n;
  if (alg == PERM_ALG_GLYNN) {
    s->P = n;
    s->B = n - 1;
    s->v0.assign(n, 0);
    s->U.assign((size_t)(n - 1) * n, 0);
    // initial column sums, sequential checked adds from the pad
    // (src/_kernels.py:415-425, 583-594)
    for (int j = 0; j < n; ++j) {
      int64_t acc = n - m;
      s128 mag = n - m;
      for (int i = 0; i < m; ++i) {
        if (__builtin_add_overflow(acc, A.at(i, j), &acc)) s->pre_overflow = true;
        mag += (A.at(i, j) < 0) ? -(s128)A.at(i, j) : (s128)A.at(i, j);
      }
      s->v0[j] = acc;
      s->bound = std::max(s->bound, mag);
      s128 exact = n - m;
      for (int i = 0; i < m; ++i) exact += A.at(i, j);
      s->v0w.push_back((int64_t)(uint64_t)exact);
      s->v0w.push_back((int64_t)(uint64_t)((unsigned __int128)exact >> 64));
    }
    // rows 1..n-1 are flipped; a real row whose doubled entry leaves int64
    // is flagged by the reference (src/_kernels.py:461-464, 631-634)
    s->R.assign((size_t)(n - 1) * n, 0);
    s->rscale = -2;
    for (int t = 0; t < n - 1; ++t) {
      const int i = n - 1 - t;
      for (int j = 0; j < n; ++j) {
        int64_t y = (i < m) ? A.at(i, j) : 1, d2;
        s->R[(size_t)t * n + j] = y;
        if (__builtin_add_overflow(y, y, &d2)) {
          s->pre_overflow = true;
          d2 = 0;
        }
        s->U[(size_t)t * n + j] = -d2;
      }
    }
    return;
  }
  // Ryser: state = row sums; Gray bit t = column t
  s->P = m;
  s->B = n;
  s->v0.assign(m, 0);
  s->U.assign((size_t)n * m, 0);
  for (int t = 0; t < n; ++t)
    for (int i = 0; i < m; ++i) s->U[(size_t)t * m + i] = A.at(i, t);
  s->R = s->U;
  s->rscale = 1;
  s->v0w.assign(2 * (size_t)m, 0);
  for (int i = 0; i < m; ++i) {
    s128 mag = 0;
    for (int j = 0; j < n; ++j) mag += (A.at(i, j) < 0) ? -(s128)A.at(i, j) : (s128)A.at(i, j);
    s->bound = std::max(s->bound, mag);
  }
  if (m < n) {
    s->weighted = true;
    s->w.assign(n + 1, 0);
    for (int k = 1; k <= m; ++k) {
      unsigned __int128 c = 1;
      for (int i = 1; i <= m - k; ++i) c = c * (unsigned __int128)(n - k - (m - k) + i) / i;
      s->w[k] = ((m - k) & 1) ? -(int64_t)c : (int64_t)c;
    }
  }
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// ------------------------------------------------------------ CHECKED walk
// Returns PERM_OK with *ovf and *value (the raw walk sum when !ovf).
static int checked_walk(const IntSetup& s, cudaStream_t stream, bool* ovf, int64_t* value) {
  *ovf = s.pre_overflow;
  *value = 0;
  if (*ovf) return PERM_OK;
  const uint64_t steps = 1ull << s.B;
  int log2L = 0;
  while ((steps >> log2L) > (1ull << 17)) ++log2L;
  const uint64_t nchunks = steps >> log2L;
  const uint64_t blocks = (nchunks + kIntThreads - 1) / kIntThreads;
  const size_t nv0 = s.v0.size(), nU = s.U.size();
  const size_t bytes = (nv0 + nU) * 8 + blocks * 64;
  DevBuf buf;
  PERM_CUDA_TRY(cudaMallocAsync(&buf.p, bytes, stream));
  int64_t* d = static_cast<int64_t*>(buf.p);
  PERM_CUDA_TRY(cudaMemcpyAsync(d, s.v0.data(), nv0 * 8, cudaMemcpyHostToDevice, stream));
  if (nU) PERM_CUDA_TRY(cudaMemcpyAsync(d + nv0, s.U.data(), nU * 8, cudaMemcpyHostToDevice, stream));
  IntWalkArgs a;
  a.v0 = d;
  a.U = d + nv0;
  a.w = nullptr;
  a.P = s.P;
  a.B = s.B;
  a.log2L = log2L;
  a.wlen = 0;
  a.k_begin = 0;
  a.nchunks = nchunks;
  a.out = d + nv0 + nU;
  int_walk_checked_kernel<<<(unsigned)blocks, kIntThreads, 0, stream>>>(a);
  PERM_CUDA_TRY(cudaGetLastError());
  std::vector<int64_t> h(blocks * 8);
  PERM_CUDA_TRY(cudaMemcpyAsync(h.data(), a.out, blocks * 64, cudaMemcpyDeviceToHost, stream));
  PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  PERM_CUDA_TRY(cudaFreeAsync(buf.p, stream));
  buf.p = nullptr;
  // ordered combine of block summaries (Gray order = block order)
  s128 G = 0;
  bool flag = false;
  for (uint64_t b = 0; b < blocks; ++b) {
    const int64_t* o = &h[b * 8];
    auto get = [&](int q) { return (s128)(((unsigned __int128)(uint64_t)o[q + 1] << 64) | (uint64_t)o[q]); };
    if (o[6]) flag = true;
    s128 S = get(0), mn = get(2), mx = get(4);
    if (G + mn < kI64Min || G + mx > kI64Max) flag = true;
    G += S;
  }
  *ovf = flag;
  *value = flag ? 0 : (int64_t)G;
  return PERM_OK;
}

// ------------------------------------------------------------ WRAP walk
walk_fn_i int_wrap_lookup(int P);
walk_fn_if int_wrap_fp_lookup(int P);

// Fused path: FP64-exact state and group products (|state| <= 83), the
// int128 sum and its FP64 estimate / magnitude sum from one kernel.
static bool fp_walk_ok(const IntSetup& s) {
  return !s.weighted && s.bound <= 83 && s.B >= 8 && s.P >= 1 && s.P <= 64;
}

static int wrap_walk_fp(const IntSetup& s, cudaStream_t stream, s128* raw, long double* est, long double* mag) {
  const uint64_t steps = 1ull << s.B;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t lanes = (uint64_t)nsm * 8 * kIntThreads;
  int log2L = 3;
  while (log2L < 14 && (steps >> (log2L + 1)) >= 16 * lanes) ++log2L;
  const uint64_t nchunks = steps >> log2L;
  const uint64_t blocks = std::min<uint64_t>((nchunks + kIntThreads - 1) / kIntThreads, (uint64_t)nsm * 8);
  std::vector<double> buf(s.v0.size() + s.U.size());
  for (size_t i = 0; i < s.v0.size(); ++i) buf[i] = (double)s.v0[i];
  for (size_t i = 0; i < s.U.size(); ++i) buf[s.v0.size() + i] = (double)s.U[i];
  const size_t bytes = buf.size() * 8 + blocks * 64 + 256;
  DevBuf dbuf;
  PERM_CUDA_TRY(cudaMallocAsync(&dbuf.p, bytes, stream));
  double* d = static_cast<double*>(dbuf.p);
  PERM_CUDA_TRY(cudaMemcpyAsync(d, buf.data(), buf.size() * 8, cudaMemcpyHostToDevice, stream));
  IntWalkFArgs a;
  a.v0 = d;
  a.U = d + s.v0.size();
  a.P = s.P;
  a.B = s.B;
  a.log2L = log2L;
  a.k_begin = 0;
  a.nchunks = nchunks;
  a.out = reinterpret_cast<int64_t*>(d + buf.size());
  walk_fn_if fn = int_wrap_fp_lookup(s.P);
  if (!fn) {
    set_error("no fp int walk for this size");
    return PERM_BAD_SHAPE;
  }
  PERM_CUDA_TRY(fn(a, (int)blocks, stream));
  std::vector<int64_t> h(blocks * 8);
  PERM_CUDA_TRY(cudaMemcpyAsync(h.data(), a.out, blocks * 64, cudaMemcpyDeviceToHost, stream));
  PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  PERM_CUDA_TRY(cudaFreeAsync(dbuf.p, stream));
  dbuf.p = nullptr;
  unsigned __int128 acc = 0;
  double H = 0, L = 0, M = 0;
  for (uint64_t b = 0; b < blocks; ++b) {
    const int64_t* o = &h[b * 8];
    acc += ((unsigned __int128)(uint64_t)o[1] << 64) | (uint64_t)o[0];
    double hh, ll, mm;
    std::memcpy(&hh, &o[2], 8);
    std::memcpy(&ll, &o[3], 8);
    std::memcpy(&mm, &o[4], 8);
    dd_add(H, L, hh, ll);
    M += mm;
  }
  *raw = (s128)acc;
  *est = (long double)H + (long double)L;
  *mag = M;
  return PERM_OK;
}

static int wrap_walk(const IntSetup& s, cudaStream_t stream, s128* raw) {
  const bool wide = s.bound >= ((s128)1 << 62);  // int64 state could wrap
  const uint64_t steps = 1ull << s.B;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // exact int64 groups of 8 factors need bound^8 < 2^63
  const bool g8 = !wide && !s.weighted && (long double)s.bound < std::pow(2.0L, 63.0L / 8.0L) && steps >= 8;
  const uint64_t lanes = (uint64_t)nsm * 8 * kIntThreads;
  int log2L = 3;
  while (log2L < 14 && (steps >> (log2L + 1)) >= 16 * lanes) ++log2L;
  while (log2L > 0 && (steps >> log2L) < 1) --log2L;
  if (!g8 && log2L > 10) log2L = 10;
  if (steps < 8) log2L = 0;
  const uint64_t nchunks = steps >> log2L;
  uint64_t blocks = std::min<uint64_t>((nchunks + kIntThreads - 1) / kIntThreads, (uint64_t)nsm * 8);
  const size_t nv0 = wide ? s.v0w.size() : s.v0.size(), nU = s.U.size(), nw = s.w.size();
  const size_t bytes = (nv0 + nU + nw) * 8 + blocks * 16;
  DevBuf buf;
  PERM_CUDA_TRY(cudaMallocAsync(&buf.p, bytes, stream));
  int64_t* d = static_cast<int64_t*>(buf.p);
  PERM_CUDA_TRY(cudaMemcpyAsync(d, (wide ? s.v0w : s.v0).data(), nv0 * 8, cudaMemcpyHostToDevice, stream));
  if (nU) PERM_CUDA_TRY(cudaMemcpyAsync(d + nv0, (wide ? s.R : s.U).data(), nU * 8, cudaMemcpyHostToDevice, stream));
  if (nw) PERM_CUDA_TRY(cudaMemcpyAsync(d + nv0 + nU, s.w.data(), nw * 8, cudaMemcpyHostToDevice, stream));
  IntWalkArgs a;
  a.v0 = d;
  a.U = d + nv0;
  a.w = nw ? d + nv0 + nU : nullptr;
  a.P = s.P;
  a.B = s.B;
  a.log2L = log2L;
  a.wlen = (int)nw;
  a.k_begin = 0;
  a.nchunks = nchunks;
  a.out = d + nv0 + nU + nw;
  walk_fn_i fast = (g8 && log2L >= 3) ? int_wrap_lookup(s.P) : nullptr;
  if (fast) {
    PERM_CUDA_TRY(fast(a, (int)blocks, stream));
  } else {
    if (wide)
      int_walk_wrap_wide_kernel<<<(unsigned)blocks, kIntThreads, 0, stream>>>(a, s.weighted ? 1 : 0, s.rscale);
    else
      int_walk_wrap_generic_kernel<<<(unsigned)blocks, kIntThreads, 0, stream>>>(a, s.weighted ? 1 : 0);
    PERM_CUDA_TRY(cudaGetLastError());
  }
  std::vector<int64_t> h(blocks * 2);
  PERM_CUDA_TRY(cudaMemcpyAsync(h.data(), a.out, blocks * 16, cudaMemcpyDeviceToHost, stream));
  PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  PERM_CUDA_TRY(cudaFreeAsync(buf.p, stream));
  buf.p = nullptr;
  unsigned __int128 acc = 0;
  for (uint64_t b = 0; b < blocks; ++b)
    acc += ((unsigned __int128)(uint64_t)h[2 * b + 1] << 64) | (uint64_t)h[2 * b];
  *raw = (s128)acc;
  return PERM_OK;
}

// Float estimate for the int128 fit certificate: same algorithm in FP64
// with the magnitude sum M; |per - per_fp| <= (P + 2^14 + 16) * 2^-52 * M
// (exact integer state entries; <= P-1 product roundings; chunk sums of at
// most 2^14 terms; double-double above that).
static int float_estimate(int alg, const IntMat& A, cudaStream_t stream, double* per, double* mag) {
  HostMat H;
  H.m = A.m;
  H.n = A.n;
  H.cplx = false;
  H.d.resize(A.d.size());
  for (size_t i = 0; i < A.d.size(); ++i) H.d[i] = (double)A.d[i];
  WalkSetup ws;
  int st = build_walk(alg, H, &ws);
  if (st) return st;
  Scratch* sc = scratch();
  if (!sc) return cuda_fail(cudaErrorNoDevice, "scratch");
  const size_t part_bytes = (size_t)kMaxPartials * kPartialStride * sizeof(double);
  st = ensure_dev(sc, part_bytes + ws.buf.size() * sizeof(double) + 64 * sizeof(double) + 256);
  if (st) return st;
  double* dst = reinterpret_cast<double*>(static_cast<char*>(sc->dev) + sc->dev_cap) - 8;
  st = run_walk(ws, 0, walk_steps(alg, A.m, A.n), 1, dst, stream);
  if (st) return st;
  PERM_CUDA_TRY(cudaMemcpyAsync(sc->host, dst, 8 * sizeof(double), cudaMemcpyDeviceToHost, stream));
  PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  double re = sc->host[0] + sc->host[1], im = 0.0, mg = sc->host[4];
  normalize(alg, A.m, A.n, ws.scale_log2, &re, &im, &mg);
  *per = re;
  *mag = mg;
  return PERM_OK;
}

static bool fits_bound(double per_fp, double mag, int P, long double denom) {
  const long double E = (long double)(P + (1 << 14) + 16) * std::ldexp(1.0L, -52) * (long double)mag;
  const long double hi = ((long double)std::fabs(per_fp) + E) * denom;
  return hi < std::ldexp(1.0L, 126);  // one bit of margin below 2^127
}

static int to_out(s128 v, int64_t* out, int* fits_int64) {
  out[0] = (int64_t)(uint64_t)v;
  out[1] = (int64_t)(uint64_t)((unsigned __int128)v >> 64);
  if (fits_int64) *fits_int64 = (v >= kI64Min && v <= kI64Max) ? 1 : 0;
  return PERM_OK;
}

int int_permanent(int alg, int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, int64_t* out,
                  int* fits_int64, void* stream_) {
  clear_error();
  cudaStream_t stream = pick_stream(stream_);
  IntMat A;
  int st = load_int_matrix(m, n, a, lda, dev_ptr, &A, stream);
  if (st) return st;
  IntSetup s;
  setup_int(alg, A, &s);
  s128 denom = 1;
  if (alg == PERM_ALG_GLYNN) {
    denom = (s128)1 << (n - 1);
    for (int i = 2; i <= n - m; ++i) denom *= i;
  }
  if (width == 64) {
    // reference semantics: PERM_OVERFLOW whenever the reference flags
    bool ovf = false;
    int64_t raw = 0;
    st = checked_walk(s, stream, &ovf, &raw);
    if (st) return st;
    if (ovf) {
      set_error("an int64 intermediate overflowed (reference semantics)");
      return PERM_OVERFLOW;
    }
    s128 v = raw;
    if (alg == PERM_ALG_GLYNN) {
      if (v % denom != 0) {  // src/algorithms.py:436-437, 459-460
        set_error("Glynn sum not divisible by its normalization");
        return PERM_OVERFLOW;
      }
      v /= denom;
    } else if (m == n && (n & 1)) {
      v = (s128)(int64_t)(0 - (uint64_t)(int64_t)v);  // int64 negation as in src/_kernels.py:216-217
    }
    return to_out(v, out, fits_int64);
  }
  if (width != 128) {
    set_error("width must be 64 or 128");
    return PERM_BAD_ARG;
  }
  // Fit certificate for |walk sum| < 2^127: (a) a priori, or (b) an FP64 run
  // with its magnitude-sum error bound (state entries must then be exactly
  // representable, i.e. magnitudes < 2^52).
  // (a): |walk sum| = |per| * denom <= per(|A|) * denom, and per(|A|) is at most
  // the product of the row sums of |A| (and, square, of the column sums)
  long double rows = 1.0L, cols = 1.0L;
  for (int i = 0; i < m; ++i) {
    long double r = 0;
    for (int j = 0; j < n; ++j) r += std::fabs((long double)A.at(i, j));
    rows *= r;
  }
  for (int j = 0; j < n; ++j) {
    long double c = 0;
    for (int i = 0; i < m; ++i) c += std::fabs((long double)A.at(i, j));
    cols *= c;
  }
  const long double apriori = (m == n ? std::min(rows, cols) : rows) * (long double)denom;
  const bool cert_apriori = apriori < std::ldexp(1.0L, 126);
  if (fp_walk_ok(s)) {
    // one pass: exact int128 walk + its own FP64 estimate.  Error of the
    // estimate of the raw sum: <= 3 product roundings per term (group
    // products are exact) and chunk sums of <= 2^14 terms, i.e.
    // E <= (3 + 2^14 + 16) u M_raw.
    s128 raw = 0;
    long double est = 0, mag_raw = 0;
    st = wrap_walk_fp(s, stream, &raw, &est, &mag_raw);
    if (st) return st;
    const long double E = (long double)(3 + (1 << 14) + 16) * std::ldexp(1.0L, -52) * mag_raw;
    if (!cert_apriori && std::fabs(est) + E >= std::ldexp(1.0L, 126)) {
      set_error("exact value not certified to fit the int128 walk");
      return PERM_OVERFLOW;
    }
    if (std::fabs((long double)raw - est) > E + 1.0L) {
      set_error("internal: int128 walk disagrees with its FP64 estimate");
      return PERM_CUDA;
    }
    s128 v = raw;
    if (alg == PERM_ALG_GLYNN) {
      if (v % denom != 0) {
        set_error("internal: Glynn int128 sum not divisible by its normalization");
        return PERM_CUDA;
      }
      v /= denom;
    } else if (m == n && (n & 1)) {
      v = -v;
    }
    return to_out(v, out, fits_int64);
  }
  double per_fp = 0, mag = 0;
  if (!cert_apriori) {
    if (s.bound >= ((s128)1 << 52)) {
      set_error("exact value not certified to fit int128 (entries too large for the FP64 certificate)");
      return PERM_OVERFLOW;
    }
    st = float_estimate(alg, A, stream, &per_fp, &mag);
    if (st) return st;
    if (!fits_bound(per_fp, mag, s.P, (long double)denom)) {
      set_error("exact value not certified to fit the int128 walk");
      return PERM_OVERFLOW;
    }
  }
  s128 raw = 0;
  st = wrap_walk(s, stream, &raw);
  if (st) return st;
  s128 v = raw;
  if (alg == PERM_ALG_GLYNN) {
    if (v % denom != 0) {
      set_error("internal: Glynn int128 sum not divisible by its normalization");
      return PERM_CUDA;
    }
    v /= denom;
  } else if (m == n && (n & 1)) {
    v = -v;
  }
  // consistency with the FP64 estimate (catches a corrupted exact sum)
  const long double E = (long double)(s.P + (1 << 14) + 16) * std::ldexp(1.0L, -52) * (long double)mag;
  if (!cert_apriori && std::fabs((long double)v - (long double)per_fp) > E + 1.0L) {
    set_error("internal: int128 result disagrees with the FP64 estimate");
    return PERM_CUDA;
  }
  return to_out(v, out, fits_int64);
}

}  // namespace permb200
