// Host side of the combination-ordered Ryser and the combinatoric DFS.
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "comb.cuh"
#include "engine.cuh"

namespace permb200 {

typedef __int128 s128;

static uint64_t nperm(int n, int k) {  // P(n, k), saturating
  unsigned __int128 r = 1;
  for (int i = 0; i < k; ++i) {
    r *= (unsigned)(n - i);
    if (r > (unsigned __int128)UINT64_MAX) return UINT64_MAX;
  }
  return (uint64_t)r;
}

static const std::vector<uint64_t>& binom_table() {
  static const std::vector<uint64_t> table = [] {  // thread-safe one-time init
    std::vector<uint64_t> t;
    const int R = kCombMaxN + 1, W = kBinomCols;
    t.assign((size_t)R * W, 0);
    for (int i = 0; i < R; ++i) {
      t[(size_t)i * W] = 1;
      for (int j = 1; j <= i && j < W; ++j) {  // saturating Pascal rule
        const uint64_t x = t[(size_t)(i - 1) * W + j - 1], y = (j <= i - 1) ? t[(size_t)(i - 1) * W + j] : 0;
        t[(size_t)i * W + j] = (x > UINT64_MAX - y) ? UINT64_MAX : x + y;
      }
    }
    return t;
  }();
  return table;
}

static int device_binom_table(const uint64_t** out) {
  static uint64_t* tabs[16] = {nullptr};
  int dev = 0;
  PERM_CUDA_TRY(cudaGetDevice(&dev));
  if (!tabs[dev & 15]) {
    const auto& bt = binom_table();
    uint64_t* d = nullptr;
    PERM_CUDA_TRY(cudaMalloc(&d, bt.size() * 8));
    PERM_CUDA_TRY(cudaMemcpy(d, bt.data(), bt.size() * 8, cudaMemcpyHostToDevice));
    tabs[dev & 15] = d;
  }
  *out = tabs[dev & 15];
  return PERM_OK;
}

static int target_threads() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm * 4 * kCombThreads;
}

// Enqueue one ryser_comb / comb_dfs kernel writing its per-block partials
// (8 slots each) at dOut; returns the number of blocks.
template <int MODE>
static int enqueue_comb(bool ryser, const void* dA, const uint64_t* dB, int m, int n, int s, int depth,
                        uint64_t total, void* dOut, uint64_t* nblocks, cudaStream_t stream) {
  const uint64_t thr = (uint64_t)target_threads();
  uint64_t per = (total + thr - 1) / thr;
  if (per < 1) per = 1;
  const uint64_t nthreads = (total + per - 1) / per;
  const uint64_t blocks = (nthreads + kCombThreads - 1) / kCombThreads;
  CombArgs a;
  a.a = dA;
  a.binom = dB;
  a.m = m;
  a.n = n;
  a.s = s;
  a.total = total;
  a.per_thread = per;
  a.depth = depth;
  a.out = dOut;
  a.fused = 0;
  a.smem_binom = 0;
  a.smem_matrix = 0;
  if (ryser) ryser_comb_kernel<MODE><<<(unsigned)blocks, kCombThreads, 0, stream>>>(a);
  else comb_dfs_kernel<MODE><<<(unsigned)blocks, kCombThreads, 0, stream>>>(a);
  PERM_CUDA_TRY(cudaGetLastError());
  *nblocks = blocks;
  return PERM_OK;
}

// All subset sizes s = m..1 of the combination-order Ryser in ONE launch
// (blocks of size s at first[s] .. first[s] + cnt[s]); binomials and, when
// small, the matrix are staged in shared memory.
template <int MODE>
static int enqueue_ryser_fused(const void* dA, const uint64_t* dB, int m, int n, size_t esz,
                               const std::vector<uint64_t>& bt, void* dOut, std::vector<uint64_t>* first,
                               std::vector<uint64_t>* cnt, uint64_t* nblocks, cudaStream_t stream) {
  const uint64_t thr = (uint64_t)target_threads();
  CombArgs a;
  a.a = dA;
  a.binom = dB;
  a.m = m;
  a.n = n;
  a.s = 0;
  a.total = 0;
  a.per_thread = 1;
  a.depth = 0;
  a.out = dOut;
  a.fused = 1;
  uint64_t off = 0;
  for (int s = m; s >= 1; --s) {
    const uint64_t total = bt[(size_t)n * kBinomCols + s];
    uint64_t per = (total + thr - 1) / thr;
    if (per < 1) per = 1;
    const uint64_t blocks = ((total + per - 1) / per + kCombThreads - 1) / kCombThreads;
    a.blk_first[s] = off;
    a.blk_count[s] = blocks;
    a.tot[s] = total;
    a.per[s] = per;
    (*first)[s] = off;
    (*cnt)[s] = blocks;
    off += blocks;
  }
  const size_t mat = (((size_t)m * n * esz) + 15) & ~(size_t)15, bin = (size_t)m * n * 8;
  a.smem_matrix = (mat + bin <= 40 * 1024) ? 1 : 0;
  a.smem_binom = (bin <= 40 * 1024) ? 1 : 0;
  const size_t smem = (a.smem_matrix ? mat : 0) + (a.smem_binom ? bin : 0);
  ryser_comb_kernel<MODE><<<(unsigned)off, kCombThreads, smem, stream>>>(a);
  PERM_CUDA_TRY(cudaGetLastError());
  *nblocks = off;
  return PERM_OK;
}

// One D2H of `count` 8-slot partials, then a single synchronization.
static int fetch_partials(const void* dOut, uint64_t count, std::vector<int64_t>* host, cudaStream_t stream) {
  host->resize(count * 8);
  Scratch* sc = scratch();
  if (count * 8 <= kHostResultDoubles) {
    PERM_CUDA_TRY(cudaMemcpyAsync(sc->host, dOut, count * 64, cudaMemcpyDeviceToHost, stream));
    PERM_CUDA_TRY(cudaStreamSynchronize(stream));
    std::memcpy(host->data(), sc->host, count * 64);
  } else {
    PERM_CUDA_TRY(cudaMemcpyAsync(host->data(), dOut, count * 64, cudaMemcpyDeviceToHost, stream));
    PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  }
  return PERM_OK;
}

// Ordered combine of checked summaries; false on overflow.
static bool combine_checked(const std::vector<int64_t>& h, s128* total) {
  s128 G = 0;
  const s128 lo = (s128)INT64_MIN, hi = (s128)INT64_MAX;
  for (size_t b = 0; b * 8 < h.size(); ++b) {
    const int64_t* o = &h[b * 8];
    auto get = [&](int q) { return (s128)(((unsigned __int128)(uint64_t)o[q + 1] << 64) | (uint64_t)o[q]); };
    if (o[6]) return false;
    if (G + get(2) < lo || G + get(4) > hi) return false;
    G += get(0);
  }
  *total = G;
  return true;
}

static void combine_float(const std::vector<int64_t>& h, double* re_h, double* re_l, double* im_h, double* im_l) {
  for (size_t b = 0; b * 8 < h.size(); ++b) {
    const double* o = reinterpret_cast<const double*>(&h[b * 8]);
    dd_add(*re_h, *re_l, o[0], o[1]);
    dd_add(*im_h, *im_l, o[2], o[3]);
  }
}

// mode 0 f64, 1 c128, 2 int64 checked, 3 exact int128 (combinatoric only).
// Float: out[0..1] = re, im.  Mode 2: *ivalue, PERM_OVERFLOW on reference
// overflow.  Mode 3: ivalue[0..1] = lo, hi; PERM_OVERFLOW when the a-priori
// bound (product of the row sums of |A|) does not certify int128.
int tiny_permanent(int alg, bool cplx, int m, int n, const double* a, double* out);  // engine_batch.cu

int comb_permanent(bool ryser, int mode, int m, int n, const void* a, int64_t lda, int dev_ptr,
                   uint64_t step_budget, double* out, int64_t* ivalue, void* stream_) {
  clear_error();
  if (m < 1 || n < 1) {
    set_error("matrix must have m >= 1 and n >= 1");
    return PERM_BAD_SHAPE;
  }
  if (m > n || n > kCombMaxN || m > 62) {
    set_error(m > n ? "need m <= n; transpose first"
                    : (m > 62 ? "more than 62 rows" : "more than kCombMaxN = 256 columns"));
    return PERM_BAD_SHAPE;
  }
  if (ryser) {  // sum_{s<=m} C(n, s) combinations, counted in uint64 ranks
    const auto& bt0 = binom_table();
    unsigned __int128 tot = 0;
    for (int s = 1; s <= m; ++s) tot += bt0[(size_t)n * kBinomCols + s];
    if (tot > ((unsigned __int128)1 << 62)) {
      set_error("combination-order Ryser over more than 2^62 column subsets");
      return PERM_BUDGET;
    }
  }
  if (!ryser) {  // src/algorithms.py:78-84
    const uint64_t perms = nperm(n, m);
    if (perms > step_budget) {
      set_error("combinatoric step budget exceeded");
      return PERM_BUDGET;
    }
  }
  if (mode == 3 && ryser) {
    set_error("exact int128 combination-order Ryser is not provided; use the int128 walk");
    return PERM_BAD_ARG;
  }
  // tiny float combinatoric from host memory: the zero-copy batch-of-one path
  // (memoized-DP kernel, m <= 4; the generic thread-per-matrix DFS is slower
  // than the tree-split comb kernel below from 5x5 on)
  static const int tiny_max_m = [] {  // PERM_TINY_COMB_MAX_M (measurement knob)
    const char* e = std::getenv("PERM_TINY_COMB_MAX_M");
    return (e && *e) ? std::atoi(e) : 4;
  }();
  if (!ryser && mode <= 1 && !dev_ptr && lda == n && stream_ == nullptr && m <= tiny_max_m && n <= 12) {
    const int tst = tiny_permanent(PERM_ALG_COMBINATORIC, mode == 1, m, n, static_cast<const double*>(a), out);
    if (tst >= 0) return tst;
  }
  cudaStream_t stream = pick_stream(stream_);
  const int esz = (mode == 1) ? 16 : 8;
  std::vector<unsigned char> hA((size_t)m * n * esz);
  if (dev_ptr) {
    PERM_CUDA_TRY(cudaMemcpy2DAsync(hA.data(), (size_t)n * esz, a, (size_t)lda * esz, (size_t)n * esz, m,
                                    cudaMemcpyDeviceToHost, stream));
    PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  } else {
    for (int i = 0; i < m; ++i)
      std::memcpy(&hA[(size_t)i * n * esz], static_cast<const unsigned char*>(a) + (size_t)i * lda * esz,
                  (size_t)n * esz);
  }
  const auto& bt = binom_table();
  // device buffers: matrix, binomials, partials
  const uint64_t thr = (uint64_t)target_threads();
  const size_t max_blocks = ((thr + kCombThreads - 1) / kCombThreads + 1) * (size_t)(ryser ? m : 1);
  const size_t bytes = hA.size() + bt.size() * 8 + max_blocks * 64 + 256;
  // engine-owned scratch (no per-call allocation): [matrix][block partials];
  // the binomial table lives on the device once per device
  Scratch* sc = scratch();
  if (!sc) return cuda_fail(cudaErrorNoDevice, "scratch");
  int st0 = ensure_dev(sc, bytes);
  if (st0) return st0;
  const uint64_t* dB = nullptr;
  st0 = device_binom_table(&dB);
  if (st0) return st0;
  unsigned char* base = static_cast<unsigned char*>(sc->dev);
  void* dA = base;
  void* dOut = base + ((hA.size() + 255) & ~(size_t)255);
  st0 = stage_h2d(sc, dA, hA.data(), hA.size(), stream);
  if (st0) return st0;
  std::vector<int64_t> h;
  int st = PERM_OK;
  if (ryser) {
    // src/_kernels.py:226-262 / 265-365: s = m..1, total += w[s] * size_sum
    double th = 0, tl = 0, ih = 0, il = 0;
    int64_t itotal = 0;
    bool ovf = false;
    // all subset sizes enqueued back to back, one read-back
    std::vector<uint64_t> first(m + 2, 0), cnt(m + 2, 0);
    uint64_t off = 0;
    st = (mode == 2) ? enqueue_ryser_fused<kCombI64>(dA, dB, m, n, esz, bt, dOut, &first, &cnt, &off, stream)
         : (mode == 0) ? enqueue_ryser_fused<kCombF64>(dA, dB, m, n, esz, bt, dOut, &first, &cnt, &off, stream)
                       : enqueue_ryser_fused<kCombC128>(dA, dB, m, n, esz, bt, dOut, &first, &cnt, &off, stream);
    if (st) return st;
    std::vector<int64_t> all;
    st = fetch_partials(dOut, off, &all, stream);
    if (st) return st;
    for (int s = m; s >= 1 && !ovf; --s) {
      int64_t c = (int64_t)bt[(size_t)(n - s) * kBinomCols + (m - s)];  // <= C(n, m) < 2^62 (checked above)
      const int64_t w = ((m - s) & 1) ? -c : c;
      h.assign(all.begin() + first[s] * 8, all.begin() + (first[s] + cnt[s]) * 8);
      if (mode == 2) {
        s128 size_sum;
        if (!combine_checked(h, &size_sum)) { ovf = true; break; }
        int64_t ss = (int64_t)size_sum, p;
        if (__builtin_mul_overflow(w, ss, &p) || __builtin_add_overflow(itotal, p, &itotal)) ovf = true;
      } else {
        double rh = 0, rl = 0, jh = 0, jl = 0;
        combine_float(h, &rh, &rl, &jh, &jl);
        const double wd = (double)w;
        // w * size_sum in double-double (w exact up to 2^53)
        dd_add(th, tl, wd * rh, std::fma(wd, rh, -(wd * rh)) + wd * rl);
        dd_add(ih, il, wd * jh, std::fma(wd, jh, -(wd * jh)) + wd * jl);
      }
    }
    if (mode == 2) {
      if (ovf) {
        set_error("an int64 intermediate overflowed (reference semantics)");
        return PERM_OVERFLOW;
      }
      *ivalue = itotal;
    } else {
      out[0] = th + tl;
      if (mode == 1) out[1] = ih + il;
    }
  } else {
    // prefix depth: enough prefixes to fill the device, at most m
    int D = 0;
    while (D < m && nperm(n, D) < thr * 4) ++D;
    if (D < 1) D = 1;
    const uint64_t total = nperm(n, D);
    if (mode == 3) {
      // every prefix product and partial sum is bounded by prod_i max(1, sum_j |a_ij|)
      long double bound = 1.0L;
      for (int i = 0; i < m; ++i) {
        long double r = 0;
        for (int j = 0; j < n; ++j) {
          int64_t x;
          std::memcpy(&x, &hA[((size_t)i * n + j) * 8], 8);
          r += std::fabs((long double)x);
        }
        bound *= std::max(1.0L, r);
      }
      if (!(bound < std::ldexp(1.0L, 126))) {
        set_error("exact value not certified to fit int128 (product of the row sums of |A| >= 2^126)");
        return PERM_OVERFLOW;
      }
      uint64_t nb = 0;
      st = enqueue_comb<kCombI128>(false, dA, dB, m, n, 0, D, total, dOut, &nb, stream);
      if (st) return st;
      st = fetch_partials(dOut, nb, &h, stream);
      if (st) return st;
      unsigned __int128 acc = 0;
      for (uint64_t b = 0; b < nb; ++b)
        acc += ((unsigned __int128)(uint64_t)h[b * 8 + 1] << 64) | (uint64_t)h[b * 8];
      ivalue[0] = (int64_t)(uint64_t)acc;
      ivalue[1] = (int64_t)(uint64_t)(acc >> 64);
    } else if (mode == 2) {
      uint64_t nb = 0;
      st = enqueue_comb<kCombI64>(false, dA, dB, m, n, 0, D, total, dOut, &nb, stream);
      if (st) return st;
      st = fetch_partials(dOut, nb, &h, stream);
      if (st) return st;
      s128 t;
      if (!combine_checked(h, &t)) {
        set_error("an int64 intermediate overflowed (reference semantics)");
        return PERM_OVERFLOW;
      }
      *ivalue = (int64_t)t;
    } else {
      uint64_t nb = 0;
      st = (mode == 0) ? enqueue_comb<kCombF64>(false, dA, dB, m, n, 0, D, total, dOut, &nb, stream)
                       : enqueue_comb<kCombC128>(false, dA, dB, m, n, 0, D, total, dOut, &nb, stream);
      if (st) return st;
      st = fetch_partials(dOut, nb, &h, stream);
      if (st) return st;
      double rh = 0, rl = 0, jh = 0, jl = 0;
      combine_float(h, &rh, &rl, &jh, &jl);
      out[0] = rh + rl;
      if (mode == 1) out[1] = jh + jl;
    }
  }
  PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  return PERM_OK;
}

}  // namespace permb200
