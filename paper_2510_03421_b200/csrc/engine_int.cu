// Exact integer path (north_star item 3): host planning for the CHECKED
// (reference int64 semantics) and WRAP (certified int128) Gray walks.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "engine.cuh"
#include "int_walk.cuh"
#include "int_walk32.cuh"

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
  std::vector<s128> cb;       // per state entry: bound on |entry| along the walk
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
      s->cb.push_back(mag);
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
    s->cb.push_back(mag);
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


// One range's inputs go to the thread's device scratch in one pinned-staged
// copy, and its block outputs come back through the pinned result buffer:
// per-call cudaMallocAsync / pageable copies cost ~10-15 us of a 40 us
// small-matrix call (round 2).  Sequential within a call (each range
// synchronizes before the next uses the scratch).
static int int_stage(const void* host, size_t in_bytes, size_t out_bytes, cudaStream_t stream, char** d,
                     size_t* out_off) {
  Scratch* sc = scratch();
  if (!sc) return cuda_fail(cudaErrorNoDevice, "scratch");
  *out_off = (in_bytes + 255) & ~(size_t)255;
  int st = ensure_dev(sc, *out_off + out_bytes + 256);
  if (st) return st;
  *d = static_cast<char*>(sc->dev);
  return in_bytes ? stage_h2d(sc, *d, host, in_bytes, stream) : PERM_OK;
}
static int int_fetch(const void* dout, size_t bytes, cudaStream_t stream, void* host) {
  Scratch* sc = scratch();
  if (!sc) return cuda_fail(cudaErrorNoDevice, "scratch");
  if (bytes <= kHostResultDoubles * sizeof(double)) {
    PERM_CUDA_TRY(cudaMemcpyAsync(sc->host, dout, bytes, cudaMemcpyDeviceToHost, stream));
    PERM_CUDA_TRY(cudaStreamSynchronize(stream));
    std::memcpy(host, sc->host, bytes);
  } else {
    PERM_CUDA_TRY(cudaMemcpyAsync(host, dout, bytes, cudaMemcpyDeviceToHost, stream));
    PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  }
  return PERM_OK;
}

// ------------------------------------------------------------ Gray ranges
// Every integer walk below runs over one Gray range [k0, k1) (the whole walk
// for a single call, one shard for a sharded one).  Chunks of 2^log2L must
// tile the range, so log2L is capped by the alignment of k0 and k1 - k0.
static int range_align(uint64_t k0, uint64_t k1) {
  const uint64_t len = k1 - k0;
  int a = len ? __builtin_ctzll(len) : 0;
  if (k0) a = std::min(a, __builtin_ctzll(k0));
  return a;
}

// One Gray range's contribution to an exact integer permanent; serialized
// as 8 int64 by perm_walk_partial_i64.
struct IntPart {
  // CHECKED (width 64): ordered summary (sum, min/max running prefix) of the
  // range's terms and the reference's overflow flag
  s128 S = 0, mn = 0, mx = 0;
  bool flag = false;
  // WRAP (width 128): the range's sum mod 2^128, and an FP64 estimate of it
  // (raw-sum units) with its magnitude sum for the fit certificate
  unsigned __int128 raw = 0;
  double est_hi = 0, est_lo = 0, mag = 0;
  int est_kind = 0;  // 0 none, 1 fused FP64-exact walk, 2 separate float walk, 3 fused FP32-quad walk (FP32 estimate), 4 FP32-quad walk with FP64 upper levels
  bool refused = false;  // entries too large for the FP64 certificate
};

// ------------------------------------------------------------ CHECKED walk
static int checked_range(const IntSetup& s, uint64_t k0, uint64_t k1, cudaStream_t stream, IntPart* p) {
  p->flag = s.pre_overflow;
  if (p->flag || k1 == k0) return PERM_OK;
  const uint64_t steps = k1 - k0;
  const int amax = range_align(k0, k1);
  int log2L = 0;
  while (log2L < amax && (steps >> log2L) > (1ull << 17)) ++log2L;
  const uint64_t nchunks = steps >> log2L;
  const uint64_t blocks = (nchunks + kIntThreads - 1) / kIntThreads;
  const size_t nv0 = s.v0.size(), nU = s.U.size();
  std::vector<int64_t> in(s.v0);
  in.insert(in.end(), s.U.begin(), s.U.end());
  char* base = nullptr;
  size_t out_off = 0;
  int st = int_stage(in.data(), in.size() * 8, blocks * 64, stream, &base, &out_off);
  if (st) return st;
  int64_t* d = reinterpret_cast<int64_t*>(base);
  IntWalkArgs a;
  a.v0 = d;
  a.U = d + nv0;
  a.w = nullptr;
  a.P = s.P;
  a.B = s.B;
  a.log2L = log2L;
  a.wlen = 0;
  a.k_begin = k0;
  a.nchunks = nchunks;
  a.out = reinterpret_cast<int64_t*>(base + out_off);
  int_walk_checked_kernel<<<(unsigned)blocks, kIntThreads, 0, stream>>>(a);
  PERM_CUDA_TRY(cudaGetLastError());
  std::vector<int64_t> h(blocks * 8);
  st = int_fetch(a.out, blocks * 64, stream, h.data());
  if (st) return st;
  // ordered combine of block summaries (Gray order = block order); the
  // empty prefix (0) is included, as in the kernel's identity element
  s128 G = 0, mn = 0, mx = 0;
  for (uint64_t b = 0; b < blocks; ++b) {
    const int64_t* o = &h[b * 8];
    auto get = [&](int q) { return (s128)(((unsigned __int128)(uint64_t)o[q + 1] << 64) | (uint64_t)o[q]); };
    if (o[6]) p->flag = true;
    mn = std::min(mn, G + get(2));
    mx = std::max(mx, G + get(4));
    G += get(0);
  }
  p->S = G;
  p->mn = mn;
  p->mx = mx;
  return PERM_OK;
}

// ------------------------------------------------------------ WRAP walk
walk_fn_i int_wrap_lookup(int P);

// Fused path: FP64-exact state and group products, the int128 sum and its
// FP64 estimate / magnitude sum from one kernel.  The P state entries are
// cut into NG groups of P/NG (+1) entries; a group's products are exact when
// the product of its entries' bounds is below 2^51.  int_fp_groups takes the
// smallest instantiated NG for which a grouping exists (longest-processing-
// time assignment of the entries, largest bound first, to the group with the
// smallest log-product and room left) and returns the state-entry order that
// realizes it (per(A) and the walk sum do not depend on that order).
struct FpGroups {
  int ng = 0;
  std::vector<int> order;  // kernel index -> original state index
};
static bool int_fp_groups(const IntSetup& s, FpGroups* out) {
  const int P = s.P;
  if ((int)s.cb.size() != P) return false;
  std::vector<int> idx(P);
  for (int j = 0; j < P; ++j) idx[j] = j;
  std::sort(idx.begin(), idx.end(), [&](int x, int y) { return s.cb[x] > s.cb[y]; });
  for (int k = 2; k >= 0; --k) {  // fewest groups first
    const int NG = int_fp_ng(P, k);
    if (k < 2 && NG == int_fp_ng(P, k + 1)) continue;
    std::vector<int> cap(NG), start(NG);
    for (int q = 0; q < NG; ++q) {
      start[q] = q * P / NG;
      cap[q] = (q + 1) * P / NG - start[q];
    }
    std::vector<long double> lg(NG, 0.0L);
    std::vector<std::vector<int>> grp(NG);
    bool ok = true;
    for (int j : idx) {
      int best = -1;
      for (int q = 0; q < NG; ++q)
        if ((int)grp[q].size() < cap[q] && (best < 0 || lg[q] < lg[best])) best = q;
      grp[best].push_back(j);
      const s128 b = s.cb[j] < 1 ? 1 : s.cb[j];
      lg[best] += std::log2((long double)b);
      if (lg[best] >= 50.99L) ok = false;
    }
    if (!ok) continue;
    // exact check of each group's bound product against 2^51
    for (int q = 0; q < NG && ok; ++q) {
      unsigned __int128 prod = 1;
      for (int j : grp[q]) {
        const s128 b = s.cb[j] < 1 ? 1 : s.cb[j];
        prod *= (unsigned __int128)b;
        if (prod >= ((unsigned __int128)1 << 51)) ok = false;
      }
    }
    if (!ok) continue;
    out->ng = NG;
    out->order.assign(P, 0);
    for (int q = 0; q < NG; ++q)
      for (size_t i = 0; i < grp[q].size(); ++i) out->order[start[q] + i] = grp[q][i];
    return true;
  }
  return false;
}

static bool fp_walk_ok(const IntSetup& s, uint64_t k0, uint64_t k1, FpGroups* g) {
  return !s.weighted && s.B >= 8 && s.P >= 1 && s.P <= 64 && k1 - k0 >= 8 && range_align(k0, k1) >= 3 &&
         int_fp_groups(s, g);
}

static int wrap_range_fp(const IntSetup& s, const FpGroups& g, uint64_t k0, uint64_t k1, cudaStream_t stream,
                         IntPart* p) {
  const uint64_t steps = k1 - k0;
  const int amax = range_align(k0, k1);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t lanes = (uint64_t)nsm * 8 * kIntThreads;
  int log2L = 3;
  while (log2L < 14 && log2L < amax && (steps >> (log2L + 1)) >= 16 * lanes) ++log2L;
  const uint64_t nchunks = steps >> log2L;
  const uint64_t blocks = std::min<uint64_t>((nchunks + kIntThreads - 1) / kIntThreads, (uint64_t)nsm * 8);
  // state entries in the kernel's group order
  std::vector<double> buf(s.v0.size() + s.U.size());
  const int P = s.P;
  for (int j = 0; j < P; ++j) buf[j] = (double)s.v0[g.order[j]];
  for (int t = 0; t < s.B; ++t)
    for (int j = 0; j < P; ++j) buf[P + (size_t)t * P + j] = (double)s.U[(size_t)t * P + g.order[j]];
  char* base = nullptr;
  size_t out_off = 0;
  int st = int_stage(buf.data(), buf.size() * 8, blocks * 64, stream, &base, &out_off);
  if (st) return st;
  double* d = reinterpret_cast<double*>(base);
  IntWalkFArgs a;
  a.v0 = d;
  a.U = d + s.v0.size();
  a.P = s.P;
  a.B = s.B;
  a.log2L = log2L;
  a.k_begin = k0;
  a.nchunks = nchunks;
  a.out = reinterpret_cast<int64_t*>(base + out_off);
  walk_fn_if fn = int_wrap_fp_lookup(s.P, g.ng);
  if (!fn) {
    set_error("no fp int walk for this size");
    return PERM_BAD_SHAPE;
  }
  PERM_CUDA_TRY(fn(a, (int)blocks, stream));
  std::vector<int64_t> h(blocks * 8);
  st = int_fetch(a.out, blocks * 64, stream, h.data());
  if (st) return st;
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
  p->raw = acc;
  p->est_hi = H;
  p->est_lo = L;
  p->mag = M;
  p->est_kind = 1;
  return PERM_OK;
}

// FP32-quad path (int_walk32.cuh): the P state entries (padded with constant
// ones to 4 NQ) are cut into NQ quads whose products of per-entry bounds stay
// below 2^23, so state, pair and quad products are exact in FP32 and each
// |quad| is a 23-bit integer.  Same longest-processing-time assignment as
// int_fp_groups; `pos` maps the kernel's entry positions (oct-interleaved,
// Walk32) to original state indices, -1 for a pad.
constexpr int kQuadBoundLog2 = 23;
struct F32Quads {
  int nq = 0;
  std::vector<int> pos;
  int scale_log2 = 0;  // the estimate product carries 2^-scale_log2
  // FP64 upper levels: every product of four consecutive quads' bounds is
  // below 2^83 (dmul96s / dmul96 in int_walk32.cuh)
  bool dl4 = false;
};
static bool int_f32_quads(const IntSetup& s, F32Quads* out) {
  const int P = s.P;
  if ((int)s.cb.size() != P || P < 1 || P > 4 * kInt32MaxQuads) return false;
  const int NQ = (P + 3) / 4;
  std::vector<int> idx(P);
  for (int j = 0; j < P; ++j) idx[j] = j;
  std::sort(idx.begin(), idx.end(), [&](int x, int y) { return s.cb[x] > s.cb[y]; });
  std::vector<std::vector<int>> quad(NQ);
  std::vector<long double> lg(NQ, 0.0L);
  long double total = 0.0L;
  for (int j : idx) {
    if (s.cb[j] >= ((s128)1 << kQuadBoundLog2)) return false;
    int best = -1;
    for (int q = 0; q < NQ; ++q)
      if (quad[q].size() < 4 && (best < 0 || lg[q] < lg[best])) best = q;
    quad[best].push_back(j);
    const long double l = std::log2((long double)(s.cb[j] < 1 ? (s128)1 : s.cb[j]));
    lg[best] += l;
    total += l;
  }
  for (int q = 0; q < NQ; ++q) {
    uint64_t prod = 1;  // < 2^23 * 2^23 at every step
    for (int j : quad[q]) {
      prod *= (uint64_t)(s.cb[j] < 1 ? (s128)1 : s.cb[j]);
      if (prod >= (1ull << kQuadBoundLog2)) return false;
    }
  }
  // dmul96 multiplies quads [0, 4) (NQ >= 3) and quads [4, 8) (NQ >= 7)
  out->dl4 = true;
  for (int q0 = 0; q0 < 8; q0 += 4) {
    if (NQ < q0 + 3) break;
    unsigned __int128 prod = 1;  // four quads: < 2^92
    for (int q = q0; q < std::min(NQ, q0 + 4); ++q)
      for (int j : quad[q]) prod *= (unsigned __int128)(uint64_t)(s.cb[j] < 1 ? (s128)1 : s.cb[j]);
    if (prod >= ((unsigned __int128)1 << 83)) out->dl4 = false;
  }
  // the FP32 product of all quads must stay a normal float: 2^-scale keeps it
  // below 2^100, and the smallest nonzero |term| (>= 1) above 2^-120
  const int scale = std::max(0, (int)std::ceil(total) - 100);
  if (scale > 120) return false;
  out->nq = NQ;
  out->scale_log2 = scale;
  out->pos.assign((size_t)4 * NQ, -1);
  const int full = 2 * (NQ / 2);  // quads living in full octs
  for (int q = 0; q < NQ; ++q)
    for (size_t i = 0; i < quad[q].size(); ++i) {
      const int at = q < full ? 8 * (q / 2) + 2 * (int)i + (q & 1) : 8 * (NQ / 2) + (int)i;
      out->pos[at] = quad[q][i];
    }
  return true;
}

static bool f32_walk_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PERM_INT_F32");
    return !(e && e[0] == '0');
  }();
  return on;
}
static bool f32_walk_ok(const IntSetup& s, uint64_t k0, uint64_t k1, F32Quads* g) {
  return f32_walk_enabled() && !s.weighted && s.B >= 8 && s.B <= 62 && k1 - k0 >= 8 && range_align(k0, k1) >= 3 &&
         int_f32_quads(s, g);
}

static int wrap_range_f32(const IntSetup& s, const F32Quads& g, uint64_t k0, uint64_t k1, cudaStream_t stream,
                          IntPart* p) {
  const uint64_t steps = k1 - k0;
  const int amax = range_align(k0, k1);
  int dev = 0, nsm = 148, resident = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  walk_fn_i32 fn = int_wrap_f32_lookup(g.nq, g.dl4, &resident);
  if (!fn) {
    set_error("no FP32-quad int walk for this size");
    return PERM_BAD_SHAPE;
  }
  const uint64_t max_blocks = (uint64_t)nsm * resident;
  const uint64_t lanes = max_blocks * kInt32Threads;
  // chunk length: the slowest lane walks ceil(chunks / lanes) chunks of L
  // steps plus a seed worth ~8 steps (B/2 divergent row adds, the chunk's
  // double-double fold); take the cheapest L
  int log2L = 3;
  double best = 1e300;
  for (int r = 3; r <= 14 && r <= amax; ++r) {
    const uint64_t nch = steps >> r;
    const double cost = (double)((nch + lanes - 1) / lanes) * ((double)(1ull << r) + 8.0);
    if (cost < best * 0.999) {
      best = cost;
      log2L = r;
    }
  }
  const uint64_t nchunks = steps >> log2L;
  const uint64_t blocks = std::min<uint64_t>((nchunks + kInt32Threads - 1) / kInt32Threads, max_blocks);
  const int P4 = 4 * g.nq;
  std::vector<float> buf((size_t)(s.B + 1) * P4);
  for (int j = 0; j < P4; ++j) buf[j] = g.pos[j] < 0 ? 1.0f : (float)s.v0[g.pos[j]];
  for (int t = 0; t < s.B; ++t)
    for (int j = 0; j < P4; ++j)
      buf[(size_t)(t + 1) * P4 + j] = g.pos[j] < 0 ? 0.0f : (float)s.U[(size_t)t * s.P + g.pos[j]];
  char* base = nullptr;
  size_t out_off = 0;
  int st = int_stage(buf.data(), buf.size() * sizeof(float), blocks * 64, stream, &base, &out_off);
  if (st) return st;
  IntWalk32Args a;
  a.v0 = reinterpret_cast<const float*>(base);
  a.U = a.v0 + P4;
  for (int j = 0; j < 2 * kInt32MaxQuads; ++j)  // row 0 of U as packed pairs (kernel parameter)
    a.row0[j] = 2 * j + 1 < P4 ? make_float2(buf[(size_t)P4 + 2 * j], buf[(size_t)P4 + 2 * j + 1]) : make_float2(0.f, 0.f);
  a.B = s.B;
  a.log2L = log2L;
  a.escale = std::ldexp(1.0f, -g.scale_log2);
  a.k_begin = k0;
  a.nchunks = nchunks;
  a.out = reinterpret_cast<int64_t*>(base + out_off);
  PERM_CUDA_TRY(fn(a, (int)blocks, stream));
  std::vector<int64_t> h(blocks * 8);
  st = int_fetch(a.out, blocks * 64, stream, h.data());
  if (st) return st;
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
  p->raw = acc;
  const int sc = g.dl4 ? 0 : g.scale_log2;  // the FP64 estimate is unscaled
  p->est_hi = std::ldexp(H, sc);
  p->est_lo = std::ldexp(L, sc);
  p->mag = std::ldexp(M, sc);
  p->est_kind = g.dl4 ? 4 : 3;
  return PERM_OK;
}

static int wrap_range(const IntSetup& s, uint64_t k0, uint64_t k1, cudaStream_t stream, IntPart* p) {
  if (k1 == k0) return PERM_OK;
  const bool wide = s.bound >= ((s128)1 << 62);  // int64 state could wrap
  const uint64_t steps = k1 - k0;
  const int amax = range_align(k0, k1);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // exact int64 groups of 8 factors need bound^8 < 2^63
  const bool g8 = !wide && !s.weighted && (long double)s.bound < std::pow(2.0L, 63.0L / 8.0L) && steps >= 8;
  const uint64_t lanes = (uint64_t)nsm * 8 * kIntThreads;
  int log2L = std::min(3, amax);
  while (log2L < 14 && log2L < amax && (steps >> (log2L + 1)) >= 16 * lanes) ++log2L;
  if (!g8 && log2L > 10) log2L = 10;
  const uint64_t nchunks = steps >> log2L;
  uint64_t blocks = std::min<uint64_t>((nchunks + kIntThreads - 1) / kIntThreads, (uint64_t)nsm * 8);
  const size_t nv0 = wide ? s.v0w.size() : s.v0.size(), nU = s.U.size(), nw = s.w.size();
  std::vector<int64_t> in(wide ? s.v0w : s.v0);
  in.insert(in.end(), (wide ? s.R : s.U).begin(), (wide ? s.R : s.U).end());
  in.insert(in.end(), s.w.begin(), s.w.end());
  char* base = nullptr;
  size_t out_off = 0;
  int st = int_stage(in.data(), in.size() * 8, blocks * 16, stream, &base, &out_off);
  if (st) return st;
  int64_t* d = reinterpret_cast<int64_t*>(base);
  IntWalkArgs a;
  a.v0 = d;
  a.U = d + nv0;
  a.w = nw ? d + nv0 + nU : nullptr;
  a.P = s.P;
  a.B = s.B;
  a.log2L = log2L;
  a.wlen = (int)nw;
  a.k_begin = k0;
  a.nchunks = nchunks;
  a.out = reinterpret_cast<int64_t*>(base + out_off);
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
  st = int_fetch(a.out, blocks * 16, stream, h.data());
  if (st) return st;
  unsigned __int128 acc = 0;
  for (uint64_t b = 0; b < blocks; ++b)
    acc += ((unsigned __int128)(uint64_t)h[2 * b + 1] << 64) | (uint64_t)h[2 * b];
  p->raw = acc;
  return PERM_OK;
}

// FP64 estimate of a range's raw sum for the fit certificate: the float walk
// with the magnitude sum M.  |raw - est| <= (P + 2^14 + 16) u M (exact state
// entries, <= P-1 product roundings, chunk sums of <= 2^14 terms, double-
// double above).  Rectangular Glynn walks the pre-scaled matrix 2^s A, whose
// raw sum is 2^(s m) times the integer walk's: undone exactly.
static int float_range(int alg, const IntMat& A, uint64_t k0, uint64_t k1, cudaStream_t stream, IntPart* p) {
  p->est_kind = 2;
  if (k1 == k0) return PERM_OK;
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
  st = run_walk(ws, k0, k1, 1, dst, stream);
  if (st) return st;
  PERM_CUDA_TRY(cudaMemcpyAsync(sc->host, dst, 8 * sizeof(double), cudaMemcpyDeviceToHost, stream));
  PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  const int e = -ws.scale_log2 * A.m;
  p->est_hi = std::ldexp(sc->host[0], e);
  p->est_lo = std::ldexp(sc->host[1], e);
  p->mag = std::ldexp(sc->host[4], e);
  return PERM_OK;
}

// ------------------------------------------------------------ certificate
struct IntPlan {
  IntMat A;
  IntSetup s;
  s128 denom = 1;           // Glynn: 2^(n-1) (n-m)!
  bool cert_apriori = false;  // |raw| < 2^126 from row/column sums alone
};

static int plan_int(int alg, int m, int n, const int64_t* a, int64_t lda, int dev_ptr, cudaStream_t stream,
                    IntPlan* pl) {
  int st = load_int_matrix(m, n, a, lda, dev_ptr, &pl->A, stream);
  if (st) return st;
  setup_int(alg, pl->A, &pl->s);
  pl->denom = 1;
  if (alg == PERM_ALG_GLYNN) {
    pl->denom = (s128)1 << (n - 1);
    for (int i = 2; i <= n - m; ++i) pl->denom *= i;
  }
  // |raw| = |per| * denom <= per(|A|) * denom, and per(|A|) is at most the
  // product of the row sums of |A| (and, square, of the column sums)
  long double rows = 1.0L, cols = 1.0L;
  for (int i = 0; i < m; ++i) {
    long double r = 0;
    for (int j = 0; j < n; ++j) r += std::fabs((long double)pl->A.at(i, j));
    rows *= r;
  }
  for (int j = 0; j < n; ++j) {
    long double c = 0;
    for (int i = 0; i < m; ++i) c += std::fabs((long double)pl->A.at(i, j));
    cols *= c;
  }
  const long double apriori = (m == n ? std::min(rows, cols) : rows) * (long double)pl->denom;
  pl->cert_apriori = apriori < std::ldexp(1.0L, 126);
  return PERM_OK;
}

static long double est_error(const IntPart& p, int P) {
  // kind 4: FP64 product of <= 5 exact pair products (4 roundings)
  const long double c = p.est_kind == 2 ? (P + (1 << 14) + 16) : ((p.est_kind == 4 ? 4 : 3) + (1 << 14) + 16);
  // kind 3: each term's estimate is an FP32 product of exact quads (at most
  // 6 roundings, relative error < 2^-21 of |term| <= |estimate| / (1 - 2^-21))
  const long double f32 = p.est_kind == 3 ? std::ldexp(1.0L, -20) : 0.0L;
  return (c * std::ldexp(1.0L, -52) + f32) * (long double)p.mag;
}

// One range.  `full` (the whole walk on one device) lets the separate float
// estimate refuse before the exact walk is spent.
static int int_part(int alg, const IntPlan& pl, int width, uint64_t k0, uint64_t k1, bool full, cudaStream_t stream,
                    IntPart* p) {
  const IntSetup& s = pl.s;
  if (width == 64) return checked_range(s, k0, k1, stream, p);
  F32Quads gq;
  if (f32_walk_ok(s, k0, k1, &gq)) {
    int st = wrap_range_f32(s, gq, k0, k1, stream, p);
    if (st) return st;
    // the FP32 estimate's certificate is looser than the FP64-exact walk's:
    // when it cannot certify the fit on its own, take the FP64 paths below
    if (!full || pl.cert_apriori ||
        (long double)std::fabs(p->est_hi) + est_error(*p, s.P) < std::ldexp(1.0L, 126))
      return PERM_OK;
    *p = IntPart();
  }
  FpGroups g;
  if (fp_walk_ok(s, k0, k1, &g)) return wrap_range_fp(s, g, k0, k1, stream, p);
  if (!pl.cert_apriori) {
    if (s.bound >= ((s128)1 << 52)) {  // state entries not exact in FP64
      p->refused = true;
      return PERM_OK;
    }
    int st = float_range(alg, pl.A, k0, k1, stream, p);
    if (st) return st;
    if (full && (long double)std::fabs(p->est_hi) + est_error(*p, s.P) >= std::ldexp(1.0L, 126)) {
      p->refused = true;
      return PERM_OK;
    }
  }
  return wrap_range(s, k0, k1, stream, p);
}

static int to_out(s128 v, int64_t* out, int* fits_int64) {
  out[0] = (int64_t)(uint64_t)v;
  out[1] = (int64_t)(uint64_t)((unsigned __int128)v >> 64);
  if (fits_int64) *fits_int64 = (v >= kI64Min && v <= kI64Max) ? 1 : 0;
  return PERM_OK;
}

// Combine the ranges' parts in Gray order and normalize.
static int int_finish(int alg, const IntPlan& pl, int width, const IntPart* parts, int G, int64_t* out,
                      int* fits_int64) {
  const int m = pl.A.m, n = pl.A.n;
  if (width == 64) {
    // reference semantics: PERM_OVERFLOW whenever the reference flags
    s128 T = 0;
    bool flag = false;
    for (int g = 0; g < G && !flag; ++g) {
      const IntPart& p = parts[g];
      if (p.flag || T + p.mn < kI64Min || T + p.mx > kI64Max) flag = true;
      T += p.S;
    }
    if (flag) {
      set_error("an int64 intermediate overflowed (reference semantics)");
      return PERM_OVERFLOW;
    }
    s128 v = (int64_t)T;
    if (alg == PERM_ALG_GLYNN) {
      if (v % pl.denom != 0) {  // src/algorithms.py:155-157, 178-180
        set_error("Glynn sum not divisible by its normalization");
        return PERM_OVERFLOW;
      }
      v /= pl.denom;
    } else if (m == n && (n & 1)) {
      v = (s128)(int64_t)(0 - (uint64_t)(int64_t)v);  // int64 negation as in src/_kernels.py:216-217
    }
    return to_out(v, out, fits_int64);
  }
  // width 128: sum mod 2^128; certify |raw| < 2^126 (a priori, or by the
  // summed FP64 estimate and its error bound) and cross-check the estimate
  unsigned __int128 acc = 0;
  double H = 0, L = 0;
  long double E = 0;
  bool have_est = true;
  for (int g = 0; g < G; ++g) {
    const IntPart& p = parts[g];
    if (p.refused) {
      set_error(pl.s.bound >= ((s128)1 << 52)
                    ? "exact value not certified to fit int128 (entries too large for the FP64 certificate)"
                    : "exact value not certified to fit the int128 walk");
      return PERM_OVERFLOW;
    }
    acc += p.raw;
    if (p.est_kind == 0) {
      have_est = false;
    } else {
      dd_add(H, L, p.est_hi, p.est_lo);
      E += est_error(p, pl.s.P);
    }
  }
  const long double est = (long double)H + (long double)L;
  if (!pl.cert_apriori) {
    if (!have_est) {
      set_error("internal: no FP64 estimate for the int128 fit certificate");
      return PERM_CUDA;
    }
    if (std::fabs(est) + E >= std::ldexp(1.0L, 126)) {
      set_error("exact value not certified to fit the int128 walk");
      return PERM_OVERFLOW;
    }
  }
  const s128 raw = (s128)acc;
  if (have_est && std::fabs((long double)raw - est) > E + 1.0L + std::ldexp(std::fabs(est), -60)) {
    set_error("internal: int128 walk disagrees with its FP64 estimate");
    return PERM_CUDA;
  }
  s128 v = raw;
  if (alg == PERM_ALG_GLYNN) {
    if (v % pl.denom != 0) {
      set_error("internal: Glynn int128 sum not divisible by its normalization");
      return PERM_CUDA;
    }
    v /= pl.denom;
  } else if (m == n && (n & 1)) {
    v = -v;
  }
  return to_out(v, out, fits_int64);
}

int int_permanent(int alg, int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, int64_t* out,
                  int* fits_int64, void* stream_) {
  clear_error();
  if (width != 64 && width != 128) {
    set_error("width must be 64 or 128");
    return PERM_BAD_ARG;
  }
  cudaStream_t stream = pick_stream(stream_);
  IntPlan pl;
  int st = plan_int(alg, m, n, a, lda, dev_ptr, stream, &pl);
  if (st) return st;
  IntPart p;
  st = int_part(alg, pl, width, 0, walk_steps(alg, m, n), true, stream, &p);
  if (st) return st;
  return int_finish(alg, pl, width, &p, 1, out, fits_int64);
}

// ------------------------------------------------------------ sharded
static const int64_t kTag64 = 0x7065726d36340000LL, kTag128 = 0x7065726d31323800LL;

static void put128(int64_t* o, s128 v) {
  o[0] = (int64_t)(uint64_t)v;
  o[1] = (int64_t)(uint64_t)((unsigned __int128)v >> 64);
}
static s128 get128(const int64_t* o) {
  return (s128)(((unsigned __int128)(uint64_t)o[1] << 64) | (uint64_t)o[0]);
}

static int check_int_shardable(int alg, int m, int n, int width) {
  if (width != 64 && width != 128) {
    set_error("width must be 64 or 128");
    return PERM_BAD_ARG;
  }
  if (width == 64 && alg == PERM_ALG_RYSER && m < n) {
    set_error("checked rectangular Ryser replays the lexicographic combination order (not sharded); use width 128");
    return PERM_BAD_ARG;
  }
  if (alg != PERM_ALG_GLYNN && alg != PERM_ALG_RYSER) {
    set_error("sharded walks are Glynn or Ryser");
    return PERM_BAD_ARG;
  }
  return PERM_OK;
}

// Host-only: which exact int128 walk the full range of this (host) matrix
// takes.  kind 4 / 3 = quad walk (FP64 / integer upper levels), 1 =
// FP64-exact groups, 0 = generic int64 / 128-bit state; groups = quads or
// FP64 groups.  No CUDA call (CPU tests of the planning logic).
int int_walk_plan(int alg, int m, int n, const int64_t* a, int64_t lda, int* kind, int* groups) {
  clear_error();
  int st = check_int_shardable(alg, m, n, 128);
  if (st) return st;
  IntPlan pl;
  st = load_int_matrix(m, n, a, lda, 0, &pl.A, nullptr);
  if (st) return st;
  setup_int(alg, pl.A, &pl.s);
  const uint64_t k1 = walk_steps(alg, m, n);
  F32Quads gq;
  FpGroups g;
  if (f32_walk_ok(pl.s, 0, k1, &gq)) {
    *kind = gq.dl4 ? 4 : 3;
    *groups = gq.nq;
  } else if (fp_walk_ok(pl.s, 0, k1, &g)) {
    *kind = 1;
    *groups = g.ng;
  } else {
    *kind = 0;
    *groups = 0;
  }
  return PERM_OK;
}

int int_walk_partial(int alg, int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, uint64_t k0,
                     uint64_t k1, int64_t* partial, void* stream_) {
  clear_error();
  int st = check_int_shardable(alg, m, n, width);
  if (st) return st;
  cudaStream_t stream = pick_stream(stream_);
  IntPlan pl;
  st = plan_int(alg, m, n, a, lda, dev_ptr, stream, &pl);
  if (st) return st;
  if (k0 > k1 || k1 > walk_steps(alg, m, n)) {
    set_error("Gray range outside the walk");
    return PERM_BAD_ARG;
  }
  IntPart p;
  st = int_part(alg, pl, width, k0, k1, false, stream, &p);
  if (st) return st;
  std::fill(partial, partial + 8, 0);
  if (width == 64) {
    put128(partial, p.S);
    put128(partial + 2, p.mn);
    put128(partial + 4, p.mx);
    partial[6] = p.flag ? 1 : 0;
    partial[7] = kTag64;
  } else {
    put128(partial, (s128)p.raw);
    std::memcpy(&partial[2], &p.est_hi, 8);
    std::memcpy(&partial[3], &p.est_lo, 8);
    std::memcpy(&partial[4], &p.mag, 8);
    partial[5] = p.est_kind;
    partial[6] = p.refused ? 1 : 0;
    partial[7] = kTag128;
  }
  return PERM_OK;
}

int int_walk_finish(int alg, int m, int n, const int64_t* a, int64_t lda, int width, const int64_t* partials, int G,
                    int64_t* out, int* fits_int64) {
  clear_error();
  int st = check_int_shardable(alg, m, n, width);
  if (st) return st;
  if (G < 1) {
    set_error("no partials");
    return PERM_BAD_ARG;
  }
  IntPlan pl;
  st = plan_int(alg, m, n, a, lda, 0, nullptr, &pl);
  if (st) return st;
  std::vector<IntPart> parts(G);
  for (int g = 0; g < G; ++g) {
    const int64_t* o = partials + 8 * (size_t)g;
    IntPart& p = parts[g];
    if (o[7] != (width == 64 ? kTag64 : kTag128)) {
      set_error("partial was not produced by perm_walk_partial_i64 with this width");
      return PERM_BAD_ARG;
    }
    if (width == 64) {
      p.S = get128(o);
      p.mn = get128(o + 2);
      p.mx = get128(o + 4);
      p.flag = o[6] != 0;
    } else {
      p.raw = (unsigned __int128)get128(o);
      std::memcpy(&p.est_hi, &o[2], 8);
      std::memcpy(&p.est_lo, &o[3], 8);
      std::memcpy(&p.mag, &o[4], 8);
      p.est_kind = (int)o[5];
      p.refused = o[6] != 0;
    }
  }
  return int_finish(alg, pl, width, parts.data(), G, out, fits_int64);
}

}  // namespace permb200
