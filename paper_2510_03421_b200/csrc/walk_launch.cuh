// Host-side planning and launch of the Gray-walk kernels.
#pragma once
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "walk.cuh"

namespace permb200 {

struct WalkJob {
  int dtype;             // 0 = f64, 1 = c128
  int P, B;
  bool weighted;
  const void* v0;        // device
  const void* U;         // device
  const double* w;       // device (weighted) or null
  int wlen;
  int mag;
  uint64_t k_begin, k_end;  // Gray range; k_begin, k_end multiples of 32*L (or tiny range)
  int force_log2L = 0;       // tuning / test knob: chunk length exponent (0 = cost model)
  double* partials;      // device scratch, >= max_partials() * kPartialStride doubles
  double* final_out;     // device, 8 doubles (combined result)
  unsigned int* done;    // device counter, zero on entry
  // zero-copy launch: setup as kernel parameters, result + flag in mapped memory
  const double* inline_host = nullptr;  // host copy of [v0 | U] to pass as kernel parameters
  unsigned int* flag = nullptr;         // mapped host flag set to seq after final_out
  unsigned int seq = 0;
};

// Inline setups (kernel parameters) up to this size: real P <= 26, complex
// P <= 18.  A launch with 4-8 KB of parameters costs ~1-3 us more than an
// empty one on B200 and the blocks read it at ~0.35 us/KB, which beats a
// staged host-to-device copy (~5 us per call) while the walk is short; from
// P = 28 the inline variant's walk measured 0.6-1.8% slower
// (tools/small_walk_exp.cu, profiles/r2_small_walks.txt).
constexpr size_t kWalkInlineMaxBytes = 5632;
template <typename T, int P, bool W>
__host__ __device__ constexpr bool walk_inline_ok() {
  return sizeof(WalkInline<T, P, W>) <= kWalkInlineMaxBytes;
}

struct WalkPlan {
  int grid = 0;          // number of block partials written
  int log2L = 0;
  uint64_t ngroups = 0;
  bool small = false;
};

using walk_fn = cudaError_t (*)(const WalkJob&, WalkPlan*, cudaStream_t);

#ifndef WALK_DEFAULT_MAX_LOG2L
#define WALK_DEFAULT_MAX_LOG2L 10  // accuracy: C5 relative error 8.5e-10 at 2^11, 4.1e-10 at 2^10 (+0.4% time)
#endif
constexpr int kWalkDefaultMaxLog2L = WALK_DEFAULT_MAX_LOG2L;

// Upper bound on block partials any plan writes (grid <= 148 * 8).
constexpr int kMaxPartials = 148 * 16;

// Chunk length for a range of `steps` Gray indices over `lanes` threads:
// long chunks amortize seeding (~6 row FMAs + B/64 sums per chunk), many
// chunks per lane bound the tail of the static lane->chunk assignment.
// Cost model: a warp processes ceil(groups / warps) groups of 32 chunks, each
// chunk costing L steps plus ~3 steps' worth of seeding (6 row FMAs + the
// warp-cooperative column sums); pick the L = 2^r (8 <= L <= 2^14) that
// minimizes the slowest warp's work.
inline int choose_log2L(uint64_t steps, uint64_t lanes, int per_group = 32) {
  const uint64_t warps = lanes / 32 ? lanes / 32 : 1;
  int best = 3;
  double best_cost = 1e300;
  for (int r = 3; r <= 14; ++r) {
    const uint64_t groups = (steps >> r) / per_group;
    if (groups < 1) break;
    const uint64_t per_warp = (groups + warps - 1) / warps;
    const double cost = (double)per_warp * ((double)(1ull << r) + 3.0);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = r;
    }
  }
  return best;
}

// Upper bound on the chunk length exponent: the state drifts by rounding over
// the L updates of a chunk (it is re-seeded exactly at each chunk start), so
// L also sets the walk's accuracy.  PERM_WALK_MAX_LOG2L overrides (tuning).
inline int walk_max_log2L() {
  static const int v = [] {
    const char* e = std::getenv("PERM_WALK_MAX_LOG2L");
    const int x = (e && *e) ? std::atoi(e) : kWalkDefaultMaxLog2L;
    return x < 3 ? 3 : (x > 14 ? 14 : x);
  }();
  return v;
}

// Largest power-of-two alignment that divides x (x != 0), capped.
inline int align_log2(uint64_t x) { return x ? __builtin_ctzll(x) : 64; }

// Resident blocks per SM of `kern` with `smem` dynamic bytes, cached per
// (kernel, smem, device): the query costs microseconds, comparable to a whole
// n <= 22 walk.
template <typename K>
cudaError_t walk_occupancy(K kern, size_t smem, int* nsm_out, int* bps_out) {
  // one slot per kernel (kernels of one signature share this instantiation)
  static thread_local const void* cached_kern = nullptr;
  static thread_local uint64_t cache = 0;  // smem << 32 | dev << 24 | bps << 12 | nsm; 0 = empty
  int dev = 0, nsm = 148, bps = 1;
  cudaGetDevice(&dev);
  const uint64_t c = cached_kern == reinterpret_cast<const void*>(kern) ? cache : 0;
  if (c && (c >> 32) == smem && (int)((c >> 24) & 0xff) == dev) {
    bps = (int)((c >> 12) & 0xfff);
    nsm = (int)(c & 0xfff);
  } else {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kWalkThreads, smem);
    if (e != cudaSuccess) return e;
    if (bps < 1) bps = 1;
    cache = ((uint64_t)smem << 32) | ((uint64_t)(dev & 0xff) << 24) | ((uint64_t)(bps & 0xfff) << 12) |
            (uint64_t)(nsm & 0xfff);
    cached_kern = reinterpret_cast<const void*>(kern);
  }
  *nsm_out = nsm;
  *bps_out = bps;
  return cudaSuccess;
}

// The chunked walk kernel applies when [k_begin, k_begin + steps) tiles into
// groups of 32 chunks of >= 8 steps; other ranges run walk_small_kernel.
inline bool walk_tiled(uint64_t k_begin, uint64_t steps) { return steps >= 256 && ((k_begin | steps) & 255) == 0; }

template <typename T, int P, bool W, bool INL>
cudaError_t launch_walk_impl(const WalkJob& job, WalkPlan* plan, cudaStream_t stream) {
  constexpr int PS = row_stride<T, P>();
  const uint64_t steps = job.k_end - job.k_begin;
  const size_t smem = (size_t)(job.B * PS + PS + kWalkWarps * PS) * sizeof(T) + (size_t)(W ? job.wlen : 0) * 8;
  auto kern = walk_kernel<T, P, W, INL>;
  static int attr_smem = 0;  // benign race: idempotent
  if ((int)smem > 48 * 1024 && attr_smem < (int)smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_smem = (int)smem;
  }
  int nsm = 148, bps = 1;
  cudaError_t e = walk_occupancy(kern, smem, &nsm, &bps);
  if (e != cudaSuccess) return e;
  if (bps * nsm > kMaxPartials) bps = kMaxPartials / nsm;
  const uint64_t lanes = (uint64_t)bps * nsm * kWalkThreads;
  // alignment: chunks of L must tile [k_begin, k_end) in groups of 32
  int r = job.force_log2L > 0 ? job.force_log2L : std::min(choose_log2L(steps, lanes), walk_max_log2L());
  const int amax = std::min(align_log2(job.k_begin), align_log2(steps)) - 5;
  if (r > amax) r = amax;
  if (r < 3 || (steps >> r) < 32) {
    if constexpr (INL) {  // short range, setup inline: one warp (walk_tiny_kernel)
      if (steps > 4096) return cudaErrorInvalidValue;
      WalkBlob<T, P, W, true> blob{};
      const size_t nd = (size_t)(P + (size_t)job.B * P) * Num<T>::kDoubles + (W ? (size_t)job.wlen : 0);
      std::memcpy(blob.d, job.inline_host, nd * sizeof(double));
      WalkArgs a{};
      a.B = job.B; a.wlen = job.wlen; a.mag = job.mag; a.k_begin = job.k_begin;
      a.final_out = job.final_out; a.flag = job.flag; a.seq = job.seq;
      plan->small = true;
      plan->grid = 1;
      plan->log2L = 0;
      walk_tiny_kernel<T, P, W><<<1, 32, 0, stream>>>(a, blob, job.k_end);
      return cudaGetLastError();
    }
    if (job.flag) return cudaErrorInvalidValue;  // the flag path is inline-only
    plan->small = true;
    plan->grid = 1;
    plan->log2L = 0;
    walk_small_kernel<T, P><<<1, 32, 0, stream>>>(static_cast<const T*>(job.v0), static_cast<const T*>(job.U), job.w,
                                               P, job.B, W ? 1 : 0, job.mag, job.k_begin, job.k_end, job.final_out);
    return cudaGetLastError();
  }
  if (!INL && job.U != static_cast<const T*>(job.v0) + P) return cudaErrorInvalidValue;  // [v0 | U] contiguous
  WalkBlob<T, P, W, INL> blob{};
  WalkArgs a;
  a.v0 = job.v0; a.U = job.U; a.w = job.w; a.B = job.B; a.log2L = r; a.wlen = job.wlen; a.mag = job.mag;
  a.k_begin = job.k_begin;
  a.ngroups = (steps >> r) / 32;
  a.partials = job.partials;
  a.final_out = job.final_out;
  a.done = job.done;
  a.flag = job.flag;
  a.seq = job.seq;
  if constexpr (INL) {
    const size_t nd = (size_t)(P + (size_t)job.B * P) * Num<T>::kDoubles + (W ? (size_t)job.wlen : 0);
    std::memcpy(blob.d, job.inline_host, nd * sizeof(double));
  }
  uint64_t grid = (uint64_t)bps * nsm;
  const uint64_t need = (a.ngroups + kWalkWarps - 1) / kWalkWarps;
  if (grid > need) grid = need;
  plan->small = false;
  plan->grid = (int)grid;
  plan->log2L = r;
  plan->ngroups = a.ngroups;
  kern<<<(unsigned)grid, kWalkThreads, smem, stream>>>(a, blob);
  return cudaGetLastError();
}

template <typename T, int P, bool W>
cudaError_t launch_walk(const WalkJob& job, WalkPlan* plan, cudaStream_t stream) {
  if constexpr (walk_inline_ok<T, P, W>()) {
    if (job.inline_host) {
      if (W ? (job.B > 62 || job.wlen > 63) : job.B > P) return cudaErrorInvalidValue;
      return launch_walk_impl<T, P, W, true>(job, plan, stream);
    }
  }
  if (job.inline_host) return cudaErrorInvalidValue;
  return launch_walk_impl<T, P, W, false>(job, plan, stream);
}

// ---- many square Glynn walks in one launch (batches of n = 17..30) -------
struct WalkMultiPlan {
  int segs = 1, log2L = 3;
  uint64_t groups_per_seg = 0;
  int grid = 0;
};
// Segments per matrix: work items (matrix, segment) are dealt round-robin to
// a grid of at most 8 blocks per resident slot, so the last wave's fill
// decides the efficiency; split each matrix until there are >= 8 waves of
// items, keeping >= 8 groups of 32 chunks of L >= 2^8 per segment (one group
// per warp).  Chunk length as long as the segment allows, capped like
// single walks.
inline WalkMultiPlan plan_walk_multi(int n, int64_t nmats, int nsm, int bps) {
  WalkMultiPlan pl;
  const int bits = n - 1;  // log2 of the steps per matrix
  const int64_t slots = (int64_t)nsm * bps;
  int lseg = 0;
  while ((nmats << lseg) < 8 * slots && bits - 8 - (lseg + 1) >= 8) ++lseg;
  pl.segs = 1 << lseg;
  pl.log2L = std::min(walk_max_log2L(), bits - 8 - lseg);  // 8 warps x 32 lanes x L per segment pass
  if (pl.log2L < 3) pl.log2L = 3;
  pl.groups_per_seg = ((1ull << bits) >> (pl.log2L + 5)) >> lseg;
  const int64_t items = nmats * pl.segs;
  pl.grid = (int)std::min<int64_t>(items, slots * 8);
  return pl;
}

template <typename T, int P>
cudaError_t launch_walk_multi(const void* a, void* out, int64_t nmats, int m, double* partials, unsigned int* done,
                              const WalkMultiPlan& pl, cudaStream_t stream) {
  constexpr int PS = row_stride<T, P>();
  const size_t smem = (size_t)((P - 1) * PS + PS + kWalkWarps * PS) * sizeof(T);
  WalkMultiArgs args;
  args.a = a;
  args.out = out;
  args.partials = partials;
  args.done = done;
  args.nmats = nmats;
  args.m = m;
  args.segs = pl.segs;
  args.log2L = pl.log2L;
  args.groups_per_seg = pl.groups_per_seg;
  double f = 1.0;
  for (int i = 2; i <= P - m; ++i) f *= (double)i;
  args.scale = std::ldexp(1.0, -(P - 1)) / f;
  walk_multi_kernel<T, P><<<pl.grid, kWalkThreads, smem, stream>>>(args);
  return cudaGetLastError();
}
template <typename T, int P>
int walk_multi_blocks_per_sm() {
  constexpr int PS = row_stride<T, P>();
  const size_t smem = (size_t)((P - 1) * PS + PS + kWalkWarps * PS) * sizeof(T);
  int bps = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, walk_multi_kernel<T, P>, kWalkThreads, smem) != cudaSuccess)
    bps = 1;
  return bps < 1 ? 1 : bps;
}
using walk_multi_fn = cudaError_t (*)(const void*, void*, int64_t, int, double*, unsigned int*,
                                      const WalkMultiPlan&, cudaStream_t);
using walk_multi_bps_fn = int (*)();
// walk_multi_inst.cu: P = 17..30, double and cd
walk_multi_fn walk_multi_lookup(bool cplx, int P);
walk_multi_bps_fn walk_multi_bps_lookup(bool cplx, int P);
constexpr int kWalkMultiMinN = 17, kWalkMultiMaxN = 30;

template <typename T, bool W, int... Ps>
walk_fn walk_pick(int P, std::integer_sequence<int, Ps...>) {
  walk_fn fn = nullptr;
  ((P == Ps + 1 ? (fn = &launch_walk<T, Ps + 1, W>, 0) : 0), ...);
  return fn;
}

// Per-translation-unit lookup tables (instantiated in walk_inst_*.cu).
walk_fn walk_lookup(int dtype, bool weighted, int P);

}  // namespace permb200
