// Exact integer Gray walks (north_star item 3), two modes:
//
// CHECKED (reference semantics).  Replays the reference's pre-checked int64
// arithmetic (src/_kernels.py:148-218 ryser_sq_int, :412-523 glynn_sq_int,
// :580-697 glynn_rect_int).  The reference returns (0, True) at the first
// int64 overflow; since every value before that point is exact, its flag is
// the OR, over the exact computation, of "this checked operation left int64".
// That OR is evaluated in parallel: each thread replays one contiguous Gray
// range with checked state updates and checked prefix products (stopping at
// the first zero factor exactly as the reference does), and summarizes its
// terms as (S, min prefix, max prefix) in 128-bit.  Ranges combine with the
// associative (S1,m1,M1)+(S2,m2,M2) = (S1+S2, min(m1,S1+m2), max(M1,S1+M2)),
// in Gray order (lanes, then warps, then blocks on the host), so the running
// total's int64 excursions are detected exactly as the sequential walk would.
//
// WRAP (exact int128, opt-in).  Mod-2^128 ring arithmetic: the
// walk sum is exact whenever the true value lies in (-2^127, 2^127), which the
// host certifies with an FP64 run plus its magnitude-sum error bound.
#pragma once
#include <utility>

#include "common.cuh"
#include "walk.cuh"

namespace permb200 {

constexpr int kIntThreads = 128;
constexpr int kIntWarps = kIntThreads / 32;

struct IntWalkArgs {
  const int64_t* v0;   // [P]
  const int64_t* U;    // [B][P]
  const int64_t* w;    // [wlen] (weighted wrap walks)
  int P, B, log2L, wlen;
  uint64_t k_begin;
  uint64_t nchunks;
  int64_t* out;        // per block: 8 int64 slots
};

// --- CHECKED summary combine ---------------------------------------------
struct Summ {
  i128 S, mn, mx;
  int flag;
};
__device__ __forceinline__ Summ summ_cat(const Summ& a, const Summ& b) {  // a precedes b
  Summ r;
  r.flag = a.flag | b.flag;
  r.S = i128_add(a.S, b.S);
  i128 bm = i128_add(a.S, b.mn), bM = i128_add(a.S, b.mx);
  r.mn = i128_lt(bm, a.mn) ? bm : a.mn;
  r.mx = i128_lt(a.mx, bM) ? bM : a.mx;
  return r;
}
__device__ __forceinline__ i128 shfl_down_i128(i128 x, int off) {
  i128 r;
  r.lo = __shfl_down_sync(0xffffffffu, x.lo, off);
  r.hi = __shfl_down_sync(0xffffffffu, x.hi, off);
  return r;
}

__device__ __forceinline__ bool add_ovf(int64_t a, int64_t b, int64_t& r) {
  r = (int64_t)((uint64_t)a + (uint64_t)b);
  return ((a ^ r) & (b ^ r)) < 0;
}
__device__ __forceinline__ bool sub_ovf(int64_t a, int64_t b, int64_t& r) {
  r = (int64_t)((uint64_t)a - (uint64_t)b);
  return ((a ^ b) & (a ^ r)) < 0;
}
__device__ __forceinline__ bool mul_ovf(int64_t a, int64_t b, int64_t& r) {
  r = (int64_t)((uint64_t)a * (uint64_t)b);
  const int64_t hi = __mul64hi(a, b);
  return hi != (r >> 63);
}

// One contiguous range of 2^log2L indices per thread; grid covers nchunks exactly.
static __global__ void __launch_bounds__(kIntThreads) int_walk_checked_kernel(IntWalkArgs a) {
  const uint64_t gtid = (uint64_t)blockIdx.x * kIntThreads + threadIdx.x;
  const int P = a.P, B = a.B;
  Summ s;
  s.S = i128_from(0);
  s.mn = i128_from(0);
  s.mx = i128_from(0);
  s.flag = 0;
  bool have = false;
  if (gtid < a.nchunks) {
    const uint64_t k0 = a.k_begin + (gtid << a.log2L);
    const uint64_t k1 = k0 + (1ull << a.log2L);
    int64_t v[64];
    const uint64_t g0 = k0 ^ (k0 >> 1);
    for (int j = 0; j < P; ++j) {
      i128 acc = i128_from(a.v0[j]);
      for (int t = 0; t < B; ++t)
        if ((g0 >> t) & 1) acc = i128_add(acc, i128_from(a.U[(size_t)t * P + j]));
      if (!i128_fits_i64(acc)) s.flag = 1;  // the reference's update producing this state overflowed
      v[j] = (int64_t)acc.lo;
    }
    for (uint64_t k = k0; k < k1 && !s.flag; ++k) {
      if (k != k0) {
        const int t = __ffsll((long long)k) - 1;
        const bool set = ((k ^ (k >> 1)) >> t) & 1;
        const int64_t* u = a.U + (size_t)t * P;
        for (int j = 0; j < P; ++j) {
          int64_t r;
          bool o = set ? add_ovf(v[j], u[j], r) : sub_ovf(v[j], u[j], r);
          if (o) s.flag = 1;
          v[j] = r;
        }
        if (s.flag) break;
      }
      int64_t p = 1;
      for (int j = 0; j < P; ++j) {  // src/_kernels.py:486-507: stop at the first zero factor
        if (v[j] == 0) { p = 0; break; }
        int64_t r;
        if (mul_ovf(p, v[j], r)) { s.flag = 1; break; }
        p = r;
      }
      if (s.flag) break;
      i128 x = i128_from(p);
      if (k & 1) x = i128_sub(i128_from(0), x);
      s.S = i128_add(s.S, x);
      if (!have) {
        s.mn = s.S;
        s.mx = s.S;
        have = true;
      } else {
        if (i128_lt(s.S, s.mn)) s.mn = s.S;
        if (i128_lt(s.mx, s.S)) s.mx = s.S;
      }
    }
  }
  // empty summaries (threads past nchunks) are identities: S = 0, mn = mx = 0
  // would wrongly clamp; give them mn = +big, mx = -big instead.
  if (!have) {
    s.mn.lo = ~0ull; s.mn.hi = 0x3fffffffffffffffull;       // +2^126-ish
    s.mx.lo = 0ull;  s.mx.hi = 0xc000000000000000ull;       // -2^126
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Summ o;
    o.S = shfl_down_i128(s.S, off);
    o.mn = shfl_down_i128(s.mn, off);
    o.mx = shfl_down_i128(s.mx, off);
    o.flag = __shfl_down_sync(0xffffffffu, s.flag, off);
    // lane i combines with lane i+off only when aligned (ordered tree)
    if ((lane & (2 * off - 1)) == 0 && lane + off < 32) s = summ_cat(s, o);
  }
  __shared__ Summ ws[kIntWarps];
  if (lane == 0) ws[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    Summ t = ws[0];
    for (int w = 1; w < kIntWarps; ++w) t = summ_cat(t, ws[w]);
    int64_t* o = a.out + (size_t)blockIdx.x * 8;
    o[0] = (int64_t)t.S.lo; o[1] = (int64_t)t.S.hi;
    o[2] = (int64_t)t.mn.lo; o[3] = (int64_t)t.mn.hi;
    o[4] = (int64_t)t.mx.lo; o[5] = (int64_t)t.mx.hi;
    o[6] = t.flag; o[7] = 0;
  }
}

// ---- WRAP: exact mod-2^128 walk -------------------------------------------
// Generic (runtime P, optional popcount weights); grid-stride over chunks.
static __global__ void __launch_bounds__(kIntThreads) int_walk_wrap_generic_kernel(IntWalkArgs a, int weighted) {
  const int P = a.P, B = a.B;
  i128 acc = i128_from(0);
  const uint64_t nthr = (uint64_t)gridDim.x * kIntThreads;
  for (uint64_t c = (uint64_t)blockIdx.x * kIntThreads + threadIdx.x; c < a.nchunks; c += nthr) {
    const uint64_t k0 = a.k_begin + (c << a.log2L);
    const uint64_t k1 = k0 + (1ull << a.log2L);
    int64_t v[64];
    const uint64_t g0 = k0 ^ (k0 >> 1);
    for (int j = 0; j < P; ++j) {
      int64_t x = a.v0[j];
      for (int t = 0; t < B; ++t)
        if ((g0 >> t) & 1) x += a.U[(size_t)t * P + j];
      v[j] = x;
    }
    int pc = __popcll(g0);
    for (uint64_t k = k0; k < k1; ++k) {
      if (k != k0) {
        const int t = __ffsll((long long)k) - 1;
        const bool set = ((k ^ (k >> 1)) >> t) & 1;
        const int64_t* u = a.U + (size_t)t * P;
        if (set) for (int j = 0; j < P; ++j) v[j] += u[j];
        else for (int j = 0; j < P; ++j) v[j] -= u[j];
        pc += set ? 1 : -1;
      }
      i128 p = i128_from(v[0]);
      for (int j = 1; j < P; ++j) p = i128_mul_s64(p, v[j]);
      if (weighted) acc = i128_add(acc, i128_mul_s64(p, a.w[pc]));
      else acc = (k & 1) ? i128_sub(acc, p) : i128_add(acc, p);
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc = i128_add(acc, shfl_down_i128(acc, off));
  __shared__ i128 ws[kIntWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) ws[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = ws[0];
    for (int w = 1; w < kIntWarps; ++w) t = i128_add(t, ws[w]);
    a.out[(size_t)blockIdx.x * 2] = (int64_t)t.lo;
    a.out[(size_t)blockIdx.x * 2 + 1] = (int64_t)t.hi;
  }
}

// WRAP walk with 128-bit state entries, for matrices whose row / column
// magnitudes reach 2^62 (where the int64 state of the kernels above could
// wrap).  Runtime P, optional weights; everything mod 2^128.
static __global__ void __launch_bounds__(kIntThreads) int_walk_wrap_wide_kernel(IntWalkArgs a, int weighted, int64_t rscale) {
  const int P = a.P, B = a.B;
  i128 acc = i128_from(0);
  const uint64_t nthr = (uint64_t)gridDim.x * kIntThreads;
  for (uint64_t c = (uint64_t)blockIdx.x * kIntThreads + threadIdx.x; c < a.nchunks; c += nthr) {
    const uint64_t k0 = a.k_begin + (c << a.log2L);
    const uint64_t k1 = k0 + (1ull << a.log2L);
    i128 v[64];
    const uint64_t g0 = k0 ^ (k0 >> 1);
    for (int j = 0; j < P; ++j) {
      i128 x;
      x.lo = (uint64_t)a.v0[2 * j];
      x.hi = (uint64_t)a.v0[2 * j + 1];
      for (int t = 0; t < B; ++t)
        if ((g0 >> t) & 1) x = i128_add(x, i128_mul_s64(i128_from(a.U[(size_t)t * P + j]), rscale));
      v[j] = x;
    }
    int pc = __popcll(g0);
    for (uint64_t k = k0; k < k1; ++k) {
      if (k != k0) {
        const int t = __ffsll((long long)k) - 1;
        const bool set = ((k ^ (k >> 1)) >> t) & 1;
        const int64_t* u = a.U + (size_t)t * P;
        for (int j = 0; j < P; ++j) {
          const i128 du = i128_mul_s64(i128_from(u[j]), rscale);
          v[j] = set ? i128_add(v[j], du) : i128_sub(v[j], du);
        }
        pc += set ? 1 : -1;
      }
      i128 p = v[0];
      for (int j = 1; j < P; ++j) p = i128_mul(p, v[j]);
      if (weighted) acc = i128_add(acc, i128_mul_s64(p, a.w[pc]));
      else acc = (k & 1) ? i128_sub(acc, p) : i128_add(acc, p);
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc = i128_add(acc, shfl_down_i128(acc, off));
  __shared__ i128 ws[kIntWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) ws[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = ws[0];
    for (int w = 1; w < kIntWarps; ++w) t = i128_add(t, ws[w]);
    a.out[(size_t)blockIdx.x * 2] = (int64_t)t.lo;
    a.out[(size_t)blockIdx.x * 2 + 1] = (int64_t)t.hi;
  }
}

// Fast unweighted WRAP walk, compile-time P; factors multiplied exactly in
// int64 in groups of 8 (host guarantees |state|^8 < 2^63), groups folded
// into the 128-bit product.  Same 8-step unrolled schedule as walk_kernel.
template <int P>
__device__ __forceinline__ i128 int_prod_g8(const int64_t (&v)[P]) {
  constexpr int NG = (P + 7) / 8;
  int64_t g[NG];
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    int64_t x = v[8 * q];
#pragma unroll
    for (int j = 8 * q + 1; j < 8 * q + 8 && j < P; ++j) x *= v[j];
    g[q] = x;
  }
  i128 p = i128_from(g[0]);
#pragma unroll
  for (int q = 1; q < NG; ++q) p = i128_mul_s64(p, g[q]);
  return p;
}

template <int P>
__device__ __forceinline__ void irow(int64_t (&v)[P], const int64_t* __restrict__ row, int64_t sign) {
  // v += sign * row, sign in {+1, -1}: two's-complement negate via xor/sub
  const int64_t msk = sign >> 63;  // 0 or -1
#pragma unroll
  for (int j = 0; j < P; ++j) v[j] += (((const volatile int64_t*)row)[j] ^ msk) - msk;
}
template <int P>
__device__ __forceinline__ void irow_add(int64_t (&v)[P], const int64_t* __restrict__ row) {
#pragma unroll
  for (int j = 0; j < P; ++j) v[j] += ((const volatile int64_t*)row)[j];
}
template <int P>
__device__ __forceinline__ void irow_sub(int64_t (&v)[P], const int64_t* __restrict__ row) {
#pragma unroll
  for (int j = 0; j < P; ++j) v[j] -= ((const volatile int64_t*)row)[j];
}

template <int P>
__global__ void __launch_bounds__(kIntThreads) int_walk_wrap_kernel(IntWalkArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int64_t* sU = reinterpret_cast<int64_t*>(smem_raw);
  const int B = a.B;
  for (int i = threadIdx.x; i < B * P; i += kIntThreads) sU[i] = a.U[i];
  __syncthreads();
  const uint64_t L = 1ull << a.log2L;
  const uint64_t nq = L >> 3;
  i128 acc = i128_from(0);
  const uint64_t nthr = (uint64_t)gridDim.x * kIntThreads;
  for (uint64_t c = (uint64_t)blockIdx.x * kIntThreads + threadIdx.x; c < a.nchunks; c += nthr) {
    const uint64_t k0 = a.k_begin + (c << a.log2L);
    int64_t v[P];
    const uint64_t g0 = k0 ^ (k0 >> 1);
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = a.v0[j];
    for (int t = 0; t < B; ++t)
      if ((g0 >> t) & 1) irow_add<P>(v, sU + t * P);
    for (uint64_t q = 0; q < nq; ++q) {
      const uint64_t l0 = q << 3;
      if (q) {
        const int t = __ffsll((long long)l0) - 1;
        const uint64_t k = k0 + l0;
        const int set = (int)(((k ^ (k >> 1)) >> t) & 1);
        irow<P>(v, sU + t * P, set ? 1 : -1);
      }
      acc = i128_add(acc, int_prod_g8<P>(v));
      irow_add<P>(v, sU);
      acc = i128_sub(acc, int_prod_g8<P>(v));
      irow_add<P>(v, sU + P);
      acc = i128_add(acc, int_prod_g8<P>(v));
      irow_sub<P>(v, sU);
      acc = i128_sub(acc, int_prod_g8<P>(v));
      {
        const int b3 = (int)(((k0 + l0) >> 3) & 1);
        irow<P>(v, sU + 2 * P, b3 ? -1 : 1);
      }
      acc = i128_add(acc, int_prod_g8<P>(v));
      irow_add<P>(v, sU);
      acc = i128_sub(acc, int_prod_g8<P>(v));
      irow_sub<P>(v, sU + P);
      acc = i128_add(acc, int_prod_g8<P>(v));
      irow_sub<P>(v, sU);
      acc = i128_sub(acc, int_prod_g8<P>(v));
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc = i128_add(acc, shfl_down_i128(acc, off));
  __shared__ i128 ws[kIntWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) ws[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = ws[0];
    for (int w = 1; w < kIntWarps; ++w) t = i128_add(t, ws[w]);
    a.out[(size_t)blockIdx.x * 2] = (int64_t)t.lo;
    a.out[(size_t)blockIdx.x * 2 + 1] = (int64_t)t.hi;
  }
}

// FP64-exact WRAP walk for small integer entries (state entries grouped so
// that each group's product of per-entry bounds is < 2^51; the default
// groups of 8 need |state| <= 83): state updates and group products
// run on the FP64 pipe exactly, each group product is converted to int64
// and folded into the mod-2^128 term.  The same products give the FP64
// estimate of every term for free, so the int128 fit certificate (FP64 sum
// + magnitude sum) is accumulated in the same pass.  Per block out slots:
// [0..1] int128 sum, [2..3] FP64 double-double sum, [4] magnitude sum.
struct IntWalkFArgs {
  const double* v0;   // [P] exact integers
  const double* U;    // [B][P] exact integers
  int P, B, log2L;
  uint64_t k_begin, nchunks;
  int64_t* out;       // [blocks][8]
};

// Exact double -> int64 for integer values |x| < 2^51 without F2I (whose
// variable latency stalled the walk on the short scoreboard): adding
// 1.5 * 2^52 puts x in the low mantissa bits.
__device__ __forceinline__ int64_t exact_d2ll(double x) {
  return __double_as_longlong(x + 6755399441055744.0) - 0x4338000000000000LL;
}

// signed 64 x 64 -> 128 (exact)
__device__ __forceinline__ i128 i128_mul_s64s64(int64_t a, int64_t b) {
  i128 r;
  r.lo = (uint64_t)a * (uint64_t)b;
  r.hi = (uint64_t)__mul64hi(a, b);
  return r;
}

// The group products as int64, multiplied as a pairwise tree: exact signed
// 64x64->128 products of neighbouring groups, then mod-2^128 products of
// those (P = 32: 2 wide products + 1 mod-2^128 product instead of 3
// i128 x int64 products in a chain).
template <int NG>
__device__ __forceinline__ i128 group_product_i128(const int64_t (&c)[NG]) {
  if constexpr (NG == 1) {
    return i128_from(c[0]);
  } else if constexpr (NG == 2) {
    return i128_mul_s64s64(c[0], c[1]);
  } else if constexpr (NG == 3) {
    return i128_mul_s64(i128_mul_s64s64(c[0], c[1]), c[2]);
  } else {
    i128 p = i128_mul(i128_mul_s64s64(c[0], c[1]), i128_mul_s64s64(c[2], c[3]));
#pragma unroll
    for (int q = 4; q + 1 < NG; q += 2) p = i128_mul(p, i128_mul_s64s64(c[q], c[q + 1]));
    if constexpr (NG > 4 && (NG & 1)) p = i128_mul_s64(p, c[NG - 1]);
    return p;
  }
}

// Product of state entries [Q P / NG, (Q + 1) P / NG) as a balanced tree:
// every sub-product is an exact integer below 2^51 (the host certified the
// group's product of per-entry bounds), so the order is free, and B200's FP64
// pipe wants many independent DMULs in a row.
template <int P, int NG, int Q>
__device__ __forceinline__ double fp_group(const double (&v)[P]) {
  constexpr int lo = Q * P / NG, W = (Q + 1) * P / NG - lo;
  double t[W];
#pragma unroll
  for (int j = 0; j < W; ++j) t[j] = v[lo + j];
#pragma unroll
  for (int h = 1; h < W; h <<= 1)
#pragma unroll
    for (int j = 0; j + h < W; j += 2 * h) t[j] *= t[j + h];
  return t[0];
}
template <int P, int NG, int... Qs>
__device__ __forceinline__ void fp_groups(const double (&v)[P], double (&g)[NG], std::integer_sequence<int, Qs...>) {
  ((g[Qs] = fp_group<P, NG, Qs>(v)), ...);
}

// One term: NG group products (FP64, exact), their int128 product (mod
// 2^128) into acc, and the FP64 estimate / magnitude of the term.  Fewer,
// larger groups cut the 64x64 -> 128-bit integer products per step (NG = 4:
// ~40 IMAD, NG = 3: ~18).
template <int P, int NG>
__device__ __forceinline__ void fp_term(const double (&v)[P], bool neg, i128& acc, double& est, double& mag) {
  double g[NG];
  fp_groups<P, NG>(v, g, std::make_integer_sequence<int, NG>{});
  int64_t c[NG];
  double f = g[0];
#pragma unroll
  for (int q = 0; q < NG; ++q) c[q] = exact_d2ll(g[q]);
#pragma unroll
  for (int q = 1; q < NG; ++q) f *= g[q];
  const i128 p = group_product_i128<NG>(c);
  if (neg) {
    acc = i128_sub(acc, p);
    est -= f;
  } else {
    acc = i128_add(acc, p);
    est += f;
  }
  mag += fabs(f);
}

#ifndef INT_FP_MINB
#define INT_FP_MINB 2  // 220 regs, no spills: 8 warps/SM beat 12 spilling ones (C4a 20.1 -> 15.4 ms)
#endif
template <int P, int NG>
__global__ void __launch_bounds__(kIntThreads, INT_FP_MINB) int_walk_wrap_fp_kernel(IntWalkFArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sU = reinterpret_cast<double*>(smem_raw);
  constexpr int PS = (P + 1) & ~1;
  const int B = a.B;
  for (int i = threadIdx.x; i < B * P; i += kIntThreads) sU[(i / P) * PS + (i % P)] = a.U[i];
  __syncthreads();
  const uint64_t nq = (1ull << a.log2L) >> 3;
  i128 acc = i128_from(0);
  double hi = 0.0, lo = 0.0, mag = 0.0;
  // (U[0] in registers, as in the float walk, measured slower here: C4a
  // 15.5 -> 16.8 ms at 255 registers)
#define INT_ROW0(op) row_##op<double, P>(v, sU);
  const uint64_t nthr = (uint64_t)gridDim.x * kIntThreads;
  for (uint64_t c = (uint64_t)blockIdx.x * kIntThreads + threadIdx.x; c < a.nchunks; c += nthr) {
    const uint64_t k0 = a.k_begin + (c << a.log2L);
    double v[P];
    const uint64_t g0 = k0 ^ (k0 >> 1);
    PERM_CHECK(a.log2L >= 3 && a.log2L <= B && (B >= 63 || (k0 >> B) == 0));
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = a.v0[j];
    for (int t = 0; t < B; ++t)
      if ((g0 >> t) & 1) row_add<double, P>(v, sU + t * PS);
    double est = 0.0;
    for (uint64_t q = 0; q < nq; ++q) {
      const uint64_t l0 = q << 3;
      if (q) {
        const int t = __ffsll((long long)l0) - 1;
        const uint64_t k = k0 + l0;
        const int set = (int)(((k ^ (k >> 1)) >> t) & 1);
        row_fma<double, P>(v, set ? 1.0 : -1.0, sU + t * PS);
      }
      fp_term<P, NG>(v, false, acc, est, mag);
      INT_ROW0(add);
      fp_term<P, NG>(v, true, acc, est, mag);
      row_add<double, P>(v, sU + PS);
      fp_term<P, NG>(v, false, acc, est, mag);
      INT_ROW0(sub);
      fp_term<P, NG>(v, true, acc, est, mag);
      row_fma<double, P>(v, (((k0 + l0) >> 3) & 1) ? -1.0 : 1.0, sU + 2 * PS);
      fp_term<P, NG>(v, false, acc, est, mag);
      INT_ROW0(add);
      fp_term<P, NG>(v, true, acc, est, mag);
      row_sub<double, P>(v, sU + PS);
      fp_term<P, NG>(v, false, acc, est, mag);
      INT_ROW0(sub);
      fp_term<P, NG>(v, true, acc, est, mag);
    }
    dd_acc(hi, lo, est);
#undef INT_ROW0
  }
  for (int off = 16; off > 0; off >>= 1) {
    acc = i128_add(acc, shfl_down_i128(acc, off));
    dd_add(hi, lo, __shfl_down_sync(0xffffffffu, hi, off), __shfl_down_sync(0xffffffffu, lo, off));
    mag += __shfl_down_sync(0xffffffffu, mag, off);
  }
  __shared__ i128 ws[kIntWarps];
  __shared__ double wd[kIntWarps][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    ws[warp] = acc;
    wd[warp][0] = hi; wd[warp][1] = lo; wd[warp][2] = mag;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = ws[0];
    double H = wd[0][0], L = wd[0][1], M = wd[0][2];
    for (int w = 1; w < kIntWarps; ++w) {
      t = i128_add(t, ws[w]);
      dd_add(H, L, wd[w][0], wd[w][1]);
      M += wd[w][2];
    }
    int64_t* o = a.out + (size_t)blockIdx.x * 8;
    o[0] = (int64_t)t.lo; o[1] = (int64_t)t.hi;
    o[2] = __double_as_longlong(H); o[3] = __double_as_longlong(L); o[4] = __double_as_longlong(M);
  }
}

using walk_fn_i = cudaError_t (*)(const IntWalkArgs&, int blocks, cudaStream_t);
using walk_fn_if = cudaError_t (*)(const IntWalkFArgs&, int blocks, cudaStream_t);
// Group counts instantiated for the fp walk at state length P: groups of
// about 8, 11 and 14 entries (the host takes the smallest count whose groups
// it can certify, int_fp_groups in engine_int.cu).
__host__ __device__ constexpr int int_fp_ng(int P, int k) {
  const int gs = k == 0 ? 8 : (k == 1 ? 11 : 14);
  return (P + gs - 1) / gs;
}
walk_fn_if int_wrap_fp_lookup(int P, int NG);

template <int P, int NG>
cudaError_t launch_int_wrap_fp(const IntWalkFArgs& a, int blocks, cudaStream_t stream) {
  const size_t smem = (size_t)a.B * ((P + 1) & ~1) * sizeof(double);
  auto kern = int_walk_wrap_fp_kernel<P, NG>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<blocks, kIntThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

template <int P>
cudaError_t launch_int_wrap(const IntWalkArgs& a, int blocks, cudaStream_t stream) {
  const size_t smem = (size_t)a.B * P * sizeof(int64_t);
  auto kern = int_walk_wrap_kernel<P>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<blocks, kIntThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace permb200
