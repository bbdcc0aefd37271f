// Shared device helpers for the exact-permanent engine (sm_100a).
//
// * cd: complex128 as an aligned double pair (numpy complex128 layout), so a
//   warp-uniform shared-memory read of one element is a single LDS.128.
// * error-free transforms (two_sum) and double-double accumulation for the
//   compensated partial sums of every walk.
// * 128-bit two's-complement helpers for the exact integer path.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// Bounds-assert build mode (`make debug` -> libpermanent_b200_debug.so,
// -DPERM_DEBUG_BOUNDS): PERM_CHECK traps with the failing condition and its
// source line; compute-sanitizer is closed on this GPU pool, so the debug
// library runs the GPU parity tests instead (tools/debug_bounds_check.sh).
// Compiled out otherwise.
#ifdef PERM_DEBUG_BOUNDS
#define PERM_CHECK(cond)                                                                      \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("PERM_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                              \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define PERM_CHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace permb200 {

struct __align__(16) cd {
  double x, y;
};

__host__ __device__ __forceinline__ cd cd_make(double x, double y) { cd r; r.x = x; r.y = y; return r; }
__host__ __device__ __forceinline__ cd operator+(cd a, cd b) { return cd_make(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cd operator-(cd a, cd b) { return cd_make(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cd cmul(cd a, cd b) {
  // 2 DMUL + 2 DFMA: the (6n-2)-op complex step of SURVEY 8(d)
  return cd_make(fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ cd cfma_s(double s, cd u, cd v) {  // v + s*u, s = +-1
  return cd_make(fma(s, u.x, v.x), fma(s, u.y, v.y));
}

// ---- scalar traits so one walk template serves f64 and c128 -------------
template <typename T> struct Num;
template <> struct Num<double> {
  static constexpr int kDoubles = 1;
  __device__ __forceinline__ static double zero() { return 0.0; }
  __device__ __forceinline__ static double one() { return 1.0; }
  __device__ __forceinline__ static double mul(double a, double b) { return a * b; }
  __device__ __forceinline__ static double add(double a, double b) { return a + b; }
  __device__ __forceinline__ static double sub(double a, double b) { return a - b; }
  __device__ __forceinline__ static double fmas(double s, double u, double v) { return fma(s, u, v); }
  __device__ __forceinline__ static double scale(double w, double p) { return w * p; }
  __device__ __forceinline__ static double absval(double a) { return fabs(a); }
  __device__ __forceinline__ static double re(double a) { return a; }
  __device__ __forceinline__ static double im(double) { return 0.0; }
};
template <> struct Num<cd> {
  static constexpr int kDoubles = 2;
  __device__ __forceinline__ static cd zero() { return cd_make(0.0, 0.0); }
  __device__ __forceinline__ static cd one() { return cd_make(1.0, 0.0); }
  __device__ __forceinline__ static cd mul(cd a, cd b) { return cmul(a, b); }
  __device__ __forceinline__ static cd add(cd a, cd b) { return a + b; }
  __device__ __forceinline__ static cd sub(cd a, cd b) { return a - b; }
  __device__ __forceinline__ static cd fmas(double s, cd u, cd v) { return cfma_s(s, u, v); }
  __device__ __forceinline__ static cd scale(double w, cd p) { return cd_make(w * p.x, w * p.y); }
  __device__ __forceinline__ static double absval(cd a) { return hypot(a.x, a.y); }
  __device__ __forceinline__ static double re(cd a) { return a.x; }
  __device__ __forceinline__ static double im(cd a) { return a.y; }
};

// ---- compensated summation ----------------------------------------------
struct dd { double hi, lo; };

__host__ __device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
// (hi, lo) += x
__host__ __device__ __forceinline__ void dd_acc(double& hi, double& lo, double x) {
  double s, e;
  two_sum(hi, x, s, e);
  hi = s;
  lo += e;
}
// (ah, al) += (bh, bl), renormalized
__host__ __device__ __forceinline__ void dd_add(double& ah, double& al, double bh, double bl) {
  double s, e;
  two_sum(ah, bh, s, e);
  e += al + bl;
  ah = s + e;
  al = e - (ah - s);
}

// ---- balanced product of a register array (compile-time length) --------
// A pairwise tree keeps the dependency depth at log2(P) so the FP64 pipe sees
// P/2 independent multiplies per level instead of one serial chain.
template <typename T, int P>
__device__ __forceinline__ T tree_product(const T (&v)[P]) {
  if constexpr (P == 1) {
    return v[0];
  } else {
    constexpr int H = (P + 1) / 2;
    T t[H];
#pragma unroll
    for (int i = 0; i < P / 2; ++i) t[i] = Num<T>::mul(v[2 * i], v[2 * i + 1]);
    if constexpr (P & 1) t[H - 1] = v[P - 1];
    return tree_product<T, H>(t);
  }
}

// ---- 128-bit two's complement (exact integer path) ----------------------
struct i128 { uint64_t lo, hi; };

__host__ __device__ __forceinline__ i128 i128_from(int64_t x) {
  i128 r; r.lo = (uint64_t)x; r.hi = (x < 0) ? ~0ull : 0ull; return r;
}
__device__ __forceinline__ i128 i128_add(i128 a, i128 b) {
  i128 r;
  asm("add.cc.u64 %0, %2, %4;\n\taddc.u64 %1, %3, %5;"
      : "=l"(r.lo), "=l"(r.hi) : "l"(a.lo), "l"(a.hi), "l"(b.lo), "l"(b.hi));
  return r;
}
__device__ __forceinline__ i128 i128_sub(i128 a, i128 b) {
  i128 r;
  asm("sub.cc.u64 %0, %2, %4;\n\tsubc.u64 %1, %3, %5;"
      : "=l"(r.lo), "=l"(r.hi) : "l"(a.lo), "l"(a.hi), "l"(b.lo), "l"(b.hi));
  return r;
}
// (a * c) mod 2^128 for signed 64-bit c
__device__ __forceinline__ i128 i128_mul_s64(i128 a, int64_t c) {
  uint64_t uc = (uint64_t)c;
  i128 r;
  r.lo = a.lo * uc;
  r.hi = __umul64hi(a.lo, uc) + a.hi * uc - ((c < 0) ? a.lo : 0ull);
  return r;
}
// (a * b) mod 2^128
__device__ __forceinline__ i128 i128_mul(i128 a, i128 b) {
  i128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
__device__ __forceinline__ bool i128_fits_i64(i128 a) { return a.hi == (uint64_t)((int64_t)a.lo >> 63); }
__device__ __forceinline__ bool i128_lt(i128 a, i128 b) {  // signed
  if (a.hi != b.hi) return (int64_t)a.hi < (int64_t)b.hi;
  return a.lo < b.lo;
}

}  // namespace permb200
