// Double-double Gray walks: the validation kernels of SURVEY 8(c) C5.
//
// FP64 Ryser is useless as a cross-check at n = 36 on the C5 law (its
// magnitude-sum conditioning M_R/|per| is ~1e18); in
// double-double (~2^-104 unit roundoff) it is accurate to ~1e-14, so
// "Glynn (FP64) vs Ryser (double-double, GPU)" validates sizes the reference
// cannot reach.  Same walk as walk.cuh (v0, U, weights from build_walk), but
// the state, every product and the accumulator are double-double; one chunk
// of 2^log2L consecutive indices per thread, grid-stride.  Not timed.
#pragma once
#include "common.cuh"

namespace permb200 {

struct ddn { double hi, lo; };

__device__ __forceinline__ ddn ddn_quick(double a, double b) {
  ddn r;
  r.hi = a + b;
  r.lo = b - (r.hi - a);
  return r;
}
__device__ __forceinline__ ddn ddn_add(ddn a, ddn b) {
  double s, e, t, f;
  two_sum(a.hi, b.hi, s, e);
  two_sum(a.lo, b.lo, t, f);
  e += t;
  ddn r = ddn_quick(s, e);
  r.lo += f;
  return ddn_quick(r.hi, r.lo);
}
__device__ __forceinline__ ddn ddn_add_d(ddn a, double b) {
  double s, e;
  two_sum(a.hi, b, s, e);
  e += a.lo;
  return ddn_quick(s, e);
}
__device__ __forceinline__ ddn ddn_neg(ddn a) { return ddn{-a.hi, -a.lo}; }
__device__ __forceinline__ ddn ddn_mul(ddn a, ddn b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  return ddn_quick(p, e);
}
__device__ __forceinline__ ddn ddn_mul_d(ddn a, double b) {
  const double p = a.hi * b;
  double e = fma(a.hi, b, -p);
  e = fma(a.lo, b, e);
  return ddn_quick(p, e);
}

struct cddn { ddn re, im; };
__device__ __forceinline__ cddn cddn_mul(cddn a, cddn b) {
  return cddn{ddn_add(ddn_mul(a.re, b.re), ddn_neg(ddn_mul(a.im, b.im))),
              ddn_add(ddn_mul(a.re, b.im), ddn_mul(a.im, b.re))};
}

struct WalkDDArgs {
  const double* v0;  // [P] (x2 if complex)
  const double* U;   // [B][P] (x2 if complex)
  const double* w;   // [wlen] or null
  int P, B, log2L, weighted;
  uint64_t k_begin, nchunks;
  double* out;       // per block: re_hi, re_lo, im_hi, im_lo
};

// PMAX: compile-time bound on the state length (register arrays), P <= PMAX.
template <bool CPLX, int PMAX>
__global__ void __launch_bounds__(128) walk_dd_kernel(WalkDDArgs a) {
  constexpr int W = CPLX ? 2 : 1;
  const int P = a.P, B = a.B;
  cddn acc = {{0, 0}, {0, 0}};
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < a.nchunks; c += nthr) {
    const uint64_t k0 = a.k_begin + (c << a.log2L);
    const uint64_t k1 = k0 + (1ull << a.log2L);
    cddn v[PMAX];
    const uint64_t g0 = k0 ^ (k0 >> 1);
#pragma unroll
    for (int j = 0; j < PMAX; ++j) {
      if (j < P) {
        v[j].re = ddn{a.v0[j * W], 0.0};
        v[j].im = ddn{CPLX ? a.v0[j * W + 1] : 0.0, 0.0};
        for (int t = 0; t < B; ++t)
          if ((g0 >> t) & 1) {
            v[j].re = ddn_add_d(v[j].re, a.U[((size_t)t * P + j) * W]);
            if (CPLX) v[j].im = ddn_add_d(v[j].im, a.U[((size_t)t * P + j) * W + 1]);
          }
      }
    }
    int pc = __popcll(g0);
    for (uint64_t k = k0; k < k1; ++k) {
      if (k != k0) {
        const int t = __ffsll((long long)k) - 1;
        const bool set = ((k ^ (k >> 1)) >> t) & 1;
        const double sg = set ? 1.0 : -1.0;
#pragma unroll
        for (int j = 0; j < PMAX; ++j) {
          if (j < P) {
            v[j].re = ddn_add_d(v[j].re, sg * a.U[((size_t)t * P + j) * W]);
            if (CPLX) v[j].im = ddn_add_d(v[j].im, sg * a.U[((size_t)t * P + j) * W + 1]);
          }
        }
        pc += set ? 1 : -1;
      }
      cddn p = v[0];
#pragma unroll
      for (int j = 1; j < PMAX; ++j) {
        if (j < P) {
          if (CPLX) p = cddn_mul(p, v[j]);
          else p.re = ddn_mul(p.re, v[j].re);
        }
      }
      if (a.weighted) {
        const double wt = a.w[pc];
        p.re = ddn_mul_d(p.re, wt);
        p.im = ddn_mul_d(p.im, wt);
      } else if (k & 1) {
        p.re = ddn_neg(p.re);
        p.im = ddn_neg(p.im);
      }
      acc.re = ddn_add(acc.re, p.re);
      if (CPLX) acc.im = ddn_add(acc.im, p.im);
    }
  }
  // block reduction (shuffles, then shared memory), fixed order
  for (int off = 16; off > 0; off >>= 1) {
    ddn o{__shfl_down_sync(0xffffffffu, acc.re.hi, off), __shfl_down_sync(0xffffffffu, acc.re.lo, off)};
    acc.re = ddn_add(acc.re, o);
    ddn q{__shfl_down_sync(0xffffffffu, acc.im.hi, off), __shfl_down_sync(0xffffffffu, acc.im.lo, off)};
    acc.im = ddn_add(acc.im, q);
  }
  __shared__ cddn ws[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) ws[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    cddn t = ws[0];
    for (int i = 1; i < (int)(blockDim.x / 32); ++i) {
      t.re = ddn_add(t.re, ws[i].re);
      t.im = ddn_add(t.im, ws[i].im);
    }
    double* o = a.out + (size_t)blockIdx.x * 4;
    o[0] = t.re.hi; o[1] = t.re.lo; o[2] = t.im.hi; o[3] = t.im.lo;
  }
}

}  // namespace permb200
