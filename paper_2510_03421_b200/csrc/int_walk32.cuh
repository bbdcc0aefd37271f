// Exact int128 WRAP walk for small integer entries on the FP32 / integer
// pipes (round 2; the exact path of src/_kernels.py:148-218 ryser_sq_int and
// :412-523 glynn_sq_int with unbounded intermediates).
//
// The FP64-exact walk (int_walk.cuh) issues ~67 FP64 + ~70 integer
// instructions per Gray step and holds 64+ state registers.  When the state
// entries can be cut into QUADS of four whose products of per-entry bounds
// stay < 2^23, everything below the quad level is exact in FP32:
//   * the state is NQ*4 floats held as packed pairs; one step's update is
//     NQ*2 add.f32x2 (two entries per instruction);
//   * quad products are a two-level packed tree: 3 mul.f32x2 per 8 entries;
//   * each |quad| becomes a 24-bit integer by the 2^23 magic add, and the
//     quads are multiplied as unsigned integers: 24x24 -> 48 (one IMAD.WIDE),
//     48x48 -> 96 (4 IMAD), 96x96 -> mod 2^128 (8 IMAD);
//   * the term's sign is the sign bit of the FP32 product of the quads (a
//     2^-s pre-scale keeps that product inside FP32's range), which is also
//     the per-term estimate of the int128 fit certificate: it is summed in
//     FP64 (F2F + DADD on the otherwise idle FP64 pipe) with its magnitude.
// About 100 issue slots per step instead of ~137, a third of the registers.
#pragma once
#include "int_walk.cuh"

namespace permb200 {

constexpr int kInt32MaxQuads = 10;  // state length <= 40
struct IntWalk32Args {
  const float* v0;  // [4 NQ] exact integers, pad entries 1
  const float* U;   // [B][4 NQ] exact integers, pad entries 0
  // row 0 of U (flipped every other step), read as uniform-register operands.  (Rows 1 and 2 as
  // parameters too: ptxas runs out of uniform registers, hoists them into vector registers, 164 regs.)
  float2 row0[2 * kInt32MaxQuads];
  int B, log2L;
  float escale;     // 2^-s applied to the estimate product
  uint64_t k_begin, nchunks;
  int64_t* out;     // [blocks][8]: int128 sum, dd estimate (scaled), magnitude (scaled)
};

// Packed pairs through the sm_100 float2 intrinsics (FADD2 / FMUL2 / FFMA2):
// unlike inline PTX they let ptxas take an operand from the uniform
// registers / the constant bank (row 0 of U arrives as a kernel parameter),
// which spares the vector register file's read ports -- the quad walk is
// bound by instruction dispatch, not by a pipe.
using f32x2 = float2;

__device__ __forceinline__ f32x2 f2_add(f32x2 a, f32x2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ f32x2 f2_sub(f32x2 a, f32x2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ f32x2 f2_mul(f32x2 a, f32x2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ f32x2 f2_fma(f32x2 a, f32x2 b, f32x2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ f32x2 f2_pack(float lo, float hi) { return make_float2(lo, hi); }
__device__ __forceinline__ void f2_unpack(f32x2 a, float& lo, float& hi) {
  lo = a.x;
  hi = a.y;
}

// |x| of an exact FP32 integer below 2^23 as uint32: 2^23 + |x| lies in
// [2^23, 2^24), where the ulp is 1, so its mantissa field is |x| (the host
// certifies every quad's bound product < 2^23, kQuadBoundLog2).
__device__ __forceinline__ uint32_t quad_mag(float x) {
  return (uint32_t)__float_as_int(fabsf(x) + 8388608.0f) & 0x7fffffu;
}

struct u96 {
  uint32_t w0, w1, w2;
};
struct u128w {
  uint32_t w0, w1, w2, w3;
};

__device__ __forceinline__ uint32_t lo32(uint64_t x) { return (uint32_t)x; }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }

// a, b < 2^48 -> a b < 2^96 as three words (here a, b < 2^46: two quads)
__device__ __forceinline__ u96 mul48(uint64_t a, uint64_t b) {
  const uint32_t al = lo32(a), ah = hi32(a), bl = lo32(b), bh = hi32(b);
  const uint64_t t0 = (uint64_t)al * bl;
  const uint64_t t1 = (uint64_t)ah * bl + hi32(t0);
  const uint64_t t2 = (uint64_t)al * bh + lo32(t1);
  u96 r;
  r.w0 = lo32(t0);
  r.w1 = lo32(t2);
  r.w2 = ah * bh + hi32(t1) + hi32(t2);
  return r;
}

// (A B) mod 2^128, A and B below 2^96
__device__ __forceinline__ u128w mul96(const u96& A, const u96& B) {
  u128w c;
  const uint64_t t = (uint64_t)A.w0 * B.w0;
  c.w0 = lo32(t);
  const uint64_t u = (uint64_t)A.w0 * B.w1 + hi32(t);
  const uint64_t v = (uint64_t)A.w1 * B.w0 + lo32(u);
  c.w1 = lo32(v);
  const uint64_t x1 = (uint64_t)A.w0 * B.w2 + hi32(u);
  const uint64_t x2 = (uint64_t)A.w1 * B.w1 + hi32(v);
  const uint64_t x3 = (uint64_t)A.w2 * B.w0 + lo32(x1);
  const uint64_t s = (uint64_t)lo32(x3) + lo32(x2);
  c.w2 = lo32(s);
  uint32_t k = hi32(s) + hi32(x1) + hi32(x2) + hi32(x3);
  k = A.w1 * B.w2 + k;
  k = A.w2 * B.w1 + k;
  c.w3 = k;
  return c;
}

// (C r) mod 2^128, r < 2^48
__device__ __forceinline__ u128w mul128x48(const u128w& C, uint64_t r) {
  const uint32_t rl = lo32(r), rh = hi32(r);
  u128w d;
  uint64_t t = (uint64_t)C.w0 * rl;
  d.w0 = lo32(t);
  t = (uint64_t)C.w1 * rl + hi32(t);
  uint32_t d1 = lo32(t);
  t = (uint64_t)C.w2 * rl + hi32(t);
  uint32_t d2 = lo32(t);
  uint32_t d3 = C.w3 * rl + hi32(t);
  t = (uint64_t)C.w0 * rh + d1;
  d.w1 = lo32(t);
  t = (uint64_t)C.w1 * rh + d2 + hi32(t);
  d.w2 = lo32(t);
  d.w3 = C.w2 * rh + d3 + hi32(t);
  return d;
}

__device__ __forceinline__ u128w widen(const u96& a) {
  u128w c;
  c.w0 = a.w0; c.w1 = a.w1; c.w2 = a.w2; c.w3 = 0;
  return c;
}
__device__ __forceinline__ u96 widen48(uint64_t r) {
  u96 a;
  a.w0 = lo32(r); a.w1 = hi32(r); a.w2 = 0;
  return a;
}

// |term| mod 2^128 from the NQ quad magnitudes
template <int NQ>
__device__ __forceinline__ u128w term_mag(const uint32_t (&q)[NQ]) {
  constexpr int NR = (NQ + 1) / 2;
  uint64_t r[NR];
#pragma unroll
  for (int i = 0; i < NQ / 2; ++i) r[i] = (uint64_t)q[2 * i] * q[2 * i + 1];
  if constexpr (NQ & 1) r[NR - 1] = q[NQ - 1];
  if constexpr (NR == 1) {
    return widen(widen48(r[0]));
  } else if constexpr (NR == 2) {
    return widen(mul48(r[0], r[1]));
  } else if constexpr (NR == 3) {
    return mul128x48(widen(mul48(r[0], r[1])), r[2]);
  } else {
    u128w p = mul96(mul48(r[0], r[1]), mul48(r[2], r[3]));
#pragma unroll
    for (int i = 4; i < NR; ++i) p = mul128x48(p, r[i]);
    return p;
  }
}

// acc += (-1)^neg sign(e) |term|: conditional two's-complement negate fused
// into the 128-bit add (x ^ m) + (m & 1)
__device__ __forceinline__ void acc_signed(uint32_t (&acc)[4], const u128w& p, uint32_t m) {
  const uint32_t x0 = p.w0 ^ m, x1 = p.w1 ^ m, x2 = p.w2 ^ m, x3 = p.w3 ^ m;
  [[maybe_unused]] uint32_t scratch;
  // m + m carries out exactly when m = 0xffffffff: the +1 of the negation
  asm("add.cc.u32 %4, %9, %9;\n\t"
      "addc.cc.u32 %0, %0, %5;\n\t"
      "addc.cc.u32 %1, %1, %6;\n\t"
      "addc.cc.u32 %2, %2, %7;\n\t"
      "addc.u32 %3, %3, %8;"
      : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "=r"(scratch)
      : "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(m));
}

// ---- FP64 upper levels (DL4) --------------------------------------------
// The FP64 pipe is idle in this walk, while the 32x32 -> 64 integer multiplies
// of the upper product levels saturate the heavy FMA pipe (ncu: IMAD.WIDE is
// 4 cycles there).  With the quads converted to double, a pair of quads
// r = q q' (|r| < 2^46) is one exact DMUL, and the product of two such r
// (|a b| < 2^83, certified by the host) comes out of three more FP64
// operations as an exact (high, low) split at 2^32, rounding DOWN:
//   t  = fma_rd(a, b, 1.5 2^84)      mantissa of t = 2^51 + H, H = floor(a b / 2^32)
//   e  = fma(a, b, -(t - 1.5 2^84))  exact remainder, 0 <= e < 2^32
// so a b = H 2^32 + e with H in two's complement: the words of the signed
// 128-bit product need one integer subtract and one shift.  The term's sign
// (the other pair products' signs and the (-1)^k of the step) is moved into
// `a` beforehand, so the 128-bit accumulate is a plain add.
struct s128w {
  uint32_t w0, w1, w2, w3;  // two's complement, w3 = sign extension of w2
};
template <bool NEG>
__device__ __forceinline__ s128w dmul96s(double a, double b) {
  const double M = 0x1.8p84;
  const double t = NEG ? __fma_rd(-a, b, M) : __fma_rd(a, b, M);
  const double ph = __dadd_rn(t, -M);
  const double e = NEG ? __fma_rn(-a, b, -ph) : __fma_rn(a, b, -ph);
  const long long eb = __double_as_longlong(__dadd_rn(e, 0x1p52));
  const long long tb = __double_as_longlong(t);
  s128w r;
  r.w0 = (uint32_t)eb;
  r.w1 = (uint32_t)tb;
  r.w2 = (uint32_t)(tb >> 32) - 0x45380000u;
  r.w3 = (uint32_t)((int32_t)r.w2 >> 31);
  return r;
}
// |a b| < 2^84 as three words (unsigned operand of the last product)
__device__ __forceinline__ u96 dmul96(double a, double b) {
  const double M = 0x1p84;
  const double aa = fabs(a), bb = fabs(b);
  const double t = __fma_rd(aa, bb, M);
  const double ph = __dadd_rn(t, -M);
  const double e = __fma_rn(aa, bb, -ph);
  const long long eb = __double_as_longlong(__dadd_rn(e, 0x1p52));
  const long long tb = __double_as_longlong(t);
  u96 r;
  r.w0 = (uint32_t)eb;
  r.w1 = (uint32_t)tb;
  r.w2 = (uint32_t)(tb >> 32) - 0x45300000u;
  return r;
}
// |x| < 2^46, an exact integer -> uint64
__device__ __forceinline__ uint64_t dmag48(double x) {
  return (uint64_t)__double_as_longlong(__dadd_rn(fabs(x), 0x1p52)) & 0xfffffffffffffull;
}
// x with its sign flipped when s is negative
__device__ __forceinline__ double flip_sign(double x, double s) {
  const int hi = __double2hiint(x) ^ (__double2hiint(s) & (int)0x80000000);
  return __hiloint2double(hi, __double2loint(x));
}
// (A B) mod 2^128 for a signed A (two's complement, |A| < 2^96) and B < 2^96:
// mul96 on A's words plus the sign word's product (-B 2^96 when A < 0)
__device__ __forceinline__ u128w mul96s(const s128w& A, const u96& B) {
  u96 a;
  a.w0 = A.w0; a.w1 = A.w1; a.w2 = A.w2;
  u128w c = mul96(a, B);
  c.w3 = A.w3 * B.w0 + c.w3;
  return c;
}

// The signed term (-1)^NEG prod(quads) mod 2^128 from the quads as doubles;
// f = the FP64 product of the pair products (the term's estimate, unsigned by NEG)
template <int NQ, bool NEG>
__device__ __forceinline__ u128w term_signed_d(const double (&qd)[NQ], double& f) {
  constexpr int NR = (NQ + 1) / 2;
  double r[NR];
#pragma unroll
  for (int i = 0; i < NQ / 2; ++i) r[i] = __dmul_rn(qd[2 * i], qd[2 * i + 1]);
  if constexpr (NQ & 1) r[NR - 1] = qd[NQ - 1];
  u128w p;
  if constexpr (NR == 1) {
    f = r[0];
    const long long x = NEG ? -__double2ll_rn(r[0]) : __double2ll_rn(r[0]);
    p.w0 = (uint32_t)x; p.w1 = (uint32_t)(x >> 32); p.w2 = p.w3 = (uint32_t)(x >> 63);
  } else if constexpr (NR == 2) {
    f = __dmul_rn(r[0], r[1]);
    const s128w A = dmul96s<NEG>(r[0], r[1]);
    p.w0 = A.w0; p.w1 = A.w1; p.w2 = A.w2; p.w3 = A.w3;
  } else {
    // rest = the product of the other pair products: its sign moves into r[0]
    double rest;
    if constexpr (NR == 3) rest = r[2];
    if constexpr (NR == 4) rest = __dmul_rn(r[2], r[3]);
    if constexpr (NR == 5) rest = __dmul_rn(__dmul_rn(r[2], r[3]), r[4]);
    f = __dmul_rn(__dmul_rn(r[0], r[1]), rest);
    const s128w A = dmul96s<NEG>(flip_sign(r[0], rest), r[1]);
    if constexpr (NR == 3) {
      u128w a;
      a.w0 = A.w0; a.w1 = A.w1; a.w2 = A.w2; a.w3 = A.w3;
      p = mul128x48(a, dmag48(r[2]));
    } else {
      p = mul96s(A, dmul96(r[2], r[3]));
      if constexpr (NR == 5) p = mul128x48(p, dmag48(r[4]));
    }
  }
  return p;
}

__device__ __forceinline__ void acc_add(uint32_t (&acc)[4], const u128w& p) {
  asm("add.cc.u32 %0, %0, %4;\n\t"
      "addc.cc.u32 %1, %1, %5;\n\t"
      "addc.cc.u32 %2, %2, %6;\n\t"
      "addc.u32 %3, %3, %7;"
      : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3])
      : "r"(p.w0), "r"(p.w1), "r"(p.w2), "r"(p.w3));
}

// State: NQ quads = 2 NQ packed pairs.  Full octs (8 entries, 4 packed regs
// v[4o..4o+3]) give the packed pair of quads (v[4o] v[4o+2]) (v[4o+1]
// v[4o+3]): quad 2o holds entries 8o + {0,2,4,6}, quad 2o+1 entries 8o +
// {1,3,5,7}.  An odd last quad (2 packed regs) multiplies its two halves.
template <int NQ, bool DL4>
struct Walk32 {
  static constexpr int NP = 2 * NQ;   // packed registers
  static constexpr int NO = NQ / 2;   // full octs

  // Rows are read with volatile shared loads: plain loads of the loop-
  // invariant rows 1 and 2 get hoisted out of the 8-step loop and spill
  // (the same ptxas behaviour as in walk.cuh).  Row 0 lives in registers.
  struct Pair2 {
    f32x2 x, y;
  };
  static __device__ __forceinline__ Pair2 lds2(const f32x2* p) {
    Pair2 u;
    asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(u.x.x), "=f"(u.x.y), "=f"(u.y.x), "=f"(u.y.y)
                 : "r"((unsigned)__cvta_generic_to_shared(p)));
    return u;
  }
  static __device__ __forceinline__ void reg_add(f32x2 (&v)[NP], const f32x2* __restrict__ r) {
#pragma unroll
    for (int j = 0; j < NP; ++j) v[j] = f2_add(v[j], r[j]);
  }
  static __device__ __forceinline__ void reg_sub(f32x2 (&v)[NP], const f32x2* __restrict__ r) {
#pragma unroll
    for (int j = 0; j < NP; ++j) v[j] = f2_sub(v[j], r[j]);
  }
  static __device__ __forceinline__ void row_add(f32x2 (&v)[NP], const f32x2* __restrict__ row) {
#pragma unroll
    for (int j = 0; j < NP; j += 2) {
      const Pair2 u = lds2(row + j);
      v[j] = f2_add(v[j], u.x);
      v[j + 1] = f2_add(v[j + 1], u.y);
    }
  }
  static __device__ __forceinline__ void row_sub(f32x2 (&v)[NP], const f32x2* __restrict__ row) {
#pragma unroll
    for (int j = 0; j < NP; j += 2) {
      const Pair2 u = lds2(row + j);
      v[j] = f2_sub(v[j], u.x);
      v[j + 1] = f2_sub(v[j + 1], u.y);
    }
  }
  static __device__ __forceinline__ void row_fma(f32x2 (&v)[NP], f32x2 s, const f32x2* __restrict__ row) {
#pragma unroll
    for (int j = 0; j < NP; j += 2) {
      const Pair2 u = lds2(row + j);
      v[j] = f2_fma(s, u.x, v[j]);
      v[j + 1] = f2_fma(s, u.y, v[j + 1]);
    }
  }

  // One term into the int128 accumulator and the FP64 estimate.
  static __device__ __forceinline__ void term(const f32x2 (&v)[NP], bool neg, float escale, uint32_t (&acc)[4],
                                              double& est, double& mag) {
    float qf[NQ];
    if constexpr (DL4) {
#pragma unroll
      for (int o = 0; o < NO; ++o) {
        const f32x2 qq = f2_mul(f2_mul(v[4 * o], v[4 * o + 2]), f2_mul(v[4 * o + 1], v[4 * o + 3]));
        f2_unpack(qq, qf[2 * o], qf[2 * o + 1]);
      }
      if constexpr (NQ & 1) {
        float a, b;
        f2_unpack(f2_mul(v[NP - 2], v[NP - 1]), a, b);
        qf[NQ - 1] = a * b;
      }
      double qd[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) qd[i] = (double)qf[i];
      double d;
      if (neg) {
        acc_add(acc, term_signed_d<NQ, true>(qd, d));
        est -= d;
      } else {
        acc_add(acc, term_signed_d<NQ, false>(qd, d));
        est += d;
      }
      mag += fabs(d);
    } else {
    f32x2 e;  // packed running product of the quad pairs (estimate)
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      const f32x2 qq = f2_mul(f2_mul(v[4 * o], v[4 * o + 2]), f2_mul(v[4 * o + 1], v[4 * o + 3]));
      f2_unpack(qq, qf[2 * o], qf[2 * o + 1]);
      if (o == 0)
        e = f2_mul(qq, f2_pack(escale, 1.0f));
      else
        e = f2_mul(e, qq);
    }
    float f;
    if constexpr (NO > 0) {
      float elo, ehi;
      f2_unpack(e, elo, ehi);
      f = elo * ehi;
    }
    if constexpr (NQ & 1) {
      float a, b;
      f2_unpack(f2_mul(v[NP - 2], v[NP - 1]), a, b);
      qf[NQ - 1] = a * b;
      if constexpr (NO > 0)
        f *= qf[NQ - 1];
      else
        f = qf[NQ - 1] * escale;
    }
    uint32_t q[NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) q[i] = quad_mag(qf[i]);
    const u128w p = term_mag<NQ>(q);
    uint32_t m = (uint32_t)(__float_as_int(f) >> 31);
    if (neg) m = ~m;
    acc_signed(acc, p, m);
    const double d = (double)f;
    est = neg ? est - d : est + d;
    mag += fabs(d);
    }
  }
};

constexpr int kInt32Threads = 128;
#ifndef INT32_MINB
#define INT32_MINB 4
#endif

template <int NQ, bool DL4>
__global__ void __launch_bounds__(kInt32Threads, INT32_MINB) int_walk_wrap_f32_kernel(const __grid_constant__ IntWalk32Args a) {
  using W = Walk32<NQ, DL4>;
  constexpr int NP = W::NP;
  extern __shared__ __align__(16) unsigned char smem_raw32[];
  f32x2* sU = reinterpret_cast<f32x2*>(smem_raw32);  // [B][NP] rows, then v0
  const int B = a.B;
  {
    const f32x2* gU = reinterpret_cast<const f32x2*>(a.U);
    for (int i = threadIdx.x; i < B * NP; i += kInt32Threads) sU[i] = gU[i];
    const f32x2* gv = reinterpret_cast<const f32x2*>(a.v0);
    for (int i = threadIdx.x; i < NP; i += kInt32Threads) sU[B * NP + i] = gv[i];
  }
  __syncthreads();
  const uint64_t nq = (1ull << a.log2L) >> 3;
  const float escale = a.escale;
  uint32_t acc[4] = {0u, 0u, 0u, 0u};
  double hi = 0.0, lo = 0.0, mag = 0.0;
  const f32x2 one2 = f2_pack(1.0f, 1.0f), mone2 = f2_pack(-1.0f, -1.0f);
  const f32x2* r0 = a.row0;  // constant-bank operands
  const uint64_t nthr = (uint64_t)gridDim.x * kInt32Threads;
  for (uint64_t c = (uint64_t)blockIdx.x * kInt32Threads + threadIdx.x; c < a.nchunks; c += nthr) {
    const uint64_t k0 = a.k_begin + (c << a.log2L);
    const uint64_t g0 = k0 ^ (k0 >> 1);
    PERM_CHECK(a.log2L >= 3 && a.log2L <= B && (B >= 63 || (k0 >> B) == 0));
    f32x2 v[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) v[j] = sU[B * NP + j];
    for (int t = 0; t < B; ++t)
      if ((g0 >> t) & 1) W::row_add(v, sU + t * NP);
    double est = 0.0;
    for (uint64_t q = 0; q < nq; ++q) {
      const uint64_t l0 = q << 3;
      if (q) {
        const int t = __ffsll((long long)l0) - 1;
        const uint64_t k = k0 + l0;
        const int set = (int)(((k ^ (k >> 1)) >> t) & 1);
        W::row_fma(v, set ? one2 : mone2, sU + t * NP);
      }
      W::term(v, false, escale, acc, est, mag);
      W::reg_add(v, r0);
      W::term(v, true, escale, acc, est, mag);
      W::row_add(v, sU + NP);
      W::term(v, false, escale, acc, est, mag);
      W::reg_sub(v, r0);
      W::term(v, true, escale, acc, est, mag);
      W::row_fma(v, (((k0 + l0) >> 3) & 1) ? mone2 : one2, sU + 2 * NP);
      W::term(v, false, escale, acc, est, mag);
      W::reg_add(v, r0);
      W::term(v, true, escale, acc, est, mag);
      W::row_sub(v, sU + NP);
      W::term(v, false, escale, acc, est, mag);
      W::reg_sub(v, r0);
      W::term(v, true, escale, acc, est, mag);
    }
    dd_acc(hi, lo, est);
  }
  i128 A;
  A.lo = ((uint64_t)acc[1] << 32) | acc[0];
  A.hi = ((uint64_t)acc[3] << 32) | acc[2];
  for (int off = 16; off > 0; off >>= 1) {
    A = i128_add(A, shfl_down_i128(A, off));
    dd_add(hi, lo, __shfl_down_sync(0xffffffffu, hi, off), __shfl_down_sync(0xffffffffu, lo, off));
    mag += __shfl_down_sync(0xffffffffu, mag, off);
  }
  constexpr int NW = kInt32Threads / 32;
  __shared__ i128 ws[NW];
  __shared__ double wd[NW][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    ws[warp] = A;
    wd[warp][0] = hi; wd[warp][1] = lo; wd[warp][2] = mag;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = ws[0];
    double H = wd[0][0], L = wd[0][1], M = wd[0][2];
    for (int w = 1; w < NW; ++w) {
      t = i128_add(t, ws[w]);
      dd_add(H, L, wd[w][0], wd[w][1]);
      M += wd[w][2];
    }
    int64_t* o = a.out + (size_t)blockIdx.x * 8;
    o[0] = (int64_t)t.lo; o[1] = (int64_t)t.hi;
    o[2] = __double_as_longlong(H); o[3] = __double_as_longlong(L); o[4] = __double_as_longlong(M);
  }
}

using walk_fn_i32 = cudaError_t (*)(const IntWalk32Args&, int blocks, cudaStream_t);
// launcher for NQ quads (nullptr outside 1..kInt32MaxQuads); dl4 = FP64 upper
// levels; *resident = blocks per SM
walk_fn_i32 int_wrap_f32_lookup(int NQ, bool dl4, int* resident);

template <int NQ, bool DL4>
cudaError_t launch_int_wrap_f32(const IntWalk32Args& a, int blocks, cudaStream_t stream) {
  const size_t smem = (size_t)(a.B + 1) * NQ * 4 * sizeof(float);
  auto kern = int_walk_wrap_f32_kernel<NQ, DL4>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<blocks, kInt32Threads, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace permb200
