// Gray-code walk engine: the FP64 / complex128 Glynn and Ryser kernels.
//
// One template covers every floating-point enumeration kernel of the
// reference (src/_kernels.py = /root/reference/pkg/src/permanent/_kernels.py):
//
//   Glynn square      glynn_sq    :373-409   P = n, B = n-1, v0 = column sums,
//                                            U[t] = -2 * row(n-1-t), term (-1)^k
//   Glynn rectangular glynn_rect  :531-577   same on the ones-padded n x n matrix
//                                            (real rows pre-scaled by a power of two)
//   Ryser square      ryser_sq    :115-145   P = n, B = n, v0 = 0, U[t] = column t,
//                                            term (-1)^k, per = (-1)^n * sum
//   Ryser rectangular ryser_rect  :226-262   P = m, B = n, all 2^n subsets, term
//                                            w[popcount(gray(k))] * prod
//
// State after Gray index k: v = v0 + sum_{t : bit t of gray(k)} U[t]; step k
// flips Gray bit t = ctz(k) (v += U[t] if the bit becomes set, else -=).
//
// Work decomposition.  The index space [k_begin, k_begin+steps)
// is cut into chunks of L = 2^r consecutive indices; lane `l` of warp-group g
// owns chunk 32*g + l, so the 32 chunks of a warp are adjacent.  Inside a
// chunk every lane performs the *same* flip schedule (Gray bit ctz(local
// index), same direction) -- the only lane-dependent step is local index L/2,
// whose direction is bit 0 of the chunk number -- so every U[t] read is a
// warp-uniform shared-memory broadcast and the steps are unrolled by 8 with
// compile-time flip rows t = 0, 1, 0, 2, 0, 1, 0.  Seeding a chunk costs
// ~B/64 column sums per lane (warp-cooperative) plus <= 6 row FMAs.
//
// Accumulation: a plain FP64 sum over each chunk (<= L terms), folded into a
// per-thread double-double with two_sum; double-double warp-shuffle and block
// reductions; one partial (hi, lo) per block, combined in fixed block order
// by the last block to finish -> deterministic for a given launch shape.
#pragma once
#include "common.cuh"

namespace permb200 {

#ifndef WALK_THREADS
#define WALK_THREADS 256
#endif
constexpr int kWalkThreads = WALK_THREADS;
constexpr int kWalkWarps = kWalkThreads / 32;
constexpr int kPartialStride = 8;  // doubles per block partial: hi, lo, im_hi, im_lo, mag, -, -, -

struct WalkArgs {
  const void* v0;        // [P] T
  const void* U;         // [B][P] T
  const double* w;       // [wlen] popcount weights (weighted walks only)
  int B;                 // Gray bits
  int log2L;             // chunk length exponent (>= 3)
  int wlen;              // number of weights
  int mag;               // also accumulate sum |term| (metric (ii) scale)
  uint64_t k_begin;      // first Gray index, multiple of 32*L
  uint64_t ngroups;      // number of 32-chunk groups
  double* partials;      // [gridDim.x][kPartialStride]
  double* final_out;     // 8 doubles: fixed-order sum of all block partials (device or mapped host)
  unsigned int* done;    // block-completion counter (0 on entry, reset on exit)
  unsigned int* flag;    // optional mapped host flag, set to seq once final_out is written
  unsigned int seq;
};

// Last-block-done combine: every block publishes its partial, the block that
// arrives last sums all partials in block order (deterministic for a given
// grid) and writes the final 8 doubles -- no separate finalize launch.
// `flag` (optional, mapped host memory): after final_out -- then also host
// memory -- is written, a system-scope fence and flag = seq, so the caller
// can spin on the flag instead of a device-to-host copy and a stream sync.
__device__ __forceinline__ void walk_last_block_combine(const double* partials, double* final_out,
                                                        unsigned int* done, unsigned int* flag = nullptr,
                                                        unsigned int seq = 0) {
  __shared__ bool last;
  PERM_CHECK(gridDim.x <= (unsigned)(148 * 16));  // kMaxPartials partial slots
  if (threadIdx.x == 0) {
    __threadfence();
    last = (atomicAdd(done, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int tid = threadIdx.x;
  double h = 0, l = 0, h2 = 0, l2 = 0, mg = 0;
  for (int i = tid; i < (int)gridDim.x; i += blockDim.x) {
    const volatile double* p = partials + (size_t)i * kPartialStride;
    dd_add(h, l, p[0], p[1]);
    dd_add(h2, l2, p[2], p[3]);
    mg += p[4];
  }
  __shared__ double red[32][5];
  // fixed-order tree over the block: shuffles then warp leaders
  for (int off = 16; off > 0; off >>= 1) {
    dd_add(h, l, __shfl_down_sync(0xffffffffu, h, off), __shfl_down_sync(0xffffffffu, l, off));
    dd_add(h2, l2, __shfl_down_sync(0xffffffffu, h2, off), __shfl_down_sync(0xffffffffu, l2, off));
    mg += __shfl_down_sync(0xffffffffu, mg, off);
  }
  if ((tid & 31) == 0) {
    red[tid >> 5][0] = h; red[tid >> 5][1] = l; red[tid >> 5][2] = h2; red[tid >> 5][3] = l2; red[tid >> 5][4] = mg;
  }
  __syncthreads();
  if (tid == 0) {
    double H = red[0][0], Lo = red[0][1], H2 = red[0][2], L2 = red[0][3], M = red[0][4];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      dd_add(H, Lo, red[w][0], red[w][1]);
      dd_add(H2, L2, red[w][2], red[w][3]);
      M += red[w][4];
    }
    final_out[0] = H; final_out[1] = Lo; final_out[2] = H2; final_out[3] = L2; final_out[4] = M;
    final_out[5] = 0.0; final_out[6] = 0.0; final_out[7] = 0.0;
    *done = 0u;  // ready for the next launch on this scratch
    if (flag) {  // release at system scope: final_out (this thread's stores) first
#ifdef WALK_FLAG_FENCE
      __threadfence_system();
      *reinterpret_cast<volatile unsigned int*>(flag) = seq;
#else
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(seq) : "memory");
#endif
    }
  }
}

// Shared-memory reads of U rows go through `asm volatile` 128-bit loads on
// purpose: with plain loads NVVM hoists every row read of the 8 unrolled
// steps to the top of the block (the rows are loop-invariant), keeping ~8
// rows live and spilling at P >= 20; C++ `volatile` stops that but splits
// each pair into two LDS.64, which saturated the LSU pipe (ncu: 85% LSU next
// to 86% FP64).  One LDS.128 per pair of doubles / per complex element, and
// a warp-uniform address is a single broadcast wavefront.
#ifndef WALK_LDS
#define WALK_LDS 1
#endif
__device__ __forceinline__ double2 lds2(const void* p) {
#if WALK_LDS == 0
  const volatile double* q = static_cast<const volatile double*>(p);
  double2 r;
  r.x = q[0];
  r.y = q[1];
  return r;
#else
  double2 r;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(a));
  return r;
#endif
}
__device__ __forceinline__ double lds1(const void* p) {
  double r;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(r) : "r"(a));
  return r;
}

template <typename T>
__device__ __forceinline__ T ld_row(const T* row, int j) {
  if constexpr (sizeof(T) == 16) {
    const double2 u = lds2(row + j);
    return cd_make(u.x, u.y);
  } else {
    return lds1(row + j);
  }
}

template <typename T, int P>
__device__ __forceinline__ void row_add(T (&v)[P], const T* __restrict__ row) {
  if constexpr (sizeof(T) == 8 && P >= 2) {
#pragma unroll
    for (int j = 0; j < P / 2; ++j) {
      const double2 u = lds2(row + 2 * j);
      v[2 * j] = Num<T>::add(v[2 * j], u.x);
      v[2 * j + 1] = Num<T>::add(v[2 * j + 1], u.y);
    }
    if constexpr (P & 1) v[P - 1] = Num<T>::add(v[P - 1], ld_row<T>(row, P - 1));
  } else {
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = Num<T>::add(v[j], ld_row<T>(row, j));
  }
}

template <typename T, int P>
__device__ __forceinline__ void row_sub(T (&v)[P], const T* __restrict__ row) {
  if constexpr (sizeof(T) == 8 && P >= 2) {
#pragma unroll
    for (int j = 0; j < P / 2; ++j) {
      const double2 u = lds2(row + 2 * j);
      v[2 * j] = Num<T>::sub(v[2 * j], u.x);
      v[2 * j + 1] = Num<T>::sub(v[2 * j + 1], u.y);
    }
    if constexpr (P & 1) v[P - 1] = Num<T>::sub(v[P - 1], ld_row<T>(row, P - 1));
  } else {
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = Num<T>::sub(v[j], ld_row<T>(row, j));
  }
}

template <typename T, int P>
__device__ __forceinline__ void row_fma(T (&v)[P], double s, const T* __restrict__ row) {
  if constexpr (sizeof(T) == 8 && P >= 2) {
#pragma unroll
    for (int j = 0; j < P / 2; ++j) {
      const double2 u = lds2(row + 2 * j);
      v[2 * j] = Num<T>::fmas(s, u.x, v[2 * j]);
      v[2 * j + 1] = Num<T>::fmas(s, u.y, v[2 * j + 1]);
    }
    if constexpr (P & 1) v[P - 1] = Num<T>::fmas(s, ld_row<T>(row, P - 1), v[P - 1]);
  } else {
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = Num<T>::fmas(s, ld_row<T>(row, j), v[j]);
  }
}

// Row stride (elements) of U in shared memory: even for doubles so a row
// starts 16-byte aligned and can be read with LDS.128.
template <typename T, int P>
__host__ __device__ constexpr int row_stride() { return (sizeof(T) == 8) ? ((P + 1) & ~1) : P; }

// Product of the state vector with kChains interleaved multiply chains: depth
// P/kChains, only kChains temporaries live (a full pairwise tree keeps P/2
// extra values live and spills at P >= 20).
#ifndef WALK_CHAINS
#define WALK_CHAINS 4
#endif
constexpr int kChains = WALK_CHAINS;
// Per-state-length chain count from a measured sweep on B200
// (tools/walk_csweep.cu, profiles/r1_walk_r0_sweep.txt).  With U[0] in
// registers (walk_r0) 4 chains are within 1% of the best everywhere except
// P = 25, 43, 44 (6 chains: +5 / +7 / +6%); WALK_CHAINS (default 4) elsewhere.
template <typename T, int P>
__host__ __device__ constexpr bool walk_r0();
template <typename T, int P>
__host__ __device__ constexpr int walk_chains() {
#ifdef WALK_CHAINS_FIXED
  return kChains;
#else
  if constexpr (sizeof(T) == 8) {
    if (walk_r0<T, P>()) return (P == 25 || P == 43 || P == 44) ? 6 : kChains;
    return kChains;
  } else {
    return P == 22 ? 6 : kChains;
  }
#endif
}
#ifndef WALK_FUSED
#define WALK_FUSED 1
#endif
// U[0] -- the row flipped at every other step -- held in registers for real
// walks whose state leaves room (P real state + P row registers under the
// 255 cap, one 256-thread block per SM).  Measured (tools/walk_p36.cu,
// tools/walk_csweep.cu -> profiles/r1_walk_r0_sweep.txt): P = 36 Glynn
// 9.70 -> 8.88 ms per 2^31 steps, 86 -> 94% of the FP64 pipe; P = 17..52
// gain 5-25% except P = 24 (-5%).  The limiter was short_scoreboard waits
// on the row loads, not the product chains or occupancy.
template <typename T, int P>
__host__ __device__ constexpr bool walk_r0() {
#ifdef WALK_R0_FORCE_C
  if (sizeof(T) == 16) return WALK_R0_FORCE_C;
#endif
#ifdef WALK_R0_FORCE
  return WALK_R0_FORCE && sizeof(T) == 8;
#else
  return sizeof(T) == 8 && P >= 17 && P <= 52 && P != 24;
#endif
}
#if WALK_FUSED
#define WALK_CHUNK walk_chunk_fused
#else
#define WALK_CHUNK walk_chunk
#endif
template <typename T, int N>
__device__ __forceinline__ T tree_of(const T (&c)[N]) {
  if constexpr (N == 1) {
    return c[0];
  } else {
    constexpr int H = (N + 1) / 2;
    T t[H];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) t[i] = Num<T>::mul(c[2 * i], c[2 * i + 1]);
    if constexpr (N & 1) t[H - 1] = c[N - 1];
    return tree_of<T, H>(t);
  }
}
template <typename T, int P>
__device__ __forceinline__ T chain_product(const T (&v)[P]) {
  constexpr int K = walk_chains<T, P>();
  constexpr int C = (P < K) ? P : K;
  T c[C];
#pragma unroll
  for (int i = 0; i < C; ++i) c[i] = v[i];
#pragma unroll
  for (int j = C; j < P; ++j) c[j % C] = Num<T>::mul(c[j % C], v[j]);
  return tree_of<T, C>(c);
}

// Occupancy target: cap registers so at least 16 warps per SM stay resident
// where the state vector fits (FP64-pipe bound code needs ILP x warps, not
// maximal occupancy); large complex vectors get the whole register file.
template <typename T, int P>
__host__ __device__ constexpr int walk_min_blocks() {
#ifdef WALK_MINB
  return WALK_MINB;
#endif
  if (walk_r0<T, P>()) return 1;
  return (Num<T>::kDoubles == 1) ? ((P <= 20) ? 3 : (P <= 41) ? 2 : 1) : ((P <= 14) ? 2 : 1);
}

template <typename T, int P, bool W, bool MAG>
struct Term {
  // chunk sum, magnitude sum
  __device__ __forceinline__ static void add(const T (&v)[P], int sign, int pc, const double* sW, T& acc,
                                             double& mag) {
    T p = chain_product<T, P>(v);
    if constexpr (W) {
      double wt = sW[pc];
      acc = Num<T>::add(acc, Num<T>::scale(wt, p));
      if constexpr (MAG) mag += fabs(wt) * Num<T>::absval(p);
    } else {
      acc = (sign > 0) ? Num<T>::add(acc, p) : Num<T>::sub(acc, p);
      if constexpr (MAG) mag += Num<T>::absval(p);
    }
  }
};

// Fused step: the term of the current state (sign or popcount weight) and
// the update to the next state, interleaved column by column -- column j
// enters its product chain, then takes its row update -- so each U row pair
// is loaded right where it is consumed and the products of step s overlap
// the shared-memory latency of step s+1's row.  UPD: 0 add, 1 sub, 2 fma(s).
template <typename T, int P, bool W, bool MAG, int UPD>
__device__ __forceinline__ void term_update(T (&v)[P], const T* __restrict__ row, double s, int sign, int pc,
                                            const double* sW, T& acc, double& mag) {
  constexpr int K = walk_chains<T, P>();
  constexpr int C = (P < K) ? P : K;
  T c[C];
  auto upd = [&](T x, T u) -> T {
    if constexpr (UPD == 0) return Num<T>::add(x, u);
    else if constexpr (UPD == 1) return Num<T>::sub(x, u);
    else return Num<T>::fmas(s, u, x);
  };
#pragma unroll
  for (int j = 0; j < P; ++j) {
    T u;
    if constexpr (sizeof(T) == 8) {
      if ((j & 1) == 0 && j + 1 < P) {
        const double2 u2 = lds2(row + j);
        u = u2.x;
        if (j < C) c[j] = v[j]; else c[j % C] = Num<T>::mul(c[j % C], v[j]);
        v[j] = upd(v[j], u);
        if (j + 1 < C) c[j + 1] = v[j + 1]; else c[(j + 1) % C] = Num<T>::mul(c[(j + 1) % C], v[j + 1]);
        v[j + 1] = upd(v[j + 1], u2.y);
        continue;
      }
      if (j & 1) continue;  // consumed with its pair
      u = lds1(row + j);
    } else {
      u = ld_row<T>(row, j);
    }
    if (j < C) c[j] = v[j]; else c[j % C] = Num<T>::mul(c[j % C], v[j]);
    v[j] = upd(v[j], u);
  }
  const T p = tree_of<T, C>(c);
  if constexpr (W) {
    const double wt = sW[pc];
    acc = Num<T>::add(acc, Num<T>::scale(wt, p));
    if constexpr (MAG) mag += fabs(wt) * Num<T>::absval(p);
  } else {
    acc = (sign > 0) ? Num<T>::add(acc, p) : Num<T>::sub(acc, p);
    if constexpr (MAG) mag += Num<T>::absval(p);
  }
}

// term_update with the row held in registers (row 0: half of all steps).
template <typename T, int P, bool W, bool MAG, int UPD>
__device__ __forceinline__ void term_update_reg(T (&v)[P], const T (&row)[P], int sign, int pc, const double* sW,
                                                T& acc, double& mag) {
  constexpr int K = walk_chains<T, P>();
  constexpr int C = (P < K) ? P : K;
  T c[C];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    if (j < C) c[j] = v[j]; else c[j % C] = Num<T>::mul(c[j % C], v[j]);
    v[j] = (UPD == 0) ? Num<T>::add(v[j], row[j]) : Num<T>::sub(v[j], row[j]);
  }
  const T p = tree_of<T, C>(c);
  if constexpr (W) {
    const double wt = sW[pc];
    acc = Num<T>::add(acc, Num<T>::scale(wt, p));
    if constexpr (MAG) mag += fabs(wt) * Num<T>::absval(p);
  } else {
    acc = (sign > 0) ? Num<T>::add(acc, p) : Num<T>::sub(acc, p);
    if constexpr (MAG) mag += Num<T>::absval(p);
  }
}

// walk_chunk_fused with U[0] in registers (u0): the four row-0 steps of
// every eight read no shared memory.
template <typename T, int P, bool W, bool MAG>
__device__ __forceinline__ T walk_chunk_fused_r0(T (&v)[P], const T (&u0)[P], const T* sU, const double* sW,
                                                 uint64_t k0, uint64_t nq, int pc, double& mag) {
  constexpr int PS = row_stride<T, P>();
  T acc = Num<T>::zero();
  for (uint64_t q = 0; q < nq; ++q) {
    term_update_reg<T, P, W, MAG, 0>(v, u0, +1, pc, sW, acc, mag);
    if constexpr (W) ++pc;
    term_update<T, P, W, MAG, 0>(v, sU + PS, 0.0, -1, pc, sW, acc, mag);
    if constexpr (W) ++pc;
    term_update_reg<T, P, W, MAG, 1>(v, u0, +1, pc, sW, acc, mag);
    if constexpr (W) --pc;
    const int b3 = (int)(((k0 + (q << 3)) >> 3) & 1);
    term_update<T, P, W, MAG, 2>(v, sU + 2 * PS, b3 ? -1.0 : 1.0, -1, pc, sW, acc, mag);
    if constexpr (W) pc += b3 ? -1 : 1;
    term_update_reg<T, P, W, MAG, 0>(v, u0, +1, pc, sW, acc, mag);
    if constexpr (W) ++pc;
    term_update<T, P, W, MAG, 1>(v, sU + PS, 0.0, -1, pc, sW, acc, mag);
    if constexpr (W) --pc;
    term_update_reg<T, P, W, MAG, 1>(v, u0, +1, pc, sW, acc, mag);
    if constexpr (W) --pc;
    if (q + 1 < nq) {
      const uint64_t l0 = (q + 1) << 3;
      const int t = __ffsll((long long)l0) - 1;
      const uint64_t k = k0 + l0;
      const int set = (int)(((k ^ (k >> 1)) >> t) & 1);
      term_update<T, P, W, MAG, 2>(v, sU + t * PS, set ? 1.0 : -1.0, -1, pc, sW, acc, mag);
      if constexpr (W) pc += set ? 1 : -1;
    } else {
      Term<T, P, W, MAG>::add(v, -1, pc, sW, acc, mag);
    }
  }
  return acc;
}

template <typename T, int P, bool W, bool MAG>
__device__ __forceinline__ T walk_chunk_fused(T (&v)[P], const T* sU, const double* sW, uint64_t k0, uint64_t nq,
                                              int pc, double& mag) {
  constexpr int PS = row_stride<T, P>();
  T acc = Num<T>::zero();
  for (uint64_t q = 0; q < nq; ++q) {
    // T0+U1(+U0), T1+U2(+U1), T2+U3(-U0), T3+U4(+-U2), T4+U5(+U0), T5+U6(-U1), T6+U7(-U0)
    term_update<T, P, W, MAG, 0>(v, sU, 0.0, +1, pc, sW, acc, mag);
    if constexpr (W) ++pc;
    term_update<T, P, W, MAG, 0>(v, sU + PS, 0.0, -1, pc, sW, acc, mag);
    if constexpr (W) ++pc;
    term_update<T, P, W, MAG, 1>(v, sU, 0.0, +1, pc, sW, acc, mag);
    if constexpr (W) --pc;
    const int b3 = (int)(((k0 + (q << 3)) >> 3) & 1);  // U4: bit 2 set iff bit 3 of k0+8q clear
    term_update<T, P, W, MAG, 2>(v, sU + 2 * PS, b3 ? -1.0 : 1.0, -1, pc, sW, acc, mag);
    if constexpr (W) pc += b3 ? -1 : 1;
    term_update<T, P, W, MAG, 0>(v, sU, 0.0, +1, pc, sW, acc, mag);
    if constexpr (W) ++pc;
    term_update<T, P, W, MAG, 1>(v, sU + PS, 0.0, -1, pc, sW, acc, mag);
    if constexpr (W) --pc;
    term_update<T, P, W, MAG, 1>(v, sU, 0.0, +1, pc, sW, acc, mag);
    if constexpr (W) --pc;
    if (q + 1 < nq) {  // T7 + the runtime row update that opens the next 8 steps
      const uint64_t l0 = (q + 1) << 3;
      const int t = __ffsll((long long)l0) - 1;
      const uint64_t k = k0 + l0;
      const int set = (int)(((k ^ (k >> 1)) >> t) & 1);
      term_update<T, P, W, MAG, 2>(v, sU + t * PS, set ? 1.0 : -1.0, -1, pc, sW, acc, mag);
      if constexpr (W) pc += set ? 1 : -1;
    } else {
      Term<T, P, W, MAG>::add(v, -1, pc, sW, acc, mag);
    }
  }
  return acc;
}

// The 8-step unrolled walk over one chunk of nq*8 indices starting at k0
// (state v already seeded): every flip row but one per 8 steps is a
// compile-time row of U (t = 0, 1, 0, 2, 0, 1, 0).
template <typename T, int P, bool W, bool MAG>
__device__ __forceinline__ T walk_chunk(T (&v)[P], const T* sU, const double* sW, uint64_t k0, uint64_t nq, int pc,
                                        double& mag) {
  constexpr int PS = row_stride<T, P>();
  using Tm = Term<T, P, W, MAG>;
  T acc = Num<T>::zero();
  for (uint64_t q = 0; q < nq; ++q) {
    const uint64_t l0 = q << 3;
    if (q) {
      const int t = __ffsll((long long)l0) - 1;
      const uint64_t k = k0 + l0;
      const int set = (int)(((k ^ (k >> 1)) >> t) & 1);
      row_fma<T, P>(v, set ? 1.0 : -1.0, sU + t * PS);
      if constexpr (W) pc += set ? 1 : -1;
    }
    Tm::add(v, +1, pc, sW, acc, mag);
    row_add<T, P>(v, sU);  // l = 1: bit 0 set
    if constexpr (W) ++pc;
    Tm::add(v, -1, pc, sW, acc, mag);
    row_add<T, P>(v, sU + PS);  // l = 2: bit 1 set
    if constexpr (W) ++pc;
    Tm::add(v, +1, pc, sW, acc, mag);
    row_sub<T, P>(v, sU);  // l = 3: bit 0 cleared
    if constexpr (W) --pc;
    Tm::add(v, -1, pc, sW, acc, mag);
    {  // l = 4: bit 2 toggles; set iff bit 3 of (k0 + l0) is clear
      const int b3 = (int)(((k0 + l0) >> 3) & 1);
      row_fma<T, P>(v, b3 ? -1.0 : 1.0, sU + 2 * PS);
      if constexpr (W) pc += b3 ? -1 : 1;
    }
    Tm::add(v, +1, pc, sW, acc, mag);
    row_add<T, P>(v, sU);  // l = 5: bit 0 set
    if constexpr (W) ++pc;
    Tm::add(v, -1, pc, sW, acc, mag);
    row_sub<T, P>(v, sU + PS);  // l = 6: bit 1 cleared
    if constexpr (W) --pc;
    Tm::add(v, +1, pc, sW, acc, mag);
    row_sub<T, P>(v, sU);  // l = 7: bit 0 cleared
    if constexpr (W) --pc;
    Tm::add(v, -1, pc, sW, acc, mag);
  }
  return acc;
}

// Partial sums of one thread: double-double real / imaginary parts and the
// magnitude sum.
struct WalkAcc {
  double hi = 0.0, lo = 0.0, hi_i = 0.0, lo_i = 0.0, mag = 0.0;
};

template <typename T, int P>
using WalkRow0 = T[walk_r0<T, P>() ? P : 1];

// The walk over warp-groups g = g_first, g_first + g_stride, ... < g_end of
// one setup staged in shared memory (sU: B rows, sV0, this warp's seed row
// myWarp): group g is 32 chunks of L = 2^log2L indices starting at
// k_begin + g * 32 * L, lane l owns chunk l of the group.
template <typename T, int P, bool W>
__device__ __forceinline__ void walk_group_range(const T* sU, const T* sV0, T* myWarp, const double* sW,
                                                 const WalkRow0<T, P>& u0, int B, int log2L, uint64_t k_begin,
                                                 uint64_t g_first, uint64_t g_end, uint64_t g_stride, int mag_on,
                                                 WalkAcc& A) {
  constexpr int PS = row_stride<T, P>();
  const int lane = threadIdx.x & 31;
  const uint64_t L = 1ull << log2L;
  const uint64_t nq = L >> 3;
  const uint64_t bmask = (B >= 64) ? ~0ull : ((1ull << B) - 1);
  const uint64_t hmask = (~0ull << (log2L + 5)) & bmask;  // warp-uniform Gray bits
  PERM_CHECK(log2L >= 3 && log2L <= B);  // in-chunk flip rows ctz(l) < log2L must be rows of U
  for (uint64_t g = g_first; g < g_end; g += g_stride) {
    const uint64_t kb = k_begin + ((g * 32) << log2L);
    const uint64_t k0 = kb + ((uint64_t)lane << log2L);
    // ---- warp-cooperative seed of the bits shared by the 32 chunks
    {
      const uint64_t gb = (kb ^ (kb >> 1)) & hmask;
      for (int j = lane; j < P; j += 32) {
        T acc = sV0[j];
        uint64_t bits = gb;
        while (bits) {
          int t = __ffsll((long long)bits) - 1;
          bits &= bits - 1;
          PERM_CHECK(t < B);
          acc = Num<T>::add(acc, sU[t * PS + j]);
        }
        myWarp[j] = acc;
      }
    }
    __syncwarp();
    T v[P];
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = myWarp[j];
    __syncwarp();
    const uint64_t g0 = k0 ^ (k0 >> 1);
    // ---- lane-dependent Gray bits: positions log2L-1 .. log2L+4
#pragma unroll
    for (int d = -1; d <= 4; ++d) {
      const int b = log2L + d;
      if (b < B) {
        const double s = (double)((g0 >> b) & 1);
        row_fma<T, P>(v, s, sU + b * PS);
      }
    }
    const int pc = __popcll(g0);
    T acc;
    if constexpr (walk_r0<T, P>()) {
      acc = mag_on ? walk_chunk_fused_r0<T, P, W, true>(v, u0, sU, sW, k0, nq, pc, A.mag)
                   : walk_chunk_fused_r0<T, P, W, false>(v, u0, sU, sW, k0, nq, pc, A.mag);
    } else {
      acc = mag_on ? WALK_CHUNK<T, P, W, true>(v, sU, sW, k0, nq, pc, A.mag)
                   : WALK_CHUNK<T, P, W, false>(v, sU, sW, k0, nq, pc, A.mag);
    }
    dd_acc(A.hi, A.lo, Num<T>::re(acc));
    if constexpr (sizeof(T) == 16) dd_acc(A.hi_i, A.lo_i, Num<T>::im(acc));
  }
}

// Deterministic block reduction (warp shuffles, then warp leaders in order);
// thread 0 writes {hi, lo, im_hi, im_lo, mag} to out.
template <bool CPLX>
__device__ __forceinline__ void walk_block_reduce(WalkAcc A, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double h2 = __shfl_down_sync(0xffffffffu, A.hi, off), l2 = __shfl_down_sync(0xffffffffu, A.lo, off);
    dd_add(A.hi, A.lo, h2, l2);
    if constexpr (CPLX) {
      double h3 = __shfl_down_sync(0xffffffffu, A.hi_i, off), l3 = __shfl_down_sync(0xffffffffu, A.lo_i, off);
      dd_add(A.hi_i, A.lo_i, h3, l3);
    }
    A.mag += __shfl_down_sync(0xffffffffu, A.mag, off);
  }
  __shared__ double red[kWalkWarps][5];
  if (lane == 0) {
    red[warp][0] = A.hi; red[warp][1] = A.lo; red[warp][2] = A.hi_i; red[warp][3] = A.lo_i; red[warp][4] = A.mag;
  }
  __syncthreads();
  // warp leaders combined by warp 0 with a 3-level shuffle tree (a serial
  // loop on one thread was ~0.3 us of dependent double-double adds)
  if (warp == 0) {
    double H = 0.0, Lo = 0.0, H2 = 0.0, L2 = 0.0, M = 0.0;
    if (lane < kWalkWarps) {
      H = red[lane][0]; Lo = red[lane][1]; H2 = red[lane][2]; L2 = red[lane][3]; M = red[lane][4];
    }
#pragma unroll
    for (int off = kWalkWarps / 2; off > 0; off >>= 1) {
      double h = __shfl_down_sync(0xffffffffu, H, off), l = __shfl_down_sync(0xffffffffu, Lo, off);
      dd_add(H, Lo, h, l);
      if constexpr (CPLX) {
        double h3 = __shfl_down_sync(0xffffffffu, H2, off), l3 = __shfl_down_sync(0xffffffffu, L2, off);
        dd_add(H2, L2, h3, l3);
      }
      M += __shfl_down_sync(0xffffffffu, M, off);
    }
    if (lane == 0) {
      out[0] = H; out[1] = Lo; out[2] = H2; out[3] = L2; out[4] = M;
    }
  }
}

// Setup passed by value in the launch (kernel parameters, <= 32 KB) for the
// small walks, where a staged host-to-device copy costs as much as the walk:
// [v0 (P) | U (B x P)], B <= P, unpadded (WalkSetup::buf's layout).
// Doubles of the inline blob: [v0 | U | w] with B <= P rows (unweighted) or
// B <= 62 rows and <= 63 popcount weights (weighted rectangular Ryser).
__host__ __device__ constexpr int walk_inline_doubles(int P, int kD, bool W) {
  return W ? 63 * P * kD + 64 : (P + 1) * P * kD;
}
template <typename T, int P, bool W>
struct WalkInline {
  alignas(16) double d[walk_inline_doubles(P, Num<T>::kDoubles, W)];
};
// The kernel's second parameter: the inline setup, or nothing.  (WalkArgs
// stays a separate by-value parameter: folded into one __grid_constant__
// struct its fields were read per thread, and the chunk loop's bookkeeping
// left the uniform datapath -- 6% slower at n = 32..36.)
template <typename T, int P, bool W, bool INL>
struct WalkBlob {
  int unused;
};
template <typename T, int P, bool W>
struct WalkBlob<T, P, W, true> : WalkInline<T, P, W> {};

// Timeline probe (tools/small_walk_exp.cu builds with -DWALK_TIMELINE):
// %globaltimer of thread 0 of every block at each phase boundary.
#ifdef WALK_TIMELINE
__device__ unsigned long long* g_walk_tl;
#define WALK_TL(i)                                                  \
  do {                                                               \
    if (threadIdx.x == 0 && g_walk_tl) {                             \
      unsigned long long t_;                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));         \
      g_walk_tl[blockIdx.x * 8 + (i)] = t_;                          \
    }                                                                \
  } while (0)
#else
#define WALK_TL(i) \
  do {             \
  } while (0)
#endif

// Stage [v0 | U] (contiguous, inline or in device memory) into shared memory
// in batches of 4 independent loads per thread before their stores: one load
// latency per batch instead of one per element (a plain loop serialized them).
template <typename T, int P>
__device__ __forceinline__ void walk_stage(const T* __restrict__ src, int B, T* sU, T* sV0) {
  constexpr int PS = row_stride<T, P>();
  const int total = (B + 1) * P;
  for (int base = 0; base < total; base += 4 * kWalkThreads) {
    T r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = base + k * kWalkThreads + (int)threadIdx.x;
      if (e < total) r[k] = src[e];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = base + k * kWalkThreads + (int)threadIdx.x;
      if (e < P) sV0[e] = r[k];
      else if (e < total) {
        PERM_CHECK(e / P - 1 < B);
        sU[(e / P - 1) * PS + (e % P)] = r[k];
      }
    }
  }
}

template <typename T, int P, bool W, bool INL>
__global__ void __launch_bounds__(kWalkThreads, walk_min_blocks<T, P>())
    walk_kernel(WalkArgs args, const __grid_constant__ WalkBlob<T, P, W, INL> blob) {
  constexpr int PS = row_stride<T, P>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sU = reinterpret_cast<T*>(smem_raw);        // [B][PS]
  T* sV0 = sU + (size_t)args.B * PS;              // [PS]
  T* sWarp = sV0 + PS;                            // [kWalkWarps][PS]
  double* sW = reinterpret_cast<double*>(sWarp + kWalkWarps * PS);  // [wlen]

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int B = args.B;
  WALK_TL(0);
  if constexpr (INL) walk_stage<T, P>(reinterpret_cast<const T*>(blob.d), B, sU, sV0);
  else walk_stage<T, P>(static_cast<const T*>(args.v0), B, sU, sV0);
  if constexpr (W) {
    const double* w = args.w;
    if constexpr (INL) w = blob.d + (size_t)(B + 1) * P * Num<T>::kDoubles;
    for (int i = tid; i < args.wlen; i += kWalkThreads) sW[i] = w[i];
  }
  __syncthreads();

  WalkRow0<T, P> u0;
  if constexpr (walk_r0<T, P>()) {
#pragma unroll
    for (int j = 0; j < P; ++j) u0[j] = sU[j];
  }
  WALK_TL(1);
  WalkAcc A;
  walk_group_range<T, P, W>(sU, sV0, sWarp + warp * PS, sW, u0, B, args.log2L, args.k_begin,
                            (uint64_t)blockIdx.x * kWalkWarps + warp, args.ngroups,
                            (uint64_t)gridDim.x * kWalkWarps, args.mag, A);
  WALK_TL(2);
  walk_block_reduce<sizeof(T) == 16>(A, args.partials + (size_t)blockIdx.x * kPartialStride);
  WALK_TL(3);
  walk_last_block_combine(args.partials, args.final_out, args.done, args.flag, args.seq);
  WALK_TL(4);
}

// Many square Glynn permanents in one launch (batches of n = 17..30): work
// item w = (matrix w / segs, segment w % segs); each block builds its
// matrix's walk setup (v0 = column sums, U[t] = -2 row(n-1-t)) in shared
// memory straight from the [B][n][n] batch, walks its segment's groups,
// writes a block partial, and the last segment of a matrix to finish
// (per-matrix counter) combines its segments in order -> out[matrix].
struct WalkMultiArgs {
  const void* a;          // [nmats][m][P] row-major, device
  void* out;              // [nmats] permanents
  double* partials;       // [nmats * segs][kPartialStride]
  unsigned int* done;     // [nmats], zero on entry, reset on exit
  int64_t nmats;
  int m;                  // rows (m < P: rectangular Glynn on [2^s A; J])
  int segs, log2L;
  uint64_t groups_per_seg;
  double scale;           // 2^-(n-1) / (n-m)!
};

template <typename T, int P>
__global__ void __launch_bounds__(kWalkThreads, walk_min_blocks<T, P>()) walk_multi_kernel(WalkMultiArgs args) {
  constexpr int PS = row_stride<T, P>();
  constexpr int B = P - 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sU = reinterpret_cast<T*>(smem_raw);  // [B][PS]
  T* sV0 = sU + (size_t)B * PS;             // [PS]
  T* sWarp = sV0 + PS;                      // [kWalkWarps][PS]
  __shared__ bool last;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t items = args.nmats * args.segs;
  for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
    const int64_t mat = w / args.segs;
    const int seg = (int)(w - mat * args.segs);
    PERM_CHECK(mat < args.nmats && seg < args.segs);
    const int m = args.m;
    const T* A = static_cast<const T*>(args.a) + mat * m * P;
    __syncthreads();  // previous item's shared memory is free
    // rectangular: ones rows below the m real rows, which are pre-scaled by
    // 2^s, s = round(-log2 RMS of the nonzero entries) (as prescale_log2)
    int sl = 0;
    if (m < P) {
      double ss = 0.0;
      int nz = 0;
      for (int i = tid; i < m * P; i += kWalkThreads) {
        const double q = Num<T>::re(A[i]) * Num<T>::re(A[i]) + Num<T>::im(A[i]) * Num<T>::im(A[i]);
        if (q != 0.0) {
          ss += q;
          ++nz;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        ss += __shfl_down_sync(0xffffffffu, ss, off);
        nz += __shfl_down_sync(0xffffffffu, nz, off);
      }
      __shared__ double red_ss[kWalkWarps];
      __shared__ int red_nz[kWalkWarps];
      if ((tid & 31) == 0) {
        red_ss[warp] = ss;
        red_nz[warp] = nz;
      }
      __syncthreads();
      double S = 0.0;
      int Z = 0;
      for (int w2 = 0; w2 < kWalkWarps; ++w2) {
        S += red_ss[w2];
        Z += red_nz[w2];
      }
      if (Z > 0 && S > 0.0) {
        const double e = -0.5 * log2(S / Z);
        if (isfinite(e)) sl = (int)rint(e);
      }
    }
    const double k = ldexp(1.0, sl);
    for (int i = tid; i < B * P; i += kWalkThreads) {
      const int t = i / P, j = i - t * P;
      const int row = P - 1 - t;
      sU[t * PS + j] = (row < m) ? Num<T>::scale(-2.0 * k, A[row * P + j]) : Num<T>::scale(-2.0, Num<T>::one());
    }
    for (int j = tid; j < P; j += kWalkThreads) {
      T c = Num<T>::zero();
      for (int i = 0; i < m; ++i) c = Num<T>::add(c, A[i * P + j]);
      sV0[j] = Num<T>::add(Num<T>::scale(k, c), Num<T>::scale((double)(P - m), Num<T>::one()));
    }
    __syncthreads();
    WalkRow0<T, P> u0;
    if constexpr (walk_r0<T, P>()) {
#pragma unroll
      for (int j = 0; j < P; ++j) u0[j] = sU[j];
    }
    WalkAcc acc;
    const uint64_t g0 = (uint64_t)seg * args.groups_per_seg;
    walk_group_range<T, P, false>(sU, sV0, sWarp + warp * PS, nullptr, u0, B, args.log2L, 0, g0 + warp,
                                  g0 + args.groups_per_seg, kWalkWarps, 0, acc);
    double* part = args.partials + (size_t)w * kPartialStride;
    walk_block_reduce<sizeof(T) == 16>(acc, part);
    if (tid == 0) {
      __threadfence();
      last = (atomicAdd(&args.done[mat], 1u) == (unsigned)args.segs - 1);
    }
    __syncthreads();
    if (last && tid == 0) {
      __threadfence();
      const volatile double* p = args.partials + (size_t)mat * args.segs * kPartialStride;
      double H = p[0], Lo = p[1], H2 = p[2], L2 = p[3];
      for (int s = 1; s < args.segs; ++s) {
        dd_add(H, Lo, p[s * kPartialStride], p[s * kPartialStride + 1]);
        dd_add(H2, L2, p[s * kPartialStride + 2], p[s * kPartialStride + 3]);
      }
      // 2^(-s m) applied with ldexp on the value (the factor alone can
      // underflow where the permanent does not)
      T r;
      if constexpr (sizeof(T) == 16)
        r = cd_make(ldexp((H + Lo) * args.scale, -sl * m), ldexp((H2 + L2) * args.scale, -sl * m));
      else r = ldexp((H + Lo) * args.scale, -sl * m);
      static_cast<T*>(args.out)[mat] = r;
      args.done[mat] = 0u;
    }
  }
}

// One warp over a short range (< 256 steps: Glynn n <= 8, Ryser n <= 7) with
// the setup as kernel parameters and the result published through mapped
// memory (final_out, flag): the zero-copy single-permanent path below the
// chunked kernel's minimum.  Lane l walks [k_begin + l s / 32, ...) from its
// own seed (v0 + the rows of its Gray code), fixed-order warp reduction.
template <typename T, int P, bool W>
__global__ void __launch_bounds__(32) walk_tiny_kernel(WalkArgs args, const __grid_constant__ WalkBlob<T, P, W, true> blob,
                                                       uint64_t k_end) {
  const int lane = threadIdx.x;
  const T* v0 = reinterpret_cast<const T*>(blob.d);
  const T* U = v0 + P;
  const double* w = blob.d + (size_t)(args.B + 1) * P * Num<T>::kDoubles;
  const uint64_t steps = k_end - args.k_begin;
  const uint64_t k0 = args.k_begin + steps * lane / 32, k1 = args.k_begin + steps * (lane + 1) / 32;
  T v[P];
  const uint64_t g0 = k0 ^ (k0 >> 1);
#pragma unroll
  for (int j = 0; j < P; ++j) v[j] = v0[j];
  PERM_CHECK(args.B <= 62 && (args.B == 0 || k_end <= (1ull << args.B)));
  for (int t = 0; t < args.B; ++t)
    if ((g0 >> t) & 1) {
#pragma unroll
      for (int j = 0; j < P; ++j) v[j] = Num<T>::add(v[j], U[t * P + j]);
    }
  int pc = __popcll(g0);
  T acc = Num<T>::zero();
  double mag = 0.0;
  for (uint64_t k = k0; k < k1; ++k) {
    if (k != k0) {
      const int t = __ffsll((long long)k) - 1;
      const int set = (int)(((k ^ (k >> 1)) >> t) & 1);
      PERM_CHECK(t < args.B);
#pragma unroll
      for (int j = 0; j < P; ++j) v[j] = set ? Num<T>::add(v[j], U[t * P + j]) : Num<T>::sub(v[j], U[t * P + j]);
      pc += set ? 1 : -1;
    }
    const T p = tree_product<T, P>(v);
    if constexpr (W) {
      acc = Num<T>::add(acc, Num<T>::scale(w[pc], p));
      if (args.mag) mag += fabs(w[pc]) * Num<T>::absval(p);
    } else {
      acc = (k & 1) ? Num<T>::sub(acc, p) : Num<T>::add(acc, p);
      if (args.mag) mag += Num<T>::absval(p);
    }
  }
  double h = Num<T>::re(acc), l = 0.0, h2 = Num<T>::im(acc), l2 = 0.0;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    dd_add(h, l, __shfl_down_sync(0xffffffffu, h, off), __shfl_down_sync(0xffffffffu, l, off));
    dd_add(h2, l2, __shfl_down_sync(0xffffffffu, h2, off), __shfl_down_sync(0xffffffffu, l2, off));
    mag += __shfl_down_sync(0xffffffffu, mag, off);
  }
  if (lane == 0) {
    double* o = args.final_out;
    o[0] = h; o[1] = l; o[2] = h2; o[3] = l2; o[4] = mag; o[5] = 0.0; o[6] = 0.0; o[7] = 0.0;
    if (args.flag) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(args.flag), "r"(args.seq) : "memory");
  }
}

// Single-thread walk for tiny index spaces (< 32 chunks of 8): runtime P.
// Same arithmetic as walk_kernel (plain sum per 'chunk' of the whole range).
template <typename T, int P>
__global__ void walk_small_kernel(const T* __restrict__ v0, const T* __restrict__ U, const double* __restrict__ w,
                                  int /*P*/, int B, int weighted, int mag_on, uint64_t k_begin, uint64_t k_end,
                                  double* partials) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  T v[P];
  const uint64_t g0 = k_begin ^ (k_begin >> 1);
  for (int j = 0; j < P; ++j) v[j] = v0[j];
  for (int t = 0; t < B; ++t)
    if ((g0 >> t) & 1)
      for (int j = 0; j < P; ++j) v[j] = Num<T>::add(v[j], U[t * P + j]);
  int pc = __popcll(g0);
  T acc = Num<T>::zero();
  double mag = 0.0;
  for (uint64_t k = k_begin; k < k_end; ++k) {
    if (k != k_begin) {
      const int t = __ffsll((long long)k) - 1;
      const int set = (int)(((k ^ (k >> 1)) >> t) & 1);
      for (int j = 0; j < P; ++j) v[j] = set ? Num<T>::add(v[j], U[t * P + j]) : Num<T>::sub(v[j], U[t * P + j]);
      pc += set ? 1 : -1;
    }
    T p = v[0];
    for (int j = 1; j < P; ++j) p = Num<T>::mul(p, v[j]);
    if (weighted) {
      acc = Num<T>::add(acc, Num<T>::scale(w[pc], p));
      if (mag_on) mag += fabs(w[pc]) * Num<T>::absval(p);
    } else {
      acc = (k & 1) ? Num<T>::sub(acc, p) : Num<T>::add(acc, p);
      if (mag_on) mag += Num<T>::absval(p);
    }
  }
  partials[0] = Num<T>::re(acc); partials[1] = 0.0;
  partials[2] = Num<T>::im(acc); partials[3] = 0.0;
  partials[4] = mag; partials[5] = 0.0; partials[6] = 0.0; partials[7] = 0.0;
}


}  // namespace permb200
