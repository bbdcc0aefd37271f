// Bulk-pipelined batch kernels: the HBM-streaming form of north_star item 4
// for the two C2 shapes (and every shape the same formulas cover).
//
// Pipeline.  A persistent grid (one CTA per SM) streams the row-major
// [B][m][n] batch through shared memory in tiles of whole matrices with
// `cp.async.bulk` (1-D TMA: one elected thread, completion on an mbarrier),
// kStages tiles in flight per SM, so HBM sees a few hundred KB of
// outstanding reads per SM instead of the 32-thread blocks' per-thread loads.
// Tile t+kStages is issued into slot t % kStages as soon as every thread is
// done reading tile t.  A partial last tile is copied with its exact byte
// count (needs m*n*8 % 16 == 0 and a 16-byte aligned batch; otherwise the
// caller uses the classic kernels in batch.cuh).
//
// Bank conflicts.  Bulk copies land matrices contiguously, so lanes reading
// "their" matrix at the same offset all hit one bank group.  Both formulas
// below are invariant under permuting a matrix's columns (all rows alike) and
// under the row permutations they are symmetric in, so each lane reads its
// matrix with a lane-dependent column rotation / row order instead of
// padding: every LDS.128 of a warp is 4 wavefronts, the minimum.
//
// Formulas (cheaper per matrix than any reference algorithm, exact algebra):
//
//  * Rectangular m <= 6 (C2b 4x10): the Moebius inversion over set partitions
//    of the rows (sum over injective row->column maps =
//    sum_pi mu(pi) prod_{blocks b} p_b,  p_b = sum_j prod_{i in b} a_ij,
//    mu(pi) = prod_b (-1)^(|b|-1) (|b|-1)!):  m = 4 costs (2^m-1-m) muls +
//    (2^m-1) adds per column = 26n + 30 flops (C2b: 290, against 3080 for the
//    reference's cheapest exact algorithm, Ryser-rect).
//    Thread per matrix.
//  * Square 8x8 (C2a): generalised Laplace expansion over the 4+4 row split,
//    per = sum_{|X|=4} per(A[0:4, X]) per(A[4:8, X^c]), with the 4x4 minors
//    built from 2x2 row-pair permanents q(P):
//      per(A[0:4, X]) = sum_{P subset X, |P|=2} q01(P) q23(X \ P).
//    A thread owns one matrix: its 4 x 28 q-tables, the top half's 70 minors
//    parked in shared memory, the bottom half's 70 minors on the complements.
//    1134 flops per matrix against 2048 for Glynn.
#pragma once
#include <utility>
#include "common.cuh"

namespace permb200 {

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned bb_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bb_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bb_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bb_fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bb_fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bb_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb_smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bb_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          bb_smem(dst)),
      "l"(src), "r"(bytes), "r"(bb_smem(bar)), "l"(0x12F0000000000000ull)  // evict-first: streamed once
      : "memory");
}
__device__ __forceinline__ void bb_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bb_smem(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// ------------------------------------------------------------- the pipeline
// Op: static constexpr int kLanes (lanes per matrix);
//     template <class R> static __device__ void run(const T* tile_smem, int64_t first, int count,
//                                                   T* out, int thread_in_tile, R&& release)
//     -- every thread calls release() exactly once, after its last read of tile_smem
template <typename T, int M, int N, int TPB, int STAGES, class Op, bool kComputeOnly = false, int MINB = 1>
__global__ void __launch_bounds__(TPB, MINB) batch_bulk_kernel(const T* __restrict__ a, T* __restrict__ out,
                                                           int64_t nb) {
  constexpr int MATS = TPB / Op::kLanes;
  constexpr unsigned MAT_BYTES = M * N * sizeof(T);
  constexpr unsigned TILE_BYTES = MATS * MAT_BYTES;
  static_assert(MAT_BYTES % 16 == 0, "bulk copies move 16-byte multiples");
  extern __shared__ __align__(128) unsigned char bb_smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES];
  const int64_t ntiles = (nb + MATS - 1) / MATS;
  auto issue = [&](int64_t tile, int slot) {
    const int64_t first = tile * MATS;
    const int64_t cnt = (nb - first < MATS) ? nb - first : MATS;
    const unsigned bytes = (unsigned)cnt * MAT_BYTES;
    bb_expect_tx(&full[slot], bytes);
    bb_bulk_g2s(bb_smem_raw + (size_t)slot * TILE_BYTES, reinterpret_cast<const char*>(a) + first * MAT_BYTES, bytes,
                &full[slot]);
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) bb_mbar_init(&full[s], 1);
    bb_fence_mbar_init();
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  }
  __syncthreads();
  int slot = 0;
  unsigned phase = 0;
  int64_t it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    if (!kComputeOnly || it < STAGES) bb_wait(&full[slot], phase);  // (kComputeOnly: timing experiments)
    const int64_t first = tile * MATS;
    const int cnt = (int)((nb - first < MATS) ? nb - first : MATS);
    // release: called by every thread once it holds what it needs from the
    // slot (before its arithmetic), so the next copy overlaps the compute
    auto release = [&]() {
      __syncthreads();
      if (threadIdx.x == 0 && !kComputeOnly) {
        const int64_t t = tile + (int64_t)STAGES * gridDim.x;
        if (t < ntiles) {
          bb_fence_proxy_async();  // generic-proxy reads before the async-proxy overwrite
          issue(t, slot);
        }
      }
    };
    PERM_CHECK(cnt >= 1 && cnt <= MATS && first + cnt <= nb);
    Op::run(reinterpret_cast<const T*>(bb_smem_raw + (size_t)slot * TILE_BYTES), first, cnt, out, threadIdx.x,
            release);
    if (++slot == STAGES) {
      slot = 0;
      phase ^= 1u;
    }
  }
}

// Per-warp pipelines: every warp streams its own ring of STAGES warp-tiles
// (32 / kLanes matrices each), lane 0 arming the warp's mbarriers and issuing
// its copies, so warps never wait on each other (no block barrier) and the
// warps per SM are set by registers, not by a block-wide tile ring.
template <typename T, int M, int N, int WARPS, int STAGES, class Op, int MINB = 1>
__global__ void __launch_bounds__(32 * WARPS, MINB) batch_bulk_warp_kernel(const T* __restrict__ a, T* __restrict__ out,
                                                                       int64_t nb) {
  constexpr int MATS = 32 / Op::kLanes;
  constexpr unsigned MAT_BYTES = M * N * sizeof(T);
  constexpr unsigned TILE_BYTES = MATS * MAT_BYTES;
  static_assert(MAT_BYTES % 16 == 0, "bulk copies move 16-byte multiples");
  extern __shared__ __align__(128) unsigned char bb_smem_raw[];
  __shared__ __align__(8) uint64_t full[WARPS][STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = bb_smem_raw + (size_t)warp * STAGES * TILE_BYTES;
  uint64_t* bar = full[warp];
  const int64_t ntiles = (nb + MATS - 1) / MATS;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp, nw = (int64_t)gridDim.x * WARPS;
  auto issue = [&](int64_t tile, int slot) {
    const int64_t first = tile * MATS;
    const int64_t cnt = (nb - first < MATS) ? nb - first : MATS;
    const unsigned bytes = (unsigned)cnt * MAT_BYTES;
    bb_expect_tx(&bar[slot], bytes);
    bb_bulk_g2s(ring + (size_t)slot * TILE_BYTES, reinterpret_cast<const char*>(a) + first * MAT_BYTES, bytes,
                &bar[slot]);
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) bb_mbar_init(&bar[s], 1);
    bb_fence_mbar_init();
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const int64_t t = gw + (int64_t)s * nw;
      if (t < ntiles) issue(t, s);
    }
  }
  __syncwarp();
  int slot = 0;
  unsigned phase = 0;
  for (int64_t tile = gw; tile < ntiles; tile += nw) {
    bb_wait(&bar[slot], phase);
    const int64_t first = tile * MATS;
    const int cnt = (int)((nb - first < MATS) ? nb - first : MATS);
    auto release = [&]() {
      __syncwarp();  // the warp is done reading this slot
      if (lane == 0) {
        const int64_t t = tile + (int64_t)STAGES * nw;
        if (t < ntiles) {
          bb_fence_proxy_async();
          issue(t, slot);
        }
      }
    };
    PERM_CHECK(cnt >= 1 && cnt <= MATS && first + cnt <= nb);
    Op::run(reinterpret_cast<const T*>(ring + (size_t)slot * TILE_BYTES), first, cnt, out, lane, release);
    if (++slot == STAGES) {
      slot = 0;
      phase ^= 1u;
    }
  }
}

// ------------------------------------------- rectangular m <= 4: partitions
__host__ __device__ constexpr int bb_hibit(int x) {
  int h = 0;
  while (x >> (h + 1)) ++h;
  return h;
}

// Set partitions of {0..M-1} (M <= 6, Bell(6) = 203) with their Moebius
// coefficients, generated at compile time from restricted growth strings.
struct BbParts {
  int n;
  int nb[256];
  int blk[256][6];
  int coef[256];
};
template <int M>
__host__ __device__ constexpr BbParts bb_parts() {
  BbParts P{};
  int a[6] = {0, 0, 0, 0, 0, 0};
  for (;;) {
    int nb = 0;
    for (int i = 0; i < M; ++i) nb = (a[i] + 1 > nb) ? a[i] + 1 : nb;
    int masks[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < M; ++i) masks[a[i]] |= 1 << i;
    int c = 1;
    for (int b = 0; b < nb; ++b) {
      int sz = 0;
      for (int i = 0; i < M; ++i) sz += (masks[b] >> i) & 1;
      for (int f = 2; f < sz; ++f) c *= f;  // (|b| - 1)!
      if ((sz - 1) & 1) c = -c;
    }
    P.nb[P.n] = nb;
    for (int b = 0; b < 6; ++b) P.blk[P.n][b] = (b < nb) ? masks[b] : 0;
    P.coef[P.n] = c;
    ++P.n;
    int i = M - 1;  // next restricted growth string
    for (; i > 0; --i) {
      int mx = 0;
      for (int j = 0; j < i; ++j) mx = (a[j] > mx) ? a[j] : mx;
      if (a[i] <= mx) {
        ++a[i];
        for (int j = i + 1; j < M; ++j) a[j] = 0;
        break;
      }
    }
    if (i == 0) break;
  }
  return P;
}
template <int M>
struct BbPartsOf {
  static constexpr BbParts value = bb_parts<M>();
};
template <typename T, int M, int Q>
__device__ __forceinline__ T bb_part_term(const T (&S)[1 << M]) {
  using X = Num<T>;
  constexpr int nb = BbPartsOf<M>::value.nb[Q];
  constexpr int c = BbPartsOf<M>::value.coef[Q];
  T prod = S[BbPartsOf<M>::value.blk[Q][0]];
  if constexpr (nb > 1) prod = X::mul(prod, S[BbPartsOf<M>::value.blk[Q][1]]);
  if constexpr (nb > 2) prod = X::mul(prod, S[BbPartsOf<M>::value.blk[Q][2]]);
  if constexpr (nb > 3) prod = X::mul(prod, S[BbPartsOf<M>::value.blk[Q][3]]);
  if constexpr (nb > 4) prod = X::mul(prod, S[BbPartsOf<M>::value.blk[Q][4]]);
  if constexpr (nb > 5) prod = X::mul(prod, S[BbPartsOf<M>::value.blk[Q][5]]);
  return (c == 1) ? prod : X::scale((double)c, prod);
}
template <typename T, int M, int... Qs>
__device__ __forceinline__ T bb_combine_generic(const T (&S)[1 << M], std::integer_sequence<int, Qs...>) {
  T acc[4] = {Num<T>::zero(), Num<T>::zero(), Num<T>::zero(), Num<T>::zero()};
  ((acc[Qs & 3] = Num<T>::add(acc[Qs & 3], bb_part_term<T, M, Qs>(S))), ...);
  return Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3]));
}

// per of an M x N matrix from the subset sums S[b] = sum_j prod_{i in b} a_ij
// (M <= 4 written out with shared sub-products; M = 5, 6 from the table)
template <typename T, int M>
__device__ __forceinline__ T partition_combine(const T (&S)[1 << M]) {
  using X = Num<T>;
  if constexpr (M == 1) {
    return S[1];
  } else if constexpr (M == 2) {
    return X::sub(X::mul(S[1], S[2]), S[3]);
  } else if constexpr (M == 3) {
    // p0p1p2 - p01p2 - p02p1 - p12p0 + 2p012
    T r = X::mul(X::mul(S[1], S[2]), S[4]);
    r = X::sub(r, X::mul(S[3], S[4]));
    r = X::sub(r, X::mul(S[5], S[2]));
    r = X::sub(r, X::mul(S[6], S[1]));
    return X::add(r, X::scale(2.0, S[7]));
  } else if constexpr (M >= 5) {
    return bb_combine_generic<T, M>(S, std::make_integer_sequence<int, BbPartsOf<M>::value.n>{});
  } else {
    // singletons: p0p1p2p3
    const T s01 = X::mul(S[1], S[2]), s23 = X::mul(S[4], S[8]);
    T r = X::mul(s01, s23);
    // {ij}{k}{l}: -6 terms
    T t = X::mul(S[3], s23);                 // {01}{2}{3}
    t = X::add(t, X::mul(S[12], s01));       // {23}{0}{1}
    t = X::add(t, X::mul(S[5], X::mul(S[2], S[8])));   // {02}{1}{3}
    t = X::add(t, X::mul(S[10], X::mul(S[1], S[4])));  // {13}{0}{2}
    t = X::add(t, X::mul(S[9], X::mul(S[2], S[4])));   // {03}{1}{2}
    t = X::add(t, X::mul(S[6], X::mul(S[1], S[8])));   // {12}{0}{3}
    r = X::sub(r, t);
    // {ij}{kl}: +3 terms
    r = X::add(r, X::mul(S[3], S[12]));
    r = X::add(r, X::mul(S[5], S[10]));
    r = X::add(r, X::mul(S[9], S[6]));
    // {ijk}{l}: +2 x 4 terms
    T u = X::mul(S[7], S[8]);
    u = X::add(u, X::mul(S[11], S[4]));
    u = X::add(u, X::mul(S[13], S[2]));
    u = X::add(u, X::mul(S[14], S[1]));
    r = X::add(r, X::scale(2.0, u));
    // {0123}: -6
    return X::sub(r, X::scale(6.0, S[15]));
  }
}

template <typename T, int M, int N>
struct PartitionOp {
  static constexpr int kLanes = 1;
  static_assert(M >= 1 && M <= 6 && M <= N, "m <= 6, m <= n");
  static_assert((N * sizeof(T)) % 16 == 0 || sizeof(T) == 16, "rows read as 16-byte chunks");
  template <class R>
  __device__ __forceinline__ static void run(const T* tile, int64_t first, int cnt, T* out, int me, R&& release) {
    using X = Num<T>;
    constexpr int NS = 1 << M;
    const T* A = tile + (size_t)me * M * N;
    // row order rotated by (lane / 8) % M: the 16-byte chunk a lane reads
    // spreads over all 8 bank groups (4 wavefronts per LDS.128)
    const int tau = ((me & 31) >> 3) % M;
    const T* rowp[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int r = (i + tau) % M;
      rowp[i] = A + r * N;
    }
    T S[NS];
#pragma unroll
    for (int b = 0; b < NS; ++b) S[b] = X::zero();
    constexpr int CW = (sizeof(T) == 8) ? 2 : 1;  // elements per 16-byte chunk
#pragma unroll
    for (int c = 0; c < N / CW; ++c) {
      T col[M][CW];
#pragma unroll
      for (int i = 0; i < M; ++i) {
        if constexpr (CW == 2) {
          const double2 v = *reinterpret_cast<const double2*>(rowp[i] + 2 * c);
          col[i][0] = v.x;
          col[i][1] = v.y;
        } else {
          col[i][0] = rowp[i][c];
        }
      }
#pragma unroll
      for (int e = 0; e < CW; ++e) {
        T p[NS];
#pragma unroll
        for (int i = 0; i < M; ++i) p[1 << i] = col[i][e];
#pragma unroll
        for (int b = 3; b < NS; ++b) {
          if ((b & (b - 1)) == 0) continue;
          const int h = bb_hibit(b);
          p[b] = X::mul(p[b ^ (1 << h)], p[1 << h]);
        }
#pragma unroll
        for (int b = 1; b < NS; ++b) S[b] = X::add(S[b], p[b]);
      }
    }
    release();
    // the row rotation relabels rows; the combine is symmetric in them
    const T r = partition_combine<T, M>(S);
    if (me < cnt) out[first + me] = r;
  }
};

// Wide rectangles (16 < n <= 62, m <= 6): the same partition formula with a
// runtime column count, one thread per matrix reading its rows straight from
// global memory (sequential 8-byte loads through L1: every 32-byte sector a
// thread touches is consumed by its next loads).
template <typename T, int M>
__global__ void __launch_bounds__(128) partition_rt_kernel(const T* __restrict__ a, T* __restrict__ out, int64_t nb,
                                                           int n) {
  using X = Num<T>;
  constexpr int NS = 1 << M;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const T* A = a + i * M * n;
  T S[NS];
#pragma unroll
  for (int b = 0; b < NS; ++b) S[b] = X::zero();
  for (int j = 0; j < n; ++j) {
    T p[NS];
#pragma unroll
    for (int r = 0; r < M; ++r) p[1 << r] = A[r * n + j];
#pragma unroll
    for (int b = 3; b < NS; ++b) {
      if ((b & (b - 1)) == 0) continue;
      const int h = bb_hibit(b);
      p[b] = X::mul(p[b ^ (1 << h)], p[1 << h]);
    }
#pragma unroll
    for (int b = 1; b < NS; ++b) S[b] = X::add(S[b], p[b]);
  }
  out[i] = partition_combine<T, M>(S);
}

// ---------------------------------------------------- square 8x8: Laplace
__host__ __device__ constexpr int lp_pidx(int i, int k) { return i * (15 - i) / 2 + (k - i - 1); }  // i < k < 8
struct LpSub {
  int x[4], c[4];
};
// the p-th 4-subset X of {0..7} containing column 0 (35 of them), and X^c
__host__ __device__ constexpr LpSub lp_sub(int p) {
  LpSub s{};
  int q = 0;
  for (int a = 1; a < 8; ++a)
    for (int b = a + 1; b < 8; ++b)
      for (int c = b + 1; c < 8; ++c) {
        if (q == p) {
          s.x[0] = 0; s.x[1] = a; s.x[2] = b; s.x[3] = c;
          int k = 0;
          for (int j = 1; j < 8; ++j)
            if (j != a && j != b && j != c) s.c[k++] = j;
        }
        ++q;
      }
  return s;
}
// per(H[:, {a,b,c,d}]) of a 4-row half H from its row-pair tables qa (rows
// 0,1) and qb (rows 2,3) is the sum over the 6 ordered splits of {a,b,c,d}
// into two pairs, qa(pair) * qb(other pair): one DMUL + five DFMAs.
// Term s (0..5, the ordered splits (ab|cd) (cd|ab) (ac|bd) (bd|ac) (ad|bc)
// (bc|ad)) of minor slot (pair, side) of the 35 (X, X^c) pairs: the index of
// its qa (which = 0) or qb (which = 1) factor.
__host__ __device__ constexpr int lp_term(int pair, int side, int s, int which) {
  const LpSub q = lp_sub(pair);
  const int a = side ? q.c[0] : q.x[0], b = side ? q.c[1] : q.x[1];
  const int c = side ? q.c[2] : q.x[2], d = side ? q.c[3] : q.x[3];
  // the 6 ordered splits: (ab|cd) (cd|ab) (ac|bd) (bd|ac) (ad|bc) (bc|ad)
  const int p0[6][2] = {{a, b}, {c, d}, {a, c}, {b, d}, {a, d}, {b, c}};
  const int p1[6][2] = {{c, d}, {a, b}, {b, d}, {a, c}, {b, c}, {a, d}};
  return which == 0 ? lp_pidx(p0[s][0], p0[s][1]) : lp_pidx(p1[s][0], p1[s][1]);
}
// 2x2 row-pair permanents of the 8 logical columns held as 16 doubles (row r0 = v[0..7], r1 = v[8..15])
__device__ __forceinline__ void lp_qtable(const double (&v)[16], double (&q)[28]) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int k = i + 1; k < 8; ++k) q[lp_pidx(i, k)] = fma(v[i], v[8 + k], v[k] * v[8 + i]);
}


// Thread per matrix: the top half's 70 minors go to the thread's column of a
// shared-memory buffer (conflict-free: consecutive threads, consecutive
// words), then the bottom half's minors on the complements consume them --
// no shuffles or selects.  Minors are built G at a time, term-major, so each
// warp issues runs of G independent DFMAs.  The matrix is read with a
// lane-dependent column rotation (pairs of columns, rho) and a swap of the
// two rows of each 128-byte row (t): per is invariant under both, and every
// LDS.128 of a warp is 4 wavefronts.
template <int TPB, int G>
struct Laplace8TOp {
  static constexpr int kLanes = 1;
  // term T of minor slot X (X = 2*pair + side; FLIP: the complement's minor)
  template <int T, int FLIP, int X0, int... Ms>
  __device__ __forceinline__ static void term(const double (&qa)[28], const double (&qb)[28], double (&g)[sizeof...(Ms)],
                                              std::integer_sequence<int, Ms...>) {
    if constexpr (T == 0) {
      ((g[Ms] = qa[lp_term((X0 + Ms) >> 1, ((X0 + Ms) & 1) ^ FLIP, 0, 0)] *
                qb[lp_term((X0 + Ms) >> 1, ((X0 + Ms) & 1) ^ FLIP, 0, 1)]),
       ...);
    } else {
      ((g[Ms] = fma(qa[lp_term((X0 + Ms) >> 1, ((X0 + Ms) & 1) ^ FLIP, T, 0)],
                    qb[lp_term((X0 + Ms) >> 1, ((X0 + Ms) & 1) ^ FLIP, T, 1)], g[Ms])),
       ...);
    }
  }
  template <int FLIP, int X0, int... Ms>
  __device__ __forceinline__ static void minors(const double (&qa)[28], const double (&qb)[28],
                                                double (&g)[sizeof...(Ms)], std::integer_sequence<int, Ms...> seq) {
    term<0, FLIP, X0>(qa, qb, g, seq);
    term<1, FLIP, X0>(qa, qb, g, seq);
    term<2, FLIP, X0>(qa, qb, g, seq);
    term<3, FLIP, X0>(qa, qb, g, seq);
    term<4, FLIP, X0>(qa, qb, g, seq);
    term<5, FLIP, X0>(qa, qb, g, seq);
  }
  template <int X0, int... Ms>
  __device__ __forceinline__ static void minors_store(const double (&qa)[28], const double (&qb)[28], double* gcol,
                                                      std::integer_sequence<int, Ms...> seq) {
    double g[sizeof...(Ms)];
    minors<0, X0>(qa, qb, g, seq);
    ((gcol[(X0 + Ms) * TPB] = g[Ms]), ...);
  }
  template <int X0, int... Ms>
  __device__ __forceinline__ static void minors_use(const double (&qc)[28], const double (&qd)[28], const double* gcol,
                                                    double (&acc)[8], std::integer_sequence<int, Ms...> seq) {
    double h[sizeof...(Ms)];
    minors<1, X0>(qc, qd, h, seq);
    ((acc[Ms & 7] = fma(gcol[(X0 + Ms) * TPB], h[Ms], acc[Ms & 7])), ...);
  }
  template <int... Ks>
  __device__ __forceinline__ static void all_store(const double (&qa)[28], const double (&qb)[28], double* gcol,
                                                   std::integer_sequence<int, Ks...>) {
    (minors_store<Ks * G>(qa, qb, gcol, std::make_integer_sequence<int, (70 - Ks * G < G) ? 70 - Ks * G : G>{}), ...);
  }
  template <int... Ks>
  __device__ __forceinline__ static void all_use(const double (&qc)[28], const double (&qd)[28], const double* gcol,
                                                 double (&acc)[8], std::integer_sequence<int, Ks...>) {
    (minors_use<Ks * G>(qc, qd, gcol, acc, std::make_integer_sequence<int, (70 - Ks * G < G) ? 70 - Ks * G : G>{}),
     ...);
  }
  __device__ __forceinline__ static void load_q(const double2* H, int rho, int t, double (&q)[28]) {
    double v[16];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double2 x = H[(((c & 3) + rho) & 3) | (((c >> 2) ^ t) << 2)];
      v[(c >> 2) * 8 + 2 * (c & 3)] = x.x;
      v[(c >> 2) * 8 + 2 * (c & 3) + 1] = x.y;
    }
    lp_qtable(v, q);
  }
  template <class R>
  __device__ __forceinline__ static void run(const double* tile, int64_t first, int cnt, double* out, int me,
                                             R&& release) {
    __shared__ double gbuf[70 * TPB];
    const int lane = me & 31;
    const int rho = lane & 3, t = (lane >> 2) & 1;
    const double2* M = reinterpret_cast<const double2*>(tile + (size_t)me * 64);
    double* gcol = gbuf + me;
    {
      double qa[28], qb[28];
      load_q(M, rho, t, qa);
      load_q(M + 8, rho, t, qb);
      all_store(qa, qb, gcol, std::make_integer_sequence<int, (70 + G - 1) / G>{});
    }
    double qc[28], qd[28];
    load_q(M + 16, rho, t, qc);
    load_q(M + 24, rho, t, qd);
    release();
    double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    all_use(qc, qd, gcol, acc, std::make_integer_sequence<int, (70 + G - 1) / G>{});
    const double r = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    if (me < cnt) out[first + me] = r;
  }
};

  // 4 steps = 16 minors per group

// 32 threads (matrices) per block, 7 minors per group: C2a 0.115 ms
using Laplace8Op = Laplace8TOp<32, 7>;

}  // namespace permb200
