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
//  * Square 8x8 (C2a): the row-by-row subset recursion
//    f_L(S) = sum_{j in S} a_{L-1,j} f_{L-1}(S \ {j}), per = f_8({0..7}),
//    1016 flops per matrix against 2048 for Glynn; one thread per matrix,
//    the middle level parked in tensor memory (perm8_tmem_kernel, RowDp8Tm).
//    (The round-1 4+4 Laplace split, 1134 flops, now lives in
//    tools/laplace8_variants.cuh as a measured alternative.)
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

// ---------------------------------------- TMEM as per-thread scratch (8x8)
// A thread-per-matrix 8x8 kernel needs ~1.3 KB of scratch per matrix beyond
// its registers.  In shared memory that scratch plus a 16 KB tile slot per
// stage per warp held the round-1 kernel at 4 warps per SM (one per
// scheduler, FP64 pipe ~60% busy on fixed-latency waits).  Here the scratch
// lives in tensor memory: 256 KB per SM that nothing else on this path uses.
// Lane i of warp w owns TMEM lane 32*(w%4)+i and 256 columns of it
// (tcgen05.st / tcgen05.ld, 32x32b shape: one thread, consecutive 32-bit
// columns).  A thread copies its whole matrix out of the tile at once (rows
// 0..3 -> registers, rows 4..7 -> TMEM), so a warp releases its slot before
// any arithmetic and one stage per warp keeps the copy of its next tile in
// flight during the whole compute.  Shared memory is then just the tile ring,
// 16 KB per warp: 8 warps per SM.
__device__ __forceinline__ uint32_t tm_lo(double x) { return (uint32_t)__double2loint(x); }
__device__ __forceinline__ uint32_t tm_hi(double x) { return (uint32_t)__double2hiint(x); }
__device__ __forceinline__ double tm_pack(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }
#define TM_D2(d, i) "r"(tm_lo(d[i])), "r"(tm_hi(d[i]))
// store D doubles (2D consecutive columns) of this thread's TMEM lane at column address ta
__device__ __forceinline__ void tm_st8(uint32_t ta, const double* d) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      TM_D2(d, 0), TM_D2(d, 1), TM_D2(d, 2), TM_D2(d, 3), TM_D2(d, 4), TM_D2(d, 5), TM_D2(d, 6), TM_D2(d, 7)
      : "memory");
}
__device__ __forceinline__ void tm_st4(uint32_t ta, const double* d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), TM_D2(d, 0),
               TM_D2(d, 1), TM_D2(d, 2), TM_D2(d, 3)
               : "memory");
}
__device__ __forceinline__ void tm_st2(uint32_t ta, const double* d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta), TM_D2(d, 0), TM_D2(d, 1)
               : "memory");
}
#undef TM_D2
__device__ __forceinline__ void tm_ld16(uint32_t ta, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(ta)
               : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t ta, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta)
               : "memory");
}
__device__ __forceinline__ void tm_ld4(uint32_t ta, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(ta)
               : "memory");
}
// tcgen05.wait::ld, tied to the loaded registers so no use is scheduled above it
__device__ __forceinline__ void tm_wait_ld(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Column map of a thread's TMEM lane (one CTA slice of kTmCols columns):
// the parked level (70 doubles, 140 columns) from column 0, in groups of G
// at 2G*k; rows 4..7 as two rotated 16-entry row-pair vectors at kTmRaw.
constexpr int kTmCols = 256, kTmRaw = 144;

// C doubles of this thread's TMEM lane from / to column ta: 8-double chunks, then 4, then 2
template <int C>
__device__ __forceinline__ void tm_st_n(uint32_t ta, const double* g) {
#pragma unroll
  for (int i = 0; i < C / 8; ++i) tm_st8(ta + 16 * i, g + 8 * i);
  if constexpr (C % 8 >= 4) tm_st4(ta + 16 * (C / 8), g + 8 * (C / 8));
  if constexpr (C % 4 >= 2) tm_st2(ta + 16 * (C / 8) + 8 * ((C % 8) / 4), g + 8 * (C / 8) + 4 * ((C % 8) / 4));
  static_assert(C % 2 == 0, "pairs of minors");
}
template <int C>
__device__ __forceinline__ void tm_ld_n(uint32_t ta, uint32_t (&r)[((2 * C + 15) / 16) * 16]) {
  constexpr int F = C / 8;
#pragma unroll
  for (int i = 0; i < F; ++i) tm_ld16(ta + 16 * i, *reinterpret_cast<uint32_t(*)[16]>(r + 16 * i));
  if constexpr (C % 8 != 0) {
#pragma unroll
    for (int i = 16 * F; i < 16 * F + 16; ++i) r[i] = 0u;
    if constexpr (C % 8 >= 4) tm_ld8(ta + 16 * F, r + 16 * F);
    if constexpr (C % 4 >= 2) tm_ld4(ta + 16 * F + 8 * ((C % 8) / 4), r + 16 * F + 8 * ((C % 8) / 4));
  }
}
template <int NR>
__device__ __forceinline__ void tm_wait_ld_n(uint32_t (&r)[NR]) {
  tm_wait_ld(*reinterpret_cast<uint32_t(*)[16]>(r));
#pragma unroll
  for (int i = 1; i < NR / 16; ++i) {  // tie the other chunks behind the wait
    uint32_t(&q)[16] = *reinterpret_cast<uint32_t(*)[16]>(r + 16 * i);
    asm volatile(""
                 : "+r"(q[0]), "+r"(q[1]), "+r"(q[2]), "+r"(q[3]), "+r"(q[4]), "+r"(q[5]), "+r"(q[6]), "+r"(q[7]),
                   "+r"(q[8]), "+r"(q[9]), "+r"(q[10]), "+r"(q[11]), "+r"(q[12]), "+r"(q[13]), "+r"(q[14]), "+r"(q[15]));
  }
}
// the rotated row pair (2p, 2p+1) of a lane's matrix as 16 doubles (row 2p^t in v[0..7])
__device__ __forceinline__ void rd_pair(const double2* M, int p, int rho, int t, double (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double2 x = M[8 * p + ((((c & 3) + rho) & 3) | (((c >> 2) ^ t) << 2))];
    v[(c >> 2) * 8 + 2 * (c & 3)] = x.x;
    v[(c >> 2) * 8 + 2 * (c & 3) + 1] = x.y;
  }
}
__device__ __forceinline__ void tm_ld_pair(uint32_t ta, double (&v)[16]) {
  uint32_t r0[16], r1[16];
  tm_ld16(ta, r0);
  tm_ld16(ta + 16, r1);
  tm_wait_ld(r0);
  tm_wait_ld(r1);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = tm_pack(r0[2 * i], r0[2 * i + 1]);
    v[8 + i] = tm_pack(r1[2 * i], r1[2 * i + 1]);
  }
}

// ------------------------------------------ 8x8 row-by-row subset recursion
// per(A) = f_8({0..7}) with f_1(S) = a_0j (S = {j}) and
//   f_L(S) = sum_{j in S} a_{L-1,j} f_{L-1}(S \ {j})        (|S| = L),
// the permanent of rows 0..L-1 on the columns S.  Level L costs L * C(8, L)
// FP64 ops: 56 + 168 + 280 + 280 + 168 + 56 + 8 = 1016 per matrix for
// levels 2..8, against 1134 for the 4+4 Laplace split (which pays 6 ops per
// 4x4 minor on both halves).  Levels 2, 3 and 6..8 pull from the level below
// in registers; level 4 (70 values) is parked in TMEM while level 5 is built
// by pushing each parked value into the 56 level-5 accumulators (the first
// push to an accumulator is a DMUL, the rest DFMAs), so neither level has to
// be register-resident at the same time as its neighbour.  Subsets of size L
// are ranked by increasing bit mask.
__host__ __device__ constexpr int rd_popc(int m) { return m ? (m & 1) + rd_popc(m >> 1) : 0; }
__host__ __device__ constexpr int rd_mask(int k, int r) {
  int q = 0;
  for (int m = 0; m < 256; ++m)
    if (rd_popc(m) == k) {
      if (q == r) return m;
      ++q;
    }
  return -1;
}
__host__ __device__ constexpr int rd_rank(int m) {
  int q = 0;
  for (int x = 0; x < m; ++x) q += rd_popc(x) == rd_popc(m);
  return q;
}
__host__ __device__ constexpr int rd_bit(int m, int t) {  // t-th set bit of m (t-th clear bit: pass ~m & 255)
  for (int j = 0; j < 8; ++j)
    if ((m >> j) & 1) {
      if (t == 0) return j;
      --t;
    }
  return -1;
}
__host__ __device__ constexpr int rd_first_push(int m) {  // rank of the smallest-rank (|m|-1)-subset of m
  int best = 1 << 20;
  for (int j = 0; j < 8; ++j)
    if ((m >> j) & 1) best = rd_rank(m & ~(1 << j)) < best ? rd_rank(m & ~(1 << j)) : best;
  return best;
}
template <int L, int R, int T>
constexpr int rd_col_v = rd_bit(rd_mask(L, R), T);  // column of term T of entry R of level L
template <int L, int R, int T>
constexpr int rd_src_v = rd_rank(rd_mask(L, R) & ~(1 << rd_bit(rd_mask(L, R), T)));  // its level L-1 entry
// term T of level-L entries R0 + Ms (term-major: runs of independent DFMAs)
template <int L, int R0, int T, int NS, int ND, int... Ms>
__device__ __forceinline__ void rd_term(const double (&src)[NS], const double* row, double (&dst)[ND], int dofs,
                                        std::integer_sequence<int, Ms...>) {
  if constexpr (T == 0)
    ((dst[dofs + Ms] = row[rd_col_v<L, R0 + Ms, 0>] * src[rd_src_v<L, R0 + Ms, 0>]), ...);
  else
    ((dst[dofs + Ms] = fma(row[rd_col_v<L, R0 + Ms, T>], src[rd_src_v<L, R0 + Ms, T>], dst[dofs + Ms])), ...);
}
template <int L, int R0, int NS, int ND, int... Ms, int... Ts>
__device__ __forceinline__ void rd_pull(const double (&src)[NS], const double* row, double (&dst)[ND], int dofs,
                                        std::integer_sequence<int, Ms...> ms, std::integer_sequence<int, Ts...>) {
  (rd_term<L, R0, Ts>(src, row, dst, dofs, ms), ...);
}
// level L entries [R0, R0 + C) into dst[dofs ...]
template <int L, int R0, int C, int NS, int ND>
__device__ __forceinline__ void rd_level_part(const double (&src)[NS], const double* row, double (&dst)[ND], int dofs) {
  rd_pull<L, R0>(src, row, dst, dofs, std::make_integer_sequence<int, C>{}, std::make_integer_sequence<int, L>{});
}
// level L (all C(8, L) entries) in groups of G
template <int L, int G, int NS, int ND, int... Ks>
__device__ __forceinline__ void rd_level(const double (&src)[NS], const double* row, double (&dst)[ND],
                                         std::integer_sequence<int, Ks...>) {
  ((rd_level_part<L, G * Ks, (ND - G * Ks < G ? ND - G * Ks : G)>(src, row, dst, G * Ks)), ...);
}
// level 4 group K (G entries) -> TMEM columns 2GK
template <int G, int K>
__device__ __forceinline__ void rd_l4_group(const double (&f3)[56], const double* r3, uint32_t tb) {
  constexpr int C = (70 - G * K < G) ? 70 - G * K : G;
  double g[C];
  rd_level_part<4, G * K, C>(f3, r3, g, 0);
  tm_st_n<C>(tb + 2 * G * K, g);
}
template <int G, int... Ks>
__device__ __forceinline__ void rd_l4(const double (&f3)[56], const double* r3, uint32_t tb,
                                      std::integer_sequence<int, Ks...>) {
  (rd_l4_group<G, Ks>(f3, r3, tb), ...);
}
// push level-4 entry T = T0 + I/4 times a_4j (j its (I%4)-th missing column) into level 5
template <int T0, int I>
__device__ __forceinline__ void rd_push1(const double* x, const double* r4, double (&f5)[56]) {
  constexpr int T = T0 + I / 4, MT = rd_mask(4, T), J = rd_bit(~MT & 255, I % 4), S = rd_rank(MT | (1 << J));
  if constexpr (rd_first_push(MT | (1 << J)) == T) f5[S] = r4[J] * x[I / 4];
  else f5[S] = fma(r4[J], x[I / 4], f5[S]);
}
template <int T0, int... Is>
__device__ __forceinline__ void rd_push(const double* x, const double* r4, double (&f5)[56],
                                        std::integer_sequence<int, Is...>) {
  (rd_push1<T0, Is>(x, r4, f5), ...);
}
// level 5 from the parked level 4, G entries per TMEM load; group K+1's load
// is issued before group K's pushes, so the TMEM latency hides behind them
template <int G, int K>
__device__ __forceinline__ void rd_l5_group(uint32_t tb, const double* r4, double (&f5)[56],
                                            uint32_t (&cur)[((2 * G + 15) / 16) * 16]) {
  constexpr int NG = (70 + G - 1) / G;
  constexpr int C = (70 - G * K < G) ? 70 - G * K : G;
  constexpr int NR = ((2 * G + 15) / 16) * 16;
  tm_wait_ld_n(cur);
  double x[C];
#pragma unroll
  for (int i = 0; i < C; ++i) x[i] = tm_pack(cur[2 * i], cur[2 * i + 1]);
  if constexpr (K + 1 < NG) {
    constexpr int C1 = (70 - G * (K + 1) < G) ? 70 - G * (K + 1) : G;
    static_assert(((2 * C1 + 15) / 16) * 16 <= NR, "");
    tm_ld_n<C1>(tb + 2 * G * (K + 1), *reinterpret_cast<uint32_t(*)[((2 * C1 + 15) / 16) * 16]>(cur));
  }
  rd_push<G * K>(x, r4, f5, std::make_integer_sequence<int, 4 * C>{});
}
template <int G, int... Ks>
__device__ __forceinline__ void rd_l5(uint32_t tb, const double* r4, double (&f5)[56],
                                      std::integer_sequence<int, Ks...>) {
  uint32_t cur[((2 * G + 15) / 16) * 16];
  tm_ld_n<(G < 70 ? G : 70)>(tb, cur);
  (rd_l5_group<G, Ks>(tb, r4, f5, cur), ...);
}

template <int G>
struct RowDp8Tm {
  static_assert(G % 2 == 0 && 2 * 70 <= kTmRaw, "level-4 groups fit below the raw block");
  template <class R>
  __device__ __forceinline__ static double run(const double2* M, int rho, int t, uint32_t tb, R&& release) {
    double v01[16], v23[16];
    rd_pair(M, 0, rho, t, v01);
    rd_pair(M, 1, rho, t, v23);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // rows 4..7 wait in TMEM
      double v[16];
      rd_pair(M, 2 + h, rho, t, v);
      tm_st8(tb + kTmRaw + 32 * h, v);
      tm_st8(tb + kTmRaw + 32 * h + 16, v + 8);
    }
    release();
    double f3[56];
    {
      double f1[8], f2[28];
#pragma unroll
      for (int j = 0; j < 8; ++j) f1[j] = v01[j];
      rd_level<2, 28>(f1, v01 + 8, f2, std::make_integer_sequence<int, 1>{});
      rd_level<3, 14>(f2, v23, f3, std::make_integer_sequence<int, 4>{});
    }
    rd_l4<G>(f3, v23 + 8, tb, std::make_integer_sequence<int, (70 + G - 1) / G>{});
    tm_wait_st();
    double v45[16], v67[16];
    tm_ld_pair(tb + kTmRaw, v45);
    double f5[56];
    rd_l5<G>(tb, v45, f5, std::make_integer_sequence<int, (70 + G - 1) / G>{});
    tm_ld_pair(tb + kTmRaw + 32, v67);
    double f6[28], f7[8];
    rd_level<6, 14>(f5, v45 + 8, f6, std::make_integer_sequence<int, 2>{});
    rd_level<7, 8>(f6, v67, f7, std::make_integer_sequence<int, 1>{});
    // level 8 as two 4-term chains
    double e0 = v67[8] * f7[rd_rank(255 & ~1)], e1 = v67[12] * f7[rd_rank(255 & ~16)];
#pragma unroll
    for (int j = 1; j < 4; ++j) {
      e0 = fma(v67[8 + j], f7[7 - j], e0);
      e1 = fma(v67[12 + j], f7[3 - j], e1);
    }
    return e0 + e1;
  }
};

// One CTA of WARPS warps per TMEM slice: per-warp single-stage tile rings
// (lane 0 arms the warp's mbarrier and issues its bulk copies), each thread
// one matrix, Body::run calls release() once the lane's matrix is out of the
// slot (registers + TMEM), so the warp's next tile streams in during the
// arithmetic.
template <int WARPS, class Body, bool kComputeOnly = false>
__global__ void __launch_bounds__(32 * WARPS, 8 / WARPS) perm8_tmem_kernel(const double* __restrict__ a,
                                                                           double* __restrict__ out, int64_t nb) {
  static_assert(WARPS == 4 || WARPS == 8, "4 warps (two CTAs per SM) or 8 (one CTA) share the 512 TMEM columns");
  constexpr unsigned TILE_BYTES = 32 * 64 * sizeof(double);
  extern __shared__ __align__(128) unsigned char bb_smem_raw[];
  __shared__ __align__(8) uint64_t full[WARPS];
  __shared__ uint32_t tmem_base_sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(bb_smem(&tmem_base_sh)),
                 "n"(kTmCols * WARPS / 4)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  unsigned char* ring = bb_smem_raw + (size_t)warp * TILE_BYTES;
  uint64_t* bar = &full[warp];
  const int64_t ntiles = (nb + 31) / 32;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp, nw = (int64_t)gridDim.x * WARPS;
  auto issue = [&](int64_t tile) {
    const int64_t first = tile * 32;
    const int64_t cnt = (nb - first < 32) ? nb - first : 32;
    const unsigned bytes = (unsigned)cnt * 512u;
    bb_expect_tx(bar, bytes);
    bb_bulk_g2s(ring, reinterpret_cast<const char*>(a) + first * 512, bytes, bar);
  };
  if (lane == 0) {
    bb_mbar_init(bar, 1);
    bb_fence_mbar_init();
    if (gw < ntiles) issue(gw);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base_sh + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kTmCols);
  const int rho = lane & 3, t = (lane >> 2) & 1;
  unsigned phase = 0;
  for (int64_t tile = gw; tile < ntiles; tile += nw) {
    if (!kComputeOnly || tile == gw) bb_wait(bar, phase);  // (kComputeOnly: timing experiments)
    phase ^= 1u;
    const int64_t first = tile * 32;
    const int cnt = (int)((nb - first < 32) ? nb - first : 32);
    PERM_CHECK(cnt >= 1 && cnt <= 32 && first + cnt <= nb);
    const double2* M = reinterpret_cast<const double2*>(ring + (size_t)lane * 512);
    const double res = Body::run(M, rho, t, tb, [&]() {
      __syncwarp();  // every lane holds its matrix: the slot is free
      if (lane == 0) {
        const int64_t nt = tile + nw;
        if (nt < ntiles && !kComputeOnly) {
          bb_fence_proxy_async();
          issue(nt);
        }
      }
    });
    if (lane < cnt) out[first + lane] = res;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh),
                 "n"(kTmCols * WARPS / 4)
                 : "memory");
  }
}

}  // namespace permb200
