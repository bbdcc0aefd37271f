// EXPERIMENT (not used by the engine; see profiles/r1_walk_experiments.txt):
// split-state Gray walk (real, unweighted), measured 5-15% SLOWER than
// walk_kernel at P = 20..36 on B200 -- kept as the record of that design.
//
// walk_kernel keeps the whole state vector in one lane and re-reads every
// flip row from shared memory at every step: P/2 LDS.128 per step next to 2P
// FP64 ops, and the FP64 pipe stalls on those loads (ncu: short_scoreboard
// is the top stall at P = 36).  Here a chunk is owned by a lane PAIR (lanes
// l and l+16): each lane holds half of the state (H = ceil(P/2) entries) and
// half of flip rows 0 and 1 in registers -- they are 6 of every 8 flips and
// constant for the whole kernel -- so only rows 2 and the runtime row come
// from shared memory (H LDS.128 per lane per 8 steps instead of 4P).  A step
// is H updates + H-1 products per lane; the two half products of 8 steps are
// exchanged with 8 shuffles and combined 4 per lane, so the FP64 work per
// step stays 2P and the non-FP64 instructions drop from ~P/2+8 to ~4.
//
// Gray structure as in walk.cuh: a warp owns 16 adjacent chunks of L = 2^r
// indices, every lane performs the same flip schedule, the 8-step unroll has
// compile-time rows t = 0, 1, 0, 2, 0, 1, 0 and one runtime row.
#pragma once
#include "../paper_2510_03421_b200/csrc/walk_launch.cuh"

namespace permb200 {

// half width, stride of one half in shared memory (even for LDS.128, and
// off a multiple of 16 doubles so the two halves' broadcasts hit different
// banks), row stride
template <int P>
struct SplitShape {
  static constexpr int H = (P + 1) / 2;
  static constexpr int HE = (H + 1) & ~1;
  static constexpr int HS = (HE % 16 == 0) ? HE + 2 : HE;
  static constexpr int RS = 2 * HS;
};

#ifndef SPLIT_RREG
#define SPLIT_RREG 1  // flip rows held in registers (1: row 0; 2: rows 0 and 1)
#endif
#ifndef SPLIT_PH
#define SPLIT_PH 4    // steps per exchange of half products (2, 4 or 8)
#endif
#ifndef SPLIT_MINB
#define SPLIT_MINB 2
#endif
template <int P>
__host__ __device__ constexpr int split_min_blocks() {
  return SPLIT_MINB;
}

// v[j] (+|-|fma s) row[j], j < H, row in shared memory (pairs via LDS.128)
template <int H, int UPD>
__device__ __forceinline__ void split_update_smem(double (&v)[H], const double* row, double s) {
#pragma unroll
  for (int j = 0; j + 1 < H; j += 2) {
    const double2 u = lds2(row + j);
    if constexpr (UPD == 0) { v[j] += u.x; v[j + 1] += u.y; }
    else if constexpr (UPD == 1) { v[j] -= u.x; v[j + 1] -= u.y; }
    else { v[j] = fma(s, u.x, v[j]); v[j + 1] = fma(s, u.y, v[j + 1]); }
  }
  if constexpr (H & 1) {
    const double u = lds1(row + H - 1);
    if constexpr (UPD == 0) v[H - 1] += u;
    else if constexpr (UPD == 1) v[H - 1] -= u;
    else v[H - 1] = fma(s, u, v[H - 1]);
  }
}

// half product with K interleaved chains
template <int H>
__device__ __forceinline__ double split_product(const double (&v)[H]) {
  constexpr int K = H >= 16 ? 4 : (H >= 8 ? 2 : 1);
  double c[K];
#pragma unroll
  for (int i = 0; i < K; ++i) c[i] = v[i];
#pragma unroll
  for (int j = K; j < H; ++j) c[j % K] *= v[j];
  return tree_of<double, K>(c);
}

template <int P>
__global__ void __launch_bounds__(kWalkThreads, split_min_blocks<P>()) walk_split_kernel(WalkArgs args) {
  using S = SplitShape<P>;
  constexpr int H = S::H, HS = S::HS, RS = S::RS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sU = reinterpret_cast<double*>(smem_raw);  // [B][RS]: half 0 at 0, half 1 at HS
  double* sV0 = sU + (size_t)args.B * RS;             // [RS]

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, cl = lane & 15;
  const int B = args.B;
  {
    const double* gU = static_cast<const double*>(args.U);
    const double* gV0 = static_cast<const double*>(args.v0);
    // odd P: the last entry of half 1 is a padding column (state 1, rows 0)
    for (int i = tid; i < B * RS; i += kWalkThreads) {
      const int t = i / RS, c = i % RS, hh = c / HS, j = c % HS, col = hh * H + j;
      sU[i] = (j < H && col < P) ? gU[(size_t)t * P + col] : 0.0;
    }
    for (int c = tid; c < RS; c += kWalkThreads) {
      const int hh = c / HS, j = c % HS, col = hh * H + j;
      sV0[c] = (j < H) ? (col < P ? gV0[col] : 1.0) : 0.0;
    }
  }
  __syncthreads();

  const double* myU = sU + half * HS;  // this lane's half of every row
  double r0[H];
  double r1[SPLIT_RREG >= 2 ? H : 1];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    r0[j] = myU[j];
    if constexpr (SPLIT_RREG >= 2) r1[j] = myU[RS + j];
  }

  const int log2L = args.log2L;
  const uint64_t nq = (1ull << log2L) >> 3;
  const uint64_t bmask = (B >= 64) ? ~0ull : ((1ull << B) - 1);
  const uint64_t hmask = (~0ull << (log2L + 4)) & bmask;  // Gray bits shared by a warp's 16 chunks
  double hi = 0.0, lo = 0.0;
  const uint64_t total_warps = (uint64_t)gridDim.x * kWalkWarps;
  constexpr int PH = SPLIT_PH;  // steps per half-product exchange
  const double sg = half ? -1.0 : 1.0;

  for (uint64_t g = (uint64_t)blockIdx.x * kWalkWarps + warp; g < args.ngroups; g += total_warps) {
    const uint64_t kb = args.k_begin + ((g * 16) << log2L);
    const uint64_t k0 = kb + ((uint64_t)cl << log2L);
    const uint64_t g0 = k0 ^ (k0 >> 1);
    double v[H];
#pragma unroll
    for (int j = 0; j < H; ++j) v[j] = sV0[half * HS + j];
    {  // warp-uniform high Gray bits
      uint64_t bits = (kb ^ (kb >> 1)) & hmask;
      while (bits) {
        const int t = __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        split_update_smem<H, 0>(v, myU + t * RS, 0.0);
      }
    }
    // lane-dependent Gray bits: positions log2L-1 .. log2L+3
#pragma unroll
    for (int d = -1; d <= 3; ++d) {
      const int b = log2L + d;
      if (b < B) split_update_smem<H, 2>(v, myU + b * RS, (double)((g0 >> b) & 1));
    }

    double acc = 0.0;
    for (uint64_t q = 0; q < nq; ++q) {
      double ph[PH];
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        ph[l % PH] = split_product<H>(v);
        if ((l % PH) == PH - 1) {
          // half 0 finishes the first PH/2 steps of the batch, half 1 the rest;
          // term sign (-1)^l
#pragma unroll
          for (int i = 0; i < PH / 2; ++i) {
            const double mine = half ? ph[PH / 2 + i] : ph[i];
            const double send = half ? ph[i] : ph[PH / 2 + i];
            const double other = __shfl_xor_sync(0xffffffffu, send, 16);
            const double p = mine * other;
            if constexpr ((PH / 2) & 1) acc = fma((i & 1) ? -sg : sg, p, acc);
            else acc = (i & 1) ? acc - p : acc + p;
          }
        }
        // update to step l+1: rows 0, 1, 0, 2, 0, 1, 0, runtime
        if (l == 0 || l == 4) {
#pragma unroll
          for (int j = 0; j < H; ++j) v[j] += r0[j];
        } else if (l == 2 || l == 6) {
#pragma unroll
          for (int j = 0; j < H; ++j) v[j] -= r0[j];
        } else if (l == 1 || l == 5) {
          if constexpr (SPLIT_RREG >= 2) {
#pragma unroll
            for (int j = 0; j < H; ++j) v[j] = (l == 1) ? v[j] + r1[j] : v[j] - r1[j];
          } else {
            if (l == 1) split_update_smem<H, 0>(v, myU + RS, 0.0);
            else split_update_smem<H, 1>(v, myU + RS, 0.0);
          }
        } else if (l == 3) {
          const int b3 = (int)(((k0 + (q << 3)) >> 3) & 1);  // bit 2 set iff bit 3 of k0+8q clear
          split_update_smem<H, 2>(v, myU + 2 * RS, b3 ? -1.0 : 1.0);
        } else if (q + 1 < nq) {  // l == 7: the runtime row that opens the next 8 steps
          const uint64_t l0 = (q + 1) << 3;
          const int t = __ffsll((long long)l0) - 1;
          const uint64_t k = k0 + l0;
          const int set = (int)(((k ^ (k >> 1)) >> t) & 1);
          split_update_smem<H, 2>(v, myU + t * RS, set ? 1.0 : -1.0);
        }
      }
    }
    dd_acc(hi, lo, acc);
  }

  // ---- deterministic reduction: warp shuffle, then warp 0 over the block
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double h2 = __shfl_down_sync(0xffffffffu, hi, off), l2 = __shfl_down_sync(0xffffffffu, lo, off);
    dd_add(hi, lo, h2, l2);
  }
  __shared__ double red[kWalkWarps][2];
  if (lane == 0) {
    red[warp][0] = hi;
    red[warp][1] = lo;
  }
  __syncthreads();
  if (tid == 0) {
    double Hh = red[0][0], Lo = red[0][1];
    for (int w = 1; w < kWalkWarps; ++w) dd_add(Hh, Lo, red[w][0], red[w][1]);
    double* out = args.partials + (size_t)blockIdx.x * kPartialStride;
    out[0] = Hh; out[1] = Lo; out[2] = 0.0; out[3] = 0.0; out[4] = 0.0;
  }
  walk_last_block_combine(args.partials, args.final_out, args.done);
}

// Split-state walk (walk_split.cuh): real, unweighted, no magnitude sum.
// Returns cudaErrorNotSupported (nothing launched) when the range is too
// short or misaligned for groups of 16 chunks; the caller then uses
// launch_walk.
template <int P>
cudaError_t launch_walk_split(const WalkJob& job, WalkPlan* plan, cudaStream_t stream) {
  using S = SplitShape<P>;
  const uint64_t steps = job.k_end - job.k_begin;
  const size_t smem = (size_t)(job.B * S::RS + S::RS) * sizeof(double);
  auto kern = walk_split_kernel<P>;
  static int attr_smem = 0;  // benign race: idempotent
  if ((int)smem > 48 * 1024 && attr_smem < (int)smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_smem = (int)smem;
  }
  int dev = 0, nsm = 148, bps = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kWalkThreads, smem);
  if (e != cudaSuccess) return e;
  if (bps < 1) bps = 1;
  if (bps * nsm > kMaxPartials) bps = kMaxPartials / nsm;
  const uint64_t chunk_lanes = (uint64_t)bps * nsm * kWalkThreads / 2;
  int r = job.force_log2L > 0 ? job.force_log2L : choose_log2L(steps, chunk_lanes * 2, 16);
  const int amax = std::min(align_log2(job.k_begin), align_log2(steps)) - 4;
  if (r > amax) r = amax;
  if (r < 3 || (steps >> r) < 16) return cudaErrorNotSupported;
  WalkArgs a;
  a.v0 = job.v0; a.U = job.U; a.w = nullptr; a.B = job.B; a.log2L = r; a.wlen = 0; a.mag = 0;
  a.k_begin = job.k_begin;
  a.ngroups = (steps >> r) / 16;
  a.partials = job.partials;
  a.final_out = job.final_out;
  a.done = job.done;
  uint64_t grid = (uint64_t)bps * nsm;
  const uint64_t need = (a.ngroups + kWalkWarps - 1) / kWalkWarps;
  if (grid > need) grid = need;
  plan->small = false;
  plan->grid = (int)grid;
  plan->log2L = r;
  plan->ngroups = a.ngroups;
  kern<<<(unsigned)grid, kWalkThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace permb200
