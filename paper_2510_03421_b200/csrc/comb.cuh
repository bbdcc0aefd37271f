// Combination- and permutation-ordered kernels:
//
//  * ryser_comb_kernel: the binomial-weighted rectangular Ryser of
//    src/_kernels.py:226-262 (float) / :265-365 (checked int64), walking the
//    size-s column combinations in the reference's lexicographic order.  Each
//    thread unranks the first combination of its rank range and advances with
//    the reference's suffix-incremental row-sum update, so the int64 checks
//    (including every intermediate row-sum value of each transition) are
//    exactly the reference's.  Cost sum_{s<=m} C(n,s): far below the 2^n of
//    the all-subsets Gray walk for very rectangular shapes.
//
//  * comb_dfs_kernel: the combinatoric algorithm of src/_kernels.py:28-56 /
//    :59-108 (depth-first over m-permutations with prefix products, zero
//    partial products pruned).  The DFS tree is cut at depth D; thread t owns
//    the t-th depth-D prefix in lexicographic order and runs the reference's
//    DFS below it.  Float partials are compensated; checked-int partials are
//    (S, min prefix, max prefix, flag) summaries combined in DFS order.
#pragma once
#include "int_walk.cuh"

namespace permb200 {

constexpr int kCombThreads = 128;
// Column limit of the combination-ordered kernels.  The reference caps only
// its Gray walks at 62 columns (src/algorithms.py:47); its combinatoric and
// rectangular Ryser take any width (work P(n, m), sum_{s<=m} C(n, s)), so
// these kernels index columns up to kCombMaxN; rows stay <= 62.
constexpr int kCombMaxN = 256;
constexpr int kBinomCols = 64;  // binomial table C(i, j): i <= kCombMaxN, j < 64, saturating

enum CombMode { kCombF64 = 0, kCombC128 = 1, kCombI64 = 2, kCombI128 = 3 };

struct CombArgs {
  const void* a;          // m x n row-major (double / cd / int64)
  const uint64_t* binom;  // [kCombMaxN + 1][kBinomCols] binomial table C(i, j)
  int m, n, s;            // ryser: subset size s
  uint64_t total;         // number of items (combinations / prefixes)
  uint64_t per_thread;    // items per thread
  int depth;              // comb_dfs: prefix depth D
  void* out;              // per block partials
  // ryser, fused launch (all subset sizes s = m..1 in one grid): block range
  // [blk_first[s], blk_first[s] + blk_count[s]) walks the C(n, s) subsets of
  // size s, tot[s] items, per[s] per thread
  int fused;
  int smem_binom, smem_matrix;  // stage binomials (rows < n, cols < m) / the matrix in shared memory
  uint64_t blk_first[64], blk_count[64], tot[64], per[64];
};

__device__ __forceinline__ uint64_t binom_at(const uint64_t* tab, int i, int j) {
  return (j < 0 || j > i || i < 0) ? 0ull : tab[i * kBinomCols + j];
}

// ---------------------------------------------------------------- Ryser
template <int MODE>
__global__ void __launch_bounds__(kCombThreads) ryser_comb_kernel(CombArgs A) {
  const int m = A.m, n = A.n;
  int s = A.s;
  uint64_t bid = blockIdx.x, total = A.total, per_thread = A.per_thread;
  if (A.fused) {
    for (int q = m; q >= 1; --q)
      if (bid >= A.blk_first[q] && bid < A.blk_first[q] + A.blk_count[q]) {
        bid -= A.blk_first[q];
        s = q;
        total = A.tot[q];
        per_thread = A.per[q];
        break;
      }
  }
  // tiny launches are latency-bound: the binomials the unranking reads
  // (rows < n, columns < m) and the matrix go to shared memory first
  using Te = typename std::conditional<MODE == kCombF64, double,
                                       typename std::conditional<MODE == kCombC128, cd, int64_t>::type>::type;
  extern __shared__ __align__(16) unsigned char comb_smem[];
  const uint64_t* bt = A.binom;
  int bstride = kBinomCols;
  const Te* abase = static_cast<const Te*>(A.a);
  {
    unsigned char* p = comb_smem;
    if (A.smem_matrix) {
      Te* sa = reinterpret_cast<Te*>(p);
      for (int i = threadIdx.x; i < m * n; i += kCombThreads) sa[i] = abase[i];
      abase = sa;
      p += (((size_t)m * n * sizeof(Te)) + 15) & ~(size_t)15;
    }
    if (A.smem_binom) {
      uint64_t* sb = reinterpret_cast<uint64_t*>(p);
      for (int i = threadIdx.x; i < n * m; i += kCombThreads) sb[i] = binom_at(A.binom, i / m, i % m);
      bt = sb;
      bstride = m;
    }
    if (A.smem_matrix || A.smem_binom) __syncthreads();
  }
  const uint64_t gtid = bid * kCombThreads + threadIdx.x;
  const uint64_t r0 = gtid * per_thread;
  uint64_t r1 = r0 + per_thread;
  if (r1 > total) r1 = total;
  int comb[64];
  // accumulators
  double hi = 0, lo = 0, hi_i = 0, lo_i = 0;
  Summ sm;
  sm.S = i128_from(0); sm.mn = i128_from(0); sm.mx = i128_from(0); sm.flag = 0;
  bool have = false;
  if (r0 < r1) {
    // unrank r0 (lexicographic, 0-based)
    uint64_t r = r0;
    int x = 0;
    for (int q = 0; q < s; ++q) {
      for (;;) {
        const int bi = n - x - 1, bj = s - q - 1;  // 0 <= bj < m
        const uint64_t cnt = (bi < 0 || bj > bi) ? 0ull : bt[bi * bstride + bj];
        if (r < cnt) { comb[q] = x++; break; }
        r -= cnt;
        ++x;
        PERM_CHECK(x < n);  // the rank lies inside C(n, s)
      }
    }
    if constexpr (MODE == kCombI64) {
      const int64_t* a = abase;
      int64_t rs[64];
      for (int i = 0; i < m; ++i) {
        if (r0 == 0) {  // reference initial sums: sequential checked adds
          int64_t acc = 0;
          for (int q = 0; q < s; ++q)
            if (add_ovf(acc, a[i * n + comb[q]], acc)) sm.flag = 1;
          rs[i] = acc;
        } else {        // state reached by the previous transition: must fit
          i128 acc = i128_from(0);
          for (int q = 0; q < s; ++q) acc = i128_add(acc, i128_from(a[i * n + comb[q]]));
          if (!i128_fits_i64(acc)) sm.flag = 1;
          rs[i] = (int64_t)acc.lo;
        }
      }
      // walk [r0, r1); the transition out of r1-1 into r1 is replayed (and
      // checked) here, the state it produces is re-checked by the next range
      for (uint64_t rk = r0; rk < r1 && !sm.flag; ++rk) {
        int64_t p = 1;
        for (int i = 0; i < m; ++i) {
          if (rs[i] == 0) { p = 0; break; }
          int64_t t;
          if (mul_ovf(p, rs[i], t)) { sm.flag = 1; break; }
          p = t;
        }
        if (sm.flag) break;
        sm.S = i128_add(sm.S, i128_from(p));
        if (!have) { sm.mn = sm.S; sm.mx = sm.S; have = true; }
        else {
          if (i128_lt(sm.S, sm.mn)) sm.mn = sm.S;
          if (i128_lt(sm.mx, sm.S)) sm.mx = sm.S;
        }
        int pos = s - 1;
        while (pos >= 0 && comb[pos] == n - s + pos) --pos;
        if (pos < 0) break;
        // reference order (src/_kernels.py:319-340): remove comb[pos..s),
        // then add the new suffix, row by row inside each column
        for (int q = pos; q < s; ++q)
          for (int i = 0; i < m; ++i)
            if (sub_ovf(rs[i], a[i * n + comb[q]], rs[i])) sm.flag = 1;
        const int v = comb[pos] + 1;
        for (int q = pos; q < s; ++q) {
          comb[q] = v + (q - pos);
          for (int i = 0; i < m; ++i)
            if (add_ovf(rs[i], a[i * n + comb[q]], rs[i])) sm.flag = 1;
        }
      }
    } else {
      using T = typename std::conditional<MODE == kCombF64, double, cd>::type;
      const T* a = reinterpret_cast<const T*>(abase);
      T rs[64];
      for (int i = 0; i < m; ++i) {
        T acc = Num<T>::zero();
        for (int q = 0; q < s; ++q) acc = Num<T>::add(acc, a[i * n + comb[q]]);
        rs[i] = acc;
      }
      T chunk = Num<T>::zero();
      int cnt = 0;
      for (uint64_t rk = r0; rk < r1; ++rk) {
        T p = rs[0];
        for (int i = 1; i < m; ++i) p = Num<T>::mul(p, rs[i]);
        chunk = Num<T>::add(chunk, p);
        if (++cnt == 1024) {
          dd_acc(hi, lo, Num<T>::re(chunk));
          dd_acc(hi_i, lo_i, Num<T>::im(chunk));
          chunk = Num<T>::zero();
          cnt = 0;
        }
        if (rk + 1 == r1) break;
        int pos = s - 1;
        while (pos >= 0 && comb[pos] == n - s + pos) --pos;
        for (int q = pos; q < s; ++q)
          for (int i = 0; i < m; ++i) rs[i] = Num<T>::sub(rs[i], a[i * n + comb[q]]);
        const int v = comb[pos] + 1;
        for (int q = pos; q < s; ++q) {
          comb[q] = v + (q - pos);
          for (int i = 0; i < m; ++i) rs[i] = Num<T>::add(rs[i], a[i * n + comb[q]]);
        }
      }
      dd_acc(hi, lo, Num<T>::re(chunk));
      dd_acc(hi_i, lo_i, Num<T>::im(chunk));
    }
  }
  // ---- block reduction (ordered for the checked mode)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (MODE == kCombI64) {
    if (!have) {
      sm.mn.lo = ~0ull; sm.mn.hi = 0x3fffffffffffffffull;
      sm.mx.lo = 0ull;  sm.mx.hi = 0xc000000000000000ull;
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Summ o;
      o.S = shfl_down_i128(sm.S, off);
      o.mn = shfl_down_i128(sm.mn, off);
      o.mx = shfl_down_i128(sm.mx, off);
      o.flag = __shfl_down_sync(0xffffffffu, sm.flag, off);
      if ((lane & (2 * off - 1)) == 0 && lane + off < 32) sm = summ_cat(sm, o);
    }
    __shared__ Summ ws[kCombThreads / 32];
    if (lane == 0) ws[warp] = sm;
    __syncthreads();
    if (threadIdx.x == 0) {
      Summ t = ws[0];
      for (int w = 1; w < kCombThreads / 32; ++w) t = summ_cat(t, ws[w]);
      int64_t* o = static_cast<int64_t*>(A.out) + (size_t)blockIdx.x * 8;
      o[0] = (int64_t)t.S.lo; o[1] = (int64_t)t.S.hi;
      o[2] = (int64_t)t.mn.lo; o[3] = (int64_t)t.mn.hi;
      o[4] = (int64_t)t.mx.lo; o[5] = (int64_t)t.mx.hi;
      o[6] = t.flag; o[7] = 0;
    }
  } else {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      dd_add(hi, lo, __shfl_down_sync(0xffffffffu, hi, off), __shfl_down_sync(0xffffffffu, lo, off));
      dd_add(hi_i, lo_i, __shfl_down_sync(0xffffffffu, hi_i, off), __shfl_down_sync(0xffffffffu, lo_i, off));
    }
    __shared__ double red[kCombThreads / 32][4];
    if (lane == 0) { red[warp][0] = hi; red[warp][1] = lo; red[warp][2] = hi_i; red[warp][3] = lo_i; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double H = red[0][0], L = red[0][1], H2 = red[0][2], L2 = red[0][3];
      for (int w = 1; w < kCombThreads / 32; ++w) { dd_add(H, L, red[w][0], red[w][1]); dd_add(H2, L2, red[w][2], red[w][3]); }
      double* o = static_cast<double*>(A.out) + (size_t)blockIdx.x * 8;
      o[0] = H; o[1] = L; o[2] = H2; o[3] = L2; o[4] = 0; o[5] = 0; o[6] = 0; o[7] = 0;
    }
  }
}

// ---------------------------------------------------------------- combinatoric
// Prefix of depth D with lexicographic index `idx` among the P(n, D)
// D-permutations: digit q picks the (idx_q)-th unused column.
// MODE kCombI128: exact wrapping int128 products and sums (the host only
// launches it when an a-priori bound keeps every prefix product and partial
// sum inside int128, so the zero pruning sees true zeros).
template <int MODE>
__global__ void __launch_bounds__(kCombThreads) comb_dfs_kernel(CombArgs A) {
  const int m = A.m, n = A.n, D = A.depth;
  const uint64_t gtid = (uint64_t)blockIdx.x * kCombThreads + threadIdx.x;
  constexpr bool kInt = (MODE == kCombI64 || MODE == kCombI128);
  double hi = 0, lo = 0, hi_i = 0, lo_i = 0;
  Summ sm;
  sm.S = i128_from(0); sm.mn = i128_from(0); sm.mx = i128_from(0); sm.flag = 0;
  i128 wide = i128_from(0);  // kCombI128 running sum (mod 2^128)
  bool have = false;
  // element type of the matrix, and of the prefix products
  using Te = typename std::conditional<MODE == kCombF64, double,
                                       typename std::conditional<MODE == kCombC128, cd, int64_t>::type>::type;
  using T = typename std::conditional<MODE == kCombI128, i128, Te>::type;
  const Te* a = static_cast<const Te*>(A.a);
  auto is_zero = [](const T& p) -> bool {
    if constexpr (MODE == kCombI128) return (p.lo | p.hi) == 0;
    else if constexpr (MODE == kCombI64) return p == 0;
    else if constexpr (MODE == kCombF64) return p == 0.0;
    else return p.x == 0.0 && p.y == 0.0;
  };
  auto leaf = [&](const T& p) {
    if constexpr (MODE == kCombI64) {
      sm.S = i128_add(sm.S, i128_from(p));
      if (!have) { sm.mn = sm.S; sm.mx = sm.S; have = true; }
      else { if (i128_lt(sm.S, sm.mn)) sm.mn = sm.S; if (i128_lt(sm.mx, sm.S)) sm.mx = sm.S; }
    } else if constexpr (MODE == kCombI128) {
      wide = i128_add(wide, p);
    }
  };
  const uint64_t p0 = gtid * A.per_thread;
  uint64_t p1 = p0 + A.per_thread;
  if (p1 > A.total) p1 = A.total;
  PERM_CHECK(D >= 1 && D <= m && m <= 64 && n <= kCombMaxN);
  // Whole permutations in the prefix (D == m, n <= 32; every single
  // combinatoric of up to ~1e6 permutations): the used columns are a bit
  // mask and the k-th free column is __fns -- no local-memory arrays, whose
  // per-thread setup was most of a small call's 9 us kernel.  Same products
  // in the same order, same zero pruning (src/_kernels.py:52).
  const bool whole = !kInt && D == m && n <= 32;
  if constexpr (!kInt) {
  for (uint64_t pidx = p0; whole && pidx < p1; ++pidx) {
    uint64_t rem = pidx, radix_prod = 1;
    for (int q = 1; q < D; ++q) radix_prod *= (uint64_t)(n - q);
    unsigned freem = (n == 32) ? 0xffffffffu : ((1u << n) - 1u);
    T p = Num<T>::one();
    bool pruned = false;
    for (int q = 0; q < m; ++q) {
      const uint64_t digit = rem / radix_prod;
      rem -= digit * radix_prod;
      if (q + 1 < D) radix_prod /= (uint64_t)(n - q - 1);
      const int c = (int)__fns(freem, 0u, (int)digit + 1);
      freem &= ~(1u << c);
      p = Num<T>::mul(p, a[q * n + c]);
      if (q < m - 1 && is_zero(p)) {
        pruned = true;
        break;
      }
    }
    if (!pruned) {
      dd_acc(hi, lo, Num<T>::re(p));
      dd_acc(hi_i, lo_i, Num<T>::im(p));
    }
  }
  }
  for (uint64_t pidx = p0; !whole && pidx < p1 && !sm.flag; ++pidx) {
    // decode prefix: mixed radix (n, n-1, ..., n-D+1), most significant first
    int choice[64];
    bool used[kCombMaxN];
    for (int j = 0; j < n; ++j) used[j] = false;
    {
      uint64_t rem = pidx;
      uint64_t radix_prod = 1;
      for (int q = 1; q < D; ++q) radix_prod *= (uint64_t)(n - q);
      for (int q = 0; q < D; ++q) {
        const uint64_t digit = rem / radix_prod;
        rem -= digit * radix_prod;
        if (q + 1 < D) radix_prod /= (uint64_t)(n - q - 1);
        int c = -1;
        uint64_t k = digit;
        for (int j = 0; j < n; ++j)
          if (!used[j]) {
            if (k == 0) { c = j; break; }
            --k;
          }
        choice[q] = c;
        used[c] = true;
      }
    }
    // prefix products (checked / pruned exactly like the reference DFS)
    T prod[65];
    bool dead = false;
    if constexpr (MODE == kCombI64) prod[0] = 1;
    else if constexpr (MODE == kCombI128) prod[0] = i128_from(1);
    else prod[0] = Num<T>::one();
    for (int q = 0; q < D; ++q) {
      T p;
      if constexpr (MODE == kCombI64) {
        if (prod[q] != 0 && a[q * n + choice[q]] != 0) {
          if (mul_ovf(prod[q], a[q * n + choice[q]], p)) { sm.flag = 1; dead = true; break; }
        } else {
          p = prod[q] * a[q * n + choice[q]];
        }
      } else if constexpr (MODE == kCombI128) {
        p = i128_mul_s64(prod[q], a[q * n + choice[q]]);
      } else {
        p = Num<T>::mul(prod[q], a[q * n + choice[q]]);
      }
      if (q == m - 1) {  // leaf inside the prefix (D == m)
        if constexpr (kInt) {
          leaf(p);
        } else {
          dd_acc(hi, lo, Num<T>::re(p));
          dd_acc(hi_i, lo_i, Num<T>::im(p));
        }
        dead = true;
        break;
      }
      if (is_zero(p)) { dead = true; break; }  // src/_kernels.py:52 prune
      prod[q + 1] = p;
    }
    if (dead) continue;
    // DFS below the prefix (src/_kernels.py:37-55 with d starting at D)
    int ch[64];
    for (int q = 0; q < m; ++q) ch[q] = -1;
    int d = D;
    Te chunk;
    if constexpr (kInt) chunk = 0; else chunk = Num<Te>::zero();
    while (d >= D) {
      int j = ch[d];
      if (j >= 0) used[j] = false;
      ++j;
      while (j < n && used[j]) ++j;
      if (j >= n) { ch[d] = -1; --d; continue; }
      ch[d] = j;
      T p;
      if constexpr (MODE == kCombI64) {
        if (mul_ovf(prod[d], a[d * n + j], p)) { sm.flag = 1; break; }
      } else if constexpr (MODE == kCombI128) {
        p = i128_mul_s64(prod[d], a[d * n + j]);
      } else {
        p = Num<T>::mul(prod[d], a[d * n + j]);
      }
      if (d == m - 1) {
        if constexpr (kInt) leaf(p);
        else chunk = Num<T>::add(chunk, p);
      } else if (!is_zero(p)) {
        used[j] = true;
        prod[d + 1] = p;
        ++d;
      }
    }
    if constexpr (!kInt) {
      dd_acc(hi, lo, Num<Te>::re(chunk));
      dd_acc(hi_i, lo_i, Num<Te>::im(chunk));
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (MODE == kCombI64) {
    if (!have) {
      sm.mn.lo = ~0ull; sm.mn.hi = 0x3fffffffffffffffull;
      sm.mx.lo = 0ull;  sm.mx.hi = 0xc000000000000000ull;
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Summ o;
      o.S = shfl_down_i128(sm.S, off);
      o.mn = shfl_down_i128(sm.mn, off);
      o.mx = shfl_down_i128(sm.mx, off);
      o.flag = __shfl_down_sync(0xffffffffu, sm.flag, off);
      if ((lane & (2 * off - 1)) == 0 && lane + off < 32) sm = summ_cat(sm, o);
    }
    __shared__ Summ ws[kCombThreads / 32];
    if (lane == 0) ws[warp] = sm;
    __syncthreads();
    if (threadIdx.x == 0) {
      Summ t = ws[0];
      for (int w = 1; w < kCombThreads / 32; ++w) t = summ_cat(t, ws[w]);
      int64_t* o = static_cast<int64_t*>(A.out) + (size_t)blockIdx.x * 8;
      o[0] = (int64_t)t.S.lo; o[1] = (int64_t)t.S.hi;
      o[2] = (int64_t)t.mn.lo; o[3] = (int64_t)t.mn.hi;
      o[4] = (int64_t)t.mx.lo; o[5] = (int64_t)t.mx.hi;
      o[6] = t.flag; o[7] = 0;
    }
  } else if constexpr (MODE == kCombI128) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) wide = i128_add(wide, shfl_down_i128(wide, off));
    __shared__ i128 wsum[kCombThreads / 32];
    if (lane == 0) wsum[warp] = wide;
    __syncthreads();
    if (threadIdx.x == 0) {
      i128 t = wsum[0];
      for (int w = 1; w < kCombThreads / 32; ++w) t = i128_add(t, wsum[w]);
      int64_t* o = static_cast<int64_t*>(A.out) + (size_t)blockIdx.x * 8;
      o[0] = (int64_t)t.lo; o[1] = (int64_t)t.hi;
      for (int q = 2; q < 8; ++q) o[q] = 0;
    }
  } else {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      dd_add(hi, lo, __shfl_down_sync(0xffffffffu, hi, off), __shfl_down_sync(0xffffffffu, lo, off));
      dd_add(hi_i, lo_i, __shfl_down_sync(0xffffffffu, hi_i, off), __shfl_down_sync(0xffffffffu, lo_i, off));
    }
    __shared__ double red[kCombThreads / 32][4];
    if (lane == 0) { red[warp][0] = hi; red[warp][1] = lo; red[warp][2] = hi_i; red[warp][3] = lo_i; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double H = red[0][0], L = red[0][1], H2 = red[0][2], L2 = red[0][3];
      for (int w = 1; w < kCombThreads / 32; ++w) { dd_add(H, L, red[w][0], red[w][1]); dd_add(H2, L2, red[w][2], red[w][3]); }
      double* o = static_cast<double*>(A.out) + (size_t)blockIdx.x * 8;
      o[0] = H; o[1] = L; o[2] = H2; o[3] = L2; o[4] = 0; o[5] = 0; o[6] = 0; o[7] = 0;
    }
  }
}

}  // namespace permb200
