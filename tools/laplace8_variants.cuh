// The 4+4 Laplace forms of the 8x8 batch permanent, kept as measured
// alternatives to the row recursion the engine uses (csrc/batch_bulk.cuh,
// RowDp8Tm): tools/bulk_bench.cu times them side by side.
//   per(A) = sum_{|X|=4} per(A[0:4, X]) per(A[4:8, X^c]),
//   per(A[0:4, X]) = sum_{P subset X, |P|=2} q01(P) q23(X \ P)   (1134 FP64 ops)
// Laplace8TOp: minors parked in shared memory (4 warps/SM, C2a 0.114 ms);
// Laplace8Tm: minors parked in TMEM (8 warps/SM, 0.096 ms).
#pragma once
#include "../paper_2510_03421_b200/csrc/batch_bulk.cuh"

namespace permb200 {

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

// minor group K of the top half (G minors, fewer in the last group) -> TMEM column 2GK
template <int G, int K>
__device__ __forceinline__ void lp_tm_top_group(const double (&qa)[28], const double (&qb)[28], uint32_t tb) {
  constexpr int C = (70 - G * K < G) ? 70 - G * K : G;
  double g[C];
  Laplace8TOp<32, G>::template minors<0, G * K>(qa, qb, g, std::make_integer_sequence<int, C>{});
  tm_st_n<C>(tb + 2 * G * K, g);
}
template <int G, int... Ks>
__device__ __forceinline__ void lp_tm_top(const double (&qa)[28], const double (&qb)[28], uint32_t tb,
                                          std::integer_sequence<int, Ks...>) {
  (lp_tm_top_group<G, Ks>(qa, qb, tb), ...);
}
// minor group K of the bottom half on the complements, times the parked top minors
template <int G, int K>
__device__ __forceinline__ void lp_tm_bottom_group(const double (&qc)[28], const double (&qd)[28], uint32_t tb,
                                                   double (&acc)[8]) {
  constexpr int C = (70 - G * K < G) ? 70 - G * K : G;
  uint32_t r[((2 * C + 15) / 16) * 16];
  tm_ld_n<C>(tb + 2 * G * K, r);
  double hm[C];
  Laplace8TOp<32, G>::template minors<1, G * K>(qc, qd, hm, std::make_integer_sequence<int, C>{});
  tm_wait_ld_n(r);
#pragma unroll
  for (int i = 0; i < C; ++i) acc[i & 7] = fma(tm_pack(r[2 * i], r[2 * i + 1]), hm[i], acc[i & 7]);
}
template <int G, int... Ks>
__device__ __forceinline__ void lp_tm_bottom(const double (&qc)[28], const double (&qd)[28], uint32_t tb,
                                             double (&acc)[8], std::integer_sequence<int, Ks...>) {
  (lp_tm_bottom_group<G, Ks>(qc, qd, tb, acc), ...);
}

// Laplace body: the 4+4 split above (1134 FP64 ops per matrix)
template <int G>
struct Laplace8Tm {
  using L = Laplace8TOp<32, G>;
  static_assert(G % 2 == 0 && 2 * 70 <= kTmRaw, "minor groups fit below the raw block");
  template <class R>
  __device__ __forceinline__ static double run(const double2* M, int rho, int t, uint32_t tb, R&& release) {
    double qa[28], qb[28];
    L::load_q(M, rho, t, qa);
    L::load_q(M + 8, rho, t, qb);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // bottom rows (4,5) and (6,7), same rotation as load_q
      double v[16];
      rd_pair(M, 2 + h, rho, t, v);
      tm_st8(tb + kTmRaw + 32 * h, v);
      tm_st8(tb + kTmRaw + 32 * h + 16, v + 8);
    }
    release();
    // top half: 70 minors, G at a time, parked in TMEM
    lp_tm_top<G>(qa, qb, tb, std::make_integer_sequence<int, (70 + G - 1) / G>{});
    tm_wait_st();
    double qc[28], qd[28];
    {
      double v[16];
      tm_ld_pair(tb + kTmRaw, v);
      lp_qtable(v, qc);
      tm_ld_pair(tb + kTmRaw + 32, v);
      lp_qtable(v, qd);
    }
    // bottom half: the complements' minors against the parked ones
    double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    lp_tm_bottom<G>(qc, qd, tb, acc, std::make_integer_sequence<int, (70 + G - 1) / G>{});
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  }
};

}  // namespace permb200
