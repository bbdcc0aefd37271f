// Accuracy experiment for the Gray walk's chunked FP64 state (SURVEY 7.4.1,
// VERDICT r1 W2): where does the n >= 34 relative error come from?
//
// Walks Gray indices [k0, k0 + S) of the C5 Glynn setup (v0 = column sums,
// U[t] = -2 row(n-1-t)) in chunks of L, each chunk re-seeded exactly
// (double-double seed rounded once), and compares the raw sum against a
// double-double walk of the same range.  Variants:
//   A  state updated in place (v += U[t] every step), plain chunk sum (the
//      r1 kernel's arithmetic)
//   B  as A, chunk sum in double-double (isolates the summation error)
//   E  state in double-double, rounded per step (isolates the state drift)
//   R1 base state without row 0: w += U[t] only for t >= 1, the term uses
//      w + U[0] computed fresh when bit 0 is set (same DADD count as A)
//   R2 base state without rows 0, 1: combos U0, U1, U0+U1 fresh
//   R3 base state without rows 0..2: 7 combos fresh
// Product: 4 interleaved chains + pairwise tree (as chain_product<T,P>).
//
//   gcc -O2 -ffp-contract=off -fopenmp tools/chunk_drift_exp.c -o /tmp/cde -lm
//   /tmp/cde n log2S log2L_min log2L_max matrix.bin
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define PMAX 64
typedef struct { double h, l; } dd;
static inline void two_sum(double a, double b, double* s, double* e) {
  double x = a + b, bb = x - a;
  *e = (a - (x - bb)) + (b - bb);
  *s = x;
}
static inline void two_prod(double a, double b, double* p, double* e) {
  *p = a * b;
  *e = fma(a, b, -*p);
}
static inline dd dd_add(dd a, dd b) {
  double s, e;
  two_sum(a.h, b.h, &s, &e);
  e += a.l + b.l;
  dd r;
  two_sum(s, e, &r.h, &r.l);
  return r;
}
static inline dd dd_add_d(dd a, double b) {
  double s, e;
  two_sum(a.h, b, &s, &e);
  e += a.l;
  dd r;
  two_sum(s, e, &r.h, &r.l);
  return r;
}
static inline dd dd_mul(dd a, dd b) {
  double p, e;
  two_prod(a.h, b.h, &p, &e);
  e += a.h * b.l + a.l * b.h;
  dd r;
  two_sum(p, e, &r.h, &r.l);
  return r;
}
static int n;
static double v0[PMAX], U[PMAX][PMAX];

static inline uint64_t gray(uint64_t k) { return k ^ (k >> 1); }
static double v0q[PMAX], Uq[PMAX][PMAX];
static void seed_q(uint64_t k, double* v) {
  uint64_t g = gray(k);
  for (int j = 0; j < n; ++j) {
    double a = v0q[j];
    for (int t = 0; t < n - 1; ++t)
      if ((g >> t) & 1) a += Uq[t][j];
    v[j] = a;
  }
}
static inline double prod4(const double* v) {
  double c[4] = {v[0], v[1], v[2], v[3]};
  for (int j = 4; j < n; ++j) c[j & 3] *= v[j];
  return (c[0] * c[1]) * (c[2] * c[3]);
}

// exact-ish seed of the state at Gray index k (bits >= lo only if mask)
static void seed(uint64_t k, uint64_t mask, double* v) {
  uint64_t g = gray(k) & mask;
  for (int j = 0; j < n; ++j) {
    dd a = {v0[j], 0};
    for (int t = 0; t < n - 1; ++t)
      if ((g >> t) & 1) a = dd_add_d(a, U[t][j]);
    v[j] = a.h;
  }
}

// variant: 'A','B','E', or 1,2,3 (base state without rows < r)
static dd walk_chunk(uint64_t k0, uint64_t L, int var) {
  double v[PMAX], w[PMAX], t[PMAX];
  dd vs[PMAX];
  double acc = 0.0;
  dd accd = {0, 0};
  if (var == 'A' || var == 'B' || var == 'E') {
    seed(k0, ~0ull, v);
    for (int j = 0; j < n; ++j) vs[j].h = v[j], vs[j].l = 0;
    for (uint64_t k = k0; k < k0 + L; ++k) {
      if (k != k0) {
        int b = __builtin_ctzll(k);
        double s = ((gray(k) >> b) & 1) ? 1.0 : -1.0;
        if (var == 'E') {
          for (int j = 0; j < n; ++j) {
            vs[j] = dd_add_d(vs[j], s * U[b][j]);
            v[j] = vs[j].h + vs[j].l;
          }
        } else {
          for (int j = 0; j < n; ++j) v[j] += s * U[b][j];
        }
      }
      double p = prod4(v);
      if (k & 1) p = -p;
      if (var == 'B') accd = dd_add_d(accd, p);
      else acc += p;
    }
  } else if (var == 'Q' || var == 'q') {
    // quantized setup: v0 and U rounded to the grid q (exact sums), state exact
    double vq[PMAX];
    for (int j = 0; j < n; ++j) vq[j] = 0;
    seed_q(k0, vq);
    for (uint64_t k = k0; k < k0 + L; ++k) {
      if (k != k0) {
        int b = __builtin_ctzll(k);
        double s = ((gray(k) >> b) & 1) ? 1.0 : -1.0;
        for (int j = 0; j < n; ++j) vq[j] += s * Uq[b][j];
      }
      double p = prod4(vq);
      if (k & 1) p = -p;
      if (var == 'Q') acc += p;
      else accd = dd_add_d(accd, p);
    }
    if (var == 'q') return accd;
  } else {
    const int dstate = (var == 'D');
    const int r = dstate ? 3 : var;
    const uint64_t lowmask = (1ull << r) - 1;
    // combos[c] = sum_{t < r, bit t of c} U[t], rounded once from dd
    static __thread double combos[32][PMAX];
    for (int c = 0; c < (1 << r); ++c)
      for (int j = 0; j < n; ++j) {
        dd a = {0, 0};
        for (int tt = 0; tt < r; ++tt)
          if ((c >> tt) & 1) a = dd_add_d(a, U[tt][j]);
        combos[c][j] = a.h;
      }
    seed(k0, ~lowmask, w);
    dd wd[PMAX];
    for (int j = 0; j < n; ++j) wd[j].h = w[j], wd[j].l = 0;
    for (uint64_t k = k0; k < k0 + L; ++k) {
      if (k != k0) {
        int b = __builtin_ctzll(k);
        if (b >= r) {
          double s = ((gray(k) >> b) & 1) ? 1.0 : -1.0;
          if (dstate) {
            for (int j = 0; j < n; ++j) {
              wd[j] = dd_add_d(wd[j], s * U[b][j]);
              w[j] = wd[j].h + wd[j].l;
            }
          } else {
            for (int j = 0; j < n; ++j) w[j] += s * U[b][j];
          }
        }
      }
      const int c = (int)(gray(k) & lowmask);
      double p;
      if (c) {
        for (int j = 0; j < n; ++j) t[j] = w[j] + combos[c][j];
        p = prod4(t);
      } else {
        p = prod4(w);
      }
      if (k & 1) p = -p;
      acc += p;
    }
  }
  if (var == 'B') return accd;
  dd r = {acc, 0};
  return r;
}

static dd walk_dd_ref(uint64_t k0, uint64_t L) {
  dd v[PMAX];
  double g[PMAX];
  seed(k0, ~0ull, g);
  // exact dd seed
  uint64_t gg = gray(k0);
  for (int j = 0; j < n; ++j) {
    dd a = {v0[j], 0};
    for (int t = 0; t < n - 1; ++t)
      if ((gg >> t) & 1) a = dd_add_d(a, U[t][j]);
    v[j] = a;
  }
  dd acc = {0, 0};
  for (uint64_t k = k0; k < k0 + L; ++k) {
    if (k != k0) {
      int b = __builtin_ctzll(k);
      double s = ((gray(k) >> b) & 1) ? 1.0 : -1.0;
      for (int j = 0; j < n; ++j) v[j] = dd_add_d(v[j], s * U[b][j]);
    }
    dd p = v[0];
    for (int j = 1; j < n; ++j) p = dd_mul(p, v[j]);
    if (k & 1) p.h = -p.h, p.l = -p.l;
    acc = dd_add(acc, p);
  }
  return acc;
}

int main(int argc, char** argv) {
  if (argc < 6) {
    fprintf(stderr, "usage: n log2S log2Lmin log2Lmax matrix.bin\n");
    return 2;
  }
  n = atoi(argv[1]);
  const int lS = atoi(argv[2]), lmin = atoi(argv[3]), lmax = atoi(argv[4]);
  double* a = malloc(sizeof(double) * n * n);
  FILE* f = fopen(argv[5], "rb");
  if (!f || fread(a, sizeof(double), n * n, f) != (size_t)(n * n)) return 3;
  fclose(f);
  for (int j = 0; j < n; ++j) {
    double s = 0;
    for (int i = 0; i < n; ++i) s += a[i * n + j];
    v0[j] = s;
  }
  for (int t = 0; t < n - 1; ++t)
    for (int j = 0; j < n; ++j) U[t][j] = -2.0 * a[(n - 1 - t) * n + j];
  {  // quantization grid: every partial column sum of |v0| + sum|U| stays < 2^52 q
    double cmax = 0;
    for (int j = 0; j < n; ++j) {
      double s = 0;
      for (int i = 0; i < n; ++i) s += 3.0 * fabs(a[i * n + j]);
      if (s > cmax) cmax = s;
    }
    (void)cmax;
    for (int j = 0; j < n; ++j) {  // per-column grid q_j = 2^(ceil(log2 sum_i |a_ij|) - 52)
      double c = 0;
      for (int i = 0; i < n; ++i) c += fabs(a[i * n + j]);
      const double q = ldexp(1.0, (int)ceil(log2(c)) - 52);
      double s = 0;
      for (int i = 0; i < n; ++i) s += rint(a[i * n + j] / q) * q;
      v0q[j] = s;
      for (int t = 0; t < n - 1; ++t) Uq[t][j] = -2.0 * rint(a[(n - 1 - t) * n + j] / q) * q;
    }
  }
  const uint64_t S = 1ull << lS;
  const uint64_t k_start = (1ull << (n - 1)) - S;  // the last S indices (all high bits exercised)
  // reference, in chunks of 2^lmin (dd everywhere)
  const uint64_t Lr = 1ull << lmin;
  const int64_t nref = (int64_t)(S / Lr);
  dd ref = {0, 0};
  double mag = 0;
  {
    dd* parts = malloc(sizeof(dd) * nref);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < nref; ++c) parts[c] = walk_dd_ref(k_start + c * Lr, Lr);
    for (int64_t c = 0; c < nref; ++c) {
      ref = dd_add(ref, parts[c]);
      mag += fabs(parts[c].h);
    }
    free(parts);
  }
  printf("n=%d range=[2^%d-2^%d, 2^%d) ref=%.17e sum|chunk|=%.3e\n", n, n - 1, lS, n - 1, ref.h, mag);
  const int vars[] = {'A', 'E', 2, 3, 'D', 5, 'Q', 'q'};
  const char* names[] = {"A (r1)", "E (dd state)", "R2 base w/o rows0-1", "R3 base w/o rows0-2",
                         "R3 with dd base state", "R5 base w/o rows0-4", "Q quantized A, exact state", "Q + dd chunk sum"};
  const int NV = 8;
  for (int lL = lmin; lL <= lmax; ++lL) {
    const uint64_t L = 1ull << lL;
    const int64_t nc = (int64_t)(S / L);
    for (int vi = 0; vi < NV; ++vi) {
      dd* parts = malloc(sizeof(dd) * nc);
#pragma omp parallel for schedule(dynamic, 16)
      for (int64_t c = 0; c < nc; ++c) parts[c] = walk_chunk(k_start + c * L, L, vars[vi]);
      dd tot = {0, 0};
      for (int64_t c = 0; c < nc; ++c) tot = dd_add(tot, parts[c]);
      free(parts);
      const double err = fabs((tot.h - ref.h) + (tot.l - ref.l));
      printf("L=2^%-2d %-22s err/|ref| %.3e\n", lL, names[vi], err / fabs(ref.h));
      fflush(stdout);
    }
  }
  return 0;
}
