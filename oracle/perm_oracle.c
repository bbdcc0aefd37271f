/*
 * oracle/perm_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference permanent kernels
 * (/root/reference/pkg/src/permanent/_kernels.py, "src/_kernels.py" below),
 * used as the CHECKER for the CUDA engine in tests/, as the smoke() checker
 * and as bench.py's cpu_baseline / --impl reference arm.  It is never linked
 * into, loaded by, or called from the product path
 * (paper_2510_03421_b200/).
 *
 * Parity pin: the float/complex kernels reproduce the reference bit for bit
 * (same sequential evaluation order, no FMA contraction: build with
 * -ffp-contract=off).  tests/test_oracle_golden.py checks them against the
 * reference's own 300 golden vectors (pkg/frontend/tests/fixtures/parity.json)
 * and against fixtures produced by running the reference in this container
 * (oracle/gen_golden.py -> tests/golden/).
 *
 * Sections:
 *   1. literal restatements of the 10 reference kernels (f64, c128, checked
 *      int64) -- src/_kernels.py:28-697
 *   2. Gray-range forms (start anywhere in the walk; the sharding identity
 *      of SURVEY Appendix A) in f64 / c128 / wrapping int128 / double-double,
 *      plus pthread drivers that split a walk over host cores.  These are the
 *      "higher-precision restatement" oracles of SURVEY 8(c) and the CPU
 *      baseline of bench.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Column limit of the permutation / combination forms: the reference caps
 * only its Gray walks at 62 columns (src/algorithms.py:47), so the DFS and
 * the combination-order Ryser take any width up to this bound. */
#define ORC_MAX_COLS 256

typedef struct { double re, im; } cplx;
typedef __int128 i128;
typedef unsigned __int128 u128;

static inline cplx c_add(cplx a, cplx b) { cplx r = {a.re + b.re, a.im + b.im}; return r; }
static inline cplx c_sub(cplx a, cplx b) { cplx r = {a.re - b.re, a.im - b.im}; return r; }
/* numba / numpy complex multiply: (ac - bd) + (ad + bc)i, no FMA. */
static inline cplx c_mul(cplx a, cplx b) {
  double ac = a.re * b.re, bd = a.im * b.im, ad = a.re * b.im, bc = a.im * b.re;
  cplx r = {ac - bd, ad + bc};
  return r;
}
static inline int c_ne(cplx a, cplx b) { return a.re != b.re || a.im != b.im; }

static inline int ctz64(uint64_t k) { return __builtin_ctzll(k); }

/* ======================================================================
 * 1. Literal restatements
 * ====================================================================== */

/* comb_dfs: src/_kernels.py:28-56.  DFS over m-permutations, prefix
 * products, zero partial products pruned (:52). */
double orc_comb_f64(int m, int n, const double* a) {
  double zero = a[0] - a[0];
  int64_t choice[64];
  double prod[65];
  unsigned char used[ORC_MAX_COLS];
  for (int i = 0; i < m; ++i) choice[i] = -1;
  memset(used, 0, sizeof used);
  prod[0] = zero + 1.0;
  double total = zero;
  int d = 0;
  while (d >= 0) {
    int64_t j = choice[d];
    if (j >= 0) used[j] = 0;
    j += 1;
    while (j < n && used[j]) j += 1;
    if (j >= n) { choice[d] = -1; d -= 1; continue; }
    choice[d] = j;
    double p = prod[d] * a[d * n + j];
    if (d == m - 1) {
      total = total + p;
    } else if (p != zero) {
      used[j] = 1;
      prod[d + 1] = p;
      d += 1;
    }
  }
  return total;
}

void orc_comb_c128(int m, int n, const double* a_, double* out) {
  const cplx* a = (const cplx*)a_;
  cplx zero = c_sub(a[0], a[0]);
  int64_t choice[64];
  cplx prod[65];
  unsigned char used[ORC_MAX_COLS];
  for (int i = 0; i < m; ++i) choice[i] = -1;
  memset(used, 0, sizeof used);
  prod[0] = zero; prod[0].re = zero.re + 1.0; prod[0].im = zero.im + 0.0;
  cplx total = zero;
  int d = 0;
  while (d >= 0) {
    int64_t j = choice[d];
    if (j >= 0) used[j] = 0;
    j += 1;
    while (j < n && used[j]) j += 1;
    if (j >= n) { choice[d] = -1; d -= 1; continue; }
    choice[d] = j;
    cplx p = c_mul(prod[d], a[d * n + j]);
    if (d == m - 1) {
      total = c_add(total, p);
    } else if (c_ne(p, zero)) {
      used[j] = 1;
      prod[d + 1] = p;
      d += 1;
    }
  }
  out[0] = total.re; out[1] = total.im;
}

/* The reference's pre-checked int64 arithmetic (src/_kernels.py:80-103 and
 * the repeated blocks) tests "does the exact result fit in int64" before
 * every add/sub/mul; __builtin_*_overflow is exactly that predicate. */
#define CHK_ADD(x, y, r) __builtin_add_overflow((x), (y), (r))
#define CHK_SUB(x, y, r) __builtin_sub_overflow((x), (y), (r))
#define CHK_MUL(x, y, r) __builtin_mul_overflow((x), (y), (r))

/* comb_dfs_int: src/_kernels.py:59-108.  Returns overflow flag. */
int orc_comb_i64(int m, int n, const int64_t* a, int64_t* out) {
  int64_t choice[64];
  int64_t prod[65];
  unsigned char used[ORC_MAX_COLS];
  for (int i = 0; i < m; ++i) choice[i] = -1;
  memset(used, 0, sizeof used);
  prod[0] = 1;
  int64_t total = 0;
  int d = 0;
  *out = 0;
  while (d >= 0) {
    int64_t j = choice[d];
    if (j >= 0) used[j] = 0;
    j += 1;
    while (j < n && used[j]) j += 1;
    if (j >= n) { choice[d] = -1; d -= 1; continue; }
    choice[d] = j;
    int64_t x = prod[d], y = a[d * n + j], p;
    if (CHK_MUL(x, y, &p)) return 1;
    if (d == m - 1) {
      if (CHK_ADD(total, p, &total)) return 1;
    } else if (p != 0) {
      used[j] = 1;
      prod[d + 1] = p;
      d += 1;
    }
  }
  *out = total;
  return 0;
}

/* ryser_sq: src/_kernels.py:115-145. */
double orc_ryser_sq_f64(int n, const double* a) {
  double zero = a[0] - a[0];
  double rowsum[64];
  for (int i = 0; i < n; ++i) rowsum[i] = 0.0;
  double total = zero;
  int neg = 0;
  uint64_t steps = (n >= 64) ? ~0ull : ((1ull << n) - 1);
  for (uint64_t k = 1; k <= steps; ++k) {
    int t = ctz64(k);
    uint64_t g = k ^ (k >> 1);
    if ((g >> t) & 1) {
      for (int i = 0; i < n; ++i) rowsum[i] = rowsum[i] + a[i * n + t];
    } else {
      for (int i = 0; i < n; ++i) rowsum[i] = rowsum[i] - a[i * n + t];
    }
    double p = zero + 1.0;
    for (int i = 0; i < n; ++i) p = p * rowsum[i];
    neg = !neg;
    if (neg) total = total - p; else total = total + p;
  }
  if (n & 1) total = -total;
  return total;
}

void orc_ryser_sq_c128(int n, const double* a_, double* out) {
  const cplx* a = (const cplx*)a_;
  cplx zero = c_sub(a[0], a[0]);
  cplx one = {zero.re + 1.0, zero.im + 0.0};
  cplx rowsum[64];
  for (int i = 0; i < n; ++i) { rowsum[i].re = 0.0; rowsum[i].im = 0.0; }
  cplx total = zero;
  int neg = 0;
  uint64_t steps = (1ull << n) - 1;
  for (uint64_t k = 1; k <= steps; ++k) {
    int t = ctz64(k);
    uint64_t g = k ^ (k >> 1);
    if ((g >> t) & 1) {
      for (int i = 0; i < n; ++i) rowsum[i] = c_add(rowsum[i], a[i * n + t]);
    } else {
      for (int i = 0; i < n; ++i) rowsum[i] = c_sub(rowsum[i], a[i * n + t]);
    }
    cplx p = one;
    for (int i = 0; i < n; ++i) p = c_mul(p, rowsum[i]);
    neg = !neg;
    if (neg) total = c_sub(total, p); else total = c_add(total, p);
  }
  if (n & 1) { total.re = -total.re; total.im = -total.im; }
  out[0] = total.re; out[1] = total.im;
}

/* ryser_sq_int: src/_kernels.py:148-218. */
int orc_ryser_sq_i64(int n, const int64_t* a, int64_t* out) {
  int64_t rowsum[64];
  for (int i = 0; i < n; ++i) rowsum[i] = 0;
  int64_t total = 0;
  int neg = 0;
  uint64_t steps = (1ull << n) - 1;
  *out = 0;
  for (uint64_t k = 1; k <= steps; ++k) {
    int t = ctz64(k);
    uint64_t g = k ^ (k >> 1);
    if ((g >> t) & 1) {
      for (int i = 0; i < n; ++i) if (CHK_ADD(rowsum[i], a[i * n + t], &rowsum[i])) return 1;
    } else {
      for (int i = 0; i < n; ++i) if (CHK_SUB(rowsum[i], a[i * n + t], &rowsum[i])) return 1;
    }
    int64_t p = 1;
    for (int i = 0; i < n; ++i) {
      int64_t x = p, y = rowsum[i];
      if (x == 0 || y == 0) { p = 0; break; }
      if (CHK_MUL(x, y, &p)) return 1;
    }
    neg = !neg;
    if (neg) { if (CHK_SUB(total, p, &total)) return 1; }
    else { if (CHK_ADD(total, p, &total)) return 1; }
  }
  if (n & 1) total = -total; /* |total| < 2^63 here; -MIN cannot occur for n>=1 */
  *out = total;
  return 0;
}

/* Binomial C(a, b) exactly, or -1 when it exceeds int64 (the running
 * product C(a-b+i, i) stays exact: each step is an exact division). */
static int64_t binom_i64(int a, int b) {
  if (b < 0 || b > a) return 0;
  u128 r = 1;
  for (int i = 1; i <= b; ++i) {
    if (r > ((u128)1 << 120) / (u128)(a - b + i)) return -1;
    r = r * (u128)(a - b + i) / (u128)i;
  }
  return r > (u128)INT64_MAX ? -1 : (int64_t)r;
}

/* _ryser_weights (src/algorithms.py:110-115) converted to float64 the way
 * np.array(weights, dtype=float64) does (correctly rounded). */
static void ryser_weights_f64(int m, int n, double* w) {
  for (int s = 0; s <= m; ++s) w[s] = 0.0;
  for (int s = 1; s <= m; ++s) {
    int64_t c = binom_i64(n - s, m - s);
    w[s] = ((m - s) & 1) ? -(double)c : (double)c;
  }
}

/* ryser_rect: src/_kernels.py:226-262; weights as src/algorithms.py:110-115. */
double orc_ryser_rect_f64(int m, int n, const double* a) {
  double w[65];
  ryser_weights_f64(m, n, w);
  double zero = a[0] - a[0];
  int64_t comb[64];
  double rowsum[64];
  double total = zero;
  for (int s = m; s >= 1; --s) {
    for (int q = 0; q < s; ++q) comb[q] = q;
    for (int i = 0; i < m; ++i) {
      double acc = zero;
      for (int q = 0; q < s; ++q) acc = acc + a[i * n + comb[q]];
      rowsum[i] = acc;
    }
    double size_sum = zero;
    for (;;) {
      double p = zero + 1.0;
      for (int i = 0; i < m; ++i) p = p * rowsum[i];
      size_sum = size_sum + p;
      int pos = s - 1;
      while (pos >= 0 && comb[pos] == n - s + pos) pos -= 1;
      if (pos < 0) break;
      for (int q = pos; q < s; ++q) {
        int64_t c = comb[q];
        for (int i = 0; i < m; ++i) rowsum[i] = rowsum[i] - a[i * n + c];
      }
      int64_t v = comb[pos] + 1;
      for (int q = pos; q < s; ++q) {
        comb[q] = v + (q - pos);
        int64_t c = comb[q];
        for (int i = 0; i < m; ++i) rowsum[i] = rowsum[i] + a[i * n + c];
      }
    }
    total = total + w[s] * size_sum;
  }
  return total;
}

void orc_ryser_rect_c128(int m, int n, const double* a_, double* out) {
  const cplx* a = (const cplx*)a_;
  double wr[65];
  ryser_weights_f64(m, n, wr);
  cplx zero = c_sub(a[0], a[0]);
  cplx one = {zero.re + 1.0, zero.im + 0.0};
  int64_t comb[64];
  cplx rowsum[64];
  cplx total = zero;
  for (int s = m; s >= 1; --s) {
    for (int q = 0; q < s; ++q) comb[q] = q;
    for (int i = 0; i < m; ++i) {
      cplx acc = zero;
      for (int q = 0; q < s; ++q) acc = c_add(acc, a[i * n + comb[q]]);
      rowsum[i] = acc;
    }
    cplx size_sum = zero;
    for (;;) {
      cplx p = one;
      for (int i = 0; i < m; ++i) p = c_mul(p, rowsum[i]);
      size_sum = c_add(size_sum, p);
      int pos = s - 1;
      while (pos >= 0 && comb[pos] == n - s + pos) pos -= 1;
      if (pos < 0) break;
      for (int q = pos; q < s; ++q) {
        int64_t c = comb[q];
        for (int i = 0; i < m; ++i) rowsum[i] = c_sub(rowsum[i], a[i * n + c]);
      }
      int64_t v = comb[pos] + 1;
      for (int q = pos; q < s; ++q) {
        comb[q] = v + (q - pos);
        int64_t c = comb[q];
        for (int i = 0; i < m; ++i) rowsum[i] = c_add(rowsum[i], a[i * n + c]);
      }
    }
    cplx w = {wr[s], 0.0};
    total = c_add(total, c_mul(w, size_sum));
  }
  out[0] = total.re; out[1] = total.im;
}

/* ryser_rect_int: src/_kernels.py:265-365; a weight above int64 is the
 * src/algorithms.py:129-130 overflow. */
int orc_ryser_rect_i64(int m, int n, const int64_t* a, int64_t* out) {
  int64_t w[65];
  for (int s = 1; s <= m; ++s) {
    int64_t c = binom_i64(n - s, m - s);
    if (c < 0) { *out = 0; return 1; }
    w[s] = ((m - s) & 1) ? -c : c;
  }
  int64_t comb[64];
  int64_t rowsum[64];
  int64_t total = 0;
  *out = 0;
  for (int s = m; s >= 1; --s) {
    for (int q = 0; q < s; ++q) comb[q] = q;
    for (int i = 0; i < m; ++i) {
      int64_t acc = 0;
      for (int q = 0; q < s; ++q) if (CHK_ADD(acc, a[i * n + comb[q]], &acc)) return 1;
      rowsum[i] = acc;
    }
    int64_t size_sum = 0;
    for (;;) {
      int64_t p = 1;
      for (int i = 0; i < m; ++i) {
        int64_t x = p, y = rowsum[i];
        if (x == 0 || y == 0) { p = 0; break; }
        if (CHK_MUL(x, y, &p)) return 1;
      }
      if (CHK_ADD(size_sum, p, &size_sum)) return 1;
      int pos = s - 1;
      while (pos >= 0 && comb[pos] == n - s + pos) pos -= 1;
      if (pos < 0) break;
      for (int q = pos; q < s; ++q) {
        int64_t c = comb[q];
        for (int i = 0; i < m; ++i) if (CHK_SUB(rowsum[i], a[i * n + c], &rowsum[i])) return 1;
      }
      int64_t v = comb[pos] + 1;
      for (int q = pos; q < s; ++q) {
        comb[q] = v + (q - pos);
        int64_t c = comb[q];
        for (int i = 0; i < m; ++i) if (CHK_ADD(rowsum[i], a[i * n + c], &rowsum[i])) return 1;
      }
    }
    int64_t p;
    if (CHK_MUL(w[s], size_sum, &p)) return 1;
    if (CHK_ADD(total, p, &total)) return 1;
  }
  *out = total;
  return 0;
}

/* glynn_sq: src/_kernels.py:373-409 (raw accumulator). */
double orc_glynn_sq_f64(int n, const double* a) {
  double zero = a[0] - a[0];
  double colsum[64];
  for (int j = 0; j < n; ++j) {
    double acc = zero;
    for (int i = 0; i < n; ++i) acc = acc + a[i * n + j];
    colsum[j] = acc;
  }
  double total = zero + 1.0;
  for (int j = 0; j < n; ++j) total = total * colsum[j];
  int neg = 0;
  uint64_t steps = (1ull << (n - 1)) - 1;
  for (uint64_t k = 1; k <= steps; ++k) {
    int t = ctz64(k);
    int i = n - 1 - t;
    uint64_t g = k ^ (k >> 1);
    if ((g >> t) & 1) {
      for (int j = 0; j < n; ++j) colsum[j] = colsum[j] - (a[i * n + j] + a[i * n + j]);
    } else {
      for (int j = 0; j < n; ++j) colsum[j] = colsum[j] + (a[i * n + j] + a[i * n + j]);
    }
    double p = zero + 1.0;
    for (int j = 0; j < n; ++j) p = p * colsum[j];
    neg = !neg;
    if (neg) total = total - p; else total = total + p;
  }
  return total;
}

void orc_glynn_sq_c128(int n, const double* a_, double* out) {
  const cplx* a = (const cplx*)a_;
  cplx zero = c_sub(a[0], a[0]);
  cplx one = {zero.re + 1.0, zero.im + 0.0};
  cplx colsum[64];
  for (int j = 0; j < n; ++j) {
    cplx acc = zero;
    for (int i = 0; i < n; ++i) acc = c_add(acc, a[i * n + j]);
    colsum[j] = acc;
  }
  cplx total = one;
  for (int j = 0; j < n; ++j) total = c_mul(total, colsum[j]);
  int neg = 0;
  uint64_t steps = (1ull << (n - 1)) - 1;
  for (uint64_t k = 1; k <= steps; ++k) {
    int t = ctz64(k);
    int i = n - 1 - t;
    uint64_t g = k ^ (k >> 1);
    if ((g >> t) & 1) {
      for (int j = 0; j < n; ++j) colsum[j] = c_sub(colsum[j], c_add(a[i * n + j], a[i * n + j]));
    } else {
      for (int j = 0; j < n; ++j) colsum[j] = c_add(colsum[j], c_add(a[i * n + j], a[i * n + j]));
    }
    cplx p = one;
    for (int j = 0; j < n; ++j) p = c_mul(p, colsum[j]);
    neg = !neg;
    if (neg) total = c_sub(total, p); else total = c_add(total, p);
  }
  out[0] = total.re; out[1] = total.im;
}

/* glynn_sq_int: src/_kernels.py:412-523. */
int orc_glynn_sq_i64(int n, const int64_t* a, int64_t* out) {
  int64_t colsum[64];
  *out = 0;
  for (int j = 0; j < n; ++j) {
    int64_t acc = 0;
    for (int i = 0; i < n; ++i) if (CHK_ADD(acc, a[i * n + j], &acc)) return 1;
    colsum[j] = acc;
  }
  int64_t total = 1;
  for (int j = 0; j < n; ++j) {
    int64_t x = total, y = colsum[j];
    if (x == 0 || y == 0) { total = 0; break; }
    if (CHK_MUL(x, y, &total)) return 1;
  }
  int neg = 0;
  uint64_t steps = (1ull << (n - 1)) - 1;
  for (uint64_t k = 1; k <= steps; ++k) {
    int t = ctz64(k);
    int i = n - 1 - t;
    uint64_t g = k ^ (k >> 1);
    int down = (int)((g >> t) & 1);
    for (int j = 0; j < n; ++j) {
      int64_t y = a[i * n + j], d2;
      if (CHK_ADD(y, y, &d2)) return 1;
      if (down) { if (CHK_SUB(colsum[j], d2, &colsum[j])) return 1; }
      else { if (CHK_ADD(colsum[j], d2, &colsum[j])) return 1; }
    }
    int64_t p = 1;
    for (int j = 0; j < n; ++j) {
      int64_t x = p, y = colsum[j];
      if (x == 0 || y == 0) { p = 0; break; }
      if (CHK_MUL(x, y, &p)) return 1;
    }
    neg = !neg;
    if (neg) { if (CHK_SUB(total, p, &total)) return 1; }
    else { if (CHK_ADD(total, p, &total)) return 1; }
  }
  *out = total;
  return 0;
}

/* glynn_rect: src/_kernels.py:531-577 (virtual all-ones rows m..n-1). */
double orc_glynn_rect_f64(int m, int n, const double* a) {
  double zero = a[0] - a[0];
  double two = zero + 2.0;
  double colsum[64];
  double pad = zero + (double)(n - m);
  for (int j = 0; j < n; ++j) {
    double acc = pad;
    for (int i = 0; i < m; ++i) acc = acc + a[i * n + j];
    colsum[j] = acc;
  }
  double total = zero + 1.0;
  for (int j = 0; j < n; ++j) total = total * colsum[j];
  int neg = 0;
  uint64_t steps = (1ull << (n - 1)) - 1;
  for (uint64_t k = 1; k <= steps; ++k) {
    int t = ctz64(k);
    int i = n - 1 - t;
    uint64_t g = k ^ (k >> 1);
    if ((g >> t) & 1) {
      if (i < m) for (int j = 0; j < n; ++j) colsum[j] = colsum[j] - (a[i * n + j] + a[i * n + j]);
      else for (int j = 0; j < n; ++j) colsum[j] = colsum[j] - two;
    } else {
      if (i < m) for (int j = 0; j < n; ++j) colsum[j] = colsum[j] + (a[i * n + j] + a[i * n + j]);
      else for (int j = 0; j < n; ++j) colsum[j] = colsum[j] + two;
    }
    double p = zero + 1.0;
    for (int j = 0; j < n; ++j) p = p * colsum[j];
    neg = !neg;
    if (neg) total = total - p; else total = total + p;
  }
  return total;
}

void orc_glynn_rect_c128(int m, int n, const double* a_, double* out) {
  const cplx* a = (const cplx*)a_;
  cplx zero = c_sub(a[0], a[0]);
  cplx one = {zero.re + 1.0, zero.im + 0.0};
  cplx two = {zero.re + 2.0, zero.im + 0.0};
  cplx pad = {zero.re + (double)(n - m), zero.im + 0.0};
  cplx colsum[64];
  for (int j = 0; j < n; ++j) {
    cplx acc = pad;
    for (int i = 0; i < m; ++i) acc = c_add(acc, a[i * n + j]);
    colsum[j] = acc;
  }
  cplx total = one;
  for (int j = 0; j < n; ++j) total = c_mul(total, colsum[j]);
  int neg = 0;
  uint64_t steps = (1ull << (n - 1)) - 1;
  for (uint64_t k = 1; k <= steps; ++k) {
    int t = ctz64(k);
    int i = n - 1 - t;
    uint64_t g = k ^ (k >> 1);
    if ((g >> t) & 1) {
      if (i < m) for (int j = 0; j < n; ++j) colsum[j] = c_sub(colsum[j], c_add(a[i * n + j], a[i * n + j]));
      else for (int j = 0; j < n; ++j) colsum[j] = c_sub(colsum[j], two);
    } else {
      if (i < m) for (int j = 0; j < n; ++j) colsum[j] = c_add(colsum[j], c_add(a[i * n + j], a[i * n + j]));
      else for (int j = 0; j < n; ++j) colsum[j] = c_add(colsum[j], two);
    }
    cplx p = one;
    for (int j = 0; j < n; ++j) p = c_mul(p, colsum[j]);
    neg = !neg;
    if (neg) total = c_sub(total, p); else total = c_add(total, p);
  }
  out[0] = total.re; out[1] = total.im;
}

/* glynn_rect_int: src/_kernels.py:580-697. */
int orc_glynn_rect_i64(int m, int n, const int64_t* a, int64_t* out) {
  int64_t colsum[64];
  int64_t pad = n - m;
  *out = 0;
  for (int j = 0; j < n; ++j) {
    int64_t acc = pad;
    for (int i = 0; i < m; ++i) if (CHK_ADD(acc, a[i * n + j], &acc)) return 1;
    colsum[j] = acc;
  }
  int64_t total = 1;
  for (int j = 0; j < n; ++j) {
    int64_t x = total, y = colsum[j];
    if (x == 0 || y == 0) { total = 0; break; }
    if (CHK_MUL(x, y, &total)) return 1;
  }
  int neg = 0;
  uint64_t steps = (1ull << (n - 1)) - 1;
  for (uint64_t k = 1; k <= steps; ++k) {
    int t = ctz64(k);
    int i = n - 1 - t;
    uint64_t g = k ^ (k >> 1);
    int down = (int)((g >> t) & 1);
    if (i < m) {
      for (int j = 0; j < n; ++j) {
        int64_t y = a[i * n + j], d2;
        if (CHK_ADD(y, y, &d2)) return 1;
        if (down) { if (CHK_SUB(colsum[j], d2, &colsum[j])) return 1; }
        else { if (CHK_ADD(colsum[j], d2, &colsum[j])) return 1; }
      }
    } else {
      for (int j = 0; j < n; ++j) {
        if (down) { if (CHK_SUB(colsum[j], (int64_t)2, &colsum[j])) return 1; }
        else { if (CHK_ADD(colsum[j], (int64_t)2, &colsum[j])) return 1; }
      }
    }
    int64_t p = 1;
    for (int j = 0; j < n; ++j) {
      int64_t x = p, y = colsum[j];
      if (x == 0 || y == 0) { p = 0; break; }
      if (CHK_MUL(x, y, &p)) return 1;
    }
    neg = !neg;
    if (neg) { if (CHK_SUB(total, p, &total)) return 1; }
    else { if (CHK_ADD(total, p, &total)) return 1; }
  }
  *out = total;
  return 0;
}

/* ======================================================================
 * 2. Gray-range forms.
 *
 * The generic walk of SURVEY Appendix A: a state vector v of length P is
 * seeded at Gray index k0 as v = v0 + sum_{t : bit t of gray(k0)} U[t], and
 * step k flips Gray bit t = ctz(k): v += U[t] if bit t of gray(k) is set,
 * else v -= U[t].  The term of step k is sign(k) * prod(v).
 *   Glynn (square, or rectangular on the ones-padded n x n matrix):
 *     P = n, B = n-1 Gray bits, v0 = column sums, U[t] = -2 * row (n-1-t),
 *     sign(k) = (-1)^k, per = sum / 2^(n-1) [/ (n-m)!]
 *     (src/_kernels.py:373-409, 531-577; flip row n-1-ctz(k) at :393).
 *   Ryser (square): P = n, B = n, v0 = 0, U[t] = column t, sign(k) = (-1)^k,
 *     per = (-1)^n * sum  (src/_kernels.py:115-145).
 *   Ryser (rectangular, over all 2^n subsets): P = m, B = n, v0 = 0,
 *     U[t] = column t, term weight w[popcount(gray(k))] with
 *     w[s] = (-1)^(m-s) C(n-s, m-s) for s <= m and 0 above
 *     (equivalent form of src/_kernels.py:226-262).
 * Summing the terms over any partition of [0, 2^B) into contiguous ranges
 * gives the whole walk (the sharding identity).
 * ====================================================================== */

typedef struct {
  int P, B;           /* product length, Gray bits */
  int weighted;       /* 0: sign (-1)^k ; 1: w[popcount(gray(k))] */
} walk_t;

/* f64 range: plain sequential sum, as the reference accumulates. */
double orc_walk_f64_range(int P, int B, const double* v0, const double* U /*[B][P]*/,
                          int weighted, const double* w, uint64_t k0, uint64_t k1) {
  double v[64];
  uint64_t g0 = k0 ^ (k0 >> 1);
  for (int j = 0; j < P; ++j) v[j] = v0[j];
  for (int t = 0; t < B; ++t)
    if ((g0 >> t) & 1) for (int j = 0; j < P; ++j) v[j] = v[j] + U[t * P + j];
  int pc = __builtin_popcountll(g0);
  double total = 0.0;
  for (uint64_t k = k0; k < k1; ++k) {
    if (k != k0) {
      int t = ctz64(k);
      uint64_t g = k ^ (k >> 1);
      if ((g >> t) & 1) { for (int j = 0; j < P; ++j) v[j] = v[j] + U[t * P + j]; ++pc; }
      else { for (int j = 0; j < P; ++j) v[j] = v[j] - U[t * P + j]; --pc; }
    }
    double p = 1.0;
    for (int j = 0; j < P; ++j) p = p * v[j];
    if (weighted) total = total + w[pc] * p;
    else if (k & 1) total = total - p; else total = total + p;
  }
  return total;
}

/* Double-double helpers (Dekker/Knuth error-free transforms; -ffp-contract
 * =off keeps them exact; fma() is used explicitly for the product error). */
typedef struct { double hi, lo; } dd;
static inline dd two_sum(double a, double b) {
  double s = a + b, bb = s - a, e = (a - (s - bb)) + (b - bb);
  dd r = {s, e};
  return r;
}
static inline dd quick_two_sum(double a, double b) {
  double s = a + b, e = b - (s - a);
  dd r = {s, e};
  return r;
}
static inline dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
static inline dd dd_neg(dd a) { dd r = {-a.hi, -a.lo}; return r; }
static inline dd dd_mul(dd a, dd b) {
  double p = a.hi * b.hi, e = fma(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p, e);
}
static inline dd dd_from(double x) { dd r = {x, 0.0}; return r; }

typedef struct { dd re, im; } cdd;
static inline cdd cdd_add(cdd a, cdd b) { cdd r = {dd_add(a.re, b.re), dd_add(a.im, b.im)}; return r; }
static inline cdd cdd_sub(cdd a, cdd b) { cdd r = {dd_add(a.re, dd_neg(b.re)), dd_add(a.im, dd_neg(b.im))}; return r; }
static inline cdd cdd_mul(cdd a, cdd b) {
  cdd r = {dd_add(dd_mul(a.re, b.re), dd_neg(dd_mul(a.im, b.im))),
           dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re))};
  return r;
}

/* double-double range walk, real (cplx = 0) or complex (cplx = 1; v0/U/w
 * interleaved re,im).  The state is re-seeded exactly (in dd) at k0, so
 * colsum drift is at the dd level.  out: [re_hi, re_lo, im_hi, im_lo,
 * mag_hi, mag_lo], mag = sum_k |w_k| |term_k| (the raw magnitude sum behind
 * the scale of SURVEY 8(c) metric (ii); |complex| from the dd parts rounded
 * to double). */
void orc_walk_dd_range(int P, int B, int is_cplx, const double* v0, const double* U,
                       int weighted, const double* w, uint64_t k0, uint64_t k1, double* out) {
  cdd v[64];
  cdd total = {{0, 0}, {0, 0}};
  dd mag = {0, 0};
  uint64_t g0 = k0 ^ (k0 >> 1);
  int st = is_cplx ? 2 : 1;
  for (int j = 0; j < P; ++j) {
    v[j].re = dd_from(v0[j * st]);
    v[j].im = dd_from(is_cplx ? v0[j * st + 1] : 0.0);
  }
  for (int t = 0; t < B; ++t)
    if ((g0 >> t) & 1)
      for (int j = 0; j < P; ++j) {
        cdd u = {dd_from(U[(t * P + j) * st]), dd_from(is_cplx ? U[(t * P + j) * st + 1] : 0.0)};
        v[j] = cdd_add(v[j], u);
      }
  int pc = __builtin_popcountll(g0);
  for (uint64_t k = k0; k < k1; ++k) {
    if (k != k0) {
      int t = ctz64(k);
      uint64_t g = k ^ (k >> 1);
      int set = (int)((g >> t) & 1);
      for (int j = 0; j < P; ++j) {
        cdd u = {dd_from(U[(t * P + j) * st]), dd_from(is_cplx ? U[(t * P + j) * st + 1] : 0.0)};
        v[j] = set ? cdd_add(v[j], u) : cdd_sub(v[j], u);
      }
      pc += set ? 1 : -1;
    }
    cdd p;
    if (is_cplx) {
      p = v[0];
      for (int j = 1; j < P; ++j) p = cdd_mul(p, v[j]);
    } else {
      p.re = v[0].re; p.im = dd_from(0.0);
      for (int j = 1; j < P; ++j) p.re = dd_mul(p.re, v[j].re);
    }
    if (weighted) {
      dd ww = dd_from(w[pc]);
      p.re = dd_mul(p.re, ww); p.im = dd_mul(p.im, ww);
      total = cdd_add(total, p);
    } else if (k & 1) total = cdd_sub(total, p);
    else total = cdd_add(total, p);
    if (is_cplx) mag = dd_add(mag, dd_from(hypot(p.re.hi + p.re.lo, p.im.hi + p.im.lo)));
    else mag = dd_add(mag, p.re.hi < 0 ? dd_neg(p.re) : p.re);
  }
  out[0] = total.re.hi; out[1] = total.re.lo; out[2] = total.im.hi; out[3] = total.im.lo;
  out[4] = mag.hi; out[5] = mag.lo;
}

/* Wrapping int128 range walk (mod 2^128 ring arithmetic).
 * v0/U are int64 and the caller guarantees |v| stays below 2^63 along the
 * walk (true for the bounded integer matrices of config C4).
 * out: [lo, hi] of the 128-bit two's-complement sum. */
void orc_walk_i128_range(int P, int B, const int64_t* v0, const int64_t* U,
                         int weighted, const int64_t* w, uint64_t k0, uint64_t k1, uint64_t* out) {
  int64_t v[64];
  uint64_t g0 = k0 ^ (k0 >> 1);
  for (int j = 0; j < P; ++j) v[j] = v0[j];
  for (int t = 0; t < B; ++t)
    if ((g0 >> t) & 1) for (int j = 0; j < P; ++j) v[j] += U[t * P + j];
  int pc = __builtin_popcountll(g0);
  u128 total = 0;
  for (uint64_t k = k0; k < k1; ++k) {
    if (k != k0) {
      int t = ctz64(k);
      uint64_t g = k ^ (k >> 1);
      if ((g >> t) & 1) { for (int j = 0; j < P; ++j) v[j] += U[t * P + j]; ++pc; }
      else { for (int j = 0; j < P; ++j) v[j] -= U[t * P + j]; --pc; }
    }
    u128 p = (u128)(i128)v[0];
    for (int j = 1; j < P; ++j) p = p * (u128)(i128)v[j];
    if (weighted) total += p * (u128)(i128)w[pc];
    else if (k & 1) total -= p; else total += p;
  }
  out[0] = (uint64_t)total;
  out[1] = (uint64_t)(total >> 64);
}

/* ---------------- pthread drivers over contiguous sub-ranges ---------- */

typedef struct {
  int kind; /* 0 f64, 1 dd (real or complex), 2 i128 */
  int P, B, is_cplx, weighted;
  const void *v0, *U, *w;
  uint64_t k0, k1;
  double f64_out;
  double dd_out[6];
  uint64_t i128_out[2];
} job_t;

static void* job_run(void* arg) {
  job_t* j = (job_t*)arg;
  if (j->kind == 0)
    j->f64_out = orc_walk_f64_range(j->P, j->B, (const double*)j->v0, (const double*)j->U, j->weighted,
                                    (const double*)j->w, j->k0, j->k1);
  else if (j->kind == 1)
    orc_walk_dd_range(j->P, j->B, j->is_cplx, (const double*)j->v0, (const double*)j->U, j->weighted,
                      (const double*)j->w, j->k0, j->k1, j->dd_out);
  else
    orc_walk_i128_range(j->P, j->B, (const int64_t*)j->v0, (const int64_t*)j->U, j->weighted,
                        (const int64_t*)j->w, j->k0, j->k1, j->i128_out);
  return NULL;
}

/* Split [k0, k1) into `nthreads` contiguous ranges and combine in range
 * order.  f64: partials combined with a double-double sum (out[0..1]);
 * dd: out[0..3] = re hi/lo, im hi/lo; i128: out = (lo, hi) as two u64
 * (passed through a double* reinterpreted as uint64_t*). */
void orc_walk_mt(int kind, int P, int B, int is_cplx, int weighted, const void* v0, const void* U,
                 const void* w, uint64_t k0, uint64_t k1, int nthreads, void* out) {
  if (nthreads < 1) nthreads = 1;
  if ((uint64_t)nthreads > k1 - k0) nthreads = (int)(k1 - k0 ? k1 - k0 : 1);
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  uint64_t span = k1 - k0;
  for (int i = 0; i < nthreads; ++i) {
    job_t* j = &jobs[i];
    j->kind = kind; j->P = P; j->B = B; j->is_cplx = is_cplx; j->weighted = weighted;
    j->v0 = v0; j->U = U; j->w = w;
    j->k0 = k0 + (uint64_t)((u128)span * (u128)i / (u128)nthreads);
    j->k1 = k0 + (uint64_t)((u128)span * (u128)(i + 1) / (u128)nthreads);
    pthread_create(&th[i], NULL, job_run, j);
  }
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  if (kind == 0) {
    dd s = {0, 0};
    for (int i = 0; i < nthreads; ++i) s = dd_add(s, dd_from(jobs[i].f64_out));
    ((double*)out)[0] = s.hi; ((double*)out)[1] = s.lo;
  } else if (kind == 1) {
    cdd s = {{0, 0}, {0, 0}};
    dd mg = {0, 0};
    for (int i = 0; i < nthreads; ++i) {
      cdd x = {{jobs[i].dd_out[0], jobs[i].dd_out[1]}, {jobs[i].dd_out[2], jobs[i].dd_out[3]}};
      s = cdd_add(s, x);
      dd y = {jobs[i].dd_out[4], jobs[i].dd_out[5]};
      mg = dd_add(mg, y);
    }
    double* o = (double*)out;  /* 6 doubles */
    o[0] = s.re.hi; o[1] = s.re.lo; o[2] = s.im.hi; o[3] = s.im.lo; o[4] = mg.hi; o[5] = mg.lo;
  } else {
    u128 s = 0;
    for (int i = 0; i < nthreads; ++i) s += ((u128)jobs[i].i128_out[1] << 64) | jobs[i].i128_out[0];
    uint64_t* o = (uint64_t*)out;
    o[0] = (uint64_t)s; o[1] = (uint64_t)(s >> 64);
  }
  free(jobs);
  free(th);
}
