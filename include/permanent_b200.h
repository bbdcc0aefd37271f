/*
 * permanent_b200.h -- C ABI of the B200 exact-permanent engine
 * (libpermanent_b200.so, built from paper_2510_03421_b200/csrc/).
 *
 * The reference package (`permanent`, /root/reference/pkg/src/permanent) has
 * no native boundary: its engine seam is the kernel registry
 * `_kernels.get_kernel(name, compiled)` (src/_kernels.py:718-728), whose
 * callables are invoked only from the wrappers in src/algorithms.py
 * (:87-89, 104-106, 133-136, 152-159, 175-182).  Every entry point below
 * replaces one of those kernels *plus* its wrapper's normalization, so the
 * Python shim (paper_2510_03421_b200/) keeps the reference's public API
 * (src/__init__.py:55-111) and calls straight through.  Paths are relative to
 * /root/reference/pkg.
 *
 * Conventions
 *   - matrices are row-major m x n with row stride `lda` elements, m <= n
 *     (the caller transposes, as src/__init__.py:50-52 does);
 *   - complex128 is interleaved (re, im) doubles: numpy's complex128 layout;
 *   - `dev_ptr` = 1: `a` is a device pointer on the current device (read in
 *     place); 0: host memory (copied; never written);
 *   - `stream` is a cudaStream_t (NULL = per-thread default stream); calls
 *     that return a host value synchronize that stream;
 *   - every function returns a status:
 */
#ifndef PERMANENT_B200_H
#define PERMANENT_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PERM_OK = 0,
  PERM_OVERFLOW = 1,   /* int: an int64 intermediate overflowed (reference semantics)
                          or the exact value is not certified to fit */
  PERM_BAD_SHAPE = 2,  /* m > n, m < 1, n > 62, unsupported size */
  PERM_BUDGET = 3,     /* combinatoric step budget exceeded */
  PERM_CUDA = 4,       /* CUDA / NCCL runtime error (see perm_last_error) */
  PERM_BAD_ARG = 5
};

/* algorithm ids, same order as AlgorithmId in src/algorithms.py:26-31 */
enum { PERM_ALG_COMBINATORIC = 0, PERM_ALG_RYSER = 1, PERM_ALG_GLYNN = 2 };
/* batch-only formulas (perm_batch_*; no reference counterpart, exact algebra):
 * PARTITION = Moebius inversion over set partitions of the rows, m <= 6 (complex m <= 5);
 * LAPLACE = 4+4-row Laplace expansion from 2x2 row-pair permanents, 8x8 real. */
enum { PERM_ALG_BATCH_PARTITION = 3, PERM_ALG_BATCH_LAPLACE = 4 };

/* Library version (major*10000 + minor*100 + patch). */
int perm_version(void);
/* Message of the last failing call on this host thread ("" if none). */
const char* perm_last_error(void);
/* Select the CUDA device used by subsequent calls from this host thread. */
int perm_set_device(int device);
/* Number of SMs of the current device (planning helper). */
int perm_device_sm_count(void);
/* Instrumentation: device time (ms, CUDA events on the launching stream) of
 * the last Gray-walk kernel launched by this host thread (-1 if none), and
 * its launch plan (grid size, log2 of the per-lane chunk length). */
double perm_last_kernel_ms(void);
/* Enable (1) / disable (0) the CUDA-event bracketing of walk kernels read by
 * perm_last_kernel_ms (off by default: two event records per call). */
int perm_set_timing(int on);
int perm_last_kernel_plan(int* grid, int* log2L);
/* FP64-pipe roofline denominator: DFMA/s sustained by an 8-chain DFMA
 * kernel over the whole device for about `seconds`. */
int perm_fp64_peak_probe(double seconds, double* dfma_per_s);
/* op 0: DFMA (as above); op 1: alternating DADD / DMUL chains, the walk's
 * instruction mix -- on B200 it reaches the nominal 64 op/clk/SM while DFMA
 * tops out ~8% lower, so the walk's FP64-pipe roofline is op 1's figure. */
int perm_fp64_pipe_probe(int op, double seconds, double* ops_per_s);
/* Measurement: device time of the float Gray walk of one host matrix
 * (alg GLYNN / RYSER, cplx 0/1), launched `reps` times back to back on a
 * private stream after one warm-up -- the setup is built once, so the
 * figure is the kernel's per-permanent device time including the
 * launch-to-launch gap, without the per-call host work.  *ms_per_launch
 * receives the CUDA-event time divided by reps. */
int perm_walk_repeat_ms(int alg, int cplx, int m, int n, const double* a, int64_t lda, int reps,
                        double* ms_per_launch);

/* ---- single permanents, float64 / complex128 --------------------------
 * Replace glynn_sq/glynn_rect + permanent_glynn_{square,rectangular}
 * (src/_kernels.py:373-409, 531-577; src/algorithms.py:140-184):
 * `out` receives the *normalized* permanent (1 double, or re/im for c128).
 * Rectangular Glynn pre-scales the real rows by a power of two
 * (SURVEY 7.4.2), which is exact algebra.  `magsum` (optional, may be NULL)
 * receives M = the normalized sum of |terms|.
 * stream NULL with a host matrix: the zero-copy route (the walk setup passed
 * as kernel parameters up to 5.5 KB, the result through mapped pinned memory
 * and a release-store flag); a caller's stream keeps stream-ordered staged
 * copies.  Like the reference's kernels, whose sums start at
 * a[0,0] - a[0,0], a non-finite a[0,0] gives NaN (real / imaginary part). */
int perm_glynn_f64(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, double* magsum,
                   void* stream);
int perm_glynn_c128(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, double* magsum,
                    void* stream);
/* Replace ryser_sq / ryser_rect + permanent_ryser_{square,rectangular}
 * (src/_kernels.py:115-145, 226-262; src/algorithms.py:93-137).  The
 * rectangular form walks all 2^n column subsets with the binomial weight of
 * each subset size (src/algorithms.py:110-115). */
int perm_ryser_f64(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, double* magsum,
                   void* stream);
int perm_ryser_c128(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, double* magsum,
                    void* stream);

/* The reference's rectangular Ryser kernel for any m <= n, square included
 * (permanent_ryser_rectangular accepts m == n, src/algorithms.py:118-137;
 * ryser_rect / ryser_rect_int, src/_kernels.py:226-365): subset sizes
 * s = m..1 in lexicographic combination order, weights (-1)^(m-s) C(n-s, m-s).
 * n up to 256 columns (the reference caps only its Gray walks at 62).
 * i64 = checked int64, PERM_OVERFLOW exactly where ryser_rect_int reports
 * overflow; out[0], out[1] = low, high 64 bits. */
int perm_ryser_rect_f64(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, void* stream);
int perm_ryser_rect_c128(int m, int n, const double* a, int64_t lda, int dev_ptr, double* out, void* stream);
int perm_ryser_rect_i64(int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int64_t* out, void* stream);

/* ---- combinatoric (src/_kernels.py:28-56, 59-108; src/algorithms.py:71-90)
 * Depth-first enumeration of the m-permutations with prefix products and
 * zero pruning, the DFS tree split at a prefix depth across threads.
 * PERM_BUDGET when P(n, m) > step_budget (StepBudgetExceeded). */
int perm_comb_f64(int m, int n, const double* a, int64_t lda, int dev_ptr, uint64_t step_budget, double* out,
                  void* stream);
int perm_comb_c128(int m, int n, const double* a, int64_t lda, int dev_ptr, uint64_t step_budget, double* out,
                   void* stream);
/* Integer combinatoric: width 64 = comb_dfs_int (src/_kernels.py:59-108)
 * with its checked-int64 overflow semantics (PERM_OVERFLOW exactly where the
 * reference reports overflowed); width 128 = exact DFS in int128, certified a
 * priori (product of the row sums of |A| < 2^126, else PERM_OVERFLOW).
 * out[0], out[1] = low, high 64 bits; *fits_int64 set (may be NULL). */
int perm_comb_i64(int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, uint64_t step_budget,
                  int64_t* out, int* fits_int64, void* stream);

/* ---- exact integer path (north_star item 3) -----------------------------
 * width = 64: the reference's checked-int64 semantics bit for bit
 *   (glynn_sq_int / glynn_rect_int / ryser_sq_int / ryser_rect_int,
 *   src/_kernels.py:148-365, 412-697, and the exact-division checks of
 *   src/algorithms.py:150-181): PERM_OVERFLOW exactly when the reference
 *   reports overflowed=True (its OverflowError, src/__init__.py:43-47).
 * width = 128: exact permanent via a mod-2^128 walk, certified to fit by an
 *   FP64 run and its magnitude-sum error bound; PERM_OVERFLOW if the
 *   certificate fails.
 * out[0], out[1] = low, high 64 bits (two's complement); *fits_int64 set. */
int perm_glynn_i64(int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, int64_t* out,
                   int* fits_int64, void* stream);
int perm_ryser_i64(int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width, int64_t* out,
                   int* fits_int64, void* stream);

/* ---- batched small matrices (north_star item 4; no reference counterpart:
 * the reference evaluates one matrix per Python call) --------------------
 * a = [B][m][n] row-major contiguous (host, or device if dev_ptr = 1),
 * out = [B] (same memory space).  alg = PERM_ALG_* (incl. the batch-only
 * formulas) or -1 for the batch dispatch (perm_batch_select: LAPLACE for 8x8
 * real, Glynn for other squares, PARTITION for m <= 4 < n and for m = 5, 6
 * with n >= m + 2, Glynn on the ones-padded pre-scaled matrix for the other
 * rectangles with n >= 9, subset-skipping Ryser otherwise).  PARTITION / LAPLACE stream the batch through shared
 * memory with 1-D bulk copies (persistent grid); other algorithms run one
 * thread (or warp) per matrix.
 * Requires m <= n <= 16, except Glynn up to n = 30 (square, or rectangular
 * on the ones-padded 2^s-scaled matrix) -- every matrix's Gray walk split
 * into segments over one launch (walk_multi_kernel), combined per matrix in
 * segment order -- and PARTITION up to n = 62 (m <= 6, complex m <= 5).
 * Device-pointer calls are asynchronous on `stream`. */
int perm_batch_f64(int alg, int64_t B, int m, int n, const double* a, double* out, int dev_ptr, void* stream);
int perm_batch_c128(int alg, int64_t B, int m, int n, const double* a, double* out, int dev_ptr, void* stream);
int perm_batch_select(int m, int n);

/* ---- sharded walks (one Gray range per GPU / rank) --------
 * perm_walk_steps: length of the Gray index space of (alg, m, n): 2^(n-1)
 * for Glynn, 2^n for Ryser.  perm_walk_shard: the [k_begin, k_end) of
 * `rank` out of `world`, aligned so every shard runs the full-speed kernel.
 * perm_walk_partial_*: raw compensated partial sum over one range, written
 * as 8 doubles {re_hi, re_lo, im_hi, im_lo, mag, 0, 0, 0} to `partial`
 * (host memory, or device memory when partial_on_device = 1, in which case
 * the call is asynchronous on `stream`).
 * perm_walk_finish_*: combine G partials in rank order (double-double) and
 * apply the algorithm's normalization -> the permanent (and M). */
uint64_t perm_walk_steps(int alg, int m, int n);
int perm_walk_shard(int alg, int m, int n, int rank, int world, uint64_t* k_begin, uint64_t* k_end);
int perm_walk_partial_f64(int alg, int m, int n, const double* a, int64_t lda, int dev_ptr, uint64_t k_begin,
                          uint64_t k_end, int mag, double* partial, int partial_on_device, void* stream);
int perm_walk_partial_c128(int alg, int m, int n, const double* a, int64_t lda, int dev_ptr, uint64_t k_begin,
                           uint64_t k_end, int mag, double* partial, int partial_on_device, void* stream);
int perm_walk_finish_f64(int alg, int m, int n, const double* a, int64_t lda, const double* partials, int G,
                         double* out, double* magsum);
int perm_walk_finish_c128(int alg, int m, int n, const double* a, int64_t lda, const double* partials, int G,
                          double* out, double* magsum);

/* Exact integer shards.  width 64: the checked-int64 walk of one range,
 * summarized as (sum, min/max running prefix, overflow flag) so that
 * perm_walk_finish_i64 reproduces the reference's overflow flag exactly
 * across shards (combined in rank order); not available for rectangular
 * Ryser, whose checked kernel follows the lexicographic combination order
 * (src/_kernels.py:265-365).  width 128: the range's walk sum mod 2^128
 * plus its FP64 estimate and magnitude sum; the finish certifies the total
 * fits and checks it against the summed estimate.  partial = 8 int64
 * (opaque, tagged with the width).  finish: out[0..1] = lo/hi, as
 * perm_glynn_i64. */
int perm_walk_partial_i64(int alg, int m, int n, const int64_t* a, int64_t lda, int dev_ptr, int width,
                          uint64_t k_begin, uint64_t k_end, int64_t* partial, void* stream);
int perm_walk_finish_i64(int alg, int m, int n, const int64_t* a, int64_t lda, int width, const int64_t* partials,
                         int G, int64_t* out, int* fits_int64);
/* Host-only planning query (no CUDA call): which exact width-128 walk the
 * full Gray range of this host matrix takes.  *kind = 4 / 3: quad walk
 * (FP32 quads under FP64 / integer upper levels), 1: FP64-exact groups,
 * 0: generic 128-bit state; *groups = quads or FP64 groups per step.  The
 * walks replace src/_kernels.py:412-523 (glynn_int / ryser_int) and are all
 * exact; the plan only decides which pipes carry the products. */
int perm_int_walk_plan(int alg, int m, int n, const int64_t* a, int64_t lda, int* kind, int* groups);

/* ---- single-process multi-device driver (SURVEY 8(b) perm_sharded_*) -----
 * One permanent over `ngpu` devices from one host process: shard i (of
 * perm_walk_shard(i, ngpu)) runs on devices[i] from a persistent host worker,
 * the caller combines in shard order.  `a` is host memory.  A device may be
 * listed more than once (its shards then share it).  Synchronous. */
int perm_sharded_f64(int alg, int m, int n, const double* a, int64_t lda, int ngpu, const int* devices, double* out,
                     double* magsum);
int perm_sharded_c128(int alg, int m, int n, const double* a, int64_t lda, int ngpu, const int* devices,
                      double* out, double* magsum);
int perm_sharded_i64(int alg, int m, int n, const int64_t* a, int64_t lda, int width, int ngpu, const int* devices,
                     int64_t* out, int* fits_int64);
/* Exchange the float drivers will use for this device list: 1 = NCCL
 * (ncclCommInitAll clique + one grouped ncclAllGather of the partials; the
 * default for >= 2 distinct devices when libnccl.so.2 loads), 0 = pinned
 * host memory (a device listed twice, no NCCL, or PERM_SHARDED_EXCHANGE=host),
 * -1 = bad arguments.  The integer driver always exchanges through the host
 * (its partials are read back to certify the int128 fit). */
int perm_sharded_exchange(int ngpu, const int* devices);

/* ---- double-double validation walks -------------
 * Glynn or Ryser with double-double state, products and sums (~1e-30 unit
 * roundoff): the GPU cross-check where the reference cannot run and FP64
 * Ryser is ill-conditioned.  out4 = {re_hi, re_lo, im_hi, im_lo} of the
 * normalized permanent.  Synchronous; several times slower than the FP64
 * walk (not a benchmark path). */
int perm_permanent_dd(int alg, int cplx, int m, int n, const double* a, int64_t lda, int dev_ptr, double* out4,
                      void* stream);

/* ---- dispatch (src/dispatch.py:84-95) -----------------------------------
 * The reference's selection rule over (m, n) with parameters p[0..7] =
 * p1..p8; returns PERM_ALG_*.  batch/ngpu are reserved (0). */
int perm_select(int m, int n, const double* p, int64_t batch, int ngpu);

#ifdef __cplusplus
}
#endif
#endif /* PERMANENT_B200_H */
