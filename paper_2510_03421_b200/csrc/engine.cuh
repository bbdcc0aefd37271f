// Host-side engine internals shared by the C-ABI translation units:
// error state, per-thread device scratch, matrix staging, walk setup.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/permanent_b200.h"
#include "walk_launch.cuh"

namespace permb200 {

// ---- errors --------------------------------------------------------------
void set_error(const std::string& msg);
void clear_error();
int cuda_fail(cudaError_t e, const char* what);

#define PERM_CUDA_TRY(expr)                                      \
  do {                                                           \
    cudaError_t _e = (expr);                                     \
    if (_e != cudaSuccess) return ::permb200::cuda_fail(_e, #expr); \
  } while (0)

// ---- per-(thread, device) scratch ----------------------------------------
struct Scratch {
  int device = -1;
  void* dev = nullptr;       // device scratch
  size_t dev_cap = 0;
  double* host = nullptr;    // pinned host result buffer (kHostResultDoubles)
  void* stage = nullptr;     // pinned host staging buffer for H2D copies
  size_t stage_cap = 0;
  unsigned int* done = nullptr;  // walk kernels' last-block counter (device)
  bool async_pending = false;    // a device-output call may still be running
  cudaStream_t own = nullptr;
  // mapped pinned result slot of the zero-copy single-walk path: the walk's
  // last block writes 8 doubles here and then flag = seq (walk.cuh)
  double* mres_host = nullptr;
  double* mres_dev = nullptr;
  unsigned int* mflag_host = nullptr;
  unsigned int* mflag_dev = nullptr;
  unsigned int mseq = 0;
};
constexpr size_t kHostResultDoubles = 16384;    // pinned result buffer size
Scratch* scratch();                              // for the current device
// copy host bytes to device through the pinned staging buffer (async DMA)
int stage_h2d(Scratch* s, void* dst, const void* src, size_t bytes, cudaStream_t stream);
int ensure_dev(Scratch* s, size_t bytes);        // grow device scratch
cudaStream_t pick_stream(void* stream);

// ---- matrices --------------------------------------------------------------
// A dense row-major copy in host memory (doubles; complex interleaved).
struct HostMat {
  int m = 0, n = 0;
  bool cplx = false;
  std::vector<double> d;  // m*n*(cplx?2:1)
  double re(int i, int j) const { return cplx ? d[2 * ((size_t)i * n + j)] : d[(size_t)i * n + j]; }
  double im(int i, int j) const { return cplx ? d[2 * ((size_t)i * n + j) + 1] : 0.0; }
};
int load_matrix(int m, int n, const double* a, int64_t lda, int dev_ptr, bool cplx, HostMat* out,
                cudaStream_t stream);

// ---- walk setup --------------------------------------
struct WalkSetup {
  int P = 0, B = 0;
  bool weighted = false;
  bool cplx = false;
  int scale_log2 = 0;                // Glynn rectangular pre-scale k = 2^scale_log2
  std::vector<double> buf;           // v0 [P], U [B][P] (complex interleaved), then w [n+1]
  size_t v0_off = 0, U_off = 0, w_off = 0;  // offsets in doubles
  int wlen = 0;
  bool exact = false;                // state lines on the exact grid (no re-seeding needed)
};
// exact_state: round each state line (Glynn column / Ryser row) to a grid on
// which every walk state is exact (the float walks; not the double-double
// validation walks, which see the matrix as given).
int build_walk(int alg, const HostMat& A, WalkSetup* ws, bool exact_state = false);
// Power-of-two pre-scale exponent for rectangular Glynn: round(-log2(RMS|a|)).
int prescale_log2(const HostMat& A);
// Normalize a raw walk sum (re, im, mag) into the permanent.
void normalize(int alg, int m, int n, int scale_log2, double* re, double* im, double* mag);
// Run the walk over [k_begin, k_end) -> 8 raw doubles at `dst` (device).
int run_walk(const WalkSetup& ws, uint64_t k_begin, uint64_t k_end, int mag, double* dst, cudaStream_t stream);
// The same launch with the setup already resident in the device scratch
// (an earlier run_walk of this WalkSetup on this thread): no staging copy.
int run_walk_resident(const WalkSetup& ws, uint64_t k_begin, uint64_t k_end, int mag, double* dst,
                      cudaStream_t stream);
// Whole walk with the 8 raw result doubles returned in host memory: the
// zero-copy path (setup as kernel parameters, result + flag in mapped pinned
// memory, spin on the flag) where it applies, else run_walk + copy + sync.
int run_walk_host(const WalkSetup& ws, uint64_t k_begin, uint64_t k_end, int mag, double* host8,
                  cudaStream_t stream, bool zero_copy);

uint64_t walk_steps(int alg, int m, int n);

// ---- bulk-pipelined batch kernels (engine_bulk.cu) --------------------------
bool bulk_batch_supported(int alg, bool cplx, int m, int n);
// PERM_OK / CUDA failure, or -1 when no bulk kernel applies (shape, alignment)
int launch_bulk_batch(int alg, bool cplx, int64_t B, int m, int n, const void* dA, void* dOut, cudaStream_t stream);
// partition formula for 16 < n <= 62 (runtime n)
int launch_partition_wide(bool cplx, int64_t B, int m, int n, const void* dA, void* dOut, cudaStream_t stream);

// ---- instrumentation -------------------------------------------------------
struct KernelTimer {
  bool init = false, ok = false, pending = false;
  cudaEvent_t start = nullptr, stop = nullptr;
  int last_grid = 0, last_log2L = 0;
};
KernelTimer& kernel_timer();
bool timing_enabled();
void set_timing(bool on);
int fp64_peak_probe(double seconds, int op, double* ops_per_s);

}  // namespace permb200
