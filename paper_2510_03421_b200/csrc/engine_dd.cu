// Host side of the double-double validation walks (perm_permanent_dd).
#include <algorithm>
#include <cmath>
#include <vector>

#include "engine.cuh"
#include "walk_dd.cuh"

namespace permb200 {

template <bool CPLX>
static cudaError_t launch_dd(const WalkDDArgs& a, int blocks, cudaStream_t s) {
  const int P = a.P;
#define DD_CASE(PM)                                                     \
  if (P <= PM) {                                                        \
    walk_dd_kernel<CPLX, PM><<<blocks, 128, 0, s>>>(a);                 \
    return cudaGetLastError();                                          \
  }
  DD_CASE(8)
  DD_CASE(16)
  DD_CASE(24)
  DD_CASE(32)
  DD_CASE(40)
  DD_CASE(48)
  DD_CASE(56)
  DD_CASE(64)
#undef DD_CASE
  return cudaErrorInvalidValue;
}

static void hdd_add(double& ah, double& al, double bh, double bl) { dd_add(ah, al, bh, bl); }

int dd_permanent(int alg, bool cplx, int m, int n, const double* a, int64_t lda, int dev_ptr, double* out4,
                 void* stream_) {
  clear_error();
  if (m < 1 || n < 1 || m > n || n > 62) {
    set_error("need 1 <= m <= n <= 62");
    return PERM_BAD_SHAPE;
  }
  if (alg != PERM_ALG_GLYNN && alg != PERM_ALG_RYSER) {
    set_error("double-double walks exist for Glynn and Ryser");
    return PERM_BAD_ARG;
  }
  cudaStream_t stream = pick_stream(stream_);
  HostMat A;
  int st = load_matrix(m, n, a, lda, dev_ptr, cplx, &A, stream);
  if (st) return st;
  WalkSetup ws;
  st = build_walk(alg, A, &ws);
  if (st) return st;
  const uint64_t steps = walk_steps(alg, m, n);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t target = (uint64_t)nsm * 4 * 128;
  int log2L = 0;
  while ((steps >> (log2L + 1)) >= target && log2L < 40) ++log2L;
  const uint64_t nchunks = steps >> log2L;
  const int blocks = (int)std::min<uint64_t>((nchunks + 127) / 128, (uint64_t)nsm * 4);
  Scratch* s = scratch();
  if (!s) return cuda_fail(cudaErrorNoDevice, "scratch");
  const size_t data_bytes = ws.buf.size() * sizeof(double);
  st = ensure_dev(s, data_bytes + (size_t)blocks * 32 + 512);
  if (st) return st;
  double* data = static_cast<double*>(s->dev);
  double* parts = data + ((ws.buf.size() + 31) & ~(size_t)31);
  st = stage_h2d(s, data, ws.buf.data(), data_bytes, stream);
  if (st) return st;
  WalkDDArgs args;
  args.v0 = data + ws.v0_off;
  args.U = data + ws.U_off;
  args.w = ws.weighted ? data + ws.w_off : nullptr;
  args.P = ws.P;
  args.B = ws.B;
  args.log2L = log2L;
  args.weighted = ws.weighted ? 1 : 0;
  args.k_begin = 0;
  args.nchunks = nchunks;
  args.out = parts;
  cudaError_t e = cplx ? launch_dd<true>(args, blocks, stream) : launch_dd<false>(args, blocks, stream);
  if (e != cudaSuccess) return cuda_fail(e, "dd walk launch");
  std::vector<double> h((size_t)blocks * 4);
  if (h.size() > kHostResultDoubles) return cuda_fail(cudaErrorInvalidValue, "dd partials");
  PERM_CUDA_TRY(cudaMemcpyAsync(s->host, parts, h.size() * 8, cudaMemcpyDeviceToHost, stream));
  PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  std::copy(s->host, s->host + h.size(), h.begin());
  double rh = 0, rl = 0, ih = 0, il = 0;
  for (int b = 0; b < blocks; ++b) {
    hdd_add(rh, rl, h[4 * b], h[4 * b + 1]);
    hdd_add(ih, il, h[4 * b + 2], h[4 * b + 3]);
  }
  if (alg == PERM_ALG_GLYNN) {
    const int ex = -(n - 1) - m * ws.scale_log2;
    rh = std::ldexp(rh, ex); rl = std::ldexp(rl, ex);
    ih = std::ldexp(ih, ex); il = std::ldexp(il, ex);
    double f = 1.0;
    for (int i = 2; i <= n - m; ++i) f *= (double)i;  // exact up to 22!
    auto div = [f](double& hi, double& lo) {
      const double q1 = hi / f;
      const double r = std::fma(-q1, f, hi) + lo;
      const double q2 = r / f;
      hi = q1 + q2;
      lo = q2 - (hi - q1);
    };
    div(rh, rl);
    div(ih, il);
  } else if (m == n && (n & 1)) {
    rh = -rh; rl = -rl; ih = -ih; il = -il;
  }
  out4[0] = rh; out4[1] = rl; out4[2] = ih; out4[3] = il;
  return PERM_OK;
}

}  // namespace permb200
