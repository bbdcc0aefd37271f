// Explicit instantiation of the Gray-walk kernels, one (scalar type,
// weighted, P range) slice per object file so the 256 kernels build in
// parallel.  Built by the Makefile with -DWALK_T=double|cd -DWALK_W=0|1
// -DWALK_TAG=<name> -DWALK_PART=0..3; walk_lookup.cu joins the slices.
#include "walk_launch.cuh"

#ifndef WALK_T
#define WALK_T double
#define WALK_W 0
#define WALK_TAG f64_w0
#endif
#ifndef WALK_PART
#define WALK_PART 0
#endif
#define WALK_CAT2(a, b) a##b
#define WALK_CAT(a, b) WALK_CAT2(a, b)
#define WALK_CAT4(a, b, c, d) WALK_CAT(WALK_CAT(WALK_CAT(a, b), c), d)

namespace permb200 {
namespace {
// slices of P = 1..64, sized so the larger (slower to compile) kernels spread out
constexpr int kLo[4] = {1, 25, 41, 53}, kHi[4] = {25, 41, 53, 65};

template <int... Ps>
walk_fn pick_slice(int P, std::integer_sequence<int, Ps...>) {
  constexpr int lo = kLo[WALK_PART];
  walk_fn fn = nullptr;
  ((P == lo + Ps ? (fn = &launch_walk<WALK_T, lo + Ps, (bool)WALK_W>, 0) : 0), ...);
  return fn;
}
}  // namespace

walk_fn WALK_CAT4(walk_lookup_, WALK_TAG, _p, WALK_PART)(int P) {
  return pick_slice(P, std::make_integer_sequence<int, kHi[WALK_PART] - kLo[WALK_PART]>{});
}
}  // namespace permb200
