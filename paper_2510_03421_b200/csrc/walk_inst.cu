// Explicit instantiation of the Gray-walk kernels for P = 1..64, one
// (scalar type, weighted) combination per object file.  Built four times by
// the Makefile with -DWALK_T=double|cd -DWALK_W=0|1 -DWALK_TAG=<name>.
#include "walk_launch.cuh"

#ifndef WALK_T
#define WALK_T double
#define WALK_W 0
#define WALK_TAG f64_w0
#endif
#define WALK_CAT2(a, b) a##b
#define WALK_CAT(a, b) WALK_CAT2(a, b)

namespace permb200 {
walk_fn WALK_CAT(walk_lookup_, WALK_TAG)(int P) {
  return walk_pick<WALK_T, (bool)WALK_W>(P, std::make_integer_sequence<int, 64>{});
}
}  // namespace permb200
