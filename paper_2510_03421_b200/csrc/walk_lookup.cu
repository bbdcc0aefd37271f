// Joins the walk_inst.cu slices: walk_lookup_<tag>(P) for P = 1..64.
#include "walk_launch.cuh"

namespace permb200 {
#define WALK_SLICES(tag)                                                              \
  walk_fn walk_lookup_##tag##_p0(int);                                                \
  walk_fn walk_lookup_##tag##_p1(int);                                                \
  walk_fn walk_lookup_##tag##_p2(int);                                                \
  walk_fn walk_lookup_##tag##_p3(int);                                                \
  walk_fn walk_lookup_##tag(int P) {                                                  \
    if (P < 25) return walk_lookup_##tag##_p0(P);                                     \
    if (P < 41) return walk_lookup_##tag##_p1(P);                                     \
    if (P < 53) return walk_lookup_##tag##_p2(P);                                     \
    return walk_lookup_##tag##_p3(P);                                                 \
  }
WALK_SLICES(f64_w0)
WALK_SLICES(f64_w1)
WALK_SLICES(c128_w0)
WALK_SLICES(c128_w1)
}  // namespace permb200
