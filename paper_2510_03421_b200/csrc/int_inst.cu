// Instantiation of the fast exact int128 walk for P = 1..64.
#include <utility>

#include "int_walk.cuh"

namespace permb200 {
template <int... Ps>
static walk_fn_i int_pick(int P, std::integer_sequence<int, Ps...>) {
  walk_fn_i fn = nullptr;
  ((P == Ps + 1 ? (fn = &launch_int_wrap<Ps + 1>, 0) : 0), ...);
  return fn;
}
walk_fn_i int_wrap_lookup(int P) { return int_pick(P, std::make_integer_sequence<int, 64>{}); }
}  // namespace permb200

namespace permb200 {
template <int... Ps>
static walk_fn_if int_pick_fp(int P, std::integer_sequence<int, Ps...>) {
  walk_fn_if fn = nullptr;
  ((P == Ps + 1 ? (fn = &launch_int_wrap_fp<Ps + 1>, 0) : 0), ...);
  return fn;
}
walk_fn_if int_wrap_fp_lookup(int P) { return int_pick_fp(P, std::make_integer_sequence<int, 64>{}); }
}  // namespace permb200
