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
template <int P, int K>
static walk_fn_if fp_entry(int NG) {
  constexpr int ng = int_fp_ng(P, K);
  return NG == ng ? &launch_int_wrap_fp<P, ng> : nullptr;
}
template <int... Ps>
static walk_fn_if int_pick_fp(int P, int NG, std::integer_sequence<int, Ps...>) {
  walk_fn_if fn = nullptr;
  ((P == Ps + 1 && !fn ? (fn = fp_entry<Ps + 1, 0>(NG), fn = fn ? fn : fp_entry<Ps + 1, 1>(NG),
                          fn = fn ? fn : fp_entry<Ps + 1, 2>(NG), 0)
                       : 0),
   ...);
  return fn;
}
walk_fn_if int_wrap_fp_lookup(int P, int NG) { return int_pick_fp(P, NG, std::make_integer_sequence<int, 64>{}); }
}  // namespace permb200
