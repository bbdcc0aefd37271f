// Instantiation of the many-matrix Glynn walk (batches of n = 17..30).
#include "walk_launch.cuh"

namespace permb200 {
namespace {
template <typename T, int... Ps>
walk_multi_fn pick(int P, std::integer_sequence<int, Ps...>) {
  walk_multi_fn fn = nullptr;
  ((P == kWalkMultiMinN + Ps ? (fn = &launch_walk_multi<T, kWalkMultiMinN + Ps>, 0) : 0), ...);
  return fn;
}
template <typename T, int... Ps>
walk_multi_bps_fn pick_bps(int P, std::integer_sequence<int, Ps...>) {
  walk_multi_bps_fn fn = nullptr;
  ((P == kWalkMultiMinN + Ps ? (fn = &walk_multi_blocks_per_sm<T, kWalkMultiMinN + Ps>, 0) : 0), ...);
  return fn;
}
using Seq = std::make_integer_sequence<int, kWalkMultiMaxN - kWalkMultiMinN + 1>;
}  // namespace

walk_multi_fn walk_multi_lookup(bool cplx, int P) {
  return cplx ? pick<cd>(P, Seq{}) : pick<double>(P, Seq{});
}
walk_multi_bps_fn walk_multi_bps_lookup(bool cplx, int P) {
  return cplx ? pick_bps<cd>(P, Seq{}) : pick_bps<double>(P, Seq{});
}
}  // namespace permb200
