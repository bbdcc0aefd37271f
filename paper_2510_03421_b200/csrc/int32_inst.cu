// Instantiation of the FP32-quad exact int128 walk for 1..10 quads.
#include <utility>

#include "int_walk32.cuh"

namespace permb200 {
template <int NQ, bool DL4>
static walk_fn_i32 f32_entry(int* resident) {
  if (resident) {
    int r = 0;
    const size_t smem = 33 * NQ * 4 * sizeof(float);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, int_walk_wrap_f32_kernel<NQ, DL4>, kInt32Threads, smem) !=
            cudaSuccess ||
        r < 1)
      r = 1;
    *resident = r;
  }
  return &launch_int_wrap_f32<NQ, DL4>;
}
template <int... Qs>
static walk_fn_i32 int_pick_f32(int NQ, bool dl4, int* resident, std::integer_sequence<int, Qs...>) {
  walk_fn_i32 fn = nullptr;
  ((NQ == Qs + 1 ? (fn = dl4 ? f32_entry<Qs + 1, true>(resident) : f32_entry<Qs + 1, false>(resident), 0) : 0), ...);
  return fn;
}
walk_fn_i32 int_wrap_f32_lookup(int NQ, bool dl4, int* resident) {
  return int_pick_f32(NQ, dl4, resident, std::make_integer_sequence<int, kInt32MaxQuads>{});
}
}  // namespace permb200
