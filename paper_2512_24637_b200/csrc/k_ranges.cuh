// Range-list work units (k_ranges.cu).
#pragma once
#include "msched_internal.cuh"

namespace msg {

// bits of bitmap word w that lie in the dense page range [lo, hi)
__device__ __forceinline__ uint32_t unit_mask(int64_t lo, int64_t hi, int64_t w) {
  int64_t p0 = w << 5;
  uint32_t m = ~0u;
  if (p0 < lo) m &= ~0u << (lo - p0);
  if (p0 + 32 > hi) m &= (hi - p0) >= 32 ? ~0u : ((1u << (hi - p0)) - 1u);
  return m;
}

__device__ __forceinline__ int64_t block_scan_excl_i64(int64_t v, int64_t* smem_warp, int64_t* total) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t s = lane < nw ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) smem_warp[lane] = s;
  }
  __syncthreads();
  int64_t before = (wid ? smem_warp[wid - 1] : 0) + x - v;
  if (total) *total = smem_warp[nw - 1];
  __syncthreads();
  return before;
}

void ranges_from_actual(Ctx& c, TaskTab& t, int32_t c0, int32_t c1, RangeBuf& B);
// one cooperative launch: missing pages of R against residency, per-tag
// counts (optional), plan scalars against plan_capacity into DevState
// (optional), capped fill
void units_plan(Ctx& c, const RangeSet& R, int64_t units_cap, int64_t* tag_cnt, int32_t ntags, int64_t cap,
                int32_t* out, int64_t plan_capacity /* < 0: no plan scalars */, int64_t* total_out);
void touch_counts_dev(Ctx& c, TaskTab& t, int32_t lo, int32_t hi, int64_t* out);
int32_t* next_barrier(Ctx& c);   // a zeroed grid-barrier counter for one cooperative launch

}  // namespace msg
