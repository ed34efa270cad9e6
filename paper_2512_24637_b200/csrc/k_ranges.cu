// Load-balanced work over ordered lists of dense page ranges.
//
// Window demand runs and per-command actual sets are lists of ranges whose
// sizes span five orders of magnitude (a 58 K-page weight slice next to a
// one-page KV tail).  Assigning a warp per range left one warp walking 1.8 K
// bitmap words while the rest of the GPU idled (k_demand_fill was 19 % of a
// replay).  Here every 32-page bitmap word of every range is one work unit:
// units are counted (popc of ~resident & range mask), exclusively scanned
// with a device-sized scan, and then expanded in order — an order-preserving
// stream compaction whose output order is the ranges' order, exactly the
// first-access order plan_migration needs (memman.py:284-291).
#include "msched_internal.cuh"
#include "k_ranges.cuh"

namespace msg {

__device__ __forceinline__ uint32_t unit_mask(int64_t lo, int64_t hi, int64_t w) {
  int64_t p0 = w << 5;
  uint32_t m = ~0u;
  if (p0 < lo) m &= ~0u << (lo - p0);
  if (p0 + 32 > hi) m &= (hi - p0) >= 32 ? ~0u : ((1u << (hi - p0)) - 1u);
  return m;
}

__device__ __forceinline__ int64_t range_of_unit(const RangeSet& R, int64_t nr, int64_t u) {
  int64_t a = 0, b = nr;   // largest r with uoff[r] <= u
  while (b - a > 1) {
    int64_t mid = (a + b) >> 1;
    if (R.uoff[mid] <= u) a = mid; else b = mid;
  }
  return a;
}

__global__ void k_units_count(RangeSet R, const uint32_t* __restrict__ bits, int32_t* ucnt, int64_t* tag_cnt,
                              int64_t* range_cnt) {
  int64_t nr = *R.nr;
  int64_t nu = nr ? R.uoff[nr] : 0;
  int lane = threadIdx.x & 31;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < nu; base += stride) {
    int64_t u = base + threadIdx.x;
    int64_t r = -1;
    int32_t c = 0;
    if (u < nu) {
      r = range_of_unit(R, nr, u);
      int64_t lo = R.lo[r], hi = lo + R.len[r];
      int64_t w = (lo >> 5) + (u - R.uoff[r]);
      c = __popc(~bits[w] & unit_mask(lo, hi, w));
      if (ucnt) ucnt[u] = c;
    }
    if (!tag_cnt && !range_cnt) continue;
    // warp-aggregate when the whole warp works on one range (the common case)
    int64_t r0 = __shfl_sync(0xffffffffu, r, 0);
    if (__all_sync(0xffffffffu, r == r0)) {
      int32_t s = c;
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0 && r0 >= 0 && s) {
        if (tag_cnt) atomicAdd(reinterpret_cast<unsigned long long*>(&tag_cnt[R.tag[r0]]), (unsigned long long)s);
        if (range_cnt) atomicAdd(reinterpret_cast<unsigned long long*>(&range_cnt[r0]), (unsigned long long)s);
      }
    } else if (r >= 0 && c) {
      if (tag_cnt) atomicAdd(reinterpret_cast<unsigned long long*>(&tag_cnt[R.tag[r]]), (unsigned long long)c);
      if (range_cnt) atomicAdd(reinterpret_cast<unsigned long long*>(&range_cnt[r]), (unsigned long long)c);
    }
  }
}

__global__ void k_units_fill(RangeSet R, const uint32_t* __restrict__ bits, const int64_t* __restrict__ uofs,
                             const int64_t* cap_ptr, int32_t* __restrict__ out) {
  int64_t nr = *R.nr;
  int64_t nu = nr ? R.uoff[nr] : 0;
  int64_t cap = cap_ptr ? *cap_ptr : INT64_MAX;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = uofs[u];
    if (o >= cap) continue;
    int64_t r = range_of_unit(R, nr, u);
    int64_t lo = R.lo[r], hi = lo + R.len[r];
    int64_t w = (lo >> 5) + (u - R.uoff[r]);
    uint32_t m = ~bits[w] & unit_mask(lo, hi, w);
    while (m && o < cap) {
      int b = __ffs(m) - 1;
      m &= m - 1;
      out[o++] = (int32_t)((w << 5) + b);
    }
  }
}

// Ranges = the actual intervals of commands [c0, c1) of one task; tag = command - c0.
__global__ void __launch_bounds__(1024, 1) k_ranges_from_iv(const Iv* pool, const int64_t* off, int32_t c0, int32_t c1,
                                                          RangeOut O) {
  int64_t i0 = off[c0], n = off[c1] - i0;
  __shared__ int64_t ws[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t words = 0;
    if (i < n) {
      const Iv v = pool[i0 + i];
      int64_t lo = v.d, hi = v.d + (v.b - v.a);
      O.lo[i] = lo;
      O.len[i] = hi - lo;
      words = ((hi + 31) >> 5) - (lo >> 5);
      int32_t a = c0, b = c1;   // command of interval i0 + i
      while (a < b) {
        int32_t mid = (a + b) >> 1;
        if (off[mid + 1] <= i0 + i) a = mid + 1; else b = mid;
      }
      O.tag[i] = a - c0;
    }
    int64_t tot;
    int64_t ex = block_scan_excl_i64(words, ws, &tot);
    if (i < n) O.uoff[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) { O.uoff[n] = carry; *O.nr = n; }
}

// ---- exclusive scan of int32 counts whose length lives in device memory ----

constexpr int DS_BLOCKS = 296, DS_THREADS = 1024;

__device__ __forceinline__ void ds_slice(int64_t n, int64_t* a, int64_t* b) {
  int64_t L = (n + DS_BLOCKS - 1) / DS_BLOCKS;
  *a = blockIdx.x * L;
  *b = *a + L < n ? *a + L : n;
}

__global__ void __launch_bounds__(DS_THREADS, 1) k_dscan_reduce(const int32_t* in, const int64_t* n_ptr,
                                                              const int64_t* n_off, int64_t* sums) {
  __shared__ int64_t ws[32];
  int64_t n = *n_ptr + (n_off ? 0 : 0);
  int64_t a, b;
  ds_slice(n, &a, &b);
  int64_t acc = 0;
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) acc += in[i];
  int64_t tot;
  block_scan_excl_i64(acc, ws, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(DS_THREADS, 1) k_dscan_sums(int64_t* sums, int64_t* total) {
  __shared__ int64_t ws[32];
  int64_t v = threadIdx.x < DS_BLOCKS ? sums[threadIdx.x] : 0;
  int64_t tot;
  int64_t ex = block_scan_excl_i64(v, ws, &tot);
  if (threadIdx.x < DS_BLOCKS) sums[threadIdx.x] = ex;
  if (threadIdx.x == 0 && total) *total = tot;
}

__global__ void __launch_bounds__(DS_THREADS, 1) k_dscan_down(const int32_t* in, const int64_t* n_ptr,
                                                            const int64_t* sums, int64_t* out) {
  __shared__ int64_t ws[32];
  __shared__ int64_t carry;
  int64_t n = *n_ptr;
  int64_t a, b;
  ds_slice(n, &a, &b);
  if (threadIdx.x == 0) carry = sums[blockIdx.x];
  __syncthreads();
  for (int64_t base = a; base < b; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < b ? in[i] : 0;
    int64_t tot;
    int64_t ex = block_scan_excl_i64(v, ws, &tot);
    if (i < b) out[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// units count of a RangeSet = uoff[nr]; copy it next to nr for the scans
__global__ void k_units_total(RangeSet R, int64_t* nu) {
  int64_t nr = *R.nr;
  *nu = nr ? R.uoff[nr] : 0;
}

void units_scan(Ctx& c, const RangeSet& R, const int32_t* ucnt, int64_t* uofs, int64_t* total, int64_t* scratch) {
  // scratch: [0] = unit count, [1 .. DS_BLOCKS] = block sums
  k_units_total<<<1, 1, 0, c.st>>>(R, scratch);
  k_dscan_reduce<<<DS_BLOCKS, DS_THREADS, 0, c.st>>>(ucnt, scratch, nullptr, scratch + 1);
  k_dscan_sums<<<1, DS_THREADS, 0, c.st>>>(scratch + 1, total);
  k_dscan_down<<<DS_BLOCKS, DS_THREADS, 0, c.st>>>(ucnt, scratch, scratch + 1, uofs);
  MSG_CHECK_LAUNCH();
  add_launches(4);
}

void units_count(Ctx& c, const RangeSet& R, int32_t* ucnt, int64_t* tag_cnt, int64_t* range_cnt) {
  k_units_count<<<4 * 148, 256, 0, c.st>>>(R, c.bits.p, ucnt, tag_cnt, range_cnt);
  MSG_CHECK_LAUNCH();
  add_launches(1);
}

void units_fill(Ctx& c, const RangeSet& R, const int64_t* uofs, const int64_t* cap_ptr, int32_t* out) {
  k_units_fill<<<4 * 148, 256, 0, c.st>>>(R, c.bits.p, uofs, cap_ptr, out);
  MSG_CHECK_LAUNCH();
  add_launches(1);
}

void ranges_from_actual(Ctx& c, TaskTab& t, int32_t c0, int32_t c1, RangeBuf& B) {
  int64_t n = t.act_off[c1] - t.act_off[c0];
  B.reserve(n, c.st);
  k_ranges_from_iv<<<1, 1024, 0, c.st>>>(t.act_pool.p, t.d_act_off.p, c0, c1, B.out());
  MSG_CHECK_LAUNCH();
  add_launches(1);
}

}  // namespace msg
