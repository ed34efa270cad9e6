// Work over ordered lists of dense page ranges.
//
// Window demand runs and per-command actual sets are lists of ranges whose
// sizes span five orders of magnitude (a 58 K-page weight slice next to a
// one-page KV tail).  Every 32-page bitmap word of every range is one work
// unit, so work is balanced regardless of range sizes.  k_units_plan counts
// the missing pages of a range list (popcount of ~resident & range mask),
// scans, and expands them in order in one cooperative launch — an
// order-preserving stream compaction whose output order is the ranges'
// order, exactly the first-access order plan_migration needs
// (memman.py:284-291).
#include "msched_internal.cuh"
#include "k_ranges.cuh"

namespace msg {



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

// ---- one cooperative launch: count, per-tag counts, scan, plan, fill ------
//
// The missing pages of an ordered range list against the resident bitmap,
// in range order (memman.py:284-291, engine.py:310-313, 350-355): every CTA
// owns a contiguous run of 32-page units; phase 1 counts (popcount of
// ~resident & range mask) and accumulates per-tag counts in shared memory;
// one grid barrier; phase 2 turns the per-CTA totals into offsets (and the
// plan scalars, memman.py:284-299); phase 3 recounts each unit (the bitmap is
// unchanged) and writes its pages at their offsets, capped.  Replaces the
// count / 3-kernel scan / scalars / fill chain (six launches).

__global__ void __launch_bounds__(UP_THREADS, 1) k_units_plan(UnitsPlan P) {
  extern __shared__ __align__(16) unsigned char up_raw[];
  int nbar = 0;
  units_plan_body(P, up_raw, nbar);
}

// per command of [c0, c1) of a task: missing pages of its actual set against
// the resident bitmap (engine.py:396-397).  blockIdx.y = command; the
// command's bitmap words are strided over blockIdx.x so a command touching a
// gigabyte is not walked by one CTA; out is zeroed by the caller.
constexpr int TC_SPLIT = 8;

__global__ void __launch_bounds__(256) k_touch_counts(const Iv* __restrict__ pool, const int64_t* __restrict__ off,
                                                     int32_t c0, const uint32_t* __restrict__ bits,
                                                     unsigned long long* __restrict__ out) {
  __shared__ unsigned long long red[8];
  const int32_t cmd = c0 + blockIdx.y;
  const int64_t i0 = off[cmd], i1 = off[cmd + 1];
  const int64_t T = (int64_t)gridDim.x * blockDim.x, me = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long acc = 0;
  int64_t skip = 0;
  for (int64_t i = i0; i < i1; ++i) {
    const Iv v = pool[i];
    const int64_t lo = v.d, hi = v.d + (v.b - v.a), w0 = lo >> 5, nw = ((hi + 31) >> 5) - w0;
    int64_t k = (T & (T - 1)) == 0 ? ((me - skip) & (T - 1)) : (((me - skip) % T) + T) % T;   // (me - skip) mod T
    for (; k < nw; k += T) acc += __popc(~bits[w0 + k] & unit_mask(lo, hi, w0 + k));
    skip += nw;
  }
  acc = __reduce_add_sync(0xffffffffu, (unsigned)acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    if (s) atomicAdd(&out[blockIdx.y], s);
  }
}

void touch_counts_dev(Ctx& c, TaskTab& t, int32_t lo, int32_t hi, int64_t* out) {
  if (hi <= lo) return;
  MSG_CUDA(cudaMemsetAsync(out, 0, (hi - lo) * sizeof(int64_t), c.st));
  k_touch_counts<<<dim3(TC_SPLIT, hi - lo), 256, 0, c.st>>>(t.act_pool.p, t.d_act_off.p, lo, c.bits.p,
                                                            reinterpret_cast<unsigned long long*>(out));
  MSG_CHECK_LAUNCH();
  add_launches(1);
}

UnitsPlan units_plan_args(Ctx& c, const RangeSet& R, int32_t grid, int64_t* tag_cnt, int32_t ntags, int64_t cap,
                          int32_t* out, int64_t plan_capacity, int64_t* total_out, int32_t* bar) {
  if (ntags > UP_MAX_TAGS) throw Error(MSG_E_INVAL, "too many commands in one window for the units plan");
  c.up_hist.resize((int64_t)grid * (1 + std::max(ntags, 0)) + 1, c.st);
  const int nt = tag_cnt ? ntags : 0;
  return UnitsPlan{R, c.bits.p, tag_cnt, nt, cap, out, plan_capacity >= 0 ? c.dstate : nullptr,
                   plan_capacity, c.len, total_out, c.up_hist.p, bar, 1};
}

void units_plan(Ctx& c, const RangeSet& R, int64_t units_cap, int64_t* tag_cnt, int32_t ntags, int64_t cap,
                int32_t* out, int64_t plan_capacity, int64_t* total_out) {
  if (c.up_per_sm < 0) {
    const int max_smem = (int)units_plan_smem(UP_MAX_TAGS, UP_THREADS);
    MSG_CUDA(cudaFuncSetAttribute(k_units_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
    MSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.up_per_sm, k_units_plan, UP_THREADS, max_smem));
    MSG_CUDA(cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, c.device));
  }
  const int per_sm = c.up_per_sm, sms = c.nsm;
  if (ntags > UP_MAX_TAGS) throw Error(MSG_E_INVAL, "too many commands in one window for the units plan");
  int G = (int)std::min<int64_t>(std::max<int64_t>((units_cap + 511) / 512, 1), (int64_t)std::max(per_sm, 1) * sms);
  c.up_hist.resize((int64_t)G * (1 + std::max(ntags, 0)) + 1, c.st);
  const int nt = tag_cnt ? ntags : 0;
  const size_t smem = units_plan_smem(nt, UP_THREADS);
  UnitsPlan P{R, c.bits.p, tag_cnt, nt, cap, out, plan_capacity >= 0 ? c.dstate : nullptr,
              plan_capacity, c.len, total_out, c.up_hist.p, next_barrier(c), 1};
  void* args[] = {&P};
  MSG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_units_plan), dim3(G), dim3(UP_THREADS), args, smem,
                                       c.st));
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
