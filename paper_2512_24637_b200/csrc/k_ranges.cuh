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

// k-th grid-wide barrier on one monotone counter (zero at launch): the
// arrival is a gpu-scope release add (it publishes this CTA's writes, which
// __syncthreads ordered before it), the wait a gpu-scope acquire poll
__device__ __forceinline__ void grid_barrier(int32_t* bar, int k) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(bar) : "memory");
    const int32_t target = (k + 1) * (int32_t)gridDim.x;
    int32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

struct UnitsPlan {
  RangeSet R;
  const uint32_t* bits;
  int64_t* tag_cnt;      // per-tag totals (ntags), or nullptr
  int32_t ntags;
  int64_t cap;           // fill cap (pages), < 0: none
  int32_t* out;          // fill output, or nullptr
  DevState* S;           // plan scalars, or nullptr
  int64_t C, len;        // capacity and resident pages (for the scalars)
  int64_t* total_out;    // missing pages, or nullptr
  int32_t* hist;         // [gridDim] CTA totals, then [gridDim][ntags] tag partials
  int32_t* bar;          // grid barrier counter (zero at launch)
  int32_t stage;         // the range table fits the dynamic shared memory
};

constexpr int UP_THREADS = 512;
constexpr int UP_MAX_TAGS = 8192;
constexpr int UP_SMEM_RANGES = 4096;   // range tables up to this size are searched in shared memory

// dynamic shared memory of units_plan_body for nt tags and NT threads
__host__ __device__ constexpr size_t units_plan_smem(int nt, int NT) {
  return ((4 * (size_t)nt + 15) & ~size_t(15)) + 16 * ((size_t)UP_SMEM_RANGES + 1) + 8 * 34 + 20 * (size_t)NT;
}

// The body runs as its own cooperative launch (k_units_plan, 512 threads) or as
// the first phase of the per-switch cooperative kernel (k_switch_coop, 1024
// threads): block-size generic; its shared memory is the caller's dynamic
// buffer (units_plan_smem bytes); nbar counts the grid barriers used so far
// on P.bar.
// Returns the missing total (every CTA computes it).
__device__ __forceinline__ int64_t units_plan_body(const UnitsPlan& P, unsigned char* up_raw, int& nbar) {
  const int NT = (int)blockDim.x;
  int32_t* tagc = reinterpret_cast<int32_t*>(up_raw);                          // ntags
  int64_t* r_uoff = reinterpret_cast<int64_t*>(up_raw + ((4 * (int64_t)P.ntags + 15) & ~int64_t(15)));
  int64_t* r_lo = r_uoff + UP_SMEM_RANGES + 1;
  int64_t* ws = r_lo + UP_SMEM_RANGES;          // [32] block-scan scratch
  int64_t* carry_p = ws + 32;                    // [1]
  int64_t* uo_s = carry_p + 2;                   // [NT] unit offsets (phase 3)
  int64_t* uw_s = uo_s + NT;                     // [NT] unit words
  uint32_t* um_s = reinterpret_cast<uint32_t*>(uw_s + NT);   // [NT] unit masks
  const int t = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const int64_t nr = *P.R.nr;
  const int64_t nu = nr ? P.R.uoff[nr] : 0;
  const int64_t U = (nu + G - 1) / G;
  const int64_t u0 = (int64_t)b * U, u1 = u0 + U < nu ? u0 + U : nu;
  const bool staged = P.stage && nr <= UP_SMEM_RANGES;
  for (int i = t; i < P.ntags; i += NT) tagc[i] = 0;
  if (staged)
    for (int64_t i = t; i <= nr; i += NT) {
      r_uoff[i] = P.R.uoff[i];
      if (i < nr) r_lo[i] = P.R.lo[i];
    }
  __syncthreads();
  const int64_t* uoff = staged ? r_uoff : P.R.uoff;
  const int64_t* rlo = staged ? r_lo : P.R.lo;
  auto unit = [&](int64_t u, int64_t* r_out, int64_t* w_out, uint32_t* m_out) {
    int64_t a = 0, z = nr;   // largest r with uoff[r] <= u
    while (z - a > 1) { int64_t mid = (a + z) >> 1; if (uoff[mid] <= u) a = mid; else z = mid; }
    // a range's units are the bitmap words it overlaps, so its end is the next range's start only
    // as far as units go; the page extent needs len, read once per unit (cached in L1)
    int64_t lo = rlo[a], hi = lo + P.R.len[a];
    int64_t w = (lo >> 5) + (u - uoff[a]);
    *r_out = a; *w_out = w; *m_out = ~P.bits[w] & unit_mask(lo, hi, w);
  };
  // ---- phase 1: counts.  When the CTA's units fit one pass (one unit per
  // thread), phase 3 reuses each thread's word and mask instead of recomputing
  const bool single = u1 - u0 <= NT;
  int64_t keep_w = 0;
  uint32_t keep_m = 0;
  int64_t acc = 0;
  for (int64_t base = u0; base < u1; base += NT) {
    int64_t u = base + t, r = -1, w = 0;
    uint32_t m = 0;
    if (u < u1) unit(u, &r, &w, &m);
    keep_w = w; keep_m = m;
    int c = __popc(m);
    acc += c;
    if (P.tag_cnt) {
      int tag = (r >= 0 && c) ? P.R.tag[r] : -1;
      unsigned peers = __match_any_sync(0xffffffffu, tag);
      int sum = __reduce_add_sync(peers, (unsigned)c);
      if (tag >= 0 && (int)(t & 31) == __ffs(peers) - 1) atomicAdd(&tagc[tag], sum);
    }
  }
  int64_t tot;
  block_scan_excl_i64(acc, ws, &tot);
  int64_t pre_tot = 0, all_tot = tot;
  if (G == 1) {
    // one CTA: its totals are the grid's; no histogram round trip, no barrier
    if (P.tag_cnt) {
      __syncthreads();
      for (int i = t; i < P.ntags; i += NT) P.tag_cnt[i] = tagc[i];
    }
  } else {
  if (t == 0) __stcg(P.hist + b, (int32_t)tot);
  __syncthreads();
  if (P.tag_cnt)
    for (int i = t; i < P.ntags; i += NT) __stcg(P.hist + G + (int64_t)b * P.ntags + i, tagc[i]);
  // ---- grid barrier
  grid_barrier(P.bar, nbar++);
  // ---- phase 2: offsets, totals, scalars, per-tag totals
  int64_t pre = 0, all = 0;
  for (int i = t; i < G; i += NT) {
    int64_t v = __ldcg(P.hist + i);
    all += v;
    if (i < b) pre += v;
  }
  block_scan_excl_i64(pre, ws, &pre_tot);
  block_scan_excl_i64(all, ws, &all_tot);
  if (P.tag_cnt) {
    if (G <= 32) {
      // few CTAs: one thread per tag sums the G partials (coalesced over tags)
      for (int i = b * NT + t; i < P.ntags; i += G * NT) {
        int64_t sum = 0;
        for (int c2 = 0; c2 < G; ++c2) sum += __ldcg(P.hist + G + (int64_t)c2 * P.ntags + i);
        P.tag_cnt[i] = sum;
      }
    } else {
      // many CTAs: CTA b sums tags b, b+G, ... with all its threads (one CTA
      // row per thread)
      for (int i = b; i < P.ntags; i += G) {
        int64_t part = 0;
        for (int c2 = t; c2 < G; c2 += NT) part += __ldcg(P.hist + G + (int64_t)c2 * P.ntags + i);
        int64_t sum;
        block_scan_excl_i64(part, ws, &sum);
        if (t == 0) P.tag_cnt[i] = sum;
      }
    }
  }
  }   // G > 1
  if (b == 0 && t == 0) {
    if (P.total_out) *P.total_out = all_tot;
    if (P.S) {
      DevState* S = P.S;
      S->missing = all_tot;
      int64_t pop = all_tot < P.C ? all_tot : P.C;
      S->populate = pop;
      S->truncated = all_tot - pop;
      S->free_before = P.C - P.len;
      int64_t ev = pop - (P.C - P.len);
      S->evict = ev > 0 ? ev : 0;
      S->skip = all_tot == 0;
      S->aux[2] = 0;   // the switch's multisplit pass count, until the multisplit publishes it
    }
  }
  if (!P.out) return all_tot;   // (callers running later phases follow with a grid barrier)
  // ---- phase 3: fill in range order, capped.  Offsets per unit (thread per
  // unit, block scan), then one warp writes a unit's pages with one
  // coalesced store (lane k writes page 32w+k when missing).
  const int64_t cap = P.cap < 0 ? INT64_MAX : P.cap;
  const int lane = t & 31, warp = t >> 5;
  if (t == 0) (*carry_p) = pre_tot;
  __syncthreads();
  for (int64_t base = u0; base < u1; base += NT) {
    int64_t u = base + t, r, w = 0;
    uint32_t m = 0;
    if (u < u1) {
      if (single) { w = keep_w; m = keep_m; }
      else unit(u, &r, &w, &m);
    }
    int64_t rt;
    int64_t o = (*carry_p) + block_scan_excl_i64(__popc(m), ws, &rt);
    uo_s[t] = o; uw_s[t] = w; um_s[t] = m;
    __syncthreads();
    for (int k = 0; k < 32; ++k) {
      const int i = warp * 32 + k;
      const uint32_t mk = um_s[i];
      if (!mk) continue;
      const int64_t ok = uo_s[i] + __popc(mk & ((1u << lane) - 1u));
      if (((mk >> lane) & 1u) && ok < cap) P.out[ok] = (int32_t)((uw_s[i] << 5) + lane);
    }
    __syncthreads();
    if (t == 0) (*carry_p) += rt;
    __syncthreads();
  }
  return all_tot;
}

void ranges_from_actual(Ctx& c, TaskTab& t, int32_t c0, int32_t c1, RangeBuf& B);
// one cooperative launch: missing pages of R against residency, per-tag
// counts (optional), plan scalars against plan_capacity into DevState
// (optional), capped fill
void units_plan(Ctx& c, const RangeSet& R, int64_t units_cap, int64_t* tag_cnt, int32_t ntags, int64_t cap,
                int32_t* out, int64_t plan_capacity /* < 0: no plan scalars */, int64_t* total_out);
// the same plan as one phase of a cooperative kernel of `grid` CTAs (bar: its
// grid-barrier counter)
UnitsPlan units_plan_args(Ctx& c, const RangeSet& R, int32_t grid, int64_t* tag_cnt, int32_t ntags, int64_t cap,
                          int32_t* out, int64_t plan_capacity, int64_t* total_out, int32_t* bar);
void touch_counts_dev(Ctx& c, TaskTab& t, int32_t lo, int32_t hi, int64_t* out);
int32_t* next_barrier(Ctx& c);   // a zeroed grid-barrier counter for one cooperative launch

}  // namespace msg
