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

__global__ void __launch_bounds__(UP_THREADS, 1) k_units_plan(UnitsPlan P) {
  __shared__ int64_t ws[32];
  __shared__ int64_t carry_s;
  extern __shared__ __align__(16) unsigned char up_raw[];
  int32_t* tagc = reinterpret_cast<int32_t*>(up_raw);                          // ntags
  int64_t* r_uoff = reinterpret_cast<int64_t*>(up_raw + ((4 * (int64_t)P.ntags + 15) & ~int64_t(15)));
  int64_t* r_lo = r_uoff + UP_SMEM_RANGES + 1;
  const int t = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const int64_t nr = *P.R.nr;
  const int64_t nu = nr ? P.R.uoff[nr] : 0;
  const int64_t U = (nu + G - 1) / G;
  const int64_t u0 = (int64_t)b * U, u1 = u0 + U < nu ? u0 + U : nu;
  const bool staged = P.stage && nr <= UP_SMEM_RANGES;
  for (int i = t; i < P.ntags; i += UP_THREADS) tagc[i] = 0;
  if (staged)
    for (int64_t i = t; i <= nr; i += UP_THREADS) {
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
  // ---- phase 1: counts
  int64_t acc = 0;
  for (int64_t base = u0; base < u1; base += UP_THREADS) {
    int64_t u = base + t, r = -1, w;
    uint32_t m = 0;
    if (u < u1) unit(u, &r, &w, &m);
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
      for (int i = t; i < P.ntags; i += UP_THREADS) P.tag_cnt[i] = tagc[i];
    }
  } else {
  if (t == 0) __stcg(P.hist + b, (int32_t)tot);
  __syncthreads();
  if (P.tag_cnt)
    for (int i = t; i < P.ntags; i += UP_THREADS) __stcg(P.hist + G + (int64_t)b * P.ntags + i, tagc[i]);
  // ---- grid barrier
  __syncthreads();
  if (t == 0) {   // release arrival / acquire poll at gpu scope (see k_plan.cu grid_barrier)
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(P.bar) : "memory");
    int32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(P.bar) : "memory");
    } while (v < G);
  }
  __syncthreads();
  // ---- phase 2: offsets, totals, scalars, per-tag totals
  int64_t pre = 0, all = 0;
  for (int i = t; i < G; i += UP_THREADS) {
    int64_t v = __ldcg(P.hist + i);
    all += v;
    if (i < b) pre += v;
  }
  block_scan_excl_i64(pre, ws, &pre_tot);
  block_scan_excl_i64(all, ws, &all_tot);
  if (P.tag_cnt) {
    if (G <= 32) {
      // few CTAs: one thread per tag sums the G partials (coalesced over tags)
      for (int i = b * UP_THREADS + t; i < P.ntags; i += G * UP_THREADS) {
        int64_t sum = 0;
        for (int c2 = 0; c2 < G; ++c2) sum += __ldcg(P.hist + G + (int64_t)c2 * P.ntags + i);
        P.tag_cnt[i] = sum;
      }
    } else {
      // many CTAs: CTA b sums tags b, b+G, ... with all its threads (one CTA
      // row per thread)
      for (int i = b; i < P.ntags; i += G) {
        int64_t part = 0;
        for (int c2 = t; c2 < G; c2 += UP_THREADS) part += __ldcg(P.hist + G + (int64_t)c2 * P.ntags + i);
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
  if (!P.out) return;
  // ---- phase 3: fill in range order, capped.  Offsets per unit (thread per
  // unit, block scan), then one warp writes a unit's pages with one
  // coalesced store (lane k writes page 32w+k when missing).
  __shared__ int64_t uo_s[UP_THREADS];
  __shared__ int64_t uw_s[UP_THREADS];
  __shared__ uint32_t um_s[UP_THREADS];
  const int64_t cap = P.cap < 0 ? INT64_MAX : P.cap;
  const int lane = t & 31, warp = t >> 5;
  if (t == 0) carry_s = pre_tot;
  __syncthreads();
  for (int64_t base = u0; base < u1; base += UP_THREADS) {
    int64_t u = base + t, r, w = 0;
    uint32_t m = 0;
    if (u < u1) unit(u, &r, &w, &m);
    int64_t rt;
    int64_t o = carry_s + block_scan_excl_i64(__popc(m), ws, &rt);
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
    if (t == 0) carry_s += rt;
    __syncthreads();
  }
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
    int64_t k = (me - skip) % T;
    if (k < 0) k += T;
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

void units_plan(Ctx& c, const RangeSet& R, int64_t units_cap, int64_t* tag_cnt, int32_t ntags, int64_t cap,
                int32_t* out, int64_t plan_capacity, int64_t* total_out) {
  if (c.up_per_sm < 0) {
    const int max_smem = 4 * UP_MAX_TAGS + 16 * (UP_SMEM_RANGES + 1) + 64;
    MSG_CUDA(cudaFuncSetAttribute(k_units_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
    MSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.up_per_sm, k_units_plan, UP_THREADS, max_smem));
    MSG_CUDA(cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, c.device));
  }
  const int per_sm = c.up_per_sm, sms = c.nsm;
  if (ntags > UP_MAX_TAGS) throw Error(MSG_E_INVAL, "too many commands in one window for the units plan");
  int G = (int)std::min<int64_t>(std::max<int64_t>((units_cap + 511) / 512, 1), (int64_t)std::max(per_sm, 1) * sms);
  c.up_hist.resize((int64_t)G * (1 + std::max(ntags, 0)) + 1, c.st);
  const int nt = tag_cnt ? ntags : 0;
  const size_t smem = ((4 * (size_t)nt + 15) & ~size_t(15)) + 16 * ((size_t)UP_SMEM_RANGES + 1);
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
