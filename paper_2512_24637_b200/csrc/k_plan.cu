// K3-K6, K8, K9 — the placement planner on the device.
//
// Data layout in HBM (per context):
//   bits[]    resident bitmap over the dense page space (1 bit / page)
//   order[2]  the eviction list as a dense array of page ids, head -> tail
//             (ping-pong buffers; live region order[cur][head, head+len))
//   frame[]   HBM frame of every resident dense page (-1 otherwise)
//   fifo[]    free-frame ring: populate j takes the j-th free frame, frames
//             released by eviction are appended in eviction order, so the
//             frame reuse order matches the pipelined-swap model
//             (engine.py:139-158).
//
// reorder_for_opt (memman.py:218-241) is restated exactly as ONE stable
// multisplit of the eviction list: every resident page gets a class equal to
// the dense rank of its tuple (class in window 0, ..., class in window W-1),
// where a page's class in window w is (K_w - r) for the r-th first-access run
// of that window (0 if absent).  Stable partition by that class reproduces the
// reference's sequence of per-run madvise calls (windows last to first, runs
// last to first) — see DESIGN.md §3 for the proof sketch.  Victims are then
// the list head (plan_migration reads evlist._runs head-first,
// memman.py:292-301), so victim selection is a prefix, not a search.
#include "msched_internal.cuh"
#include "k_ranges.cuh"

#include <algorithm>

namespace msg {

#ifdef MSG_MC_PHASE_TS
// k_windows_fused phase stamps: [phase] summed SM cycles since the kernel's first stamp, and launches
__device__ unsigned long long g_fw_sum[16], g_fw_n;
#define FWTS(i)                                                                   \
  do {                                                                            \
    __syncthreads();                                                              \
    if (threadIdx.x == 0) {                                                       \
      const unsigned long long t_ = (unsigned long long)clock64();  /* one CTA: SM cycles */ \
      if ((i) == 0) fw_t0 = t_;                                                   \
      atomicAdd(&g_fw_sum[i], t_ - fw_t0);                                        \
      if ((i) == 15) atomicAdd(&g_fw_n, 1ull);                                     \
    }                                                                             \
  } while (0)
// k_switch_coop phase stamps (block 0, after each grid barrier: every CTA is
// past the previous phase): [phase] summed ns since the kernel's start, and launches
__device__ unsigned long long g_sw_sum[8], g_sw_n;
// gap from the window kernel's last stamp to the switch kernel's first
// (launches that directly follow a window kernel): sum, count
__device__ unsigned long long g_fw_end, g_gap_sum, g_gap_n;
__shared__ unsigned long long sw_t0;
#define SWTS(i)                                                                   \
  do {                                                                            \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                    \
      unsigned long long t_;                                                      \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                       \
      if ((i) == 0) {                                                             \
        sw_t0 = t_;                                                               \
        const unsigned long long fe_ = *(volatile unsigned long long*)&g_fw_end;  \
        if (fe_ && t_ > fe_) { atomicAdd(&g_gap_sum, t_ - fe_); atomicAdd(&g_gap_n, 1ull); } \
        *(volatile unsigned long long*)&g_fw_end = 0;                             \
      }                                                                           \
      atomicAdd(&g_sw_sum[i], t_ - sw_t0);                                        \
      if ((i) == 7) atomicAdd(&g_sw_n, 1ull);                                     \
    }                                                                             \
  } while (0)
// k_window_combine_wide / k_window_runs (block 0) phase stamps: [phase]
// summed SM cycles since the kernel's first stamp, and launches
__device__ unsigned long long g_cw_sum[16], g_cw_n, g_wr_sum[16], g_wr_n;
#define PHTS(arr, cnt, i, last)                                                   \
  do {                                                                            \
    __syncthreads();                                                              \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                                    \
      const unsigned long long t_ = (unsigned long long)clock64();                \
      if ((i) == 0) ph_t0 = t_;                                                   \
      atomicAdd(&arr[i], t_ - ph_t0);                                             \
      if (last) atomicAdd(&cnt, 1ull);                                            \
    }                                                                             \
  } while (0)
#define CWTS(i) PHTS(g_cw_sum, g_cw_n, i, (i) == 15)
#define WRTS(i) PHTS(g_wr_sum, g_wr_n, i, (i) == 15)
#define PHTS_DECL unsigned long long ph_t0 = 0; (void)ph_t0
#else
#define FWTS(i) do {} while (0)
#define SWTS(i) do {} while (0)
#define CWTS(i) do {} while (0)
#define WRTS(i) do {} while (0)
#define PHTS_DECL do {} while (0)
#endif

static int64_t g_launches = 0;
int64_t kernel_launches() { return g_launches; }
void add_launches(int64_t n) { g_launches += n; }

// ---------------------------------------------------------------------------
// block-level helpers

template <class T>
__device__ T block_excl_scan(T v, T* smem_warp, T* total) {
  // blockDim.x multiple of 32, <= 1024
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nw ? smem_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) smem_warp[lane] = s;
  }
  __syncthreads();
  T before = (wid ? smem_warp[wid - 1] : T(0)) + x - v;
  if (total) *total = smem_warp[nw - 1];
  __syncthreads();
  return before;
}

// Block-wide exclusive scan of a[0..n) in place (any n); returns the total.
template <class T>
__device__ T block_scan_array(T* a, int64_t n) {
  __shared__ T warp_s[32];
  __shared__ T carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    T v = i < n ? a[i] : T(0);
    T tot;
    T ex = block_excl_scan<T>(v, warp_s, &tot);
    T carry = carry_s;
    if (i < n) a[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + tot;
    __syncthreads();
  }
  return carry_s;
}

// Bitonic sort of uint64 keys with int64 payload, n padded to a power of two.
__device__ void bitonic_kv(uint64_t* key, int64_t* val, int64_t npow2) {
  for (int64_t k = 2; k <= npow2; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < npow2; i += blockDim.x) {
        int64_t l = i ^ j;
        if (l > i) {
          bool up = (i & k) == 0;
          if ((key[i] > key[l]) == up) {
            uint64_t tk = key[i]; key[i] = key[l]; key[l] = tk;
            int64_t tv = val[i]; val[i] = val[l]; val[l] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}


__host__ __device__ inline int64_t pow2_at_least(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// ---------------------------------------------------------------------------
// K3: per-window first-access runs (memman.py:174-196).  One CTA per window.

struct WinDesc {
  const Iv* pool;               // the task's predicted intervals
  int64_t pool_lo, pool_hi;    // predicted intervals of commands [c0, c1)
  int32_t c0, c1, w, pad;
  const int64_t* cmd_off;      // task CSR offsets (pool indices), ncmd+1
  const uint8_t* selfpop;
  int64_t scratch;             // offset of this window's scratch region (elements)
};

struct WinOut {
  // per window: runs in first-access order (label asc, start asc)
  int64_t* run_a;   // abs start
  int64_t* run_b;   // abs end
  int64_t* run_d;   // dense start
  int32_t* run_lab; // command index
  int64_t* run_base;// per-window offset into the run arrays (= scratch base)
  int64_t* nruns;   // per window
  int64_t* pages;   // per window |w.pages|
};

extern __shared__ __align__(16) unsigned char dyn_smem[];
constexpr int64_t kWinSmem = 200 * 1024;

template <int NW>
__device__ bool block_radix_sort(uint64_t* a0, uint64_t* a1, int32_t* av, uint64_t* b0, uint64_t* b1, int32_t* bv,
                                 int n, int nbits, int32_t (*cnt)[256], int32_t* warp_s, int sh0);

// Scratch lives in shared memory when the window fits (44 B per padded
// endpoint: key[4mp] val[mp] label[mp]), else in the global region the host
// reserved (same layout).
__global__ void __launch_bounds__(1024, 1) k_window_runs(const WinDesc* wins, int64_t* gkey_u, int64_t* gval,
                              int32_t* glab, WinOut out, int64_t smem_cap) {
  PHTS_DECL;
  WRTS(0);
  const WinDesc W = wins[blockIdx.x];
  const Iv* pool = W.pool;
  int64_t n = W.pool_hi - W.pool_lo;
  int64_t base = W.scratch;           // scratch: 4n slots of key/val, 2n labels
  uint64_t* key = reinterpret_cast<uint64_t*>(gkey_u) + base;
  int64_t* val = gval + base;
  int32_t* L = glab + base;
  // on-chip windows that leave room for the digit counters sort with the
  // block radix sort (a few 8-bit passes) instead of the bitonic network
  const int64_t mp0 = pow2_at_least(2 * n);
  const bool radix = 44 * mp0 + 32 * 256 * 4 <= smem_cap && mp0 <= (1 << 20);
  int32_t(*rcnt)[256] = reinterpret_cast<int32_t(*)[256]>(dyn_smem + 44 * mp0);
  __shared__ int32_t rws[32];
  __shared__ unsigned long long rmn_s, rmx_s;
  if (44 * mp0 <= smem_cap) {
    key = reinterpret_cast<uint64_t*>(dyn_smem);
    val = reinterpret_cast<int64_t*>(key + 4 * mp0);
    L = reinterpret_cast<int32_t*>(val + mp0);
  }
  __shared__ int64_t tot_s;
  if (n == 0) {
    if (threadIdx.x == 0) { out.nruns[W.w] = 0; out.pages[W.w] = 0; out.run_base[W.w] = base; }
    return;
  }
  // 1. endpoints, sorted
  int64_t m = 2 * n, mp = pow2_at_least(m);
  for (int64_t i = threadIdx.x; i < mp; i += blockDim.x) {
    if (i < m) {
      const Iv& v = pool[W.pool_lo + (i >> 1)];
      key[i] = (uint64_t)((i & 1) ? v.b : v.a) ^ 0x8000000000000000ull;  // order-preserving
    } else {
      key[i] = ~0ull;
    }
    val[i] = 0;
  }
  __syncthreads();
  WRTS(1);
  if (radix) {
    // keys relative to the smallest endpoint: only the spanned bits are sorted
    unsigned long long vmn = ~0ull, vmx = 0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      vmn = key[i] < vmn ? key[i] : vmn;
      vmx = key[i] > vmx ? key[i] : vmx;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long a2 = __shfl_xor_sync(0xffffffffu, vmn, o), b2 = __shfl_xor_sync(0xffffffffu, vmx, o);
      vmn = a2 < vmn ? a2 : vmn;
      vmx = b2 > vmx ? b2 : vmx;
    }
    if (threadIdx.x == 0) { rmn_s = ~0ull; rmx_s = 0; }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { atomicMin(&rmn_s, vmn); atomicMax(&rmx_s, vmx); }
    __syncthreads();
    const unsigned long long mn = rmn_s;
    const int ebits = rmx_s > mn ? 64 - __clzll((long long)(rmx_s - mn)) : 0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) key[i] -= mn;
    __syncthreads();
    const bool in_b = block_radix_sort<1>(key, nullptr, nullptr, key + mp, nullptr, nullptr, (int)m, ebits, rcnt, rws, 0);
    const uint64_t* src = in_b ? key + mp : key;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) key[i] = src[i] + mn;
    __syncthreads();
  } else {
    bitonic_kv(key, val, mp);
  }
  WRTS(2);
  // 2. unique: flag first occurrences, scan to positions (val holds flags)
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) val[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
  __syncthreads();
  int64_t* pos = val;
  int64_t nu = block_scan_array<int64_t>(pos, m);
  // compact unique endpoints into E (reuse key region after m: use val2 area)
  int64_t* E = reinterpret_cast<int64_t*>(key) + mp;  // scratch has room: 4n >= mp + m
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    bool first = (i == 0 || key[i] != key[i - 1]);
    if (first) E[pos[i]] = (int64_t)(key[i] ^ 0x8000000000000000ull);
  }
  __syncthreads();
  int64_t nseg = nu - 1;
  for (int64_t k = threadIdx.x; k < nseg; k += blockDim.x) L[k] = kNone;
  __syncthreads();
  WRTS(3);
  // 3. label = min covering command (first access)
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const Iv& v = pool[W.pool_lo + i];
    // command of interval i: largest c with cmd_off[c] <= pool_lo + i
    int64_t gi = W.pool_lo + i;
    int32_t lo = W.c0, hi = W.c1;
    while (lo < hi) {
      int32_t mid = (lo + hi) >> 1;
      if (W.cmd_off[mid + 1] <= gi) lo = mid + 1; else hi = mid;
    }
    int32_t cmd = lo;
    int64_t s0 = lower_bound_i64(E, nu, v.a), s1 = lower_bound_i64(E, nu, v.b);
    for (int64_t k = s0; k < s1; ++k) atomicMin(&L[k], cmd);
  }
  __syncthreads();
  WRTS(4);
  // 4. runs: maximal segment groups with one label (segments abut by construction)
  int64_t* rflag = val;  // reuse: run-start flags -> run ids
  for (int64_t k = threadIdx.x; k < nseg; k += blockDim.x)
    rflag[k] = (L[k] != kNone && (k == 0 || L[k - 1] != L[k])) ? 1 : 0;
  __syncthreads();
  int64_t nr = block_scan_array<int64_t>(rflag, nseg);
  // run r: start segment = the k with flag; end = first k' > k with L[k'] != L[k]
  int64_t* ra = out.run_a + base;
  int64_t* rb = out.run_b + base;
  int32_t* rl = out.run_lab + base;
  for (int64_t k = threadIdx.x; k < nseg; k += blockDim.x) {
    if (L[k] == kNone) continue;
    bool start = (k == 0 || L[k - 1] != L[k]);
    bool end = (k + 1 == nseg || L[k + 1] != L[k]);
    int64_t r = rflag[k] - (start ? 0 : 0);
    // rflag is an exclusive scan of start flags: for a start segment it is its run id;
    // for non-start segments it equals (id of its run) + 1.
    int64_t id = start ? r : r - 1;
    if (start) { ra[id] = E[k]; rl[id] = L[k]; }
    if (end) rb[id] = E[k + 1];
  }
  __syncthreads();
  // 5. order runs by (label, start): key = label << 32 | run id (ids are in start order)
  int64_t rp = pow2_at_least(nr);
  uint64_t* k2 = key;       // reuse sort buffers (E no longer needed after this)
  int64_t* v2 = val;
  // E lives at key + mp; make sure we do not overwrite it before use: copy runs first
  __syncthreads();
  WRTS(5);
  if (radix) {
    // key = (label - c0, run id): labels are commands of [c0, c1)
    const int ib = nr > 1 ? 64 - __clzll((long long)(nr - 1)) : 0;
    const int lb = W.c1 - W.c0 > 1 ? 32 - __clz(W.c1 - W.c0 - 1) : 0;
    for (int64_t i = threadIdx.x; i < nr; i += blockDim.x)
      k2[i] = ((uint64_t)(uint32_t)(rl[i] - W.c0) << ib) | (uint64_t)i;
    __syncthreads();
    const bool in_b = block_radix_sort<1>(k2, nullptr, nullptr, k2 + rp, nullptr, nullptr, (int)nr, ib + lb, rcnt, rws, 0);
    const uint64_t* src = in_b ? k2 + rp : k2;
    for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) v2[i] = (int64_t)(src[i] & ((1ull << ib) - 1));
  } else {
    for (int64_t i = threadIdx.x; i < rp; i += blockDim.x) {
      k2[i] = i < nr ? (((uint64_t)(uint32_t)rl[i] << 32) | (uint64_t)i) : ~0ull;
      v2[i] = i;
    }
    __syncthreads();
    bitonic_kv(k2, v2, rp);
  }
  WRTS(6);
  // gather into final order (use the label area beyond nr as temp for permuted copy)
  int64_t* ta = reinterpret_cast<int64_t*>(key) + rp;   // temp arrays
  int64_t* tb = ta + nr;
  int32_t* tl = reinterpret_cast<int32_t*>(tb + nr);
  for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) {
    int64_t src = v2[i];
    ta[i] = ra[src]; tb[i] = rb[src]; tl[i] = rl[src];
  }
  __syncthreads();
  if (threadIdx.x == 0) tot_s = 0;
  __syncthreads();
  int64_t mine = 0;
  for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) {
    ra[i] = ta[i]; rb[i] = tb[i]; rl[i] = tl[i];
    mine += tb[i] - ta[i];
  }
  // one shared atomic per warp (1024 contended ones were ~10 % of the kernel)
#pragma unroll
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(reinterpret_cast<unsigned long long*>(&tot_s), (unsigned long long)mine);
  __syncthreads();
  if (threadIdx.x == 0) {
    out.nruns[W.w] = nr;
    out.pages[W.w] = tot_s;
    out.run_base[W.w] = base;
  }
  WRTS(15);
}

// ---------------------------------------------------------------------------
// Cross-window class table: elementary segments of all windows' runs, each
// with its tuple of per-window classes, ranked lexicographically.

struct CombineParams {
  int32_t nwin;
  const int64_t* run_a; const int64_t* run_b; const int32_t* run_lab;
  const int64_t* run_base; const int64_t* nruns;
  const int32_t* run_cls;   // optional explicit class per run (facade); else K_w - rank
  // dense map
  const int64_t* span_first; const int64_t* span_n; const int64_t* span_dense; int32_t nspans;
  // scratch (sized by host)
  uint64_t* key; int64_t* val; int64_t* E; int32_t* T; int64_t* idx;
  // outputs: covered segments sorted by dense start
  int64_t* seg_lo; int64_t* seg_hi; int32_t* seg_cls; int64_t* nseg_out; int64_t* ncls_out;
  uint64_t* wide;   // k_window_combine_wide's global scratch (3 x pow2(2M) words) when smem is short
};

__device__ int64_t dense_at(const CombineParams& P, int64_t a) {
  int lo = 0, hi = P.nspans;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (P.span_first[mid] <= a) lo = mid + 1; else hi = mid;
  }
  int s = lo - 1;
  return P.span_dense[s] + (a - P.span_first[s]);
}

__device__ __forceinline__ int tuple_cmp(const int32_t* T, int64_t i, int64_t j, int W) {
  for (int w = 0; w < W; ++w) {
    int32_t a = T[i * W + w], b = T[j * W + w];
    if (a != b) return a < b ? -1 : 1;
  }
  return 0;
}

__global__ void __launch_bounds__(1024, 1) k_window_combine(CombineParams P, int64_t smem_cap,
                                                             const int32_t* skip) {
  __shared__ int64_t tot_runs_s;
  if (skip && *skip) return;   // k_window_combine_wide already built the table
  int W = P.nwin;
  // gather all runs' endpoints
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < W; ++w) t += P.nruns[w];
    tot_runs_s = t;
  }
  __syncthreads();
  int64_t M = tot_runs_s;
  if (M == 0) {
    if (threadIdx.x == 0) { *P.nseg_out = 0; *P.ncls_out = 0; }
    return;
  }
  int64_t m = 2 * M, mp = pow2_at_least(m);
  if (8 * (4 * mp + m) + 4 * m * W <= smem_cap) {   // stage the scratch in shared memory
    P.key = reinterpret_cast<uint64_t*>(dyn_smem);
    P.val = reinterpret_cast<int64_t*>(P.key + mp);
    P.E = P.val + mp;
    P.idx = P.E + 2 * mp;
    P.T = reinterpret_cast<int32_t*>(P.idx + m);
  }
  // flatten (w, r) -> global run index g via per-window prefix (small W: linear walk)
  for (int64_t i = threadIdx.x; i < mp; i += blockDim.x) {
    if (i < m) {
      int64_t g = i >> 1, w = 0;
      while (g >= P.nruns[w]) { g -= P.nruns[w]; ++w; }
      int64_t r = P.run_base[w] + g;
      P.key[i] = (uint64_t)((i & 1) ? P.run_b[r] : P.run_a[r]) ^ 0x8000000000000000ull;
    } else {
      P.key[i] = ~0ull;
    }
    P.val[i] = 0;
  }
  __syncthreads();
  bitonic_kv(P.key, P.val, mp);
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) P.val[i] = (i == 0 || P.key[i] != P.key[i - 1]) ? 1 : 0;
  __syncthreads();
  int64_t nu = block_scan_array<int64_t>(P.val, m);
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x)
    if (i == 0 || P.key[i] != P.key[i - 1]) P.E[P.val[i]] = (int64_t)(P.key[i] ^ 0x8000000000000000ull);
  __syncthreads();
  int64_t ns = nu - 1;
  for (int64_t i = threadIdx.x; i < ns * W; i += blockDim.x) P.T[i] = 0;
  __syncthreads();
  // paint each run's class (K_w - rank) over its segments
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    int64_t g = i, w = 0;
    while (g >= P.nruns[w]) { g -= P.nruns[w]; ++w; }
    int64_t r = P.run_base[w] + g;
    int32_t cls = P.run_cls ? P.run_cls[r] : (int32_t)(P.nruns[w] - g);
    int64_t s0 = lower_bound_i64(P.E, nu, P.run_a[r]), s1 = lower_bound_i64(P.E, nu, P.run_b[r]);
    for (int64_t k = s0; k < s1; ++k) P.T[k * W + w] = cls;
  }
  __syncthreads();
  // covered segments -> compact indices
  for (int64_t k = threadIdx.x; k < ns; k += blockDim.x) {
    bool cov = false;
    for (int w = 0; w < W; ++w) cov |= P.T[k * W + w] != 0;
    P.val[k] = cov ? 1 : 0;
  }
  __syncthreads();
  int64_t nc = block_scan_array<int64_t>(P.val, ns);
  for (int64_t k = threadIdx.x; k < ns; k += blockDim.x) {
    bool cov = (k + 1 < ns ? P.val[k + 1] : nc) != P.val[k];
    if (cov) P.idx[P.val[k]] = k;
  }
  __syncthreads();
  // sort covered segments by tuple (comparison bitonic over indices)
  int64_t cp = pow2_at_least(nc);
  int64_t* perm = P.val;  // reuse
  for (int64_t i = threadIdx.x; i < cp; i += blockDim.x) perm[i] = i < nc ? P.idx[i] : -1;
  __syncthreads();
  // Tuples fit a mixed-radix 64-bit key (radix K_w + 1 per window) in all
  // practical cases; then sort plain keys.  Otherwise compare tuples.
  __shared__ int use_key_s;
  if (threadIdx.x == 0) {
    double bits = 0;
    for (int w = 0; w < W; ++w) bits += log2((double)P.nruns[w] + 1.0);
    use_key_s = bits <= 40.0 && nc < (1ll << 24);   // 24 low bits: the segment index tie-break
  }
  __syncthreads();
  bool use_key = use_key_s;
  if (use_key) {
    uint64_t* k3 = reinterpret_cast<uint64_t*>(P.key);
    for (int64_t i = threadIdx.x; i < cp; i += blockDim.x) {
      if (i < nc) {
        int64_t sidx = P.idx[i];
        uint64_t kk = 0;
        for (int w = 0; w < W; ++w) kk = kk * (uint64_t)(P.nruns[w] + 1) + (uint64_t)P.T[sidx * W + w];
        k3[i] = (kk << 24) | (uint64_t)i;
        perm[i] = sidx;
      } else {
        k3[i] = ~0ull;
        perm[i] = -1;
      }
    }
    __syncthreads();
    bitonic_kv(k3, perm, cp);
  }
  for (int64_t k = 2; k <= cp && !use_key; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < cp; i += blockDim.x) {
        int64_t l = i ^ j;
        if (l > i) {
          bool up = (i & k) == 0;
          int64_t a = perm[i], b = perm[l];
          int c;
          if (a < 0 && b < 0) c = 0;
          else if (a < 0) c = 1;
          else if (b < 0) c = -1;
          else { c = tuple_cmp(P.T, a, b, W); if (c == 0) c = a < b ? -1 : (a > b ? 1 : 0); }
          if ((c > 0) == up) { perm[i] = b; perm[l] = a; }
        }
      }
      __syncthreads();
    }
  }
  // dense rank of distinct tuples (1-based); write class per segment via key scratch
  int64_t* rk = reinterpret_cast<int64_t*>(P.key);   // sort keys are dead here
  for (int64_t i = threadIdx.x; i < nc; i += blockDim.x)
    rk[i] = (i == 0 || tuple_cmp(P.T, perm[i - 1], perm[i], W) != 0) ? 1 : 0;
  __syncthreads();
  int64_t ndist = block_scan_array<int64_t>(rk, nc);
  // rk[i] = (#distinct before i); class = rk + (first? 1 : 0) ... recompute inclusive
  for (int64_t i = threadIdx.x; i < nc; i += blockDim.x) {
    bool first = (i == 0 || tuple_cmp(P.T, perm[i - 1], perm[i], W) != 0);
    int64_t cls = rk[i] + (first ? 1 : 0);
    // store into T's first column slot of that segment is unsafe (needed by neighbours);
    // write to the output by covered position instead: segments in E order
    P.E[nu + perm[i]] = cls;      // scratch after E: class per segment index
  }
  __syncthreads();
  for (int64_t ci = threadIdx.x; ci < nc; ci += blockDim.x) {
    int64_t k = P.idx[ci];
    P.seg_lo[ci] = dense_at(P, P.E[k]);
    P.seg_hi[ci] = P.seg_lo[ci] + (P.E[k + 1] - P.E[k]);
    P.seg_cls[ci] = (int32_t)P.E[nu + k];
  }
  if (threadIdx.x == 0) { *P.nseg_out = nc; *P.ncls_out = ndist; }
}

// Wide variant of the class table for many runs (fragmented windows: hundreds
// of single-page runs per window).  The per-window classes fold into one
// 128-bit mixed-radix key per elementary segment (window 0 most significant,
// radix = max class + 1 per window), painted window by window (runs of one
// window are disjoint, so no two threads write one segment in a pass); the
// segments are then sorted by key in shared memory (uncovered segments carry
// the all-ones key and sort last) and dense-ranked.  Replaces the tuple
// comparison sort of k_window_combine whenever the radices fit 127 bits.
typedef unsigned __int128 u128;
constexpr int64_t kWideSmem = 224 * 1024;   // + ~1.6 KB static: within the 227 KB opt-in

__device__ void bitonic_u128(uint64_t* klo, uint64_t* khi, int32_t* idx, int64_t npow2) {
  for (int64_t k = 2; k <= npow2; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < npow2; i += blockDim.x) {
        int64_t l = i ^ j;
        if (l > i) {
          bool up = (i & k) == 0;
          bool gt = khi[i] > khi[l] || (khi[i] == khi[l] && klo[i] > klo[l]);
          if (gt == up) {
            uint64_t t = klo[i]; klo[i] = klo[l]; klo[l] = t;
            t = khi[i]; khi[i] = khi[l]; khi[l] = t;
            int32_t ti = idx[i]; idx[i] = idx[l]; idx[l] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ void bitonic_u64(uint64_t* key, int64_t npow2) {
  for (int64_t k = 2; k <= npow2; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < npow2; i += blockDim.x) {
        int64_t l = i ^ j;
        if (l > i) {
          bool up = (i & k) == 0;
          if ((key[i] > key[l]) == up) { uint64_t t = key[i]; key[i] = key[l]; key[l] = t; }
        }
      }
      __syncthreads();
    }
  }
}

// *ok_out = 0 when the radices do not fit 127 bits (the caller then runs
// k_window_combine); otherwise the outputs of k_window_combine.
// Stable block-wide LSD radix sort (8-bit digits, 1024 threads) of n
// elements held in shared memory as SoA: NW 64-bit key words (k0 = low word,
// k1 = high word when NW == 2) and an optional int32 payload.  Warp w owns
// the contiguous elements [w * per, (w + 1) * per): counting and scattering
// walk them in order, so equal digits keep their relative order.  The sort
// ping-pongs between buffers a and b; returns true when the result is in b.
template <int NW>
__device__ bool block_radix_sort(uint64_t* a0, uint64_t* a1, int32_t* av, uint64_t* b0, uint64_t* b1, int32_t* bv,
                                 int n, int nbits, int32_t (*cnt)[256], int32_t* warp_s, int sh0) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const int per = ((n + 31) / 32 + 31) & ~31;
  const int lo = w * per, hi = lo + per < n ? lo + per : n;
  bool in_b = false;
  for (int sh = sh0; sh < nbits; sh += 8) {   // key bits [sh0, nbits)
    uint64_t* s0 = in_b ? b0 : a0; uint64_t* s1 = in_b ? b1 : a1; int32_t* sv = in_b ? bv : av;
    uint64_t* d0 = in_b ? a0 : b0; uint64_t* d1 = in_b ? a1 : b1; int32_t* dv = in_b ? av : bv;
    auto digit = [&](int i) -> int {
      const uint64_t word = (NW == 2 && sh >= 64) ? s1[i] : s0[i];
      return (int)((word >> (sh & 63)) & 255);
    };
    for (int j = lane; j < 256; j += 32) cnt[w][j] = 0;
    __syncwarp();
    // counts need no order: one shared atomic per element on the warp's own
    // row (__match_any_sync here cost 9x more: tools/radix_probe.cu)
    for (int i0 = lo; i0 < hi; i0 += 32) {
      const int i = i0 + lane;
      if (i < hi) atomicAdd(&cnt[w][digit(i)], 1);
    }
    __syncthreads();
    // exclusive offsets in (digit, warp) order: thread d < 256 walks digit d's
    // column over the 32 warp rows (consecutive digits: conflict-free), the
    // 256 digit totals are scanned by warps 0-7, and the digit bases are added
    // back down the columns -- two barriers instead of a 1024-wide block scan
    // (the scan was the fixed cost of a pass: tools/radix_probe.cu)
    {
      const int t = threadIdx.x, ln = t & 31, wid = t >> 5;
      int32_t excl = 0;
      if (t < 256) {
        int32_t tot = 0;
#pragma unroll 8
        for (int ww = 0; ww < 32; ++ww) { const int32_t c = cnt[ww][t]; cnt[ww][t] = tot; tot += c; }
        int32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (ln >= o) x += y;
        }
        if (ln == 31) warp_s[wid] = x;
        excl = x - tot;
      }
      __syncthreads();
      if (t < 256) {
        int32_t base = excl;
        for (int k = 0; k < wid; ++k) base += warp_s[k];
#pragma unroll 8
        for (int ww = 0; ww < 32; ++ww) cnt[ww][t] += base;
      }
    }
    __syncthreads();
    for (int i0 = lo; i0 < hi; i0 += 32) {
      const int i = i0 + lane;
      const int d = i < hi ? digit(i) : 256;
      // lanes holding the same digit, built from nine ballots (the stable
      // rank is the count of such lanes below this one)
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int bt = 0; bt < 9; ++bt) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> bt) & 1);
        peers &= ((d >> bt) & 1) ? bal : ~bal;
      }
      const int32_t before = d < 256 ? cnt[w][d] : 0;
      __syncwarp();
      if (d < 256) {
        const int o = before + __popc(peers & lt);
        d0[o] = s0[i];
        if (NW == 2) d1[o] = s1[i];
        if (sv) dv[o] = sv[i];
        if (lane == __ffs(peers) - 1) cnt[w][d] = before + __popc(peers);
      }
      __syncwarp();
    }
    __syncthreads();
    in_b = !in_b;
  }
  return in_b;
}

__global__ void __launch_bounds__(1024, 1) k_window_combine_wide(CombineParams P, int64_t smem_cap, int32_t* ok_out) {
  PHTS_DECL;
  CWTS(0);
  __shared__ int64_t tot_runs_s;
  __shared__ u128 mult_s[64];
  __shared__ int32_t rad_s[64];
  __shared__ int ok_s;
  __shared__ int64_t npre_s[65], rbase_s[64];   // per-window run prefix and scratch base (W <= 64)
  const int W = P.nwin;
  if (threadIdx.x < 64) rad_s[threadIdx.x] = 0;
  // per-window counts and bases loaded by one thread each (one thread walking
  // them was a chain of dependent global round trips), then prefixed
  if (threadIdx.x < W && threadIdx.x < 64) {
    npre_s[threadIdx.x + 1] = P.nruns[threadIdx.x];
    rbase_s[threadIdx.x] = P.run_base[threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int Wc = W < 64 ? W : 64;   // (W > 64 exits below, before the total is used)
    npre_s[0] = 0;
    for (int w = 0; w < Wc; ++w) npre_s[w + 1] += npre_s[w];
    tot_runs_s = npre_s[Wc];
  }
  __syncthreads();
  const int64_t M = tot_runs_s;
  if (W > 64) {   // beyond the radix table: the tuple-comparison kernel takes it
    if (threadIdx.x == 0) *ok_out = 0;
    return;
  }
  // radix per window: max class + 1
  for (int64_t i0 = 0; i0 < M; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    int w = -1;
    int32_t cls = 0;
    if (i < M) {
      w = 0;
      while (i >= npre_s[w + 1]) ++w;   // (shared memory; empty windows are skipped)
      const int64_t g = i - npre_s[w];
      const int64_t r = rbase_s[w] + g;
      cls = P.run_cls ? P.run_cls[r] : (int32_t)(npre_s[w + 1] - npre_s[w] - g);
    }
    // one shared atomic per window present in the warp (lanes of a window
    // are contiguous): 1024 contended atomics on <= 64 words were serialised
    const uint32_t peers = __match_any_sync(0xffffffffu, w);
    const int32_t mx = __reduce_max_sync(peers, cls);
    if (w >= 0 && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicMax(&rad_s[w], mx);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ok_s = W <= 64;
    u128 m = 1;
    for (int w = W - 1; w >= 0 && ok_s; --w) {
      mult_s[w] = m;
      // m * rad <= 2^127 (the radices fit), decided from the 64-bit halves of
      // the product instead of a 128-bit division
      const uint64_t rad = (uint64_t)(uint32_t)rad_s[w] + 1;
      const u128 lo = (u128)(uint64_t)m * rad;
      const u128 hi = (m >> 64) * rad + (lo >> 64);   // product >> 64 (< 2^97)
      if (hi > ((u128)1 << 63) || (hi == ((u128)1 << 63) && (uint64_t)lo != 0)) ok_s = 0;
      else m *= rad;
    }
    *ok_out = ok_s;
  }
  __syncthreads();
  if (!ok_s) return;
  if (M == 0) {
    if (threadIdx.x == 0) { *P.nseg_out = 0; *P.ncls_out = 0; }
    return;
  }
  const int64_t m0 = 2 * M;
  // ---- on-chip radix path: shared memory holds R0 [0, 16m) (endpoint sort,
  // then the per-segment keys, then one sort buffer) | E [16m, 24m) | digit
  // counters (32 KB) | X (the covered segments, 20 B each)
  {
    const int64_t e_off = 16 * m0, cnt_off = 24 * m0, x_off = 24 * m0 + 32 * 256 * 4;
    __shared__ unsigned long long mn_s, mx_s, klo_max_s, khi_max_s;
    __shared__ int32_t rwarp_s[32];
    __shared__ int64_t nc_s;
    if (x_off <= smem_cap && m0 < (1ll << 30)) {
      const int m = (int)m0;
      uint64_t* ea = reinterpret_cast<uint64_t*>(dyn_smem);
      uint64_t* eb = ea + m;
      int64_t* E = reinterpret_cast<int64_t*>(dyn_smem + e_off);
      int32_t(*cnt)[256] = reinterpret_cast<int32_t(*)[256]>(dyn_smem + cnt_off);
      if (threadIdx.x == 0) { mn_s = ~0ull; mx_s = 0; klo_max_s = 0; khi_max_s = 0; }
      // endpoints as dense page ids when the span table fits the X region
      // (unused until the painting is done): the dense map is monotone and
      // only closes the gaps between spans, which no run covers, so the
      // covered segments are the same and the keys span fewer bits (one radix
      // pass less at the fragmented configuration: 30 -> 22 bits)
      const bool dmode = P.nspans <= 1024 && x_off + 16ll * P.nspans <= smem_cap;
      int64_t* sfirst = reinterpret_cast<int64_t*>(dyn_smem + x_off);
      int64_t* sdense = sfirst + P.nspans;
      if (dmode)
        for (int i = threadIdx.x; i < P.nspans; i += blockDim.x) { sfirst[i] = P.span_first[i]; sdense[i] = P.span_dense[i]; }
      __syncthreads();
      auto to_dense = [&](int64_t a) -> int64_t {
        if (!dmode) return a;
        int lo = 0, hi = P.nspans;
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (sfirst[mid] <= a) lo = mid + 1; else hi = mid; }
        return sdense[lo - 1] + (a - sfirst[lo - 1]);
      };
      {
        unsigned long long vmn = ~0ull, vmx = 0;
#pragma unroll 4
        for (int i = threadIdx.x; i < m; i += blockDim.x) {   // (unrolled: the endpoint loads overlap)
          const int64_t gi = i >> 1;
          int w = 0;
          while (gi >= npre_s[w + 1]) ++w;
          const int64_t r = rbase_s[w] + (gi - npre_s[w]);
          const uint64_t v = (uint64_t)to_dense((i & 1) ? P.run_b[r] : P.run_a[r]);
          ea[i] = v;
          vmn = v < vmn ? v : vmn;
          vmx = v > vmx ? v : vmx;
        }
        // warp-reduced, then one shared atomic per warp (was two per endpoint)
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const unsigned long long a2 = __shfl_xor_sync(0xffffffffu, vmn, o), b2 = __shfl_xor_sync(0xffffffffu, vmx, o);
          vmn = a2 < vmn ? a2 : vmn;
          vmx = b2 > vmx ? b2 : vmx;
        }
        if ((threadIdx.x & 31) == 0) { atomicMin(&mn_s, vmn); atomicMax(&mx_s, vmx); }
      }
      __syncthreads();
      CWTS(1);
      const uint64_t mn = mn_s;
      for (int i = threadIdx.x; i < m; i += blockDim.x) ea[i] -= mn;
      const int ebits = mx_s > mn ? 64 - __clzll((long long)(mx_s - mn)) : 0;
      __syncthreads();
      const bool ein_b = block_radix_sort<1>(ea, nullptr, nullptr, eb, nullptr, nullptr, m, ebits, cnt, rwarp_s, 0);
      CWTS(2);
      const uint64_t* es = ein_b ? eb : ea;
      // unique endpoints -> E: each thread owns a contiguous run of the sorted
      // endpoints, one block scan of the per-thread unique counts
      int nu;
      {
        const int per_e = (m + (int)blockDim.x - 1) / (int)blockDim.x;
        const int i0 = (int)threadIdx.x * per_e, i1 = i0 + per_e < m ? i0 + per_e : m;
        int mine = 0;
        for (int i = i0; i < i1; ++i) mine += (i == 0 || es[i] != es[i - 1]);
        int32_t tot;
        int o = block_excl_scan<int32_t>(mine, rwarp_s, &tot);
        for (int i = i0; i < i1; ++i)
          if (i == 0 || es[i] != es[i - 1]) E[o++] = (int64_t)(es[i] + mn);
        nu = tot;
      }
      __syncthreads();
      const int ns = nu - 1;
      // per-segment 128-bit keys in R0 (the endpoint buffers are dead)
      uint64_t* klo = ea;
      uint64_t* khi = ea + ns;
      for (int k = threadIdx.x; k < ns; k += blockDim.x) { klo[k] = 0; khi[k] = 0; }
      __syncthreads();
      CWTS(3);
      // every window's runs at once (was one window per barrier round): a
      // segment several windows cover sums their contributions with 64-bit
      // shared atomics, each low-word add's carry added to the high word, so
      // the 128-bit total does not depend on the order
      for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
        int w = 0;
        while (i >= npre_s[w + 1]) ++w;
        const int64_t g = i - npre_s[w], nr = npre_s[w + 1] - npre_s[w];
        const int64_t r = rbase_s[w] + g;
        const int32_t cls = P.run_cls ? P.run_cls[r] : (int32_t)(nr - g);
        const u128 add = mult_s[w] * (u128)(uint32_t)cls;
        const unsigned long long alo = (uint64_t)add, ahi = (uint64_t)(add >> 64);
        const int64_t s0 = lower_bound_i64(E, nu, to_dense(P.run_a[r])), s1 = lower_bound_i64(E, nu, to_dense(P.run_b[r]));
        for (int64_t k = s0; k < s1; ++k) {
          const unsigned long long old = atomicAdd(reinterpret_cast<unsigned long long*>(klo + k), alo);
          const unsigned long long c = old + alo < old ? 1ull : 0ull;
          if (ahi | c) atomicAdd(reinterpret_cast<unsigned long long*>(khi + k), ahi + c);
        }
      }
      __syncthreads();
      CWTS(4);
      // covered segments -> X (key lo, key hi, segment index), in segment order.
      // Each thread owns a contiguous run of segments: one count and one
      // block scan give every thread its output offset (was a barrier-bound
      // scan round per 1024 segments)
      const int per_t = (ns + (int)blockDim.x - 1) / (int)blockDim.x;
      const int k0 = (int)threadIdx.x * per_t, k1 = k0 + per_t < ns ? k0 + per_t : ns;
      int mine = 0;
      for (int k = k0; k < k1; ++k) mine += (klo[k] | khi[k]) != 0;
      int32_t nc_tot;
      const int32_t my_off = block_excl_scan<int32_t>(mine, rwarp_s, &nc_tot);
      const int nc = nc_tot;
      if (20ll * nc > 16 * m0 || x_off + 20ll * nc > smem_cap) {
        // the covered set does not fit on chip: the tuple-comparison kernel takes it
        if (threadIdx.x == 0) *ok_out = 0;
        return;
      }
      uint64_t* xlo = reinterpret_cast<uint64_t*>(dyn_smem + x_off);
      uint64_t* xhi = xlo + nc;
      int32_t* xid = reinterpret_cast<int32_t*>(xhi + nc);
      for (int k = threadIdx.x; k < ns; k += blockDim.x) P.E[nu + k] = 0;
      int64_t rcarry = 0;
      // ---- grouped path.  In key order the covered segments fall into
      // groups by (w*, c*): the first window a segment is in and its class
      // there (every earlier window's digit is 0), w* descending, then c*
      // ascending; within a group (the segments of one run of window w*) the
      // later windows decide.  Sorting by that short primary key (a few
      // radix passes instead of up to sixteen over the 128-bit key) and
      // insertion-sorting the groups by the full key gives the same order.
      // Groups are single segments when windows hold scattered pages; a
      // group of more than 32 segments falls back to the full-key sort.
      bool ranked = false;
      {
        constexpr int IDB = 20;   // segment index bits of a packed key
        int wb = 0;
        while ((1 << wb) < W) ++wb;
        int32_t cmax = 0;
        for (int w = 0; w < W; ++w) cmax = rad_s[w] > cmax ? rad_s[w] : cmax;
        int cb = 0;
        while ((1ll << cb) <= (int64_t)cmax) ++cb;
        __shared__ int big_s;
        if (IDB + wb + cb <= 64 && ns < (1 << IDB)) {
          uint64_t* pk = xlo;   // packed (primary << IDB | segment), in segment order
          uint64_t* pk2 = xhi;  // the sort's second buffer
          int o = my_off;
          for (int k = k0; k < k1; ++k) {
            if ((klo[k] | khi[k]) == 0) continue;
            const u128 key = ((u128)khi[k]) << 64 | klo[k];
            int ws = 0;   // smallest w with mult[w] <= key (mult falls with w)
            while (ws + 1 < W && mult_s[ws] > key) ++ws;
            // c* = key / mult[w*]: a double-precision estimate (within one of
            // the quotient, which is < 2^20), corrected exactly -- a 128-bit
            // division per segment was the phase's cost
            const u128 mw = mult_s[ws];
            const double kd = (double)khi[k] * 18446744073709551616.0 + (double)klo[k];
            const double md = (double)(uint64_t)(mw >> 64) * 18446744073709551616.0 + (double)(uint64_t)mw;
            uint64_t cs = (uint64_t)(kd / md);
            while (cs > 0 && (u128)cs * mw > key) --cs;
            while ((u128)(cs + 1) * mw <= key) ++cs;
            pk[o++] = ((((uint64_t)(W - 1 - ws)) << cb | cs) << IDB) | (uint64_t)k;
          }
          if (threadIdx.x == 0) big_s = 0;
          __syncthreads();
          CWTS(5);
          const bool in_b = block_radix_sort<1>(pk, nullptr, nullptr, pk2, nullptr, nullptr, nc, IDB + wb + cb, cnt,
                                                rwarp_s, IDB);
          uint64_t* ps = in_b ? pk2 : pk;
          constexpr uint64_t kSeg = (1ull << IDB) - 1;
          auto kless = [&](uint64_t u, uint64_t v) {
            const int a = (int)(u & kSeg), b = (int)(v & kSeg);
            return khi[a] < khi[b] || (khi[a] == khi[b] && klo[a] < klo[b]);
          };
          // group starts first (the free payload slots of X hold the flags), so
          // a group's thread reads and writes only its own group's entries
          int32_t* gstart = xid;
          for (int i = threadIdx.x; i < nc; i += blockDim.x)
            gstart[i] = i == 0 || (ps[i - 1] >> IDB) != (ps[i] >> IDB);
          __syncthreads();
          for (int i = threadIdx.x; i < nc; i += blockDim.x) {
            if (!gstart[i]) continue;
            int j = i + 1;
            while (j < nc && !gstart[j] && j - i <= 32) ++j;
            if (j - i > 32) { atomicOr(&big_s, 1); continue; }
            for (int a = i + 1; a < j; ++a) {
              const uint64_t v = ps[a];
              int b = a;
              while (b > i && kless(v, ps[b - 1])) { ps[b] = ps[b - 1]; --b; }
              ps[b] = v;
            }
          }
          __syncthreads();
          CWTS(6);
          if (!big_s) {
            for (int base = 0; base < nc; base += blockDim.x) {
              const int i = base + threadIdx.x;
              bool first = false;
              if (i < nc) {
                const int a = (int)(ps[i] & kSeg);
                first = i == 0;
                if (!first) {
                  const int b = (int)(ps[i - 1] & kSeg);
                  first = klo[a] != klo[b] || khi[a] != khi[b];
                }
              }
              int32_t tot;
              const int32_t ex = block_excl_scan<int32_t>(first ? 1 : 0, rwarp_s, &tot);
              if (i < nc) P.E[nu + (int64_t)(ps[i] & kSeg)] = rcarry + ex + (first ? 1 : 0);
              rcarry += tot;
            }
            ranked = true;
          }
        }
      }
      if (!ranked) {
      int64_t carry = 0;
      unsigned long long hmax = 0, lmax = 0;
      for (int base = 0; base < ns; base += blockDim.x) {
        const int k = base + threadIdx.x;
        const bool cov = k < ns && (klo[k] | khi[k]) != 0;
        int32_t tot;
        const int32_t ex = block_excl_scan<int32_t>(cov ? 1 : 0, rwarp_s, &tot);
        if (cov) {
          const int o = (int)(carry + ex);
          xlo[o] = klo[k]; xhi[o] = khi[k]; xid[o] = k;
          hmax = khi[k] > hmax ? khi[k] : hmax;
          lmax = klo[k] > lmax ? klo[k] : lmax;
        }
        carry += tot;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long a2 = __shfl_xor_sync(0xffffffffu, hmax, o), b2 = __shfl_xor_sync(0xffffffffu, lmax, o);
        hmax = a2 > hmax ? a2 : hmax;
        lmax = b2 > lmax ? b2 : lmax;
      }
      if ((threadIdx.x & 31) == 0) { atomicMax(&khi_max_s, hmax); atomicMax(&klo_max_s, lmax); }
      __syncthreads();
      const int kbits = khi_max_s ? 128 - __clzll((long long)khi_max_s) : (klo_max_s ? 64 - __clzll((long long)klo_max_s) : 0);
      // the sort's second buffer in R0 (the per-segment keys are dead)
      uint64_t* ylo = ea;
      uint64_t* yhi = ylo + nc;
      int32_t* yid = reinterpret_cast<int32_t*>(yhi + nc);
      const bool kin_b = block_radix_sort<2>(xlo, xhi, xid, ylo, yhi, yid, nc, kbits, cnt, rwarp_s, 0);
      const uint64_t* slo = kin_b ? ylo : xlo;
      const uint64_t* shi = kin_b ? yhi : xhi;
      const int32_t* sid = kin_b ? yid : xid;
      // dense rank of the distinct keys; class per segment (0 = uncovered) in P.E[nu + k]
      for (int base = 0; base < nc; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const bool first = i < nc && (i == 0 || slo[i] != slo[i - 1] || shi[i] != shi[i - 1]);
        int32_t tot;
        const int32_t ex = block_excl_scan<int32_t>(first ? 1 : 0, rwarp_s, &tot);
        if (i < nc) P.E[nu + sid[i]] = rcarry + ex + (first ? 1 : 0);
        rcarry += tot;
      }
      }   // !ranked
      __syncthreads();
      CWTS(7);
      // covered segments in E order -> the class table
      int64_t oc = 0;
      for (int base = 0; base < ns; base += blockDim.x) {
        const int k = base + threadIdx.x;
        const int64_t cls = k < ns ? P.E[nu + k] : 0;
        int32_t tot;
        const int32_t ex = block_excl_scan<int32_t>(cls > 0 ? 1 : 0, rwarp_s, &tot);
        if (cls > 0) {
          const int64_t ci = oc + ex;
          P.seg_lo[ci] = dmode ? E[k] : dense_at(P, E[k]);
          P.seg_hi[ci] = P.seg_lo[ci] + (E[k + 1] - E[k]);
          P.seg_cls[ci] = (int32_t)cls;
        }
        oc += tot;
      }
      if (threadIdx.x == 0) { *P.nseg_out = nc; *P.ncls_out = rcarry; }
      CWTS(15);
      return;
    }
  }
  // 1. sorted unique endpoints -> E.  On chip when the segment sort (20 B per
  // padded segment, <= mp) and E (8 B per endpoint) fit: the endpoint sort
  // runs in the segment-sort region, E after it, so every search below is a
  // shared-memory search.
  const int64_t m = 2 * M, mp = pow2_at_least(m);
  const bool on_chip = 20 * mp + 8 * m <= smem_cap;
  uint64_t* ek = on_chip ? reinterpret_cast<uint64_t*>(dyn_smem) : P.key;
  int64_t* E = on_chip ? reinterpret_cast<int64_t*>(dyn_smem + 20 * mp) : P.E;
  for (int64_t i = threadIdx.x; i < mp; i += blockDim.x) {
    if (i < m) {
      int64_t g = i >> 1, w = 0;
      while (g >= P.nruns[w]) { g -= P.nruns[w]; ++w; }
      int64_t r = P.run_base[w] + g;
      ek[i] = (uint64_t)((i & 1) ? P.run_b[r] : P.run_a[r]) ^ 0x8000000000000000ull;
    } else {
      ek[i] = ~0ull;
    }
  }
  __syncthreads();
  bitonic_u64(ek, mp);
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) P.val[i] = (i == 0 || ek[i] != ek[i - 1]) ? 1 : 0;
  __syncthreads();
  const int64_t nu = block_scan_array<int64_t>(P.val, m);
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x)
    if (i == 0 || ek[i] != ek[i - 1]) E[P.val[i]] = (int64_t)(ek[i] ^ 0x8000000000000000ull);
  __syncthreads();
  const int64_t ns = nu - 1, sp = pow2_at_least(ns > 0 ? ns : 1);
  // 2. per-segment 128-bit keys, painted window by window
  uint64_t *klo, *khi;
  int32_t* idx;
  if (on_chip) {
    klo = reinterpret_cast<uint64_t*>(dyn_smem); khi = klo + sp; idx = reinterpret_cast<int32_t*>(khi + sp);
  } else {
    klo = P.wide; khi = P.wide + mp; idx = reinterpret_cast<int32_t*>(P.wide + 2 * mp);
  }
  for (int64_t k = threadIdx.x; k < sp; k += blockDim.x) { klo[k] = 0; khi[k] = 0; idx[k] = (int32_t)k; }
  __syncthreads();
  int64_t g0 = 0;
  for (int w = 0; w < W; ++w) {
    const int64_t nr = P.nruns[w];
    const u128 mw = mult_s[w];
    for (int64_t g = threadIdx.x; g < nr; g += blockDim.x) {
      const int64_t r = P.run_base[w] + g;
      const int32_t cls = P.run_cls ? P.run_cls[r] : (int32_t)(nr - g);
      const u128 add = mw * (u128)(uint32_t)cls;
      const int64_t s0 = lower_bound_i64(E, nu, P.run_a[r]), s1 = lower_bound_i64(E, nu, P.run_b[r]);
      for (int64_t k = s0; k < s1; ++k) {
        u128 v = (((u128)khi[k]) << 64 | klo[k]) + add;
        klo[k] = (uint64_t)v; khi[k] = (uint64_t)(v >> 64);
      }
    }
    g0 += nr;
    __syncthreads();
  }
  // uncovered segments (key 0) and padding sort last
  for (int64_t k = threadIdx.x; k < sp; k += blockDim.x)
    if (k >= ns || (klo[k] == 0 && khi[k] == 0)) { klo[k] = ~0ull; khi[k] = ~0ull; }
  __syncthreads();
  bitonic_u128(klo, khi, idx, sp);
  // 3. dense rank of distinct covered keys; class per segment into E[nu + k]
  int64_t* rk = P.val;
  for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) {
    const bool cov = !(klo[i] == ~0ull && khi[i] == ~0ull);
    rk[i] = cov && (i == 0 || klo[i] != klo[i - 1] || khi[i] != khi[i - 1]) ? 1 : 0;
  }
  __syncthreads();
  const int64_t ndist = block_scan_array<int64_t>(rk, ns);
  // class per segment (0 = uncovered; global P.E[nu + k]): every slot first, since sorted
  // positions below ns may hold padding entries whose index is >= ns
  for (int64_t k = threadIdx.x; k < ns; k += blockDim.x) P.E[nu + k] = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) {
    const bool cov = !(klo[i] == ~0ull && khi[i] == ~0ull);
    const bool first = cov && (i == 0 || klo[i] != klo[i - 1] || khi[i] != khi[i - 1]);
    if (cov) P.E[nu + idx[i]] = rk[i] + (first ? 1 : 0);
  }
  __syncthreads();
  // 4. covered segments in E order -> the class table
  for (int64_t k = threadIdx.x; k < ns; k += blockDim.x) P.val[k] = P.E[nu + k] > 0 ? 1 : 0;
  __syncthreads();
  const int64_t nc = block_scan_array<int64_t>(P.val, ns);
  for (int64_t k = threadIdx.x; k < ns; k += blockDim.x) {
    const int64_t cls = P.E[nu + k];
    if (cls > 0) {
      const int64_t ci = P.val[k];
      P.seg_lo[ci] = dense_at(P, E[k]);
      P.seg_hi[ci] = P.seg_lo[ci] + (E[k + 1] - E[k]);
      P.seg_cls[ci] = (int32_t)cls;
    }
  }
  if (threadIdx.x == 0) { *P.nseg_out = nc; *P.ncls_out = ndist; }
}

// ---------------------------------------------------------------------------
// K3 fast path: every window's first-access runs, the cross-window class
// table and window 0's demand runs in ONE single-CTA launch (memman.py:174-206
// + the reorder classes of DESIGN.md section 3 + engine.py:310-313).  Used
// when the windows hold <= 512 predicted intervals in total (all configs
// here: <= 168), so every sort is one element per thread: a 1024-wide
// bitonic network with shuffles for strides < 32 and shared memory above.
// Descriptors travel as kernel parameters; all searches run in shared memory.

constexpr int FW_MAX_WIN = 16;
constexpr int FW_MAX_IV = 512;   // 2 x 512 endpoints: one per thread of a 1024-thread CTA
constexpr int FW_MAX_SPANS = 1024;
constexpr uint64_t FW_POS = (1ull << 48) - 1;
constexpr int FW_SP_CAP = 4096;    // window-0 commands whose self-populating flags are staged
constexpr int FW_LAB_SCAN = 128;   // up to this many intervals, labels are a per-segment scan (else atomics)

struct FusedWinParams {
  WinDesc wd[FW_MAX_WIN];
  int32_t nwin;
  WinOut out;
  const int64_t* span_first; const int64_t* span_dense; int32_t nspans;
  int64_t* seg_lo; int64_t* seg_hi; int32_t* seg_cls; int64_t* nseg_out; int64_t* ncls_out;
  RangeOut R;            // window 0 demand runs (R.nr == nullptr: not wanted)
};

struct FwSmem {
  int64_t ia[FW_MAX_IV], ib[FW_MAX_IV];
  int32_t iw[FW_MAX_IV], icmd[FW_MAX_IV];
  uint64_t E[1024];             // unique window-tagged endpoints
  int32_t L[1024];              // first-access command per segment
  uint64_t xk[1024], xk2[1024]; // bitonic exchange (two buffers: one barrier per wide stage)
  int32_t xv[1024];
  uint64_t yk[1024], yk2[1024];
  int32_t yv[1024];
  int64_t ra[1024], rb[1024];   // runs by id (start order), abs
  int32_t rl[1024], rsk[1024], rek[1024];
  int64_t sa[1024], sb[1024];   // runs in first-access order (window, label, start)
  int32_t sl[1024], sw[1024], scls[1024];
  uint8_t isb[1024];
  uint64_t E2[1024];            // unique run boundaries (abs)
  unsigned __int128 skey[1024]; // mixed-radix class tuple per elementary segment
  int32_t cls_of[1024];
  uint16_t wcls[FW_MAX_WIN * 1024];   // class of each elementary segment per window
  int64_t span_first[FW_MAX_SPANS], span_dense[FW_MAX_SPANS];
  int64_t ws[32];
  int64_t ioff[FW_MAX_WIN + 1], coff[FW_MAX_WIN + 1];
  int32_t wfirst[FW_MAX_WIN], K[FW_MAX_WIN];
  unsigned long long pages[FW_MAX_WIN];
  unsigned __int128 M[FW_MAX_WIN];
  uint8_t sp0[FW_SP_CAP];       // window 0's self-populating flags, prefetched with the intervals
  int32_t nu, R, nu2;
};

// Bitonic sort of the first n triples (n a power of two <= 1024), one
// (hi, lo, payload) triple per thread, ordered lexicographically; on return
// thread t < n holds the triple of rank t.  Triples must be distinct (the
// payload is a unique index) and threads count..n-1 must hold padding that
// sorts last.  Strides < 32 use shuffles; wider ones exchange through shared
// memory (every thread reaches the barriers; only t < max(n, 32) computes).
constexpr int FW_RANK_SORT_MAX = 128;

// Small inputs (n <= FW_RANK_SORT_MAX): each thread counts the keys below its
// own (ties broken by payload, else by thread index) with independent
// broadcast shared loads, then stores itself at that rank -- three barriers
// instead of the network's log^2 stages of dependent exchanges.
template <bool HI, bool PAY>
__device__ __forceinline__ void fw_rank_sortT(uint64_t& hi, uint64_t& lo, int32_t& v, FwSmem& s, int n) {
  const int t = threadIdx.x;
  __syncthreads();   // callers' earlier uses of the exchange buffers are done
  if (t < n) { if (HI) s.xk[t] = hi; s.xk2[t] = lo; if (PAY) s.xv[t] = v; }
  __syncthreads();
  if (t < n) {
    int r = 0;
    const int32_t me = PAY ? v : t;
    // every operand loaded unconditionally and combined with bitwise ops: a
    // short-circuit chain compiles to dependent load-compare-branch steps
#pragma unroll 8
    for (int i = 0; i < n; ++i) {
      const uint64_t ol = s.xk2[i];
      const uint64_t oh = HI ? s.xk[i] : 0;
      const int32_t ov = PAY ? s.xv[i] : i;
      const bool lt = (ol < lo) | ((ol == lo) & (ov < me));
      const bool less = HI ? ((oh < hi) | ((oh == hi) & lt)) : lt;
      r += (int)less;
    }
    if (HI) s.yk[r] = hi;
    s.yk2[r] = lo;
    if (PAY) s.yv[r] = v;
  }
  __syncthreads();
  if (t < n) { if (HI) hi = s.yk[t]; lo = s.yk2[t]; if (PAY) v = s.yv[t]; }
  __syncthreads();   // the reads above, before callers reuse the buffers
}

template <bool HI, bool PAY>
__device__ __forceinline__ void fw_sortT(uint64_t& hi, uint64_t& lo, int32_t& v, FwSmem& s, int n) {
  if (n <= FW_RANK_SORT_MAX) { fw_rank_sortT<HI, PAY>(hi, lo, v, s, n); return; }
  const int t = threadIdx.x;
  const bool act = t < (n < 32 ? 32 : n);
  int buf = 0;   // wide stages alternate exchange buffers, so one barrier each suffices
  if (n > 32) __syncthreads();   // callers' earlier uses of the exchange buffers are done
  for (int kk = 2; kk <= n; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      uint64_t ph = 0, pl = 0; int32_t pv = 0;
      if (j >= 32) {
        uint64_t* bk = buf ? s.yk : s.xk;
        uint64_t* bk2 = buf ? s.yk2 : s.xk2;
        int32_t* bv = buf ? s.yv : s.xv;
        buf ^= 1;
        if (act) { if (HI) bk[t] = hi; bk2[t] = lo; if (PAY) bv[t] = v; }
        __syncthreads();
        if (act) { if (HI) ph = bk[t ^ j]; pl = bk2[t ^ j]; if (PAY) pv = bv[t ^ j]; }
      } else if (act) {
        if (HI) ph = __shfl_xor_sync(0xffffffffu, hi, j);
        pl = __shfl_xor_sync(0xffffffffu, lo, j);
        if (PAY) pv = __shfl_xor_sync(0xffffffffu, v, j);
      }
      if (act) {
        const bool up = (t & kk) == 0, lower = (t & j) == 0;
        bool less;
        if (HI) less = ph < hi || (ph == hi && (pl < lo || (PAY && pl == lo && pv < v)));
        else less = pl < lo || (PAY && pl == lo && pv < v);
        if (lower == up ? less : !less) { if (HI) hi = ph; lo = pl; if (PAY) v = pv; }
      }
    }
  }
  if (n > 32) __syncthreads();   // last wide stage's reads, before callers reuse the buffers
}

// (hi, lo, payload) triples, lexicographic; payloads unique
__device__ __forceinline__ void fw_sort2(uint64_t& hi, uint64_t& lo, int32_t& v, FwSmem& s, int n) {
  fw_sortT<true, true>(hi, lo, v, s, n);
}

// plain 64-bit keys (duplicates allowed)
__device__ __forceinline__ void fw_sort(uint64_t& k, FwSmem& s, int n) {
  uint64_t z = 0;
  int32_t v = 0;
  fw_sortT<false, false>(z, k, v, s, n);
}

__device__ __forceinline__ int fw_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

__device__ __forceinline__ int32_t fw_lb(const uint64_t* a, int32_t n, uint64_t x) {
  int32_t lo = 0, hi = n;
  while (lo < hi) { int32_t mid = (lo + hi) >> 1; if (a[mid] < x) lo = mid + 1; else hi = mid; }
  return lo;
}

__global__ void __launch_bounds__(1024, 1) k_windows_fused(FusedWinParams P) {
#ifdef MSG_MC_PHASE_TS
  unsigned long long fw_t0 = 0;
#endif
  FWTS(0);
  extern __shared__ __align__(16) unsigned char fw_raw[];
  FwSmem& s = *reinterpret_cast<FwSmem*>(fw_raw);
  const int t = threadIdx.x;
  const int W = P.nwin;
  if (t == 0) {
    s.ioff[0] = 0; s.coff[0] = 0;
    for (int w = 0; w < W; ++w) {
      s.ioff[w + 1] = s.ioff[w] + (P.wd[w].pool_hi - P.wd[w].pool_lo);
      s.coff[w + 1] = s.coff[w] + (P.wd[w].c1 - P.wd[w].c0);
    }
  }
  if (t < FW_MAX_WIN) { s.wfirst[t] = 0x7fffffff; s.K[t] = 0; s.pages[t] = 0; }
  __syncthreads();
  const int32_t N = (int32_t)s.ioff[W];
  const int64_t NC = s.coff[W];
  FWTS(1);
  // ---- every global input in one round: spans, intervals and their
  // commands, window 0's self-populating flags (independent loads)
  for (int i = t; i < P.nspans; i += blockDim.x) { s.span_first[i] = P.span_first[i]; s.span_dense[i] = P.span_dense[i]; }
  const int32_t ncw0 = W > 0 ? P.wd[0].c1 - P.wd[0].c0 : 0;
  if (P.R.nr && ncw0 <= FW_SP_CAP)
    for (int i = t; i < ncw0; i += blockDim.x) s.sp0[i] = P.wd[0].selfpop[P.wd[0].c0 + i];
  for (int64_t k = t; k < NC; k += blockDim.x) {
    int w = 0;
    while (k >= s.coff[w + 1]) ++w;
    const WinDesc& D = P.wd[w];
    int32_t c = D.c0 + (int32_t)(k - s.coff[w]);
    int64_t j0 = D.cmd_off[c], j1 = D.cmd_off[c + 1];
    for (int64_t j = j0; j < j1; ++j) s.icmd[s.ioff[w] + (j - D.pool_lo)] = c;
  }
  if (t < N) {
    int w = 0;
    while (t >= s.ioff[w + 1]) ++w;
    const Iv v = P.wd[w].pool[P.wd[w].pool_lo + (t - s.ioff[w])];
    s.ia[t] = v.a; s.ib[t] = v.b; s.iw[t] = w;
  }
  __syncthreads();
  FWTS(2);
  // ---- unique window-tagged endpoints
  {
    uint64_t k = ~0ull;
    if (t < 2 * N) {
      int i = t >> 1;
      k = ((uint64_t)s.iw[i] << 48) | (uint64_t)((t & 1) ? s.ib[i] : s.ia[i]);
    }
    fw_sort(k, s, fw_pow2(2 * N));
    s.xk[t] = k;
    __syncthreads();
    bool f = t < 2 * N && (t == 0 || s.xk[t - 1] != k);
    int64_t tot;
    int64_t pos = block_scan_excl_i64(f ? 1 : 0, s.ws, &tot);
    if (f) s.E[pos] = k;
    if (t == 0) s.nu = (int32_t)tot;
  }
  s.L[t] = kNone;
  s.isb[t] = 0;
  __syncthreads();
  const int32_t nu = s.nu;
  FWTS(3);
  // ---- first-access label per elementary segment (memman.py:187-193)
  {
    int4* span4 = reinterpret_cast<int4*>(s.yk);   // (first segment, end segment, command) per interval
    if (t < N) {
      uint64_t tag = (uint64_t)s.iw[t] << 48;
      int32_t s0 = fw_lb(s.E, nu, tag | (uint64_t)s.ia[t]), s1 = fw_lb(s.E, nu, tag | (uint64_t)s.ib[t]);
      if (N <= FW_LAB_SCAN) span4[t] = make_int4(s0, s1, s.icmd[t], 0);
      else for (int32_t k = s0; k < s1; ++k) atomicMin(&s.L[k], s.icmd[t]);
    }
    if (N <= FW_LAB_SCAN) {
      // few intervals: each segment takes the min over the intervals covering
      // it (broadcast loads), instead of one thread walking a long interval
      __syncthreads();
      if (t < nu - 1) {
        int32_t m = kNone;
#pragma unroll 4
        for (int i = 0; i < N; ++i) {
          const int4 q = span4[i];
          m = (t >= q.x && t < q.y && q.z < m) ? q.z : m;
        }
        s.L[t] = m;
      }
    }
  }
  __syncthreads();
  FWTS(4);
  // ---- maximal runs of one label (consecutive covered segments share a window)
  {
    const int32_t k = t;
    const bool in = k < nu - 1 && s.L[k] != kNone;
    const bool st = in && (k == 0 || s.L[k - 1] != s.L[k]);
    const bool en = in && (k == nu - 2 || s.L[k + 1] != s.L[k]);
    int64_t tot;
    int64_t ex = block_scan_excl_i64(st ? 1 : 0, s.ws, &tot);
    int32_t rid = (int32_t)(ex + (st ? 1 : 0)) - 1;
    if (st) { s.ra[rid] = (int64_t)(s.E[k] & FW_POS); s.rl[rid] = s.L[k]; s.rsk[rid] = k; }
    if (en) { s.rb[rid] = (int64_t)(s.E[k + 1] & FW_POS); s.rek[rid] = k + 1; }
    if (t == 0) s.R = (int32_t)tot;
  }
  __syncthreads();
  const int32_t R = s.R;
  FWTS(5);
  // ---- runs in first-access order per window: (window, label, start)
  {
    uint64_t k = ~0ull;
    if (t < R) k = ((s.E[s.rsk[t]] >> 48) << 52) | ((uint64_t)(uint32_t)s.rl[t] << 20) | (uint64_t)t;
    fw_sort(k, s, fw_pow2(R));
    if (t < R) {
      int w = (int)(k >> 52);
      atomicMin(&s.wfirst[w], t);
      atomicAdd(&s.K[w], 1);
    }
    __syncthreads();
    if (t < R) {
      int w = (int)(k >> 52);
      int32_t rid = (int32_t)(k & 0xfffff);
      int32_t r = t - s.wfirst[w];
      int64_t a = s.ra[rid], b = s.rb[rid];
      s.sa[t] = a; s.sb[t] = b; s.sl[t] = s.rl[rid]; s.sw[t] = w; s.scls[t] = s.K[w] - r;
      int64_t o = P.wd[w].scratch + r;
      P.out.run_a[o] = a; P.out.run_b[o] = b; P.out.run_lab[o] = s.rl[rid];
      atomicAdd(&s.pages[w], (unsigned long long)(b - a));
      s.isb[s.rsk[rid]] = 1;   // run boundaries, marked on the endpoint list
      s.isb[s.rek[rid]] = 1;
    }
  }
  __syncthreads();
  if (t < W) {
    P.out.nruns[t] = s.K[t];
    P.out.pages[t] = (int64_t)s.pages[t];
    P.out.run_base[t] = P.wd[t].scratch;
  }
  auto dense_of = [&](int64_t a) -> int64_t {
    int32_t lo = 0, hi = P.nspans;
    while (lo < hi) { int32_t mid = (lo + hi) >> 1; if (s.span_first[mid] <= a) lo = mid + 1; else hi = mid; }
    return s.span_dense[lo - 1] + (a - s.span_first[lo - 1]);
  };
  FWTS(6);
  // ---- window 0 demand runs: not self-populating, dense, first-access order
  if (P.R.nr) {
    const int32_t K0 = W > 0 ? s.K[0] : 0;
    const int32_t r = t;   // window 0 runs are ranks [0, K0)
    bool keep = false;
    int64_t dlo = 0, dlen = 0;
    if (r < K0) {
      const int32_t c = s.sl[r];
      keep = !(ncw0 <= FW_SP_CAP ? s.sp0[c - P.wd[0].c0] : P.wd[0].selfpop[c]);
      dlo = dense_of(s.sa[r]);
      dlen = s.sb[r] - s.sa[r];
    }
    int64_t words = keep ? ((dlo + dlen + 31) >> 5) - (dlo >> 5) : 0;
    int64_t tot, utot;
    int64_t ex = block_scan_excl_i64(keep ? 1 : 0, s.ws, &tot);
    int64_t uex = block_scan_excl_i64(words, s.ws, &utot);
    if (keep) {
      P.R.lo[ex] = dlo; P.R.len[ex] = dlen; P.R.tag[ex] = s.sl[r] - P.wd[0].c0; P.R.uoff[ex] = uex;
    }
    if (t == 0) { *P.R.nr = tot; P.R.uoff[tot] = utot; }
  }
  FWTS(7);
  // ---- cross-window class table: elementary segments of all run boundaries
  {
    uint64_t k = ~0ull;
    if (t < nu && s.isb[t]) k = s.E[t] & FW_POS;
    fw_sort(k, s, fw_pow2(nu));
    FWTS(8);
    s.xk[t] = k;
    __syncthreads();
    bool f = k != ~0ull && (t == 0 || s.xk[t - 1] != k);
    int64_t tot;
    int64_t pos = block_scan_excl_i64(f ? 1 : 0, s.ws, &tot);
    if (f) s.E2[pos] = k;
    if (t == 0) {
      s.nu2 = (int32_t)tot;
      unsigned __int128 m = 1;
      for (int w = W - 1; w >= 0; --w) { s.M[w] = m; m *= (unsigned __int128)(s.K[w] + 1); }
    }
    s.skey[t] = 0;
  }
  __syncthreads();
  const int32_t nu2 = s.nu2;
  FWTS(9);
  // paint each window's class over the elementary segments (all windows in
  // parallel: runs of one window are disjoint), then fold to the mixed radix
  for (int i = t; i < W * nu2; i += blockDim.x) s.wcls[(i / nu2) * 1024 + i % nu2] = 0;
  __syncthreads();
  if (t < R) {
    int32_t s0 = fw_lb(s.E2, nu2, (uint64_t)s.sa[t]), s1 = fw_lb(s.E2, nu2, (uint64_t)s.sb[t]);
    uint16_t c = (uint16_t)s.scls[t];
    for (int32_t k = s0; k < s1; ++k) s.wcls[s.sw[t] * 1024 + k] = c;
  }
  __syncthreads();
  FWTS(10);
  if (t < nu2 - 1) {
    unsigned __int128 key = 0;
    for (int w = 0; w < W; ++w) key += (unsigned __int128)s.wcls[w * 1024 + t] * s.M[w];
    s.skey[t] = key;
  }
  __syncthreads();
  FWTS(11);
  // dense rank of the distinct tuples over covered segments
  {
    const int32_t k = t;
    const bool cov = k < nu2 - 1 && s.skey[k] != 0;
    uint64_t hi = cov ? (uint64_t)(s.skey[k] >> 64) : ~0ull;   // valid tuples are < 2^97
    uint64_t lo = cov ? (uint64_t)s.skey[k] : ~0ull;
    int32_t v = k;
    const int ns = fw_pow2(nu2 > 1 ? nu2 - 1 : 1);
    if (__syncthreads_or(cov && hi != 0)) fw_sort2(hi, lo, v, s, ns);
    else fw_sortT<false, true>(hi, lo, v, s, ns);
    FWTS(12);
    const bool valid = t < ns && v < nu2 - 1 && s.skey[v] != 0;
    if (valid) { hi = (uint64_t)(s.skey[v] >> 64); lo = (uint64_t)s.skey[v]; }
    s.xk[t] = hi; s.xk2[t] = lo;
    __syncthreads();
    const bool first = valid && (t == 0 || s.xk[t - 1] != hi || s.xk2[t - 1] != lo);
    int64_t tot;
    int64_t ex = block_scan_excl_i64(first ? 1 : 0, s.ws, &tot);
    if (valid) s.cls_of[v] = (int32_t)(ex + (first ? 1 : 0));
    if (t == 0) *P.ncls_out = tot;
  }
  __syncthreads();
  FWTS(13);
  // ---- covered segments in position order, dense
  {
    const int32_t k = t;
    const bool cov = k < nu2 - 1 && s.skey[k] != 0;
    int64_t tot;
    int64_t ci = block_scan_excl_i64(cov ? 1 : 0, s.ws, &tot);
    if (cov) {
      int64_t a = (int64_t)s.E2[k], b = (int64_t)s.E2[k + 1];
      int64_t d = dense_of(a);
      P.seg_lo[ci] = d; P.seg_hi[ci] = d + (b - a); P.seg_cls[ci] = s.cls_of[k];
    }
    if (t == 0) *P.nseg_out = tot;
  }
  FWTS(15);
#ifdef MSG_MC_PHASE_TS
  if (t == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));
    *(volatile unsigned long long*)&g_fw_end = t_;
  }
#endif
}

static void win_kernels_init(Ctx& c) {
  if (c.win_init) return;
  MSG_CUDA(cudaFuncSetAttribute(k_window_runs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWinSmem));
  MSG_CUDA(cudaFuncSetAttribute(k_window_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWinSmem));
  MSG_CUDA(cudaFuncSetAttribute(k_window_combine_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWideSmem));
  MSG_CUDA(cudaFuncSetAttribute(k_windows_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FwSmem)));
  c.win_init = true;
}

// ---------------------------------------------------------------------------
// Demand runs of window 0 vs the resident bitmap (engine.py:310-313,
// memman.py:284-291, engine.py:350-355).

__device__ __forceinline__ bool is_res(const uint32_t* bits, int64_t p) {
  return (bits[p >> 5] >> (p & 31)) & 1u;
}

// count non-resident pages of dense ranges [lo, lo+len): one warp per range
__device__ int64_t warp_count_nonres(const uint32_t* bits, int64_t lo, int64_t len) {
  int lane = threadIdx.x & 31;
  int64_t hi = lo + len, acc = 0;
  int64_t w0 = lo >> 5, w1 = (hi + 31) >> 5;
  for (int64_t w = w0 + lane; w < w1; w += 32) {
    uint32_t word = ~bits[w];
    int64_t p0 = w << 5;
    if (p0 < lo) word &= ~0u << (lo - p0);
    if (p0 + 32 > hi) word &= (hi - p0) >= 32 ? ~0u : ((1u << (hi - p0)) - 1u);
    acc += __popc(word);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

struct DemandParams {
  const int64_t* run_a; const int64_t* run_b; const int32_t* run_lab; int64_t run_base; const int64_t* nruns;
  const uint8_t* selfpop; int32_t c0;
  const int64_t* span_first; const int64_t* span_n; const int64_t* span_dense; int32_t nspans;
  RangeOut R;            // compacted demand runs (dense), tag = first-access command - c0
};

// Window-0 runs whose first-access command is not self-populating, as a
// RangeSet in first-access order (memman.py:189-193).  Single block.
__global__ void __launch_bounds__(1024, 1) k_demand_collect(DemandParams P) {
  int64_t nr = P.nruns[0];
  __shared__ int64_t ws[32];
  __shared__ int64_t carry, ucarry;
  if (threadIdx.x == 0) { carry = 0; ucarry = 0; }
  __syncthreads();
  for (int64_t base = 0; base < nr; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    bool keep = false;
    int64_t r = P.run_base + i;
    int64_t dlo = 0, dlen = 0;
    if (i < nr) {
      keep = !P.selfpop[P.run_lab[r]];
      int64_t a = P.run_a[r];
      int lo = 0, hi = P.nspans;
      while (lo < hi) { int mid = (lo + hi) >> 1; if (P.span_first[mid] <= a) lo = mid + 1; else hi = mid; }
      int s = lo - 1;
      dlo = P.span_dense[s] + (a - P.span_first[s]);
      dlen = P.run_b[r] - a;
    }
    int64_t words = keep ? ((dlo + dlen + 31) >> 5) - (dlo >> 5) : 0;
    int64_t tot, utot;
    int64_t ex = block_scan_excl_i64(keep ? 1 : 0, ws, &tot);
    int64_t uex = block_scan_excl_i64(words, ws, &utot);
    if (keep) {
      int64_t o = carry + ex;
      P.R.lo[o] = dlo;
      P.R.len[o] = dlen;
      P.R.tag[o] = P.run_lab[r] - P.c0;
      P.R.uoff[o] = ucarry + uex;
    }
    __syncthreads();
    if (threadIdx.x == 0) { carry += tot; ucarry += utot; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { *P.R.nr = carry; P.R.uoff[carry] = ucarry; }
}

// ---------------------------------------------------------------------------
// Multisplit of the eviction list (the reorder / madvise / remove kernel).

constexpr int MS_THREADS = 256;
constexpr int MS_WARPS = MS_THREADS / 32;
constexpr int MS_CHUNK = 128;                             // entries per warp step (4 per lane, striped)
constexpr int MS_CHUNKS = 4;                              // warp steps per tile
constexpr int MS_ITEMS = MS_CHUNKS * 4;                   // entries per thread per tile
constexpr int MS_TILE = MS_WARPS * MS_CHUNKS * MS_CHUNK;  // 4096 entries
constexpr int MS_SMEM_SEGS = 2048;
constexpr int MS_CTAS_PER_SM = 4;
constexpr int MS_MAX_PASSES = 4;

struct SegTab {
  const int64_t* lo; const int64_t* hi; const int32_t* cls; const int64_t* n;
  int64_t cap = 0;   // allocated entries of lo/hi/cls when known (0: unknown)
};

// Segment table staged in shared memory as 32-bit dense bounds (dense ids
// are < 2^31), the per-warp digit counters of the ranking, and the per-CTA
// digit bookkeeping of the look-back.
struct MsSmem {
  int32_t lo[MS_SMEM_SEGS];
  int32_t hi[MS_SMEM_SEGS];
  int32_t cls[MS_SMEM_SEGS];
  int32_t cnt[MS_WARPS][256];   // per-warp digit counts, then exclusive warp offsets
  int64_t gbase[256];           // first output index of each digit (all tiles)
  int64_t base[256];            // gbase + this tile's look-back prefix
  int32_t agg[256];             // this tile's digit counts
  int32_t act[256];             // digits present anywhere in the list
  int32_t nact;
  int32_t tile;
};

struct SegView {
  const int32_t* lo32; const int32_t* hi32; const int32_t* cls32;   // smem copy (n <= MS_SMEM_SEGS)
  const int64_t* lo; const int64_t* hi; const int32_t* cls;         // global fallback
  int32_t n, steps;                                                 // steps = log2(pow2 >= n)
  bool small;
};

// The interval [ilo, ihi) around page p on which the class is constant (a
// segment, or the gap between two), and that class.  Branchless binary search
// with a fixed trip count.
struct Span { int32_t lo, hi, cls; };

__device__ __forceinline__ Span seg_find(const SegView& S, int32_t p) {
  int32_t pos = 0;
  Span r;
  if (S.small) {
    for (int32_t step = 1 << S.steps; step > 0; step >>= 1) {
      int32_t q = pos + step;
      if (q <= S.n && S.lo32[q - 1] <= p) pos = q;
    }
    if (pos > 0 && p < S.hi32[pos - 1]) { r.lo = S.lo32[pos - 1]; r.hi = S.hi32[pos - 1]; r.cls = S.cls32[pos - 1]; }
    else { r.lo = pos > 0 ? S.hi32[pos - 1] : INT32_MIN; r.hi = pos < S.n ? S.lo32[pos] : INT32_MAX; r.cls = 0; }
    return r;
  }
  for (int32_t step = 1 << S.steps; step > 0; step >>= 1) {
    int32_t q = pos + step;
    if (q <= S.n && S.lo[q - 1] <= (int64_t)p) pos = q;
  }
  if (pos > 0 && (int64_t)p < S.hi[pos - 1]) {
    r.lo = (int32_t)S.lo[pos - 1]; r.hi = (int32_t)S.hi[pos - 1]; r.cls = S.cls[pos - 1];
  } else {
    r.lo = pos > 0 ? (int32_t)S.hi[pos - 1] : INT32_MIN;
    r.hi = pos < S.n ? (int32_t)S.lo[pos] : INT32_MAX;
    r.cls = 0;
  }
  return r;
}

__device__ SegView ms_load_table(const SegTab& T, MsSmem& sm) {
  SegView S;
  int64_t nn = *T.n;
  S.n = (int32_t)nn;
  int steps = 0;
  while ((1ll << steps) < nn) ++steps;
  S.steps = steps;
  S.small = nn <= MS_SMEM_SEGS;
  S.lo = T.lo; S.hi = T.hi; S.cls = T.cls;
  S.lo32 = sm.lo; S.hi32 = sm.hi; S.cls32 = sm.cls;
  if (S.small)
    for (int64_t i = threadIdx.x; i < nn; i += blockDim.x) {
      sm.lo[i] = (int32_t)T.lo[i]; sm.hi[i] = (int32_t)T.hi[i]; sm.cls[i] = T.cls[i];
    }
  return S;
}

// Digit totals of every pass without reading the list: the list holds
// exactly the resident pages, so the entries of class c are the resident
// pages of c's segments (popcount of the resident bitmap over the segment);
// everything else is class 0.  One CTA per segment (grid-stride).
// tot[p*257 + d] for pass p, tot[p*257 + 256] = all advised entries.
__global__ void k_ms_digit_totals(SegTab T, const uint32_t* __restrict__ bits, int passes,
                                  unsigned long long* tot) {
  __shared__ unsigned long long red[8];
  int64_t ns = *T.n;
  for (int64_t s = blockIdx.x; s < ns; s += gridDim.x) {
    int64_t lo = T.lo[s], hi = T.hi[s];
    unsigned long long acc = 0;
    for (int64_t w = (lo >> 5) + threadIdx.x; w < (hi + 31) >> 5; w += blockDim.x) {
      int64_t p0 = w << 5;
      uint32_t m = ~0u;
      if (p0 < lo) m &= ~0u << (lo - p0);
      if (p0 + 32 > hi) m &= (hi - p0) >= 32 ? ~0u : ((1u << (hi - p0)) - 1u);
      acc += __popc(__ldg(bits + w) & m);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < passes) {
      unsigned long long t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      if (t) {
        int p = threadIdx.x;
        atomicAdd(&tot[p * 257 + ((T.cls[s] >> (8 * p)) & 255)], t);
        atomicAdd(&tot[p * 257 + 256], t);
      }
    }
    __syncthreads();
  }
}

// Single-pass stable multisplit with decoupled look-back, persistent CTAs.
//
// Tiles of 4096 list entries are claimed in order through an atomic counter.
// A warp owns 4 consecutive 128-entry chunks of its tile and reads each with
// four coalesced 128-byte loads (entry lane + 32k).  The eviction list is
// made of long runs of consecutive page ids (pages are appended run by run,
// and every multisplit keeps relative order), so a chunk that is one run
// inside one constant-class interval is classified with one check against
// the warp's cached interval — no search, no per-entry work — and later
// written back as four coalesced stores of computed ids.  Anything else takes
// the per-entry path (ranked with match_any in array order, so the split is
// stable).
//
// Look-back: status[d * stride + tile] = epoch (16) | flag (2: 1 aggregate,
// 2 inclusive) | count (46).  Only digits present in the list take part (the
// digit totals are known up front); one warp resolves a digit 32 predecessor
// tiles at a time with one coalesced load.  The epoch makes stale words from
// earlier passes invisible without clearing.
struct Onesweep {
  unsigned long long* status;
  int64_t stride;               // tiles per digit row
  int32_t* tile_ctr;
  const unsigned long long* tot;
  uint32_t epoch;
};

__device__ __forceinline__ unsigned long long os_pack(uint32_t epoch, uint32_t flag, unsigned long long v) {
  return ((unsigned long long)epoch << 48) | ((unsigned long long)flag << 46) | v;
}

__global__ void __launch_bounds__(MS_THREADS, MS_CTAS_PER_SM)
k_ms_onesweep(const int32_t* __restrict__ src, int64_t n, SegTab T, int shift, int32_t* __restrict__ dst,
              Onesweep O) {
  __shared__ MsSmem sm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lt = (1u << lane) - 1u;
  SegView S = ms_load_table(T, sm);
  // digit totals -> global digit bases and the list of present digits
  {
    const int d = tid;
    unsigned long long td = O.tot[d] + (d == 0 ? (unsigned long long)n - O.tot[256] : 0ull);
    unsigned long long x = td;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t present = __ballot_sync(0xffffffffu, td != 0);
    if (lane == 31) { sm.gbase[warp] = (int64_t)x; sm.agg[warp] = __popc(present); }
    __syncthreads();
    int64_t wp = 0;
    int32_t ap = 0;
    for (int w = 0; w < warp; ++w) { wp += sm.gbase[w]; ap += sm.agg[w]; }
    __syncthreads();
    sm.gbase[d] = wp + (int64_t)(x - td);
    if (td) sm.act[ap + __popc(present & lt)] = d;
    if (d == MS_THREADS - 1) sm.nact = ap + __popc(present);
  }
  const int64_t ntiles = (n + MS_TILE - 1) / MS_TILE;
  int32_t c_lo = 1, c_hi = 0, c_d = 0;   // warp's cached constant-class interval
  for (;;) {
    if (tid == 0) sm.tile = atomicAdd(O.tile_ctr, 1);
    for (int i = lane; i < 256; i += 32) sm.cnt[warp][i] = 0;
    __syncthreads();
    const int64_t tile = sm.tile;
    if (tile >= ntiles) break;
    const int64_t wbase = tile * MS_TILE + warp * (MS_CHUNKS * MS_CHUNK);
    // ---- phase 1: load, classify and rank (per warp, in array order)
    int32_t val[MS_ITEMS];
    int32_t dig[MS_ITEMS];   // digit | rank-within-warp << 9; digit 256 = past the end
    uint32_t fast = 0;       // bit j: chunk j is one run of one digit (val[4j] = first id)
#pragma unroll
    for (int j = 0; j < MS_CHUNKS; ++j) {
      const int64_t cb = wbase + j * MS_CHUNK;
      int32_t x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int64_t i = cb + 32 * k + lane;
        x[k] = i < n ? __ldg(src + i) : 0;
      }
      const int32_t v0 = __shfl_sync(0xffffffffu, x[0], 0);
      bool ok = cb + MS_CHUNK <= n;
#pragma unroll
      for (int k = 0; k < 4; ++k) ok = ok && x[k] == v0 + 32 * k + lane;
      int d = -1;
      if (__all_sync(0xffffffffu, ok)) {
        if (!(v0 >= c_lo && v0 + (MS_CHUNK - 1) < c_hi)) {
          Span s = seg_find(S, v0);
          c_lo = s.lo; c_hi = s.hi; c_d = (s.cls >> shift) & 255;
        }
        if (v0 + (MS_CHUNK - 1) < c_hi) d = c_d;
      }
      if (d >= 0) {
        fast |= 1u << j;
        int32_t before = sm.cnt[warp][d];
        __syncwarp();
        if (lane == 0) sm.cnt[warp][d] = before + MS_CHUNK;
        __syncwarp();
        val[4 * j] = v0;
        dig[4 * j] = d | (before << 9);
        continue;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int dk = 256;
        if (cb + 32 * k + lane < n) {
          if (x[k] >= c_lo && x[k] < c_hi) dk = c_d;
          else dk = (seg_find(S, x[k]).cls >> shift) & 255;
        }
        uint32_t peers = __match_any_sync(0xffffffffu, dk);
        int32_t before = dk < 256 ? sm.cnt[warp][dk] : 0;
        __syncwarp();
        if (dk < 256 && lane == __ffs(peers) - 1) sm.cnt[warp][dk] = before + __popc(peers);
        __syncwarp();
        val[4 * j + k] = x[k];
        dig[4 * j + k] = dk | ((before + __popc(peers & lt)) << 9);
      }
    }
    __syncthreads();
    // ---- tile aggregate per digit; exclusive warp offsets; publish
    {
      const int d = tid;
      int32_t acc = 0;
#pragma unroll
      for (int w = 0; w < MS_WARPS; ++w) { int32_t t = sm.cnt[w][d]; sm.cnt[w][d] = acc; acc += t; }
      sm.agg[d] = acc;
      if (O.tot[d] + (d == 0 ? (unsigned long long)n - O.tot[256] : 0ull))
        atomicExch(O.status + d * O.stride + tile, os_pack(O.epoch, tile == 0 ? 2u : 1u, (unsigned long long)acc));
    }
    __syncthreads();
    // ---- decoupled look-back: one warp per present digit, 32 tiles per step
    for (int a = warp; a < sm.nact; a += MS_WARPS) {
      const int d = sm.act[a];
      const unsigned long long* row = O.status + d * O.stride;
      unsigned long long prefix = 0;
      int64_t j = tile - 1;
      while (j >= 0) {
        int64_t t = j - lane;
        unsigned long long w = t >= 0 ? *reinterpret_cast<const volatile unsigned long long*>(row + t)
                                      : os_pack(O.epoch, 2u, 0ull);
        bool ready = (uint32_t)(w >> 48) == O.epoch && ((w >> 46) & 3) != 0;
        uint32_t nr = __ballot_sync(0xffffffffu, !ready);
        uint32_t inc = __ballot_sync(0xffffffffu, ready && ((w >> 46) & 3) == 2);
        int lim = nr ? __ffs(nr) - 1 : 32;      // lanes [0, lim) are ready
        int fi = inc ? __ffs(inc) - 1 : 32;     // nearest inclusive
        int take = fi < lim ? fi + 1 : lim;
        unsigned long long v = lane < take ? (w & ((1ull << 46) - 1)) : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        prefix += v;
        if (fi < lim) break;
        j -= take;
      }
      if (lane == 0) {
        if (tile > 0) atomicExch(O.status + d * O.stride + tile, os_pack(O.epoch, 2u, prefix + sm.agg[d]));
        sm.base[d] = sm.gbase[d] + (int64_t)prefix;
      }
    }
    __syncthreads();
    // ---- scatter
#pragma unroll
    for (int j = 0; j < MS_CHUNKS; ++j) {
      if (fast & (1u << j)) {
        const int d = dig[4 * j] & 511;
        int64_t p = sm.base[d] + sm.cnt[warp][d] + (dig[4 * j] >> 9) + lane;
        const int32_t v = val[4 * j] + lane;
#pragma unroll
        for (int k = 0; k < 4; ++k) dst[p + 32 * k] = v + 32 * k;
        continue;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int dd = dig[4 * j + k] & 511, r = dig[4 * j + k] >> 9;
        if (dd < 256) dst[sm.base[dd] + sm.cnt[warp][dd] + r] = val[4 * j + k];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// On-chip multisplit (one cooperative launch for all digit passes; per pass
// one grid barrier, plus one between passes).
//
// One 1024-thread CTA per SM owns a contiguous slice of the list, staged in
// shared memory by one TMA bulk copy (slices are cut on 16-byte boundaries of
// the underlying buffer, so every 512-entry block is 16-byte aligned in both
// global and shared memory).  Each of the 32 warps owns a contiguous run of
// blocks.  The eviction list is made of long runs of consecutive page ids
// (pages are appended run by run, and every multisplit keeps relative
// order), so phase 1 checks a whole block with four 16-byte shared loads per
// lane: a block that is one run inside one constant-class interval is
// recorded as (first id, digit) and never looked at again.  Other blocks are
// split into 128-entry chunks (run chunk or per-entry, ranked with match_any
// in array order, so the split is stable).  The CTA's digit histogram goes
// to global memory (totals by atomics); after the grid barrier each CTA sums
// the rows of the CTAs before it, so there is no look-back and no separate
// totals kernel.  Phase 3 replays the blocks in order: run blocks are written
// as computed ids with aligned 16-byte stores.  Traffic: 4 B read + 4 B
// written per entry per pass.  A second pass (>= 256 classes) re-stages the
// first pass's output after a grid barrier (async-proxy fence before the
// TMA read of data the generic proxy wrote).
constexpr int MC_THREADS = 1024;
constexpr int MC_WARPS = MC_THREADS / 32;
constexpr int MC_BLOCK = 512;                       // entries per fast block (16 per lane)
constexpr int MC_SMEM = 224 * 1024;
constexpr int MC_PIECES = 4;                // TMA pieces of a slice, one mbarrier each
constexpr int MC_FIXED = MC_WARPS * 256 * 4 + 256 * 8 + 16 * 256 * 4 + 8 * (8 + MC_PIECES) + 16;
constexpr int MC_TCAP_MIN = MS_SMEM_SEGS;   // class-table segments always kept on chip
constexpr int MC_TCAP_MAX = 16384;          // more when the staged slice leaves room (fragmented lists)
// ms_coop_body's int32 scratch `red` ([16][256] words): phase-2 slots, then
// the per-entry chunk queue.  A chunk that is not one run in one
// constant-class interval is queued (up to MC_QCAP per CTA) instead of being
// classified by the warp that owns it: after phase 1 every warp takes queued
// chunks round-robin, stores each entry's digit (one byte) and adds the
// counts to the owner's row, so the slowest warp no longer carries its
// blocks' per-entry searches alone; phase 3 reads the stored digits.
constexpr int kRedSlice = 256;    // [256] this slice's digit counts
constexpr int kRedDl = 512;       // [256] digits present in the slice
constexpr int kRedQ = 768;        // [MC_QCAP] queued chunks: chunk index << 5 | owner warp
constexpr int kRedNq = 832;       // queued-chunk count (may pass MC_QCAP: the rest run inline)
constexpr int kRedNd = 833;       // present-digit count
constexpr int kRedCol = 1024;     // [4][256] column sums (many-digit slices)
constexpr int kRedDig = 2048;     // [MC_QCAP][128] stored digits (bytes)
constexpr int MC_QCAP = 64;

struct McArgs {
  const int32_t* src0;   // pass 0 source, 16-byte aligned: list entry i is src0[i + a]
  int32_t* bufA;         // base of pass 0's source buffer (destination of odd passes)
  int32_t* bufB;         // the other buffer (destination of even passes, source of odd ones)
  int64_t n;             // list entries
  int32_t a;             // pass 0's leading pad entries (0..3)
  SegTab T;
  int32_t* hist;         // [gridDim.x][256] per-CTA digit counts
  int32_t* totb;         // [2][256] digit totals; row par is zero at launch
  int32_t par;
  int32_t* bar;          // grid barrier counter (zero at launch; barrier k waits for (k+1) * grid)
  int64_t E;             // aligned entries per CTA (multiple of MC_BLOCK)
  int32_t vcap;          // entries per CTA kept in shared memory (multiple of MC_BLOCK)
  int32_t nch_cap;       // chunk records per CTA
  int32_t passes;        // digit passes (LSD, 8 bits each), all in this launch
  unsigned long long* t_first;   // globaltimer of the first CTA to start (atomicMin)
  unsigned long long* t_last;    // globaltimer of the last CTA to finish (atomicMax)
  int32_t dbg_id;                // launch ordinal (phase-timing build)
  int32_t tcap;                  // class-table segments staged in shared memory (after the slice cache)
  // device-decided pass count (the async switch path, no host round trip):
  // passes = digits of *ncls_dev, 0 when *missing_dev == 0 and !reorder_always;
  // CTA 0 publishes it to *passes_out
  const int64_t* ncls_dev;
  const int64_t* missing_dev;
  int32_t reorder_always;
  int64_t* passes_out;
  int32_t force_stream;          // test / tuning hook (MSG_MS_STREAM=1): stream even slices that fit
};

// TMA bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBAR_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// cp.async (16-byte global -> shared, L2 only) with per-thread groups
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ int ms_digit(const SegView& S, int32_t x, int32_t c_lo, int32_t c_hi, int c_d, int shift) {
  if (x >= c_lo && x < c_hi) return c_d;
  return (seg_find(S, x).cls >> shift) & 255;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Phase timestamps of k_ms_coop (instrumented build only: `make phase-ts`,
// read by tools/mc_phase_replay.py): per stamp the earliest / latest CTA and
// the sum over CTAs of the time since that CTA's start.
#ifdef MSG_MC_PHASE_TS
__device__ unsigned long long g_mc_min[16], g_mc_max[16], g_mc_sum[16], g_mc_n;
// per-CTA absolute stamps of the last 256 launches: [launch & 255][cta][stamp]
__device__ unsigned long long g_mc_cta[256][160][8];
// per-warp phase-1 profile of the last 64 launches: [launch & 63][cta][warp] =
// (globaltimer ns spent in phase 1 after the warp's first piece wait) << 32 | slow chunks << 16 | blocks
__device__ unsigned long long g_mc_warp[64][160][32];
__device__ __forceinline__ unsigned long long mc_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MCTS(i)                                                                            \
  do {                                                                                     \
    if (threadIdx.x == 0) {                                                                \
      const unsigned long long t_ = mc_now();                                              \
      atomicMin(&g_mc_min[i], t_); atomicMax(&g_mc_max[i], t_); atomicAdd(&g_mc_sum[i], t_ - mc_t0); \
      if (blockIdx.x < 160 && (i) < 8) g_mc_cta[A.dbg_id & 255][blockIdx.x][i] = t_;      \
    }                                                                                      \
  } while (0)
#define MCTS_START const unsigned long long mc_t0 = mc_now(); MCTS(0)
#else
#define MCTS(i) do {} while (0)
#define MCTS_START do {} while (0)
#endif

// The multisplit runs as its own cooperative launch (k_ms_coop) or as a phase
// of the per-switch cooperative kernel (k_switch_coop); nbar counts the grid
// barriers used so far on A.bar.
__device__ __forceinline__ void ms_coop_body(const McArgs& A, unsigned char* mc_raw, int& nbar) {
  MCTS_START;
  if (threadIdx.x == 0) atomicMin(A.t_first, global_ns());   // device-side duration of the multisplit (stats)
  int32_t(*cnt)[256] = reinterpret_cast<int32_t(*)[256]>(mc_raw);
  int64_t* base = reinterpret_cast<int64_t*>(cnt + MC_WARPS);
  int32_t* red = reinterpret_cast<int32_t*>(base + 256);          // [16][256]
  int64_t* misc = reinterpret_cast<int64_t*>(red + 16 * 256);     // [0, 8): warp totals; [8, 12): mbarriers
  int2* info = reinterpret_cast<int2*>(misc + 8 + MC_PIECES);     // chunk records (16-B aligned)
  int32_t* cache = reinterpret_cast<int32_t*>(info + ((A.nch_cap + 1) & ~1));   // 16-B aligned
  // the class table after the slice (+ 4 entries of TMA rounding slack)
  int32_t* lo32 = cache + A.vcap + 4;
  int32_t* hi32 = lo32 + A.tcap;
  int32_t* cls32 = hi32 + A.tcap;
  // the mbarriers live for every pass: they must not share a slot with the
  // phase-2 warp totals.  The staged slice arrives in MC_PIECES block-aligned
  // pieces, one mbarrier each, so a warp starts on its blocks as soon as the
  // piece holding them has landed instead of waiting for the whole slice.
  uint64_t* bar = reinterpret_cast<uint64_t*>(misc + 8);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t cE = (int64_t)blockIdx.x * A.E;                    // aligned index of the slice start
  auto piece_len = [](int32_t m) { return (m + MC_PIECES * MC_BLOCK - 1) / (MC_PIECES * MC_BLOCK) * MC_BLOCK; };
  auto issue = [&](const int32_t* src, int32_t m) {   // thread 0
    const int32_t P4 = piece_len(m);
    for (int k = 0; k < MC_PIECES; ++k) {
      const int32_t lo = k * P4, hi = lo + P4 < m ? lo + P4 : m;
      const int32_t cntk = hi > lo ? hi - lo : 0;
      const uint32_t bytes = (uint32_t)(((int64_t)cntk * 4 + 15) & ~int64_t(15));
      mbar_expect_tx(bar + k, bytes);
      if (cntk > 0) tma_bulk_g2s(cache + lo, src + cE + lo, bytes, bar + k);
    }
  };
  if (tid == 0) {
    // pass 0's slice goes to shared memory first -- before the pass count
    // and the class table are read -- so the copy overlaps those loads.
    // (An earlier phase of the same kernel may have used this shared memory
    // through the generic proxy.)
    asm volatile("fence.proxy.async;" ::: "memory");
    for (int k = 0; k < MC_PIECES; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar + k)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int64_t nA0 = A.n + A.a;
    const int64_t cEnd0 = cE + A.E < nA0 ? cE + A.E : nA0;
    const int64_t len0 = cEnd0 > cE ? cEnd0 - cE : 0;
    issue(A.src0, (int32_t)(len0 <= A.vcap && !A.force_stream ? len0 : 0));   // staged whole or streamed (below)
  }
  // class table -> smem (once for all passes).  When the host knows the
  // table's allocated length, every entry up to it is loaded without waiting
  // for the segment count, so the count's load and the entries' loads are one
  // round trip instead of two (entries past the count are never searched).
  SegView S;
  {
    // (the first kEager entries are loaded before the count arrives; the rest,
    // up to the count, after it: loading the whole allocated capacity staged 4x
    // the table for fragmented windows)
    constexpr int64_t kEager = 2048;
    const int64_t nn = *A.T.n;
    int64_t eager = 0;
    if (A.T.cap > 0) {
      eager = A.T.cap < A.tcap ? A.T.cap : A.tcap;
      eager = eager < kEager ? eager : kEager;
      for (int64_t i = tid; i < eager; i += MC_THREADS) {
        lo32[i] = (int32_t)A.T.lo[i]; hi32[i] = (int32_t)A.T.hi[i]; cls32[i] = A.T.cls[i];
      }
    }
    S.n = (int32_t)nn;
    S.steps = nn > 1 ? 64 - __clzll(nn - 1) : 0;
    S.small = nn <= A.tcap;
    S.lo = A.T.lo; S.hi = A.T.hi; S.cls = A.T.cls;
    S.lo32 = lo32; S.hi32 = hi32; S.cls32 = cls32;
    if (S.small)
      for (int64_t i = eager + tid; i < nn; i += MC_THREADS) {
        lo32[i] = (int32_t)A.T.lo[i]; hi32[i] = (int32_t)A.T.hi[i]; cls32[i] = A.T.cls[i];
      }
  }
  int passes = A.passes;
  if (A.ncls_dev) {
    // (L2 loads: an earlier phase of the same kernel may have written them)
    const bool skip = A.missing_dev && __ldcg(A.missing_dev) == 0 && !A.reorder_always;
    int64_t nc = skip ? 0 : __ldcg(A.ncls_dev);
    passes = 0;
    while (nc > 0) { ++passes; nc >>= 8; }
    if (blockIdx.x == 0 && threadIdx.x == 0) *A.passes_out = passes;
    if (passes == 0) {   // uniform over the grid: no barrier is entered (t_last stays unset)
      // the staged copy is in flight into this CTA's shared memory: let it land first
      if (tid == 0)
        for (int k = 0; k < MC_PIECES; ++k) mbar_wait(bar + k, 0);
      return;
    }
  }
  __syncthreads();   // the initialised mbarrier and the class table, before any use
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = 8 * pass;
    // pass p reads what pass p-1 wrote (buffers alternate; only pass 0 is offset)
    const int32_t* __restrict__ srcA = pass == 0 ? A.src0 : (pass & 1) ? A.bufB : A.bufA;
    int32_t* __restrict__ dst = (pass & 1) ? A.bufA : A.bufB;
    const int32_t pa = pass == 0 ? A.a : 0;
    const int64_t nA = A.n + pa;
    const int64_t cEnd = cE + A.E < nA ? cE + A.E : nA;
    const int64_t lenA = cEnd > cE ? cEnd - cE : 0;
    const int32_t m = (int32_t)(lenA <= A.vcap && !A.force_stream ? lenA : 0);   // staged entries (all or none)
    // a slice larger than the cache streams through it instead: every warp
    // double-buffers its own blocks with cp.async (two 2 KB buffers per warp),
    // so two blocks per warp are in flight instead of one
    const bool stream = m == 0 && lenA > 0 && A.vcap >= 2 * MC_BLOCK * MC_WARPS;
    if (tid == 0 && pass > 0) {   // (pass 0's copy was issued at kernel start)
      // every piece of the previous pass has landed (each was waited on by a
      // warp; this makes re-arming safe regardless), then the previous pass's
      // generic-proxy writes (this CTA's shared reads, every CTA's global
      // scatter, ordered by the grid barrier) before the async-proxy copy
      for (int k = 0; k < MC_PIECES; ++k) mbar_wait(bar + k, (pass - 1) & 1);
      asm volatile("fence.proxy.async;" ::: "memory");
      issue(srcA, m);
    }
    for (int i = lane; i < 256; i += 32) cnt[warp][i] = 0;
    if (tid == 0) red[kRedNq] = 0;
    __syncthreads();
    if (pass == 0) MCTS(1);
    const int32_t P4 = piece_len(m);
    int waited = -1;   // the highest piece this warp has waited for in this pass
    auto need = [&](int32_t boff) {   // the block at boff may read the staged slice
      if (boff >= m) return;
      const int pc = boff / P4;
      if (pc > waited) { for (int k = waited + 1; k <= pc; ++k) mbar_wait(bar + k, pass & 1); waited = pc; }
    };
    auto valid = [&](int32_t off) { int64_t ia = cE + off; return ia >= pa && ia < nA; };
    auto fetch = [&](int32_t off) -> int32_t { return off < m ? cache[off] : __ldcs(srcA + cE + off); };
    const int32_t nblk = (int32_t)((lenA + MC_BLOCK - 1) / MC_BLOCK);
    const int32_t b0 = (int32_t)((int64_t)nblk * warp / MC_WARPS);
    const int32_t b1 = (int32_t)((int64_t)nblk * (warp + 1) / MC_WARPS);
    int32_t c_lo = 1, c_hi = 0, c_d = 0;   // the warp's cached constant-class interval
    int32_t l_lo = 1, l_hi = 0, l_d = 0;   // this lane's (per-entry paths: lane k sees every 32nd entry)
    auto lane_digit = [&](int32_t x) -> int {
      if (x >= c_lo && x < c_hi) return c_d;
      if (x < l_lo || x >= l_hi) {
        const Span sp = seg_find(S, x);
        l_lo = sp.lo; l_hi = sp.hi; l_d = (sp.cls >> shift) & 255;
      }
      return l_d;
    };
    // digit of a run [v, v + len) if it lies in one constant-class interval, else -1
    auto run_digit = [&](int32_t v, int32_t len) -> int {
      if (!(v >= c_lo && v + (len - 1) < c_hi)) {
        Span sp = seg_find(S, v);
        c_lo = sp.lo; c_hi = sp.hi; c_d = (sp.cls >> shift) & 255;
      }
      return v + (len - 1) < c_hi ? c_d : -1;
    };
    // ---- phase 1: classify and count
#ifdef MSG_MC_PHASE_TS
    unsigned long long wp_t0 = 0;
    int wp_slow = 0;
#endif
    int32_t* const wbuf = cache + warp * 2 * MC_BLOCK;
    auto gfull = [&](int32_t b) { return cE + (int64_t)(b + 1) * MC_BLOCK <= nA; };
    auto prefetch = [&](int32_t b) {
      int32_t* d = wbuf + (b & 1) * MC_BLOCK;
      const int32_t* s = srcA + cE + (int64_t)b * MC_BLOCK;
#pragma unroll
      for (int t = 0; t < 4; ++t) cp_async16(d + 4 * lane + 128 * t, s + 4 * lane + 128 * t);
      cp_async_commit();
    };
    if (stream && b0 < b1 && gfull(b0)) prefetch(b0);
    for (int32_t b = b0; b < b1; ++b) {
      const int32_t boff = b * MC_BLOCK;
      need(boff);
#ifdef MSG_MC_PHASE_TS
      if (!wp_t0) wp_t0 = mc_now();
#endif
      const bool full = cE + boff >= pa && cE + boff + MC_BLOCK <= nA;
      // lane reads the 16-byte words lane + 32 t: each load instruction covers
      // 512 contiguous bytes (no shared-memory bank conflicts)
      int4 q[4];
      if (boff + MC_BLOCK <= m) {
#pragma unroll
        for (int t = 0; t < 4; ++t) q[t] = *reinterpret_cast<const int4*>(cache + boff + 4 * lane + 128 * t);
      } else if (stream && gfull(b)) {
        // block b was prefetched (before the loop, or in the previous iteration)
        const bool nxt = b + 1 < b1 && gfull(b + 1);
        if (nxt) { prefetch(b + 1); cp_async_wait<1>(); } else { cp_async_wait<0>(); }
        const int32_t* s = wbuf + (b & 1) * MC_BLOCK;   // each lane reads the 16-byte words it copied
#pragma unroll
        for (int t = 0; t < 4; ++t) q[t] = *reinterpret_cast<const int4*>(s + 4 * lane + 128 * t);
      } else if (cE + boff + MC_BLOCK <= nA) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          q[t] = __ldcs(reinterpret_cast<const int4*>(srcA + cE + boff + 4 * lane + 128 * t));
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          int32_t o = boff + 4 * lane + 128 * t;
          q[t].x = valid(o) ? fetch(o) : 0; q[t].y = valid(o + 1) ? fetch(o + 1) : 0;
          q[t].z = valid(o + 2) ? fetch(o + 2) : 0; q[t].w = valid(o + 3) ? fetch(o + 3) : 0;
        }
      }
      const int32_t v0 = __shfl_sync(0xffffffffu, q[0].x, 0);
      bool ok = full;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        int32_t e = v0 + 4 * lane + 128 * t;
        ok = ok && q[t].x == e && q[t].y == e + 1 && q[t].z == e + 2 && q[t].w == e + 3;
      }
      int d = __all_sync(0xffffffffu, ok) ? run_digit(v0, MC_BLOCK) : -1;
      if (d >= 0) {
        if (lane < 4) info[4 * b + lane] = make_int2(v0 + MS_CHUNK * lane, d);
        if (lane == 0) cnt[warp][d] += MC_BLOCK;
        __syncwarp();
        continue;
      }
      // mixed block: per 128-entry chunk, entries striped (32k + lane)
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        const int32_t coff = boff + MS_CHUNK * j;
        int32_t x[4];
        bool okc = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          int32_t o = coff + 32 * k + lane;
          bool vk = valid(o);
          x[k] = vk ? fetch(o) : 0;
          okc = okc && vk;
        }
        const int32_t c0 = __shfl_sync(0xffffffffu, x[0], 0);
#pragma unroll
        for (int k = 0; k < 4; ++k) okc = okc && x[k] == c0 + 32 * k + lane;
        int dc = __all_sync(0xffffffffu, okc) ? run_digit(c0, MS_CHUNK) : -1;
        if (dc >= 0) {
          if (lane == 0) { info[4 * b + j] = make_int2(c0, dc); cnt[warp][dc] += MS_CHUNK; }
          __syncwarp();
          continue;
        }
#ifdef MSG_MC_PHASE_TS
        ++wp_slow;
#endif
        // per-entry chunk: queued for the whole CTA when there is room
        int q = 0;
        if (lane == 0) q = atomicAdd(&red[kRedNq], 1);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q < MC_QCAP) {
          if (lane == 0) { info[4 * b + j] = make_int2(q, -2); red[kRedQ + q] = ((coff / MS_CHUNK) << 5) | warp; }
          __syncwarp();
          continue;
        }
        if (lane == 0) info[4 * b + j] = make_int2(0, -1);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          int dk = valid(coff + 32 * k + lane) ? lane_digit(x[k]) : 256;
          uint32_t peers = __match_any_sync(0xffffffffu, dk);
          if (dk < 256 && lane == __ffs(peers) - 1) cnt[warp][dk] += __popc(peers);
          __syncwarp();
        }
      }
    }
    __syncthreads();
    // ---- phase 1b: the queued per-entry chunks, round-robin over the warps;
    // counts go to the owner's row (shared atomics: several warps may add to
    // one row), digits to the byte store phase 3 reads
    {
      const int nq = red[kRedNq] < MC_QCAP ? red[kRedNq] : MC_QCAP;
      uint8_t* const dig = reinterpret_cast<uint8_t*>(red + kRedDig);
      for (int q = warp; q < nq; q += MC_WARPS) {
        const int32_t qi = red[kRedQ + q];
        const int own = qi & 31;
        const int32_t coff = (qi >> 5) * MS_CHUNK;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int32_t o = coff + 32 * k + lane;
          const bool vk = valid(o);
          const int dk = vk ? lane_digit(fetch(o)) : 256;
          if (vk) dig[q * MS_CHUNK + 32 * k + lane] = (uint8_t)dk;
          if (dk < 256) atomicAdd(&cnt[own][dk], 1);   // (counts need no lane match)
        }
      }
      if (nq) __syncthreads();
    }
#ifdef MSG_MC_PHASE_TS
    if (pass == 0 && lane == 0 && blockIdx.x < 160) {
      const unsigned long long t1 = mc_now();
      g_mc_warp[A.dbg_id & 63][blockIdx.x][warp] = ((t1 - (wp_t0 ? wp_t0 : t1)) << 32) | ((unsigned long long)wp_slow << 16) |
                                                   (unsigned long long)(b1 - b0);
    }
#endif
    if (pass == 0) MCTS(2);
    // ---- CTA histogram; exclusive warp offsets; digit totals by atomics
    int32_t* tot = A.totb + 256 * ((A.par + pass) & 1);
    if (tid < 256) {
      int32_t acc = 0;
#pragma unroll 8
      for (int w = 0; w < MC_WARPS; ++w) { int32_t t = cnt[w][tid]; cnt[w][tid] = acc; acc += t; }
      __stcg(A.hist + (int64_t)blockIdx.x * 256 + tid, acc);
      if (acc) atomicAdd(tot + tid, acc);
      red[kRedSlice + tid] = acc;   // this slice's digit counts
      red[tid] = 0;            // prefix accumulators
    }
    if (tid == 0) red[kRedNd] = 0;
    if (pass == 0) MCTS(3);
    grid_barrier(A.bar, nbar++);
    if (pass == 0) MCTS(4);
    // ---- phase 2: digit bases = totals scan + this CTA's prefix over the
    // CTAs before it.  Only the digits present in this slice need a base (long
    // runs make that a handful), so the CTA reads those columns of the earlier
    // rows -- one round of independent loads -- instead of whole rows.
    {
      int32_t* dl = red + kRedDl;   // present digits
      if (tid < 256 && red[kRedSlice + tid] > 0) dl[atomicAdd(&red[kRedNd], 1)] = tid;
      __syncthreads();
      const int nd = red[kRedNd], me = (int)blockIdx.x;
      if (nd <= 16) {
        for (int k = tid; k < nd * me; k += MC_THREADS) {
          const int j = k / me, c2 = k - j * me;
          const int d = dl[j];
          const int32_t v = __ldcg(A.hist + (int64_t)c2 * 256 + d);
          if (v) atomicAdd(&red[d], v);
        }
      } else {
        // many digits (fragmented lists): whole columns, four threads per
        // digit each summing a quarter of the earlier rows (coalesced rows,
        // independent loads, no shared-memory atomics)
        const int d = tid & 255, q = tid >> 8;
        const int r0 = me * q / 4, r1 = me * (q + 1) / 4;
        int32_t acc = 0;
#pragma unroll 8
        for (int c2 = r0; c2 < r1; ++c2) acc += __ldcg(A.hist + (int64_t)c2 * 256 + d);
        red[kRedCol + q * 256 + d] = acc;
        __syncthreads();
        if (tid < 256)
          red[tid] = red[kRedCol + tid] + red[kRedCol + 256 + tid] + red[kRedCol + 512 + tid] + red[kRedCol + 768 + tid];
      }
    }
    __syncthreads();
    {
      int64_t pre = 0, tt = 0, x = 0;
      if (tid < 256) {
        pre = red[tid];
        tt = __ldcg(tot + tid);
        x = tt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int64_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) misc[warp] = x;
      }
      __syncthreads();
      if (tid < 256) {
        int64_t wp = 0;
        for (int w = 0; w < warp; ++w) wp += misc[w];
        base[tid] = wp + (x - tt) + pre;
        // the other totals row starts the next pass (or launch) at zero; its
        // last readers finished before the previous pass's closing barrier
        if (blockIdx.x == 0) A.totb[256 * ((A.par + pass + 1) & 1) + tid] = 0;
      }
    }
    __syncthreads();
    if (pass == 0) MCTS(5);
    // ---- phase 3: replay the blocks in order and scatter
    for (int32_t b = b0; b < b1; ++b) {
      const int32_t boff = b * MC_BLOCK;
      int2 r = lane < 4 ? info[4 * b + lane] : make_int2(0, -1);
      const int32_t v0 = __shfl_sync(0xffffffffu, r.x, 0);
      const int d0 = __shfl_sync(0xffffffffu, r.y, 0);
      const bool same = lane >= 4 || (r.y == d0 && r.x == v0 + MS_CHUNK * lane);
      if (d0 >= 0 && __all_sync(0xffffffffu, same)) {
        const int32_t before = cnt[warp][d0];
        const int64_t p = base[d0] + before;
        const int32_t ph = (int32_t)((4 - (p & 3)) & 3);          // entries before a 16-B boundary
        if (lane < ph) dst[p + lane] = v0 + lane;
        const int32_t nb = (MC_BLOCK - ph) >> 2;
        for (int32_t k = lane; k < nb; k += 32) {
          int32_t t = ph + 4 * k;
          *reinterpret_cast<int4*>(dst + p + t) = make_int4(v0 + t, v0 + t + 1, v0 + t + 2, v0 + t + 3);
        }
        const int32_t ts = ph + 4 * nb;
        if (lane < MC_BLOCK - ts) dst[p + ts + lane] = v0 + ts + lane;
        __syncwarp();
        if (lane == 0) cnt[warp][d0] = before + MC_BLOCK;
        __syncwarp();
        continue;
      }
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        const int32_t rx = __shfl_sync(0xffffffffu, r.x, j);
        const int ry = __shfl_sync(0xffffffffu, r.y, j);
        const int32_t coff = boff + MS_CHUNK * j;
        if (ry >= 0) {
          const int32_t before = cnt[warp][ry];
          const int64_t p = base[ry] + before + lane;
#pragma unroll
          for (int k = 0; k < 4; ++k) dst[p + 32 * k] = rx + lane + 32 * k;
          __syncwarp();
          if (lane == 0) cnt[warp][ry] = before + MS_CHUNK;
          __syncwarp();
          continue;
        }
        const uint8_t* const dq = reinterpret_cast<const uint8_t*>(red + kRedDig) + rx * MS_CHUNK;   // ry == -2
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int32_t o = coff + 32 * k + lane;
          const bool vk = valid(o);
          const int32_t xv = vk ? fetch(o) : 0;
          int dk = vk ? (ry == -2 ? (int)dq[32 * k + lane] : lane_digit(xv)) : 256;
          uint32_t peers = __match_any_sync(0xffffffffu, dk);
          int32_t before = dk < 256 ? cnt[warp][dk] : 0;
          __syncwarp();
          if (dk < 256 && lane == __ffs(peers) - 1) cnt[warp][dk] = before + __popc(peers);
          __syncwarp();
          if (dk < 256) dst[base[dk] + before + __popc(peers & lt)] = xv;
        }
      }
    }
    // the next pass reads this pass's output grid-wide
    if (pass + 1 < passes) grid_barrier(A.bar, nbar++);
  }
  __syncthreads();
  MCTS(6);
#ifdef MSG_MC_PHASE_TS
  if (threadIdx.x == 0) atomicAdd(&g_mc_n, 1ull);
#endif
  if (threadIdx.x == 0) atomicMax(A.t_last, global_ns());
}

__global__ void __launch_bounds__(MC_THREADS, 1) k_ms_coop(McArgs A) {
  extern __shared__ __align__(16) unsigned char mc_raw[];
  int nbar = 0;
  ms_coop_body(A, mc_raw, nbar);
}

// generic exclusive scan (int32 in -> int64 out), 3 phases
constexpr int SCAN_BLOCK = 1024, SCAN_ITEMS = 4, SCAN_CHUNK = SCAN_BLOCK * SCAN_ITEMS;

__global__ void __launch_bounds__(1024, 1) k_scan_reduce(const int32_t* in, int64_t n, int64_t* sums) {
  __shared__ int64_t ws[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_CHUNK;
  int64_t acc = 0;
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + k * SCAN_BLOCK + threadIdx.x;
    if (i < n) acc += in[i];
  }
  int64_t tot;
  block_excl_scan<int64_t>(acc, ws, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024, 1) k_scan_sums(int64_t* sums, int64_t nb) { block_scan_array<int64_t>(sums, nb); }

__global__ void __launch_bounds__(1024, 1) k_scan_down(const int32_t* in, int64_t n, const int64_t* sums, int64_t* out) {
  __shared__ int64_t ws[32];
  __shared__ int64_t carry;
  int64_t base = (int64_t)blockIdx.x * SCAN_CHUNK;
  if (threadIdx.x == 0) carry = sums[blockIdx.x];
  __syncthreads();
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + k * SCAN_BLOCK + threadIdx.x;
    int64_t v = i < n ? in[i] : 0;
    int64_t tot;
    int64_t ex = block_excl_scan<int64_t>(v, ws, &tot);
    if (i < n) out[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

static void scan_i32_to_i64(Ctx& c, const int32_t* in, int64_t n, int64_t* out) {
  int64_t nb = (n + SCAN_CHUNK - 1) / SCAN_CHUNK;
  c.s.i64e.resize(std::max<int64_t>(nb, 1), c.st);
  k_scan_reduce<<<nb, SCAN_BLOCK, 0, c.st>>>(in, n, c.s.i64e.p);
  k_scan_sums<<<1, SCAN_BLOCK, 0, c.st>>>(c.s.i64e.p, nb);
  k_scan_down<<<nb, SCAN_BLOCK, 0, c.st>>>(in, n, c.s.i64e.p, out);
  MSG_CHECK_LAUNCH();
  add_launches(3);
}

void scan_flags(Ctx& c, const int32_t* in, int64_t n, int64_t* out) { scan_i32_to_i64(c, in, n, out); }

int32_t* next_barrier(Ctx& c) {
  if (!c.ms_ctr.p) {
    c.ms_ctr.exact(1 << 16);
    c.ms_tot.exact(257 * MS_MAX_PASSES);
  }
  if (++c.ms_epoch >= (1u << 16)) {   // epochs wrap: clear the look-back status words too
    if (c.ms_status.p) MSG_CUDA(cudaMemsetAsync(c.ms_status.p, 0, c.ms_status.n * 8, c.st));
    c.ms_epoch = 1;
  }
  if (c.ms_epoch == 1) MSG_CUDA(cudaMemsetAsync(c.ms_ctr.p, 0, (1 << 16) * 4, c.st));
  return c.ms_ctr.p + c.ms_epoch;
}

// Sum the device-timed durations of the cooperative multisplit launches not
// yet counted (stats); syncs the planner stream.
void ms_harvest(Ctx& c) {
  if (!c.ms_tring.p || c.ms_tslot <= c.ms_tbase) return;
  const int64_t R = (int64_t)c.ms_tring.n / 2;
  std::vector<unsigned long long> h(2 * R);
  MSG_CUDA(cudaMemcpyAsync(h.data(), c.ms_tring.p, h.size() * 8, cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaStreamSynchronize(c.st));
  // launches that ran no pass (the async path's early exits) leave their
  // last-CTA stamp unset and are not counted
  for (int64_t k = c.ms_tbase; k < c.ms_tslot; ++k)
    if (h[R + k] > h[k]) { c.ms_dev_ms_acc += (double)(h[R + k] - h[k]) * 1e-6; ++c.stats.ms_dev_launches; }
  c.ms_tbase = c.ms_tslot;
}

static void ms_init(Ctx& c) {
  if (!c.ms_ctr.p) {
    c.ms_ctr.exact(1 << 16);
    c.ms_tot.exact(257 * MS_MAX_PASSES);
  }
  if (!c.ms_grid_cap) {
    int per_sm = 0, sms = 0, coop_per_sm = 0;
    MSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ms_onesweep, MS_THREADS, 0));
    MSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    MSG_CUDA(cudaFuncSetAttribute(k_ms_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, MC_SMEM));
    MSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&coop_per_sm, k_ms_coop, MC_THREADS, MC_SMEM));
    c.ms_grid_cap = std::max(1, per_sm) * std::max(1, sms);
    c.ms_coop_grid = coop_per_sm * sms;
  }
}

// Launch the cooperative multisplit of the current list, all digit passes in
// one launch (a grid barrier between passes).  Returns false when the list
// does not fit the on-chip path (the caller falls back).
// whether the cooperative multisplit can take the current list (the same
// geometry test ms_coop_launch makes), without launching it
static bool ms_coop_fits(Ctx& c, int grid = 0) {
  ms_init(c);
  const int coop_grid = grid ? grid : c.ms_coop_grid;
  if (c.len == 0 || coop_grid <= 0 || (c.debug & 8) || (c.fallback & 2)) return c.len == 0;
  const int64_t nA = c.len + 3;
  int64_t E = (nA + coop_grid - 1) / coop_grid;
  E = (E + MC_BLOCK - 1) / MC_BLOCK * MC_BLOCK;
  const int64_t nch = E / MS_CHUNK;
  const int64_t avail = (int64_t)MC_SMEM - MC_FIXED - 8 * (((nch + 1) + 1) & ~int64_t(1)) - 16;
  return (avail - 12 * (int64_t)MC_TCAP_MIN) / 4 - 4 >= 0;
}

struct DevPasses {   // the async path: pass count decided on the device
  const int64_t* ncls = nullptr;
  const int64_t* missing = nullptr;
  int reorder_always = 0;
  int64_t* out = nullptr;
};

// The multisplit's arguments for a cooperative grid of `grid` CTAs (false when
// the list does not fit the on-chip path).  Claims a device-timing slot.
static bool ms_args(Ctx& c, const SegTab& T, int passes, DevPasses dp, int grid, int32_t* bar, McArgs& A) {
  ms_init(c);
  const int64_t n = c.len;
  if (n == 0 || grid <= 0 || (c.debug & 8) || (c.fallback & 2)) return false;
  const int32_t* src0 = c.order[c.cur].p + c.head;
  const int32_t a = (int32_t)((reinterpret_cast<uintptr_t>(src0) & 15) >> 2);
  const int64_t nA = n + a;
  int64_t E = (nA + grid - 1) / grid;
  E = (E + MC_BLOCK - 1) / MC_BLOCK * MC_BLOCK;
  const int64_t nch = E / MS_CHUNK;
  // shared memory after the fixed part and the chunk records: the slice
  // cache (+ 4 entries of TMA rounding slack) and the class table (12 B per
  // segment; at least MC_TCAP_MIN, up to MC_TCAP_MAX when the slice is short)
  const int64_t avail = (int64_t)MC_SMEM - MC_FIXED - 8 * (((nch + 1) + 1) & ~int64_t(1)) - 16;
  int64_t tcap = (avail - 4 * (E + 4)) / 12;
  tcap = std::max<int64_t>(MC_TCAP_MIN, std::min<int64_t>(tcap, MC_TCAP_MAX)) & ~int64_t(3);
  if (c.ms_force_stream) tcap = MC_TCAP_MIN;   // the whole cache for the per-warp stream buffers
  int64_t vcap = (avail - 12 * tcap) / 4 - 4;
  if (!c.ms_force_stream) vcap = std::min<int64_t>(vcap, E);
  vcap &= ~int64_t(3);
  if (vcap < 0) return false;
  if ((int64_t)c.ms_hist.n < 256 * ((int64_t)grid + 2)) {
    c.ms_hist.exact(256 * ((int64_t)grid + 2));   // rows + two digit-total rows
    MSG_CUDA(cudaMemsetAsync(c.ms_hist.p, 0, c.ms_hist.n * 4, c.st));
    c.ms_tot_par = 0;
  }
  if (!c.ms_tring.p || c.ms_tslot >= (int64_t)c.ms_tring.n / 2) {   // (first, last) slot per launch
    if (!c.ms_tring.p) c.ms_tring.exact(2 * 4096);
    else ms_harvest(c);
    MSG_CUDA(cudaMemsetAsync(c.ms_tring.p, 0xff, 4096 * 8, c.st));
    MSG_CUDA(cudaMemsetAsync(c.ms_tring.p + 4096, 0, 4096 * 8, c.st));
    c.ms_tslot = 0;
    c.ms_tbase = 0;
  }
  unsigned long long* tf = c.ms_tring.p + c.ms_tslot;
  unsigned long long* tl = c.ms_tring.p + 4096 + c.ms_tslot;
  ++c.ms_tslot;
  A = McArgs{src0 - a, c.order[c.cur].p, c.order[c.cur ^ 1].p, n, a, T, c.ms_hist.p,
             c.ms_hist.p + 256 * (int64_t)grid, c.ms_tot_par, bar, E, (int32_t)vcap, (int32_t)nch,
             passes, tf, tl, (int32_t)(c.ms_launch_id++), (int32_t)tcap, dp.ncls, dp.missing, dp.reorder_always,
             dp.out, c.ms_force_stream};
  return true;
}

static bool ms_coop_launch(Ctx& c, const SegTab& T, int passes, DevPasses dp = DevPasses{}) {
  ms_init(c);
  McArgs A;
  if (!ms_args(c, T, passes, dp, c.ms_coop_grid, next_barrier(c), A)) return false;
  cudaEvent_t e0, e1;
  MSG_CUDA(cudaEventCreate(&e0));
  MSG_CUDA(cudaEventCreate(&e1));
  c.ev_pool.push_back(e0);
  c.ev_pool.push_back(e1);
  MSG_CUDA(cudaEventRecord(e0, c.st));
  void* args[] = {&A};
  MSG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_ms_coop), dim3(c.ms_coop_grid), dim3(MC_THREADS),
                                       args, MC_SMEM, c.st));
  MSG_CHECK_LAUNCH();
  add_launches(1);
  MSG_CUDA(cudaEventRecord(e1, c.st));
  c.busy_ms.push_back({e0, e1});
  c.ms_events_pending = true;
  return true;
}

// host bookkeeping once the number of passes a cooperative launch ran is known
static void ms_coop_done(Ctx& c, int passes) {
  if (c.ms_events_pending) c.stats.ms_ev_passes += std::max(passes, 0);
  c.ms_events_pending = false;
  if (passes <= 0) return;
  c.cur ^= passes & 1;
  c.head = 0;
  c.ms_tot_par ^= passes & 1;
  c.stats.ms_passes += passes;
  c.stats.ms_bytes += 8 * c.len * passes;
}

// Stable multisplit of order[cur][head, head+len) by class digits; result
// at order[cur^(passes&1)][0, len).  `passes` LSD passes.
static void multisplit(Ctx& c, const SegTab& T, int passes) {
  int64_t n = c.len;
  if (n == 0 || passes <= 0) return;
  if (ms_coop_launch(c, T, passes)) {
    ms_coop_done(c, passes);
    return;
  }
  // decoupled look-back fallback: one launch per pass
  if (passes > MS_MAX_PASSES) throw Error(MSG_E_INVAL, "too many reorder classes");
  int64_t ntiles = (n + MS_TILE - 1) / MS_TILE;
  if ((int64_t)c.ms_status.n < 256 * ntiles) {
    c.ms_status.exact(256 * ntiles);
    MSG_CUDA(cudaMemsetAsync(c.ms_status.p, 0, 256 * ntiles * 8, c.st));
    c.ms_epoch = 0;
  }
  const int grid_cap = c.ms_grid_cap;
  cudaEvent_t e0, e1;
  MSG_CUDA(cudaEventCreate(&e0));
  MSG_CUDA(cudaEventCreate(&e1));
  c.ev_pool.push_back(e0);
  c.ev_pool.push_back(e1);
  MSG_CUDA(cudaEventRecord(e0, c.st));
  unsigned long long* tot = c.ms_tot.p;
  // digit totals of all passes from the resident bitmap (one launch)
  MSG_CUDA(cudaMemsetAsync(tot, 0, 257 * passes * 8, c.st));
  k_ms_digit_totals<<<296, 256, 0, c.st>>>(T, c.bits.p, passes, tot);
  add_launches(1);
  for (int pass = 0; pass < passes; ++pass) {
    int32_t* bar = next_barrier(c);   // the onesweep tile counter of this pass
    const int32_t* src = c.order[c.cur].p + c.head;
    int32_t* dst = c.order[c.cur ^ 1].p;
    Onesweep O{c.ms_status.p, (int64_t)(c.ms_status.n / 256), bar, tot + 257 * pass, c.ms_epoch};
    int grid = (int)std::min<int64_t>(ntiles, grid_cap);
    k_ms_onesweep<<<grid, MS_THREADS, 0, c.st>>>(src, n, T, 8 * pass, dst, O);
    MSG_CHECK_LAUNCH();
    add_launches(1);
    c.cur ^= 1;
    c.head = 0;
  }
  MSG_CUDA(cudaEventRecord(e1, c.st));
  c.busy_ms.push_back({e0, e1});
  c.stats.ms_passes += passes;
  c.stats.ms_ev_passes += passes;
  c.stats.ms_bytes += 8 * n * passes;
}

// ---------------------------------------------------------------------------
// apply: evict the list head, install pages at the tail (memman.py:43-56, 93-112)

// Copy-ordering epochs (migration only): inst_ep[f] = batch whose H2D last
// wrote frame f, free_ep[f] = batch whose D2H last read it.  A batch's D2H
// waits only for the H2D batch that wrote the newest frame it evicts, and its
// H2D into previously free frames only for the D2H batch that freed the
// newest of them (dep[0], dep[1]).
struct Epochs {
  int32_t* inst_ep;
  int32_t* free_ep;
  int32_t batch;
  int* dep;   // [0] max inst_ep over evicted frames, [1] max free_ep over reused free frames
};

// Warp-aggregated residency-bit update: lanes whose pages share a bitmap word
// combine their bits and one lane issues the atomic (list runs put 32
// consecutive pages in one word, which would otherwise serialise 32 atomics).
__device__ __forceinline__ void bits_update(uint32_t* bits, int32_t p, bool valid, bool set) {
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const int32_t wd = p >> 5;
  const unsigned peers = __match_any_sync(act, wd);
  const unsigned m = __reduce_or_sync(peers, 1u << (p & 31));
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) {
    if (set) atomicOr(&bits[wd], m); else atomicAnd(&bits[wd], ~m);
  }
}

__device__ __forceinline__ void evict_body(const int32_t* __restrict__ order, int64_t n, uint32_t* bits,
                                           int32_t* frame, int32_t* fifo, int64_t fifo_tail, int64_t C, int64_t* mig,
                                           Epochs ep) {
  // EV_ILP elements per thread per step, their loads issued together: the
  // order -> frame chain is paid once per step, not once per element
  constexpr int EV_ILP = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int dep = -1;
  for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x; e0 < n; e0 += EV_ILP * stride) {
    int32_t p[EV_ILP], f[EV_ILP];
    bool v[EV_ILP];
#pragma unroll
    for (int k = 0; k < EV_ILP; ++k) {
      const int64_t e = e0 + k * stride + threadIdx.x;
      v[k] = e < n;
      p[k] = v[k] ? __ldcg(order + e) : 0;
    }
#pragma unroll
    for (int k = 0; k < EV_ILP; ++k) f[k] = v[k] ? frame[p[k]] : -1;
#pragma unroll
    for (int k = 0; k < EV_ILP; ++k) {
      bits_update(bits, p[k], v[k], false);
      if (!v[k]) continue;
      const int64_t e = e0 + k * stride + threadIdx.x;
      frame[p[k]] = -1;
      int64_t q = fifo_tail + e;
      if (q >= C) q -= C;
      if (q >= C) q -= C;
      fifo[q] = f[k];
      if (mig) mig[e] = ((int64_t)p[k] << 32) | (uint32_t)f[k];
      if (ep.inst_ep) {
        dep = max(dep, ep.inst_ep[f[k]]);
        ep.free_ep[f[k]] = ep.batch;
      }
    }
  }
  if (ep.inst_ep) {
    dep = __reduce_max_sync(0xffffffffu, dep);
    if ((threadIdx.x & 31) == 0 && dep >= 0) atomicMax(&ep.dep[0], dep);
  }
}
__global__ void k_evict_head(const int32_t* __restrict__ order, int64_t n, uint32_t* bits, int32_t* frame,
                             int32_t* fifo, int64_t fifo_tail, int64_t C, int64_t* mig, Epochs ep) {
  evict_body(order, n, bits, frame, fifo, fifo_tail, C, mig, ep);
}

__device__ __forceinline__ void install_body(const int32_t* __restrict__ pages, int64_t n, uint32_t* bits,
                                             int32_t* frame, const int32_t* __restrict__ fifo, int64_t fifo_head,
                                             int64_t C, int32_t* order_tail, int64_t* mig, Epochs ep,
                                             int64_t old_free) {
  constexpr int IN_ILP = 4;   // as in evict_body: the loads of several elements in flight together
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int dep = -1;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x; j0 < n; j0 += IN_ILP * stride) {
    int32_t p[IN_ILP], f[IN_ILP];
    bool v[IN_ILP];
#pragma unroll
    for (int k = 0; k < IN_ILP; ++k) {
      const int64_t j = j0 + k * stride + threadIdx.x;
      v[k] = j < n;
      p[k] = v[k] ? __ldcg(pages + j) : 0;
      int64_t q = fifo_head + j;
      if (q >= C) q -= C;
      if (q >= C) q -= C;
      f[k] = v[k] ? __ldcg(fifo + q) : -1;
    }
#pragma unroll
    for (int k = 0; k < IN_ILP; ++k) {
      bits_update(bits, p[k], v[k], true);
      if (!v[k]) continue;
      const int64_t j = j0 + k * stride + threadIdx.x;
      frame[p[k]] = f[k];
      order_tail[j] = p[k];
      if (mig) mig[j] = ((int64_t)p[k] << 32) | (uint32_t)f[k];
      if (ep.inst_ep) {
        if (j < old_free) dep = max(dep, ep.free_ep[f[k]]);
        ep.inst_ep[f[k]] = ep.batch;
      }
    }
  }
  if (ep.inst_ep) {
    dep = __reduce_max_sync(0xffffffffu, dep);
    if ((threadIdx.x & 31) == 0 && dep >= 0) atomicMax(&ep.dep[1], dep);
  }
}
__global__ void k_install(const int32_t* __restrict__ pages, const int64_t* np_dev, int64_t np_host, uint32_t* bits,
                          int32_t* frame, const int32_t* __restrict__ fifo, int64_t fifo_head, int64_t C,
                          int32_t* order_tail, int64_t* mig, Epochs ep, int64_t old_free) {
  install_body(pages, np_dev ? *np_dev : np_host, bits, frame, fifo, fifo_head, C, order_tail, mig, ep, old_free);
}

// The async switch path (no host round trip between plan and apply): the
// list's position after the multisplit and the evict / populate counts are
// read on the device.  ListSel: where the live list starts -- the other
// buffer at 0 after an odd number of multisplit passes, this buffer at 0
// after an even nonzero number, unchanged when no pass ran.
struct ListSel {
  int32_t* cur; int32_t* other; int64_t head; const int64_t* passes_dev;
};
__device__ __forceinline__ int32_t* sel_base(const ListSel& L) {
  const int64_t p = L.passes_dev ? __ldcg(L.passes_dev) : 0;
  return p > 0 ? ((p & 1) ? L.other : L.cur) : L.cur + L.head;
}
// the plan fits (populate <= free frames + evictions, engine.py:338-339);
// otherwise nothing is applied and the host reports the error
__device__ __forceinline__ bool plan_fits(const DevState* S, int64_t C, int64_t len0) {
  return __ldcg(&S->populate) <= C - len0 + __ldcg(&S->evict);
}
// S != nullptr: the switch plan's counts (S->evict / S->populate), applied
// only when the plan fits; S == nullptr (touch installs): n_host evictions
// and *np_dev installs
__global__ void k_evict_head_dev(ListSel L, const DevState* S, int64_t n_host, int64_t len0, uint32_t* bits,
                                 int32_t* frame, int32_t* fifo, int64_t fifo_tail, int64_t C) {
  if (S && !plan_fits(S, C, len0)) return;
  evict_body(sel_base(L), S ? S->evict : n_host, bits, frame, fifo, fifo_tail, C, nullptr,
             Epochs{nullptr, nullptr, 0, nullptr});
}
__global__ void k_install_dev(const int32_t* __restrict__ pages, ListSel L, const DevState* S, const int64_t* np_dev,
                              int64_t len0, uint32_t* bits, int32_t* frame, const int32_t* __restrict__ fifo,
                              int64_t fifo_head, int64_t C) {
  if (S && !plan_fits(S, C, len0)) return;
  // after evicting e pages from the head the tail sits at head + e + (len0 - e)
  install_body(pages, S ? S->populate : *np_dev, bits, frame, fifo, fifo_head, C, sel_base(L) + len0, nullptr,
               Epochs{nullptr, nullptr, 0, nullptr}, 0);
}

// results gathered into the pinned readback buffer (see k_pack / apply_body)
struct PackSeg { const int64_t* src; int32_t words; int32_t dst_word; };
struct PackArgs { PackSeg seg[6]; int32_t nseg; int64_t* dst; };

// The async path's apply as ONE cooperative launch (in place of evict,
// install, the touch-count memset + scan and the result gather): evict the
// head, grid barrier, install the populate list, grid barrier, count the
// missing pages of the slice's commands against the new residency, grid
// barrier, and block 0 writes the call's results into the pinned readback
// buffer.  Counts come from DevState (a switch plan: applied only when it
// fits) or from the host / *np_dev (a touch).
struct ApplyArgs {
  ListSel L;
  const DevState* S;          // plan counts, or nullptr
  int64_t ev_host;            // touch: evictions
  const int64_t* np_dev;      // touch: installs (the missing count)
  int64_t len0;
  uint32_t* bits; int32_t* frame; int32_t* fifo;
  int64_t fifo_tail, fifo_head, C;
  const int32_t* pages;
  // touch scan of commands [tc_c0, tc_c0 + tc_n) of one task
  const Iv* act_pool; const int64_t* act_off; int32_t tc_c0, tc_n;
  unsigned long long* tc;     // tc_n counters (zeroed here)
  int32_t* bar;               // grid barrier counter (zero at launch)
  PackArgs pack;              // results -> pinned readback (pack.dst == nullptr: none)
};
constexpr int AP_SPLIT = 8;   // blocks' worth of work per command in the touch scan

// The apply: the last phase of the per-switch cooperative kernel
// (k_switch_coop).  The counts and lists it reads may come from earlier
// phases of the same kernel, so they are read from L2 (ld.cg), never from a
// stale L1 line.  red: blockDim / 32 words of shared memory.
__device__ __forceinline__ void apply_body(const ApplyArgs& A, int& nbar, unsigned long long* red) {
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < A.tc_n; i += blockDim.x) A.tc[i] = 0;
  const bool fits = A.S == nullptr || plan_fits(A.S, A.C, A.len0);
  const int64_t ev = A.S ? (fits ? __ldcg(&A.S->evict) : 0) : A.ev_host;
  int32_t* base = sel_base(A.L);
  evict_body(base, ev, A.bits, A.frame, A.fifo, A.fifo_tail, A.C, nullptr, Epochs{nullptr, nullptr, 0, nullptr});
  grid_barrier(A.bar, nbar++);
  SWTS(3);
  const int64_t np = A.S ? (fits ? __ldcg(&A.S->populate) : 0) : (A.np_dev ? __ldcg(A.np_dev) : 0);
  install_body(A.pages, np, A.bits, A.frame, A.fifo, A.fifo_head, A.C, base + A.len0, nullptr,
               Epochs{nullptr, nullptr, 0, nullptr}, 0);
  grid_barrier(A.bar, nbar++);
  SWTS(4);
  // touch scan: (command, split) work items over the blocks; each item strides
  // the command's bitmap words like k_touch_counts' blockIdx.x
  for (int item = blockIdx.x; item < A.tc_n * AP_SPLIT; item += gridDim.x) {
    const int32_t cmd = A.tc_c0 + item / AP_SPLIT, split = item % AP_SPLIT;
    const int64_t i0 = A.act_off[cmd], i1 = A.act_off[cmd + 1];
    const int64_t T = (int64_t)AP_SPLIT * blockDim.x, me = (int64_t)split * blockDim.x + threadIdx.x;
    unsigned long long acc = 0;
    int64_t skip = 0;
    for (int64_t i = i0; i < i1; ++i) {
      const Iv v = A.act_pool[i];
      const int64_t lo = v.d, hi = v.d + (v.b - v.a), w0 = lo >> 5, nw = ((hi + 31) >> 5) - w0;
      // (me - skip) mod T; T = AP_SPLIT * 1024 is a power of two: a mask instead of a 64-bit remainder per interval
      int64_t k = (T & (T - 1)) == 0 ? ((me - skip) & (T - 1)) : (((me - skip) % T) + T) % T;
      for (; k < nw; k += T) acc += __popc(~__ldcg(A.bits + w0 + k) & unit_mask(lo, hi, w0 + k));
      skip += nw;
    }
    acc = __reduce_add_sync(0xffffffffu, (unsigned)acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
      if (s) atomicAdd(&A.tc[item / AP_SPLIT], s);
    }
    __syncthreads();
  }
  if (A.pack.dst == nullptr) return;
  grid_barrier(A.bar, nbar++);
  SWTS(5);
  if (blockIdx.x == 0)
    for (int s = 0; s < A.pack.nseg; ++s)
      for (int i = threadIdx.x; i < A.pack.seg[s].words; i += blockDim.x)
        A.pack.dst[A.pack.seg[s].dst_word + i] = __ldcg(A.pack.seg[s].src + i);
  SWTS(7);
}


// The async switch path's device work after the window kernel as ONE
// cooperative launch: the units plan (missing = demand - resident, the plan
// scalars, the populate list; or a faulting command's missing list), the
// multisplit (pass count read on the device), then evict, install, the touch
// scan and the result gather -- grid barriers between the phases, all on one
// barrier counter, one CTA per SM with the multisplit's shared memory.
struct SwitchArgs {
  UnitsPlan up;
  McArgs ms;
  ApplyArgs ap;
  int32_t has_up, has_ms;
};

__global__ void __launch_bounds__(MC_THREADS, 1) k_switch_coop(SwitchArgs A) {
  extern __shared__ __align__(16) unsigned char sw_raw[];
  __shared__ unsigned long long red[MC_WARPS];
  int nbar = 0;
  SWTS(0);
  if (A.has_up) {
    units_plan_body(A.up, sw_raw, nbar);
    grid_barrier(A.ap.bar, nbar++);
  }
  SWTS(1);
  if (A.has_ms) {
    ms_coop_body(A.ms, sw_raw, nbar);
    grid_barrier(A.ap.bar, nbar++);
  }
  SWTS(2);
  apply_body(A.ap, nbar, red);
}

// MSG_F_EXECUTE: populate position of every page installed by this switch,
// and per command of the slice the populate prefix its actual set needs
__global__ void k_pos_scatter(const int32_t* __restrict__ pages, int64_t n, int64_t tag, int64_t* pos_of) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    pos_of[pages[j]] = (tag << 32) | j;
}

__global__ void k_gate_need(const Iv* __restrict__ pool, const int64_t* __restrict__ off, int32_t c0, int32_t c1,
                            const int64_t* __restrict__ pos_of, int64_t tag, unsigned long long* need) {
  // one warp per (command, interval) pair, lanes over pages
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t i0 = off[c0], n = off[c1] - i0;
  for (int64_t i = warp; i < n; i += nwarps) {
    int32_t a = c0, b = c1;   // command of interval i0 + i
    while (a < b) { int32_t mid = (a + b) >> 1; if (off[mid + 1] <= i0 + i) a = mid + 1; else b = mid; }
    const Iv v = pool[i0 + i];
    unsigned long long m = 0;
    for (int64_t k = lane; k < v.b - v.a; k += 32) {
      int64_t x = pos_of[v.d + k];
      if ((x >> 32) == tag) m = max(m, (unsigned long long)(x & 0xffffffff) + 1);
    }
    m = __reduce_max_sync(0xffffffffu, (unsigned)m);
    if (lane == 0 && m) atomicMax(&need[a - c0], m);
  }
}

// ---------------------------------------------------------------------------
// K8 touch scan: missing pages of each command's actual set (engine.py:396-397)


// missing pages of one command in page order (for installs): one warp per interval



// class table from explicit dense ranges (madvise / remove / release)
__global__ void k_table_from_ranges(const int64_t* lo, const int64_t* len, int64_t n, int64_t* tlo, int64_t* thi,
                                    int32_t* tcls, int64_t* tn) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    tlo[i] = lo[i];
    thi[i] = lo[i] + len[i];
    tcls[i] = 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *tn = n;
}

// ---------------------------------------------------------------------------
// host orchestration

static DevState& hs(Ctx& c) { return *c.hstate; }

// One launch that gathers a call's small results (DevState, per-window and
// per-command counts) from device buffers straight into the pinned readback
// buffer (mapped), in place of one device-to-host copy per buffer.
__global__ void k_pack(PackArgs A) {
  for (int s = 0; s < A.nseg; ++s)
    for (int i = threadIdx.x; i < A.seg[s].words; i += blockDim.x) A.dst[A.seg[s].dst_word + i] = A.seg[s].src[i];
}
static void pack_to_host(Ctx& c, PackArgs& A) {
  MSG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&A.dst), c.hbuf.p, 0));
  k_pack<<<1, 256, 0, c.st>>>(A);
  MSG_CHECK_LAUNCH();
  add_launches(1);
}

// grid of the per-switch cooperative kernel (one CTA per SM)
static int sw_grid(Ctx& c) {
  if (!c.sw_grid) {
    MSG_CUDA(cudaFuncSetAttribute(k_switch_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, MC_SMEM));
    int per_sm = 0;
    MSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_switch_coop, MC_THREADS, MC_SMEM));
    if (!c.nsm) MSG_CUDA(cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, c.device));
    c.sw_grid = per_sm * c.nsm;
  }
  return c.sw_grid;
}

static void switch_launch(Ctx& c, SwitchArgs& A) {
  if (A.ap.pack.nseg) MSG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&A.ap.pack.dst), c.hbuf.p, 0));
  void* args[] = {&A};
  MSG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_switch_coop), dim3(sw_grid(c)), dim3(MC_THREADS),
                                       args, MC_SMEM, c.st));
  MSG_CHECK_LAUNCH();
  add_launches(1);
}

// host phase clock (MSG_HOST_PHASES=1): mark(i) adds the time since the
// previous mark to phase i of call kind k
struct PhaseClock {
  Ctx& c; int k; std::chrono::steady_clock::time_point t;
  PhaseClock(Ctx& c_, int k_) : c(c_), k(k_), t(std::chrono::steady_clock::now()) { if (c.host_phases) ++c.hp_n[k]; }
  void mark(int i) {
    if (!c.host_phases) return;
    auto n = std::chrono::steady_clock::now();
    c.hp_sum[k][i] += std::chrono::duration<double>(n - t).count();
    t = n;
  }
};

void pull_state(Ctx& c) {
  MSG_CUDA(cudaMemcpyAsync(c.hstate, c.dstate, sizeof(DevState), cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaStreamSynchronize(c.st));
}

static inline int grid_for(int64_t n, int threads, int max_blocks = 148 * 8) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

// Build the class table for windows `win` into c.s (seg arrays) and return
// (#segments upper bound, passes).  Also fills per-window page counts and the
// window-0 run arrays (used by the demand path).
struct WinBuild {
  int64_t total_iv = 0;
  int64_t scratch_total = 0;
  std::vector<int64_t> win_base;
};

// The cross-window class table for the general (non-fused) path: the
// 128-bit-key kernel, then the tuple-comparison kernel, which exits at once
// unless the first found the radices too wide (decided on the device; no
// host round trip).  M_ub bounds the total run count.
static void launch_combine(Ctx& c, CombineParams P, int64_t M_ub) {
  const int64_t mp = pow2_at_least(2 * std::max<int64_t>(M_ub, 1));
  c.s.wide.resize(3 * mp + 2, c.st);
  P.wide = reinterpret_cast<uint64_t*>(c.s.wide.p);
  int32_t* ok = reinterpret_cast<int32_t*>(c.s.wide.p + 3 * mp);
  win_kernels_init(c);
  k_window_combine_wide<<<1, 1024, kWideSmem, c.st>>>(P, kWideSmem, ok);
  k_window_combine<<<1, 1024, kWinSmem, c.st>>>(P, kWinSmem, ok);
  MSG_CHECK_LAUNCH();
  add_launches(2);
}

static bool build_windows(Ctx& c, const msg_window* win, int32_t nwin, WinBuild& wb, const RangeOut* dem = nullptr) {
  std::vector<WinDesc> wd(nwin);
  int64_t off = 0;
  for (int w = 0; w < nwin; ++w) {
    if (win[w].task < 0 || win[w].task >= (int32_t)c.tasks.size() || !c.tasks[win[w].task])
      throw Error(MSG_E_INVAL, "unknown task in window");
    TaskTab& t = *c.tasks[win[w].task];
    if (win[w].c0 < 0 || win[w].c1 < win[w].c0 || win[w].c1 > t.ncmd) throw Error(MSG_E_INVAL, "bad window range");
    wd[w].pool = t.pred_pool.p;
    wd[w].pool_lo = t.pred_off[win[w].c0];
    wd[w].pool_hi = t.pred_off[win[w].c1];
    wd[w].c0 = win[w].c0; wd[w].c1 = win[w].c1; wd[w].w = w;
    wd[w].cmd_off = t.d_pred_off.p;
    wd[w].selfpop = t.d_selfpop.p;
    wd[w].scratch = off;
    int64_t n = wd[w].pool_hi - wd[w].pool_lo;
    wb.total_iv += n;
    off += 4 * pow2_at_least(2 * std::max<int64_t>(n, 1)) + 16;
  }
  wb.scratch_total = off;
  cudaStream_t st = c.st;
  // scratch: keys/vals/labels per window + run arrays; combine scratch
  c.s.i64a.resize(off, st);                 // keys
  c.s.i64b.resize(off, st);                 // vals
  c.s.i32a.resize(off, st);                 // labels / run labels
  c.s.i64c.resize(3 * off + 4 * nwin + 8, st);   // run_a | run_b | run_d | run_base | nruns | pages
  int64_t* rbuf = c.s.i64c.p;
  WinOut o;
  o.run_a = rbuf; o.run_b = rbuf + off; o.run_d = rbuf + 2 * off;
  o.run_base = rbuf + 3 * off; o.nruns = o.run_base + nwin; o.pages = o.nruns + nwin;
  c.s.i32b.resize(off, st);
  o.run_lab = c.s.i32b.p;
  const bool fused = wb.total_iv <= FW_MAX_IV && nwin <= FW_MAX_WIN && (int64_t)c.span_first.size() <= FW_MAX_SPANS &&
                     !(c.fallback & 1);
  if (!fused) {
    // the window descriptors go through the Iv scratch buffer, sized in Iv units
    size_t need_iv = (nwin * sizeof(WinDesc) + sizeof(Iv) - 1) / sizeof(Iv);
    c.s.iv.resize(need_iv, st);
    MSG_CUDA(cudaMemcpyAsync(c.s.iv.p, wd.data(), nwin * sizeof(WinDesc), cudaMemcpyHostToDevice, st));
    win_kernels_init(c);
    k_window_runs<<<nwin, 1024, kWinSmem, st>>>(reinterpret_cast<const WinDesc*>(c.s.iv.p),
                                                c.s.i64a.p, c.s.i64b.p, c.s.i32a.p, o, kWinSmem);
    MSG_CHECK_LAUNCH();
    add_launches(1);
  }
  // combine scratch: key[mp] | val[mp] | E[2mp] | idx[2M] | seg_lo[2M] | seg_hi[2M] | nseg | ncls
  int64_t M = 2 * wb.total_iv + 2;    // >= total runs
  int64_t mp = pow2_at_least(2 * M);
  c.s.i64d.resize(4 * mp + 6 * M + 4, st);
  c.s.u32a.resize(2 * M * (int64_t)nwin + 16, st);
  c.s.i32c.resize(2 * M + 16, st);
  CombineParams P{};
  P.nwin = nwin;
  P.run_a = o.run_a; P.run_b = o.run_b; P.run_lab = o.run_lab; P.run_base = o.run_base; P.nruns = o.nruns;
  P.run_cls = nullptr;
  P.span_first = c.d_span_first.p; P.span_n = c.d_span_n.p; P.span_dense = c.d_span_dense.p;
  P.nspans = (int32_t)c.span_first.size();
  int64_t* d = c.s.i64d.p;
  P.key = reinterpret_cast<uint64_t*>(d);
  P.val = d + mp;
  P.E = d + 2 * mp;
  P.idx = d + 4 * mp;
  P.T = reinterpret_cast<int32_t*>(c.s.u32a.p);
  P.seg_lo = d + 4 * mp + 2 * M;
  P.seg_hi = P.seg_lo + 2 * M;
  P.seg_cls = c.s.i32c.p;
  P.nseg_out = P.seg_hi + 2 * M;
  P.ncls_out = P.nseg_out + 1;
  win_kernels_init(c);
  if (fused) {
    FusedWinParams F{};
    for (int w = 0; w < nwin; ++w) F.wd[w] = wd[w];
    F.nwin = nwin;
    F.out = o;
    F.span_first = c.d_span_first.p; F.span_dense = c.d_span_dense.p; F.nspans = (int32_t)c.span_first.size();
    F.seg_lo = P.seg_lo; F.seg_hi = P.seg_hi; F.seg_cls = P.seg_cls; F.nseg_out = P.nseg_out; F.ncls_out = P.ncls_out;
    if (dem && !(c.fallback & 4)) F.R = *dem; else F.R.nr = nullptr;
    // one element per thread in every phase: 2N endpoints bound them all
    int threads = 64;
    while (threads < 2 * wb.total_iv) threads <<= 1;
    k_windows_fused<<<1, threads, sizeof(FwSmem), st>>>(F);
    MSG_CHECK_LAUNCH();
    add_launches(1);
    return F.R.nr != nullptr;
  }
  launch_combine(c, P, M);
  return false;
}

// pointers into the build outputs (must mirror build_windows)
struct WinPtrs {
  int64_t *run_a, *run_b, *run_base, *nruns, *pages;
  int32_t* run_lab;
  SegTab tab;
  int64_t* ncls;
};

static WinPtrs win_ptrs(Ctx& c, int32_t nwin, const WinBuild& wb) {
  WinPtrs p{};
  int64_t off = wb.scratch_total;
  int64_t* rbuf = c.s.i64c.p;
  p.run_a = rbuf; p.run_b = rbuf + off; p.run_base = rbuf + 3 * off; p.nruns = p.run_base + nwin;
  p.pages = p.nruns + nwin; p.run_lab = c.s.i32b.p;
  int64_t M = 2 * wb.total_iv + 2;
  int64_t mp = pow2_at_least(2 * M);
  int64_t* d = c.s.i64d.p;
  int64_t* seg_lo = d + 4 * mp + 2 * M;
  int64_t* seg_hi = seg_lo + 2 * M;
  p.tab.lo = seg_lo; p.tab.hi = seg_hi; p.tab.cls = c.s.i32c.p;
  p.tab.n = seg_hi + 2 * M;
  p.tab.cap = 2 * M;
  p.ncls = seg_hi + 2 * M + 1;
  return p;
}

static int passes_for(int64_t ncls) {
  int p = 0;
  while (ncls > 0) { ++p; ncls >>= 8; }
  return p;
}

static void compact_if_needed(Ctx& c) {
  // invariant for appends without a preceding multisplit: head <= C
  if (c.head > c.C) {
    MSG_CUDA(cudaMemcpyAsync(c.order[c.cur ^ 1].p, c.order[c.cur].p + c.head, c.len * sizeof(int32_t),
                             cudaMemcpyDeviceToDevice, c.st));
    c.cur ^= 1;
    c.head = 0;
  }
}

static int64_t* mig_buf(Ctx& c, int64_t n) {
  c.batch_old_free = c.fifo_len;
  if (!(c.cfg.flags & MSG_F_MIGRATE) && !(c.cfg.flags & MSG_F_VERIFY_TAGS)) return nullptr;
  // reset this batch's dependency maxima (DevState aux[0] holds two int32)
  MSG_CUDA(cudaMemsetAsync(&c.dstate->aux[0], 0xff, sizeof(int64_t), c.st));
  int par = c.mig_par;
  // the copy work that last used this buffer must be finished
  MSG_CUDA(cudaStreamWaitEvent(c.st, c.ev_mig[par], 0));
  c.mig_list[par].resize(std::max<int64_t>(n, 1), c.st);
  return c.mig_list[par].p;
}

// evict `n` pages from the head; pushes frames; fills mig[0..n)
static Epochs epochs(Ctx& c, int64_t* mig) {
  Epochs e{nullptr, nullptr, c.mig_batch, nullptr};
  if (mig && (c.cfg.flags & MSG_F_MIGRATE)) {
    e.inst_ep = c.inst_ep.p;
    e.free_ep = c.free_ep.p;
    e.dep = reinterpret_cast<int*>(&c.dstate->aux[0]);
  }
  return e;
}

static void evict_head_n(Ctx& c, int64_t n, int64_t* mig) {
  c.batch_old_free = c.fifo_len;   // frames already free before this batch's evictions
  if (n <= 0) return;
  // executed commands read frames through the frame table: evictions (which
  // unmap frames) come after every command executed so far, as the fault
  // handler of a later command runs after the earlier ones finished
  if (c.run_used) MSG_CUDA(cudaStreamWaitEvent(c.st, c.ev_run_last, 0));
  k_evict_head<<<grid_for(n, 256), 256, 0, c.st>>>(c.order[c.cur].p + c.head, n, c.bits.p, c.frame.p, c.fifo.p,
                                                  c.fifo_head + c.fifo_len, c.C, mig, epochs(c, mig));
  MSG_CHECK_LAUNCH();
  add_launches(1);
  c.head += n;
  c.len -= n;
  c.fifo_len += n;
}

// install `n` pages (device list) at the tail
static void install_pages(Ctx& c, const int32_t* pages, int64_t n, int64_t* mig) {
  if (n <= 0) return;
  // remapping frames also waits for the commands executed so far (see evict_head_n)
  if (c.run_used) MSG_CUDA(cudaStreamWaitEvent(c.st, c.ev_run_last, 0));
  k_install<<<grid_for(n, 256), 256, 0, c.st>>>(pages, nullptr, n, c.bits.p, c.frame.p, c.fifo.p, c.fifo_head, c.C,
                                               c.order[c.cur].p + c.head + c.len, mig, epochs(c, mig),
                                               c.batch_old_free);
  MSG_CHECK_LAUNCH();
  add_launches(1);
  c.fifo_head = (c.fifo_head + n) % c.C;
  c.fifo_len -= n;
  c.len += n;
}

static int64_t abs_of(const Ctx& c, int64_t d) {
  auto it = std::upper_bound(c.span_dense.begin(), c.span_dense.end(), d);
  int64_t s = (it - c.span_dense.begin()) - 1;
  return c.span_first[s] + (d - c.span_dense[s]);
}

static void dump_dense(Ctx& c, const int32_t* dev, int64_t n, std::vector<int64_t>& out) {
  std::vector<int32_t> h(n);
  if (n) MSG_CUDA(cudaMemcpyAsync(h.data(), dev, n * 4, cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaStreamSynchronize(c.st));
  out.resize(n);
  for (int64_t i = 0; i < n; ++i) out[i] = abs_of(c, h[i]);
}

void list_reorder(Ctx& c, const int64_t* first, const int64_t* end, const int32_t* win, int32_t n, int32_t nwin,
                  int64_t* win_pages) {
  if (nwin <= 0) return;
  // per-window runs in the given (first-access) order; class = K_w - rank
  std::vector<std::vector<std::pair<int64_t, int64_t>>> per(nwin);
  for (int i = 0; i < n; ++i) {
    if (win[i] < 0 || win[i] >= nwin) throw Error(MSG_E_INVAL, "bad window index");
    if (end[i] > first[i]) per[win[i]].push_back({first[i], end[i]});
  }
  std::vector<int64_t> ra, rb, nr(nwin), base(nwin);
  std::vector<int32_t> rc;
  for (int w = 0; w < nwin; ++w) {
    base[w] = (int64_t)ra.size();
    int64_t K = (int64_t)per[w].size();
    win_pages[w] = 0;
    for (int64_t r = 0; r < K; ++r) {
      int64_t a = per[w][r].first, b = per[w][r].second;
      win_pages[w] += b - a;
      // clip to the domain (pages outside it are never resident)
      while (a < b) {
        auto it = std::upper_bound(c.span_first.begin(), c.span_first.end(), a);
        int64_t s = (it - c.span_first.begin()) - 1;
        if (s < 0 || a >= c.span_first[s] + c.span_n[s]) {
          if ((size_t)(s + 1) >= c.span_first.size() || c.span_first[s + 1] >= b) break;
          a = c.span_first[s + 1];
          continue;
        }
        int64_t e = std::min(b, c.span_first[s] + c.span_n[s]);
        ra.push_back(a); rb.push_back(e); rc.push_back((int32_t)(K - r));
        a = e;
      }
    }
    nr[w] = (int64_t)ra.size() - base[w];
  }
  int64_t M = std::max<int64_t>((int64_t)ra.size(), 1);
  cudaStream_t st = c.st;
  c.s.i64c.resize(3 * M + 2 * nwin + 8, st);
  c.s.i32b.resize(M, st);
  int64_t* rbuf = c.s.i64c.p;
  if (!ra.empty()) {
    MSG_CUDA(cudaMemcpyAsync(rbuf, ra.data(), ra.size() * 8, cudaMemcpyHostToDevice, st));
    MSG_CUDA(cudaMemcpyAsync(rbuf + M, rb.data(), rb.size() * 8, cudaMemcpyHostToDevice, st));
    MSG_CUDA(cudaMemcpyAsync(c.s.i32b.p, rc.data(), rc.size() * 4, cudaMemcpyHostToDevice, st));
  }
  MSG_CUDA(cudaMemcpyAsync(rbuf + 3 * M, base.data(), nwin * 8, cudaMemcpyHostToDevice, st));
  MSG_CUDA(cudaMemcpyAsync(rbuf + 3 * M + nwin, nr.data(), nwin * 8, cudaMemcpyHostToDevice, st));
  int64_t Mb = (int64_t)ra.size() + 2;
  int64_t mp = pow2_at_least(2 * Mb);
  c.s.i64d.resize(4 * mp + 6 * Mb + 4, st);
  c.s.u32a.resize(2 * Mb * (int64_t)nwin + 16, st);
  c.s.i32c.resize(2 * Mb + 16, st);
  CombineParams P{};
  P.nwin = nwin;
  P.run_a = rbuf; P.run_b = rbuf + M; P.run_lab = nullptr; P.run_base = rbuf + 3 * M; P.nruns = rbuf + 3 * M + nwin;
  P.run_cls = c.s.i32b.p;
  P.span_first = c.d_span_first.p; P.span_n = c.d_span_n.p; P.span_dense = c.d_span_dense.p;
  P.nspans = (int32_t)c.span_first.size();
  int64_t* d = c.s.i64d.p;
  P.key = reinterpret_cast<uint64_t*>(d);
  P.val = d + mp;
  P.E = d + 2 * mp;
  P.idx = d + 4 * mp;
  P.T = reinterpret_cast<int32_t*>(c.s.u32a.p);
  P.seg_lo = d + 4 * mp + 2 * Mb;
  P.seg_hi = P.seg_lo + 2 * Mb;
  P.seg_cls = c.s.i32c.p;
  P.nseg_out = P.seg_hi + 2 * Mb;
  P.ncls_out = P.nseg_out + 1;
  launch_combine(c, P, Mb);
  MSG_CUDA(cudaMemcpyAsync(c.hbuf.p, P.ncls_out, 8, cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaStreamSynchronize(st));
  SegTab T{P.seg_lo, P.seg_hi, P.seg_cls, P.nseg_out, 2 * Mb};
  multisplit(c, T, passes_for(c.hbuf.p[0]));
  MSG_CUDA(cudaStreamSynchronize(st));
}

// per-command missing counts of the actual sets of commands [lo, hi) of t
// (K8, engine.py:396-397); result in c.s.tc on the device
static void touch_counts(Ctx& c, TaskTab& t, int32_t lo, int32_t hi) {
  int32_t n = hi - lo;
  c.s.tc.resize(std::max(n, 1), c.st);
  touch_counts_dev(c, t, lo, hi, c.s.tc.p);
}

void plan_switch(Ctx& c, const msg_window* win, int32_t nwin, bool reorder_always, msg_switch_out* out,
                 int64_t* win_pages, int64_t* prefix, int64_t* touch_cnt) {
  if (nwin < 1) throw Error(MSG_E_INVAL, "need at least one window");
  PhaseClock pc(c, 0);
  fold_events(c, c.event_bound);
  cudaStream_t st = c.st;
  // the call's planner-time pair: created once per context (an event create
  // and destroy per call cost more host time than the pair's two records)
  for (auto& e : c.ev_call)
    if (!e) MSG_CUDA(cudaEventCreate(&e));
  cudaEvent_t e0 = c.ev_call[0], e1 = c.ev_call[1];
  MSG_CUDA(cudaEventRecord(e0, st));
  TaskTab& t0 = *c.tasks[win[0].task];
  int32_t c0 = win[0].c0, c1 = win[0].c1, ncw = c1 - c0;
  c.hbuf.reserve(4 * (int64_t)nwin + 3 * (int64_t)ncw + 64);
  // ---- phase A: windows, class table, window-0 demand vs residency
  int64_t niv0 = t0.pred_off[c1] - t0.pred_off[c0];
  int64_t nrun_cap = std::max<int64_t>(2 * niv0 + 2, 2);
  int64_t units_cap = t0.pred_units[c1] - t0.pred_units[c0] + 2 * nrun_cap + 2;
  c.s.rdem.reserve(nrun_cap, st);
  RangeOut dem_out = c.s.rdem.out();
  WinBuild wb;
  const bool dem_done = build_windows(c, win, nwin, wb, &dem_out);
  pc.mark(0);   // window launch (host)
  WinPtrs wp = win_ptrs(c, nwin, wb);
  c.s.uscr.resize(512 + ncw, st);
  int64_t* pref_d = c.s.uscr.p + 512;   // per-command gating counts
  int64_t* total_d = c.s.uscr.p + 400;
  // populate list (pre-apply residency, first-access order, capacity-capped)
  DVec<int32_t>& poplist = c.s.poplist;
  poplist.resize(std::max<int64_t>(std::min<int64_t>(32 * units_cap, c.C), 1), st);
  DemandParams D{};
  D.run_a = wp.run_a; D.run_b = wp.run_b; D.run_lab = wp.run_lab;
  D.run_base = 0;  // window 0's scratch region starts at offset 0
  D.nruns = wp.nruns;
  D.selfpop = t0.d_selfpop.p; D.c0 = c0;
  D.span_first = c.d_span_first.p; D.span_n = c.d_span_n.p; D.span_dense = c.d_span_dense.p;
  D.nspans = (int32_t)c.span_first.size();
  D.R = c.s.rdem.out();
  RangeSet R = c.s.rdem.set();
  if (!dem_done) {
    k_demand_collect<<<1, 1024, 0, st>>>(D);
    MSG_CHECK_LAUNCH();
    add_launches(1);
  }
  // ---- async path: plain replays (no copies, no executed commands, no
  // debug dumps) run the plan, the multisplit (its pass count decided on the
  // device) and the apply as one cooperative launch behind the window
  // kernel, and the host syncs once, at the end
  const bool async = !(c.cfg.flags & (MSG_F_MIGRATE | MSG_F_VERIFY_TAGS | MSG_F_EXECUTE)) && !c.debug &&
                     ms_coop_fits(c, sw_grid(c));
  // missing = demand - resident, gating counts, plan scalars, populate list
  if (!async) units_plan(c, R, units_cap, ncw ? pref_d : nullptr, ncw, c.C, poplist.p, c.C, total_d);
  pc.mark(1);   // plan launch (host)
  int64_t* hb = c.hbuf.p;
  if (async) {
    compact_if_needed(c);
    const int64_t len0 = c.len, head0 = c.head, fifo_head0 = c.fifo_head, fifo_len0 = c.fifo_len;
    const int cur0 = c.cur;
    int64_t* passes_d = &c.dstate->aux[2];
    const int G = sw_grid(c);
    int32_t* bar = next_barrier(c);
    SwitchArgs SA{};
    // (the plan phase zeroes the pass-count slot with the plan scalars)
    SA.up = units_plan_args(c, R, G, ncw ? pref_d : nullptr, ncw, c.C, poplist.p, c.C, total_d, bar);
    SA.has_up = 1;
    SA.has_ms = len0 > 0 &&
                ms_args(c, wp.tab, 0, DevPasses{wp.ncls, &c.dstate->missing, reorder_always ? 1 : 0, passes_d}, G,
                        bar, SA.ms);
    pc.mark(3);
    const ListSel L{c.order[cur0].p, c.order[cur0 ^ 1].p, head0, passes_d};
    // evict, install, the slice's touch scan and the result gather: one launch
    // (results: win pages | prefix | touch counts | DevState)
    constexpr int kStateWords = (int)(sizeof(DevState) / sizeof(int64_t));
    static_assert(sizeof(DevState) % sizeof(int64_t) == 0, "DevState packs as 64-bit words");
    c.s.tc.resize(std::max(ncw, 1), st);
    ApplyArgs AA{};
    AA.L = L; AA.S = c.dstate; AA.len0 = len0;
    AA.bits = c.bits.p; AA.frame = c.frame.p; AA.fifo = c.fifo.p;
    AA.fifo_tail = fifo_head0 + fifo_len0; AA.fifo_head = fifo_head0; AA.C = c.C;
    AA.pages = poplist.p;
    AA.act_pool = t0.act_pool.p; AA.act_off = t0.d_act_off.p; AA.tc_c0 = c0; AA.tc_n = ncw;
    AA.tc = reinterpret_cast<unsigned long long*>(c.s.tc.p);
    AA.pack.seg[AA.pack.nseg++] = PackSeg{wp.pages, nwin, 0};
    if (ncw) {
      AA.pack.seg[AA.pack.nseg++] = PackSeg{pref_d, ncw, nwin};
      AA.pack.seg[AA.pack.nseg++] = PackSeg{c.s.tc.p, ncw, nwin + ncw};
    }
    AA.pack.seg[AA.pack.nseg++] = PackSeg{reinterpret_cast<const int64_t*>(c.dstate), kStateWords, nwin + 2 * ncw};
    AA.bar = bar;
    SA.ap = AA;
    switch_launch(c, SA);
    pc.mark(4);
    MSG_CUDA(cudaEventRecord(e1, st));
    pc.mark(6);
    MSG_CUDA(cudaStreamSynchronize(st));
    pc.mark(7);
    const DevState S = *reinterpret_cast<const DevState*>(hb + nwin + 2 * ncw);
    for (int w = 0; w < nwin; ++w) win_pages[w] = hb[w];
    for (int k = 0; k < ncw; ++k) prefix[k] = hb[nwin + k];
    out->missing = S.missing;
    out->nwin = nwin;
    out->early_exit = S.missing == 0 && !reorder_always;
    c.switch_base = c.installed_total;
    c.fault_task = -1;
    out->populate = out->evict = out->truncated = 0;
    const int64_t passes = S.aux[2];
    if (passes > 0) {   // ms_coop_done
      c.cur ^= (int)(passes & 1);
      c.head = 0;
      c.ms_tot_par ^= (int)(passes & 1);
      c.stats.ms_passes += passes;
      c.stats.ms_bytes += 8 * len0 * passes;
    }
    out->free_before = c.C - c.len;
    if (!out->early_exit) {
      const int64_t pop = S.populate, ev = S.evict;
      out->populate = pop; out->evict = ev; out->truncated = S.truncated;
      if (pop > c.C - len0 + ev) throw Error(MSG_E_CAPACITY, "migration plan overflowed HBM capacity");
      c.batch_old_free = c.fifo_len;
      c.head += ev; c.len -= ev; c.fifo_len += ev;                          // evict_head_n
      c.fifo_head = (c.fifo_head + pop) % c.C; c.fifo_len -= pop; c.len += pop;   // install_pages
    }
    out->first_missing = -1;
    out->first_missing_pages = 0;
    for (int k = 0; k < ncw; ++k) {
      touch_cnt[k] = hb[nwin + ncw + k];
      if (touch_cnt[k] && out->first_missing < 0) { out->first_missing = c0 + k; out->first_missing_pages = touch_cnt[k]; }
    }
    c.gate_task = -1;
    c.gate_c0 = c0;
    c.gate_need.clear();
    out->resident_after = c.len;
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    c.stats.plan_ms += ms;
    return;
  }
  // the reorder is queued behind the plan before the host round trip, its
  // pass count read on the device (0 on an early exit), so it starts on a
  // busy stream instead of after the host's launch latency
  const bool pre_ms = !c.debug && c.len > 0 && ms_coop_fits(c) &&
                      ms_coop_launch(c, wp.tab, 0, DevPasses{wp.ncls, &c.dstate->missing, reorder_always ? 1 : 0,
                                                             &c.dstate->aux[2]});
  MSG_CUDA(cudaMemcpyAsync(c.hstate, c.dstate, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaMemcpyAsync(hb, wp.pages, nwin * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaMemcpyAsync(hb + nwin, wp.ncls, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (ncw) MSG_CUDA(cudaMemcpyAsync(hb + nwin + 1, pref_d, ncw * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaStreamSynchronize(st));
  pc.mark(2);   // first sync (device phase A)
  DevState S = hs(c);
  if (pre_ms) ms_coop_done(c, (int)S.aux[2]);   // (before any error below: the list is reordered)
  for (int w = 0; w < nwin; ++w) win_pages[w] = hb[w];
  for (int k = 0; k < ncw; ++k) prefix[k] = hb[nwin + 1 + k];
  int64_t ncls = hb[nwin];
  out->missing = S.missing;
  out->nwin = nwin;
  out->early_exit = S.missing == 0 && !reorder_always;
  c.switch_base = c.installed_total;
  c.fault_task = -1;
  out->free_before = c.C - c.len;
  out->populate = out->evict = out->truncated = 0;
  // ---- phase B: reorder (multisplit), plan, apply, migrate
  if (!out->early_exit) {
    int64_t pop = S.populate, ev = S.evict;
    out->populate = pop; out->evict = ev; out->truncated = S.truncated;
    if (pop > c.C - c.len + ev) throw Error(MSG_E_CAPACITY, "migration plan overflowed HBM capacity");
    if (!pre_ms) multisplit(c, wp.tab, passes_for(ncls));
    pc.mark(3);   // multisplit launch (host)
    if (c.debug & 2) dump_dense(c, c.order[c.cur].p + c.head, c.len, c.dbg[0]);
    out->free_before = c.C - c.len;
    int64_t* mig = mig_buf(c, ev + pop);
    c.switch_base = c.installed_total;   // executed commands gate on this switch's populate
    c.fault_task = -1;
    if (c.debug & 3) {
      dump_dense(c, c.order[c.cur].p + c.head, ev, c.dbg[1]);
      dump_dense(c, poplist.p, pop, c.dbg[2]);
    }
    evict_head_n(c, ev, mig);
    compact_if_needed(c);
    install_pages(c, poplist.p, pop, mig ? mig + ev : nullptr);
    pc.mark(4);   // apply launches (host)
    if (mig) migrate_batch(c, ev, pop, out->free_before, true);
    pc.mark(5);   // migration issue (host, incl. its segment sync)
  }
  // ---- MSG_F_EXECUTE: what each command of the slice physically needs landed
  const bool gates = (c.cfg.flags & MSG_F_EXECUTE) && ncw > 0;
  if (gates) {
    if ((int64_t)c.pos_of.n < c.D) {
      c.pos_of.exact(std::max<int64_t>(c.D, 1));
      MSG_CUDA(cudaMemsetAsync(c.pos_of.p, 0xff, c.pos_of.n * 8, st));
    }
    ++c.switch_tag;
    c.s.tb.resize(ncw, st);
    unsigned long long* need = reinterpret_cast<unsigned long long*>(c.s.tb.p);
    MSG_CUDA(cudaMemsetAsync(need, 0, ncw * 8, st));
    if (!out->early_exit && out->populate) {
      k_pos_scatter<<<grid_for(out->populate, 256), 256, 0, st>>>(c.s.poplist.p, out->populate, c.switch_tag,
                                                                 c.pos_of.p);
      int64_t niv = t0.act_off[c1] - t0.act_off[c0];
      if (niv)
        k_gate_need<<<grid_for(32 * niv, 256), 256, 0, st>>>(t0.act_pool.p, t0.d_act_off.p, c0, c1, c.pos_of.p,
                                                            c.switch_tag, need);
      MSG_CHECK_LAUNCH();
      add_launches(2);
    }
    MSG_CUDA(cudaMemcpyAsync(hb + ncw, need, ncw * 8, cudaMemcpyDeviceToHost, st));
  }
  // ---- K8 touch scan of the slice (post-apply residency)
  touch_counts(c, t0, c0, c1);
  if (ncw) MSG_CUDA(cudaMemcpyAsync(hb, c.s.tc.p, ncw * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaEventRecord(e1, st));
  pc.mark(6);   // gates + touch scan launches (host)
  MSG_CUDA(cudaStreamSynchronize(st));
  pc.mark(7);   // final sync (device phase B)
  out->first_missing = -1;
  out->first_missing_pages = 0;
  for (int k = 0; k < ncw; ++k) {
    touch_cnt[k] = hb[k];
    if (hb[k] && out->first_missing < 0) { out->first_missing = c0 + k; out->first_missing_pages = hb[k]; }
  }
  c.gate_task = gates ? win[0].task : -1;
  c.gate_c0 = c0;
  c.gate_need.assign(gates ? hb + ncw : hb, gates ? hb + 2 * ncw : hb);
  out->resident_after = c.len;
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  c.stats.plan_ms += ms;
}

void touch_slow(Ctx& c, int32_t task, int32_t cmd, int64_t evict, const msg_window* win, int32_t nwin,
                int32_t scan_end, bool write_tags, msg_touch_out* out, int64_t* win_pages) {
  PhaseClock pc(c, 1);
  fold_events(c, c.event_bound);
  if (task < 0 || task >= (int32_t)c.tasks.size() || !c.tasks[task]) throw Error(MSG_E_INVAL, "unknown task");
  TaskTab& t = *c.tasks[task];
  if (cmd < 0 || cmd >= t.ncmd || scan_end > t.ncmd) throw Error(MSG_E_INVAL, "bad command index");
  cudaStream_t st = c.st;
  c.hbuf.reserve(4 * (int64_t)nwin + (scan_end - cmd) + 64);
  // One host round trip for both the missing count of cmd (against current
  // residency, before any eviction) and, when a refresh reorder follows, the
  // window class table; then the missing list is filled while the host
  // launches the reorder, so the multisplit starts on a busy stream.
  const bool has_iv = t.act_off[cmd + 1] != t.act_off[cmd];
  const bool refresh = evict > 0 && nwin > 0;
  // the async path gathers its results with one launch at the end
  const bool async = !(c.cfg.flags & (MSG_F_MIGRATE | MSG_F_VERIFY_TAGS | MSG_F_EXECUTE)) && !c.debug &&
                     ms_coop_fits(c, sw_grid(c));
  RangeSet R{};
  int64_t* hb = c.hbuf.p;
  if (has_iv) {
    int64_t nu = t.act_units[cmd + 1] - t.act_units[cmd];
    ranges_from_actual(c, t, cmd, cmd + 1, c.s.ract);
    c.s.uscr.resize(512, st);
    c.s.miss.resize(std::max<int64_t>(32 * nu, 1), st);
    R = c.s.ract.set();
    if (!async) {   // (the async path runs the plan inside its cooperative launch)
      units_plan(c, R, nu, nullptr, 0, -1, c.s.miss.p, -1, c.s.uscr.p + 400);
      MSG_CUDA(cudaMemcpyAsync(hb, c.s.uscr.p + 400, 8, cudaMemcpyDeviceToHost, st));
    }
  }
  WinBuild wb;
  WinPtrs wp{};
  bool pre_ms = false;   // synchronous path: the refresh reorder queued before the host round trip
  if (refresh) {
    build_windows(c, win, nwin, wb);
    wp = win_ptrs(c, nwin, wb);
    if (!async) {
      if (!c.debug && c.len > 0 && ms_coop_fits(c)) {
        MSG_CUDA(cudaMemsetAsync(&c.dstate->aux[2], 0, sizeof(int64_t), st));
        pre_ms = ms_coop_launch(c, wp.tab, 0, DevPasses{wp.ncls, nullptr, 0, &c.dstate->aux[2]});
        if (pre_ms) MSG_CUDA(cudaMemcpyAsync(hb + 2 + nwin, &c.dstate->aux[2], 8, cudaMemcpyDeviceToHost, st));
      }
      MSG_CUDA(cudaMemcpyAsync(hb + 1, wp.pages, nwin * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      MSG_CUDA(cudaMemcpyAsync(hb + 1 + nwin, wp.ncls, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    }
  }
  pc.mark(0);   // missing-set + window launches (host)
  // ---- async path (see plan_switch): refresh, evict and install follow on
  // the device with counts read there; one host sync at the end
  if (async) {
    compact_if_needed(c);
    const int64_t len0 = c.len, head0 = c.head, fifo_head0 = c.fifo_head, fifo_len0 = c.fifo_len;
    const int cur0 = c.cur;
    int64_t* passes_d = &c.dstate->aux[2];   // published by the multisplit phase (none: read as 0)
    const int G = sw_grid(c);
    int32_t* bar = next_barrier(c);
    SwitchArgs SA{};
    // the command's missing list (plan phase), the refresh multisplit, then
    // evict, install, the rescan and the result gather: one launch
    // (results: n | win pages | ncls slot (unused) | passes | touch counts)
    if (has_iv) SA.up = units_plan_args(c, R, G, nullptr, 0, -1, c.s.miss.p, -1, c.s.uscr.p + 400, bar);
    SA.has_up = has_iv ? 1 : 0;
    SA.has_ms = evict > 0 && refresh && len0 > 0 &&
                ms_args(c, wp.tab, 0, DevPasses{wp.ncls, nullptr, 0, passes_d}, G, bar, SA.ms);
    const ListSel L{c.order[cur0].p, c.order[cur0 ^ 1].p, head0, SA.has_ms ? passes_d : nullptr};
    const int64_t ev_done = evict > 0 ? std::min(evict, len0) : 0;
    const int32_t lo = cmd + 1, hi = scan_end;
    c.s.tc.resize(std::max(hi - lo, 1), st);
    ApplyArgs AA{};
    AA.L = L; AA.S = nullptr; AA.ev_host = ev_done; AA.np_dev = has_iv ? c.s.uscr.p + 400 : nullptr; AA.len0 = len0;
    AA.bits = c.bits.p; AA.frame = c.frame.p; AA.fifo = c.fifo.p;
    AA.fifo_tail = fifo_head0 + fifo_len0; AA.fifo_head = fifo_head0; AA.C = c.C;
    AA.pages = c.s.miss.p;
    AA.act_pool = t.act_pool.p; AA.act_off = t.d_act_off.p; AA.tc_c0 = lo; AA.tc_n = std::max(hi - lo, 0);
    AA.tc = reinterpret_cast<unsigned long long*>(c.s.tc.p);
    if (has_iv) AA.pack.seg[AA.pack.nseg++] = PackSeg{c.s.uscr.p + 400, 1, 0};
    if (refresh) AA.pack.seg[AA.pack.nseg++] = PackSeg{wp.pages, nwin, 1};
    if (SA.has_ms) AA.pack.seg[AA.pack.nseg++] = PackSeg{passes_d, 1, 2 + nwin};
    if (hi > lo) AA.pack.seg[AA.pack.nseg++] = PackSeg{c.s.tc.p, hi - lo, 3 + nwin};
    AA.bar = bar;
    SA.ap = AA;
    switch_launch(c, SA);
    pc.mark(5);
    MSG_CUDA(cudaStreamSynchronize(st));
    pc.mark(6);
    const int64_t n = has_iv ? hb[0] : 0;
    if (refresh)
      for (int w = 0; w < nwin; ++w) win_pages[w] = hb[1 + w];
    out->missing = n;
    out->refreshed = evict > 0 && refresh ? 1 : 0;
    out->evicted = ev_done;
    const int64_t passes = SA.has_ms ? hb[2 + nwin] : 0;
    if (passes > 0) {   // ms_coop_done
      c.cur ^= (int)(passes & 1);
      c.head = 0;
      c.ms_tot_par ^= (int)(passes & 1);
      c.stats.ms_passes += passes;
      c.stats.ms_bytes += 8 * len0 * passes;
    }
    c.batch_old_free = c.fifo_len;
    c.head += ev_done; c.len -= ev_done; c.fifo_len += ev_done;                  // evict_head_n
    c.fifo_head = (c.fifo_head + n) % c.C; c.fifo_len -= n; c.len += n;          // install_pages
    if (n) { c.fault_task = task; c.fault_cmd = cmd; c.fault_total = c.installed_total; }
    out->resident_after = c.len;
    out->next_missing = -1;
    out->next_missing_pages = 0;
    for (int k = 0; k < hi - lo; ++k)
      if (hb[3 + nwin + k]) { out->next_missing = lo + k; out->next_missing_pages = hb[3 + nwin + k]; break; }
    return;
  }
  if (has_iv || refresh) MSG_CUDA(cudaStreamSynchronize(st));
  pc.mark(1);   // first sync
  const int64_t n = has_iv ? hb[0] : 0;
  const int64_t ncls = refresh ? hb[1 + nwin] : 0;
  if (refresh)
    for (int w = 0; w < nwin; ++w) win_pages[w] = hb[1 + w];
  out->missing = n;
  out->refreshed = 0;
  out->evicted = 0;
  int64_t* mig = mig_buf(c, std::max<int64_t>(evict, 0) + n);
  // frames free BEFORE this batch's evictions: installs beyond them reuse
  // frames this batch evicts and must wait for those copies back to the host
  const int64_t free_before = c.C - c.len;
  int64_t ev_done = 0;
  if (evict > 0) {
    if (refresh) {
      if (pre_ms) ms_coop_done(c, (int)hb[2 + nwin]);
      else multisplit(c, wp.tab, passes_for(ncls));
      out->refreshed = 1;
      if (c.debug & 2) dump_dense(c, c.order[c.cur].p + c.head, c.len, c.dbg[0]);
    }
    ev_done = std::min(evict, c.len);
    if (c.debug & 3) dump_dense(c, c.order[c.cur].p + c.head, ev_done, c.dbg[1]);
    evict_head_n(c, ev_done, mig);
    out->evicted = ev_done;
  }
  if (c.debug & 3) {
    if (evict <= 0) c.dbg[1].clear();
    dump_dense(c, c.s.miss.p, n, c.dbg[2]);
  }
  pc.mark(2);   // multisplit + evict launches (host)
  compact_if_needed(c);
  install_pages(c, c.s.miss.p, n, mig ? mig + ev_done : nullptr);
  pc.mark(3);   // install launch (host)
  if (mig) migrate_batch(c, ev_done, n, free_before, !write_tags);
  pc.mark(4);
  if (n) { c.fault_task = task; c.fault_cmd = cmd; c.fault_total = c.installed_total; }
  out->resident_after = c.len;
  // rescan (cmd, scan_end)
  out->next_missing = -1;
  out->next_missing_pages = 0;
  int32_t lo = cmd + 1, hi = scan_end;
  if (hi > lo) {
    touch_counts(c, t, lo, hi);
    MSG_CUDA(cudaMemcpyAsync(c.hbuf.p, c.s.tc.p, (hi - lo) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    pc.mark(5);
    MSG_CUDA(cudaStreamSynchronize(st));
    pc.mark(6);   // final sync
    for (int k = 0; k < hi - lo; ++k)
      if (c.hbuf.p[k]) { out->next_missing = lo + k; out->next_missing_pages = c.hbuf.p[k]; break; }
  } else {
    pc.mark(5);
    MSG_CUDA(cudaStreamSynchronize(st));
    pc.mark(6);
  }
}

// madvise / remove with an explicit dense range table (class 1 = member)
static void split_by_ranges(Ctx& c, const std::vector<int64_t>& lo, const std::vector<int64_t>& len) {
  int64_t n = (int64_t)lo.size();
  DVec<int64_t>& tb = c.s.tb;
  DVec<int32_t>& tcls = c.s.tcls;
  tb.resize(4 * n + 4, c.st);
  tcls.resize(n + 1, c.st);
  if (n) {
    MSG_CUDA(cudaMemcpyAsync(tb.p, lo.data(), n * 8, cudaMemcpyHostToDevice, c.st));
    MSG_CUDA(cudaMemcpyAsync(tb.p + n, len.data(), n * 8, cudaMemcpyHostToDevice, c.st));
  }
  k_table_from_ranges<<<grid_for(n, 256), 256, 0, c.st>>>(tb.p, tb.p + n, n, tb.p + 2 * n, tb.p + 3 * n, tcls.p,
                                                         tb.p + 4 * n);
  MSG_CHECK_LAUNCH();
  add_launches(1);
  SegTab T{tb.p + 2 * n, tb.p + 3 * n, tcls.p, tb.p + 4 * n};
  multisplit(c, T, 1);
}

// sort + merge absolute runs, convert to dense ranges (host side, small inputs)
static void dense_ranges(Ctx& c, const int64_t* first, const int64_t* end, int32_t n, std::vector<int64_t>& lo,
                         std::vector<int64_t>& len, bool strict) {
  std::vector<std::pair<int64_t, int64_t>> r;
  for (int i = 0; i < n; ++i)
    if (end[i] > first[i]) r.push_back({first[i], end[i]});
  std::sort(r.begin(), r.end());
  std::vector<std::pair<int64_t, int64_t>> m;
  for (auto& x : r) {
    if (!m.empty() && x.first <= m.back().second) m.back().second = std::max(m.back().second, x.second);
    else m.push_back(x);
  }
  // clip to spans (pages outside the domain can never be resident)
  for (auto& x : m) {
    int64_t a = x.first;
    while (a < x.second) {
      auto it = std::upper_bound(c.span_first.begin(), c.span_first.end(), a);
      int64_t s = (it - c.span_first.begin()) - 1;
      if (s < 0 || a >= c.span_first[s] + c.span_n[s]) {
        if (strict) throw Error(MSG_E_DOMAIN, "page outside the dense page map");
        // skip to next span start
        if ((size_t)(s + 1) >= c.span_first.size()) break;
        a = std::max(a + 1, c.span_first[s + 1]);
        continue;
      }
      int64_t b = std::min(x.second, c.span_first[s] + c.span_n[s]);
      lo.push_back(c.span_dense[s] + (a - c.span_first[s]));
      len.push_back(b - a);
      a = b;
    }
  }
}

__global__ void k_release_pages(const int32_t* pages, int64_t n, uint32_t* bits, int32_t* frame, int32_t* fifo,
                                int64_t fifo_tail, int64_t C) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t p = pages[e];
    atomicAnd(&bits[p >> 5], ~(1u << (p & 31)));
    fifo[(fifo_tail + e) % C] = frame[p];
    frame[p] = -1;
  }
}

// resident pages of a few (possibly huge) dense ranges: one thread per
// 32-page bitmap word across all ranges, so a task span of millions of pages
// is not walked by one warp
__global__ void k_count_resident(const int64_t* __restrict__ lo, const int64_t* __restrict__ len,
                                 const int64_t* __restrict__ woff, int64_t n, const uint32_t* __restrict__ bits,
                                 unsigned long long* out) {
  const int64_t nw = woff[n];
  unsigned long long acc = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nw; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, z = n;   // largest r with woff[r] <= u
    while (z - a > 1) { int64_t mid = (a + z) >> 1; if (woff[mid] <= u) a = mid; else z = mid; }
    const int64_t l = lo[a], h = l + len[a], w = (l >> 5) + (u - woff[a]);
    const int64_t p0 = w << 5;
    uint32_t m = ~0u;
    if (p0 < l) m &= ~0u << (l - p0);
    if (p0 + 32 > h) m &= (h - p0) >= 32 ? ~0u : ((1u << (h - p0)) - 1u);
    acc += __popc(bits[w] & m);
  }
  acc = __reduce_add_sync(0xffffffffu, (unsigned)acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

static int64_t count_resident(Ctx& c, const std::vector<int64_t>& lo, const std::vector<int64_t>& len) {
  int64_t n = (int64_t)lo.size();
  if (!n) return 0;
  std::vector<int64_t> host(3 * n + 2, 0);
  for (int64_t r = 0; r < n; ++r) {
    host[r] = lo[r];
    host[n + r] = len[r];
    host[2 * n + r + 1] = host[2 * n + r] + (((lo[r] + len[r] + 31) >> 5) - (lo[r] >> 5));
  }
  DVec<int64_t>& b = c.s.rb;
  b.resize(3 * n + 2, c.st);
  MSG_CUDA(cudaMemcpyAsync(b.p, host.data(), (3 * n + 1) * 8, cudaMemcpyHostToDevice, c.st));
  MSG_CUDA(cudaMemsetAsync(b.p + 3 * n + 1, 0, 8, c.st));
  const int64_t words = host[3 * n];
  k_count_resident<<<grid_for(words, 256, 148 * 8), 256, 0, c.st>>>(
      b.p, b.p + n, b.p + 2 * n, n, c.bits.p, reinterpret_cast<unsigned long long*>(b.p + 3 * n + 1));
  MSG_CHECK_LAUNCH();
  add_launches(1);
  MSG_CUDA(cudaMemcpyAsync(c.hbuf.p, b.p + 3 * n + 1, 8, cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaStreamSynchronize(c.st));
  return c.hbuf.p[0];
}

void release_pages(Ctx& c, const int64_t* first, const int64_t* end, int32_t n, int64_t* removed) {
  c.hbuf.reserve(64);
  std::vector<int64_t> lo, len;
  dense_ranges(c, first, end, n, lo, len, false);
  int64_t k = count_resident(c, lo, len);
  *removed = k;
  if (k == 0 || c.len == 0) return;
  split_by_ranges(c, lo, len);   // members (class 1) now at the tail
  int64_t keep = c.len - k;
  const int32_t* gone = c.order[c.cur].p + c.head + keep;
  if (c.run_used) MSG_CUDA(cudaStreamWaitEvent(c.st, c.ev_run_last, 0));
  k_release_pages<<<grid_for(k, 256), 256, 0, c.st>>>(gone, k, c.bits.p, c.frame.p, c.fifo.p,
                                                      c.fifo_head + c.fifo_len, c.C);
  MSG_CHECK_LAUNCH();
  add_launches(1);
  c.fifo_len += k;
  c.len = keep;
  MSG_CUDA(cudaStreamSynchronize(c.st));
}

// ---- eviction-list facade ----------------------------------------------

void list_append_abs(Ctx& c, const int64_t* first, const int64_t* end, int32_t n) {
  // pages in the given run order; already-resident pages are skipped
  std::vector<int32_t> pages;
  for (int i = 0; i < n; ++i) {
    for (int64_t p = first[i]; p < end[i]; ++p) {
      int64_t d = dense_of_host(c, p);
      if (d < 0) throw Error(MSG_E_DOMAIN, "page outside the dense page map");
      pages.push_back((int32_t)d);
    }
  }
  if (pages.empty()) return;
  // filter resident on host via a bitmap snapshot (facade path, small)
  std::vector<uint32_t> words((c.D + 31) / 32);
  MSG_CUDA(cudaMemcpyAsync(words.data(), c.bits.p, words.size() * 4, cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaStreamSynchronize(c.st));
  std::vector<int32_t> fresh;
  for (int32_t p : pages) {
    uint32_t& w = words[p >> 5];
    if (!((w >> (p & 31)) & 1u)) { fresh.push_back(p); w |= 1u << (p & 31); }
  }
  if ((int64_t)fresh.size() + c.len > c.C) throw Error(MSG_E_CAPACITY, "eviction list exceeds HBM capacity");
  DVec<int32_t>& d = c.s.miss;
  d.resize(std::max<size_t>(fresh.size(), 1), c.st);
  MSG_CUDA(cudaMemcpyAsync(d.p, fresh.data(), fresh.size() * 4, cudaMemcpyHostToDevice, c.st));
  compact_if_needed(c);
  int64_t* mig = mig_buf(c, fresh.size());
  int64_t fb = c.C - c.len;
  install_pages(c, d.p, (int64_t)fresh.size(), mig);
  if (mig) migrate_batch(c, 0, (int64_t)fresh.size(), fb, true);
  MSG_CUDA(cudaStreamSynchronize(c.st));
}

void list_madvise_abs(Ctx& c, const int64_t* first, const int64_t* end, int32_t n) {
  std::vector<int64_t> lo, len;
  dense_ranges(c, first, end, n, lo, len, false);
  if (lo.empty() || c.len == 0) return;
  split_by_ranges(c, lo, len);
  MSG_CUDA(cudaStreamSynchronize(c.st));
}

void list_evict_head(Ctx& c, int64_t n, int64_t* pages_out, int64_t* nout) {
  n = std::min(std::max<int64_t>(n, 0), c.len);
  *nout = n;
  if (!n) return;
  std::vector<int32_t> h(n);
  MSG_CUDA(cudaMemcpyAsync(h.data(), c.order[c.cur].p + c.head, n * 4, cudaMemcpyDeviceToHost, c.st));
  int64_t* mig = mig_buf(c, n);
  int64_t fb = c.C - c.len;
  evict_head_n(c, n, mig);
  if (mig) migrate_batch(c, n, 0, fb, true);
  MSG_CUDA(cudaStreamSynchronize(c.st));
  for (int64_t i = 0; i < n; ++i) {
    int64_t d = h[i];
    auto it = std::upper_bound(c.span_dense.begin(), c.span_dense.end(), d);
    int64_t s = (it - c.span_dense.begin()) - 1;
    pages_out[i] = c.span_first[s] + (d - c.span_dense[s]);
  }
}

void list_read(Ctx& c, int64_t* pages_out, int64_t cap, int64_t* n) {
  *n = c.len;
  if (!pages_out) return;
  int64_t k = std::min(cap, c.len);
  std::vector<int32_t> h(k);
  if (k) MSG_CUDA(cudaMemcpyAsync(h.data(), c.order[c.cur].p + c.head, k * 4, cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaStreamSynchronize(c.st));
  for (int64_t i = 0; i < k; ++i) {
    int64_t d = h[i];
    auto it = std::upper_bound(c.span_dense.begin(), c.span_dense.end(), d);
    int64_t s = (it - c.span_dense.begin()) - 1;
    pages_out[i] = c.span_first[s] + (d - c.span_dense[s]);
  }
}

// ---- demand paging (Mode.um): per command, sequential on the device -------

__global__ void k_table_from_iv(const Iv* iv, int64_t n, int64_t* lo, int64_t* hi, int32_t* cls, int64_t* tn) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    lo[i] = iv[i].d;
    hi[i] = iv[i].d + (iv[i].b - iv[i].a);
    cls[i] = 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *tn = n;
}

// Demand paging slice (Mode.um, engine.py:389-445): per command, in order:
// missing count, capacity evictions from the LRU head, install, and the LRU
// refresh madvise(actual) as a two-class multisplit.
void um_slice(Ctx& c, int32_t task, int32_t c0, int32_t c1, int64_t* missing_out, int64_t* evicted_out) {
  fold_events(c, c.event_bound);
  TaskTab& t = *c.tasks[task];
  cudaStream_t st = c.st;
  c.dbg[3].clear();
  c.s.uscr.resize(512, st);
  for (int32_t cmd = c0; cmd < c1; ++cmd) {
    const int64_t i0 = t.act_off[cmd], niv = t.act_off[cmd + 1] - i0;
    int64_t n = 0;
    if (niv) {
      // missing pages of the command (count + list in page order): the one
      // host round trip of the command
      const int64_t nu = t.act_units[cmd + 1] - t.act_units[cmd];
      ranges_from_actual(c, t, cmd, cmd + 1, c.s.ract);
      c.s.miss.resize(std::max<int64_t>(32 * nu, 1), st);
      units_plan(c, c.s.ract.set(), nu, nullptr, 0, -1, c.s.miss.p, -1, c.s.uscr.p + 400);
      MSG_CUDA(cudaMemcpyAsync(c.hbuf.p, c.s.uscr.p + 400, 8, cudaMemcpyDeviceToHost, st));
      MSG_CUDA(cudaStreamSynchronize(st));
      n = c.hbuf.p[0];
    }
    missing_out[cmd - c0] = n;
    evicted_out[cmd - c0] = 0;
    if (n > c.C) {
      throw Error(MSG_E_CAPACITY, "command working set (" + std::to_string(n) + " pages) exceeds HBM capacity (" +
                                      std::to_string(c.C) + " pages)");
    }
    if (n) {
      // capacity evictions from the LRU head, then install (engine.py:408-419)
      const int64_t over = std::max<int64_t>(c.len + n - c.C, 0);
      int64_t* mig = mig_buf(c, over + n);
      const int64_t free_before = c.C - c.len;
      const int64_t ev = std::min(over, c.len);
      if (c.debug & 3) {
        dump_dense(c, c.order[c.cur].p + c.head, ev, c.dbg[1]);
        dump_dense(c, c.s.miss.p, n, c.dbg[2]);
      }
      evict_head_n(c, ev, mig);
      compact_if_needed(c);
      install_pages(c, c.s.miss.p, n, mig ? mig + ev : nullptr);
      if (mig) migrate_batch(c, ev, n, free_before, t.kind[cmd] != MSG_CMD_H2D);
      evicted_out[cmd - c0] = ev;
      if (c.debug & 3) {  // [cmd, nmiss, miss..., nev, ev...] per faulting command
        auto& u = c.dbg[3];
        u.push_back(cmd);
        u.push_back((int64_t)c.dbg[2].size());
        u.insert(u.end(), c.dbg[2].begin(), c.dbg[2].end());
        u.push_back((int64_t)c.dbg[1].size());
        u.insert(u.end(), c.dbg[1].begin(), c.dbg[1].end());
      }
    }
    // LRU refresh madvise(actual) (engine.py:398-401, 425-426): a two-class
    // multisplit -- unless every page of the set was just installed, in page
    // order, at the tail, where the refresh leaves it
    if (niv && c.len && n != t.act_pages[cmd]) {
      DVec<int64_t>& tb = c.s.tb;
      DVec<int32_t>& tcls = c.s.tcls;
      tb.resize(2 * niv + 2, st);
      tcls.resize(niv, st);
      k_table_from_iv<<<grid_for(niv, 256), 256, 0, st>>>(t.act_pool.p + i0, niv, tb.p, tb.p + niv, tcls.p,
                                                         tb.p + 2 * niv);
      MSG_CHECK_LAUNCH();
      add_launches(1);
      SegTab T{tb.p, tb.p + niv, tcls.p, tb.p + 2 * niv};
      multisplit(c, T, 1);
    }
  }
  MSG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace msg

namespace msg {

// ---- facade helpers: compute_window / plan_migration on explicit runs ----

void window_runs_explicit(Ctx& c, const int64_t* first, const int64_t* end, const int32_t* cmd, int32_t niv,
                          int32_t ncmd, int64_t* runs_out, int64_t* nruns, int64_t* pages) {
  cudaStream_t st = c.st;
  std::vector<Iv> iv(std::max(niv, 1));
  std::vector<int64_t> off(ncmd + 1, 0);
  for (int i = 0; i < niv; ++i) {
    if (cmd[i] < 0 || cmd[i] >= ncmd || (i && cmd[i] < cmd[i - 1])) throw Error(MSG_E_INVAL, "bad run command index");
    iv[i] = Iv{first[i], end[i], 0};
    off[cmd[i] + 1]++;
  }
  for (int k = 0; k < ncmd; ++k) off[k + 1] += off[k];
  DVec<Iv> d_iv; d_iv.exact(iv.size());
  DVec<int64_t> d_off; d_off.exact(ncmd + 1);
  DVec<uint8_t> d_sp; d_sp.exact(std::max(ncmd, 1));
  MSG_CUDA(cudaMemcpyAsync(d_iv.p, iv.data(), iv.size() * sizeof(Iv), cudaMemcpyHostToDevice, st));
  MSG_CUDA(cudaMemcpyAsync(d_off.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice, st));
  MSG_CUDA(cudaMemsetAsync(d_sp.p, 0, std::max(ncmd, 1), st));
  WinDesc wd{};
  wd.pool = d_iv.p;
  wd.pool_lo = 0; wd.pool_hi = niv; wd.c0 = 0; wd.c1 = ncmd; wd.w = 0;
  wd.cmd_off = d_off.p; wd.selfpop = d_sp.p; wd.scratch = 0;
  int64_t scratch = 4 * pow2_at_least(2 * std::max<int64_t>(niv, 1)) + 16;
  DVec<WinDesc> d_wd; d_wd.exact(1);
  MSG_CUDA(cudaMemcpyAsync(d_wd.p, &wd, sizeof(wd), cudaMemcpyHostToDevice, st));
  DVec<int64_t> ka, va, rb; ka.exact(scratch); va.exact(scratch); rb.exact(3 * scratch + 8);
  DVec<int32_t> lab, rl; lab.exact(scratch); rl.exact(scratch);
  WinOut o;
  o.run_a = rb.p; o.run_b = rb.p + scratch; o.run_d = rb.p + 2 * scratch;
  o.run_base = rb.p + 3 * scratch; o.nruns = o.run_base + 1; o.pages = o.nruns + 1;
  o.run_lab = rl.p;
  win_kernels_init(c);
  k_window_runs<<<1, 1024, kWinSmem, st>>>(d_wd.p, ka.p, va.p, lab.p, o, kWinSmem);
  MSG_CHECK_LAUNCH();
  add_launches(1);
  int64_t hb[3];
  MSG_CUDA(cudaMemcpyAsync(hb, o.run_base, 3 * 8, cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaStreamSynchronize(st));
  int64_t nr = hb[1];
  *nruns = nr;
  *pages = hb[2];
  if (runs_out && nr) {
    std::vector<int64_t> a(nr), b(nr);
    std::vector<int32_t> l(nr);
    MSG_CUDA(cudaMemcpyAsync(a.data(), o.run_a, nr * 8, cudaMemcpyDeviceToHost, st));
    MSG_CUDA(cudaMemcpyAsync(b.data(), o.run_b, nr * 8, cudaMemcpyDeviceToHost, st));
    MSG_CUDA(cudaMemcpyAsync(l.data(), o.run_lab, nr * 4, cudaMemcpyDeviceToHost, st));
    MSG_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < nr; ++i) { runs_out[3 * i] = a[i]; runs_out[3 * i + 1] = b[i]; runs_out[3 * i + 2] = l[i]; }
  }
}

void list_plan(Ctx& c, const int64_t* first, const int64_t* end, int32_t n, int64_t capacity, int64_t* pop_out,
               int64_t* npop, int64_t* ev_out, int64_t* nev, int64_t* truncated) {
  cudaStream_t st = c.st;
  std::vector<int64_t> a, b;
  for (int i = 0; i < n; ++i) {
    if (end[i] <= first[i]) continue;
    int64_t d0 = dense_of_host(c, first[i]), d1 = dense_of_host(c, end[i] - 1);
    if (d0 < 0 || d1 < 0 || d1 - d0 != end[i] - 1 - first[i]) throw Error(MSG_E_DOMAIN, "run outside the page map");
    a.push_back(first[i]); b.push_back(end[i]);
  }
  int64_t m = (int64_t)a.size();
  int64_t cap = std::max<int64_t>(m, 1);
  DVec<int64_t> buf; buf.exact(3 * cap + 8);
  DVec<int32_t> lab; lab.exact(cap);
  DVec<uint8_t> sp; sp.exact(cap);
  std::vector<int32_t> hl(cap);
  int64_t units = 0;
  for (int64_t i = 0; i < cap; ++i) hl[i] = (int32_t)i;
  for (int64_t i = 0; i < m; ++i) {
    int64_t d = dense_of_host(c, a[i]);
    units += ((d + (b[i] - a[i]) + 31) >> 5) - (d >> 5);
  }
  if (m) {
    MSG_CUDA(cudaMemcpyAsync(buf.p, a.data(), m * 8, cudaMemcpyHostToDevice, st));
    MSG_CUDA(cudaMemcpyAsync(buf.p + cap, b.data(), m * 8, cudaMemcpyHostToDevice, st));
  }
  MSG_CUDA(cudaMemcpyAsync(lab.p, hl.data(), cap * 4, cudaMemcpyHostToDevice, st));
  MSG_CUDA(cudaMemsetAsync(sp.p, 0, cap, st));
  MSG_CUDA(cudaMemcpyAsync(buf.p + 2 * cap, &m, 8, cudaMemcpyHostToDevice, st));
  RangeBuf rb;
  rb.reserve(cap, st);
  DemandParams D{};
  D.run_a = buf.p; D.run_b = buf.p + cap; D.run_lab = lab.p; D.run_base = 0; D.nruns = buf.p + 2 * cap;
  D.selfpop = sp.p; D.c0 = 0;
  D.span_first = c.d_span_first.p; D.span_n = c.d_span_n.p; D.span_dense = c.d_span_dense.p;
  D.nspans = (int32_t)c.span_first.size();
  D.R = rb.out();
  RangeSet R = rb.set();
  DVec<int64_t> scr; scr.exact(512);
  DVec<int32_t> pl; pl.exact(std::max<int64_t>(std::min<int64_t>(32 * units, std::max<int64_t>(capacity, 0)), 1));
  k_demand_collect<<<1, 1024, 0, st>>>(D);
  MSG_CHECK_LAUNCH();
  add_launches(1);
  units_plan(c, R, units, nullptr, 0, std::max<int64_t>(capacity, 0), pl.p, capacity, scr.p + 400);
  MSG_CUDA(cudaMemcpyAsync(c.hstate, c.dstate, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaStreamSynchronize(st));
  DevState S = *c.hstate;
  *npop = S.populate;
  *truncated = S.truncated;
  int64_t ev = std::min<int64_t>(S.evict, c.len);
  *nev = ev;
  std::vector<int64_t> tmp;
  dump_dense(c, pl.p, S.populate, tmp);
  if (pop_out) std::copy(tmp.begin(), tmp.end(), pop_out);
  dump_dense(c, c.order[c.cur].p + c.head, ev, tmp);
  if (ev_out) std::copy(tmp.begin(), tmp.end(), ev_out);
}

}  // namespace msg

#ifdef MSG_MC_PHASE_TS
extern "C" void msg_dbg_mc_ts(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, msg::g_mc_min, 16 * 8);
  cudaMemcpyFromSymbol(out + 16, msg::g_mc_max, 16 * 8);
  cudaMemcpyFromSymbol(out + 32, msg::g_mc_sum, 16 * 8);
  cudaMemcpyFromSymbol(out + 48, msg::g_mc_n, 8);
}
extern "C" void msg_dbg_mc_warp(unsigned long long* out) {   // 64 x 160 x 32 per-warp records
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, msg::g_mc_warp, sizeof(msg::g_mc_warp));
}
extern "C" void msg_dbg_mc_cta(unsigned long long* out) {   // 256 x 160 x 8 stamps
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, msg::g_mc_cta, sizeof(msg::g_mc_cta));
}
extern "C" void msg_dbg_fw_ts(unsigned long long* out) {   // 16 phase sums + launches
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, msg::g_fw_sum, 16 * 8);
  cudaMemcpyFromSymbol(out + 16, msg::g_fw_n, 8);
}
extern "C" void msg_dbg_sw_ts(unsigned long long* out) {   // 8 phase sums + launches
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, msg::g_sw_sum, 8 * 8);
  cudaMemcpyFromSymbol(out + 8, msg::g_sw_n, 8);
  cudaMemcpyFromSymbol(out + 9, msg::g_gap_sum, 8);
  cudaMemcpyFromSymbol(out + 10, msg::g_gap_n, 8);
}
extern "C" void msg_dbg_cw_ts(unsigned long long* out) {   // combine_wide 16 sums + n, window_runs 16 sums + n
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, msg::g_cw_sum, 16 * 8);
  cudaMemcpyFromSymbol(out + 16, msg::g_cw_n, 8);
  cudaMemcpyFromSymbol(out + 17, msg::g_wr_sum, 16 * 8);
  cudaMemcpyFromSymbol(out + 33, msg::g_wr_n, 8);
}
extern "C" void msg_dbg_mc_reset() {
  unsigned long long lo[16], hi[16] = {0}, z[16] = {0}, zn = 0;
  for (int i = 0; i < 16; ++i) lo[i] = ~0ull;
  cudaMemcpyToSymbol(msg::g_mc_min, lo, 128);
  cudaMemcpyToSymbol(msg::g_mc_max, hi, 128);
  cudaMemcpyToSymbol(msg::g_mc_sum, z, 128);
  cudaMemcpyToSymbol(msg::g_mc_n, &zn, 8);
  unsigned long long zf[16] = {0};
  cudaMemcpyToSymbol(msg::g_fw_sum, zf, sizeof(zf));
  cudaMemcpyToSymbol(msg::g_fw_n, &zn, 8);
  cudaMemcpyToSymbol(msg::g_sw_sum, zf, 8 * 8);
  cudaMemcpyToSymbol(msg::g_sw_n, &zn, 8);
  cudaMemcpyToSymbol(msg::g_gap_sum, &zn, 8);
  cudaMemcpyToSymbol(msg::g_gap_n, &zn, 8);
  cudaMemcpyToSymbol(msg::g_fw_end, &zn, 8);
  cudaMemcpyToSymbol(msg::g_cw_sum, zf, sizeof(zf));
  cudaMemcpyToSymbol(msg::g_cw_n, &zn, 8);
  cudaMemcpyToSymbol(msg::g_wr_sum, zf, sizeof(zf));
  cudaMemcpyToSymbol(msg::g_wr_n, &zn, 8);
}
#endif
