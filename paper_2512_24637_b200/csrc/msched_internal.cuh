// Internal declarations shared by the msched_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include <stdexcept>
#include <chrono>

#include "../../include/msched_b200.h"

namespace msg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define MSG_CUDA(x)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      throw ::msg::Error(MSG_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + " (" + \
                                         __FILE__ + ":" + std::to_string(__LINE__) + ")");   \
  } while (0)

#define MSG_CHECK_LAUNCH() MSG_CUDA(cudaGetLastError())

constexpr int32_t kNone = 0x7fffffff;

// Page interval in absolute page ids [a, b) plus its dense start d.
struct Iv {
  int64_t a, b, d;
};

// Owning device buffer with geometric growth.
template <class T>
struct DVec {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  DVec() = default;
  DVec(const DVec&) = delete;
  DVec& operator=(const DVec&) = delete;
  ~DVec() { if (p) cudaFree(p); }
  void reserve(size_t want, cudaStream_t s) {
    if (want <= cap) return;
    size_t nc = cap ? cap : 256;
    while (nc < want) nc *= 2;
    T* q = nullptr;
    if (cudaMalloc(&q, nc * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      throw Error(MSG_E_OOM, "device allocation of " + std::to_string(nc * sizeof(T)) + " bytes failed");
    }
    // zero-filled, so growth never carries uninitialised bytes (only on growth: geometric, rare)
    MSG_CUDA(cudaMemsetAsync(q, 0, nc * sizeof(T), s));
    if (n) MSG_CUDA(cudaMemcpyAsync(q, p, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p) { MSG_CUDA(cudaStreamSynchronize(s)); cudaFree(p); }
    p = q;
    cap = nc;
  }
  void resize(size_t want, cudaStream_t s) { reserve(want, s); n = want; }
  // grow-only scratch: at least `want` elements, contents discarded on growth
  // (geometric, so repeated calls stop allocating -- and cudaFree, which
  // synchronises the device, stops being called)
  void fit(size_t want) {
    if (want > cap) exact(std::max<size_t>(want, 2 * cap));
    n = want;
  }
  void exact(size_t want) {  // allocate exactly, discarding contents
    if (p) cudaFree(p);
    p = nullptr; n = cap = 0;
    if (want == 0) return;
    if (cudaMalloc(&p, want * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      throw Error(MSG_E_OOM, "device allocation of " + std::to_string(want * sizeof(T)) + " bytes failed");
    }
    n = cap = want;
  }
};

// Pinned host buffer.
template <class T>
struct HVec {
  T* p = nullptr;
  size_t cap = 0;
  ~HVec() { if (p) cudaFreeHost(p); }
  void reserve(size_t want) {
    if (want <= cap) return;
    size_t nc = cap ? cap : 256;
    while (nc < want) nc *= 2;
    if (p) cudaFreeHost(p);
    p = nullptr;
    if (cudaMallocHost(&p, nc * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      throw Error(MSG_E_OOM, "pinned allocation failed");
    }
    cap = nc;
  }
};

struct Rule {
  int32_t kind, ptr;
  int64_t off;
  msg_expr e[3];
};

struct TaskTab {
  int32_t id = -1;
  int64_t ncmd = 0;
  // host mirrors of the interval CSR offsets (pred / actual) into the pools
  std::vector<int64_t> pred_off{0}, act_off{0};
  std::vector<int64_t> pred_units{0}, act_units{0};   // cumulative bitmap-word units per command
  std::vector<int64_t> act_pages;                    // pages of each command's actual set (dense map)
  std::vector<uint8_t> selfpop, kind;
  std::vector<Rule> rules;
  std::vector<int32_t> kern_off{0};
  std::vector<msg_range> allocs;   // sorted by start
  DVec<int64_t> d_pred_off, d_act_off;
  DVec<uint8_t> d_selfpop;
  DVec<Iv> pred_pool, act_pool;   // this task's intervals (CSR by command)
};

// An ordered list of dense page ranges, processed one 32-page bitmap word
// (a "unit") at a time.  uoff[r] = units before range r; uoff[nr] = total.
struct RangeSet {
  const int64_t* lo;
  const int64_t* len;
  const int32_t* tag;
  const int64_t* uoff;
  const int64_t* nr;
};

struct RangeOut {
  int64_t* lo;
  int64_t* len;
  int32_t* tag;
  int64_t* uoff;
  int64_t* nr;
};

// Owning storage for a RangeSet plus its per-unit scratch.
struct RangeBuf {
  DVec<int64_t> i64;   // lo | len | uoff | nr
  DVec<int32_t> tag;
  int64_t cap = 0;
  void reserve(int64_t n, cudaStream_t st) {
    cap = n < 1 ? 1 : n;
    i64.resize(3 * cap + 4, st);
    tag.resize(cap, st);
  }
  RangeOut out() { return RangeOut{i64.p, i64.p + cap, tag.p, i64.p + 2 * cap, i64.p + 3 * cap + 2}; }
  RangeSet set() { return RangeSet{i64.p, i64.p + cap, tag.p, i64.p + 2 * cap, i64.p + 3 * cap + 2}; }
};

// Per-switch planner scratch.
struct Scratch {
  DVec<int64_t> i64a, i64b, i64c, i64d, i64e;
  DVec<int32_t> i32a, i32b, i32c;
  DVec<uint32_t> u32a;
  DVec<Iv> iv;
  DVec<int64_t> dem, tc, cnt, tb, rb;
  DVec<int32_t> poplist, miss, tcls;
  DVec<int32_t> mflag;
  DVec<int64_t> moff, msegs;
  RangeBuf rdem, ract;          // window-0 demand runs; actual sets of a command range
  DVec<int32_t> ucnt;           // per-unit counts
  DVec<int64_t> uofs, uscr;     // per-unit offsets, scan scratch
  DVec<int64_t> wide;           // k_window_combine_wide global scratch + its ok flag
};

// msg_add_commands' device inputs and intermediates (K1), kept across calls
struct PredScratch {
  DVec<uint8_t> comp;
  DVec<int32_t> err;
  DVec<int64_t> cnt, rawp, rawa, nn, gk, dst;
  DVec<Iv> np, na;
  DVec<uint8_t> din;        // all inputs of one call, one H2D copy
  HVec<uint8_t> hin, hio;   // pinned staging: the packed inputs; counts / offsets in and out
};

// Device-side scalar state (one struct in device memory).
struct DevState {
  int64_t head;         // index of the list head in the current order buffer
  int64_t len;          // resident pages
  int64_t fifo_head;    // free-frame FIFO (ring over capacity)
  int64_t fifo_len;
  int64_t missing;      // scratch results
  int64_t populate, evict, truncated, free_before;
  int32_t skip, first_missing;
  int64_t first_missing_pages;
  int64_t nclass;       // classes of the current multisplit
  int64_t aux[8];
};

struct Ctx {
  msg_cfg cfg{};
  std::string err;
  int device = 0;
  cudaStream_t st = nullptr;          // planner stream
  cudaStream_t st_d2h = nullptr, st_h2d = nullptr;
  cudaStream_t st_run = nullptr;      // executed commands (msg_run_command)
  DVec<int4> flush_buf;               // msg_flush_l2's 256 MiB write target (this ctx's device)
  PredScratch ps;                     // K1 scratch (predict_commands)
  // host-side phase clock of msg_plan_switch / msg_touch (MSG_HOST_PHASES=1
  // prints the sums when the context is destroyed): [call][phase] seconds
  bool host_phases = false;
  double hp_sum[2][8] = {};
  int64_t hp_n[2] = {};
  unsigned long long* d_progress = nullptr;   // populate pages landed so far (written by the H2D stream)
  unsigned long long* d_run_acc = nullptr;    // [0] pages read [1] bad tags [2] non-resident
  int64_t installed_total = 0;        // populate pages whose copies have been issued
  int64_t switch_base = 0;            // installed_total before the current switch's populate
  int32_t fault_task = -1, fault_cmd = -1;   // last touch install and the total after its batch
  int64_t fault_total = 0;
  cudaEvent_t ev_run_last = nullptr;  // the last executed command
  DVec<int64_t> pos_of;               // MSG_F_EXECUTE: (switch tag << 32 | populate position) per dense page
  int32_t switch_tag = 0;
  int32_t gate_task = -1, gate_c0 = 0;
  std::vector<int64_t> gate_need;     // per command of the last switch's slice: populate pages its actual set needs
  bool run_used = false;
  cudaEvent_t ev_plan_done = nullptr, ev_h2d_done = nullptr, ev_d2h_prev = nullptr;
  int64_t P = 4096, C = 0;            // page size, capacity pages
  // dense map
  std::vector<int64_t> span_first, span_n, span_dense;
  DVec<int64_t> d_span_first, d_span_n, d_span_dense;
  int64_t D = 0;                      // dense pages
  // residency
  DVec<uint32_t> bits;                // resident bitmap over dense pages
  DVec<int32_t> order[2];             // eviction order ping-pong buffers
  int cur = 0;                        // which order buffer is live
  int64_t head = 0, len = 0;          // host mirror of DevState head/len
  int64_t order_cap = 0;
  DVec<int32_t> frame;                // frame of each dense page, -1 if none
  DVec<int32_t> fifo;                 // free frames (ring)
  int64_t fifo_head = 0, fifo_len = 0;
  DevState* dstate = nullptr;
  DevState* hstate = nullptr;         // pinned mirror
  // tasks and interval pools
  std::vector<TaskTab*> tasks;
  DVec<msg_range> d_allocs;           // scratch for the allocation predictor
  Scratch s;
  HVec<int64_t> hbuf;                 // pinned readback buffer
  // migration
  char* arena = nullptr;              // HBM frames
  char* pool = nullptr;               // pinned host backing (mapped)
  char* pool_dev = nullptr;           // device alias of pool
  int64_t pool_pages = 0;
  DVec<int64_t> mig_list[2];          // (page<<32|frame) per migrated page: [d2h..., h2d...]
  int mig_par = 0;
  int32_t mig_batch = 0;              // migration batch id (copy-ordering epochs)
  int64_t batch_old_free = 0;         // free frames that predate the current batch
  DVec<int32_t> inst_ep, free_ep;     // per frame: last H2D batch / last D2H batch
  std::vector<cudaEvent_t> ev_d2h_of, ev_h2d_of;   // per batch completion events
  cudaEvent_t ev_mig[2] = {nullptr, nullptr};
  cudaEvent_t ev_call[2] = {nullptr, nullptr};   // plan_switch's planner-time pair (reused every call)
  std::vector<cudaEvent_t> ev_pool;
  // busy times of event pairs already folded away (fold_events)
  double fold_h2d_ms = 0, fold_d2h_ms = 0, fold_ms_ms = 0, fold_run_ms = 0;
  size_t event_bound = 1 << 15;   // events kept before folding
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> busy_h2d, busy_d2h;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> busy_plan, busy_ms, busy_run;
  msg_stats stats{};
  bool ms_events_pending = false;   // a standalone multisplit launch awaits its pass count (stats)
  // parity dumps
  int debug = 0;   // 1: plan lists, 2: full list orders
  int fallback = 0;   // MSG_FALLBACK test hook: 1 two-kernel windows, 2 look-back multisplit, 4 demand kernel
  // single-pass multisplit state
  DVec<unsigned long long> ms_status;   // 256 per tile, epoch-tagged
  DVec<int32_t> ms_ctr;                 // tile claim counter per epoch
  DVec<unsigned long long> ms_tot;      // digit totals (4 x 257)
  DVec<int32_t> ms_hist;                // per-CTA digit counts of the cooperative multisplit (+ 2 total rows)
  int ms_tot_par = 0;                   // which total row the next cooperative launch accumulates into
  DVec<int32_t> up_hist;                // k_units_plan per-CTA totals and tag partials
  DVec<unsigned long long> ms_tring;    // k_ms_coop device timestamps: [first starts | last ends] per launch
  int64_t ms_tslot = 0, ms_tbase = 0;   // next slot; slots before ms_tbase were already summed
  double ms_dev_ms_acc = 0.0;
  // per-device kernel setup (dynamic shared memory attributes are per device)
  bool win_init = false;
  int ms_grid_cap = 0, ms_coop_grid = 0, up_per_sm = -1, nsm = 0, sw_grid = 0;
  int ms_force_stream = 0;            // MSG_MS_STREAM=1 (tuning / test hook)
  uint32_t ms_epoch = 0;
  int64_t ms_launch_id = 0;           // cooperative multisplit launches (phase-timing build)
  std::vector<int64_t> dbg[4];
  ~Ctx();
};

// ---- helpers implemented in the .cu files ----
int64_t dense_of_host(const Ctx& c, int64_t abs_page);   // -1 if outside
void launch_count();                                     // bump kernel counter

// predictor
void predict_commands(Ctx& c, TaskTab& t, int32_t ncmd, const msg_cmd* cmds, const msg_arg* args,
                      const uint8_t* blob, int64_t blob_len, const msg_range* gt, uint8_t* complete_out);

// planner
void plan_switch(Ctx& c, const msg_window* win, int32_t nwin, bool reorder_always, msg_switch_out* out,
                 int64_t* win_pages, int64_t* prefix, int64_t* touch_cnt);
void touch_slow(Ctx& c, int32_t task, int32_t cmd, int64_t evict, const msg_window* win, int32_t nwin,
                int32_t scan_end, bool write_tags, msg_touch_out* out, int64_t* win_pages);
void um_slice(Ctx& c, int32_t task, int32_t c0, int32_t c1, int64_t* missing, int64_t* evicted);
void release_pages(Ctx& c, const int64_t* first, const int64_t* end, int32_t n, int64_t* removed);
void list_append_abs(Ctx& c, const int64_t* first, const int64_t* end, int32_t n);
void list_madvise_abs(Ctx& c, const int64_t* first, const int64_t* end, int32_t n);
void list_evict_head(Ctx& c, int64_t n, int64_t* pages_out, int64_t* nout);
void list_read(Ctx& c, int64_t* pages_out, int64_t cap, int64_t* n);
void window_runs_explicit(Ctx& c, const int64_t* first, const int64_t* end, const int32_t* cmd, int32_t niv,
                          int32_t ncmd, int64_t* runs_out, int64_t* nruns, int64_t* pages);
void list_plan(Ctx& c, const int64_t* first, const int64_t* end, int32_t n, int64_t capacity, int64_t* pop_out,
               int64_t* npop, int64_t* ev_out, int64_t* nev, int64_t* truncated);
void list_reorder(Ctx& c, const int64_t* first, const int64_t* end, const int32_t* win, int32_t n, int32_t nwin,
                  int64_t* win_pages);
void pull_state(Ctx& c);   // sync + copy DevState to the host mirrors
void ms_harvest(Ctx& c);   // accumulate device-timed multisplit launches into the stats
void fold_events(Ctx& c, size_t bound);   // release events past `bound` (busy times kept as sums)
void push_state(Ctx& c);

void scan_flags(Ctx& c, const int32_t* in, int64_t n, int64_t* out);   // exclusive scan

// migration
void migration_init(Ctx& c);
void migrate_batch(Ctx& c, int64_t n_d2h, int64_t n_h2d, int64_t free_before, bool copy_h2d);
void verify_tags(Ctx& c, int64_t* bad);
void run_command(Ctx& c, int32_t task, int32_t cmd, int64_t need_pages, double latency_s);
void run_wait_before_copies(Ctx& c);

int64_t kernel_launches();
void add_launches(int64_t n);

}  // namespace msg
