// The extern "C" boundary (include/msched_b200.h): context lifetime, the
// dense page map, task tables, and error mapping.  Every entry point catches
// msg::Error and returns its code; no exception crosses the ABI.
#include "msched_internal.cuh"

#include <vector>

#include <cstdlib>

#include <algorithm>
#include <cstring>

namespace msg {

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_iota_i32(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

__global__ void k_flush(int4* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_int4((int)i, 0, 0, 0);
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  if (host_phases) {
    const char* nm[2] = {"plan_switch", "touch"};
    for (int k = 0; k < 2; ++k) {
      if (!hp_n[k]) continue;
      std::fprintf(stderr, "[msg host phases] %s n=%lld us/call:", nm[k], (long long)hp_n[k]);
      for (int i = 0; i < 8; ++i) std::fprintf(stderr, " %.1f", hp_sum[k][i] * 1e6 / hp_n[k]);
      std::fprintf(stderr, "\n");
    }
  }
  if (st) cudaStreamSynchronize(st);
  if (st_d2h) cudaStreamSynchronize(st_d2h);
  if (st_h2d) cudaStreamSynchronize(st_h2d);
  if (st_run) cudaStreamSynchronize(st_run);
  for (auto* t : tasks) delete t;
  for (auto e : ev_pool) cudaEventDestroy(e);
  for (auto e : {ev_mig[0], ev_mig[1], ev_call[0], ev_call[1], ev_h2d_done, ev_plan_done, ev_d2h_prev})
    if (e) cudaEventDestroy(e);
  if (arena) cudaFree(arena);
  if (pool) cudaFreeHost(pool);
  if (dstate) cudaFree(dstate);
  if (hstate) cudaFreeHost(hstate);
  if (ev_run_last) cudaEventDestroy(ev_run_last);
  if (d_progress) cudaFree(d_progress);
  if (d_run_acc) cudaFree(d_run_acc);
  if (st_run) cudaStreamDestroy(st_run);
  if (st_d2h) cudaStreamDestroy(st_d2h);
  if (st_h2d) cudaStreamDestroy(st_h2d);
  if (st) cudaStreamDestroy(st);
}

int64_t dense_of_host(const Ctx& c, int64_t p) {
  auto it = std::upper_bound(c.span_first.begin(), c.span_first.end(), p);
  int64_t s = (it - c.span_first.begin()) - 1;
  if (s < 0 || p >= c.span_first[s] + c.span_n[s]) return -1;
  return c.span_dense[s] + (p - c.span_first[s]);
}

static void set_domain(Ctx& c, const int64_t* first, const int64_t* npages, int32_t n) {
  if (c.D) throw Error(MSG_E_INVAL, "domain already set");
  std::vector<std::pair<int64_t, int64_t>> r;
  for (int i = 0; i < n; ++i)
    if (npages[i] > 0) r.push_back({first[i], first[i] + npages[i]});
  std::sort(r.begin(), r.end());
  std::vector<std::pair<int64_t, int64_t>> m;
  for (auto& x : r) {
    if (!m.empty() && x.first <= m.back().second) m.back().second = std::max(m.back().second, x.second);
    else m.push_back(x);
  }
  int64_t d = 0;
  for (auto& x : m) d += x.second - x.first;
  // validate before touching the context: a rejected domain leaves it unset
  if (d >= (1ll << 31)) throw Error(MSG_E_DOMAIN, "dense page map exceeds 2^31 pages");
  d = 0;
  for (auto& x : m) {
    c.span_first.push_back(x.first);
    c.span_n.push_back(x.second - x.first);
    c.span_dense.push_back(d);
    d += x.second - x.first;
  }
  c.D = d;
  cudaStream_t st = c.st;
  size_t ns = std::max<size_t>(m.size(), 1);
  c.d_span_first.exact(ns); c.d_span_n.exact(ns); c.d_span_dense.exact(ns);
  if (!m.empty()) {
    MSG_CUDA(cudaMemcpyAsync(c.d_span_first.p, c.span_first.data(), m.size() * 8, cudaMemcpyHostToDevice, st));
    MSG_CUDA(cudaMemcpyAsync(c.d_span_n.p, c.span_n.data(), m.size() * 8, cudaMemcpyHostToDevice, st));
    MSG_CUDA(cudaMemcpyAsync(c.d_span_dense.p, c.span_dense.data(), m.size() * 8, cudaMemcpyHostToDevice, st));
  }
  int64_t words = (std::max<int64_t>(d, 1) + 31) / 32 + 1;
  c.bits.exact(words);
  MSG_CUDA(cudaMemsetAsync(c.bits.p, 0, words * 4, st));
  c.frame.exact(std::max<int64_t>(d, 1));
  k_fill_i32<<<1184, 256, 0, st>>>(c.frame.p, std::max<int64_t>(d, 1), -1);
  c.order_cap = 2 * c.C + 64;
  c.order[0].exact(c.order_cap);
  c.order[1].exact(c.order_cap);
  c.fifo.exact(std::max<int64_t>(c.C, 1));
  k_iota_i32<<<1184, 256, 0, st>>>(c.fifo.p, c.C);
  MSG_CHECK_LAUNCH();
  add_launches(2);
  c.fifo_head = 0;
  c.fifo_len = c.C;
  migration_init(c);
  MSG_CUDA(cudaStreamSynchronize(st));
}

static void nonneg(int64_t n) {
  if (n < 0) throw Error(MSG_E_INVAL, "negative count");
}

static TaskTab& task_of(Ctx& c, int32_t task) {
  if (task < 0 || task >= (int32_t)c.tasks.size() || !c.tasks[task]) throw Error(MSG_E_INVAL, "unknown task");
  return *c.tasks[task];
}

}  // namespace msg

using namespace msg;

struct msg_ctx {
  Ctx c;
};

template <class F>
static int guard(msg_ctx* ctx, F&& f) {
  try {
    if (ctx) cudaSetDevice(ctx->c.device);
    f();
    return MSG_OK;
  } catch (const Error& e) {
    if (ctx) ctx->c.err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.err = e.what();
    return MSG_E_INVAL;
  }
}

extern "C" {

int msg_create(const msg_cfg* cfg, msg_ctx** out) {
  if (!cfg || !out) return MSG_E_INVAL;
  *out = nullptr;
  if (cfg->page_size <= 0 || (cfg->page_size & (cfg->page_size - 1))) return MSG_E_INVAL;
  if (cfg->capacity_pages <= 0 || cfg->capacity_pages >= (1ll << 31)) return MSG_E_INVAL;
  auto* ctx = new msg_ctx();
  int rc = guard(ctx, [&] {
    Ctx& c = ctx->c;
    c.cfg = *cfg;
    c.device = cfg->device;
    MSG_CUDA(cudaSetDevice(c.device));
    MSG_CUDA(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
    c.P = cfg->page_size;
    c.C = cfg->capacity_pages;
    MSG_CUDA(cudaMalloc(&c.dstate, sizeof(DevState)));
    MSG_CUDA(cudaMemset(c.dstate, 0, sizeof(DevState)));
    MSG_CUDA(cudaMallocHost(&c.hstate, sizeof(DevState)));
    std::memset(c.hstate, 0, sizeof(DevState));
    c.hbuf.reserve(1 << 16);
    // test hook: MSG_FALLBACK=windows,onesweep,demand runs the general kernels
    // in place of the fast paths, so the golden tests cover both
    if (const char* f = std::getenv("MSG_FALLBACK")) {
      std::string v(f);
      if (v.find("windows") != std::string::npos) c.fallback |= 1;
      if (v.find("onesweep") != std::string::npos) c.fallback |= 2;
      if (v.find("demand") != std::string::npos) c.fallback |= 4;
    }
    if (const char* f = std::getenv("MSG_HOST_PHASES")) c.host_phases = f[0] == '1';
    if (const char* f = std::getenv("MSG_MS_STREAM")) c.ms_force_stream = f[0] == '1';
    // test hook: MSG_EVENT_BOUND=n folds the context's events past n (fold_events)
    if (const char* f = std::getenv("MSG_EVENT_BOUND")) c.event_bound = (size_t)std::max(1ll, std::atoll(f));
  });
  if (rc != MSG_OK) {
    std::fprintf(stderr, "msg_create: %s\n", ctx->c.err.c_str());
    delete ctx;
    return rc;
  }
  *out = ctx;
  return MSG_OK;
}

void msg_destroy(msg_ctx* ctx) { delete ctx; }

const char* msg_last_error(const msg_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

void* msg_stream(msg_ctx* ctx) { return ctx ? (void*)ctx->c.st : nullptr; }

int msg_set_domain(msg_ctx* ctx, const int64_t* first, const int64_t* npages, int32_t n) {
  return guard(ctx, [&] { set_domain(ctx->c, first, npages, n); });
}

int msg_add_task(msg_ctx* ctx, int32_t task, const msg_range* allocs, int32_t nallocs) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (!c.D && !c.span_first.size()) throw Error(MSG_E_INVAL, "set the domain first");
    if (task < 0) throw Error(MSG_E_INVAL, "negative task id");
    if (nallocs < 0) throw Error(MSG_E_INVAL, "negative count");
    if (nallocs > 0 && !allocs) throw Error(MSG_E_INVAL, "null allocation table");
    if ((int32_t)c.tasks.size() <= task) c.tasks.resize(task + 1, nullptr);
    if (c.tasks[task]) throw Error(MSG_E_INVAL, "task registered twice");
    auto* t = new TaskTab();
    t->id = task;
    t->allocs.assign(allocs, allocs + nallocs);
    std::sort(t->allocs.begin(), t->allocs.end(),
              [](const msg_range& a, const msg_range& b) { return a.start < b.start; });
    c.tasks[task] = t;
  });
}

int msg_set_rules(msg_ctx* ctx, int32_t task, const msg_rule* rules, const int32_t* kernel_rule_off,
                  int32_t nkernels) {
  return guard(ctx, [&] {
    TaskTab& t = task_of(ctx->c, task);
    if (nkernels < 0) throw Error(MSG_E_INVAL, "negative kernel count");
    int32_t nr = nkernels ? kernel_rule_off[nkernels] : 0;
    t.rules.clear();
    for (int32_t i = 0; i < nr; ++i) {
      const msg_rule& r = rules[i];
      Rule q;
      q.kind = r.kind; q.ptr = r.ptr_arg; q.off = r.offset;
      for (int k = 0; k < 3; ++k) {
        q.e[k] = r.e[k];
        if (q.e[k].nslots < 0 || q.e[k].nslots > 3) throw Error(MSG_E_INVAL, "expression has > 3 slots");
        if ((k == 0 || r.kind == 1) && q.e[k].den <= 0) throw Error(MSG_E_INVAL, "non-positive denominator");
        if (q.e[k].den <= 0) q.e[k].den = 1;
      }
      if (r.kind != 0 && r.kind != 1) throw Error(MSG_E_INVAL, "bad rule kind");
      t.rules.push_back(q);
    }
    t.kern_off.assign(kernel_rule_off, kernel_rule_off + nkernels + 1);
    if (nkernels == 0) t.kern_off = {0};
  });
}

int msg_add_commands(msg_ctx* ctx, int32_t task, int32_t ncmd, const msg_cmd* cmds, const msg_arg* args,
                     const uint8_t* blob, int64_t blob_len, const msg_range* gt, uint8_t* complete_out) {
  return guard(ctx, [&] {
    TaskTab& t = task_of(ctx->c, task);
    if (ncmd < 0 || blob_len < 0) throw Error(MSG_E_INVAL, "negative count");
    predict_commands(ctx->c, t, ncmd, cmds, args, blob, blob_len, gt, complete_out);
  });
}

int msg_read_pages(msg_ctx* ctx, int32_t task, int32_t cmd, int32_t which, int64_t* runs, int64_t cap,
                   int64_t* nruns) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    TaskTab& t = task_of(c, task);
    if (cmd < 0 || cmd >= t.ncmd) throw Error(MSG_E_INVAL, "bad command index");
    const std::vector<int64_t>& off = which ? t.act_off : t.pred_off;
    int64_t i0 = off[cmd], n = off[cmd + 1] - i0;
    *nruns = n;
    if (!runs) return;
    int64_t k = std::min(cap, n);
    std::vector<Iv> h(k);
    if (k)
      MSG_CUDA(cudaMemcpyAsync(h.data(), (which ? t.act_pool.p : t.pred_pool.p) + i0, k * sizeof(Iv),
                               cudaMemcpyDeviceToHost, c.st));
    MSG_CUDA(cudaStreamSynchronize(c.st));
    for (int64_t i = 0; i < k; ++i) { runs[2 * i] = h[i].a; runs[2 * i + 1] = h[i].b; }
  });
}

int msg_read_pages_range(msg_ctx* ctx, int32_t task, int32_t c0, int32_t c1, int32_t which, int64_t* runs,
                         int64_t cap, int64_t* off, int64_t* nruns) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    TaskTab& t = task_of(c, task);
    if (c0 < 0 || c1 < c0 || c1 > t.ncmd) throw Error(MSG_E_INVAL, "bad command range");
    if (!nruns) throw Error(MSG_E_INVAL, "null output");
    const std::vector<int64_t>& o = which ? t.act_off : t.pred_off;
    const int64_t i0 = o[c0], n = o[c1] - i0;
    *nruns = n;
    if (off)
      for (int32_t k = 0; k <= c1 - c0; ++k) off[k] = o[c0 + k] - i0;
    if (!runs) return;
    const int64_t k = std::min(cap, n);
    if (k <= 0) return;
    std::vector<Iv> h(k);
    MSG_CUDA(cudaMemcpyAsync(h.data(), (which ? t.act_pool.p : t.pred_pool.p) + i0, k * sizeof(Iv),
                             cudaMemcpyDeviceToHost, c.st));
    MSG_CUDA(cudaStreamSynchronize(c.st));
    for (int64_t i = 0; i < k; ++i) { runs[2 * i] = h[i].a; runs[2 * i + 1] = h[i].b; }
  });
}

// every window names a registered task and a command range inside it
static void check_windows(Ctx& c, const msg_window* win, int32_t nwin) {
  if (nwin < 0 || (nwin > 0 && !win)) throw Error(MSG_E_INVAL, "bad window list");
  for (int32_t w = 0; w < nwin; ++w) {
    TaskTab& t = task_of(c, win[w].task);
    if (win[w].c0 < 0 || win[w].c1 < win[w].c0 || win[w].c1 > t.ncmd) throw Error(MSG_E_INVAL, "bad window range");
  }
}

int msg_plan_switch(msg_ctx* ctx, const msg_window* win, int32_t nwin, int32_t reorder_always, msg_switch_out* out,
                    int64_t* win_pages_out, int64_t* prefix_out, int64_t* touch_cnt_out) {
  return guard(ctx, [&] {
    check_windows(ctx->c, win, nwin);
    plan_switch(ctx->c, win, nwin, reorder_always != 0, out, win_pages_out, prefix_out, touch_cnt_out);
  });
}

int msg_touch(msg_ctx* ctx, int32_t task, int32_t cmd, int64_t evict, const msg_window* win, int32_t nwin,
              int32_t scan_end, int32_t write_tags, msg_touch_out* out, int64_t* win_pages_out) {
  return guard(ctx, [&] {
    check_windows(ctx->c, win, nwin);
    touch_slow(ctx->c, task, cmd, evict, win, nwin, scan_end, write_tags != 0, out, win_pages_out);
  });
}

int msg_um_slice(msg_ctx* ctx, int32_t task, int32_t c0, int32_t c1, int64_t* missing_out, int64_t* evicted_out) {
  return guard(ctx, [&] {
    TaskTab& t = task_of(ctx->c, task);
    if (c0 < 0 || c1 < c0 || c1 > t.ncmd) throw Error(MSG_E_INVAL, "bad command range");
    um_slice(ctx->c, task, c0, c1, missing_out, evicted_out);
  });
}

int msg_release_task(msg_ctx* ctx, const int64_t* span_first, const int64_t* span_end, int32_t nspans,
                     int64_t* removed) {
  return guard(ctx, [&] {
    nonneg(nspans);
    release_pages(ctx->c, span_first, span_end, nspans, removed);
  });
}

int msg_list_append(msg_ctx* ctx, const int64_t* first, const int64_t* end, int32_t n) {
  return guard(ctx, [&] {
    nonneg(n);
    list_append_abs(ctx->c, first, end, n);
  });
}

int msg_list_madvise(msg_ctx* ctx, const int64_t* first, const int64_t* end, int32_t n) {
  return guard(ctx, [&] {
    nonneg(n);
    list_madvise_abs(ctx->c, first, end, n);
  });
}

int msg_list_evict_head(msg_ctx* ctx, int64_t n, int64_t* pages_out, int64_t* nout) {
  return guard(ctx, [&] { list_evict_head(ctx->c, n, pages_out, nout); });
}

int msg_list_len(msg_ctx* ctx, int64_t* n) {
  return guard(ctx, [&] { *n = ctx->c.len; });
}

int msg_list_read(msg_ctx* ctx, int64_t* pages_out, int64_t cap, int64_t* n) {
  return guard(ctx, [&] {
    nonneg(cap);
    list_read(ctx->c, pages_out, cap, n);
  });
}

int msg_list_reorder(msg_ctx* ctx, const int64_t* first, const int64_t* end, const int32_t* win, int32_t n,
                     int32_t nwin, int64_t* win_pages) {
  return guard(ctx, [&] {
    nonneg(n);
    nonneg(nwin);
    list_reorder(ctx->c, first, end, win, n, nwin, win_pages);
  });
}

int msg_window_runs(msg_ctx* ctx, const int64_t* iv_first, const int64_t* iv_end, const int32_t* iv_cmd, int32_t niv,
                    int32_t ncmd, int64_t* runs_out, int64_t* nruns, int64_t* pages) {
  return guard(ctx, [&] {
    nonneg(niv);
    nonneg(ncmd);
    window_runs_explicit(ctx->c, iv_first, iv_end, iv_cmd, niv, ncmd, runs_out, nruns, pages);
  });
}

int msg_list_plan(msg_ctx* ctx, const int64_t* run_first, const int64_t* run_end, int32_t nruns, int64_t capacity,
                  int64_t* populate_out, int64_t* npopulate, int64_t* evict_out, int64_t* nevict,
                  int64_t* truncated) {
  return guard(ctx, [&] {
    nonneg(nruns);
    list_plan(ctx->c, run_first, run_end, nruns, capacity, populate_out, npopulate, evict_out, nevict, truncated);
  });
}

int msg_debug(msg_ctx* ctx, int32_t enable) {
  return guard(ctx, [&] { ctx->c.debug = enable; });
}

int msg_debug_read(msg_ctx* ctx, int32_t which, int64_t* out, int64_t cap, int64_t* n) {
  return guard(ctx, [&] {
    if (which < 0 || which > 3) throw Error(MSG_E_INVAL, "bad dump id");
    const auto& v = ctx->c.dbg[which];
    *n = (int64_t)v.size();
    if (out) std::copy(v.begin(), v.begin() + std::min<int64_t>(cap, (int64_t)v.size()), out);
  });
}

int msg_sync(msg_ctx* ctx) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    MSG_CUDA(cudaStreamSynchronize(c.st));
    if (c.st_d2h) MSG_CUDA(cudaStreamSynchronize(c.st_d2h));
    if (c.st_h2d) MSG_CUDA(cudaStreamSynchronize(c.st_h2d));
    if (c.st_run) MSG_CUDA(cudaStreamSynchronize(c.st_run));
  });
}

int msg_run_command(msg_ctx* ctx, int32_t task, int32_t cmd, int64_t need_pages, double latency_s) {
  return guard(ctx, [&] { run_command(ctx->c, task, cmd, need_pages, latency_s); });
}

int msg_get_stats(msg_ctx* ctx, msg_stats* out) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    MSG_CUDA(cudaStreamSynchronize(c.st));
    if (c.st_d2h) MSG_CUDA(cudaStreamSynchronize(c.st_d2h));
    if (c.st_h2d) MSG_CUDA(cudaStreamSynchronize(c.st_h2d));
    if (c.st_run) MSG_CUDA(cudaStreamSynchronize(c.st_run));
    msg_stats s = c.stats;
    s.kernels = kernel_launches();
    if (c.d_run_acc) {
      unsigned long long acc[4];
      MSG_CUDA(cudaMemcpy(acc, c.d_run_acc, sizeof(acc), cudaMemcpyDeviceToHost));
      s.run_pages = (int64_t)acc[0]; s.run_bad_tags = (int64_t)acc[1]; s.run_missing = (int64_t)acc[2];
    }
    ms_harvest(c);
    double r = c.fold_run_ms;
    for (auto& pr : c.busy_run) { float ms = 0; if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) r += ms; }
    cudaGetLastError();
    s.run_ms = r;
    double h = c.fold_h2d_ms, d = c.fold_d2h_ms;
    for (auto& pr : c.busy_h2d) { float ms = 0; if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) h += ms; }
    for (auto& pr : c.busy_d2h) { float ms = 0; if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) d += ms; }
    cudaGetLastError();
    s.h2d_busy_ms = h;
    s.d2h_busy_ms = d;
    double m = c.fold_ms_ms;
    for (auto& pr : c.busy_ms) { float ms = 0; if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) m += ms; }
    cudaGetLastError();
    s.ms_ms = m;
    s.ms_dev_launches = c.stats.ms_dev_launches;
    s.ms_ev_passes = c.stats.ms_ev_passes;
    s.ms_dev_ms = c.ms_dev_ms_acc;
    *out = s;
  });
}

int msg_reset(msg_ctx* ctx, int32_t keep_tasks) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    MSG_CUDA(cudaStreamSynchronize(c.st));
    if (c.st_d2h) MSG_CUDA(cudaStreamSynchronize(c.st_d2h));
    if (c.st_h2d) MSG_CUDA(cudaStreamSynchronize(c.st_h2d));
    if (c.st_run) MSG_CUDA(cudaStreamSynchronize(c.st_run));
    c.installed_total = 0; c.switch_base = 0; c.fault_task = -1; c.run_used = false;
    std::memset(c.hp_sum, 0, sizeof(c.hp_sum));   // the phase clock covers the replays since the last reset
    std::memset(c.hp_n, 0, sizeof(c.hp_n));
    if (c.d_progress) MSG_CUDA(cudaMemsetAsync(c.d_progress, 0, 8, c.st));
    if (c.d_run_acc) MSG_CUDA(cudaMemsetAsync(c.d_run_acc, 0, 4 * 8, c.st));
    c.busy_run.clear();
    int64_t words = (std::max<int64_t>(c.D, 1) + 31) / 32 + 1;
    MSG_CUDA(cudaMemsetAsync(c.bits.p, 0, words * 4, c.st));
    k_fill_i32<<<1184, 256, 0, c.st>>>(c.frame.p, std::max<int64_t>(c.D, 1), -1);
    k_iota_i32<<<1184, 256, 0, c.st>>>(c.fifo.p, c.C);
    MSG_CHECK_LAUNCH();
    add_launches(2);
    c.cur = 0; c.head = 0; c.len = 0;
    c.fifo_head = 0; c.fifo_len = c.C;
    if (!keep_tasks) {
      for (auto* t : c.tasks) delete t;
      c.tasks.clear();
    }
    for (auto e : c.ev_pool) cudaEventDestroy(e);
    c.ev_pool.clear();
    c.busy_h2d.clear(); c.busy_d2h.clear(); c.busy_plan.clear(); c.busy_ms.clear();
    c.fold_h2d_ms = c.fold_d2h_ms = c.fold_ms_ms = c.fold_run_ms = 0;
    c.ev_d2h_of.clear(); c.ev_h2d_of.clear();
    c.mig_batch = 0;
    if (c.inst_ep.p) {
      MSG_CUDA(cudaMemsetAsync(c.inst_ep.p, 0xff, c.C * 4, c.st));
      MSG_CUDA(cudaMemsetAsync(c.free_ep.p, 0xff, c.C * 4, c.st));
    }
    int64_t k = c.stats.kernels;
    c.stats = msg_stats{};
    c.stats.kernels = k;
    c.ms_dev_ms_acc = 0.0;
    c.ms_tslot = (int64_t)c.ms_tring.n / 2;   // next launch re-initialises the ring
    c.ms_tbase = c.ms_tslot;
    for (auto& v : c.dbg) v.clear();
    MSG_CUDA(cudaStreamSynchronize(c.st));
  });
}

int msg_verify_residency(msg_ctx* ctx, int64_t* bad_pages) {
  return guard(ctx, [&] { verify_tags(ctx->c, bad_pages); });
}

int msg_flush_l2(msg_ctx* ctx) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (!c.flush_buf.p) c.flush_buf.exact((256ll << 20) / 16);
    k_flush<<<1184, 256, 0, c.st>>>(c.flush_buf.p, (int64_t)c.flush_buf.n);
    MSG_CHECK_LAUNCH();
    add_launches(1);
    MSG_CUDA(cudaStreamSynchronize(c.st));
  });
}

}  // extern "C"
