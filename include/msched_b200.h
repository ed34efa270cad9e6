/*
 * msched_b200.h — C ABI of the B200-native proactive memory-scheduling path.
 *
 * One context (msg_ctx) per GPU owns all device state of one simulated
 * oversubscribed GPU: the dense page map, per-command predicted/actual page
 * intervals, the resident bitmap, the eviction order, the HBM frame arena
 * and the pinned host backing pool.  The host keeps task-level scheduling
 * and every floating-point timing decision (engine.py:262-473 of the
 * reference); only integer set results cross this boundary.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/msim/):
 *   msg_add_task / msg_set_rules / msg_add_commands
 *       -> Simulator._init_task_tables / _extend_task_tables / _predict
 *          (engine.py:222-249), predictor.predict / predict_allocation /
 *          ground_truth_prediction (predictor.py:24-77),
 *          TemplateRule.predict_regions (analyzer.py:155-174)
 *   msg_plan_switch
 *       -> Simulator._prepare_slice (engine.py:305-340): timeline_windows /
 *          compute_window (memman.py:174-206), reorder_for_opt
 *          (memman.py:218-241), plan_migration (memman.py:269-302),
 *          _gating_state (engine.py:342-361), apply_plan (memman.py:305-307);
 *          plus the fast path of _touch (engine.py:389-397) for the slice
 *   msg_touch
 *       -> Simulator._touch / _refresh_opt (engine.py:389-460)
 *   msg_release_task
 *       -> Simulator._release (engine.py:462-473), EvictionList.remove
 *   msg_list_* (eviction-list facade used by the drop-in EvictionList)
 *       -> EvictionList.append_tail / madvise / evict_head / remove /
 *          pages_in_order (memman.py:43-123)
 *   msg_migrate_* -> the migration timing model (engine.py:126-166) made
 *       real: pinned host DRAM <-> HBM copies of every planned page.
 *
 * Conventions
 *   - Return 0 on success, a negative MSG_E_* code on failure; the message
 *     is available from msg_last_error(ctx) until the next call on ctx.
 *   - Inputs are caller-owned and copied during the call; outputs are
 *     caller-allocated.
 *   - A context is not thread-safe; contexts on different devices are
 *     independent (one process per GPU).
 *   - Page ids crossing the ABI are ABSOLUTE page numbers (byte address /
 *     page_size), exactly the reference's PageSet elements.
 */
#ifndef MSCHED_B200_H
#define MSCHED_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSG_OK 0
#define MSG_E_INVAL (-1)     /* bad argument */
#define MSG_E_DOMAIN (-2)    /* page outside the dense map, arithmetic overflow */
#define MSG_E_CAPACITY (-3)  /* residency guard (engine.py:402-406, 420-424) */
#define MSG_E_OOM (-4)       /* device or pinned-host allocation failed */
#define MSG_E_CUDA (-5)      /* CUDA runtime error */

/* predictor selection (engine.py:239-244) */
#define MSG_PRED_TEMPLATE 0
#define MSG_PRED_ALLOCATION 1
#define MSG_PRED_TRUTH 2

/* command kinds (core.py:210-213) */
#define MSG_CMD_KERNEL 0
#define MSG_CMD_H2D 1
#define MSG_CMD_D2H 2

/* msg_cfg.flags */
#define MSG_F_MIGRATE 1u       /* perform real host<->HBM copies of planned pages */
#define MSG_F_VERIFY_TAGS 2u   /* stamp page ids into payloads so migration is checkable */
#define MSG_F_LOOSE_DOMAIN 4u  /* predictor-only contexts: pages outside the map are allowed (no residency) */
#define MSG_F_EXECUTE 8u       /* msg_run_command: executed commands also wait for their own in-flight pages */

typedef struct msg_ctx msg_ctx;

typedef struct {
  int32_t device;
  int32_t predictor;        /* MSG_PRED_* */
  int64_t page_size;        /* bytes, power of two */
  int64_t capacity_pages;   /* HBM frames (hbm_capacity_bytes / page_size) */
  int64_t host_pool_pages;  /* pinned backing pages; 0 = whole domain; smaller pools alias */
  uint32_t flags;           /* MSG_F_* */
  uint32_t reserved;
} msg_cfg;

/* One launch-argument slot (core.py:216-227).  value is a 128-bit
 * two's-complement integer (lo, hi); raw structs point into the blob. */
typedef struct {
  uint64_t lo;
  int64_t hi;
  int32_t width;            /* 32 / 64; 0 for raw */
  int32_t raw_len;          /* -1 when not a raw struct */
  int64_t raw_off;          /* byte offset into the blob */
} msg_arg;

typedef struct {
  int32_t kind;             /* MSG_CMD_* */
  int32_t kernel;           /* index into the task's kernel table, -1 unknown */
  int32_t arg_off, nargs;   /* into the msg_arg array */
  int32_t gt_off, ngt;      /* into the ground-truth range array */
  int64_t dims[6];          /* gx gy gz bx by bz */
  int64_t dev_addr, dev_len;/* memcpy device extent (core.py:257-260) */
} msg_cmd;

typedef struct {
  int64_t start, len;       /* bytes */
} msg_range;

/* Slot code: kind in bits 0-1 (0 plain arg, 1 struct word, 2 launch dim),
 * arg/dim index in bits 2-17, struct byte offset in bits 18-49,
 * width (32/64) flag in bit 50 (1 = 64). */
typedef struct {
  int64_t num, den;         /* exact rational coefficient, den > 0 */
  int32_t nslots;           /* 0..3 */
  int32_t pad;
  int64_t slot[3];
} msg_expr;

typedef struct {
  int32_t kind;             /* 0 fixed/linear (size), 1 strided */
  int32_t ptr_arg;
  int64_t offset;
  msg_expr e[3];            /* size | stride, chunk, count */
} msg_rule;

typedef struct {
  int32_t task;
  int32_t c0, c1;           /* command range [c0, c1) */
  int32_t pad;
} msg_window;

/* Result of one proactive context switch. */
typedef struct {
  int64_t missing;          /* |demand - resident| before the switch (engine.py:310) */
  int32_t early_exit;       /* nothing missing: no reorder, no plan */
  int32_t nwin;
  int64_t populate, evict, truncated, free_before;
  int64_t resident_after;
  int32_t first_missing;    /* first command of window 0 whose actual set is not resident, -1 none */
  int32_t pad;
  int64_t first_missing_pages;
} msg_switch_out;

typedef struct {
  int64_t missing;          /* pages installed */
  int64_t evicted;          /* capacity evictions */
  int64_t resident_after;
  int32_t refreshed;
  int32_t next_missing;     /* next command in (cmd, scan_end) with missing pages, -1 none */
  int64_t next_missing_pages;
} msg_touch_out;

typedef struct {
  int64_t kernels;          /* kernel launches issued so far */
  int64_t h2d_bytes, d2h_bytes;      /* migrated payload bytes */
  int64_t h2d_segments, d2h_segments;
  int64_t ce_batches, sm_batches;
  double h2d_busy_ms, d2h_busy_ms;   /* copy-engine busy time (CUDA events) */
  double plan_ms;                     /* planner kernel time (CUDA events) */
  /* the reorder multisplit (the dominant planner kernel): launches, device
   * time over its count+scan+scatter kernels, algorithmic bytes (8 B per
   * list entry per pass: the list is read once and written once) */
  int64_t ms_passes;
  double ms_ms;
  int64_t ms_bytes;
  /* executed commands (msg_run_command): count, pages read from the HBM
   * arena, pages whose payload tag did not match (MSG_F_VERIFY_TAGS), pages
   * found non-resident, and the consumer stream's busy time (CUDA events) */
  int64_t run_cmds, run_pages, run_bad_tags, run_missing;
  double run_ms;
  /* the cooperative multisplit's launches timed on the device itself
   * (%globaltimer, first CTA start to last CTA end): ms_ms minus launch
   * latency */
  int64_t ms_dev_launches;
  double ms_dev_ms;
  /* passes whose launch ms_ms brackets with CUDA events (standalone
   * multisplit launches); the async switch path runs the multisplit as a
   * phase of its per-switch kernel, timed on the device only */
  int64_t ms_ev_passes;
} msg_stats;

/* Forget all residency (bitmap, list, frames); keep the task tables and the
 * predicted sets (keep_tasks=1) or drop the tasks too (keep_tasks=0).
 * Allocations (HBM arena, pinned pool) are kept.  Clears msg_stats. */
int msg_reset(msg_ctx *ctx, int32_t keep_tasks);

int msg_create(const msg_cfg *cfg, msg_ctx **out);
void msg_destroy(msg_ctx *ctx);
const char *msg_last_error(const msg_ctx *ctx);
void *msg_stream(msg_ctx *ctx);   /* the cudaStream_t the planner runs on */

/* Dense page map: disjoint absolute page spans [first, first+npages).  Must
 * be called once before tasks/commands; page ids outside are MSG_E_DOMAIN. */
int msg_set_domain(msg_ctx *ctx, const int64_t *span_first, const int64_t *span_npages, int32_t nspans);

/* Task registration: its allocations (byte ranges) for the allocation
 * predictor, and its kernel rule table (kernel k owns rules
 * [kernel_rule_off[k], kernel_rule_off[k+1])). */
int msg_add_task(msg_ctx *ctx, int32_t task, const msg_range *allocs, int32_t nallocs);
int msg_set_rules(msg_ctx *ctx, int32_t task, const msg_rule *rules, const int32_t *kernel_rule_off,
                  int32_t nkernels);

/* K1: evaluate predicted and actual page sets of ncmd new commands of `task`
 * on the device.  complete_out (optional, ncmd bytes) receives the
 * predictor's `complete` flag before any unpredictable_fraction override. */
int msg_add_commands(msg_ctx *ctx, int32_t task, int32_t ncmd, const msg_cmd *cmds, const msg_arg *args,
                     const uint8_t *blob, int64_t blob_len, const msg_range *gt, uint8_t *complete_out);

/* Read back a command's predicted (which=0) or actual (which=1) page runs.
 * Call with runs=NULL to get the count. */
int msg_read_pages(msg_ctx *ctx, int32_t task, int32_t cmd, int32_t which, int64_t *runs, int64_t cap,
                   int64_t *nruns);
/* The same for commands [c0, c1) in one device-to-host copy: runs of
 * command c0 + k are runs[2 * off[k] .. 2 * off[k + 1]) (off: c1 - c0 + 1
 * entries).  Call with runs=NULL to get the total in *nruns (off is filled
 * either way; pass off=NULL to skip it). */
int msg_read_pages_range(msg_ctx *ctx, int32_t task, int32_t c0, int32_t c1, int32_t which, int64_t *runs,
                         int64_t cap, int64_t *off, int64_t *nruns);

/* One proactive switch.  win[0] is the incoming slice; win_pages_out
 * (nwin entries) receives |window pages| for madvise_cost_s; prefix_out
 * (c1-c0 of win[0]) receives the per-command count of new non-resident
 * demand pages (pre-apply, uncapped; the host caps and accumulates);
 * touch_cnt_out (c1-c0 of win[0]) the post-apply missing count per command. */
int msg_plan_switch(msg_ctx *ctx, const msg_window *win, int32_t nwin, int32_t reorder_always,
                    msg_switch_out *out, int64_t *win_pages_out, int64_t *prefix_out, int64_t *touch_cnt_out);

/* Slow path of _touch for command `cmd` of `task`.  If evict > 0 the list
 * is first reordered with windows `win` (when nwin > 0) and `evict` head
 * pages are evicted; then the command's missing pages are appended.
 * Afterwards commands (cmd, scan_end) are rescanned. */
int msg_touch(msg_ctx *ctx, int32_t task, int32_t cmd, int64_t evict, const msg_window *win, int32_t nwin,
              int32_t scan_end, int32_t write_tags, msg_touch_out *out, int64_t *win_pages_out);

/* Demand-paging slice (Mode.um): commands [c0, c1) of `task` processed in
 * order on the device; per command: missing count and capacity evictions. */
int msg_um_slice(msg_ctx *ctx, int32_t task, int32_t c0, int32_t c1, int64_t *missing_out, int64_t *evicted_out);

/* Execute command `cmd` of `task` on the device (the paper's early-start
 * gating made real, engine.py:139-158, 342-361, 373-378): on a dedicated
 * stream, wait until the populate copies of the current switch have landed
 * up to `need_pages` (the command's gating prefix: demand pages first
 * accessed by commands <= cmd, in populate order) — and, if this command's
 * own touch installed pages, until that batch has landed; with MSG_F_EXECUTE
 * also until every page of its actual set that this switch populates has
 * landed (a page predicted for a later command but touched by this one is
 * in flight, and the hardware would stall on it) — then launch a
 * kernel that reads every page of the command's actual set from its HBM
 * frame (16-byte loads) and checks the payload tags when the context
 * verifies them; the kernel then occupies the GPU until `latency_s` (the
 * command's profiled duration, Command.latency_s, core.py:231) has passed
 * since it started, so an executed replay runs in the time the model
 * charges for exec_s (engine.py:373-384).  Pass need_pages = populate count
 * to wait for the whole batch (Mode.early_start = False).  Later migrations
 * wait for the executed commands before they evict or overwrite frames.
 * Needs MSG_F_MIGRATE and MSG_F_EXECUTE (the H2D stream publishes populate
 * progress only then).  latency_s < 0 or > 60 s is MSG_E_INVAL. */
int msg_run_command(msg_ctx *ctx, int32_t task, int32_t cmd, int64_t need_pages, double latency_s);

/* Release a task: drop its pages (absolute page spans) from the list. */
int msg_release_task(msg_ctx *ctx, const int64_t *span_first, const int64_t *span_end, int32_t nspans,
                     int64_t *removed);

/* Eviction-list facade (memman.py:43-123); pages are absolute ids. */
int msg_list_append(msg_ctx *ctx, const int64_t *run_first, const int64_t *run_end, int32_t nruns);
int msg_list_madvise(msg_ctx *ctx, const int64_t *run_first, const int64_t *run_end, int32_t nruns);
int msg_list_evict_head(msg_ctx *ctx, int64_t n, int64_t *pages_out, int64_t *nout);
int msg_list_len(msg_ctx *ctx, int64_t *n);
int msg_list_read(msg_ctx *ctx, int64_t *pages_out, int64_t cap, int64_t *n);
/* reorder_for_opt with explicit windows (memman.py:218-241): runs of window
 * k in first-access order, windows in timeline order.  win_pages_out gets
 * each window's page count. */
int msg_list_reorder(msg_ctx *ctx, const int64_t *run_first, const int64_t *run_end, const int32_t *run_win,
                     int32_t nruns, int32_t nwin, int64_t *win_pages_out);

/* compute_window (memman.py:174-196) over explicit per-command page runs:
 * iv_* are the normalised runs of commands [0, ncmd) (command of each run in
 * iv_cmd, non-decreasing).  Outputs the first-access runs (first, end,
 * command) and |window pages|. */
int msg_window_runs(msg_ctx *ctx, const int64_t *iv_first, const int64_t *iv_end, const int32_t *iv_cmd,
                    int32_t niv, int32_t ncmd, int64_t *runs_out, int64_t *nruns, int64_t *pages);

/* plan_migration (memman.py:269-302) against the current list, without
 * applying it: populate pages (first-access order, capacity-truncated) and
 * evict pages (head order). */
int msg_list_plan(msg_ctx *ctx, const int64_t *run_first, const int64_t *run_end, int32_t nruns,
                  int64_t capacity, int64_t *populate_out, int64_t *npopulate, int64_t *evict_out,
                  int64_t *nevict, int64_t *truncated);

/* Offline template inference, native (analyzer.py:185-441 of the reference:
 * build_descriptors / build_descriptor / infer_rule / fit_linear_expr).
 * Commands in the msg_cmd / msg_arg / blob / msg_range layout, with
 * cmds[i].kernel = the index of the command's kernel name (0..nkernels-1,
 * memcpys ignored) and latency[i] its latency.  Per kernel k: status[k] = 0
 * when done here, 1 when a value lies outside the native arithmetic (values
 * and slot values must be < 2^64) or argument counts are ragged — the host
 * analyzer then does that kernel; latency_out[k] (mean over the records),
 * unpredictable_out[k], and rules [rule_off[k], rule_off[k+1]) of rules_out.
 * A rule's expression q (size for fixed/linear; stride, chunk, count for
 * strided) is coeff * prod(slot[q][0..nslots[q])) with coeff = v0[q] divided
 * by the product of those slots in the kernel's first record (the host forms
 * the reduced fraction).  Returns MSG_E_INVAL if rules_cap is too small
 * (rule_off[nkernels] has the count).  Needs no GPU and no context. */
typedef struct {
  int32_t ptr_arg;
  int32_t kind;             /* 0 fixed, 1 linear, 2 strided */
  int64_t offset;
  int32_t nslots[3];
  int32_t pad;
  int64_t slot[3][3];       /* slot codes (see msg_expr) */
  int64_t v0[3];
} msg_arule;

int msg_analyze(const msg_cmd *cmds, int32_t ncmd, const msg_arg *args, const uint8_t *blob, int64_t blob_len,
                const msg_range *gt, const double *latency, int32_t nkernels, int32_t *status, double *latency_out,
                double *unpredictable_out, msg_arule *rules_out, int32_t rules_cap, int32_t *rule_off);

/* Parity dumps (the reference's promised but unimplemented SPEC.md:415-416
 * debug dump).  which: 0 list order after the last reorder, 1 last evicted
 * pages (head order), 2 last installed pages (install order).  enable is a
 * bit set: 1 plan dumps, 2 full list orders, 8 run the reorder multisplit on
 * the look-back (onesweep) kernel instead of the on-chip cooperative one, so
 * tests cover both. */
int msg_debug(msg_ctx *ctx, int32_t enable);
int msg_debug_read(msg_ctx *ctx, int32_t which, int64_t *out, int64_t cap, int64_t *n);

/* Migration engine. */
int msg_sync(msg_ctx *ctx);                       /* wait for all planner + copy work */
int msg_get_stats(msg_ctx *ctx, msg_stats *out);
int msg_verify_residency(msg_ctx *ctx, int64_t *bad_pages);   /* needs MSG_F_VERIFY_TAGS */
int msg_flush_l2(msg_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
