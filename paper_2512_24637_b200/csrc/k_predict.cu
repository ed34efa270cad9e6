// K1/K2 — working-set prediction on the device.
//
// Per command: evaluate the task's template rules against the live launch
// arguments with exact 128-bit rational arithmetic (analyzer.py:119-174,
// predictor.py:24-44), or the whole-allocation rule (predictor.py:47-65), or
// the ground truth (predictor.py:74-77, engine.py:246-249); turn byte ranges
// into absolute page intervals (core.py:192-207), normalise them (sort,
// merge overlapping AND touching runs: core.py:177-189) and map them into
// the dense page space.  Four passes: count, fill, normalise (one CTA per
// command, bitonic sort in shared memory), compact into the task's CSR.
#include "msched_internal.cuh"

#include <cstring>

namespace msg {

typedef __int128 i128;
typedef unsigned __int128 u128;

__device__ __forceinline__ i128 arg_value(const msg_arg& a) {
  return (i128)(((u128)(uint64_t)a.hi << 64) | (u128)a.lo);
}

// |x| as unsigned
__device__ __forceinline__ u128 uabs(i128 x) { return x < 0 ? (u128)(-(x + 1)) + 1 : (u128)x; }

// Overflow-checked signed 128-bit multiply (result must fit in +-2^126).
__device__ bool mul_ok(i128 a, i128 b, i128* r) {
  u128 ua = uabs(a), ub = uabs(b);
  const u128 lim = ((u128)1) << 126;
  if (ua != 0 && ub > lim / ua) return false;
  *r = a * b;
  return true;
}

__device__ __forceinline__ i128 floor_div_pow2(i128 x, int shift) {
  // arithmetic shift == floor division by 2^shift for two's complement
  return x >> shift;
}

struct CmdView {
  const msg_cmd* c;
  const msg_arg* args;
  const uint8_t* blob;
  int64_t blob_len;
};

// Slot lookup: returns false when the slot is absent (analyzer.py:78-96, 119-124).
__device__ bool slot_value(const CmdView& v, int64_t code, i128* out) {
  int kind = (int)(code & 3);
  int idx = (int)((code >> 2) & 0xffff);
  if (kind == 2) {
    if (idx > 5) return false;
    *out = (i128)v.c->dims[idx];
    return true;
  }
  if (idx >= v.c->nargs) return false;
  const msg_arg& a = v.args[v.c->arg_off + idx];
  bool is_raw = a.raw_len >= 0;
  if (kind == 0) {
    if (is_raw) return false;
    *out = arg_value(a);
    return true;
  }
  if (!is_raw) return false;
  int64_t off = (code >> 18) & 0xffffffffLL;
  bool wide = (code >> 50) & 1;
  int64_t L = a.raw_len;
  if (wide) {
    if (off % 8 != 0 || off + 8 > L) return false;
  } else {
    if (off % 4 != 0 || off + 4 > L) return false;
  }
  const uint8_t* p = v.blob + a.raw_off + off;
  uint64_t w = 0;
  int nb = wide ? 8 : 4;
  for (int i = nb - 1; i >= 0; --i) w = (w << 8) | p[i];
  *out = (i128)(u128)w;
  return true;
}

// 0 = ok, 1 = None (missing slot / non-integral), 2 = overflow
__device__ int eval_expr(const CmdView& v, const msg_expr& e, i128* out) {
  i128 prod = 1;
  for (int k = 0; k < e.nslots; ++k) {
    i128 s;
    if (!slot_value(v, e.slot[k], &s)) return 1;
    if (!mul_ok(prod, s, &prod)) return 2;
  }
  i128 den = (i128)e.den;
  if (prod % den != 0) return 1;
  i128 r;
  if (!mul_ok(prod / den, (i128)e.num, &r)) return 2;
  *out = r;
  return 0;
}

__device__ __forceinline__ bool to_pages(i128 start, i128 len, int shift, int64_t* a, int64_t* b) {
  i128 first = floor_div_pow2(start, shift);
  i128 last = floor_div_pow2(start + len - 1, shift);
  const i128 lim = ((i128)1) << 62;
  if (first < -lim || last >= lim) return false;
  *a = (int64_t)first;
  *b = (int64_t)last + 1;
  return true;
}

struct PredParams {
  const msg_cmd* cmds;
  const msg_arg* args;
  const uint8_t* blob;
  int64_t blob_len;
  const msg_range* gt;
  const Rule* rules;
  const int32_t* kern_off;
  int32_t nkern;
  const msg_range* allocs;
  int32_t nallocs;
  int32_t mode;       // MSG_PRED_*
  int32_t shift;      // log2(page)
  int32_t ncmd;
  int64_t* cnt_pred;  // raw interval counts
  int64_t* cnt_act;
  const int64_t* off_pred;  // raw offsets (fill pass)
  const int64_t* off_act;
  int64_t* raw_pred;  // (a, b) pairs
  int64_t* raw_act;
  uint8_t* complete;
  int32_t* err;       // 1 = overflow / domain
};

constexpr int64_t kMaxStrided = 1ll << 24;

// Emits the intervals of one command; when `out` is null only counts them.
__device__ int64_t emit_truth(const PredParams& P, const msg_cmd& c, int64_t* out, bool* bad) {
  if (c.kind != MSG_CMD_KERNEL) {
    int64_t a, b;
    if (!to_pages(c.dev_addr, c.dev_len, P.shift, &a, &b)) { *bad = true; return 0; }
    if (out) { out[0] = a; out[1] = b; }
    return 1;
  }
  for (int k = 0; k < c.ngt; ++k) {
    const msg_range& r = P.gt[c.gt_off + k];
    if (out) {
      int64_t a, b;
      if (!to_pages(r.start, r.len, P.shift, &a, &b)) { *bad = true; return 0; }
      out[2 * k] = a; out[2 * k + 1] = b;
    }
  }
  return c.ngt;
}

__device__ int64_t emit_alloc(const PredParams& P, const CmdView& v, int64_t* out, bool* bad) {
  const msg_cmd& c = *v.c;
  int64_t n = 0;
  for (int i = 0; i < c.nargs; ++i) {
    const msg_arg& a = v.args[c.arg_off + i];
    if (a.raw_len >= 0 || a.width != 64) continue;
    i128 val = arg_value(a);
    // allocations are sorted by start and pairwise disjoint (Task.validate)
    int lo = 0, hi = P.nallocs;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if ((i128)P.allocs[mid].start <= val) lo = mid + 1; else hi = mid;
    }
    int j = lo - 1;
    if (j < 0) continue;
    const msg_range& al = P.allocs[j];
    if (!(val < (i128)al.start + (i128)al.len)) continue;
    if (out) {
      int64_t pa, pb;
      if (!to_pages(al.start, al.len, P.shift, &pa, &pb)) { *bad = true; return 0; }
      out[2 * n] = pa; out[2 * n + 1] = pb;
    }
    ++n;
  }
  return n;
}

__device__ int64_t emit_template(const PredParams& P, const CmdView& v, int64_t* out, bool* bad,
                                 bool* complete) {
  const msg_cmd& c = *v.c;
  if (c.kernel < 0 || c.kernel >= P.nkern) { *complete = false; return 0; }
  int64_t n = 0;
  for (int r = P.kern_off[c.kernel]; r < P.kern_off[c.kernel + 1]; ++r) {
    const Rule& R = P.rules[r];
    if (R.ptr >= c.nargs) { *complete = false; continue; }
    i128 base = arg_value(v.args[c.arg_off + R.ptr]) + (i128)R.off;
    if (R.kind == 0) {
      i128 size;
      int st = eval_expr(v, R.e[0], &size);
      if (st == 2) { *bad = true; return 0; }
      if (st == 1) { *complete = false; continue; }
      if (size < 1) size = 1;
      if (out) {
        int64_t a, b;
        if (!to_pages(base, size, P.shift, &a, &b)) { *bad = true; return 0; }
        out[2 * n] = a; out[2 * n + 1] = b;
      }
      ++n;
    } else {
      i128 stride, chunk, count;
      int s0 = eval_expr(v, R.e[0], &stride), s1 = eval_expr(v, R.e[1], &chunk),
          s2 = eval_expr(v, R.e[2], &count);
      if (s0 == 2 || s1 == 2 || s2 == 2) { *bad = true; return 0; }
      if (s0 || s1 || s2 || count < 1) { *complete = false; continue; }
      if (count > kMaxStrided) { *bad = true; return 0; }
      if (chunk < 1) chunk = 1;
      for (int64_t j = 0; j < (int64_t)count; ++j) {
        if (out) {
          i128 off;
          if (!mul_ok((i128)j, stride, &off)) { *bad = true; return 0; }
          int64_t a, b;
          if (!to_pages(base + off, chunk, P.shift, &a, &b)) { *bad = true; return 0; }
          out[2 * (n + j)] = a; out[2 * (n + j) + 1] = b;
        }
      }
      n += (int64_t)count;
    }
  }
  return n;
}

__global__ void k_pred_pass(PredParams P, int fill) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.ncmd; i += gridDim.x * blockDim.x) {
    const msg_cmd& c = P.cmds[i];
    CmdView v{&c, P.args, P.blob, P.blob_len};
    bool bad = false, complete = true;
    int64_t* po = fill ? P.raw_pred + 2 * P.off_pred[i] : nullptr;
    int64_t* ao = fill ? P.raw_act + 2 * P.off_act[i] : nullptr;
    int64_t na = emit_truth(P, c, ao, &bad);
    int64_t np;
    if (c.kind != MSG_CMD_KERNEL || P.mode == MSG_PRED_TRUTH) {
      np = emit_truth(P, c, po, &bad);
    } else if (P.mode == MSG_PRED_ALLOCATION) {
      np = emit_alloc(P, v, po, &bad);
    } else {
      np = emit_template(P, v, po, &bad, &complete);
    }
    if (bad) atomicExch(P.err, 1);
    if (!fill) {
      P.cnt_pred[i] = np;
      P.cnt_act[i] = na;
      P.complete[i] = complete ? 1 : 0;
    }
  }
}

// ---- normalisation: one CTA per command ----------------------------------

constexpr int kNormThreads = 256;
constexpr int kNormSmem = 2048;  // intervals sorted in shared memory

struct NormParams {
  const int64_t* raw;        // (a, b) pairs
  const int64_t* off;        // raw offsets per command
  const int64_t* cnt;        // raw counts
  Iv* out;                   // normalised intervals written at raw offsets
  int64_t* nout;             // normalised counts
  int64_t* nunits;           // 32-page bitmap words the command's intervals cover
  int64_t* npages;           // pages of the command's intervals inside the dense map
  const int64_t* span_first;
  const int64_t* span_n;
  const int64_t* span_dense;
  int32_t nspans;
  int32_t* err;
  int64_t* gkeys;            // global scratch for big commands (2 * total raw)
  int32_t strict;             // out-of-map pages are an error
};

__device__ __forceinline__ void cswap(int64_t* ka, int64_t* kb, int64_t* va, int64_t* vb, bool up) {
  if ((*ka > *kb) == up) {
    int64_t t = *ka; *ka = *kb; *kb = t;
    t = *va; *va = *vb; *vb = t;
  }
}

// Block-wide bitonic sort of (key, val) of length n (padded to pow2 with +inf keys).
__device__ void block_bitonic(int64_t* key, int64_t* val, int64_t npow2) {
  for (int64_t k = 2; k <= npow2; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < npow2; i += blockDim.x) {
        int64_t l = i ^ j;
        if (l > i) cswap(&key[i], &key[l], &val[i], &val[l], (i & k) == 0);
      }
      __syncthreads();
    }
  }
}

__device__ int64_t dense_of(const NormParams& P, int64_t a, int64_t b) {
  // span containing [a, b): largest span_first <= a
  int lo = 0, hi = P.nspans;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (P.span_first[mid] <= a) lo = mid + 1; else hi = mid;
  }
  int s = lo - 1;
  if (s < 0 || b > P.span_first[s] + P.span_n[s]) return -1;
  return P.span_dense[s] + (a - P.span_first[s]);
}

__global__ void k_normalize(NormParams P) {
  __shared__ int64_t sk[kNormSmem], sv[kNormSmem];
  int c = blockIdx.x;
  int64_t n = P.cnt[c];
  int64_t base = P.off[c];
  const int64_t* raw = P.raw + 2 * base;
  if (n == 0) {
    if (threadIdx.x == 0) { P.nout[c] = 0; P.nunits[c] = 0; P.npages[c] = 0; }
    return;
  }
  int64_t npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  int64_t *key, *val;
  if (npow2 <= kNormSmem) {
    key = sk; val = sv;
  } else {
    key = P.gkeys + 4 * base;  // scratch sized 4 * total raw (>= 2 * npow2)
    val = key + npow2;
  }
  for (int64_t i = threadIdx.x; i < npow2; i += blockDim.x) {
    if (i < n) { key[i] = raw[2 * i]; val[i] = raw[2 * i + 1]; }
    else { key[i] = INT64_MAX; val[i] = INT64_MAX; }
  }
  __syncthreads();
  if (n > 1) block_bitonic(key, val, npow2);
  // merge sequentially per thread-chunk: a run starts at i when key[i] > max(val[0..i-1])
  // (touching runs merge: core.py:184 uses a <= prev_end).  Done by thread 0 for
  // small n; large n uses a chunked scan of running maxima.
  if (threadIdx.x == 0) {
    int64_t m = 0, units = 0, pages = 0;
    int64_t ca = key[0], cb = val[0];
    bool bad = false;
    Iv* out = P.out + base;
    for (int64_t i = 1; i <= n; ++i) {
      if (i < n && key[i] <= cb) {
        if (val[i] > cb) cb = val[i];
        continue;
      }
      int64_t d = dense_of(P, ca, cb);
      if (d < 0 && P.strict) bad = true;
      out[m++] = Iv{ca, cb, d};
      if (d >= 0) { units += ((d + (cb - ca) + 31) >> 5) - (d >> 5); pages += cb - ca; }
      if (i < n) { ca = key[i]; cb = val[i]; }
    }
    P.nout[c] = m;
    P.nunits[c] = units;
    P.npages[c] = pages;
    if (bad) atomicExch(P.err, 2);
  }
}

__global__ void k_compact_iv(const Iv* src, const int64_t* src_off, const int64_t* cnt, const int64_t* dst_off,
                             Iv* dst, int32_t ncmd) {
  for (int c = blockIdx.x; c < ncmd; c += gridDim.x) {
    int64_t n = cnt[c];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[dst_off[c] + i] = src[src_off[c] + i];
  }
}

static int ilog2(int64_t p) {
  int s = 0;
  while ((1ll << s) < p) ++s;
  return s;
}

void predict_commands(Ctx& c, TaskTab& t, int32_t ncmd, const msg_cmd* cmds, const msg_arg* args,
                      const uint8_t* blob, int64_t blob_len, const msg_range* gt, uint8_t* complete_out) {
  if (ncmd <= 0) return;
  cudaStream_t st = c.st;
  int64_t nargs = 0, ngt = 0;
  for (int i = 0; i < ncmd; ++i) {
    const msg_cmd& m = cmds[i];
    if (m.arg_off < 0 || m.nargs < 0 || m.gt_off < 0 || m.ngt < 0)
      throw Error(MSG_E_INVAL, "negative argument or ground-truth table offset/count");
    nargs = std::max<int64_t>(nargs, (int64_t)m.arg_off + m.nargs);
    ngt = std::max<int64_t>(ngt, (int64_t)m.gt_off + m.ngt);
    if (m.kind < 0 || m.kind > 2) throw Error(MSG_E_INVAL, "bad command kind");
    if (m.kind != MSG_CMD_KERNEL && m.dev_len <= 0) throw Error(MSG_E_INVAL, "zero or negative length range");
  }
  if (nargs && !args) throw Error(MSG_E_INVAL, "null argument table");
  if (ngt && !gt) throw Error(MSG_E_INVAL, "null ground-truth table");
  if (blob_len && !blob) throw Error(MSG_E_INVAL, "null struct blob");
  // raw struct arguments are read from the blob on the device: their byte
  // windows must lie inside it
  for (int64_t j = 0; j < nargs; ++j) {
    const msg_arg& a = args[j];
    if (a.raw_len >= 0 && (a.raw_off < 0 || a.raw_off > blob_len - a.raw_len))
      throw Error(MSG_E_INVAL, "raw struct argument outside the blob");
  }
  // ByteRange rejects empty and negative lengths (core.py:52-54)
  for (int64_t j = 0; j < ngt; ++j)
    if (gt[j].len <= 0) throw Error(MSG_E_INVAL, "zero or negative length range");
  // the inputs, packed into one pinned staging buffer (16-byte aligned
  // parts) and moved with one copy into the context's grow-only K1 scratch
  PredScratch& S = c.ps;
  const void* part_src[7] = {cmds, args, blob, gt, t.rules.data(), t.kern_off.data(), t.allocs.data()};
  const size_t part_len[7] = {ncmd * sizeof(msg_cmd), (size_t)nargs * sizeof(msg_arg), (size_t)blob_len,
                              (size_t)ngt * sizeof(msg_range), t.rules.size() * sizeof(Rule),
                              t.kern_off.size() * sizeof(int32_t), t.allocs.size() * sizeof(msg_range)};
  size_t part_off[7], total_in = 0;
  for (int k = 0; k < 7; ++k) { part_off[k] = total_in; total_in += (part_len[k] + 16 + 15) & ~size_t(15); }
  S.hin.reserve(total_in);
  S.din.fit(total_in);
  for (int k = 0; k < 7; ++k)
    if (part_len[k]) std::memcpy(S.hin.p + part_off[k], part_src[k], part_len[k]);
  MSG_CUDA(cudaMemcpyAsync(S.din.p, S.hin.p, total_in, cudaMemcpyHostToDevice, st));
  struct { msg_cmd* p; } d_cmds{reinterpret_cast<msg_cmd*>(S.din.p + part_off[0])};
  struct { msg_arg* p; } d_args{reinterpret_cast<msg_arg*>(S.din.p + part_off[1])};
  struct { uint8_t* p; } d_blob{S.din.p + part_off[2]};
  struct { msg_range* p; } d_gt{reinterpret_cast<msg_range*>(S.din.p + part_off[3])};
  struct { Rule* p; } d_rules{reinterpret_cast<Rule*>(S.din.p + part_off[4])};
  struct { int32_t* p; } d_koff{reinterpret_cast<int32_t*>(S.din.p + part_off[5])};
  struct { msg_range* p; } d_allocs{reinterpret_cast<msg_range*>(S.din.p + part_off[6])};
  // pinned host side of the small count / offset round trips
  S.hio.reserve(8 * (16 * (size_t)ncmd + 16));
  int64_t* hio = reinterpret_cast<int64_t*>(S.hio.p);

  auto& cnt = S.cnt; cnt.fit(4 * (int64_t)ncmd + 2);   // cnt_pred | cnt_act | off_pred | off_act
  auto& comp = S.comp; comp.fit(ncmd);
  auto& err = S.err; err.fit(2);
  MSG_CUDA(cudaMemsetAsync(err.p, 0, 2 * sizeof(int32_t), st));

  PredParams P{};
  P.cmds = d_cmds.p; P.args = d_args.p; P.blob = d_blob.p; P.blob_len = blob_len; P.gt = d_gt.p;
  P.rules = d_rules.p; P.kern_off = d_koff.p; P.nkern = (int32_t)t.kern_off.size() - 1;
  P.allocs = d_allocs.p; P.nallocs = (int32_t)t.allocs.size();
  P.mode = c.cfg.predictor; P.shift = ilog2(c.P); P.ncmd = ncmd;
  P.cnt_pred = cnt.p; P.cnt_act = cnt.p + ncmd; P.complete = comp.p; P.err = err.p;
  int grid = (ncmd + 127) / 128;
  k_pred_pass<<<grid, 128, 0, st>>>(P, 0);
  MSG_CHECK_LAUNCH(); add_launches(1);

  // pinned layout: hc [0, 2n) | herr [2n, 2n+1) | off [2n+2, 4n+2) | hn [4n+2, 10n+2) | dst [10n+2, 12n+2) |
  // complete bytes [12n+2, ...)
  const int64_t n2 = 2 * (int64_t)ncmd;
  int64_t* hc = hio;
  int32_t* herr = reinterpret_cast<int32_t*>(hio + n2);
  int64_t* off = hio + n2 + 2;
  int64_t* hn = off + n2;
  int64_t* dst = hn + 3 * n2;
  uint8_t* hcomp = reinterpret_cast<uint8_t*>(dst + n2);
  MSG_CUDA(cudaMemcpyAsync(hc, cnt.p, n2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaMemcpyAsync(herr, err.p, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (complete_out) MSG_CUDA(cudaMemcpyAsync(hcomp, comp.p, ncmd, cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaStreamSynchronize(st));
  if (herr[0]) throw Error(MSG_E_DOMAIN, "rule arithmetic overflow or page id out of range");
  if (complete_out) std::memcpy(complete_out, hcomp, ncmd);

  int64_t tp = 0, ta = 0;
  for (int i = 0; i < ncmd; ++i) { off[i] = tp; tp += hc[i]; off[ncmd + i] = ta; ta += hc[ncmd + i]; }
  MSG_CUDA(cudaMemcpyAsync(cnt.p + 2 * ncmd, off, n2 * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  auto& rawp = S.rawp; auto& rawa = S.rawa;
  rawp.fit(2 * std::max<int64_t>(tp, 1)); rawa.fit(2 * std::max<int64_t>(ta, 1));
  P.off_pred = cnt.p + 2 * ncmd; P.off_act = cnt.p + 3 * ncmd; P.raw_pred = rawp.p; P.raw_act = rawa.p;
  k_pred_pass<<<grid, 128, 0, st>>>(P, 1);
  MSG_CHECK_LAUNCH(); add_launches(1);

  // normalise both sets
  auto& np_ = S.np; auto& na_ = S.na;
  np_.fit(std::max<int64_t>(tp, 1)); na_.fit(std::max<int64_t>(ta, 1));
  auto& nn = S.nn; nn.fit(6 * (int64_t)ncmd);   // counts | units | pages, pred then act
  auto& gk = S.gk; gk.fit(4 * std::max(tp, ta) + 4);
  NormParams N{};
  N.span_first = c.d_span_first.p; N.span_n = c.d_span_n.p; N.span_dense = c.d_span_dense.p;
  N.nspans = (int32_t)c.span_first.size(); N.err = err.p; N.gkeys = gk.p;
  N.strict = !(c.cfg.flags & MSG_F_LOOSE_DOMAIN);
  N.raw = rawp.p; N.off = P.off_pred; N.cnt = P.cnt_pred; N.out = np_.p; N.nout = nn.p; N.nunits = nn.p + 2 * ncmd;
  N.npages = nn.p + 4 * ncmd;
  k_normalize<<<ncmd, kNormThreads, 0, st>>>(N);
  MSG_CHECK_LAUNCH();
  N.raw = rawa.p; N.off = P.off_act; N.cnt = P.cnt_act; N.out = na_.p; N.nout = nn.p + ncmd; N.nunits = nn.p + 3 * ncmd;
  N.npages = nn.p + 5 * ncmd;
  k_normalize<<<ncmd, kNormThreads, 0, st>>>(N);
  MSG_CHECK_LAUNCH(); add_launches(2);
  MSG_CUDA(cudaMemcpyAsync(hn, nn.p, 3 * n2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaMemcpyAsync(herr, err.p, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  MSG_CUDA(cudaStreamSynchronize(st));
  if (herr[0] == 2) throw Error(MSG_E_DOMAIN, "predicted or accessed page outside the dense page map");

  // append to the task CSR and the global pools
  int64_t pp = t.pred_off.back(), pa = t.act_off.back();
  for (int i = 0; i < ncmd; ++i) {
    dst[i] = pp; pp += hn[i];
    dst[ncmd + i] = pa; pa += hn[ncmd + i];
    t.pred_off.push_back(pp);
    t.act_off.push_back(pa);
    t.pred_units.push_back(t.pred_units.back() + hn[2 * ncmd + i]);
    t.act_units.push_back(t.act_units.back() + hn[3 * ncmd + i]);
    t.act_pages.push_back(hn[5 * ncmd + i]);
    t.selfpop.push_back(cmds[i].kind == MSG_CMD_H2D);
    t.kind.push_back((uint8_t)cmds[i].kind);
  }
  t.pred_pool.resize(std::max<int64_t>(pp, 1), st);
  t.act_pool.resize(std::max<int64_t>(pa, 1), st);
  auto& ddst = S.dst; ddst.fit(2 * (int64_t)ncmd);
  MSG_CUDA(cudaMemcpyAsync(ddst.p, dst, n2 * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  k_compact_iv<<<std::min(ncmd, 4096), 128, 0, st>>>(np_.p, P.off_pred, nn.p, ddst.p, t.pred_pool.p, ncmd);
  k_compact_iv<<<std::min(ncmd, 4096), 128, 0, st>>>(na_.p, P.off_act, nn.p + ncmd, ddst.p + ncmd, t.act_pool.p, ncmd);
  MSG_CHECK_LAUNCH(); add_launches(2);
  t.ncmd += ncmd;
  // device copies of the task's CSR offsets and flags
  t.d_pred_off.resize(t.pred_off.size(), st);
  t.d_act_off.resize(t.act_off.size(), st);
  t.d_selfpop.resize(std::max<size_t>(t.selfpop.size(), 1), st);
  MSG_CUDA(cudaMemcpyAsync(t.d_pred_off.p, t.pred_off.data(), t.pred_off.size() * 8, cudaMemcpyHostToDevice, st));
  MSG_CUDA(cudaMemcpyAsync(t.d_act_off.p, t.act_off.data(), t.act_off.size() * 8, cudaMemcpyHostToDevice, st));
  if (!t.selfpop.empty())
    MSG_CUDA(cudaMemcpyAsync(t.d_selfpop.p, t.selfpop.data(), t.selfpop.size(), cudaMemcpyHostToDevice, st));
  MSG_CUDA(cudaStreamSynchronize(st));  // host vectors above are stack temporaries
}

}  // namespace msg
