// Migration engine: each switch's working-set transition as one coalesced
// batch between pinned host DRAM and the HBM frame arena.
//
// The planner leaves a list of (page, frame) pairs: evictions first (head
// order), then installs (populate order).  This file
//   1. cuts the list into maximal segments that are contiguous in both the
//      host backing (slot = dense page mod pool pages) and the frame arena;
//   2. moves large segments with the copy engines (one cudaMemcpyAsync per
//      segment piece, one stream per direction so D2H and H2D overlap, full
//      duplex), gating each
//      install chunk on the eviction chunk that frees its frames — the real
//      counterpart of the pipelined-swap model (engine.py:139-166);
//   3. moves fragmented batches with SM gather/scatter kernels reading and
//      writing mapped pinned memory with 16-byte accesses.
#include "msched_internal.cuh"

#include <cuda.h>   // stream memory-op types only; the entry points come from cudaGetDriverEntryPoint

#include <algorithm>
#include <cstdlib>

namespace msg {

constexpr int64_t kTagMagic = 0x5a17c0de00000000ll;
constexpr int64_t kSegCeMax = 1 << 16;   // CE path limit on segments per batch
constexpr int64_t kMinCePages = 8;       // average segment size for the CE path (pages)

__host__ __device__ __forceinline__ int64_t tag_of(int64_t page) { return kTagMagic ^ page; }

__global__ void k_seg_mark(const int64_t* list, int64_t n, int64_t n_d2h, int64_t pool_pages, int32_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool b = (i == 0 || i == n_d2h);
    if (!b) {
      int64_t x = list[i], y = list[i - 1];
      int64_t p = x >> 32, q = y >> 32;
      int32_t f = (int32_t)(uint32_t)(x & 0xffffffff), g = (int32_t)(uint32_t)(y & 0xffffffff);
      b = (p != q + 1) || (f != g + 1) || (p % pool_pages == 0);
    }
    flag[i] = b ? 1 : 0;
  }
}

__global__ void k_seg_write(const int64_t* list, int64_t n, const int32_t* flag, const int64_t* off, int64_t* segs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (flag[i]) {
      int64_t k = off[i];
      segs[2 * k] = i;
      segs[2 * k + 1] = list[i];
    }
  }
}

// SM path: one warp per page, 16-byte accesses (page size multiple of 512 B)
__global__ void k_sm_copy(const int64_t* list, int64_t n, char* arena, char* pool, int64_t P, int64_t pool_pages,
                          int to_host) {
  int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t v16 = P / 16;
  for (int64_t i = warp; i < n; i += nwarps) {
    int64_t x = list[i];
    int64_t page = x >> 32;
    int64_t frame = (int64_t)(uint32_t)(x & 0xffffffff);
    int4* a = reinterpret_cast<int4*>(arena + frame * P);
    int4* h = reinterpret_cast<int4*>(pool + (page % pool_pages) * P);
    if (to_host) {
      for (int64_t k = lane; k < v16; k += 32) h[k] = a[k];
    } else {
      for (int64_t k = lane; k < v16; k += 32) a[k] = h[k];
    }
  }
}

__global__ void k_write_tags(const int64_t* list, int64_t n, char* arena, int64_t P) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = list[i];
    int64_t page = x >> 32, frame = (int64_t)(uint32_t)(x & 0xffffffff);
    *reinterpret_cast<int64_t*>(arena + frame * P) = tag_of(page);
  }
}

__global__ void k_verify(const uint32_t* bits, const int32_t* frame, int64_t D, const char* arena, int64_t P,
                         unsigned long long* bad) {
  unsigned long long nb = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < D; p += (int64_t)gridDim.x * blockDim.x) {
    bool res = (bits[p >> 5] >> (p & 31)) & 1u;
    int32_t f = frame[p];
    if (res != (f >= 0)) { ++nb; continue; }
    if (res && *reinterpret_cast<const int64_t*>(arena + (int64_t)f * P) != tag_of(p)) ++nb;
  }
  if (nb) atomicAdd(bad, nb);
}

// Stream memory operations (populate progress counter written by the H2D
// stream, waited on by the command stream).  Resolved through the runtime so
// the library does not link libcuda directly.
typedef CUresult (*PfnWait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PfnWrite64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
static PfnWait64 p_wait64 = nullptr;
static PfnWrite64 p_write64 = nullptr;

static void stream_memops_init() {
  if (p_wait64 && p_write64) return;
  cudaDriverEntryPointQueryResult q1, q2;
  MSG_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue64", reinterpret_cast<void**>(&p_wait64), cudaEnableDefault, &q1));
  MSG_CUDA(cudaGetDriverEntryPoint("cuStreamWriteValue64", reinterpret_cast<void**>(&p_write64), cudaEnableDefault, &q2));
  if (q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !p_wait64 || !p_write64)
    throw Error(MSG_E_CUDA, "cuStreamWaitValue64 / cuStreamWriteValue64 unavailable");
}

static void write_progress(Ctx& c, cudaStream_t st, int64_t value) {
  if (!c.d_progress || !(c.cfg.flags & MSG_F_EXECUTE)) return;
  CUresult r = p_write64(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(c.d_progress), (cuuint64_t)value,
                         CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) throw Error(MSG_E_CUDA, "cuStreamWriteValue64 failed (" + std::to_string((int)r) + ")");
}

void migration_init(Ctx& c) {
  MSG_CUDA(cudaStreamCreateWithFlags(&c.st_d2h, cudaStreamNonBlocking));
  MSG_CUDA(cudaStreamCreateWithFlags(&c.st_h2d, cudaStreamNonBlocking));
  MSG_CUDA(cudaEventCreateWithFlags(&c.ev_mig[0], cudaEventDisableTiming));
  MSG_CUDA(cudaEventCreateWithFlags(&c.ev_mig[1], cudaEventDisableTiming));
  MSG_CUDA(cudaEventCreateWithFlags(&c.ev_h2d_done, cudaEventDisableTiming));
  MSG_CUDA(cudaEventCreateWithFlags(&c.ev_plan_done, cudaEventDisableTiming));
  MSG_CUDA(cudaEventCreateWithFlags(&c.ev_d2h_prev, cudaEventDisableTiming));
  MSG_CUDA(cudaEventRecord(c.ev_d2h_prev, c.st));
  MSG_CUDA(cudaEventRecord(c.ev_mig[0], c.st));
  MSG_CUDA(cudaEventRecord(c.ev_mig[1], c.st));
  MSG_CUDA(cudaEventRecord(c.ev_h2d_done, c.st));
  MSG_CUDA(cudaEventRecord(c.ev_plan_done, c.st));
  if (!(c.cfg.flags & (MSG_F_MIGRATE | MSG_F_VERIFY_TAGS))) return;
  if (c.P % 512 != 0) throw Error(MSG_E_INVAL, "migration needs page_size to be a multiple of 512 bytes");
  size_t abytes = (size_t)c.C * (size_t)c.P;
  if (cudaMalloc(&c.arena, abytes) != cudaSuccess) {
    cudaGetLastError();
    throw Error(MSG_E_OOM, "HBM frame arena of " + std::to_string(abytes) + " bytes does not fit");
  }
  c.pool_pages = c.cfg.host_pool_pages > 0 ? std::min<int64_t>(c.cfg.host_pool_pages, c.D) : c.D;
  if (c.pool_pages < 1) c.pool_pages = 1;
  size_t pbytes = (size_t)c.pool_pages * (size_t)c.P;
  if (cudaHostAlloc(reinterpret_cast<void**>(&c.pool), pbytes, cudaHostAllocMapped | cudaHostAllocPortable) !=
      cudaSuccess) {
    cudaGetLastError();
    throw Error(MSG_E_OOM, "pinned host pool of " + std::to_string(pbytes) + " bytes failed");
  }
  MSG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.pool_dev), c.pool, 0));
  if (c.cfg.flags & MSG_F_MIGRATE) {
    stream_memops_init();
    MSG_CUDA(cudaStreamCreateWithFlags(&c.st_run, cudaStreamNonBlocking));
    MSG_CUDA(cudaEventCreateWithFlags(&c.ev_run_last, cudaEventDisableTiming));
    MSG_CUDA(cudaMalloc(&c.d_progress, 8));
    MSG_CUDA(cudaMalloc(&c.d_run_acc, 4 * 8));
    MSG_CUDA(cudaMemsetAsync(c.d_progress, 0, 8, c.st));
    MSG_CUDA(cudaMemsetAsync(c.d_run_acc, 0, 4 * 8, c.st));
    c.inst_ep.exact(std::max<int64_t>(c.C, 1));
    c.free_ep.exact(std::max<int64_t>(c.C, 1));
    MSG_CUDA(cudaMemsetAsync(c.inst_ep.p, 0xff, c.C * 4, c.st));
    MSG_CUDA(cudaMemsetAsync(c.free_ep.p, 0xff, c.C * 4, c.st));
  }
  if (c.cfg.flags & MSG_F_VERIFY_TAGS) {
    for (int64_t s = 0; s < c.pool_pages; ++s) *reinterpret_cast<int64_t*>(c.pool + s * c.P) = kTagMagic ^ s;
  }
}

static double sum_pairs(std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
  double t = 0;
  for (auto& pr : v) { float ms = 0; if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) t += ms; }
  cudaGetLastError();
  v.clear();
  return t;
}

// A long-lived context (no reset between replays) would otherwise keep every
// per-batch and per-chunk event: past a bound, wait for the streams, fold the
// busy-time pairs into running sums and release the events.  Batch events
// become null (the batches are complete; nothing needs to wait on them).
void fold_events(Ctx& c, size_t bound) {
  if (c.ev_pool.size() <= bound) return;
  for (cudaStream_t s : {c.st, c.st_d2h, c.st_h2d, c.st_run})
    if (s) MSG_CUDA(cudaStreamSynchronize(s));
  ms_harvest(c);
  c.fold_h2d_ms += sum_pairs(c.busy_h2d);
  c.fold_d2h_ms += sum_pairs(c.busy_d2h);
  c.fold_ms_ms += sum_pairs(c.busy_ms);
  c.fold_run_ms += sum_pairs(c.busy_run);
  for (auto e : c.ev_pool) cudaEventDestroy(e);
  c.ev_pool.clear();
  std::fill(c.ev_d2h_of.begin(), c.ev_d2h_of.end(), nullptr);
  std::fill(c.ev_h2d_of.begin(), c.ev_h2d_of.end(), nullptr);
}

static cudaEvent_t new_event(Ctx& c, bool timing) {
  cudaEvent_t e;
  MSG_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  c.ev_pool.push_back(e);
  return e;
}

// Issues the pending copy-engine pieces of one direction on `st`, one
// cudaMemcpyAsync each (the segments are maximal runs contiguous on both
// sides, so a piece is a large copy: cfg4 averages ~100 pieces per switch).
static void ce_batch(std::vector<void*>& d, std::vector<void*>& s, std::vector<size_t>& z, cudaStream_t st,
                     cudaMemcpyKind kind) {
  for (size_t i = 0; i < d.size(); ++i) MSG_CUDA(cudaMemcpyAsync(d[i], s[i], z[i], kind, st));
  d.clear(); s.clear(); z.clear();
}

void migrate_batch(Ctx& c, int64_t n_d2h, int64_t n_h2d, int64_t free_before, bool copy_h2d) {
  int par = c.mig_par;
  int64_t n = n_d2h + n_h2d;
  const int64_t* list = c.mig_list[par].p;
  bool real = c.cfg.flags & MSG_F_MIGRATE;
  if (n == 0) return;
  if (!real) {
    // bookkeeping only: frames receive their page's tag as if the copy happened
    if (n_h2d) {
      k_write_tags<<<std::min<int64_t>((n_h2d + 255) / 256, 1184), 256, 0, c.st>>>(list + n_d2h, n_h2d, c.arena, c.P);
      MSG_CHECK_LAUNCH();
      add_launches(1);
    }
    MSG_CUDA(cudaEventRecord(c.ev_mig[par], c.st));
    c.mig_par ^= 1;
    return;
  }
  const int64_t base = c.installed_total;   // populate progress before this batch
  c.installed_total = base + n_h2d;
  if (c.run_used) run_wait_before_copies(c);
  // 1. segments
  c.s.mflag.resize(n, c.st);
  c.s.moff.resize(n, c.st);
  c.s.msegs.resize(2 * n + 2, c.st);
  int grid = (int)std::min<int64_t>((n + 255) / 256, 1184);
  k_seg_mark<<<grid, 256, 0, c.st>>>(list, n, n_d2h, c.pool_pages, c.s.mflag.p);
  MSG_CHECK_LAUNCH();
  scan_flags(c, c.s.mflag.p, n, c.s.moff.p);
  k_seg_write<<<grid, 256, 0, c.st>>>(list, n, c.s.mflag.p, c.s.moff.p, c.s.msegs.p);
  MSG_CHECK_LAUNCH();
  add_launches(2);
  int64_t* hb = c.hbuf.p;
  MSG_CUDA(cudaMemcpyAsync(hb, c.s.moff.p + n - 1, 8, cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaMemcpyAsync(hb + 1, c.s.mflag.p + n - 1, 4, cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaMemcpyAsync(hb + 2, &c.dstate->aux[0], 8, cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaStreamSynchronize(c.st));
  int64_t nseg = hb[0] + (int64_t)(*reinterpret_cast<int32_t*>(hb + 1));
  bool use_ce = nseg <= kSegCeMax && n >= kMinCePages * nseg;
  cudaEvent_t planned = new_event(c, false);
  MSG_CUDA(cudaEventRecord(planned, c.st));
  // frames written by earlier installs must land before they are read back
  int32_t dep_d2h = reinterpret_cast<int32_t*>(hb + 2)[0];   // newest H2D batch whose frames we evict
  int32_t dep_h2d = reinterpret_cast<int32_t*>(hb + 2)[1];   // newest D2H batch that freed reused frames
  cudaEvent_t d2h_start = new_event(c, true), d2h_end = new_event(c, true);
  cudaEvent_t h2d_start = new_event(c, true), h2d_end = new_event(c, true);
  if (!use_ce) {
    c.stats.sm_batches++;
    MSG_CUDA(cudaStreamWaitEvent(c.st_h2d, planned, 0));
    MSG_CUDA(cudaStreamWaitEvent(c.st_h2d, c.ev_d2h_prev, 0));
    MSG_CUDA(cudaStreamWaitEvent(c.st_h2d, c.ev_h2d_done, 0));
    MSG_CUDA(cudaEventRecord(d2h_start, c.st_h2d));
    if (n_d2h) k_sm_copy<<<296, 256, 0, c.st_h2d>>>(list, n_d2h, c.arena, c.pool_dev, c.P, c.pool_pages, 1);
    MSG_CUDA(cudaEventRecord(d2h_end, c.st_h2d));
    MSG_CUDA(cudaEventRecord(h2d_start, c.st_h2d));
    if (n_h2d) {
      if (copy_h2d) k_sm_copy<<<296, 256, 0, c.st_h2d>>>(list + n_d2h, n_h2d, c.arena, c.pool_dev, c.P, c.pool_pages, 0);
      else if (c.cfg.flags & MSG_F_VERIFY_TAGS)
        k_write_tags<<<std::min<int64_t>((n_h2d + 255) / 256, 1184), 256, 0, c.st_h2d>>>(list + n_d2h, n_h2d, c.arena, c.P);
    }
    MSG_CHECK_LAUNCH();
    add_launches(2);
    write_progress(c, c.st_h2d, base + n_h2d);
    MSG_CUDA(cudaEventRecord(h2d_end, c.st_h2d));
    MSG_CUDA(cudaEventRecord(c.ev_h2d_done, c.st_h2d));
    MSG_CUDA(cudaEventRecord(c.ev_d2h_prev, c.st_h2d));
    MSG_CUDA(cudaEventRecord(c.ev_mig[par], c.st_h2d));
    if (copy_h2d) c.stats.h2d_bytes += n_h2d * c.P;
    c.stats.d2h_bytes += n_d2h * c.P;
  } else {
    c.stats.ce_batches++;
    std::vector<int64_t> segs(2 * nseg);
    MSG_CUDA(cudaMemcpyAsync(segs.data(), c.s.msegs.p, 2 * nseg * 8, cudaMemcpyDeviceToHost, c.st));
    MSG_CUDA(cudaStreamSynchronize(c.st));
    MSG_CUDA(cudaEventRecord(c.ev_mig[par], c.st));  // the device list is no longer needed
    auto seg_at = [&](int64_t k, int64_t* i0, int64_t* len, int64_t* page, int64_t* frame) {
      *i0 = segs[2 * k];
      int64_t nxt = k + 1 < nseg ? segs[2 * (k + 1)] : n;
      *len = nxt - *i0;
      *page = segs[2 * k + 1] >> 32;
      *frame = (int64_t)(uint32_t)(segs[2 * k + 1] & 0xffffffff);
    };
    // evictions, in chunks of ~64 MiB (8..128 per batch); each chunk's
    // completion is an event that gates the installs reusing its frames.
    // Segments are split at chunk boundaries, so one huge contiguous segment
    // (2 MiB pages, whole GEMM operands) still pipelines.
    static const int64_t kChunkBytes = getenv("MSG_MIG_CHUNK_MB") ? atoll(getenv("MSG_MIG_CHUNK_MB")) << 20 : 64ll << 20;
    int64_t nchunks = std::min<int64_t>(std::max<int64_t>((n_d2h * c.P + kChunkBytes - 1) / kChunkBytes, 8), 128);
    int64_t chunk = std::max<int64_t>((n_d2h + nchunks - 1) / nchunks, 1);
    std::vector<std::pair<int64_t, cudaEvent_t>> done;   // (evictions complete up to, event)
    std::vector<void*> dd, ss;
    std::vector<size_t> zz;
    if (dep_d2h >= 0 && dep_d2h < (int32_t)c.ev_h2d_of.size() && c.ev_h2d_of[dep_d2h])   // null: folded, done
      MSG_CUDA(cudaStreamWaitEvent(c.st_d2h, c.ev_h2d_of[dep_d2h], 0));
    MSG_CUDA(cudaEventRecord(d2h_start, c.st_d2h));
    int64_t k = 0, next_cut = chunk;
    for (; k < nseg; ++k) {
      int64_t i0, len, page, frame;
      seg_at(k, &i0, &len, &page, &frame);
      if (i0 >= n_d2h) break;
      for (int64_t pos = i0; pos < i0 + len;) {
        int64_t take = std::min(i0 + len, next_cut) - pos;
        dd.push_back(c.pool + ((page + (pos - i0)) % c.pool_pages) * c.P);
        ss.push_back(c.arena + (frame + (pos - i0)) * c.P);
        zz.push_back((size_t)(take * c.P));
        c.stats.d2h_bytes += take * c.P;
        c.stats.d2h_segments++;
        pos += take;
        if (pos == next_cut && pos < n_d2h) {
          ce_batch(dd, ss, zz, c.st_d2h, cudaMemcpyDeviceToHost);
          cudaEvent_t e = new_event(c, false);
          MSG_CUDA(cudaEventRecord(e, c.st_d2h));
          done.push_back({pos, e});
          next_cut += chunk;
        }
      }
    }
    ce_batch(dd, ss, zz, c.st_d2h, cudaMemcpyDeviceToHost);
    MSG_CUDA(cudaEventRecord(d2h_end, c.st_d2h));
    done.push_back({n_d2h, d2h_end});
    // installs: frames that were free before this batch may still be draining
    // from earlier evictions; frames freed by this batch wait for their chunk
    if (dep_h2d >= 0 && dep_h2d < (int32_t)c.ev_d2h_of.size() && c.ev_d2h_of[dep_h2d])   // null: folded, done
      MSG_CUDA(cudaStreamWaitEvent(c.st_h2d, c.ev_d2h_of[dep_h2d], 0));
    // a page evicted by an earlier batch (its D2H writes the page's host
    // slot) may be re-installed now into a frame that was already free: the
    // H2D reading that slot must follow the earlier batch's write-back
    MSG_CUDA(cudaStreamWaitEvent(c.st_h2d, c.ev_d2h_prev, 0));
    MSG_CUDA(cudaEventRecord(h2d_start, c.st_h2d));
    size_t waited = 0;
    bool any_wait = false;
    // installs go in populate order; after every flushed copy batch the H2D
    // stream publishes how many of them have landed (the early-start progress
    // that executed commands wait on), at least every 1/16 of the batch
    const bool publish = (c.cfg.flags & MSG_F_EXECUTE) != 0;   // only executed commands read the progress
    const int64_t h2d_chunk = publish ? std::max<int64_t>((n_h2d + 15) / 16, 256) : INT64_MAX;
    int64_t issued = 0, published = 0;
    auto flush_h2d = [&]() {
      ce_batch(dd, ss, zz, c.st_h2d, cudaMemcpyHostToDevice);
      if (publish && copy_h2d && issued > published) {
        write_progress(c, c.st_h2d, base + issued);
        published = issued;
      }
    };
    for (; k < nseg; ++k) {
      int64_t i0, len, page, frame;
      seg_at(k, &i0, &len, &page, &frame);
      for (int64_t pos = i0; pos < i0 + len;) {
        // install j = pos - n_d2h reuses the frame of eviction j - free_before;
        // cut pieces where that eviction index crosses a chunk boundary
        int64_t j = pos - n_d2h, take = i0 + len - pos;
        int64_t e0 = j - free_before;
        if (e0 < 0) take = std::min(take, -e0);                       // frames free before the batch
        else take = std::min(take, (e0 / chunk + 1) * chunk - e0);   // up to the next chunk boundary
        int64_t e_idx = e0 + take - 1;   // last eviction this piece depends on
        if (e_idx >= 0) {
          size_t need = 0;
          while (need + 1 < done.size() && done[need].first <= e_idx) ++need;
          if (!any_wait || need > waited) {
            flush_h2d();
            MSG_CUDA(cudaStreamWaitEvent(c.st_h2d, done[need].second, 0));
            waited = need;
            any_wait = true;
          }
        }
        if (copy_h2d && issued - published >= h2d_chunk) flush_h2d();
        issued = j + take;
        if (copy_h2d) {
          dd.push_back(c.arena + (frame + (pos - i0)) * c.P);
          ss.push_back(c.pool + ((page + (pos - i0)) % c.pool_pages) * c.P);
          zz.push_back((size_t)(take * c.P));
          c.stats.h2d_bytes += take * c.P;
          c.stats.h2d_segments++;
        }
        pos += take;
      }
    }
    flush_h2d();
    if (!copy_h2d && (c.cfg.flags & MSG_F_VERIFY_TAGS) && n_h2d) {
      // installs that carry their own data (memcpy): stamp the frames instead
      MSG_CUDA(cudaStreamWaitEvent(c.st_h2d, d2h_end, 0));
      MSG_CUDA(cudaStreamWaitEvent(c.st_h2d, planned, 0));
      k_write_tags<<<std::min<int64_t>((n_h2d + 255) / 256, 1184), 256, 0, c.st_h2d>>>(list + n_d2h, n_h2d, c.arena, c.P);
      MSG_CHECK_LAUNCH();
      add_launches(1);
      MSG_CUDA(cudaEventRecord(c.ev_mig[par], c.st_h2d));
    }
    write_progress(c, c.st_h2d, base + n_h2d);
    MSG_CUDA(cudaEventRecord(h2d_end, c.st_h2d));
    MSG_CUDA(cudaEventRecord(c.ev_h2d_done, c.st_h2d));
    MSG_CUDA(cudaEventRecord(c.ev_d2h_prev, c.st_d2h));
  }
  c.busy_d2h.push_back({d2h_start, d2h_end});
  c.ev_d2h_of.push_back(use_ce ? d2h_end : h2d_end);
  c.ev_h2d_of.push_back(h2d_end);
  c.mig_batch++;
  c.busy_h2d.push_back({h2d_start, h2d_end});
  c.mig_par ^= 1;
}

// ---------------------------------------------------------------------------
// Executed commands: the slice's kernels, started as soon as the populate
// prefix they need has landed (the paper's GPU trackers + events,
// PAPER.md:1000-1009; the early-start model of engine.py:139-158, 373-378).
// Each reads every page of its actual set from its HBM frame.

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// lat_ns: the command's profiled duration; every CTA stays resident until
// that long after it started (the grid is sized to be co-resident: at most
// kConsumeCtasPerSm CTAs of 256 threads per SM), so the command occupies its
// modeled latency even when its reads finish sooner
constexpr int kConsumeCtasPerSm = 4;
__global__ void __launch_bounds__(256, kConsumeCtasPerSm) k_consume(const Iv* __restrict__ iv, int64_t n_iv, const int32_t* __restrict__ frame,
                          const char* __restrict__ arena, int64_t P, int verify, unsigned long long* acc,
                          uint64_t lat_ns) {
  const uint64_t t_start = lat_ns ? globaltimer_ns() : 0;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t v16 = P / 16;
  unsigned long long pages = 0, bad = 0, miss = 0;
  int4 x = make_int4(0, 0, 0, 0);
  int64_t skip = 0;
  for (int64_t r = 0; r < n_iv; ++r) {
    const Iv v = iv[r];
    const int64_t np = v.b - v.a;
    // this warp's first page in range r: global page index = skip + k
    int64_t k0 = warp - skip % nwarps;
    if (k0 < 0) k0 += nwarps;
    for (int64_t k = k0; k < np; k += nwarps) {
      const int64_t d = v.d + k;
      const int32_t f = frame[d];
      if (f < 0) { if (lane == 0) ++miss; continue; }
      const int4* src = reinterpret_cast<const int4*>(arena + (int64_t)f * P);
      for (int64_t q = lane; q < v16; q += 32) {
        int4 y = __ldcs(src + q);
        x.x ^= y.x; x.y ^= y.y; x.z ^= y.z; x.w ^= y.w;
      }
      if (lane == 0) {
        ++pages;
        if (verify && *reinterpret_cast<const int64_t*>(arena + (int64_t)f * P) != tag_of(d)) ++bad;
      }
    }
    skip += np;
  }
  pages = __reduce_add_sync(0xffffffffu, (unsigned)pages);
  bad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
  miss = __reduce_add_sync(0xffffffffu, (unsigned)miss);
  unsigned sig = __reduce_xor_sync(0xffffffffu, (unsigned)(x.x ^ x.y ^ x.z ^ x.w));
  if (lane == 0) {
    if (pages) atomicAdd(&acc[0], pages);
    if (bad) atomicAdd(&acc[1], bad);
    if (miss) atomicAdd(&acc[2], miss);
    atomicXor(&acc[3], (unsigned long long)sig);
  }
  if (lat_ns && threadIdx.x == 0) {
    while (globaltimer_ns() - t_start < lat_ns) __nanosleep(2000);
  }
}

// copies of a new batch must not evict or overwrite frames that executed
// commands may still be reading
void run_wait_before_copies(Ctx& c) {
  MSG_CUDA(cudaStreamWaitEvent(c.st_d2h, c.ev_run_last, 0));
  MSG_CUDA(cudaStreamWaitEvent(c.st_h2d, c.ev_run_last, 0));
}

void run_command(Ctx& c, int32_t task, int32_t cmd, int64_t need_pages, double latency_s) {
  if (!(latency_s >= 0.0 && latency_s <= 60.0)) throw Error(MSG_E_INVAL, "command latency outside [0, 60] s");
  if (!c.nsm) MSG_CUDA(cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, c.device));
  if (!(c.cfg.flags & MSG_F_MIGRATE) || !(c.cfg.flags & MSG_F_EXECUTE) || !c.st_run)
    throw Error(MSG_E_INVAL, "executing commands needs MSG_F_MIGRATE | MSG_F_EXECUTE");
  if (task < 0 || task >= (int32_t)c.tasks.size() || !c.tasks[task]) throw Error(MSG_E_INVAL, "unknown task");
  TaskTab& t = *c.tasks[task];
  if (cmd < 0 || cmd >= t.ncmd) throw Error(MSG_E_INVAL, "bad command index");
  if (need_pages < 0) throw Error(MSG_E_INVAL, "negative gating prefix");
  if (c.gate_task == task && cmd >= c.gate_c0 && cmd - c.gate_c0 < (int64_t)c.gate_need.size())
    need_pages = std::max<int64_t>(need_pages, c.gate_need[cmd - c.gate_c0]);
  int64_t want = c.switch_base + need_pages;
  if (c.fault_task == task && c.fault_cmd == cmd) want = std::max(want, c.fault_total);
  // a wait on a value no issued copy will ever publish would hang the stream
  if (want > c.installed_total) throw Error(MSG_E_INVAL, "gating prefix beyond the issued populate copies");
  // the frame table of the plan that made the pages resident
  cudaEvent_t planned = new_event(c, false);
  MSG_CUDA(cudaEventRecord(planned, c.st));
  MSG_CUDA(cudaStreamWaitEvent(c.st_run, planned, 0));
  if (want > 0) {
    CUresult r = p_wait64(reinterpret_cast<CUstream>(c.st_run), reinterpret_cast<CUdeviceptr>(c.d_progress),
                          (cuuint64_t)want, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) throw Error(MSG_E_CUDA, "cuStreamWaitValue64 failed (" + std::to_string((int)r) + ")");
  }
  cudaEvent_t e0 = new_event(c, true), e1 = new_event(c, true);
  MSG_CUDA(cudaEventRecord(e0, c.st_run));
  int64_t i0 = t.act_off[cmd], niv = t.act_off[cmd + 1] - i0;
  int64_t pages = 0;
  const uint64_t lat_ns = (uint64_t)(latency_s * 1e9 + 0.5);
  if (niv || lat_ns) {
    // bitmap-word units bound the page count (enough to size the grid)
    pages = (t.act_units[cmd + 1] - t.act_units[cmd]) * 32;
    int blocks = (int)std::min<int64_t>(std::max<int64_t>((pages + 7) / 8, 1), (int64_t)std::max(c.nsm, 1) * kConsumeCtasPerSm);
    k_consume<<<blocks, 256, 0, c.st_run>>>(t.act_pool.p + i0, niv, c.frame.p, c.arena, c.P,
                                             (c.cfg.flags & MSG_F_VERIFY_TAGS) ? 1 : 0, c.d_run_acc, lat_ns);
    MSG_CHECK_LAUNCH();
    add_launches(1);
  }
  MSG_CUDA(cudaEventRecord(e1, c.st_run));
  MSG_CUDA(cudaEventRecord(c.ev_run_last, c.st_run));
  c.busy_run.push_back({e0, e1});
  c.run_used = true;
  c.stats.run_cmds++;
}

void verify_tags(Ctx& c, int64_t* bad) {
  if (!(c.cfg.flags & MSG_F_VERIFY_TAGS)) throw Error(MSG_E_INVAL, "context created without MSG_F_VERIFY_TAGS");
  if (c.pool_pages < c.D) throw Error(MSG_E_INVAL, "tag verification needs an unaliased host pool");
  MSG_CUDA(cudaDeviceSynchronize());
  unsigned long long* d = nullptr;
  MSG_CUDA(cudaMalloc(&d, 8));
  MSG_CUDA(cudaMemset(d, 0, 8));
  k_verify<<<1184, 256, 0, c.st>>>(c.bits.p, c.frame.p, c.D, c.arena, c.P, d);
  MSG_CHECK_LAUNCH();
  add_launches(1);
  unsigned long long h = 0;
  MSG_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, c.st));
  // non-resident pages: their host slot must hold their own payload (an
  // eviction that copied the wrong frame back would only show up here)
  std::vector<uint32_t> words((c.D + 31) / 32 + 1);
  MSG_CUDA(cudaMemcpyAsync(words.data(), c.bits.p, words.size() * 4, cudaMemcpyDeviceToHost, c.st));
  MSG_CUDA(cudaStreamSynchronize(c.st));
  cudaFree(d);
  for (int64_t p = 0; p < c.D; ++p) {
    if ((words[p >> 5] >> (p & 31)) & 1u) continue;
    if (*reinterpret_cast<const int64_t*>(c.pool + p * c.P) != tag_of(p)) ++h;
  }
  *bad = (int64_t)h;
}

}  // namespace msg
