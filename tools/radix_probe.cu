// Where a pass of the window kernels' block radix sort goes: one 1024-thread
// CTA sorts n random 22-bit keys held in shared memory (the fragmented
// configuration's sizes: 640 endpoints per window, 5120 for the class table),
// SM cycles per sub-phase (zero + count, scan, scatter) summed over the passes,
// block 0, averaged over launches.  Mirrors block_radix_sort in k_plan.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rp tools/radix_probe.cu && /tmp/rp
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ unsigned long long g_ph[4];

template <class T>
__device__ T block_excl_scan(T v, T* smem_warp, T* total) {
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

__device__ __forceinline__ uint32_t match9(int d) {
  uint32_t eq = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1);
    eq &= ((d >> b) & 1) ? bal : ~bal;
  }
  return eq;
}

// 0: match_any ranks; 1: counts by shared atomics, match_any scatter; 2: counts by atomics, ballot-built ranks
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_probe(const uint64_t* keys, int n, int nbits, uint64_t* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* a0 = reinterpret_cast<uint64_t*>(sm);
  uint64_t* b0 = a0 + n;
  int32_t(*cnt)[256] = reinterpret_cast<int32_t(*)[256]>(b0 + n);
  __shared__ int32_t warp_s[32];
  for (int i = threadIdx.x; i < n; i += blockDim.x) a0[i] = keys[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const int per = ((n + 31) / 32 + 31) & ~31;
  const int lo = w * per, hi = lo + per < n ? lo + per : n;
  bool in_b = false;
  unsigned long long t_cnt = 0, t_scan = 0, t_sc = 0;
  for (int sh = 0; sh < nbits; sh += 8) {
    uint64_t* s0 = in_b ? b0 : a0;
    uint64_t* d0 = in_b ? a0 : b0;
    const unsigned long long c0 = clock64();
    for (int j = lane; j < 256; j += 32) cnt[w][j] = 0;
    __syncwarp();
    for (int i0 = lo; i0 < hi; i0 += 32) {
      const int i = i0 + lane;
      const int d = i < hi ? (int)((s0[i] >> sh) & 255) : 256;
      if (MODE == 0) {
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (d < 256 && lane == __ffs(peers) - 1) cnt[w][d] += __popc(peers);
      } else {
        if (d < 256) atomicAdd(&cnt[w][d], 1);
      }
      __syncwarp();
    }
    __syncthreads();
    const unsigned long long c1 = clock64();
    if (MODE < 3) {
      const int d = threadIdx.x >> 2, wq = (threadIdx.x & 3) * 8;
      int32_t sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) sum += cnt[wq + j][d];
      int32_t tot;
      int32_t run = block_excl_scan<int32_t>(sum, warp_s, &tot);
#pragma unroll
      for (int j = 0; j < 8; ++j) { const int32_t c = cnt[wq + j][d]; cnt[wq + j][d] = run; run += c; }
    } else {   // column walk + 256-wide scan (the kernel's scan)
      const int t = threadIdx.x, ln = t & 31, wid = t >> 5;
      int32_t excl = 0;
      if (t < 256) {
        int32_t tot = 0;
#pragma unroll 8
        for (int ww = 0; ww < 32; ++ww) { const int32_t c = cnt[ww][t]; cnt[ww][t] = tot; tot += c; }
        int32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int32_t y = __shfl_up_sync(0xffffffffu, x, o); if (ln >= o) x += y; }
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
    const unsigned long long c2 = clock64();
    for (int i0 = lo; i0 < hi; i0 += 32) {
      const int i = i0 + lane;
      const int d = i < hi ? (int)((s0[i] >> sh) & 255) : 256;
      const uint32_t peers = MODE >= 2 ? match9(d) : __match_any_sync(0xffffffffu, d);
      const int32_t before = d < 256 ? cnt[w][d] : 0;
      __syncwarp();
      if (d < 256) {
        const int o = before + __popc(peers & lt);
        d0[o] = s0[i];
        if (lane == __ffs(peers) - 1) cnt[w][d] = before + __popc(peers);
      }
      __syncwarp();
    }
    __syncthreads();
    const unsigned long long c3 = clock64();
    t_cnt += c1 - c0; t_scan += c2 - c1; t_sc += c3 - c2;
    in_b = !in_b;
  }
  const uint64_t* r = in_b ? b0 : a0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = r[i];
  if (threadIdx.x == 0) { atomicAdd(&g_ph[0], t_cnt); atomicAdd(&g_ph[1], t_scan); atomicAdd(&g_ph[2], t_sc); atomicAdd(&g_ph[3], 1ull); }
}

int main() {
  const int nmax = 5120;
  uint64_t h[nmax];
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < nmax; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s & ((1u << 22) - 1); }
  uint64_t *dk, *dout;
  cudaMalloc(&dk, nmax * 8);
  cudaMalloc(&dout, nmax * 8);
  cudaMemcpy(dk, h, nmax * 8, cudaMemcpyHostToDevice);
  const int smem = 2 * nmax * 8 + 32 * 256 * 4;
  cudaFuncSetAttribute(k_probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int n : {640, 5120}) {
    for (int mode = 0; mode < 4; ++mode) {
      unsigned long long z[4] = {0, 0, 0, 0};
      cudaMemcpyToSymbol(g_ph, z, sizeof(z));
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      for (int r = 0; r < 100; ++r) {
        if (mode == 0) k_probe<0><<<1, 1024, smem>>>(dk, n, 22, dout);
        else if (mode == 1) k_probe<1><<<1, 1024, smem>>>(dk, n, 22, dout);
        else if (mode == 2) k_probe<2><<<1, 1024, smem>>>(dk, n, 22, dout);
        else k_probe<3><<<1, 1024, smem>>>(dk, n, 22, dout);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long o[4];
      cudaMemcpyFromSymbol(o, g_ph, sizeof(o));
      uint64_t res[nmax];
      cudaMemcpy(res, dout, n * 8, cudaMemcpyDeviceToHost);
      bool sorted = true;
      for (int i = 1; i < n; ++i) sorted &= res[i - 1] <= res[i];
      printf("n %5d %-22s kernel %.2f us; per sort (3 passes): count %.2f us, scan %.2f us, scatter %.2f us; sorted %d (%s)\n",
             n, mode == 3 ? "+ column-walk scan" : mode == 2 ? "atomics + ballot ranks" : mode ? "count by smem atomics" : "count by match_any", ms * 1e3 / 100,
             o[0] / (double)o[3] / 1965.0, o[1] / (double)o[3] / 1965.0, o[2] / (double)o[3] / 1965.0, (int)sorted,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
