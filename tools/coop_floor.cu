// Fixed cost of the multisplit's launch shape, with no list work: a
// cooperative launch of one 1024-thread CTA per SM with 224 KB of dynamic
// shared memory, optionally a 112 KB TMA-sized global read per CTA and one
// grid barrier.  Timed with CUDA events (back to back, stream busy) and with
// %globaltimer inside the kernel (first CTA start to last CTA end).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o coop_floor tools/coop_floor.cu && ./coop_floor
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_first = ~0ull, g_last = 0;
__device__ __forceinline__ unsigned long long now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(1024, 1) k_floor(int* bar, int target, const int4* src, int per_cta, int4* sink) {
  if (threadIdx.x == 0) atomicMin(&g_first, now());
  extern __shared__ int4 sm[];
  int4 acc = make_int4(0, 0, 0, 0);
  if (src) {
    const int4* p = src + (size_t)blockIdx.x * per_cta;
    for (int i = threadIdx.x; i < per_cta; i += blockDim.x) {
      int4 v = __ldcs(p + i);
      sm[i % 8192] = v;
      acc.x ^= v.x;
    }
  }
  __syncthreads();
  if (bar) {
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1);
      while (*reinterpret_cast<volatile int*>(bar) < target) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
  }
  if (acc.x == 0x7fffffff) sink[blockIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_last, now());
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 224 * 1024;
  cudaFuncSetAttribute(k_floor, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 200, per_cta = 112 * 1024 / 16;
  int* bars;
  cudaMalloc(&bars, sizeof(int) * (reps + 16) * 4);
  cudaMemset(bars, 0, sizeof(int) * (reps + 16) * 4);
  int4 *src, *sink;
  cudaMalloc(&src, (size_t)sms * per_cta * 16);
  cudaMemset(src, 1, (size_t)sms * per_cta * 16);
  cudaMalloc(&sink, sms * 16);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[4] = {"launch only", "launch + grid barrier", "launch + 112 KB read per CTA",
                          "launch + read + grid barrier"};
  int bi = 0;
  for (int v = 0; v < 4; ++v) {
    const bool use_bar = v & 1, use_src = v & 2;
    double ev_us = 0, dev_us = 0;
    for (int r = -10; r < reps; ++r) {
      unsigned long long init_first = ~0ull, init_last = 0;
      cudaMemcpyToSymbolAsync(g_first, &init_first, 8, 0, cudaMemcpyHostToDevice, st);
      cudaMemcpyToSymbolAsync(g_last, &init_last, 8, 0, cudaMemcpyHostToDevice, st);
      int* bar = use_bar ? bars + (bi++ % (reps + 16)) : nullptr;
      if (use_bar) cudaMemsetAsync(bar, 0, 4, st);
      int target = sms;
      const int4* s = use_src ? src : nullptr;
      int pc = per_cta;
      void* args[] = {&bar, &target, &s, &pc, &sink};
      cudaEventRecord(a, st);
      cudaLaunchCooperativeKernel((void*)k_floor, dim3(sms), dim3(1024), args, smem, st);
      cudaEventRecord(b, st);
      cudaStreamSynchronize(st);
      unsigned long long f, l;
      cudaMemcpyFromSymbol(&f, g_first, 8);
      cudaMemcpyFromSymbol(&l, g_last, 8);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 0) { ev_us += ms * 1e3; dev_us += (l - f) * 1e-3; }
    }
    printf("%-32s events %6.2f us   device %6.2f us\n", names[v], ev_us / reps, dev_us / reps);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
