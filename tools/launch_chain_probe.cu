// Device cost of the per-switch launch chain: a one-CTA kernel (the window
// kernel's shape, ~5 us of work) followed by a one-CTA-per-SM kernel with
// 224 KB of dynamic shared memory (the switch kernel's shape, one grid
// barrier), back to back on one stream, 300 times.  Compares the second
// launch as a cooperative launch and as a plain launch, and the chain
// without the one-CTA kernel.  Reports wall time per chain (events around
// the whole loop, so per-launch event overhead is excluded).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lcp tools/launch_chain_probe.cu && /tmp/lcp
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_one(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
}

__global__ void __launch_bounds__(1024, 1) k_grid(int* bar, int target) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(bar) : "memory");
    int v;
    do { asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while (v < target);
  }
  __syncthreads();
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int reps = 300;
  int* bars;
  cudaMalloc(&bars, sizeof(int) * reps * 8);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int smem : {4096, 224 * 1024}) {
    cudaFuncSetAttribute(k_grid, cudaFuncAttributeMaxDynamicSharedMemorySize, smem < 48 * 1024 ? 48 * 1024 : smem);
    for (int mode = 0; mode < 4; ++mode) {   // bit0: cooperative; bit1: with the one-CTA kernel in front
      const bool coop = mode & 1, one = mode & 2;
      for (int warm = 0; warm < 2; ++warm) {
        cudaMemsetAsync(bars, 0, sizeof(int) * reps * 8, st);
        k_one<<<1, 32, 0, st>>>(20000000);   // 20 ms busy: the host queues the whole loop before it starts
        cudaEventRecord(a, st);
        for (int r = 0; r < reps; ++r) {
          if (one) k_one<<<1, 128, 0, st>>>(5000);
          int* bar = bars + r;
          int target = sms;
          if (coop) {
            void* args[] = {&bar, &target};
            cudaLaunchCooperativeKernel((void*)k_grid, dim3(sms), dim3(1024), args, smem, st);
          } else {
            k_grid<<<sms, 1024, smem, st>>>(bar, target);
          }
        }
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (warm)
          printf("smem %6d  %-11s %-16s %.2f us per chain queued", smem, coop ? "cooperative" : "plain",
                 one ? "one-CTA + grid" : "grid only", ms * 1e3 / reps);
      }
      // the per-call round trip: launch the chain, wait for it (host clock)
      cudaMemsetAsync(bars, 0, sizeof(int) * reps * 8, st);
      cudaStreamSynchronize(st);
      auto t0 = std::chrono::steady_clock::now();
      for (int r = 0; r < reps; ++r) {
        if (one) k_one<<<1, 128, 0, st>>>(5000);
        int* bar = bars + r;
        int target = sms;
        if (coop) {
          void* args[] = {&bar, &target};
          cudaLaunchCooperativeKernel((void*)k_grid, dim3(sms), dim3(1024), args, smem, st);
        } else {
          k_grid<<<sms, 1024, smem, st>>>(bar, target);
        }
        cudaStreamSynchronize(st);
      }
      const double rt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      printf(", %.2f us per round trip  (%s)\n", rt * 1e6 / reps, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
