// Host-side cost of launching while the stream is busy: a spinning kernel
// occupies the stream, then we time (host clock) a plain launch and a
// cooperative launch of a trivial grid-wide kernel queued behind it.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

__global__ void spin(long long ns) {
  long long t0 = clock64();
  while (clock64() - t0 < ns * 2) {}
}
__global__ void trivial(int* p) { if (threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }

int main() {
  int* d; cudaMalloc(&d, 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto now = [] { return std::chrono::steady_clock::now(); };
  for (int shape = 0; shape < 3; ++shape) {
    int grid = shape == 0 ? sms : shape == 1 ? 4 * sms : 1;
    int threads = shape == 0 ? 1024 : 512;
    for (int mode = 0; mode < 2; ++mode) {
      double busy = 0, idle = 0;
      for (int r = 0; r < 50; ++r) {
        cudaStreamSynchronize(s);
        auto t0 = now();
        void* args[] = {&d};
        if (mode) cudaLaunchCooperativeKernel((void*)trivial, dim3(grid), dim3(threads), args, 0, s);
        else trivial<<<grid, threads, 0, s>>>(d);
        idle += std::chrono::duration<double>(now() - t0).count();
        spin<<<1, 32, 0, s>>>(100000);   // ~100 us busy
        auto t1 = now();
        if (mode) cudaLaunchCooperativeKernel((void*)trivial, dim3(grid), dim3(threads), args, 0, s);
        else trivial<<<grid, threads, 0, s>>>(d);
        busy += std::chrono::duration<double>(now() - t1).count();
      }
      cudaStreamSynchronize(s);
      printf("grid %4d x %4d %-12s host us per launch: idle stream %.1f, behind a 100 us kernel %.1f (%s)\n", grid, threads,
             mode ? "cooperative" : "plain", idle / 50 * 1e6, busy / 50 * 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
