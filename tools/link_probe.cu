// Host-link (PCIe) probe: copy-engine vs SM-driven transfers between pinned
// host memory and HBM.  Used to establish the measured host-link peak that
// the migration engine is judged against.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void sm_pull(const int4* __restrict__ host, int4* __restrict__ dev, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * s < n16; i += 4 * s) {
    int4 a = host[i], b = host[i + s], c = host[i + 2 * s], d = host[i + 3 * s];
    dev[i] = a; dev[i + s] = b; dev[i + 2 * s] = c; dev[i + 3 * s] = d;
  }
  for (; i < n16; i += s) dev[i] = host[i];
}
__global__ void sm_push(const int4* __restrict__ dev, int4* __restrict__ host, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i < n16; i += s) host[i] = dev[i];
}

int main() {
  const size_t B = 1ull << 30;
  void *h1, *h2, *d1, *d2;
  CK(cudaHostAlloc(&h1, B, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h2, B, cudaHostAllocMapped));
  memset(h1, 1, B); memset(h2, 2, B);
  CK(cudaMalloc(&d1, B)); CK(cudaMalloc(&d2, B));
  cudaStream_t s1, s2; CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, c, d; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c); cudaEventCreate(&d);
  float ms;
  auto gbs = [&](double bytes, float ms) { return bytes / (ms * 1e6); };
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a, s1); CK(cudaMemcpyAsync(d1, h1, B, cudaMemcpyHostToDevice, s1)); cudaEventRecord(b, s1); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("CE H2D 1GiB: %.1f GB/s\n", gbs(B, ms));
    cudaEventRecord(a, s1); CK(cudaMemcpyAsync(h2, d2, B, cudaMemcpyDeviceToHost, s1)); cudaEventRecord(b, s1); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("CE D2H 1GiB: %.1f GB/s\n", gbs(B, ms));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a, 0); cudaStreamWaitEvent(s1, a); cudaStreamWaitEvent(s2, a);
    CK(cudaMemcpyAsync(d1, h1, B, cudaMemcpyHostToDevice, s1)); CK(cudaMemcpyAsync(h2, d2, B, cudaMemcpyDeviceToHost, s2));
    cudaEventRecord(b, s1); cudaEventRecord(c, s2); cudaEventSynchronize(b); cudaEventSynchronize(c);
    float m1, m2; cudaEventElapsedTime(&m1, a, b); cudaEventElapsedTime(&m2, a, c);
    printf("CE duplex: H2D %.1f GB/s D2H %.1f GB/s aggregate %.1f GB/s\n", gbs(B, m1), gbs(B, m2), gbs(2.0 * B, m1 > m2 ? m1 : m2));
  }
  // 4 KiB, 64 KiB and 2 MiB pieces, one cudaMemcpyAsync each (the migration
  // engine's copy-engine path issues one call per contiguous segment piece)
  for (size_t piece : {4096ul, 65536ul, 2ul << 20}) {
    size_t n = B / piece;
    for (int dir = 0; dir < 2; ++dir) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a, s1);
        for (size_t i = 0; i < n; ++i) {
          char* dv = (char*)d1 + ((i * 7919) % n) * piece;
          char* hv = (char*)(dir ? h2 : h1) + i * piece;
          if (dir == 0) CK(cudaMemcpyAsync(dv, hv, piece, cudaMemcpyHostToDevice, s1));
          else CK(cudaMemcpyAsync(hv, dv, piece, cudaMemcpyDeviceToHost, s1));
        }
        cudaEventRecord(b, s1); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("CE per-piece %s piece=%zu n=%zu: %.1f GB/s (%.2f ms)\n", dir ? "D2H" : "H2D", piece, n, gbs(B, ms), ms);
      }
    }
  }
  void *hm1, *hm2; CK(cudaHostGetDevicePointer(&hm1, h1, 0)); CK(cudaHostGetDevicePointer(&hm2, h2, 0));
  for (int grid : {32, 74, 148, 296, 592, 1184}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, s1); sm_pull<<<grid, 512, 0, s1>>>((int4*)hm1, (int4*)d1, B / 16); cudaEventRecord(b, s1); cudaEventSynchronize(b);
      CK(cudaGetLastError()); cudaEventElapsedTime(&ms, a, b); float pull = gbs(B, ms);
      cudaEventRecord(a, s1); sm_push<<<grid, 512, 0, s1>>>((int4*)d2, (int4*)hm2, B / 16); cudaEventRecord(b, s1); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); float push = gbs(B, ms);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a, 0); cudaStreamWaitEvent(s1, a); cudaStreamWaitEvent(s2, a);
      sm_pull<<<grid, 512, 0, s1>>>((int4*)hm1, (int4*)d1, B / 16); sm_push<<<grid, 512, 0, s2>>>((int4*)d2, (int4*)hm2, B / 16);
      cudaEventRecord(b, s1); cudaEventRecord(c, s2); cudaEventSynchronize(b); cudaEventSynchronize(c);
      float m1, m2; cudaEventElapsedTime(&m1, a, b); cudaEventElapsedTime(&m2, a, c);
      printf("SM grid=%d x512: pull(H2D) %.1f GB/s push(D2H) %.1f GB/s duplex agg %.1f GB/s\n", grid, pull, push, gbs(2.0 * B, m1 > m2 ? m1 : m2));
    }
  }
  // CE H2D while SM pushes (mixed)
  cudaEventRecord(a, 0); cudaStreamWaitEvent(s1, a); cudaStreamWaitEvent(s2, a);
  CK(cudaMemcpyAsync(d1, h1, B, cudaMemcpyHostToDevice, s1)); sm_push<<<148, 512, 0, s2>>>((int4*)d2, (int4*)hm2, B / 16);
  cudaEventRecord(b, s1); cudaEventRecord(c, s2); cudaEventSynchronize(b); cudaEventSynchronize(c);
  { float m1, m2; cudaEventElapsedTime(&m1, a, b); cudaEventElapsedTime(&m2, a, c);
    printf("mixed CE-H2D + SM-D2H: %.1f / %.1f GB/s\n", gbs(B, m1), gbs(B, m2)); }
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d asyncEngines %d\n", p.name, p.multiProcessorCount, p.asyncEngineCount);
  return 0;
}
