// Probe: CDP2 pending-launch pool memory cost and device-launch throughput on
// B200.  Never launches more children than the pool holds (that hangs).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void child(int* x) { if (threadIdx.x == 0) atomicAdd(x, 1); }
__global__ void parent(int* x, int n, int* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    child<<<1, 32, 0, cudaStreamFireAndForget>>>(x);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) atomicCAS(err, 0, (int)e);
  }
}
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  size_t f0, t0;
  cudaFree(0);
  cudaMemGetInfo(&f0, &t0);
  printf("free0 %.1f MB\n", f0 / 1e6);
  int *x, *err;
  cudaMalloc(&x, 4);
  cudaMalloc(&err, 4);
  size_t def = 0;
  cudaDeviceGetLimit(&def, cudaLimitDevRuntimePendingLaunchCount);
  printf("default pending limit %zu\n", def);
  for (int lim : {2048, 4096, 16384, 65536, 262144, 1 << 20, 1 << 22}) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, lim);
    size_t f, t;
    cudaMemGetInfo(&f, &t);
    printf("limit %d set=%d pool %.1f MB (%.1f B/slot)\n", lim, (int)e, (f0 - f) / 1e6, (double)(f0 - f) / lim);
    for (int n : {1000, 10000, 100000, 1000000}) {
      if (n > lim / 2) continue;
      cudaMemset(x, 0, 4); cudaMemset(err, 0, 4);
      parent<<<(n + 127) / 128, 128>>>(x, n, err);
      cudaDeviceSynchronize();
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaMemset(x, 0, 4);
      cudaEventRecord(a);
      parent<<<(n + 127) / 128, 128>>>(x, n, err);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      int hx, he;
      cudaMemcpy(&hx, x, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(&he, err, 4, cudaMemcpyDeviceToHost);
      printf("  n=%d ms=%.3f launches/s=%.3g done=%d err=%d\n", n, ms, n / (ms * 1e-3), hx, he);
    }
  }
  cudaStream_t s; cudaStreamCreate(&s);
  int* h; cudaMallocHost(&h, 4);
  for (int w = 0; w < 10; ++w) { child<<<1, 32, 0, s>>>(x); cudaMemcpyAsync(h, x, 4, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }
  auto t1 = std::chrono::high_resolution_clock::now();
  for (int i = 0; i < 1000; i++) { child<<<1, 32, 0, s>>>(x); cudaMemcpyAsync(h, x, 4, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }
  auto t2 = std::chrono::high_resolution_clock::now();
  printf("host launch+D2H+sync roundtrip us=%.2f\n", std::chrono::duration<double, std::micro>(t2 - t1).count() / 1000);
  return 0;
}
