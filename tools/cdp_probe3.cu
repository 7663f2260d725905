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
int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  if (argc < 3) return 2;
  int lim = atoi(argv[1]), n = atoi(argv[2]);
  size_t f0, t0; cudaFree(0); cudaMemGetInfo(&f0, &t0);
  int *x, *err; cudaMalloc(&x, 4); cudaMalloc(&err, 4);
  cudaError_t e = cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, lim);
  size_t got = 0; cudaDeviceGetLimit(&got, cudaLimitDevRuntimePendingLaunchCount);
  size_t f, t; cudaMemGetInfo(&f, &t);
  printf("lim=%d set=%d readback=%zu pool=%.1fMB ", lim, (int)e, got, (f0 - f) / 1e6);
  cudaMemset(x, 0, 4); cudaMemset(err, 0, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  parent<<<(n + 127) / 128, 128>>>(x, n, err);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int hx, he; cudaMemcpy(&hx, x, 4, cudaMemcpyDeviceToHost); cudaMemcpy(&he, err, 4, cudaMemcpyDeviceToHost);
  printf("n=%d ms=%.3f rate=%.3g/s done=%d err=%d\n", n, ms, n / (ms * 1e-3), hx, he);
  return 0;
}
