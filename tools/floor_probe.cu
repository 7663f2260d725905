// floor_probe.cu -- what does a launch-free parent grid over 4 M vertices
// cost when (almost) no vertex is in the frontier?  Standalone timings of
// trivial 4 M-thread grids (CUDA events, mean of 200 launches) to compare
// with the ~21 us a BFS level of the launch-free parent variant takes.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/floor_probe tools/floor_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_k() {}
__global__ void read_k(const int* __restrict__ dist, int n, int level,
                       int* sink) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n && __ldcg(dist + u) == level) atomicAdd(sink, 1);
}
__global__ void read_scan_k(const int* __restrict__ dist, int n, int level,
                            int* sink) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = u < n && __ldcg(dist + u) == level ? 3 : 0;
  int x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  if (__ballot_sync(0xffffffffu, c > 0) && (threadIdx.x & 31) == 31)
    atomicAdd(sink, x);
}

int main() {
  const int n = 1 << 22;
  int *dist, *sink;
  cudaMalloc(&dist, n * sizeof(int));
  cudaMalloc(&sink, sizeof(int));
  cudaMemset(dist, 0x7f, n * sizeof(int));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int pb : {128, 256, 1024}) {
    const int grid = (n + pb - 1) / pb;
    for (int which = 0; which < 3; ++which) {
      for (int it = 0; it < 20; ++it) {
        if (which == 0) empty_k<<<grid, pb>>>();
        if (which == 1) read_k<<<grid, pb>>>(dist, n, 5, sink);
        if (which == 2) read_scan_k<<<grid, pb>>>(dist, n, 5, sink);
      }
      cudaDeviceSynchronize();
      float tot = 0.f;
      for (int it = 0; it < 200; ++it) {
        cudaEventRecord(a);
        if (which == 0) empty_k<<<grid, pb>>>();
        if (which == 1) read_k<<<grid, pb>>>(dist, n, 5, sink);
        if (which == 2) read_scan_k<<<grid, pb>>>(dist, n, 5, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        tot += ms;
      }
      printf("{\"kernel\": \"%s\", \"block\": %d, \"grid\": %d, \"us\": %.2f}\n",
             which == 0 ? "empty" : which == 1 ? "read_dist" : "read_scan",
             pb, grid, tot / 200 * 1e3);
    }
  }
  return 0;
}
