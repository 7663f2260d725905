// graph_probe.cu — can a CUDA graph WHILE node drive CDP2 parent grids?
//
// Body of the loop: an IF node picking one of two parent kernels from a
// device-set condition (the launching / launch-free parent variants), then a
// one-thread kernel that advances the level and sets both conditions.  The
// launching parent issues a CDP2 child from device code.  Checked: child
// work count, level count; timed against the host loop (launch + readback
// per level).
//   nvcc -O3 -rdc=true -gencode arch=compute_100a,code=sm_100a \
//        tools/graph_probe.cu -lcudadevrt -o tools/graph_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                            \
  do {                                                                   \
    cudaError_t e_ = (x);                                                \
    if (e_ != cudaSuccess) {                                             \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x,                   \
             cudaGetErrorString(e_));                                    \
      return 1;                                                          \
    }                                                                    \
  } while (0)

struct St {
  int level;
  int children;
  int flat;
  int big;
};

__global__ void child(St* st) { atomicAdd(&st->children, 1); }
#ifdef NO_CDP
#define CHILD_LAUNCH atomicAdd(&st->children, 128)
#else
#define CHILD_LAUNCH child<<<4, 32>>>(st)
#endif

__global__ void parent_cdp(St* st, int n) {
  const int lvl = *(volatile int*)&st->level;
  if (blockIdx.x * blockDim.x + threadIdx.x == 0)
    CHILD_LAUNCH;
  (void)lvl;
  (void)n;
}

__global__ void parent_flat(St* st, int n) {
  if (blockIdx.x * blockDim.x + threadIdx.x == 0) atomicAdd(&st->flat, 1);
  (void)n;
}

__global__ void advance(St* st, cudaGraphConditionalHandle hw,
                        cudaGraphConditionalHandle hi, int levels) {
  const int l = ++st->level;
  cudaGraphSetConditional(hw, l < levels);
  if (hi) cudaGraphSetConditional(hi, (l & 1) == 0);  // alternate the variants
}

__global__ void advance_host(St* st) { ++st->level; }

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;  // 0 if/else+cdp, 1 no cdp, 2 cdp no if, 3 plain graph cdp
  const int n = 1 << 22, blk = 256, grid = n / blk, levels = 6;
  St* st;
  CK(cudaMalloc(&st, sizeof(St)));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));

  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw = 0, hi = 0;
  cudaGraph_t tmp;
  if (mode == 3) {
    CK(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeRelaxed));
    for (int l = 0; l < levels; ++l) {
      if ((l & 1) == 0) parent_cdp<<<grid, blk, 0, s>>>(st, n);
      else parent_flat<<<grid, blk, 0, s>>>(st, n);
      advance_host<<<1, 1, 0, s>>>(st);
    }
    CK(cudaStreamEndCapture(s, &tmp));
  } else {
    CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    if (mode == 0)
      CK(cudaGraphConditionalHandleCreate(&hi, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    if (mode == 0) {
      cudaGraphNodeParams ip = {};
      ip.type = cudaGraphNodeTypeConditional;
      ip.conditional.handle = hi;
      ip.conditional.type = cudaGraphCondTypeIf;
      ip.conditional.size = 2;
      cudaGraphNode_t inode;
      CK(cudaGraphAddNode(&inode, body, nullptr, 0, &ip));
      cudaGraph_t thenG = ip.conditional.phGraph_out[0];
      cudaGraph_t elseG = ip.conditional.phGraph_out[1];
      CK(cudaStreamBeginCaptureToGraph(s, thenG, nullptr, nullptr, 0,
                                       cudaStreamCaptureModeRelaxed));
      parent_cdp<<<grid, blk, 0, s>>>(st, n);
      CK(cudaStreamEndCapture(s, &tmp));
      CK(cudaStreamBeginCaptureToGraph(s, elseG, nullptr, nullptr, 0,
                                       cudaStreamCaptureModeRelaxed));
      parent_flat<<<grid, blk, 0, s>>>(st, n);
      CK(cudaStreamEndCapture(s, &tmp));
      CK(cudaStreamBeginCaptureToGraph(s, body, &inode, nullptr, 1,
                                       cudaStreamCaptureModeRelaxed));
    } else {
      CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                       cudaStreamCaptureModeRelaxed));
      if (mode == 2) parent_cdp<<<grid, blk, 0, s>>>(st, n);
      else parent_flat<<<grid, blk, 0, s>>>(st, n);
    }
    advance<<<1, 1, 0, s>>>(st, hw, hi, levels);
    CK(cudaStreamEndCapture(s, &tmp));
  }

  cudaGraphExec_t ge;
  {
    cudaGraphNode_t errn = nullptr;
    char log[512] = {0};
    cudaError_t e = cudaGraphInstantiateWithParams ? cudaSuccess : cudaSuccess;
    e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) {
      printf("mode %d instantiate: %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    (void)errn; (void)log;
  }
  printf("mode %d\n", mode);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaMemsetAsync(st, 0, sizeof(St), s));
    CK(cudaEventRecord(e0, s));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaStreamSynchronize(s));
    St h;
    CK(cudaMemcpy(&h, st, sizeof(St), cudaMemcpyDeviceToHost));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("graph: levels=%d children=%d (want %d) flat=%d (want %d) %.1f us\n",
           h.level, h.children, 128 * ((levels + 1) / 2), h.flat, levels / 2,
           ms * 1e3);
  }
  // host loop: launch, one-thread readback kernel, copy + sync per level
  St* hst;
  CK(cudaHostAlloc(&hst, sizeof(St), cudaHostAllocDefault));
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaMemsetAsync(st, 0, sizeof(St), s));
    CK(cudaEventRecord(e0, s));
    for (int l = 0; l < levels; ++l) {
      if ((l & 1) == 0)
        parent_cdp<<<grid, blk, 0, s>>>(st, n);
      else
        parent_flat<<<grid, blk, 0, s>>>(st, n);
      advance_host<<<1, 1, 0, s>>>(st);
      CK(cudaMemcpyAsync(hst, st, sizeof(St), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    CK(cudaEventRecord(e1, s));
    CK(cudaStreamSynchronize(s));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("host loop: levels=%d children=%d flat=%d %.1f us\n", hst->level,
           hst->children, hst->flat, ms * 1e3);
  }
  return 0;
}
