// ceiling.cu — microbenchmarks for the ceilings that bind the BFS / SSSP edge
// work on B200 (VERDICT r1 "report against the ceiling that binds").
//
// Flat, perfectly load-balanced edge-parallel kernels over the SAME RMAT
// target stream (`col`) the nested kernels walk: no parents, no launches, no
// scheduler.  Each isolates one component of the per-edge visit:
//   stream_col      the coalesced col stream alone (HBM read ceiling)
//   red_uniform     RED.ADD at hashed uniform addresses (L2 atomic ceiling,
//                   no same-address contention)
//   red_targets     counts[col[e]] += 1 (the RMAT hub contention included)
//   red_merged      the same, lanes hitting the same v merged (match_any)
//   probe_targets   dist[col[e]] probe (L1-cached ld.ca)
//   visit_flat      the whole BFS visit: probe + merged count + CAS
//   relax_flat      the whole SSSP relaxation: col + weight + probe + atomicMin
// Built by tools/ceiling.py (nvcc -shared), timed there with CUDA events.
#include <cuda_runtime.h>
#include <cstdint>

#define FULL 0xffffffffu

namespace {

__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

constexpr int U = 4;

__global__ void stream_col(const int* __restrict__ col, long long m, int* sink) {
  int acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < m;
       e0 += stride * U) {
    int v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long e = e0 + j * stride;
      v[j] = e < m ? ld_stream(col + e) : 0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) acc ^= v[j];
  }
  if (acc == 0x7fffffff) *sink = acc;
}

__global__ void stream_col4(const int4* __restrict__ col, long long m4, int* sink) {
  int acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m4;
       e += stride) {
    int4 v = __ldcs(col + e);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) *sink = acc;
}

__global__ void red_uniform(long long m, int* counts, uint32_t nmask) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += stride)
    atomicAdd(counts + (hash32((uint32_t)e) & nmask), 1);
}

__global__ void red_targets(const int* __restrict__ col, long long m,
                            int* counts) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < m;
       e0 += stride * U) {
    int v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long e = e0 + j * stride;
      v[j] = e < m ? ld_stream(col + e) : -1;
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (v[j] >= 0) atomicAdd(counts + v[j], 1);
  }
}

__global__ void red_merged(const int* __restrict__ col, long long m,
                           int* counts) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  // warp-uniform trip count so match_any sees full warps
  const long long nit = (m + stride * U - 1) / (stride * U);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long it = 0; it < nit; ++it) {
    int v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long e = t + (it * U + j) * stride;
      v[j] = e < m ? ld_stream(col + e) : -1;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const unsigned g = __match_any_sync(FULL, v[j]);
      if (v[j] >= 0 && (threadIdx.x & 31) == __ffs(g) - 1)
        atomicAdd(counts + v[j], __popc(g));
    }
  }
}

__global__ void probe_targets(const int* __restrict__ col, long long m,
                              const int* dist, int* sink) {
  int acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < m;
       e0 += stride * U) {
    int v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long e = e0 + j * stride;
      v[j] = e < m ? ld_stream(col + e) : 0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) acc += __ldca(dist + v[j]);
  }
  if (acc == 0x7fffffff) *sink = acc;
}

constexpr int kUnreached = 1 << 30;

__global__ void visit_flat(const int* __restrict__ col, long long m, int* dist,
                           int* counts, int level, int* changed) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long nit = (m + stride * 2 - 1) / (stride * 2);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int ch = 0;
  for (long long it = 0; it < nit; ++it) {
    int v[2], d[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const long long e = t + (it * 2 + j) * stride;
      v[j] = e < m ? ld_stream(col + e) : -1;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) d[j] = v[j] >= 0 ? __ldca(dist + v[j]) : 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const unsigned g = __match_any_sync(FULL, v[j]);
      if (v[j] < 0) continue;
      if ((threadIdx.x & 31) == __ffs(g) - 1) atomicAdd(counts + v[j], __popc(g));
      if (d[j] == kUnreached &&
          atomicCAS(dist + v[j], kUnreached, level + 1) == kUnreached)
        ch = 1;
    }
  }
  if (__any_sync(FULL, ch) && (threadIdx.x & 31) == 0 && __ldcg(changed) == 0)
    *changed = 1;
}

__global__ void relax_flat(const int* __restrict__ col,
                           const int* __restrict__ w, long long m, int* dist,
                           int du, int* changed) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int ch = 0;
  for (long long e0 = t; e0 < m; e0 += stride * 2) {
    int v[2], ww[2], d[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const long long e = e0 + j * stride;
      v[j] = e < m ? ld_stream(col + e) : -1;
      ww[j] = e < m ? ld_stream(w + e) : 0;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) d[j] = v[j] >= 0 ? __ldca(dist + v[j]) : 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (v[j] < 0) continue;
      const int alt = du + ww[j];
      if (alt < d[j] && atomicMin(dist + v[j], alt) > alt) ch = 1;
    }
  }
  if (ch && __ldcg(changed) == 0) *changed = 1;
}

__global__ void cas_uniform(long long m, int* a, uint32_t nmask, int* sink) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  int acc = 0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += stride)
    acc += atomicCAS(a + (hash32((uint32_t)e) & nmask), -5, -6);
  if (acc == 0x7fffffff) *sink = acc;
}

// counts at a bijective hash of v (22-bit multiply-xorshift inside nmask):
// consecutive vertices no longer share a 128 B line / L2 slice
__device__ __forceinline__ uint32_t spread(uint32_t v, uint32_t nmask) {
  v = (v * 0x9E3779B1u) & nmask;
  v ^= v >> 11;
  v = (v * 0x85EBCA77u) & nmask;
  return v;
}

__global__ void red_hashed(const int* __restrict__ col, long long m,
                           int* counts, uint32_t nmask) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < m;
       e0 += stride * U) {
    int v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long e = e0 + j * stride;
      v[j] = e < m ? ld_stream(col + e) : -1;
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (v[j] >= 0) atomicAdd(counts + spread((uint32_t)v[j], nmask), 1);
  }
}

// every lane the same data-dependent address (no compile-time aggregation)
__global__ void red_single(const int* __restrict__ col, long long m,
                           int* counts) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += stride)
    atomicAdd(counts + ((unsigned)ld_stream(col + e) >> 31), 1);
}

// one 128 B line, lane-distinct words
__global__ void red_one_line(const int* __restrict__ col, long long m,
                             int* counts) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += stride)
    atomicAdd(counts + ((unsigned)ld_stream(col + e) >> 31) + (threadIdx.x & 31),
              1);
}

}  // namespace

extern "C" {

// the BFS visit exactly as BfsApp does it since round 2: counts in the
// spread layout (common.cuh spread_slot, 4096-vertex blocks), lanes hitting
// the same vertex merged, L1 probe, CAS on discovery -- flat and perfectly
// balanced: the ceiling of the nested BFS's per-edge work
__device__ __forceinline__ uint32_t spread_slot(uint32_t v, uint32_t mask) {
  uint32_t x = (v * 0x9E3779B1u) & mask;
  x ^= x >> 7;
  x = (x * 0x85EBCA77u) & mask;
  return (v & ~mask) | x;
}

__global__ void visit_spread(const int* __restrict__ col, long long m,
                             int* dist, int* counts, int level, int* changed) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long nit = (m + stride * 2 - 1) / (stride * 2);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int ch = 0;
  for (long long it = 0; it < nit; ++it) {
    int v[2], d[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const long long e = t + (it * 2 + j) * stride;
      v[j] = e < m ? ld_stream(col + e) : -1;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) d[j] = v[j] >= 0 ? __ldca(dist + v[j]) : 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const unsigned g = __match_any_sync(FULL, v[j]);
      if (v[j] < 0) continue;
      if ((threadIdx.x & 31) == __ffs(g) - 1)
        atomicAdd(counts + spread_slot((uint32_t)v[j], 4095u), __popc(g));
      if (d[j] == kUnreached &&
          atomicCAS(dist + v[j], kUnreached, level + 1) == kUnreached)
        ch = 1;
    }
  }
  if (__any_sync(FULL, ch) && (threadIdx.x & 31) == 0 && __ldcg(changed) == 0)
    *changed = 1;
}

int ceil_run(int which, const int* col, const int* w, long long m, int* dist,
             int* counts, uint32_t nmask, int grid, int block, int* scratch,
             cudaStream_t s) {
  switch (which) {
    case 0: stream_col<<<grid, block, 0, s>>>(col, m, scratch); break;
    case 1: stream_col4<<<grid, block, 0, s>>>(
                reinterpret_cast<const int4*>(col), m / 4, scratch); break;
    case 2: red_uniform<<<grid, block, 0, s>>>(m, counts, nmask); break;
    case 3: red_targets<<<grid, block, 0, s>>>(col, m, counts); break;
    case 4: red_merged<<<grid, block, 0, s>>>(col, m, counts); break;
    case 5: probe_targets<<<grid, block, 0, s>>>(col, m, dist, scratch); break;
    case 6: visit_flat<<<grid, block, 0, s>>>(col, m, dist, counts, 0, scratch);
            break;
    case 7: relax_flat<<<grid, block, 0, s>>>(col, w, m, dist, 1, scratch);
            break;
    case 8: cas_uniform<<<grid, block, 0, s>>>(m, counts, nmask, scratch);
            break;
    case 9: red_hashed<<<grid, block, 0, s>>>(col, m, counts, nmask); break;
    case 10: red_single<<<grid, block, 0, s>>>(col, m, counts); break;
    case 11: red_one_line<<<grid, block, 0, s>>>(col, m, counts); break;
    case 12: visit_spread<<<grid, block, 0, s>>>(col, m, dist, counts, 0,
                                                 scratch);
             break;
    default: return -1;
  }
  return (int)cudaGetLastError();
}

}
