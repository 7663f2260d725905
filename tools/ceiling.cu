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

// rank of v among the vertices with popcount(v) <= kmax (kmax <= 4, 22-bit
// ids): 0 for v = 0, then the 1-bit ids, the 2-bit ids ... (combinatorial
// number system); -1 when popcount(v) > kmax
__device__ __forceinline__ int hub_rank(unsigned v, int kmax) {
  const int k = __popc(v);
  if (k > kmax) return -1;
  // offsets: sum_{i<k} C(22, i) = 0, 1, 23, 254, 1794
  int idx = k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 23 : k == 3 ? 254 : 1794;
  for (int j = 1; j <= k; ++j) {
    const int p = __ffs(v) - 1;
    v &= v - 1;
    int c = p;  // C(p, j)
    if (j >= 2) c = c * (p - 1) / 2;
    if (j >= 3) c = c * (p - 2) / 3;
    if (j >= 4) c = c * (p - 3) / 4;
    idx += c;
  }
  return idx;
}

// visit_spread with the hub counters (popcount(v) <= kmax) replicated R ways
// (replica picked by the global warp id, replicas 8 KB apart so they sit in
// distinct lines / L2 slices)
__global__ void visit_hubrep(const int* __restrict__ col, long long m,
                             int* dist, int* counts, int* rep, int kmax,
                             int rbits, int level, int* changed) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long nit = (m + stride * 2 - 1) / (stride * 2);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int r = (int)((t >> 5) & ((1 << rbits) - 1));
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
      if ((threadIdx.x & 31) == __ffs(g) - 1) {
        const int h = hub_rank((unsigned)v[j], kmax);
        int* a = h >= 0 ? rep + (r << 11) + h
                        : counts + spread_slot((uint32_t)v[j], 4095u);
        atomicAdd(a, __popc(g));
      }
      if (d[j] == kUnreached &&
          atomicCAS(dist + v[j], kUnreached, level + 1) == kUnreached)
        ch = 1;
    }
  }
  if (__any_sync(FULL, ch) && (threadIdx.x & 31) == 0 && __ldcg(changed) == 0)
    *changed = 1;
}

// the visit without the counts (probe + CAS only): what counts cost
__global__ void visit_nocount(const int* __restrict__ col, long long m,
                              int* dist, int level, int* changed) {
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
      if (v[j] < 0) continue;
      if (d[j] == kUnreached &&
          atomicCAS(dist + v[j], kUnreached, level + 1) == kUnreached)
        ch = 1;
    }
  }
  if (__any_sync(FULL, ch) && (threadIdx.x & 31) == 0 && __ldcg(changed) == 0)
    *changed = 1;
}

__global__ void fill_hi(unsigned long long* w, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = i == 0 ? 0ull : (unsigned long long)kUnreached << 32;
}

// counts and dist fused in one 64-bit word per vertex (hi = dist, lo =
// count): the merged count's ATOM.ADD returns the old word, whose hi half
// replaces the dist probe; the first discoverer CASes the hi half
__global__ void visit_fused64(const int* __restrict__ col, long long m,
                              unsigned long long* word, unsigned mask,
                              int level, int* changed) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long nit = (m + stride * 2 - 1) / (stride * 2);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int ch = 0;
  for (long long it = 0; it < nit; ++it) {
    int v[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const long long e = t + (it * 2 + j) * stride;
      v[j] = e < m ? ld_stream(col + e) : -1;
    }
    unsigned long long old[2];
    bool lead[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const unsigned g = __match_any_sync(FULL, v[j]);
      lead[j] = v[j] >= 0 && (threadIdx.x & 31) == __ffs(g) - 1;
      old[j] = lead[j] ? atomicAdd(word + spread_slot((uint32_t)v[j], mask),
                                   (unsigned long long)__popc(g))
                       : 0ull;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (lead[j] && (int)(old[j] >> 32) == kUnreached) {
        int* hi = reinterpret_cast<int*>(
                      word + spread_slot((uint32_t)v[j], mask)) + 1;
        if (atomicCAS(hi, kUnreached, level + 1) == kUnreached) ch = 1;
      }
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
    case 13: {
      static int* rep = nullptr;
      if (!rep && cudaMalloc(&rep, (32 << 11) * sizeof(int))) return -2;
      cudaMemsetAsync(rep, 0, (32 << 11) * sizeof(int), s);
      visit_hubrep<<<grid, block, 0, s>>>(col, m, dist, counts, rep,
                                          (int)(nmask >> 8), (int)(nmask & 0xff),
                                          0, scratch);
      break;
    }
    case 14: visit_nocount<<<grid, block, 0, s>>>(col, m, dist, 0, scratch);
             break;
    case 15:
    case 16: {
      static unsigned long long* word = nullptr;
      static long long have = 0;
      const long long n = (long long)nmask + 1;
      if (have < n) {
        if (word) cudaFree(word);
        if (cudaMalloc(&word, n * 8)) return -2;
        have = n;
      }
      fill_hi<<<(int)((n + 255) / 256), 256, 0, s>>>(word, n);
      visit_fused64<<<grid, block, 0, s>>>(col, m, word,
                                           which == 16 ? 4095u : 0u, 0,
                                           scratch);
      break;
    }
    default: return -1;
  }
  return (int)cudaGetLastError();
}

}
