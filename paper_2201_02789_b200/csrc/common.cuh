// common.cuh — warp/block primitives shared by the scheduler and the apps.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define DP_FULL 0xffffffffu

namespace dp {

constexpr int kUnreached = 1 << 30;  // bench/graphs.py:29 UNREACHED

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

#ifndef DP_STREAM_NO_ALLOCATE
#define DP_STREAM_NO_ALLOCATE 1
#endif

// Streaming read of data used once per pass (CSR col / weight): read-only
// path without allocating in L1, so L1 keeps the reused dist lines.
__device__ __forceinline__ int ld_stream(const int* p) {
#if DP_STREAM_NO_ALLOCATE
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];"
               : "=r"(v)
               : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__host__ __device__ __forceinline__ int ceil_div(int a, int b) {
  return (a + b - 1) / b;
}

__host__ __device__ __forceinline__ long long ceil_div_ll(long long a,
                                                         long long b) {
  return (a + b - 1) / b;
}

// inclusive warp scan (all 32 lanes must participate)
__device__ __forceinline__ int warp_incl_scan(int x) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(DP_FULL, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(
    unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(DP_FULL, x, o);
  return x;
}

// Broadcast a 4-byte-multiple POD from lane `src` to the whole warp.
template <class T>
__device__ __forceinline__ T shfl_pod(const T& v, int src) {
  static_assert(sizeof(T) % 4 == 0, "POD must be a multiple of 4 bytes");
  T r;
  const int* pv = reinterpret_cast<const int*>(&v);
  int* pr = reinterpret_cast<int*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); ++i)
    pr[i] = __shfl_sync(DP_FULL, pv[i], src);
  return r;
}

// Block-wide exclusive scan of (participation flag, value) pairs.
// Every thread of the block must call it (contains __syncthreads).
struct BlockScan {
  int rank;   // exclusive count of participants before this thread
  int excl;   // exclusive sum of values before this thread
  int np;     // participants in the block
  int total;  // sum of values in the block
};

__device__ __forceinline__ BlockScan block_scan(int part, int val,
                                                int* smem /* >= 66 ints */) {
  const int lane = lane_id();
  const int wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  int x = val, c = part;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(DP_FULL, x, o);
    int z = __shfl_up_sync(DP_FULL, c, o);
    if (lane >= o) {
      x += y;
      c += z;
    }
  }
  if (lane == 31) {
    smem[wid] = x;
    smem[32 + wid] = c;
  }
  __syncthreads();
  if (wid == 0) {
    int wx = lane < nw ? smem[lane] : 0;
    int wc = lane < nw ? smem[32 + lane] : 0;
    int ix = warp_incl_scan(wx);
    int ic = warp_incl_scan(wc);
    if (lane < nw) {
      smem[lane] = ix - wx;
      smem[32 + lane] = ic - wc;
    }
    if (lane == 31) {
      smem[64] = ix;
      smem[65] = ic;
    }
  }
  __syncthreads();
  BlockScan s;
  s.excl = smem[wid] + x - val;
  s.rank = smem[32 + wid] + c - part;
  s.total = smem[64];
  s.np = smem[65];
  __syncthreads();  // smem may be reused by the caller
  return s;
}

// Device-side run counters: the SimReport launch/block counters
// (sim/machine.py:165-247) measured on hardware.
struct DevState {
  unsigned long long launches;  // device-initiated non-empty launches
  unsigned long long blocks;    // blocks of device-launched grids
  int err;                      // first cudaError_t seen by a device launch
  int flag[2];                  // double-buffered `changed` (levels / rounds)
  int done_round;               // device loop: round count at convergence
  unsigned long long lat_sum;   // device launch -> first child block start, ns
  unsigned long long lat_cnt;
  int skipped[2];  // per round (double-buffered like flag): a parent whose
                   // edges had not arrived yet was deferred (host-buffer
                   // calls that overlap the H2D copy with the rounds)
  // DP_PROFILE builds: warp-cycles per phase (parent, launch, agg, disagg,
  // child), the measured counterpart of SimReport.phase_time
  // (sim/report.py:12-28, folded from per-thread costs at
  // sim/machine.py:657-666); zero in the default build
  unsigned long long phase[5];
  // device launch queue: launches issued whose first child block has not
  // started yet, and its maximum over the run (SimReport.max_pending_depth,
  // the pending-queue length at sim/machine.py:237-244)
  int pending;
  int max_pending;
  // publication checker (DP_CHECK_PUBLISH builds; zero otherwise): child
  // reads of aggregation-table rows whose writer never published them, the
  // hardware stand-in for the reference's "unpublished-read" trap
  // (sim/machine.py:559-574), and reads of rows still holding the poison
  // pattern written before the parent grid (stale bytes actually observed)
  unsigned long long unpublished;
  unsigned long long poisoned;
  // partitioned apps with the fused exchange: atomics issued into other
  // parts' dist (NVLink / NVSwitch peer traffic when parts are GPUs)
  unsigned long long remote;
  // BFS: a vertex discovered for the next level would launch (degree >= T):
  // double-buffered like flag; 0 lets the host run that level's parent grid
  // as the launch-free variant
  int big[2];
  // partitioned BFS: this part's next frontier holds a launching row (set
  // by part_big_kernel, OR-ed over the parts into big[] by the flag OR)
  int big_local;
};

// ---------------------------------------------------------------------------
// Publication checker builds (the reference's fence checker, sim/machine.py:
// 543-649, and its fence-deletion mutation, tests/test_passes.py:541-554).
//   DP_CHECK_PUBLISH=1  every aggregation-table row carries a stamp that only
//                       its publication sets: the multiblock protocol's fence
//                       (aggregate.py:318-319) for cross-block hand-offs, the
//                       launch itself for warp/block rows, the parent grid's
//                       end for grid rows (the cases the reference's checker
//                       publishes on, machine.py:576-598); rows are poisoned
//                       (0xff bytes) before every parent grid
//   DP_NO_FENCE=1       deletes the protocol's fences (the mutation); with
//                       the checker on, the child's reads are then unpublished
// ---------------------------------------------------------------------------
#ifndef DP_CHECK_PUBLISH
#define DP_CHECK_PUBLISH 0
#endif
#ifndef DP_NO_FENCE
#define DP_NO_FENCE 0
#endif
#if DP_CHECK_PUBLISH
__device__ int* g_pub_stamp;      // one stamp per table row
__device__ const char* g_pub_tab; // base of the Args table
#endif

#ifndef DP_PROFILE
#define DP_PROFILE 0
#endif
enum Phase { kPhParent = 0, kPhLaunch = 1, kPhAgg = 2, kPhDisagg = 3,
             kPhChild = 4 };

__device__ __forceinline__ long long ph_now() {
#if DP_PROFILE
  return clock64();
#else
  return 0;
#endif
}

// add the time since t0 to a phase, once per (converged part of a) warp
__device__ __forceinline__ void ph_add(DevState* ds, int ph, long long t0) {
#if DP_PROFILE
  const long long d = clock64() - t0;
  const unsigned am = __activemask();
  if (lane_id() == __ffs(am) - 1 && d > 0)
    atomicAdd(&ds->phase[ph], (unsigned long long)d);
#else
  (void)ds;
  (void)ph;
  (void)t0;
#endif
}

// Spread layout of a per-vertex atomic counter (BFS `counts`): within each
// aligned block of 2^b vertices (mask = 2^b - 1), vertex v's slot is a
// bijective multiply-xorshift hash of its low b bits; the high bits stay, so
// the set of blocks touched (the L2 working set) is that of vertex order.
// mask 0 = vertex order.  RMAT hubs cluster in a few 128 B lines (vertices
// 0..31 alone take ~1 % of all edges at RMAT-22) and L2 serialises the
// atomic requests of one line: spreading them over distinct lines took the
// flat counts pass 0.81 -> 0.46 ms (profiles/ceiling_r02b.txt).  The work
// array (n rounded up to a whole block) is gathered back into vertex order
// once per run.
__host__ __device__ __forceinline__ unsigned spread_slot(unsigned v,
                                                        unsigned mask) {
  if (!mask) return v;
  unsigned x = (v * 0x9E3779B1u) & mask;
  x ^= x >> 7;
  x = (x * 0x85EBCA77u) & mask;
  return (v & ~mask) | x;
}

// Owner part and local index of vertex v >= 0 under the cyclic partition
// owner(v) = v % nparts.  Power-of-two part counts (the 1/2/4/8-GPU runs)
// take a mask and a shift instead of an integer division per edge.
__device__ __forceinline__ int part_of(int v, int nparts) {
  return (nparts & (nparts - 1)) == 0 ? v & (nparts - 1) : v % nparts;
}
__device__ __forceinline__ int local_of(int v, int nparts) {
  return (nparts & (nparts - 1)) == 0 ? v >> (__ffs(nparts) - 1)
                                      : v / nparts;
}

// Chunks of the edge arrays copied so far (monotone counter written by the
// copy stream); a parent may read edge slots [0, arrived << shift).
__device__ __forceinline__ int arrived_chunks(const int* arrived) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(arrived));
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// first block of a device-launched child: launch latency sample
__device__ __forceinline__ void note_child_start(DevState* ds,
                                                 unsigned long long ts) {
  if (ts && blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd(&ds->lat_sum, globaltimer_ns() - ts);
    atomicAdd(&ds->lat_cnt, 1ull);
    // the queue length just before this start: its maximum over the starts
    // is the queue's high-water mark (the first start after the peak sees it)
    atomicMax(&ds->max_pending, atomicSub(&ds->pending, 1));
  }
}

// a device launch is about to be issued (counted before the call, so its
// child can never leave the queue before it entered); the child's first
// block takes it out again in note_child_start
// (a reduction without a return value: no register stays live across the
// launch for it, which the parent kernels' occupancy depends on)
__device__ __forceinline__ void note_launch_issue(DevState* ds) {
  atomicAdd(&ds->pending, 1);
}

__device__ __forceinline__ void note_launch_error(DevState* ds) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) atomicCAS(&ds->err, 0, (int)e);
}

// warp-aggregated launch accounting; all 32 lanes must call
__device__ __forceinline__ void count_launches_warp(DevState* ds, bool launched,
                                                    int blocks) {
  unsigned m = __ballot_sync(DP_FULL, launched);
  if (m) {
    int sum = __reduce_add_sync(DP_FULL, launched ? blocks : 0);
    if (lane_id() == 0) {
      atomicAdd(&ds->launches, (unsigned long long)__popc(m));
      atomicAdd(&ds->blocks, (unsigned long long)sum);
    }
  }
}

}  // namespace dp
