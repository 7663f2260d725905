// sched.cuh — the policy-templated nested-launch scheduler.
//
// One parent thread owns one unit of irregular work (a vertex, an edge list,
// a curve).  App::expand() returns its child count and the scalar arguments
// the child needs; the scheduler then decides, per the paper's three
// optimizations, how that child grid runs:
//
//   T  thresholding  passes/threshold.py:86-172  (guard `_threads >= T` :149)
//      count < T  -> the child grid runs serially inside the parent
//      (make_serial_clone :60-83), no launch.
//   C  coarsening    passes/coarsen.py:65-144
//      the child grid shrinks to ceil(gd / C) blocks; each physical block
//      loops over logical blocks [bx*C, min((bx+1)*C, gDim)) (:125-135).
//   A  aggregation   passes/aggregate.py:171-495
//      launches are recorded into tables and one representative launches a
//      single aggregated grid per group; each aggregated child block finds
//      its logical grid by searching the scanned gdim table (:435-495).
//
// B200 re-design of the aggregation protocol (same launch/block counts and
// outputs as the reference, different mechanics):
//   - the per-group prefix sum is computed with warp shuffles + one shared-
//     memory pass (block_scan) instead of thread 0's serial O(np) scan
//     (aggregate.py:323-343);
//   - multiblock / grid: ONE fused 64-bit atomicAdd per parent BLOCK
//     (participants << 32 | blocks) instead of one per participant
//     (aggregate.py:298-320); the returned old value is both the block's slot
//     base and its block-offset base, so table rows land already scanned;
//   - the group's ctr/done words re-arm themselves (the last block zeroes
//     them) instead of a host memset before every launch (common.py:120-133);
//   - disaggregation is a 32-ary warp search (4 probes for 1M rows) instead
//     of a one-thread binary search;
//   - warp granularity, rejected by the reference (aggregate.py:174-175), is
//     provided.
// Child launches are CDP2 fire-and-forget launches.
#pragma once
#include <type_traits>
#include "common.cuh"


namespace dp {

enum AggKind { kAggNone = 0, kAggWarp = 1, kAggBlock = 2, kAggMulti = 3,
               kAggGrid = 4 };

struct Knobs {
  int threshold;      // 0: pass off (every non-empty child launches)
  int cf;             // coarsening factor >= 1
  int cb;             // child block size (multiple of 32)
  int group;          // multiblock group size in parent blocks
  int agg_threshold;  // block granularity: direct launches below this
  int serial_warp;    // 1: below-threshold children share the parent warp
  int agg_cf;         // 1: coarsening applies to the aggregated grid (the
                      // reference's order "A before C", pipeline.py:60-81:
                      // logical blocks of the aggregated clone span parents)
  int cf_wave;        // B200: rows of >= cf_wave logical child blocks are
                      // not coarsened (0: every row uses cf), see row_cf
};



template <class App>
struct AggTables {
  typename App::Args* args;  // one row per parent thread (compacted per group)
  int* scan;                 // exclusive block-offset of each row in its group
  unsigned long long* ctr;   // per group: participants << 32 | total blocks
  int* done;                 // per group: parent blocks that finished recording
};

// ---------------------------------------------------------------------------
// children
// ---------------------------------------------------------------------------

// Coarsening factor of one row (B200, dp_config.cf_wave): a row whose
// logical child grid alone reaches cf_wave blocks (about one wave of the
// GPU) runs uncoarsened -- coarsening exists to amortise per-block setup
// over many small children, and would only serialise one huge child (the
// RMAT-22 source's 160k edges: 1,247 logical blocks folded onto 78 physical
// ones made BFS level 0 / SSSP round 0 take ~75 us).  Under aggregation such
// a row gets a launch of its own (parent_kernel): computing a per-row factor
// inside the aggregated child cost the SSSP child 76 bytes of spills.
__host__ __device__ __forceinline__ int row_cf(int cf, int cf_wave,
                                               long long gl) {
  return cf_wave > 0 && gl >= cf_wave ? 1 : cf;
}

// Logical blocks [lb*cf, min(lb*cf+cf, ceil(cnt/cb))) of one child grid.
// Thread t owns item b*cb + t of each logical block b; U logical blocks are
// processed together so their independent load chains overlap.
#ifndef DP_CHILD_UNROLL
#define DP_CHILD_UNROLL 0  // items in flight per child thread (0: per app)
#endif
// an app's child-side unroll: App::kChildUnroll when it declares one, else
// the serial arm's App::kUnroll
template <class App, class = void>
struct ChildUnroll {
  static constexpr int value = App::kUnroll;
};
template <class App>
struct ChildUnroll<App, std::void_t<decltype(App::kChildUnroll)>> {
  static constexpr int value = App::kChildUnroll;
};
template <class App>
__device__ __forceinline__ void run_logical_blocks(const App& app,
                                                   const typename App::Args& a,
                                                   long long lb, int cf,
                                                   typename App::Acc& acc) {
  constexpr int U =
      DP_CHILD_UNROLL > 0 ? DP_CHILD_UNROLL : ChildUnroll<App>::value;
  const int cnt = App::count(a);
  const long long cb = blockDim.x;
  const long long gl = ceil_div_ll(cnt, cb);
  const long long b0 = lb * cf;
  const long long b1 = b0 + cf < gl ? b0 + cf : gl;
  if constexpr (App::kBlockMode) {
    // block-cooperative child (shared setup amortised over the CF logical
    // blocks, the paper's coarsening rationale): items [b0*cb, b1*cb)
    const long long e1 = b1 * cb < cnt ? b1 * cb : cnt;
    app.block_items(a, b0 * cb, e1, acc);
    return;
  }
  auto args = [&](int) -> const typename App::Args& { return a; };
  for (long long b = b0; b < b1; b += U) {
    int e[U];
    bool ok[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long ee = (b + j) * cb + threadIdx.x;
      ok[j] = b + j < b1 && ee < cnt;
      e[j] = (int)ee;
    }
    app.template items<U>(args, e, ok, acc);
  }
}

// Plain child: BFS `visit` etc. (benchmarks.py:92-103), coarsened.
template <class App>
__global__ void __launch_bounds__(256, App::kMinBlocks) child_kernel(App app, typename App::Args a, int cf,
                                     DevState* ds, unsigned long long ts) {
  note_child_start(ds, ts);
  const long long t0 = ph_now();
  typename App::Acc acc{};
  run_logical_blocks(app, a, blockIdx.x, cf, acc);  // cf: the row's (row_cf)
  app.flush(acc);
  ph_add(ds, kPhChild, t0);
}

// a device launch: queued in the pending count, its time added to the launch
// phase (DP_PROFILE builds) and to `tl`, so the enclosing aggregation phase
// can leave it out
#define DP_TIMED_LAUNCH(ds, tl, ...)       \
  do {                                     \
    note_launch_issue(ds);                 \
    const long long t_ = ph_now();         \
    __VA_ARGS__;                           \
    ph_add(ds, kPhLaunch, t_);             \
    tl += ph_now() - t_;                   \
  } while (0)

// Largest lo in [0, np) with scan[lo] <= p (scan[0] == 0, strictly
// increasing).  Whole warp; 32-ary: each round probes 32 evenly spaced rows.
__device__ __forceinline__ int warp_search(const int* __restrict__ scan, int np,
                                           int p) {
  const int lane = lane_id();
  int lo = 0, hi = np;
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) >> 5;
    const int idx = lo + lane * step;
    const bool ok = idx < hi && __ldcg(scan + idx) <= p;
    const unsigned m = __ballot_sync(DP_FULL, ok);
    const int last = 31 - __clz(m);  // lane 0 is always ok
    lo += last * step;
    hi = min(lo + step, hi);
  }
  return lo;
}

// Disaggregation of aggregated block `p`: the row that owns it (warp search,
// shared with the block) and its Args; returns the block's index within its
// parent's child grid.  All threads call.
// ---------------------------------------------------------------------------
// Publication of aggregation-table rows (common.cuh, DP_CHECK_PUBLISH).
// pub_mark: the row is published by the launch that follows (warp / block
// rows, the launching thread's barrier) or by the parent grid's end (grid
// rows, launched by the host glue).  pub_fence: the multiblock protocol's
// fence (aggregate.py:318-319), which publishes the rows this thread wrote
// before the group's done counter moves; DP_NO_FENCE deletes it and with it
// the publication.  Default builds: pub_mark is empty, pub_fence a fence.
// ---------------------------------------------------------------------------
template <class Args>
__device__ __forceinline__ void pub_mark(const Args* row) {
#if DP_CHECK_PUBLISH
  g_pub_stamp[((const char*)row - g_pub_tab) / (long long)sizeof(Args)] = 1;
#else
  (void)row;
#endif
}
template <class Args>
__device__ __forceinline__ void pub_fence(const Args* row) {
#if !DP_NO_FENCE
  pub_mark(row);  // stamp first: the fence orders it with the row
  __threadfence();
#else
  (void)row;
#endif
}
// acquire side of the hand-off: the group's last block, before it reads the
// counter and launches (also deleted by the mutation)
__device__ __forceinline__ void protocol_fence() {
#if !DP_NO_FENCE
  __threadfence();
#endif
}

// child side: was the row published, and does it still hold the poison?
template <class Args>
__device__ __forceinline__ void check_row(const Args* row, const Args& a,
                                          DevState* ds) {
#if DP_CHECK_PUBLISH
  if (threadIdx.x == 0) {
    const long long i =
        ((const char*)row - g_pub_tab) / (long long)sizeof(Args);
    if (__ldcg(g_pub_stamp + i) != 1) atomicAdd(&ds->unpublished, 1ull);
    const int* w = reinterpret_cast<const int*>(&a);
    bool poison = true;
#pragma unroll
    for (int j = 0; j < (int)(sizeof(Args) / 4); ++j) poison &= w[j] == -1;
    if (poison) atomicAdd(&ds->poisoned, 1ull);
  }
#else
  (void)row;
  (void)a;
  (void)ds;
#endif
}

template <class App>
__device__ __forceinline__ long long find_row(const typename App::Args* tab,
                                              const int* scan, int np, int p,
                                              typename App::Args& a,
                                              DevState* ds) {
  __shared__ int s_lo;
  int lo = 0;
  if (threadIdx.x < 32) {
    lo = warp_search(scan, np, p);
    if (threadIdx.x == 0) s_lo = lo;
  }
  if (blockDim.x > 32) {
    __syncthreads();
    lo = s_lo;
  }
  // rows are 16-byte multiples: load with 128-bit L2 reads
  static_assert(sizeof(a) % 16 == 0, "Args rows must be 16-byte multiples");
  const int4* src = reinterpret_cast<const int4*>(tab + lo);
  int4* dst = reinterpret_cast<int4*>(&a);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(a) / 16); ++i) dst[i] = __ldcg(src + i);
  check_row(tab + lo, a, ds);
  return (long long)p - __ldcg(scan + lo);
}

// Aggregated child (`<child>_agg`, aggregate.py:435-495), canonical order
// (coarsening before aggregation): one physical block = one (parent row,
// local physical block) pair, found once per block and reused across that
// parent's coarsening loop.
template <class App>
__global__ void __launch_bounds__(256, App::kMinBlocks) child_agg_kernel(App app, const typename App::Args* tab,
                                 const int* scan, int np, int cf,
                                 int agg_total, DevState* ds,
                                 unsigned long long ts) {
  (void)agg_total;
  note_child_start(ds, ts);
  const long long t0 = ph_now();
  typename App::Acc acc{};
  typename App::Args a;
  const long long lb = find_row<App>(tab, scan, np, (int)blockIdx.x, a, ds);
  ph_add(ds, kPhDisagg, t0);
  const long long t1 = ph_now();
  run_logical_blocks(app, a, lb, cf, acc);
  app.flush(acc);
  ph_add(ds, kPhChild, t1);
}

// Order "A before C" (the coarsening pass rewrote the aggregated clone
// itself, pipeline.py:60-81): physical block b runs the aggregated logical
// blocks [b*cf, min(b*cf + cf, agg_total)), each found by its own search, so
// one physical block may serve several parents.  A kernel of its own: a
// second inlined copy of the item code in child_agg_kernel cost TcApp's
// block-mode child 18 registers (32 -> 50) and TC 46 % of its time.
template <class App>
__global__ void __launch_bounds__(256, App::kMinBlocks) child_agg_lb_kernel(App app, const typename App::Args* tab,
                                    const int* scan, int np, int cf,
                                    int agg_total, DevState* ds,
                                    unsigned long long ts) {
  note_child_start(ds, ts);
  typename App::Acc acc{};
  const long long l0 = (long long)blockIdx.x * cf;
  const long long l1 = l0 + cf < agg_total ? l0 + cf : agg_total;
  for (long long l = l0; l < l1; ++l) {
    typename App::Args a;
    const long long lb = find_row<App>(tab, scan, np, (int)l, a, ds);
    run_logical_blocks(app, a, lb, 1, acc);
    if (blockDim.x > 32) __syncthreads();  // s_lo is reused
  }
  app.flush(acc);
}

// device launch of an aggregated child grid (fire-and-forget)
template <class App>
__device__ __forceinline__ void launch_agg(const App& app, int pg, int cb,
                                           const typename App::Args* tab,
                                           const int* scan, int np, int cf,
                                           int agg_total, DevState* ds) {
  if (agg_total > 0)
    child_agg_lb_kernel<App><<<pg, cb, 0, cudaStreamFireAndForget>>>(
        app, tab, scan, np, cf, agg_total, ds, globaltimer_ns());
  else
    child_agg_kernel<App><<<pg, cb, 0, cudaStreamFireAndForget>>>(
        app, tab, scan, np, cf, 0, ds, globaltimer_ns());
}

// physical blocks of an aggregated launch over `total` aggregated blocks
__device__ __forceinline__ int agg_grid(const Knobs& k, int total) {
  return k.agg_cf ? ceil_div(total, k.cf) : total;
}

// ---------------------------------------------------------------------------
// parent
// ---------------------------------------------------------------------------

// The below-threshold arm.  Thread mode is the reference's serial clone
// (threshold.py:60-83): the parent thread loops over every child item.
// Warp mode (B200) flattens the below-threshold items of all 32 lanes into
// one list and processes it 32 items per step: item k belongs to the lane
// whose inclusive count first exceeds k (5-step shuffle search), so a warp
// with degrees {1, 1, ..., 40} takes 3 fully-populated steps instead of 40
// one-lane steps.  Same items, same atomics, no launch.  All lanes call.
#ifndef DP_BIG_UNROLL
#define DP_BIG_UNROLL 0  // serial arm, lanes with >= 32 items (0: per app)
#endif
// the serial arm's unroll for a lane walked by the whole warp:
// App::kBigUnroll when declared, else App::kUnroll
template <class App, class = void>
struct BigUnroll {
  static constexpr int value = App::kUnroll;
};
template <class App>
struct BigUnroll<App, std::void_t<decltype(App::kBigUnroll)>> {
  static constexpr int value = App::kBigUnroll;
};
template <class App>
__device__ __forceinline__ void serial_arm(const App& app,
                                           const typename App::Args& a, int cnt,
                                           bool mine, bool warp_mode,
                                           typename App::Acc& acc) {
  constexpr int U = App::kUnroll;
  using Args = typename App::Args;
  if (!warp_mode) {
    if (!mine) return;
    auto args = [&](int) -> const Args& { return a; };
    for (int e0 = 0; e0 < cnt; e0 += U) {
      int e[U];
      bool ok[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        e[j] = e0 + j;
        ok[j] = e0 + j < cnt;
      }
      app.template items<U>(args, e, ok, acc);
    }
    return;
  }
  // lanes with >= 32 items: the whole warp walks that lane's items, U x 32
  // at a time (no owner search)
  unsigned big = __ballot_sync(DP_FULL, mine && cnt >= 32);
  while (big) {
    const int src = __ffs(big) - 1;
    big &= big - 1;
    const Args b = shfl_pod(a, src);
    const int cb = __shfl_sync(DP_FULL, cnt, src);
    auto args = [&](int) -> const Args& { return b; };
    constexpr int UB =
        DP_BIG_UNROLL > 0 ? DP_BIG_UNROLL : BigUnroll<App>::value;
    for (int e0 = 0; e0 < cb; e0 += 32 * UB) {
      int e[UB];
      bool ok[UB];
#pragma unroll
      for (int j = 0; j < UB; ++j) {
        e[j] = e0 + j * 32 + lane_id();
        ok[j] = e[j] < cb;
      }
      app.template items<UB>(args, e, ok, acc);
    }
  }
  // the rest (< 32 items per lane) as one flattened, load-balanced list
  const int c = mine && cnt > 0 && cnt < 32 ? cnt : 0;
  const int incl = warp_incl_scan(c);
  const int total = __shfl_sync(DP_FULL, incl, 31);
  const int excl = incl - c;
  const int lane = lane_id();
  for (int base = 0; base < total; base += 32 * U) {
    Args b[U];
    int e[U];
    bool ok[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int k = base + j * 32 + lane;
      int owner = 0;  // lanes whose inclusive count is <= k
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int probe = __shfl_sync(DP_FULL, incl, owner + step - 1);
        if (probe <= k) owner += step;
      }
      owner = owner < 31 ? owner : 31;
      e[j] = k - __shfl_sync(DP_FULL, excl, owner);
      b[j] = shfl_pod(a, owner);
      ok[j] = k < total;
    }
    app.template items<U>([&](int j) -> const Args& { return b[j]; }, e, ok,
                          acc);
  }
}

template <class App, int AGG, bool CDP>
__global__ void __launch_bounds__(256, App::kMinBlocks)
    parent_kernel(App app, Knobs k, AggTables<App> t, DevState* ds,
                  long long base) {
  using Args = typename App::Args;
  const long long t_parent = ph_now();
  typename App::Acc acc{};
  // wave-local thread index (table rows) and the parent it owns
  const long long lu = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long u = base + lu;
  app.parent_prologue();
  Args a{};
  // called by every thread (apps may use warp collectives); returns 0 when
  // the thread owns no parent
  const int cnt = app.expand((int)u, u < app.nparents(), a);
  ph_add(ds, kPhParent, t_parent);

  if constexpr (!CDP) {
    // No-CDP variant (e.g. BFS_NOCDP, benchmarks.py:122-141): no launch code
    const long long t_child = ph_now();
    serial_arm(app, a, cnt, true, k.serial_warp != 0, acc);
    app.flush(acc);
    ph_add(ds, kPhChild, t_child);
  } else {
    const long long t_agg = ph_now();
    long long tl = 0;  // launch time inside the protocol (DP_PROFILE)
    const bool go = cnt > 0 && (k.threshold == 0 || cnt >= k.threshold);
    // physical (coarsened) child grid of this parent thread; under agg_cf
    // the recorded rows stay uncoarsened and the aggregated grid is
    // coarsened instead (direct launches are per-parent coarsened always)
    int gl = go ? ceil_div(cnt, k.cb) : 0;
    const int cfr = row_cf(k.cf, k.cf_wave, gl);
    if constexpr (AGG != kAggNone) {
      // cf_wave: a row whose child fills a GPU wave is launched on its own,
      // uncoarsened, and stays out of the aggregated grid (whose per-row
      // coarsening stays uniform)
      if (cfr != k.cf) {
        DP_TIMED_LAUNCH(ds, tl,
            child_kernel<App><<<gl, k.cb, 0, cudaStreamFireAndForget>>>(
                app, a, 1, ds, globaltimer_ns());
            note_launch_error(ds));
        atomicAdd(&ds->launches, 1ull);
        atomicAdd(&ds->blocks, (unsigned long long)gl);
        gl = 0;
      }
    }
    const int gd = AGG == kAggNone || !k.agg_cf ? ceil_div(gl, cfr) : gl;
    // The launch / aggregation protocol runs BEFORE the serial arm (the
    // reference places it after the enclosing statement, aggregate.py:
    // 244-249; both orders give the same outputs): children start while the
    // parent is still busy, and the protocol's barriers never wait on a
    // long serial tail.

    if constexpr (AGG == kAggNone) {
      if (gd > 0) {
        DP_TIMED_LAUNCH(ds, tl,
            child_kernel<App><<<gd, k.cb, 0, cudaStreamFireAndForget>>>(
                app, a, cfr, ds, globaltimer_ns());
            note_launch_error(ds));
      }
      count_launches_warp(ds, gd > 0, gd);
    } else if constexpr (AGG == kAggWarp) {
      const unsigned m = __ballot_sync(DP_FULL, gd > 0);
      if (m) {
        const int lane = lane_id();
        const int incl = warp_incl_scan(gd);
        const int total = __shfl_sync(DP_FULL, incl, 31);
        const long long row0 = lu - lane;  // one 32-row segment per warp
        if (gd > 0) {
          const int rank = __popc(m & lanemask_lt());
          t.args[row0 + rank] = a;
          t.scan[row0 + rank] = incl - gd;
          pub_mark(t.args + row0 + rank);
          __threadfence();
        }
        __syncwarp();
        if (lane == __ffs(m) - 1) {
          const int pg = agg_grid(k, total);
          DP_TIMED_LAUNCH(ds, tl,
              launch_agg(app, pg, k.cb, t.args + row0, t.scan + row0,
                         __popc(m), k.cf, k.agg_cf ? total : 0, ds);
              note_launch_error(ds));
          atomicAdd(&ds->launches, 1ull);
          atomicAdd(&ds->blocks, (unsigned long long)pg);
        }
      }
    } else {
      __shared__ int smem[66];
      __shared__ unsigned long long s_old;
      // most blocks hold no launching parent once T is in the hundreds:
      // they skip the scan (one barrier instead of three) and, below, the
      // record barriers
      BlockScan s{0, 0, 0, 0};
      if (__syncthreads_or(gd > 0)) s = block_scan(gd > 0, gd, smem);
      if constexpr (AGG == kAggBlock) {
        if (k.agg_threshold > 0 && s.np < k.agg_threshold) {
          // aggregate.py:376-392: too few participants -> direct launches
          const int gdd = ceil_div(gl, k.cf);
          if (gdd > 0) {
            DP_TIMED_LAUNCH(ds, tl,
                child_kernel<App><<<gdd, k.cb, 0, cudaStreamFireAndForget>>>(
                    app, a, k.cf, ds, globaltimer_ns());
                note_launch_error(ds));
          }
          count_launches_warp(ds, gdd > 0, gdd);
        } else if (s.np > 0) {
          const long long row0 = (long long)blockIdx.x * blockDim.x;
          if (gd > 0) {
            t.args[row0 + s.rank] = a;
            t.scan[row0 + s.rank] = s.excl;
            pub_mark(t.args + row0 + s.rank);
            __threadfence();
          }
          __syncthreads();
          if (threadIdx.x == 0) {
            const int pg = agg_grid(k, s.total);
            DP_TIMED_LAUNCH(ds, tl,
                launch_agg(app, pg, k.cb, t.args + row0, t.scan + row0,
                           s.np, k.cf, k.agg_cf ? s.total : 0, ds);
                note_launch_error(ds));
            atomicAdd(&ds->launches, 1ull);
            atomicAdd(&ds->blocks, (unsigned long long)pg);
          }
        }
      } else {
        // multiblock (aggregate.py:395-422) and grid (:425-429)
        const int grp = AGG == kAggMulti ? (int)blockIdx.x / k.group : 0;
        const long long sb =
            AGG == kAggMulti ? (long long)grp * k.group * blockDim.x : 0;
        if (s.np > 0) {  // block-uniform
          if (threadIdx.x == 0)
            s_old = atomicAdd(&t.ctr[grp], ((unsigned long long)s.np << 32) +
                                               (unsigned long long)s.total);
          __syncthreads();
          if (gd > 0) {
            const unsigned long long old = s_old;
            const long long row = sb + (long long)(old >> 32) + s.rank;
            t.args[row] = a;
            t.scan[row] = (int)(old & 0xffffffffull) + s.excl;
            if constexpr (AGG == kAggMulti)
              pub_fence(t.args + row);  // publish before the done counter
            else
              pub_mark(t.args + row);  // grid: the parent grid's end publishes
          }
          if constexpr (AGG == kAggMulti) __syncthreads();
        }
        if constexpr (AGG == kAggMulti) {
          if (threadIdx.x == 0) {
            const int nblk = min(k.group, (int)gridDim.x - grp * k.group);
            const bool last = atomicAdd(&t.done[grp], 1) == nblk - 1;
            if (last) {
              protocol_fence();
              const unsigned long long c =
                  atomicAdd(&t.ctr[grp], 0ull);  // L2-coherent read
              t.ctr[grp] = 0;                     // re-arm for the next launch
              t.done[grp] = 0;
              const int np = (int)(c >> 32);
              const int total = (int)(c & 0xffffffffull);
              if (np > 0) {
                const int pg = agg_grid(k, total);
                DP_TIMED_LAUNCH(ds, tl,
                    launch_agg(app, pg, k.cb, t.args + sb, t.scan + sb, np,
                               k.cf, k.agg_cf ? total : 0, ds);
                    note_launch_error(ds));
                atomicAdd(&ds->launches, 1ull);
                atomicAdd(&ds->blocks, (unsigned long long)pg);
              }
            }
          }
        }
        // grid: the host glue reads ctr[0] after the parent grid completes
        // and performs the aggregated launch (common.py:144-164)
      }
    }
    ph_add(ds, kPhAgg, t_agg + tl);  // the protocol minus its launches
    const long long t_child = ph_now();
    serial_arm(app, a, cnt, !go, k.serial_warp != 0, acc);
    app.flush(acc);
    ph_add(ds, kPhChild, t_child);
  }
}

// ---------------------------------------------------------------------------
// Persistent parent (B200): a grid of a few blocks per SM walks the parents in
// chunks of blockDim.x twice.  Pass 1 only expands and records the launches
// (one fused atomic per chunk into the single group); the last block to
// finish pass 1 performs the aggregated launch (multiblock with one group)
// or leaves it to the host glue (grid).  Pass 2 re-expands and runs the
// serial arms, so the aggregated child overlaps with the parent's own
// below-threshold work instead of starting after the last of ~10^4 parent
// blocks.  Requires App::kPureExpand (expand has no side effects).
// ---------------------------------------------------------------------------
template <class App, int AGG>
__global__ void __launch_bounds__(256)
    parent_persistent_kernel(App app, Knobs k, AggTables<App> t, DevState* ds,
                             long long base, long long nparents) {
  static_assert(App::kPureExpand, "persistent parents re-run expand()");
  static_assert(AGG == kAggMulti || AGG == kAggGrid, "single-group only");
  using Args = typename App::Args;
  __shared__ int smem[66];
  __shared__ unsigned long long s_old;
  app.parent_prologue();
  const long long nchunks = ceil_div_ll(nparents, blockDim.x);
  // pass 1: record every launch of this block's chunks
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const long long lu = c * blockDim.x + threadIdx.x;
    Args a{};
    const int cnt = app.expand((int)(base + lu),
                               lu < nparents && base + lu < app.nparents(), a);
    const bool go = cnt > 0 && (k.threshold == 0 || cnt >= k.threshold);
    const int gl = go ? ceil_div(cnt, k.cb) : 0;
    const int gd = ceil_div(gl, k.cf);
    const BlockScan s = block_scan(gd > 0, gd, smem);
    if (threadIdx.x == 0)
      s_old = s.np > 0 ? atomicAdd(&t.ctr[0], ((unsigned long long)s.np << 32) +
                                                  (unsigned long long)s.total)
                       : 0ull;
    __syncthreads();
    if (gd > 0) {
      const unsigned long long old = s_old;
      const long long row = (long long)(old >> 32) + s.rank;
      t.args[row] = a;
      t.scan[row] = (int)(old & 0xffffffffull) + s.excl;
      if constexpr (AGG == kAggMulti)
        pub_fence(t.args + row);
      else
        pub_mark(t.args + row);
    }
    __syncthreads();  // s_old is rewritten by the next chunk
  }
  if constexpr (AGG == kAggMulti) {
    if (threadIdx.x == 0) {
      const int d = atomicAdd(&t.done[0], 1);
      if (d == (int)gridDim.x - 1) {
        protocol_fence();
        const unsigned long long c = atomicAdd(&t.ctr[0], 0ull);
        t.ctr[0] = 0;
        t.done[0] = 0;
        const int np = (int)(c >> 32);
        const int total = (int)(c & 0xffffffffull);
        if (np > 0) {
          note_launch_issue(ds);
          child_agg_kernel<App><<<total, k.cb, 0, cudaStreamFireAndForget>>>(
              app, t.args, t.scan, np, k.cf, 0, ds, globaltimer_ns());
          note_launch_error(ds);
          atomicAdd(&ds->launches, 1ull);
          atomicAdd(&ds->blocks, (unsigned long long)total);
        }
      }
    }
  }
  // pass 2: the below-threshold children, serially in the parent warps
  typename App::Acc acc{};
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const long long lu = c * blockDim.x + threadIdx.x;
    Args a{};
    const int cnt = app.expand((int)(base + lu),
                               lu < nparents && base + lu < app.nparents(), a);
    const bool go = cnt > 0 && (k.threshold == 0 || cnt >= k.threshold);
    serial_arm(app, a, cnt, !go, k.serial_warp != 0, acc);
  }
  app.flush(acc);
}

// ---------------------------------------------------------------------------
// Device-side level loop (B200, CDP2 tail launches).  The host loop of the
// reference (bench/benchmarks.py:157-168, 259-270) launches one parent grid
// per level and reads `changed` back.  Here a one-thread controller does it:
// round r's parent grid goes to the fire-and-forget stream, the controller of
// round r+1 to the tail-launch stream, so it starts only after round r and
// every grid it spawned have completed, reads the flag, and either stops or
// continues.  A chain covers at most `last - first + 1` rounds (bounded
// nesting); the host relaunches until done_round is set.
// ---------------------------------------------------------------------------
template <class App, int AGG>
__global__ void round_controller(App app0, Knobs k, AggTables<App> t,
                                 DevState* ds, int grid, int pb, int round,
                                 int first, int last) {
  if (round > 0 && round > first && ds->flag[(round - 1) & 1] == 0) {
    ds->done_round = round;  // round - 1 changed nothing
    return;
  }
  if (round > last) return;  // hand back to the host
  const App app = app0.for_round(round, ds->flag);
  parent_kernel<App, AGG, true><<<grid, pb, 0, cudaStreamFireAndForget>>>(
      app, k, t, ds, 0ll);
  note_launch_error(ds);
  round_controller<App, AGG><<<1, 1, 0, cudaStreamTailLaunch>>>(
      app0, k, t, ds, grid, pb, round + 1, first, last);
  note_launch_error(ds);
  atomicAdd(&ds->launches, 2ull);
  atomicAdd(&ds->blocks, (unsigned long long)grid + 1);
}

}  // namespace dp
