// apps.cuh — per-application parent/child functors for the scheduler.
//
// Each App supplies
//   Args                  16-byte-multiple POD of scalar child arguments (the
//                         rows of the aggregation tables, aggregate.py:103-136)
//   Acc                   per-thread accumulator flushed once per thread
//   nparents()            parent threads per host launch
//   parent_prologue()     once-per-grid bookkeeping (all threads call)
//   expand(u, valid, a)   parent work; returns the child thread count
//                         (all threads call; 0 when !valid)
//   count(a)              child thread count recorded in a row
//   item(a, e, acc)       child thread e's work
//   items<U>(args, e, ok, acc)  U independent items at once: all streaming
//                         loads, then all probes, then all updates, so a
//                         thread keeps U dependent chains in flight
//   kUnroll               U used by the scheduler
//   flush(acc)            warp-collective epilogue (all 32 lanes call)
#pragma once
#include "common.cuh"

namespace dp {

#ifndef DP_GRAPH_UNROLL
#define DP_GRAPH_UNROLL 2  // tools/ab.sh: 2 < 4 < 8 (profiles/ab_unroll_r01.txt)
#endif
#ifndef DP_MERGE_COUNTS
#define DP_MERGE_COUNTS 1
#endif
#ifndef DP_SSSP_UNROLL
#define DP_SSSP_UNROLL 2
#endif
#ifndef DP_TC_MINB
#define DP_TC_MINB 1  // TC's grid parent is at 31 registers already
#endif
#ifndef DP_BFSPART_MINB
#define DP_BFSPART_MINB 8  // <= 32 registers: BFS-26 22.0 -> 19.7 ms
#endif
#ifndef DP_BFS_MINB
#define DP_BFS_MINB 8  // <= 32 registers: 1.26 vs 1.28 ms (ab_bfs_minblocks_r01)
#endif
#ifndef DP_BT_MINB
#define DP_BT_MINB 1
#endif
#ifndef DP_SP_MINB
#define DP_SP_MINB 1
#endif
#ifndef DP_SP_UNROLL
#define DP_SP_UNROLL 1  // SP items in flight per thread (variable / ratio)
#endif
#ifndef DP_SP_VAR_UNROLL
#define DP_SP_VAR_UNROLL 2  // variable pass: eta gathers in flight per lane
                            // (1: 12.92, 2: 12.31, 4: 12.8, 8: 13.0 ms,
                            // profiles/r02/ab_sp_varunroll_r02.txt)
#endif
#ifndef DP_SP_OCC_L1
#define DP_SP_OCC_L1 1  // variable pass: L1-cached occurrence loads
#endif
#ifndef DP_SP_RATIO_MINB
#define DP_SP_RATIO_MINB 5  // 58 -> 48 registers: 5-SAT 12.29 -> 12.03 ms
                            // (profiles/r02/ab_sp_rminb_r02.txt)
#endif
#ifndef DP_MST_MINB
#define DP_MST_MINB 8  // <= 32 registers: MST 4.15 (56) -> 3.98 (48) -> 3.70 ms
#endif
#ifndef DP_SSSP_CHILD_UNROLL
#define DP_SSSP_CHILD_UNROLL 1  // hub children: 1 < 2 < 4 < 8
#endif                          // (profiles/ab_child_unroll_r01.txt)
// Discovery / relaxation as a fire-and-forget RED.MIN instead of a returning
// CAS / atomicMin: min(old, new) reaches the same final value, and the round
// flag is set from the probe (alt < d).  A probe is stale only within the
// launch that cached it (L1 is invalidated at every kernel launch,
// B300_MICROARCH.md "Per-launch flush"), so a flagged round is always one in
// which some vertex really was lowered: the flag, and hence the level /
// round count, is unchanged.
#ifndef DP_BFS_RED
#define DP_BFS_RED 0
#endif
#ifndef DP_SSSP_RED
#define DP_SSSP_RED 0
#endif
#ifndef DP_BFS_NO_COUNTS
#define DP_BFS_NO_COUNTS 0  // ablation only (wrong counts): the cost of counts
#endif
#ifndef DP_SSSPPEER_MINB
#define DP_SSSPPEER_MINB DP_SSSP_MINB  // fused-exchange SSSP (A/B knob)
#endif
#ifndef DP_SSSP_MINB
#define DP_SSSP_MINB 8  // <= 32 registers: full occupancy for the latency-
#endif                  // bound relaxations (tools/ab.sh, profiles/)

// items<U> for apps whose item is not latency-chained: plain loop
__device__ __forceinline__ void red_min(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.min.s32 [%0], %1;" ::"l"(p), "r"(v)
               : "memory");
}

template <int U, class App, class ArgsOf>
__device__ __forceinline__ void items_loop(const App& app, ArgsOf args,
                                           const int* e, const bool* ok,
                                           typename App::Acc& acc) {
#pragma unroll
  for (int j = 0; j < U; ++j)
    if (ok[j]) app.item(args(j), e[j], acc);
}

// ---------------------------------------------------------------------------
// BFS — BFS_CDP main/visit (bench/benchmarks.py:91-120)
// ---------------------------------------------------------------------------
struct BfsApp {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  int* dist;
  int* counts;        // counts[spread_slot(v, cmask)] (common.cuh)
  int* changed;       // this level's flag
  int* changed_next;  // next level's flag, cleared here
  // launch bits (bit v: v's row would launch under the policy's threshold)
  // and the flag "the next level holds such a vertex" (DevState::big); null
  // when the host does not pick the parent variant per level
  const unsigned* __restrict__ lbits;
  int* big_next;
  int* big_after;  // the level after next's flag, cleared here
  int n;
  int level;
  unsigned cmask;     // spread layout of counts (0: vertex order)
  unsigned pad_;

  struct alignas(16) Args {
    int start, deg, level, pad;
  };
  struct Acc {
    int changed;
    int big;
  };

  __device__ int nparents() const { return n; }
  __device__ void parent_prologue() const {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *changed_next = 0;
      if (lbits) *big_after = 0;
    }
  }
  // the app of level r (device-side level loop)
  __device__ BfsApp for_round(int r, int* flags) const {
    BfsApp a = *this;
    a.level = r;
    a.changed = flags + (r & 1);
    a.changed_next = flags + ((r + 1) & 1);
    a.lbits = nullptr;  // the device loop keeps the launching variant
    return a;
  }
  // a discovered vertex whose row would launch next level
  __device__ __forceinline__ void note_big(int v, Acc& acc) const {
    if (lbits && (__ldg(lbits + (v >> 5)) >> (v & 31) & 1u)) acc.big = 1;
  }
  // main (:105-119): u with dist[u] == level owns deg = rowptr[u+1]-rowptr[u]
  __device__ int expand(int u, bool valid, Args& a) const {
    if (!valid || __ldcg(dist + u) != level) return 0;
    const int s = __ldg(rowptr + u);
    const int d = __ldg(rowptr + u + 1) - s;
    a = Args{s, d, level, 0};
    return d > 0 ? d : 0;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  // visit (:92-103): count the edge, discover v with one CAS against
  // UNREACHED.  The plain pre-check only skips CASes that would fail.
  __device__ void item(const Args& a, int e, Acc& acc) const {
    const int v = __ldg(col + a.start + e);
    atomicAdd(counts + spread_slot(v, cmask), 1);
    if (__ldcg(dist + v) == kUnreached &&
        atomicCAS(dist + v, kUnreached, a.level + 1) == kUnreached) {
      acc.changed = 1;
      note_big(v, acc);
    }
  }
  // counts[v] += 1 with lanes that hit the same v merged into one atomic:
  // RMAT hub destinations otherwise serialise at one L2 slice
  __device__ __forceinline__ void count_edge(int v) const {
#if DP_MERGE_COUNTS
    const unsigned am = __activemask();
    const unsigned grp = __match_any_sync(am, v);
    if (lane_id() == __ffs(grp) - 1)
      atomicAdd(counts + spread_slot(v, cmask), __popc(grp));
#else
    atomicAdd(counts + spread_slot(v, cmask), 1);
#endif
  }
  static constexpr int kUnroll = DP_GRAPH_UNROLL;
  // hub rows walked by the whole parent warp: 4 in flight (1.27 vs 1.29 ms,
  // profiles/ab_big_unroll_r01.txt)
  static constexpr int kBigUnroll = 4;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_BFS_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    int v[U], d[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      v[j] = ok[j] ? ld_stream(col + args(j).start + e[j]) : 0;
    // L1-cached probe: dist only ever decreases, so a stale copy is >= the
    // true value and can only cost a redundant (failing) CAS, never a
    // missed discovery; RMAT hubs then hit in L1 instead of costing a 32 B
    // L2 sector each
#pragma unroll
    for (int j = 0; j < U; ++j) d[j] = ok[j] ? __ldca(dist + v[j]) : 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (!ok[j]) continue;
      if (!DP_BFS_NO_COUNTS) count_edge(v[j]);
#if DP_BFS_RED
      if (d[j] == kUnreached) {
        red_min(dist + v[j], args(j).level + 1);
        acc.changed = 1;
      }
#else
      if (d[j] == kUnreached &&
          atomicCAS(dist + v[j], kUnreached, args(j).level + 1) ==
              kUnreached) {
        acc.changed = 1;
        note_big(v[j], acc);
      }
#endif
    }
  }
  __device__ void flush(Acc& acc) const {
    // read before write: after the first success the flag line is only
    // read (shared), not re-written by every succeeding warp
    if (__any_sync(DP_FULL, acc.changed) && lane_id() == 0 &&
        __ldcg(changed) == 0)
      *changed = 1;
    if (lbits && __any_sync(DP_FULL, acc.big) && lane_id() == 0 &&
        __ldcg(big_next) == 0)
      *big_next = 1;
  }
};

// ---------------------------------------------------------------------------
// BFS on one part of a cyclic 1D vertex partition:
// owner(v) = v % nparts, owned vertices at local index v / nparts.  Each
// examined edge counts into a dense per-part `counts` (summed across parts at
// the end); a local target is discovered in place, a remote target is sent to
// its owner once per part for the whole run (`sent` bitmap), bucketed per
// owner with warp-aggregated slot reservation.  The owner applies received
// ids with the same CAS (dp_bfs_part_apply).  dist stays a level labelling,
// bit-identical to the single-part run.
// ---------------------------------------------------------------------------
// kPeer: the fused exchange (remote CAS through peer_dist) compiled alone;
// the bucketed exchange (send_buf) otherwise -- one runtime branch per edge
// between them had cost the register-capped kernels 28-36 B of spills
template <bool kPeer>
struct BfsPartAppT {
  const int* __restrict__ rowptr;  // local CSR over owned vertices
  const int* __restrict__ col;     // global target ids
  int* dist;                       // owned vertices (local index)
  int* counts;                     // dense, global ids
  unsigned* sent;                  // bitmap over global ids
  int* send_buf;                   // [nparts][stride]
  int* send_count;                 // [nparts]
  int* changed;
  // fused exchange (null: buckets): every part's dist, addressable here
  // (symmetric memory); a remote discovery is a CAS into the owner's dist
  int* const* peer_dist;
  unsigned long long* remote_ops;  // DevState::remote
  long long stride;
  int n_local;
  int nparts;
  int part;
  int level;
  unsigned cmask;  // counts in the spread layout (common.cuh; 0: vertex order)
  unsigned pad_;

  struct alignas(16) Args {
    int start, deg, level, pad;
  };
  struct Acc {
    int changed;
    int remote;
  };

  __device__ int nparents() const { return n_local; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int lu, bool valid, Args& a) const {
    if (!valid || __ldcg(dist + lu) != level) return 0;
    const int s = __ldg(rowptr + lu);
    const int d = __ldg(rowptr + lu + 1) - s;
    a = Args{s, d, level, 0};
    return d > 0 ? d : 0;
  }
  __device__ static int count(const Args& a) { return a.deg; }

  __device__ void push(int q, int v) const {
    const unsigned am = __activemask();
    const unsigned grp = __match_any_sync(am, q);
    const int leader = __ffs(grp) - 1;
    int base = 0;
    if (lane_id() == leader) base = atomicAdd(send_count + q, __popc(grp));
    base = __shfl_sync(grp, base, leader);
    send_buf[(long long)q * stride + base + __popc(grp & lanemask_lt())] = v;
  }
  __device__ void update(int v, int d_or_bits, int lvl, Acc& acc) const {
#if DP_MERGE_COUNTS
    {  // lanes hitting the same vertex merge their increments (BfsApp)
      const unsigned grp = __match_any_sync(__activemask(), v);
      if (lane_id() == __ffs(grp) - 1)
        atomicAdd(counts + spread_slot(v, cmask), __popc(grp));
    }
#else
    atomicAdd(counts + spread_slot(v, cmask), 1);
#endif
    const int q = part_of(v, nparts);
    if (q == part) {
      const int lv = local_of(v, nparts);
      if (d_or_bits == kUnreached &&
          atomicCAS(dist + lv, kUnreached, lvl + 1) == kUnreached)
        acc.changed = 1;
    } else {
      const unsigned bit = 1u << (v & 31);
      if (!((unsigned)d_or_bits & bit) &&
          !(atomicOr(sent + (v >> 5), bit) & bit)) {
        if constexpr (kPeer) {
          ++acc.remote;
          if (atomicCAS(peer_dist[q] + local_of(v, nparts), kUnreached, lvl + 1) ==
              kUnreached)
            acc.changed = 1;
        } else {
          push(q, v);
        }
      }
    }
  }
  // probe: the local dist (L1-cached, see BfsApp) or the sent-bitmap word
  __device__ int probe(int v) const {
    return part_of(v, nparts) == part ? __ldca(dist + local_of(v, nparts))
                              : (int)__ldcg(sent + (v >> 5));
  }
  __device__ void item(const Args& a, int e, Acc& acc) const {
    const int v = __ldg(col + a.start + e);
    update(v, probe(v), a.level, acc);
  }
  static constexpr int kUnroll = DP_GRAPH_UNROLL;
  // whole-warp rows: 4 in flight, as BfsApp (BFS-26 P=1: 22.0 vs 22.6 ms)
  static constexpr int kBigUnroll = 4;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  // register cap (8 blocks of 256 per SM at 32 registers; 5 at 48, 4 at 50)
  static constexpr int kMinBlocks = DP_BFSPART_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    int v[U], d[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      v[j] = ok[j] ? ld_stream(col + args(j).start + e[j]) : 0;
#pragma unroll
    for (int j = 0; j < U; ++j) d[j] = ok[j] ? probe(v[j]) : 0;
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (ok[j]) update(v[j], d[j], args(j).level, acc);
  }
  __device__ void flush(Acc& acc) const {
    // remote discoveries are visible to every part before this warp retires
    const int nr = __reduce_add_sync(DP_FULL, acc.remote);
    if (nr) {
      __threadfence_system();
      if (lane_id() == 0) atomicAdd(remote_ops, (unsigned long long)nr);
    }
    // read before write: after the first success the flag line is only
    // read (shared), not re-written by every succeeding warp
    if (__any_sync(DP_FULL, acc.changed) && lane_id() == 0 &&
        __ldcg(changed) == 0)
      *changed = 1;
  }
};
using BfsPartApp = BfsPartAppT<false>;
using BfsPeerApp = BfsPartAppT<true>;

// ---------------------------------------------------------------------------
// SSSP on one part of the cyclic 1D partition.  Local relaxations lower the
// owned dist in place; a remote relaxation (v, alt) is sent to owner(v) only
// if it strictly improves this part's best-sent value best[v] (atomicMin),
// so a part never re-sends a value that cannot lower dist[v].  Buckets hold
// packed (v << 32 | alt) pairs at per-owner offsets sized by the part's
// edges into each owner (one push per edge per round at most).
// ---------------------------------------------------------------------------
struct SsspPartApp {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const int* __restrict__ weight;
  int* dist;  // owned (local index)
  int* best;  // dense, global ids: best value sent per remote vertex
  unsigned long long* send_buf;
  const long long* send_off;  // [nparts] bucket bases
  int* send_count;            // [nparts]
  int* changed;
  int n_local;
  int nparts;
  int part;
  int pad;

  struct alignas(16) Args {
    int start, deg, du, pad;
  };
  struct Acc {
    int changed;
  };

  __device__ int nparents() const { return n_local; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int lu, bool valid, Args& a) const {
    if (!valid) return 0;
    const int du = __ldcg(dist + lu);
    if (du >= kUnreached) return 0;
    const int s = __ldg(rowptr + lu);
    const int d = __ldg(rowptr + lu + 1) - s;
    a = Args{s, d, du, 0};
    return d > 0 ? d : 0;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  __device__ void push(int q, int v, int alt) const {
    const unsigned am = __activemask();
    const unsigned grp = __match_any_sync(am, q);
    const int leader = __ffs(grp) - 1;
    int base = 0;
    if (lane_id() == leader) base = atomicAdd(send_count + q, __popc(grp));
    base = __shfl_sync(grp, base, leader);
    send_buf[send_off[q] + base + __popc(grp & lanemask_lt())] =
        ((unsigned long long)(unsigned)v << 32) | (unsigned)alt;
  }
  __device__ void relax(int v, int alt, Acc& acc) const {
    const int q = part_of(v, nparts);
    if (q == part) {
      const int lv = local_of(v, nparts);
      if (alt < __ldca(dist + lv) && atomicMin(dist + lv, alt) > alt)
        acc.changed = 1;
    } else if (alt < __ldca(best + v) && atomicMin(best + v, alt) > alt) {
      push(q, v, alt);
    }
  }
  __device__ void item(const Args& a, int e, Acc& acc) const {
    relax(ld_stream(col + a.start + e),
          (int)((unsigned)a.du + (unsigned)ld_stream(weight + a.start + e)),
          acc);
  }
  static constexpr int kUnroll = DP_SSSP_UNROLL;
  static constexpr int kChildUnroll = DP_SSSP_CHILD_UNROLL;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_SSSP_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    int v[U], alt[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = ok[j] ? args(j).start + e[j] : 0;
      v[j] = ok[j] ? ld_stream(col + i) : 0;
      alt[j] = ok[j] ? (int)((unsigned)args(j).du +
                             (unsigned)ld_stream(weight + i))
                     : 0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (ok[j]) relax(v[j], alt[j], acc);
  }
  __device__ void flush(Acc& acc) const {
    // read before write: after the first success the flag line is only
    // read (shared), not re-written by every succeeding warp
    if (__any_sync(DP_FULL, acc.changed) && lane_id() == 0 &&
        __ldcg(changed) == 0)
      *changed = 1;
  }
};

// ---------------------------------------------------------------------------
// SSSP on one part of the cyclic 1D partition, exchange fused into the
// relaxation: the parts' dist arrays are mapped into every part's address
// space (symmetric memory over NVLink / NVSwitch, or plain allocations when
// all parts share one GPU), and a remote relaxation is an atomicMin straight
// into the owner's dist — no send buckets, no all-to-all, no apply pass.
// The per-part best-sent filter still keeps each part from re-sending a value
// that cannot lower dist[v].  A warp that wrote remotely fences system-wide
// before it retires, so the round's remote lowerings are visible to every
// part once the round's flag reduction (the only collective) completes.
// ---------------------------------------------------------------------------
struct SsspPeerApp {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const int* __restrict__ weight;
  int* const* peer_dist;  // [nparts]: every part's dist (local index)
  int* my_dist;           // == peer_dist[part]
  int* best;              // dense, global ids: best value sent per vertex
  int* changed;
  unsigned long long* remote_ops;  // DevState::remote
  int n_local;
  int nparts;
  int part;
  int pad;

  struct alignas(16) Args {
    int start, deg, du, pad;
  };
  struct Acc {
    int changed;
    int remote;
  };

  __device__ int nparents() const { return n_local; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int lu, bool valid, Args& a) const {
    if (!valid) return 0;
    const int du = __ldcg(my_dist + lu);
    if (du >= kUnreached) return 0;
    const int s = __ldg(rowptr + lu);
    const int d = __ldg(rowptr + lu + 1) - s;
    a = Args{s, d, du, 0};
    return d > 0 ? d : 0;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  // probe: the owned dist (L1-cached: values only decrease, a stale copy
  // costs at most a redundant atomic, see BfsApp::items) or the best-sent
  // filter of a remote vertex
  __device__ int probe(int v) const {
    return part_of(v, nparts) == part ? __ldca(my_dist + local_of(v, nparts))
                                      : __ldcg(best + v);
  }
  __device__ void update(int v, int alt, int d, Acc& acc) const {
    if (alt >= d) return;
    const int q = part_of(v, nparts);
    if (q == part) {
      if (atomicMin(my_dist + local_of(v, nparts), alt) > alt) acc.changed = 1;
    } else if (atomicMin(best + v, alt) > alt) {
      ++acc.remote;
      if (atomicMin(peer_dist[q] + local_of(v, nparts), alt) > alt)
        acc.changed = 1;
    }
  }
  __device__ void item(const Args& a, int e, Acc& acc) const {
    const int v = ld_stream(col + a.start + e);
    update(v,
           (int)((unsigned)a.du + (unsigned)ld_stream(weight + a.start + e)),
           probe(v), acc);
  }
  static constexpr int kUnroll = DP_SSSP_UNROLL;
  static constexpr int kChildUnroll = DP_SSSP_CHILD_UNROLL;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_SSSPPEER_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    int v[U], alt[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = ok[j] ? args(j).start + e[j] : 0;
      v[j] = ok[j] ? ld_stream(col + i) : 0;
      alt[j] = ok[j] ? (int)((unsigned)args(j).du +
                             (unsigned)ld_stream(weight + i))
                     : 0;
    }
    int d[U];
#pragma unroll
    for (int j = 0; j < U; ++j) d[j] = ok[j] ? probe(v[j]) : 0;
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (ok[j]) update(v[j], alt[j], d[j], acc);
  }
  __device__ void flush(Acc& acc) const {
    const int nr = __reduce_add_sync(DP_FULL, acc.remote);
    if (nr) {
      __threadfence_system();
      if (lane_id() == 0) atomicAdd(remote_ops, (unsigned long long)nr);
    }
    if (__any_sync(DP_FULL, acc.changed) && lane_id() == 0 &&
        __ldcg(changed) == 0)
      *changed = 1;
  }
};

// ---------------------------------------------------------------------------
// SSSP — SSSP_CDP main/relax_edges/relax (bench/benchmarks.py:175-222)
// ---------------------------------------------------------------------------
// Edge weights packed as nibbles (w - 1, eight per 32-bit word, slot e in
// bits 4*(e & 7) of word e >> 3; dp_config.weight_bits = 4): slots below
// `wslots` read the packed word (the 32 lanes of a warp share one 16-byte
// sector, 1/8 of the int32 bytes), the rest the int32 array.
__device__ __forceinline__ int packed_weight(const unsigned* __restrict__ wp,
                                             int e) {
  return (int)((__ldg(wp + (e >> 3)) >> ((e & 7) << 2)) & 15u) + 1;
}

// kPacked: the weights are read from `wpack` only (a separate
// instantiation: a per-edge choice between the two arrays cost the headline
// kernel its register budget, 1.66 -> 3.1 ms)
template <bool kPacked>
struct SsspAppT {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const int* __restrict__ weight;
  const unsigned* __restrict__ wpack;  // kPacked: nibble-packed weights
  int* dist;
  int* changed;
  int* changed_next;
  int* last;  // frontier mode: distance of u's last relaxation (else null)
  // host-buffer calls: edge slots arrive in 2^shift-slot chunks while the
  // rounds run (null when the graph is resident); deferred parents set
  // *skipped so the loop cannot stop before they have relaxed
  const int* arrived;
  int* skipped;
  int* skipped_next;
  int n;
  int shift;

  struct alignas(16) Args {
    int start, deg, du, pad;
  };
  struct Acc {
    int changed;
  };

  __device__ int nparents() const { return n; }
  __device__ void parent_prologue() const {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *changed_next = 0;
      if (arrived) *skipped_next = 0;
    }
  }
  __device__ SsspAppT for_round(int r, int* flags) const {
    SsspAppT a = *this;
    a.changed = flags + (r & 1);
    a.changed_next = flags + ((r + 1) & 1);
    return a;
  }
  // main (:207-222): every reached u relaxes all its out-edges from its
  // round-start distance du
  __device__ int expand(int u, bool valid, Args& a) const {
    if (!valid) return 0;
    const int du = __ldcg(dist + u);
    if (du >= kUnreached) return 0;
    const int s = __ldg(rowptr + u);
    const int d = __ldg(rowptr + u + 1) - s;
    if (d <= 0) return 0;
    if (arrived && ((s + d - 1) >> shift) >= arrived_chunks(arrived)) {
      // edges still in flight: relax in a later round (the outputs are
      // the unique shortest distances whatever the relaxation order)
      if (__ldcg(skipped) == 0) *skipped = 1;
      return 0;
    }
    if (last) {
      // frontier mode: edges relaxed from du already cannot lower anything
      // again; a vertex lowered later in this round (after this read)
      // differs from last[u] next round and relaxes then, and a round
      // without any lowering leaves every vertex at dist == last
      if (__ldcg(last + u) == du) return 0;
      last[u] = du;
    }
    a = Args{s, d, du, 0};
    return d;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  // relax (:184-195): the CAS loop lowers dist[v] to alt and flags the round
  // when it succeeds; atomicMin reaches the same final value and succeeds
  // exactly when the old value was larger.  Arithmetic wraps like the
  // reference's 32-bit ints (sim/compile.py:36-37).
  __device__ int weight_of(int i) const {
    if constexpr (kPacked)
      return packed_weight(wpack, i);
    else
      return ld_stream(weight + i);
  }
  __device__ void item(const Args& a, int e, Acc& acc) const {
    const int v = __ldg(col + a.start + e);
    const int alt = (int)((unsigned)a.du + (unsigned)weight_of(a.start + e));
    if (alt < __ldcg(dist + v) && atomicMin(dist + v, alt) > alt)
      acc.changed = 1;
  }
  static constexpr int kUnroll = DP_SSSP_UNROLL;
  static constexpr int kChildUnroll = DP_SSSP_CHILD_UNROLL;
  static constexpr bool kBlockMode = false;
  // frontier mode writes last[] in expand: the host never pairs it with the
  // persistent parent (which re-runs expand)
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_SSSP_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    int v[U], alt[U], d[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = ok[j] ? args(j).start + e[j] : 0;
      v[j] = ok[j] ? ld_stream(col + i) : 0;
      alt[j] = ok[j] ? (int)((unsigned)args(j).du + (unsigned)weight_of(i))
                     : 0;
    }
    // L1-cached probe (stale copies are >= the true distance: a stale hit
    // only costs a redundant atomicMin, see BfsApp::items)
#pragma unroll
    for (int j = 0; j < U; ++j) d[j] = ok[j] ? __ldca(dist + v[j]) : 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
#if DP_SSSP_RED
      if (ok[j] && alt[j] < d[j]) {
        red_min(dist + v[j], alt[j]);
        acc.changed = 1;
      }
#else
      if (ok[j] && alt[j] < d[j] && atomicMin(dist + v[j], alt[j]) > alt[j])
        acc.changed = 1;
#endif
    }
  }
  __device__ void flush(Acc& acc) const {
    // read before write: after the first success the flag line is only
    // read (shared), not re-written by every succeeding warp
    if (__any_sync(DP_FULL, acc.changed) && lane_id() == 0 &&
        __ldcg(changed) == 0)
      *changed = 1;
  }
};

using SsspApp = SsspAppT<false>;
using SsspPackedApp = SsspAppT<true>;

// ---------------------------------------------------------------------------
// manylaunch — MANYLAUNCH_CDP main/spawn (bench/benchmarks.py:283-300)
// ---------------------------------------------------------------------------
struct ManyLaunchApp {
  const int* __restrict__ sizes;
  int* out;
  int* total;
  int n;
  int pad;

  struct alignas(16) Args {
    int s, i, pad0, pad1;
  };
  struct Acc {
    int cnt;
  };

  __device__ int nparents() const { return n; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int u, bool valid, Args& a) const {
    if (!valid) return 0;
    const int s = __ldg(sizes + u);
    a = Args{s, u, 0, 0};
    return s > 0 ? s : 0;
  }
  __device__ static int count(const Args& a) { return a.s; }
  // spawn (:284-290): out[i] += j + 1; total[0] += 1.  The hot total[0]
  // increment is summed per warp in flush (one atomic per warp).
  __device__ void item(const Args& a, int j, Acc& acc) const {
    atomicAdd(out + a.i, j + 1);
    acc.cnt += 1;
  }
  static constexpr int kUnroll = 1;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = 1;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    items_loop<U>(*this, args, e, ok, acc);
  }
  __device__ void flush(Acc& acc) const {
    const int c = __reduce_add_sync(DP_FULL, acc.cnt);
    if (c && lane_id() == 0) atomicAdd(total, c);
  }
};

// ---------------------------------------------------------------------------
// Graph coloring (north-star app; no reference implementation).  Jones-
// Plassmann with a deterministic priority key(v) = (hash(v), v): a vertex is
// coloured once all its higher-priority neighbours are, with the smallest
// colour they do not use — exactly the sequential greedy colouring in
// priority order, whatever the schedule.  Counter form: wait[u] = number of
// still-uncoloured higher-priority neighbours; rounds run over a worklist of
// ready vertices (wait == 0), so every vertex scans its neighbours a
// constant number of times (O(m) total) instead of once per round.  The
// worklist length lives on the device (parents beyond it exit), so rounds
// are queued without a host readback each:
//   GcCountApp   parent = vertex, child = neighbour: wait[u] += key(w) > key(u)
//   GcGatherApp  parent = ready vertex, child = neighbour: a higher-priority
//                neighbour's colour c is marked in u's (deg+1)-bit bitmap at
//                bit offset rowptr[u] + u + c  (then a flat mex pass)
//   GcNotifyApp  parent = vertex coloured this round, child = neighbour: a
//                lower-priority neighbour's wait drops; at 0 it joins the
//                next round's worklist
// ---------------------------------------------------------------------------
// Priority: largest-log-degree-first with a hash tie-break (Hasenplaugh et
// al.'s LLF ordering): key(v) = floor(log2(deg v + 1)) : 5 bits | high 27
// bits of hash32(v) | v : 32 bits.  Unique per vertex.  Against a pure hash
// order on RMAT-20 it colours with 186 instead of 240 colours and shortens
// the longest priority chain (= the rounds) from 1,644 to 1,531
// (profiles/gc_policies_r01b.txt).
__host__ __device__ __forceinline__ unsigned long long gc_key(int v, int deg) {
  unsigned x = (unsigned)v * 0x9E3779B1u;
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  unsigned lg = 0;
  for (unsigned d = (unsigned)deg + 1u; d > 1u; d >>= 1) ++lg;
  return ((unsigned long long)lg << 59) |
         ((unsigned long long)(x >> 5) << 32) | (unsigned)v;
}

struct GcCountApp {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const unsigned long long* __restrict__ key;  // gc_key per vertex
  int* wait;
  int n;
  int pad;

  struct alignas(16) Args {
    int start, deg, u, pad;
  };
  // run-length count of the vertex this thread works on (one atomic per
  // vertex per thread instead of one per edge)
  struct Acc {
    int u, c;
  };

  __device__ int nparents() const { return n; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int u, bool valid, Args& a) const {
    if (!valid) return 0;
    const int s = __ldg(rowptr + u);
    const int d = __ldg(rowptr + u + 1) - s;
    a = Args{s, d, u, 0};
    return d > 0 ? d : 0;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  __device__ void item(const Args& a, int e, Acc& acc) const {
    const int w = ld_stream(col + a.start + e);
    if (acc.c && acc.u != a.u) {
      atomicAdd(wait + acc.u, acc.c);
      acc.c = 0;
    }
    acc.u = a.u;
    acc.c += __ldg(key + w) > __ldg(key + a.u);
  }
  static constexpr int kUnroll = 1;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = 1;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    items_loop<U>(*this, args, e, ok, acc);
  }
  __device__ void flush(Acc& acc) const {
    if (acc.c) atomicAdd(wait + acc.u, acc.c);
  }
};

struct GcGatherApp {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const unsigned long long* __restrict__ key;
  const int* __restrict__ ready;  // this round's worklist
  const int* nready;              // its length (on the device)
  const int* color;
  unsigned* used;  // bit rowptr[u] + u + c: colour c taken by a neighbour

  struct alignas(16) Args {
    int start, deg, u, pad;
  };
  struct Acc {};

  __device__ int nparents() const { return __ldcg(nready); }
  __device__ void parent_prologue() const {}
  __device__ int expand(int i, bool valid, Args& a) const {
    if (!valid) return 0;
    const int u = __ldcg(ready + i);
    const int s = __ldg(rowptr + u);
    const int d = __ldg(rowptr + u + 1) - s;
    a = Args{s, d, u, 0};
    return d > 0 ? d : 0;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  __device__ void item(const Args& a, int e, Acc&) const {
    const int w = ld_stream(col + a.start + e);
    // lower priority: not coloured yet
    if (__ldg(key + w) < __ldg(key + a.u)) return;
    const int c = __ldcg(color + w);
    if (c >= 0 && c <= a.deg) {
      const long long bit = (long long)a.start + a.u + c;
      atomicOr(used + (bit >> 5), 1u << (bit & 31));
    }
  }
  static constexpr int kUnroll = 1;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = 1;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    items_loop<U>(*this, args, e, ok, acc);
  }
  __device__ void flush(Acc&) const {}
};

struct GcNotifyApp {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const unsigned long long* __restrict__ key;
  const int* __restrict__ ready;  // vertices coloured this round
  const int* nready;
  int* wait;
  int* next;        // next round's worklist
  int* next_count;

  struct alignas(16) Args {
    int start, deg, u, pad;
  };
  struct Acc {};

  __device__ int nparents() const { return __ldcg(nready); }
  __device__ void parent_prologue() const {}
  __device__ int expand(int i, bool valid, Args& a) const {
    if (!valid) return 0;
    const int u = __ldcg(ready + i);
    const int s = __ldg(rowptr + u);
    const int d = __ldg(rowptr + u + 1) - s;
    a = Args{s, d, u, 0};
    return d > 0 ? d : 0;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  __device__ void item(const Args& a, int e, Acc&) const {
    const int w = ld_stream(col + a.start + e);
    const bool last =
        __ldg(key + w) < __ldg(key + a.u) && atomicSub(wait + w, 1) == 1;
    // warp-aggregated append of the vertices that just became ready
    const unsigned am = __activemask();
    const unsigned m = __ballot_sync(am, last);
    if (!m) return;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane_id() == leader) base = atomicAdd(next_count, __popc(m));
    base = __shfl_sync(am, base, leader);
    if (last) next[base + __popc(m & lanemask_lt())] = w;
  }
  static constexpr int kUnroll = 1;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = 1;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    items_loop<U>(*this, args, e, ok, acc);
  }
  __device__ void flush(Acc&) const {}
};

// ---------------------------------------------------------------------------
// Triangle counting (no reference implementation)
//   Input: the rank-ordered CSR+ (dp_tc_orient: vertices relabelled by
//   (degree, id) rank, u -> v iff u < v, out-lists N+ ascending).  The call
//   builds its transpose on the device (in-edges, restricted to the
//   oriented-edge range [edge_lo, edge_hi) of a shard), each in-edge (u, v)
//   stored as the slot range of N+(u) above v.
//   parent = vertex v, child item = in-edge (u, v), work = |N+(u)>v ∩ N+(v)|.
//   A triangle u < v < w is found once, at v, from u's list past v: probing
//   that suffix into a set of N+(v) (built once per child block) costs
//   sum_u d+(u)(d+(u)-1)/2 probes -- half of probing all of N+(u), 14.5 G on
//   RMAT-22; the forward form, N+(v) into a set of N+(u), costs 28.9 G.
// ---------------------------------------------------------------------------
struct TcApp {
  const int* __restrict__ rowptr;     // CSR+ (out)
  const int* __restrict__ col;
  const int* __restrict__ in_rowptr;  // transpose (in), shard edges only
  const int2* __restrict__ in_rng;    // per in-edge (u, v): N+(u) slots > v
  unsigned long long* total;
  int n;
  int pad;

  struct alignas(16) Args {
    int v, first, cnt, pad;  // in-edges [first, first + cnt) of v
  };
  struct Acc {
    unsigned long long tri;
  };

  __device__ int nparents() const { return n; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int v, bool valid, Args& a) const {
    if (!valid) return 0;
    const int b = __ldg(in_rowptr + v), e = __ldg(in_rowptr + v + 1);
    if (e <= b || __ldg(rowptr + v + 1) == __ldg(rowptr + v)) return 0;
    a = Args{v, b, e - b, 0};
    return e - b;
  }
  __device__ static int count(const Args& a) { return a.cnt; }

  // |A ∩ B| of two ascending lists: walk the shorter, lower_bound into the
  // longer with a window that only moves forward.
  __device__ static int intersect(const int* __restrict__ A, int na,
                                  const int* __restrict__ B, int nb) {
    if (na > nb) {
      const int* t = A; A = B; B = t;
      int tn = na; na = nb; nb = tn;
    }
    int c = 0, lo = 0;
    for (int i = 0; i < na && lo < nb; ++i) {
      const int x = __ldg(A + i);
      int hi = nb;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(B + mid) < x) lo = mid + 1; else hi = mid;
      }
      if (lo < nb && __ldg(B + lo) == x) { ++c; ++lo; }
    }
    return c;
  }

  __device__ void item(const Args& a, int e, Acc& acc) const {
    const int2 ur = __ldg(in_rng + a.first + e);
    const int vb = __ldg(rowptr + a.v), ve = __ldg(rowptr + a.v + 1);
    acc.tri += (unsigned long long)intersect(col + ur.x, ur.y - ur.x,
                                             col + vb, ve - vb);
  }
  static constexpr int kUnroll = 1;

  // Child blocks: N+(v) goes into a shared-memory hash set once per physical
  // block; each warp then takes 32 in-edges (u, v), flattens their lists
  // N+(u) into one list (load-balanced, owner lane by shuffle search) and
  // probes the set: coalesced reads of N+(u), O(1) lookups, no per-thread
  // merge chains.  Lists longer than kSlots/2 fall back to per-thread merges.
  static constexpr bool kBlockMode = true;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_TC_MINB;
  static constexpr int kSlotBits = 12;
  static constexpr int kSlots = 1 << kSlotBits;  // 16 KB of shared memory

  __device__ static unsigned hash_slot(int x, int bits) {
    return ((unsigned)x * 2654435761u) >> (32 - bits);
  }

  __device__ void block_items(const Args& a, long long e0, long long e1,
                              Acc& acc) const {
    __shared__ int set[kSlots];
    __shared__ unsigned char owner8[8][32 * 32];  // <= 8 warps (cb <= 256)
    const int vb = __ldg(rowptr + a.v), ve = __ldg(rowptr + a.v + 1);
    if (ve - vb > kSlots / 2) {
      for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x)
        item(a, (int)e, acc);
      return;
    }
    // always the full sparse table: most probes are misses (wedges >>
    // triangles) and a linear-probing miss costs ~1/(1-load)^2 probes; the
    // clear is 16 stores per thread.  Measured (profiles/tune_tc_*): sizing
    // the table to the list (load 1/2) or to 32 KB (lower occupancy) is
    // slower.
    const int bits = kSlotBits;
    const unsigned mask = (1u << bits) - 1;
    for (int i = threadIdx.x; i <= (int)mask; i += blockDim.x) set[i] = -1;
    __syncthreads();
    for (int i = vb + threadIdx.x; i < ve; i += blockDim.x) {
      const int x = __ldg(col + i);
      unsigned h = hash_slot(x, bits);
      while (atomicCAS(&set[h], -1, x) != -1) h = (h + 1) & mask;
    }
    __syncthreads();
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned tri = 0;  // per-lane hits (<= 2^32 per block call)
    auto hit = [&](int w) -> unsigned {
      unsigned h = hash_slot(w, bits);
      int key;
      while ((key = set[h]) != -1 && key != w) h = (h + 1) & mask;
      return key == w;
    };
    for (long long base = e0 + 32LL * wid; base < e1; base += 32LL * nw) {
      const long long e = base + lane;
      int ub = 0, du = 0;
      if (e < e1) {
        const int2 ur = __ldg(in_rng + a.first + e);
        ub = ur.x;
        du = ur.y - ur.x;
      }
      // long lists: the whole warp walks one list at a time, four
      // coalesced loads in flight per lane
      unsigned big = __ballot_sync(DP_FULL, du >= 32);
      while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const int b = __shfl_sync(DP_FULL, ub, src);
        const int d = __shfl_sync(DP_FULL, du, src);
        for (int i = lane; i < d; i += 128) {
          int w[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            w[j] = i + 32 * j < d ? __ldg(col + b + i + 32 * j) : -1;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (w[j] >= 0) tri += hit(w[j]);
        }
      }
      // short lists (< 32): flattened into one load-balanced list; each
      // item's owner lane comes from a per-warp byte table filled once (one
      // shared-memory load per item instead of a 5-step shuffle search)
      const int ds = du < 32 ? du : 0;
      const int incl = warp_incl_scan(ds);
      const int total = __shfl_sync(DP_FULL, incl, 31);
      const int excl = incl - ds;
      unsigned char* own = owner8[wid];
      for (int i = 0; i < ds; ++i) own[excl + i] = (unsigned char)lane;
      __syncwarp();
      const int lbase = ub - excl;
      for (int k0 = 0; k0 < total; k0 += 32) {
        const int k = k0 + lane;
        const int owner = k < total ? own[k] : 0;
        const int pos = __shfl_sync(DP_FULL, lbase, owner) + k;
        if (k < total) tri += hit(__ldg(col + pos));
      }
      __syncwarp();  // own[] is refilled for the next 32 in-edges
    }
    acc.tri += tri;
  }
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    items_loop<U>(*this, args, e, ok, acc);
  }
  __device__ void flush(Acc& acc) const {
    const unsigned long long s = warp_sum_u64(acc.tri);
    if (s && lane_id() == 0) atomicAdd(total, s);
  }
};

// ---------------------------------------------------------------------------
// Bezier line tessellation (no reference implementation; modelled on the
// CUDA sample cdpBezierTessellation cited by PAPER.md:433; SURVEY §8(d) cfg 2)
//   parent = curve: curvature -> vertex count, bump-allocate its vertices
//   (the original's device-side cudaMalloc); child item i =
//   vertex B(i / (ntess - 1)).
// ---------------------------------------------------------------------------
struct BtApp {
  const float2* __restrict__ cp;  // [ncurves][3]
  int* ntess;
  long long* offsets;
  float2* verts;
  unsigned long long* cursor;  // bump allocator
  int* overflow;
  long long cap;  // vertex capacity
  int ncurves;
  int max_tess;
  float scale;
  int pad;

  // the row carries the curve's control points and 1/(nt-1) (loaded once
  // by the parent in expand): the warp walking a curve receives them with
  // the row's shuffle instead of re-loading them per vertex
  struct alignas(16) Args {
    int nt;
    float inv;
    long long off;
    float2 p0, p1, p2;
  };
  struct Acc {};

  __device__ int nparents() const { return ncurves; }
  __device__ void parent_prologue() const {}

  // Vertex count from curvature, fp32 with explicit round-to-nearest ops
  // (no FMA contraction) so the CPU oracle reproduces it bit-for-bit:
  //   curv = |P1 - (P0+P2)/2| / |P2 - P0|,  nt = clamp(int(curv*scale), 4, max)
  __device__ static int tess_count(float2 p0, float2 p1, float2 p2,
                                   float scale, int max_tess) {
    const float mx = __fmul_rn(0.5f, __fadd_rn(p0.x, p2.x));
    const float my = __fmul_rn(0.5f, __fadd_rn(p0.y, p2.y));
    const float dx = __fsub_rn(p1.x, mx), dy = __fsub_rn(p1.y, my);
    const float lx = __fsub_rn(p2.x, p0.x), ly = __fsub_rn(p2.y, p0.y);
    const float num = __fsqrt_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)));
    const float den = __fsqrt_rn(__fadd_rn(__fmul_rn(lx, lx), __fmul_rn(ly, ly)));
    const float t = __fmul_rn(__fdiv_rn(num, den), scale);
    int nt = t < (float)max_tess ? (int)t : max_tess;  // NaN/inf -> max
    return nt < 4 ? 4 : nt;
  }

  __device__ int expand(int u, bool valid, Args& a) const {
    int nt = 0;
    float2 q0 = make_float2(0.f, 0.f), q1 = q0, q2 = q0;
    if (valid) {
      q0 = __ldg(cp + 3 * u);
      q1 = __ldg(cp + 3 * u + 1);
      q2 = __ldg(cp + 3 * u + 2);
      nt = tess_count(q0, q1, q2, scale, max_tess);
    }
    // warp-aggregated bump allocation: one 64-bit atomic per warp
    const int incl = warp_incl_scan(nt);
    unsigned long long base = 0;
    if (lane_id() == 31 && incl > 0) base = atomicAdd(cursor, (unsigned long long)incl);
    base = __shfl_sync(DP_FULL, base, 31);
    if (!valid) return 0;
    const long long off = (long long)base + incl - nt;
    if (off + nt > cap) {  // output pool exhausted: report, do not write
      atomicExch(overflow, 1);
      ntess[u] = nt;
      offsets[u] = -1;
      return 0;
    }
    ntess[u] = nt;
    offsets[u] = off;
    a = Args{nt, __frcp_rn((float)(nt - 1)), off, q0, q1, q2};
    return nt;
  }
  __device__ static int count(const Args& a) { return a.nt; }
  __device__ void item(const Args& a, int i, Acc&) const {
    // t = i * (1/(nt-1)) (<= 1.5 ulp): vertices are checked within 1e-5, only
    // the counts (tess_count) must match the oracle bit for bit
    const float t = (float)i * a.inv;
    const float s = 1.0f - t;
    const float w0 = s * s, w1 = 2.0f * s * t, w2 = t * t;
    verts[a.off + i] = make_float2(w0 * a.p0.x + w1 * a.p1.x + w2 * a.p2.x,
                                   w0 * a.p0.y + w1 * a.p1.y + w2 * a.p2.y);
  }
  static constexpr int kUnroll = 1;
  static constexpr int kBigUnroll = 4;  // whole-warp rows: 4 stores in flight
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = false;  // bump-allocates in expand
  static constexpr int kMinBlocks = DP_BT_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    items_loop<U>(*this, args, e, ok, acc);
  }
  __device__ void flush(Acc&) const {}
};

// ---------------------------------------------------------------------------
// Minimum spanning forest, Boruvka rounds — the paper's MSTF (find) and MSTV
// (verify) kernels (from the LonestarGPU / KLAP suite; no
// reference code).  Input: symmetric simple CSR, symmetric weights, and per
// slot the canonical undirected edge id eid (the slot of its (min,max) copy).
// Edges are totally ordered by key = (weight, eid), so the forest is unique
// and equals Kruskal's in that order (oracle_mst) whatever the schedule.
//   comp[v]   component root of v (fully compressed between rounds)
//   cmin[c]   min key leaving component c (atomicMin), kNoEdge if none
// MSTF: parent = vertex, child item = out-edge: a cross-component edge lowers
// cmin[comp u].  MSTV: parent = the go-ahead vertex of its component (the
// endpoint of the edge cmin names).  If it is the smaller endpoint, the
// canonical slot lies in its own row and it marks the edge directly; the
// larger endpoint expands its row (child item = out-edge) to find the slot
// whose eid realises the minimum, marks the forest edge and records the
// partner component (LonestarGPU verify_min_elem).  Hook + pointer jumping are flat kernels in
// dynpar.cu.
// ---------------------------------------------------------------------------
constexpr unsigned long long kNoEdge = ~0ull;

// order-preserving map of a signed weight into the high half of the key
__host__ __device__ __forceinline__ unsigned long long mst_key(int w, int eid) {
  return ((unsigned long long)((unsigned)w ^ 0x80000000u) << 32) |
         (unsigned)eid;
}

struct MstFindApp {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const int* __restrict__ weight;
  const int* __restrict__ eid;
  const int* __restrict__ comp;  // read-only during the kernel
  unsigned long long* cmin;
  int* changed;  // some cross-component edge exists
  int n;
  int pad;

  struct alignas(16) Args {
    int start, deg, cu, pad;
  };
  struct Acc {
    int changed;
  };

  __device__ int nparents() const { return n; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int u, bool valid, Args& a) const {
    if (!valid) return 0;
    const int s = __ldg(rowptr + u);
    const int d = __ldg(rowptr + u + 1) - s;
    if (d <= 0) return 0;
    a = Args{s, d, __ldg(comp + u), 0};
    return d;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  __device__ __forceinline__ void offer(int cu, unsigned long long k,
                                        Acc& acc) const {
    acc.changed = 1;
    // cmin only decreases during the kernel: the plain L2 pre-check skips
    // atomics that cannot succeed
    if (k < __ldcg(cmin + cu)) atomicMin(cmin + cu, k);
  }
  __device__ void item(const Args& a, int e, Acc& acc) const {
    const int i = a.start + e;
    const int v = ld_stream(col + i);
    if (__ldg(comp + v) != a.cu)
      offer(a.cu, mst_key(ld_stream(weight + i), ld_stream(eid + i)), acc);
  }
  static constexpr int kUnroll = 4;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_MST_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    int v[U], c[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      v[j] = ok[j] ? ld_stream(col + args(j).start + e[j]) : 0;
#pragma unroll
    for (int j = 0; j < U; ++j) c[j] = ok[j] ? __ldg(comp + v[j]) : 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (!ok[j] || c[j] == args(j).cu) continue;
      const int i = args(j).start + e[j];
      offer(args(j).cu,
            mst_key(ld_stream(weight + i), ld_stream(eid + i)), acc);
    }
  }
  __device__ void flush(Acc& acc) const {
    if (__any_sync(DP_FULL, acc.changed) && lane_id() == 0 &&
        __ldcg(changed) == 0)
      *changed = 1;
  }
};

struct MstVerifyApp {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const int* __restrict__ eid;
  const int* __restrict__ comp;
  const unsigned long long* __restrict__ cmin;
  unsigned char* in_mst;  // [m], set at the canonical slot
  int* partner;           // [n] per component root: the other component
  int n;
  int pad;

  struct alignas(16) Args {
    int start, deg, cu, want;  // want = eid of the component's min edge
  };
  struct Acc {};

  __device__ int nparents() const { return n; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int u, bool valid, Args& a) const {
    if (!valid) return 0;
    const int cu = __ldg(comp + u);
    const unsigned long long k = __ldcg(cmin + cu);
    if (k == kNoEdge) return 0;
    const int want = (int)(unsigned)(k & 0xffffffffull);
    const int s = __ldg(rowptr + u);
    const int d = __ldg(rowptr + u + 1) - s;
    // u is an endpoint of the chosen edge: its smaller endpoint owns the
    // canonical slot, the larger one is that slot's target.  The endpoint in
    // the other component is checked against that component's minimum.
    if (want >= s && want < s + d) {
      // the smaller endpoint owns the canonical slot: nothing to search
      // (idempotent stores, so a re-run of expand is harmless)
      in_mst[want] = 1;
      partner[cu] = __ldg(comp + __ldg(col + want));
      return 0;
    }
    // the larger endpoint scans its row for the mirror slot
    if (__ldg(col + want) != u) return 0;
    a = Args{s, d, cu, want};
    return d > 0 ? d : 0;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  __device__ void item(const Args& a, int e, Acc&) const {
    const int i = a.start + e;
    if (ld_stream(eid + i) == a.want) {  // unique: one slot per component
      in_mst[a.want] = 1;
      partner[a.cu] = __ldg(comp + __ldg(col + i));
    }
  }
  static constexpr int kUnroll = 4;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_MST_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    items_loop<U>(*this, args, e, ok, acc);
  }
  __device__ void flush(Acc&) const {}
};

// ---------------------------------------------------------------------------
// Survey propagation on random k-SAT — the paper's SP (from the
// LonestarGPU / KLAP suite; no reference code).  Factor graph: clause a owns
// edges e in [a*k, (a+1)*k), lit[e] = var << 1 | negated; the variable-major
// CSR (occ_row, occs) lists each variable's edges, packed on the device as
// occs[t] = e << 1 | negated so the variable side never gathers lit.  One
// synchronous sweep of the surveys eta (Braunstein, Mezard, Zecchina 2005):
//   SpVarApp    parent = variable i, child item = occurrence e of i:
//               P_s(i) *= (1 - eta[e]) for the occurrence's sign s, zero
//               factors counted apart (so one factor can be divided out);
//               run once per L2 window of eta (below)
//   SpRatioApp  parent = clause a, child item = edge e = (a, i):
//               ratio[e] = Pu / (Pu + Ps + P0), S = P_s(i) / (1 - eta[e])
//               (a excluded), U = P_-s(i), Pu = (1-U) S, Ps = (1-S) U, P0 = SU
//               (products are L2-resident, eta / ratio contiguous)
//   SpClauseApp parent = clause a, child item = edge (a, i):
//               eta'[a, i] = prod_{j in a, j != i} ratio[a, j]  (contiguous)
// Only the variable pass gathers (eta by occurrence): measured on 5-SAT,
// a variable-major ratio pass costs 3.2 GB of DRAM per sweep (random eta
// gathers + ratio scatters, ~64 B per 8 B access) against ~0.5 GB here.
// The gather can be windowed (DYNPAR_SP_WINDOW_MB): the variable pass runs
// once per slice of the edge (= eta) index space small enough to stay in L2,
// each parent taking only its occurrences inside the slice (a variable's
// occurrence list is sorted by edge, so a slice is a sub-range: seg_lo /
// seg_hi).  One pass over the whole 160 MB eta of 5-SAT 200k read 1.92 GB
// of DRAM (L2 hit 32 %, profiles/ncu_full_sp_ksat5_r01.json), four 48 MB
// windows 4 x 145 MB; but once the occurrence lists are read through L1
// (DP_SP_OCC_L1) one pass is faster (5-SAT 12.96 vs 13.29 ms at 96 MB,
// 3-SAT 9.66 vs 10.36 ms: profiles/r02/ab_sp_win2_r02.txt), so it is off
// by default.  Scattering variable-major factors
// from the clause pass instead was measured slower (5-SAT 20.9 vs 19.5 ms,
// 3-SAT 14.8 vs 11.9 ms: partial-sector writes cost more than the gathers).
// Arithmetic and storage in fp64 (explicit round-to-nearest ops, no FMA
// contraction, as the CPU oracle does).  The product order of P_s depends on
// the schedule, so results match the oracle within a tolerance, not
// bit-exactly (tests state it).  fp64 storage matters: the first sweeps
// amplify perturbations ~1e6-fold (a 1-ulp fp32 change of eta0 moves 5-SAT
// surveys by 0.08 after 10 sweeps), so fp32 rounding flips would not stay
// within tolerance; fp64 order effects (~1e-16) do.
// ---------------------------------------------------------------------------
// 32 B: the ratio pass fetches a variable's record with one 256-bit load
struct alignas(16) SpVarProd {
  double p[2];  // product of the non-zero (1 - eta) factors, per sign
  int z[2];     // zero factors, per sign
  int pad[2];
};

__device__ __forceinline__ void atomic_mul_f64(double* addr, double f) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = __ldcg(a), assumed;
  do {
    assumed = old;
    old = atomicCAS(a, assumed,
                    __double_as_longlong(__dmul_rn(__longlong_as_double(assumed), f)));
  } while (old != assumed);
}

struct SpVarApp {
  const int* __restrict__ seg_lo;  // variable i's occurrences in this
  const int* __restrict__ seg_hi;  // window: occs[seg_lo[i], seg_hi[i])
  const int* __restrict__ occs;    // sp_tile(e) << 1 | negated
  const double* __restrict__ eta;
  SpVarProd* prod;
  int nvars;
  int pad;

  struct alignas(16) Args {
    int start, deg, i, pad;
  };
  // run-length partial product of the variable this thread is working on:
  // committed when the thread moves to another variable, and in flush()
  // merged across the lanes of the warp holding the same variable, so a
  // variable costs ~one CAS per sign per warp instead of one per occurrence
  // (5-SAT: ~100 occurrences per variable hitting two words)
  struct Acc {
    int has, var;
    int z[2];
    double p[2];
  };

  __device__ int nparents() const { return nvars; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int i, bool valid, Args& a) const {
    if (!valid) return 0;
    const int s = __ldg(seg_lo + i);
    const int d = __ldg(seg_hi + i) - s;
    a = Args{s, d, i, 0};
    return d > 0 ? d : 0;
  }
  __device__ static int count(const Args& a) { return a.deg; }
  __device__ void commit(int var, const double* p, const int* z) const {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (p[s] != 1.0) atomic_mul_f64(&prod[var].p[s], p[s]);
      if (z[s]) atomicAdd(&prod[var].z[s], z[s]);
    }
  }
  __device__ double factor(const Args& a, int t, int& neg) const {
#if DP_SP_OCC_L1
    // thread-mode serial arm: a lane walks its own variable's list, so the
    // next occurrences sit in the sector just fetched -- keep it in L1
    const int o = __ldg(occs + a.start + t);
#else
    const int o = ld_stream(occs + a.start + t);
#endif
    neg = o & 1;
    return __dsub_rn(1.0, __ldg(eta + (o >> 1)));
  }
  __device__ void item(const Args& a, int t, Acc& acc) const {
    int neg;
    const double f = factor(a, t, neg);
    fold(a, f, neg, acc);
  }
  __device__ __forceinline__ void fold(const Args& a, double f, int neg,
                                       Acc& acc) const {
    if (acc.has && acc.var != a.i) {
      commit(acc.var, acc.p, acc.z);
      acc.has = 0;
    }
    if (!acc.has) {
      acc.has = 1;
      acc.var = a.i;
      acc.p[0] = acc.p[1] = 1.0;
      acc.z[0] = acc.z[1] = 0;
    }
    if (f == 0.0)
      acc.z[neg] += 1;
    else
      acc.p[neg] = __dmul_rn(acc.p[neg], f);
  }
  static constexpr int kUnroll = DP_SP_VAR_UNROLL;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_SP_MINB;
  // all U gathers first, then the folds in item order (same products):
  // a fold may commit with atomics, which would otherwise keep the next
  // item's loads from being issued ahead of it
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    double f[U];
    int neg[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      f[j] = ok[j] ? factor(args(j), e[j], neg[j]) : (neg[j] = 0, 1.0);
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (ok[j]) fold(args(j), f[j], neg[j], acc);
  }
  __device__ void flush(Acc& acc) const {
    const int key = acc.has ? acc.var : -1;
    const unsigned grp = __match_any_sync(DP_FULL, key);
    const int leader = __ffs(grp) - 1;
    double p0 = 1.0, p1 = 1.0;
    int z0 = 0, z1 = 0;
    for (unsigned m = grp; m; m &= m - 1) {  // same trip count in the group
      const int src = __ffs(m) - 1;
      p0 = __dmul_rn(p0, __shfl_sync(grp, acc.p[0], src));
      p1 = __dmul_rn(p1, __shfl_sync(grp, acc.p[1], src));
      z0 += __shfl_sync(grp, acc.z[0], src);
      z1 += __shfl_sync(grp, acc.z[1], src);
    }
    if (key >= 0 && lane_id() == leader) {
      const double p[2] = {p0, p1};
      const int z[2] = {z0, z1};
      commit(key, p, z);
    }
  }
};

// the survey a variable's occurrence contributes towards its clause:
// Pu / (Pu + Ps + P0) (0 when all three vanish)
__device__ __forceinline__ double sp_ratio(const double* p, const int* z,
                                           int neg, double eta_e) {
  const double f = __dsub_rn(1.0, eta_e);
  double S;  // same-sign product with this clause divided out
  if (f == 0.0)
    S = z[neg] - 1 == 0 ? p[neg] : 0.0;
  else
    S = z[neg] == 0 ? __ddiv_rn(p[neg], f) : 0.0;
  const double U = z[neg ^ 1] == 0 ? p[neg ^ 1] : 0.0;
  const double pu = __dmul_rn(__dsub_rn(1.0, U), S);
  const double ps = __dmul_rn(__dsub_rn(1.0, S), U);
  const double p0 = __dmul_rn(S, U);
  const double den = __dadd_rn(__dadd_rn(pu, ps), p0);
  return den > 0.0 ? __ddiv_rn(pu, den) : 0.0;
}

// Clause-tiled edge layout of lit / eta / ratio on the device: literal j of
// clause a at ((a >> 5) k + j) 32 + (a & 31).  With the serial arm in thread
// mode a lane owns one clause, so the 32 lanes of a warp read literal j of
// 32 consecutive clauses: one coalesced 128 B (int) / 256 B (double) access
// instead of 32 accesses at a k-element stride (clause-major: L1 throughput
// 89 % for 18 % DRAM in the ratio pass, profiles/r02/ncu_full_sp_window_r02.json).
// The caller's clause-major eta is tiled on entry and untiled on exit.
__host__ __device__ __forceinline__ long long sp_tile(long long a, int j,
                                                      int k) {
  return (((a >> 5) * k + j) << 5) + (a & 31);
}

struct SpRatioApp {
  const int* __restrict__ lit;         // clause-tiled (sp_tile)
  const double* __restrict__ eta;      // clause-tiled
  const SpVarProd* __restrict__ prod;  // L2-resident (32 B per variable)
  double* __restrict__ ratio;          // clause-tiled
  int nclauses;
  int k;

  struct alignas(16) Args {
    int a, k, pad0, pad1;
  };
  struct Acc {};

  __device__ int nparents() const { return nclauses; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int a, bool valid, Args& r) const {
    if (!valid) return 0;
    r = Args{a, k, 0, 0};
    return k;
  }
  __device__ static int count(const Args& r) { return r.k; }
  __device__ void item(const Args& r, int t, Acc&) const {
    const long long e = sp_tile(r.a, t, r.k);
    const int l = ld_stream(lit + e);
    // the variable's 32 B record in one 256-bit L2 load (sm_100)
    unsigned long long q0, q1, q2, q3;
    asm("ld.global.cg.v4.b64 {%0, %1, %2, %3}, [%4];"
        : "=l"(q0), "=l"(q1), "=l"(q2), "=l"(q3)
        : "l"(prod + (l >> 1)));
    (void)q3;
    const double p[2] = {__longlong_as_double(q0), __longlong_as_double(q1)};
    const int z[2] = {(int)(unsigned)q2, (int)(unsigned)(q2 >> 32)};
    ratio[e] = sp_ratio(p, z, l & 1, __ldg(eta + e));
  }
  static constexpr int kUnroll = DP_SP_UNROLL;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_SP_RATIO_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    items_loop<U>(*this, args, e, ok, acc);
  }
  __device__ void flush(Acc&) const {}
};

struct SpClauseApp {
  const double* __restrict__ ratio;
  const double* __restrict__ eta;  // previous sweep
  double* eta_next;
  unsigned* max_delta;  // float bits of max |eta' - eta| (rounded up)
  int nclauses;
  int k;

  struct alignas(16) Args {
    int a, k, pad0, pad1;
  };
  struct Acc {
    float delta;
  };

  __device__ int nparents() const { return nclauses; }
  __device__ void parent_prologue() const {}
  __device__ int expand(int a, bool valid, Args& r) const {
    if (!valid) return 0;
    r = Args{a, k, 0, 0};
    return k;
  }
  __device__ static int count(const Args& r) { return r.k; }
  __device__ void item(const Args& r, int t, Acc& acc) const {
    const long long base = sp_tile(r.a, 0, r.k);  // literal j at base + 32 j
    double v = 1.0;
    for (int j = 0; j < r.k; ++j)  // fixed order: the oracle's
      if (j != t) v = __dmul_rn(v, __ldg(ratio + base + 32 * j));
    const float d =
        __double2float_ru(fabs(__dsub_rn(v, __ldg(eta + base + 32 * t))));
    acc.delta = fmaxf(acc.delta, d);
    eta_next[base + 32 * t] = v;
  }
  static constexpr int kUnroll = 1;
  static constexpr bool kBlockMode = false;
  static constexpr bool kPureExpand = true;
  static constexpr int kMinBlocks = DP_SP_MINB;
  template <int U, class ArgsOf>
  __device__ __forceinline__ void items(ArgsOf args, const int* e,
                                        const bool* ok, Acc& acc) const {
    items_loop<U>(*this, args, e, ok, acc);
  }
  __device__ void flush(Acc& acc) const {
    float d = acc.delta;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d = fmaxf(d, __shfl_xor_sync(DP_FULL, d, o));
    if (lane_id() == 0 && d > 0.f &&
        __float_as_uint(d) > __ldcg(max_delta))
      atomicMax(max_delta, __float_as_uint(d));
  }
};

}  // namespace dp
