/*
 * dynpar.h — C-ABI of libdynpar.so, the B200 (sm_100a) nested-parallel hot path.
 *
 * The reference (arXiv 2201.02789 package `dynoptc`, pure Python) has no FFI:
 * its operator API for this path is `dynoptc.bench` (pkg/src/dynoptc/bench/
 * __init__.py:3-19) and every run goes through the simulator's Machine
 * (pkg/src/dynoptc/sim/machine.py:73-184).  Each entry point below replaces
 * one reference call site; the Python layer `paper_2201_02789_b200.bench`
 * keeps the reference's names and calls these through ctypes.
 *
 *   reference call                                     -> entry point
 *   run_config(bfs, wl, cfg)      harness.py:65-80     -> dp_bfs / dp_bfs_dev
 *     (BFS_CDP main+visit, benchmarks.py:91-120, drive :157-168)
 *   run_reference(bfs, wl)        harness.py:57-62     -> dp_bfs (variant=NOCDP)
 *     (BFS_NOCDP, benchmarks.py:122-141)
 *   run_config / run_reference for sssp                -> dp_sssp / dp_sssp_dev
 *     (benchmarks.py:175-270)
 *   run_config / run_reference for manylaunch          -> dp_manylaunch / _dev
 *     (benchmarks.py:277-332)
 *   (no reference; BASELINE.json configs 2 and 4)      -> dp_tc, dp_bt (+_dev)
 *   (no reference; paper Table I MSTF / MSTV / SP, and
 *    the north star's graph colouring)                 -> dp_mst, dp_sp, dp_gc
 *   (no reference; partitioned BFS / SSSP steps, bucketed
 *    or with the exchange fused over peer memory)      -> dp_*_part_*
 *   transform(... threshold, cfactor, agg, group_size, agg_threshold)
 *                                 pipeline.py:45-81    -> dp_config (policy knobs)
 *   SimReport counters            sim/report.py:12-28  -> dp_stats
 *   SimTrap(kind, ...)            sim/machine.py:43-50 -> negative return codes
 *
 * Conventions
 *  - Plain pointers and sizes only.  `*_dev` entry points take DEVICE pointers
 *    and a cudaStream_t passed as void* (NULL = legacy default stream); the
 *    others take caller-owned HOST arrays and copy H2D/D2H inside the call.
 *  - Every call is synchronous on return.  Calls are not re-entrant per
 *    device (the library keeps one workspace per device).
 *  - Return 0 on success, a negative DP_ERR_* code otherwise; the message is
 *    in dp_last_error() (thread-local).
 *  - Knob validation mirrors passes/aggregate.py:174-179 and is ALSO done in
 *    Python before the call (ValueError there, DP_ERR_INVALID here).
 */
#ifndef DYNPAR_H
#define DYNPAR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DP_ABI_VERSION 2

/* aggregation granularity (passes/aggregate.py:84 GRANULARITIES, + warp) */
#define DP_AGG_NONE 0
#define DP_AGG_WARP 1
#define DP_AGG_BLOCK 2
#define DP_AGG_MULTIBLOCK 3
#define DP_AGG_GRID 4

/* program variant (Benchmark.cdp_source / nocdp_source, benchmarks.py:56-68) */
#define DP_VARIANT_NOCDP 0
#define DP_VARIANT_CDP 1

/* how a below-threshold child grid runs inside the parent
 * (passes/threshold.py:60-83 runs it in the parent THREAD) */
#define DP_SERIAL_THREAD 0
#define DP_SERIAL_WARP 1 /* B200 addition: the parent warp shares the loop */

/* "always serialize" sentinel, passes/common.py:10 */
#define DP_INF_THRESHOLD 2147483647

/* error codes -> SimTrap kinds (sim/machine.py:43-50) */
#define DP_OK 0
#define DP_ERR_QUEUE_OVERFLOW (-1) /* "queue-overflow": pending launch pool full */
#define DP_ERR_LAUNCH_CONFIG (-2)  /* "launch-config" */
#define DP_ERR_CUDA (-3)           /* "cuda-error" */
#define DP_ERR_INVALID (-4)        /* bad knob / argument (ValueError in Python) */
#define DP_ERR_NO_DEVICE (-5)      /* no CUDA device visible */
#define DP_ERR_ITERATIONS (-6)     /* "more levels than vertices", benchmarks.py:168 */
#define DP_ERR_UNPUBLISHED (-7)    /* "unpublished-read" (publication-checker builds
                                      only: a child read an aggregation-table row
                                      its writer never published, sim/machine.py:571) */

typedef struct dp_config {
  int32_t threshold;     /* T: child count >= T launches, else serial; 0 = pass off */
  int32_t cfactor;       /* C: logical child blocks per physical block, >= 1 */
  int32_t agg;           /* DP_AGG_* */
  int32_t group_size;    /* multiblock: parent blocks per group, >= 1 */
  int32_t agg_threshold; /* block only: < this many participants -> direct launches */
  int32_t variant;       /* DP_VARIANT_* */
  int32_t parent_block;  /* parent threads per block (reference BLOCK = 32) */
  int32_t child_block;   /* child threads per block (reference launches use 32) */
  int32_t serial_mode;   /* DP_SERIAL_* */
  int32_t pending_launch_limit; /* cudaLimitDevRuntimePendingLaunchCount; 0 = auto */
  int32_t persistent;    /* > 0: persistent parent grid of this many blocks per
                            SM (single-group multiblock / grid aggregation):
                            all launches are recorded first, the serial arms
                            run while the aggregated child uses the rest of
                            the GPU.  0 = one parent thread per parent. */
  int32_t device_loop;   /* 1: BFS levels / SSSP rounds are chained on the
                            device (CDP2 tail launches, up to 16 per host
                            launch) instead of one host launch + flag
                            readback each */
  int32_t frontier;      /* SSSP only, 1: a reached vertex relaxes its edges
                            only when its distance changed since it last did
                            (work-efficient rounds; same final distances,
                            fewer relaxations).  0 = every reached vertex
                            every round, as SSSP_CDP main does
                            (benchmarks.py:207-222) */
  int32_t agg_coarsen;   /* 1: the coarsening factor applies to the aggregated
                            child grid (logical aggregated blocks
                            [b*C, b*C + C) per physical block, possibly of
                            several parents): the reference's pass order with
                            A before C (pipeline.py:60-81).  Requires
                            agg in {warp, block, multiblock}.  0 = canonical
                            T -> C -> A (per-parent coarsening) */
  int32_t counts_spread;  /* partitioned BFS (dp_bfs_part_level*): b > 0 ->
                            d_counts holds n rounded up to a multiple of 2^b
                            slots and vertex v counts at slot spread_b(v)
                            (a bijective hash of v's low b bits that keeps
                            RMAT hubs out of shared 128 B lines); gather with
                            dp_unspread_dev.  0 = vertex order.  dp_bfs /
                            dp_bfs_dev use the spread layout internally and
                            always return vertex order */
  int32_t weight_bits;   /* SSSP: 4 -> the edge weights are read as packed
                            nibbles (w - 1, 8 per 32-bit word; 1/8 of the
                            int32 bytes) when every weight lies in [1, 16];
                            dp_sssp packs on the host chunk by chunk ahead
                            of the copy (out-of-range chunks and all later
                            ones stay int32), dp_sssp_dev packs on the
                            device.  0 = int32 weights as given */
  int32_t cf_wave;       /* B200: a row whose logical child grid has >=
                            cf_wave blocks runs uncoarsened (coarsening
                            amortises setup over many small children; one
                            huge child would only be serialised).  0 = every
                            row coarsened by cfactor (the reference) */
  int32_t col_bits;      /* dp_sssp (host buffers): 24 -> each chunk of col
                            crosses PCIe as 3-byte values (3/4 of the int32
                            bytes), packed on the host ahead of the copy and
                            expanded into the int32 col on the device before
                            the chunk is published; a chunk holding a value
                            outside [0, 2^24) travels as int32.  The rounds
                            read int32 col either way.  0 = int32 */
} dp_config;

/* SimReport (sim/report.py:12-28) counters, measured on the device */
typedef struct dp_stats {
  uint64_t num_launches;      /* device-side launches with grid, block > 0 */
  uint64_t host_launches;     /* host-side launches with grid, block > 0 */
  uint64_t blocks_scheduled;  /* sum of grid sizes over every launched grid */
  uint64_t max_pending_depth; /* deepest device launch queue (issued, not started) */
  uint64_t iterations;        /* host-loop trips (BFS levels / SSSP rounds) */
  uint64_t work_units;        /* child items executed (edges examined, ...) */
  uint64_t bytes_alg;         /* algorithmic HBM bytes (DESIGN.md per app) */
  double ns_device;           /* CUDA-event time of the whole run (device) */
  double ns_host;             /* host wall time of the call, copies included */
  double ns_kernel_max;       /* longest host-launched step (parent grid + its
                                 children [+ grid-glue launch]), CUDA events */
  double ns_kernel_sum;       /* sum of those step durations (no host gaps) */
  double ns_phase[5];         /* parent, launch, agg, disagg, child (0 unless profiled) */
  uint64_t h2d_bytes;         /* bytes copied host->device in this call */
  uint64_t d2h_bytes;         /* bytes copied device->host in this call */
  uint64_t kernel_launches;   /* launches of library kernels issued from the host */
  double launch_lat_ns_mean;  /* device launch -> first child block start
                                 (%globaltimer), mean over device launches */
  uint64_t remote_ops;        /* partitioned runs with the fused exchange:
                                 atomics issued into other parts' dist */
  uint64_t unpublished_reads; /* publication-checker builds: child reads of
                                 aggregation rows never published (0 otherwise) */
  uint64_t poisoned_reads;    /* publication-checker builds: child reads of rows
                                 still holding the pre-launch poison bytes */
} dp_stats;

/* ---- library -------------------------------------------------------------- */
int dp_abi_version(void);
const char* dp_last_error(void);
int dp_device_count(void);
/* Select `device` (sm_100) for every later call from any host thread (one
 * device per process: the library's CUDA runtime is linked statically, so
 * its current device is independent of the caller's).  0 on success. */
int dp_init(int32_t device);

/* ---- BFS (benchmarks.py:91-168) ------------------------------------------ */
/* host buffers: rowptr[n+1], col[m]; out dist[n], counts[n] */
int dp_bfs(const int32_t* rowptr, const int32_t* col, int32_t n, int64_t m,
           int32_t src, const dp_config* cfg, int32_t* dist, int32_t* counts,
           dp_stats* stats);
/* device buffers; dist/counts are initialised by the call */
int dp_bfs_dev(const int32_t* d_rowptr, const int32_t* d_col, int32_t n,
               int64_t m, int32_t src, const dp_config* cfg, int32_t* d_dist,
               int32_t* d_counts, void* stream, dp_stats* stats);

/* ---- SSSP (benchmarks.py:175-270) ---------------------------------------- */
/* host buffers: rowptr[n+1], col[m], weight[m]; out dist[n].  col / weight
 * stream in behind the rounds (chunked copy; weight_bits / col_bits pick the
 * transfer codecs).  Once every chunk has landed the call copies dist back
 * while the next round runs and returns as soon as a round lowers nothing:
 * `dist` may be written more than once during the call (its final contents
 * are the result) and stats->d2h_bytes counts every copy. */
int dp_sssp(const int32_t* rowptr, const int32_t* col, const int32_t* weight,
            int32_t n, int64_t m, int32_t src, const dp_config* cfg,
            int32_t* dist, dp_stats* stats);
int dp_sssp_dev(const int32_t* d_rowptr, const int32_t* d_col,
                const int32_t* d_weight, int32_t n, int64_t m, int32_t src,
                const dp_config* cfg, int32_t* d_dist, void* stream,
                dp_stats* stats);

/* ---- manylaunch (benchmarks.py:277-332) ---------------------------------- */
int dp_manylaunch(const int32_t* sizes, int32_t n, const dp_config* cfg,
                  int32_t* out, int32_t* total, dp_stats* stats);
int dp_manylaunch_dev(const int32_t* d_sizes, int32_t n, const dp_config* cfg,
                      int32_t* d_out, int32_t* d_total, void* stream,
                      dp_stats* stats);

/* ---- triangle counting (no reference) -------------- */
/* rank-ordered CSR+ (dp_tc_orient: every edge u -> v has u < v, rows sorted
 * ascending; the kernels probe only the part of N+(u) above v).
 * [edge_lo, edge_hi) restricts the count to a range of oriented edges
 * (the multi-GPU shard); pass 0, m for the whole graph. */
int dp_tc(const int32_t* rowptr, const int32_t* col, int32_t n, int64_t m,
          int64_t edge_lo, int64_t edge_hi, const dp_config* cfg,
          uint64_t* triangles, dp_stats* stats);
int dp_tc_dev(const int32_t* d_rowptr, const int32_t* d_col, int32_t n,
              int64_t m, int64_t edge_lo, int64_t edge_hi,
              const dp_config* cfg, uint64_t* d_triangles, void* stream,
              dp_stats* stats);

/* ---- graph colouring (north-star app, no reference) -------- */
/* Jones-Plassmann with priority key(v) = (hash32(v), v) over a symmetric
 * simple CSR (dp_symmetrize): color[n] equals the sequential greedy colouring
 * in decreasing priority order.  stats->iterations = rounds. */
int dp_gc(const int32_t* rowptr, const int32_t* col, int32_t n, int64_t m,
          const dp_config* cfg, int32_t* color, dp_stats* stats);
int dp_gc_dev(const int32_t* d_rowptr, const int32_t* d_col, int32_t n,
              int64_t m, const dp_config* cfg, int32_t* d_color, void* stream,
              dp_stats* stats);

/* ---- minimum spanning forest: MSTF / MSTV (no reference) */
/* Boruvka rounds over a symmetric simple CSR (dp_symmetrize) with symmetric
 * weights and eid[e] = the canonical slot of slot e's undirected edge
 * (min(e, mirror[e]), dp_edge_mirror).  Edges are ordered by (weight, eid),
 * so the forest is unique (= Kruskal in that order).  cfg_find drives the
 * nested find kernel (MSTF), cfg_verify the nested verify kernel (MSTV;
 * NULL = cfg_find).  Out: in_mst[m] = 1 at the canonical slot of every forest
 * edge, *total_weight, *nedges.  stats->iterations = find rounds. */
int dp_mst(const int32_t* rowptr, const int32_t* col, const int32_t* weight,
           const int32_t* eid, int32_t n, int64_t m, const dp_config* cfg_find,
           const dp_config* cfg_verify, uint8_t* in_mst, int64_t* total_weight,
           int64_t* nedges, dp_stats* stats);
int dp_mst_dev(const int32_t* d_rowptr, const int32_t* d_col,
               const int32_t* d_weight, const int32_t* d_eid, int32_t n,
               int64_t m, const dp_config* cfg_find,
               const dp_config* cfg_verify, uint8_t* d_in_mst,
               int64_t* total_weight, int64_t* nedges, void* stream,
               dp_stats* stats);

/* ---- survey propagation on random k-SAT (no reference) ----- */
/* Clause a owns edges [a*k, (a+1)*k): lits[e] = var << 1 | negated.
 * occ_row[nvars+1] / occ[nclauses*k]: each variable's edges (variable-major
 * CSR).  eta0[nclauses*k]: initial surveys.  Synchronous sweeps (nested
 * variable->occurrence product kernel, nested clause->literal survey kernel)
 * until max |eta' - eta| <= eps or max_sweeps.  Out: eta (final surveys),
 * wpos/wneg[nvars] variable biases W+ / W-, *sweeps, *delta (last max
 * change).  fp64 arithmetic and surveys, fp32 biases; the per-variable
 * product order is schedule-dependent, so results equal the CPU oracle
 * within a tolerance.  Inside the call lit / eta live clause-tiled (32
 * clauses per tile, literal-major within it); eta comes in and goes out
 * clause-major as above.  Occurrence lists sorted by edge (as the
 * reference-style generator builds them) also allow the L2-windowed
 * variable pass (DYNPAR_SP_WINDOW_MB); unsorted lists run one pass. */
int dp_sp(const int32_t* lits, int32_t k, int32_t nclauses,
          const int32_t* occ_row, const int32_t* occ, int32_t nvars,
          const double* eta0, int32_t max_sweeps, float eps,
          const dp_config* cfg, double* eta, float* wpos, float* wneg,
          int32_t* sweeps, float* delta, dp_stats* stats);
/* device buffers; d_eta holds eta0 on entry and the final surveys on return */
int dp_sp_dev(const int32_t* d_lits, int32_t k, int32_t nclauses,
              const int32_t* d_occ_row, const int32_t* d_occ, int32_t nvars,
              int32_t max_sweeps, float eps, const dp_config* cfg,
              double* d_eta, float* d_wpos, float* d_wneg, int32_t* sweeps,
              float* delta, void* stream, dp_stats* stats);

/* ---- BFS over a cyclic 1D vertex partition ------- */
/* One level on part `part` of `nparts` (owner(v) = v % nparts; local index
 * v / nparts).  d_rowptr_p/d_col_p: the part's rows (dp_rmat_csr_part),
 * d_dist_p[n_local]: owned levels, d_counts[n]: dense per-part edge counts,
 * d_sent: bitmap over global ids (zeroed once per BFS), d_send_buf:
 * [nparts][send_stride] remote discoveries bucketed by owner with
 * d_send_counts[nparts] (zero before each level), d_changed: set when a
 * local vertex was discovered.  The caller exchanges the buckets (all-to-all)
 * and applies what it receives with dp_bfs_part_apply. */
int dp_bfs_part_level(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                      int32_t n_local, int32_t nparts, int32_t part,
                      int32_t level, const dp_config* cfg, int32_t* d_dist_p,
                      int32_t* d_counts, uint32_t* d_sent, int32_t* d_send_buf,
                      int64_t send_stride, int32_t* d_send_counts,
                      int32_t* d_changed, void* stream, dp_stats* stats);
/* The same level with the exchange fused into the expansion: d_peer_dist is
 * a DEVICE array of nparts pointers to every part's dist (symmetric memory
 * across GPUs, plain pointers when all parts share one GPU; entry `part` ==
 * d_dist_p); a remote discovery (first per part, d_sent) is a CAS of the
 * owner's dist from UNREACHED to level + 1.  No buckets, no apply pass. */
int dp_bfs_part_level_peer(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                           int32_t n_local, int32_t nparts, int32_t part,
                           int32_t level, const dp_config* cfg,
                           int32_t* d_dist_p, int32_t* const* d_peer_dist,
                           int32_t* d_counts, uint32_t* d_sent,
                           int32_t* d_changed, void* stream, dp_stats* stats);
/* Whole partitioned BFS of one part, levels looped in the library (see
 * dp_sssp_part_solve_peer for d_peer_sig / epoch / concurrency): initialises
 * dist, d_counts (counts_len >= n_global, rounded up to the spread block when
 * cfg->counts_spread > 0) and the sent bitmap ((n_global + 31) / 32 words),
 * then levels until no part discovers a vertex.  stats: iterations = levels
 * (as bfs_1d_peer), remote_ops = CAS issued into other parts' dist. */
int dp_bfs_part_solve_peer(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                           int32_t n_local, int32_t n_global, int32_t nparts,
                           int32_t part, int32_t src, const dp_config* cfg,
                           int32_t* d_dist_p, int32_t* const* d_peer_dist,
                           int32_t* d_counts, int64_t counts_len,
                           uint32_t* d_sent, uint64_t* const* d_peer_sig,
                           uint64_t epoch, void* stream, dp_stats* stats);
/* free the calling host thread's workspace (tables, pinned buffers); the
 * next call on the thread re-creates it */
void dp_thread_release(void);
/* diagnostics: device time (ms, CUDA events) of every host-launched step
 * (parent grid + its children [+ grid glue]) of the calling thread's last
 * run, in order -- one per BFS level / SSSP round; copies min(count, cap)
 * into ms and returns the count */
int64_t dp_step_times(double* ms, int64_t cap);
/* out[v] = work[spread_b(v)] for v < n: counts accumulated with
 * counts_spread = b back in vertex order */
int dp_unspread_dev(const int32_t* d_work, int32_t b, int32_t n,
                    int32_t* d_out, void* stream);
/* discover received global ids at level + 1 (CAS against UNREACHED) */
int dp_bfs_part_apply(const int32_t* d_recv, int64_t nrecv, int32_t nparts,
                      int32_t level, int32_t* d_dist_p, int32_t* d_changed,
                      void* stream);

/* ---- SSSP over the cyclic 1D vertex partition --------------------------- */
/* One Bellman-Ford round on part `part`: owned dist[n_local] lowered in
 * place; a remote relaxation (v, alt) is appended to owner(v)'s bucket as
 * (uint64)v << 32 | alt when it strictly lowers d_best[v] (dense, global ids,
 * UNREACHED-initialised once per SSSP).  Bucket q starts at d_send_off[q]
 * and must hold the part's edges into owner q; d_send_counts[nparts] and
 * d_changed are zeroed by the caller before each round. */
int dp_sssp_part_round(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                       const int32_t* d_weight_p, int32_t n_local,
                       int32_t nparts, int32_t part, const dp_config* cfg,
                       int32_t* d_dist_p, int32_t* d_best, uint64_t* d_send_buf,
                       const int64_t* d_send_off, int32_t* d_send_counts,
                       int32_t* d_changed, void* stream, dp_stats* stats);
/* The same round with the exchange fused into the relaxation: d_peer_dist is
 * a DEVICE array of nparts pointers to every part's dist[n_local_q] (peer-
 * mapped symmetric memory across GPUs, or plain pointers when all parts
 * share one GPU; entry `part` == d_dist_p); a remote relaxation that lowers
 * d_best[v] is an atomicMin straight into its owner's dist.  No buckets, no apply pass: the caller
 * only reduces d_changed (max) across parts between rounds. */
int dp_sssp_part_round_peer(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                            const int32_t* d_weight_p, int32_t n_local,
                            int32_t nparts, int32_t part,
                            const dp_config* cfg, int32_t* d_dist_p,
                            int32_t* const* d_peer_dist, int32_t* d_best,
                            int32_t* d_changed, void* stream,
                            dp_stats* stats);
/* Whole partitioned SSSP of one part (all rounds, loop in the library):
 * initialises its dist (src is a global id) and best, then per round runs
 * the fused-exchange step of dp_sssp_part_round_peer and ORs every part's
 * round flag through the parts' signal slots -- no host collective.
 * d_peer_sig: DEVICE array of nparts pointers, entry q = part q's uint64
 * slots[2 * nparts] (zero-filled once; symmetric memory across GPUs, plain
 * device memory when the parts share a GPU).  epoch: equal on every part,
 * unique per call on a slot set, in [1, 2^31).  Parts must run
 * concurrently (one per process, or one per host thread with its own
 * stream); a part that waits longer than $DYNPAR_PEER_TIMEOUT_MS (default
 * 60000) for a peer fails with DP_ERR_CUDA.  stats: iterations = rounds,
 * remote_ops = atomics issued into other parts' dist. */
int dp_sssp_part_solve_peer(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                            const int32_t* d_weight_p, int32_t n_local,
                            int32_t n_global, int32_t nparts, int32_t part,
                            int32_t src, const dp_config* cfg,
                            int32_t* d_dist_p, int32_t* const* d_peer_dist,
                            int32_t* d_best, uint64_t* const* d_peer_sig,
                            uint64_t epoch, void* stream, dp_stats* stats);
/* lower owned dist by received (v << 32 | alt) pairs (atomicMin) */
int dp_sssp_part_apply(const uint64_t* d_recv, int64_t nrecv, int32_t nparts,
                       int32_t* d_dist_p, int32_t* d_changed, void* stream);

/* ---- Bezier line tessellation (no reference) ------- */
/* cp[ncurves][3][2] float32 control points.  Outputs: ntess[ncurves] vertex
 * counts, offsets[ncurves] start of each curve's vertices in verts, and
 * verts[2*vert_capacity] float32 (x,y).  Offsets come from a device bump
 * allocator (the device-side cudaMalloc of the original), so
 * they depend on scheduling; the per-curve vertices do not.
 * Returns DP_ERR_INVALID if the vertices do not fit vert_capacity. */
int dp_bt(const float* cp, int32_t ncurves, int32_t max_tess, float curv_scale,
          const dp_config* cfg, int32_t* ntess, int64_t* offsets, float* verts,
          int64_t vert_capacity, int64_t* nverts, dp_stats* stats);
int dp_bt_dev(const float* d_cp, int32_t ncurves, int32_t max_tess,
              float curv_scale, const dp_config* cfg, int32_t* d_ntess,
              int64_t* d_offsets, float* d_verts, int64_t vert_capacity,
              int64_t* nverts, void* stream, dp_stats* stats);

/* ---- host-side input generation (builder-defined, no reference) ----------- */
/* RMAT (Graph500 a,b,c = .57,.19,.19), n = 2^scale, m = edge_factor*n edges,
 * multi-edges and self-loops kept, CSR rows sorted ascending.  Deterministic
 * for (scale, edge_factor, seed) on any host.  rowptr[n+1], col[m]. */
int dp_rmat_csr(int32_t scale, int32_t edge_factor, uint64_t seed,
                int32_t* rowptr, int32_t* col, int32_t nthreads);
/* The rows of the same RMAT graph owned by `part` under the cyclic 1D
 * partition owner(v) = v % nparts: rowptr_p[n_p+1] over local vertices
 * lv = v / nparts, col_p (global ids).  Call with col_p == NULL to size
 * (*m_p), then again with col_capacity >= *m_p. */
int dp_rmat_csr_part(int32_t scale, int32_t edge_factor, uint64_t seed,
                     int32_t nparts, int32_t part, int32_t* rowptr_p,
                     int32_t* col_p, int64_t col_capacity, int64_t* m_p,
                     int32_t nthreads);
/* Device-side generation of the same graph: writes one key
 * (v / nparts) << 32 | dst per edge whose source v is owned by `part`, in
 * arbitrary order (sort them to get the CSR rows of dp_rmat_csr_part).
 * d_keys == NULL or capacity == 0 only counts (*count). */
int dp_rmat_part_keys_dev(int32_t scale, int32_t edge_factor, uint64_t seed,
                          int32_t nparts, int32_t part, uint64_t* d_keys,
                          int64_t capacity, int64_t* count, void* stream);
/* symmetrise, drop self-loops and duplicates, relabel the vertices by
 * ascending (degree, id) rank and keep u -> v iff rank u < rank v: the
 * rank-ordered CSR+ dp_tc expects (rows ascending, every edge u -> v has
 * u < v; same triangle count as the input).
 * Allocates *rowptr_plus (n+1) and *col_plus (*m_plus); free with dp_free. */
int dp_tc_orient(const int32_t* rowptr, const int32_t* col, int32_t n,
                 int32_t** rowptr_plus, int32_t** col_plus, int64_t* m_plus,
                 int32_t nthreads);
/* symmetrise, drop self-loops and duplicates (both directions kept). */
int dp_symmetrize(const int32_t* rowptr, const int32_t* col, int32_t n,
                  int32_t** rowptr_s, int32_t** col_s, int64_t* m_s,
                  int32_t nthreads);
/* symmetric CSR, sorted rows, no duplicates: mirror[e] = slot of the reverse
 * edge.  DP_ERR_INVALID if a reverse edge is missing. */
int dp_edge_mirror(const int32_t* rowptr, const int32_t* col, int32_t n,
                   int32_t* mirror, int32_t nthreads);
void dp_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* DYNPAR_H */
