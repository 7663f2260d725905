// dynpar.cu — host drivers and the C-ABI of libdynpar.so (include/dynpar.h).
//
// The host loop of each application mirrors the reference's `drive`
// functions (bench/benchmarks.py:157-168, 259-270, 328-332): one host launch
// of the parent grid per level/round, then a readback of the `changed` flag.
// What the reference's GlueRunner does around a launch (pipeline.py:99-110:
// arm tables, grid-granularity completion hook) is done here: tables re-arm
// on the device, and grid granularity reads the fused counter back and
// host-launches the aggregated child (passes/common.py:144-164).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dynpar.h"
#include "apps.cuh"
#include "sched.cuh"

using namespace dp;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define DP_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      return fail(DP_ERR_CUDA, std::string("cuda-error: ") + #call + ": " +  \
                                   cudaGetErrorString(e_));                  \
  } while (0)

constexpr int kMaxChunks = 32;

// Per-device workspace: aggregation tables, counters, pinned readback, I/O
// staging for the host-buffer entry points.  Grow-only.
struct Workspace {
  bool ready = false;
  void* tab = nullptr;  // Args rows
  size_t tab_bytes = 0;
  int* scan = nullptr;
  size_t scan_rows = 0;
  unsigned long long* ctr = nullptr;  // per group
  int* done = nullptr;
  size_t groups = 0;
  DevState* ds = nullptr;
  DevState* h_ds = nullptr;            // pinned
  unsigned long long* h_ctr = nullptr;  // pinned
  unsigned long long* d_scratch = nullptr;  // TC total / BT cursor
  int* d_flag = nullptr;                    // BT overflow
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evk0 = nullptr, evk1 = nullptr;
  // mapped (zero-copy) readback of DevState for the per-level host loop
  struct Signal {
    DevState ds;
    unsigned seq;
    unsigned pad;
    unsigned long long aux;  // d_scratch[1]: the lazy launcher count
  };
  Signal* h_sig = nullptr;  // host view (mapped pinned)
  Signal* d_sig = nullptr;  // device view of the same memory
  unsigned seq = 0;
  // staging for host-buffer calls
  void* io[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t io_bytes[6] = {0, 0, 0, 0, 0, 0};
  // copy/compute overlap of host-buffer calls: a copy stream, the device
  // counter of chunks that have landed, one event per chunk
  cudaStream_t copy_stream = nullptr;
  int* d_arrived = nullptr;
  cudaEvent_t chunk_ev[kMaxChunks] = {};
  cudaEvent_t ev_spec = nullptr;  // speculative result readback
  // BFS counts in the spread layout (2^k slots)
  void* cwork = nullptr;
  size_t cwork_bytes = 0;
  // publication-checker builds: one stamp per aggregation-table row
  void* pub = nullptr;
  size_t pub_bytes = 0;
  // BFS launch bits (bit v: v's row reaches the threshold)
  void* lbits = nullptr;
  size_t lbits_bytes = 0;
  // packed SSSP weights: device copy and the pinned host staging of dp_sssp
  void* wpack = nullptr;
  size_t wpack_bytes = 0;
  void* h_wpack = nullptr;
  size_t h_wpack_bytes = 0;
  int* d_bad = nullptr;
  // dp_config.col_bits = 24: 3-byte col values in flight (pinned host
  // staging, device landing buffer unpacked into the int32 col)
  void* cpack = nullptr;
  size_t cpack_bytes = 0;
  void* h_cpack = nullptr;
  size_t h_cpack_bytes = 0;
};

// One workspace per (host thread, device): the partitioned solve drivers
// run one part per host thread when several parts share a process
// (dp_*_part_solve_peer), each with its own stream, tables and DevState.
// dp_thread_release frees the calling thread's.
thread_local Workspace g_ws[64];

// The CDP2 pending-launch pool is a device-wide limit: one size per device
// for every thread, changed under a lock (growing it synchronises the device).
std::mutex g_pending_mu;
long long g_pending_limit[64] = {};

// The device chosen by dp_init.  libdynpar links the CUDA runtime statically,
// so its current device is independent of the caller's runtime (e.g.
// PyTorch's) and per host thread: every entry point re-selects it.
int g_device = -1;

int current_device(int* dev) {
  if (g_device >= 0) {
    cudaError_t e = cudaSetDevice(g_device);
    if (e != cudaSuccess)
      return fail(DP_ERR_NO_DEVICE, std::string("cudaSetDevice: ") +
                                        cudaGetErrorString(e));
  }
  cudaError_t e = cudaGetDevice(dev);
  if (e != cudaSuccess)
    return fail(DP_ERR_NO_DEVICE, std::string("no CUDA device: ") +
                                      cudaGetErrorString(e));
  return 0;
}

Workspace* workspace(int* rc) {
  int dev = 0;
  *rc = current_device(&dev);
  if (*rc) return nullptr;
  Workspace& w = g_ws[dev & 63];
  if (!w.ready) {
    cudaError_t e;
    if ((e = cudaMalloc(&w.ds, sizeof(DevState))) != cudaSuccess ||
        (e = cudaMallocHost(&w.h_ds, sizeof(DevState))) != cudaSuccess ||
        (e = cudaMallocHost(&w.h_ctr, 2 * sizeof(unsigned long long))) !=
            cudaSuccess ||
        (e = cudaMalloc(&w.d_scratch, 2 * sizeof(unsigned long long))) !=
            cudaSuccess ||
        (e = cudaMalloc(&w.d_flag, sizeof(int))) != cudaSuccess ||
        (e = cudaEventCreate(&w.ev0)) != cudaSuccess ||
        (e = cudaEventCreate(&w.ev1)) != cudaSuccess ||
        (e = cudaEventCreate(&w.evk0)) != cudaSuccess ||
        (e = cudaEventCreate(&w.evk1)) != cudaSuccess ||
        (e = cudaHostAlloc(&w.h_sig, sizeof(Workspace::Signal),
                           cudaHostAllocMapped)) != cudaSuccess ||
        (e = cudaHostGetDevicePointer(&w.d_sig, w.h_sig, 0)) != cudaSuccess) {
      *rc = fail(DP_ERR_CUDA,
                 std::string("workspace init: ") + cudaGetErrorString(e));
      return nullptr;
    }
    std::memset((void*)w.h_sig, 0, sizeof(Workspace::Signal));
    w.ready = true;
  }
  return &w;
}

int grow(void** p, size_t* have, size_t need) {
  if (need <= *have) return 0;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  size_t n = std::max(need, (size_t)256);
  cudaError_t e = cudaMalloc(p, n);
  if (e != cudaSuccess)
    return fail(DP_ERR_CUDA, std::string("workspace alloc of ") +
                                 std::to_string(n) + " bytes: " +
                                 cudaGetErrorString(e));
  *have = n;
  return 0;
}

int validate(const dp_config* c) {
  if (!c) return fail(DP_ERR_INVALID, "null config");
  if (c->variant != DP_VARIANT_NOCDP && c->variant != DP_VARIANT_CDP)
    return fail(DP_ERR_INVALID, "unknown variant");
  if (c->agg < DP_AGG_NONE || c->agg > DP_AGG_GRID)
    return fail(DP_ERR_INVALID, "unknown aggregation granularity");
  if (c->agg_threshold > 0 && c->agg != DP_AGG_BLOCK)
    return fail(DP_ERR_INVALID,
                "aggregation threshold requires block granularity");
  if (c->agg == DP_AGG_MULTIBLOCK && c->group_size < 1)
    return fail(DP_ERR_INVALID, "group size must be at least 1");
  if (c->cfactor < 1) return fail(DP_ERR_INVALID, "cfactor must be >= 1");
  if (c->persistent < 0 || c->persistent > 8)
    return fail(DP_ERR_INVALID, "persistent must be in [0, 8]");
  if (c->threshold < 0) return fail(DP_ERR_INVALID, "threshold must be >= 0");
  if (c->counts_spread < 0 || c->counts_spread > 30)
    return fail(DP_ERR_INVALID, "counts_spread must be in [0, 30]");
  if (c->weight_bits != 0 && c->weight_bits != 4)
    return fail(DP_ERR_INVALID, "weight_bits must be 0 or 4");
  if (c->cf_wave < 0) return fail(DP_ERR_INVALID, "cf_wave must be >= 0");
  if (c->col_bits != 0 && c->col_bits != 24)
    return fail(DP_ERR_INVALID, "col_bits must be 0 or 24");
  if (c->cf_wave > 0 && c->agg_coarsen)
    return fail(DP_ERR_INVALID,
                "cf_wave applies to per-row coarsening (canonical order)");
  if (c->agg_coarsen &&
      (c->agg < DP_AGG_WARP || c->agg > DP_AGG_MULTIBLOCK || c->persistent))
    return fail(DP_ERR_INVALID,
                "agg_coarsen requires warp, block or multiblock aggregation "
                "and a non-persistent parent");
  if (c->parent_block < 32 || c->parent_block > 256 ||
      c->parent_block % 32)
    return fail(DP_ERR_INVALID,
                "parent_block must be a multiple of 32 in [32, 256]");
  if (c->child_block < 32 || c->child_block > 256 || c->child_block % 32)
    return fail(DP_ERR_INVALID,
                "child_block must be a multiple of 32 in [32, 256]");
  return 0;
}

int map_device_error(int e) {
  if (e == 0x7fff0001)  // kErrPeerTimeout
    return fail(DP_ERR_CUDA,
                "cuda-error: partitioned exchange timed out waiting for a "
                "peer part ($DYNPAR_PEER_TIMEOUT_MS)");
  if (e == (int)cudaErrorLaunchPendingCountExceeded)
    return fail(DP_ERR_QUEUE_OVERFLOW,
                "queue-overflow: pending launch count exceeded the device "
                "runtime pool (raise pending_launch_limit)");
  if (e == (int)cudaErrorInvalidConfiguration)
    return fail(DP_ERR_LAUNCH_CONFIG, "launch-config: invalid device launch");
  return fail(DP_ERR_CUDA, std::string("cuda-error in device launch: ") +
                               cudaGetErrorString((cudaError_t)e));
}

// ---------------------------------------------------------------------------
// CDP2 pending-launch pool.  Measured on B200 (profiles/cdp_probe_r01.txt):
// a device launch beyond cudaLimitDevRuntimePendingLaunchCount does NOT fail,
// it stalls the grid indefinitely, and each slot costs ~11 KB of HBM.  So the
// pool is sized from an exact upper bound on the device launches one host
// launch can issue under the chosen policy, and a run whose bound does not
// fit the memory budget is refused up front with "queue-overflow" — the
// reference traps the same way when its bounded FIFO overflows
// (sim/machine.py:237-241; PAPER.md:417 raised this limit on the V100).
// ---------------------------------------------------------------------------

// parents whose child count can reach `thr`: CSR degree >= thr
__global__ void count_deg_ge_kernel(const int* __restrict__ rowptr, int n,
                                    int thr, unsigned long long* out) {
  unsigned long long c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    c += (__ldg(rowptr + i + 1) - __ldg(rowptr + i)) >= thr;
  c = warp_sum_u64(c);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

__global__ void count_val_ge_kernel(const int* __restrict__ v, int n, int thr,
                                    unsigned long long* out) {
  unsigned long long c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    c += __ldg(v + i) >= thr;
  c = warp_sum_u64(c);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

int effective_threshold(const dp_config* c) {
  return c->threshold > 1 ? c->threshold : 1;
}

long long launch_bound(const dp_config* c, long long parents,
                       long long launchers);
long long launch_bound_agg(const dp_config* c, long long launchers,
                           long long warps, long long blocks);

// kind 0: CSR rowptr degrees, 1: per-parent values.  Skipped (returns the
// parent count) when the policy's structural bound -- warps, blocks or
// groups -- already keeps the pool small, so aggregated runs pay no extra
// kernel + sync for pool sizing.
int count_launchers(Workspace* w, const dp_config* c, const int* data, int n,
                    int kind, cudaStream_t s, long long* out) {
  if (launch_bound(c, n, n) <= (1 << 16)) {
    *out = n;
    return 0;
  }
  const int thr = effective_threshold(c);
  DP_CUDA(cudaMemsetAsync(w->d_scratch + 1, 0, sizeof(unsigned long long), s));
  if (n > 0) {
    const int blocks = std::min(dp::ceil_div(n, 256), 148 * 8);
    if (kind == 0)
      count_deg_ge_kernel<<<blocks, 256, 0, s>>>(data, n, thr,
                                                 w->d_scratch + 1);
    else
      count_val_ge_kernel<<<blocks, 256, 0, s>>>(data, n, thr,
                                                 w->d_scratch + 1);
    DP_CUDA(cudaGetLastError());
  }
  DP_CUDA(cudaMemcpyAsync(w->h_ctr + 1, w->d_scratch + 1,
                          sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          s));
  DP_CUDA(cudaStreamSynchronize(s));
  *out = (long long)w->h_ctr[1];
  return 0;
}

// count_launchers without the host round trip (BFS / SSSP level loops).
// When a bound computed from m alone keeps the pool small, the count kernel
// is queued into d_scratch[1] and its value rides on the first round's
// readback (signal_kernel aux); *lazy_bound >= 0 then holds that pool bound
// and *out an upper bound on the launchers.  Otherwise as count_launchers
// (*lazy_bound = -1).  The stream synchronisation this saves left the GPU
// idle between the count and the first parent grid of every call.
int count_launchers_lazy(Workspace* w, const dp_config* c, const int* rowptr,
                         int n, int64_t m, cudaStream_t s, long long* out,
                         long long* lazy_bound) {
  *lazy_bound = -1;
  const long long thr = c->threshold;  // 0: every non-empty row launches
  if (c->variant == DP_VARIANT_CDP && m >= 0 &&
      launch_bound(c, n, n) > (1 << 16) && !std::getenv("DYNPAR_SYNC_COUNT")) {
    // a launcher has >= max(T, 1) items
    const long long L = std::min<long long>(n, m / std::max<long long>(thr, 1));
    if (L == 0) {  // no row can reach the threshold: exact, nothing to count
      *out = 0;
      return 0;
    }
    // a row launched on its own under cf_wave has >= (cf_wave - 1) * cb + 1
    long long solo = 0;
    if (c->cf_wave > 0 && c->agg != DP_AGG_NONE)
      solo = std::min<long long>(
          L, m / ((long long)(c->cf_wave - 1) * c->child_block + 1));
    const long long bound =
        solo + launch_bound_agg(c, L, dp::ceil_div_ll(n, 32),
                                dp::ceil_div_ll(n, c->parent_block));
    if (bound <= (1 << 14)) {
      DP_CUDA(cudaMemsetAsync(w->d_scratch + 1, 0, sizeof(unsigned long long),
                              s));
      if (n > 0) {
        count_deg_ge_kernel<<<std::min(dp::ceil_div(n, 256), 148 * 8), 256, 0,
                              s>>>(rowptr, n, effective_threshold(c),
                                   w->d_scratch + 1);
        DP_CUDA(cudaGetLastError());
      }
      *out = L;
      *lazy_bound = bound;
      return 0;
    }
  }
  return count_launchers(w, c, rowptr, n, 0, s, out);
}

// Upper bound on device launches issued by ONE host launch of the parent
// grid, given `launchers` parents that may meet the threshold.
long long launch_bound(const dp_config* c, long long parents,
                       long long launchers) {
  if (c->variant != DP_VARIANT_CDP) return 0;
  const long long warps = dp::ceil_div_ll(parents, 32);
  const long long blocks = dp::ceil_div_ll(parents, c->parent_block);
  // cf_wave: every launching row may be big enough for a launch of its own
  const long long solo =
      c->cf_wave > 0 && c->agg != DP_AGG_NONE ? launchers : 0;
  return solo + launch_bound_agg(c, launchers, warps, blocks);
}

long long launch_bound_agg(const dp_config* c, long long launchers,
                           long long warps, long long blocks) {
  switch (c->agg) {
    case DP_AGG_NONE: return launchers;
    case DP_AGG_WARP: return std::min(launchers, warps);
    case DP_AGG_BLOCK:
      if (c->agg_threshold > 0)  // direct launches below agg_threshold
        return std::min(launchers, blocks * (long long)c->agg_threshold);
      return std::min(launchers, blocks);
    case DP_AGG_MULTIBLOCK:
      return std::min(launchers, dp::ceil_div_ll(blocks, c->group_size));
    default: return 0;  // grid: the aggregated launch is a host launch
  }
}

constexpr long long kSlotBytes = 12 * 1024;  // measured ~11.3 KB per slot
// Largest pool used.  The B200 driver clamps the limit to 599,186 slots
// (cudaDeviceGetLimit readback); launching past an explicit limit below the
// clamp fails with cudaErrorLaunchPendingCountExceeded, past the clamp it
// stalls (profiles/cdp_probe_r01.txt).  Waves keep every host launch's
// worst case under this.
constexpr long long kMaxPending = 1 << 19;

int ensure_pending_limit(Workspace* w, const dp_config* c, long long bound) {
  if (c->variant != DP_VARIANT_CDP) return 0;
  bound = std::min(bound, kMaxPending);  // larger bounds run in waves
  long long want = bound + 64;
  if (c->pending_launch_limit > 0) {
    if (c->pending_launch_limit < bound)
      return fail(DP_ERR_QUEUE_OVERFLOW,
                  "queue-overflow: up to " + std::to_string(bound) +
                      " pending device launches exceed pending_launch_limit " +
                      std::to_string(c->pending_launch_limit));
    want = std::min<long long>(c->pending_launch_limit, kMaxPending + 64);
  }
  want = std::max<long long>(want, 2048);
  // Right-size: grow when needed, shrink when far oversized.  A large pool
  // slows every device launch (profiles/cdp_probe_r01.txt: 1000 launches
  // take 0.41 ms at 2048 slots, 1.15 ms at the clamp), so a naive-CDP run
  // must not tax the aggregated runs that follow it.
  int dev = 0;
  DP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_pending_mu);
  long long& have = g_pending_limit[dev & 63];
  (void)w;
  if (want <= have && !(have > 4 * want && have > 8192)) return 0;
  size_t freeb = 0, totb = 0;
  DP_CUDA(cudaMemGetInfo(&freeb, &totb));
  const long long extra =
      std::max<long long>(want - have, 0) * kSlotBytes;
  if (extra > (long long)(freeb * 0.85))
    return fail(DP_ERR_QUEUE_OVERFLOW,
                "queue-overflow: " + std::to_string(bound) +
                    " pending device launches need ~" +
                    std::to_string(extra >> 20) + " MiB of launch pool, " +
                    std::to_string(freeb >> 20) + " MiB free");
  DP_CUDA(cudaDeviceSynchronize());
  DP_CUDA(cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount,
                             (size_t)want));
  size_t got = 0;
  DP_CUDA(cudaDeviceGetLimit(&got, cudaLimitDevRuntimePendingLaunchCount));
  have = (long long)got;
  if ((long long)got < bound + 64)
    return fail(DP_ERR_QUEUE_OVERFLOW,
                "queue-overflow: the device runtime granted " +
                    std::to_string(got) + " pending launches, " +
                    std::to_string(bound) + " may be needed");
  return 0;
}

Knobs knobs_of(const dp_config* c) {
  Knobs k;
  k.threshold = c->threshold;
  k.cf = c->cfactor;
  k.cb = c->child_block;
  k.group = c->group_size;
  k.agg_threshold = c->agg_threshold;
  k.serial_warp = c->serial_mode == DP_SERIAL_WARP;
  k.agg_cf = c->agg_coarsen != 0;
  k.cf_wave = c->cf_wave;
  return k;
}

struct RunCounters {
  unsigned long long host_launches = 0;
  unsigned long long host_blocks = 0;
  unsigned long long kernel_launches = 0;
  double ms_kernel_max = 0.0;
  double ms_kernel_sum = 0.0;
};

#ifndef DP_L1_CARVEOUT
#define DP_L1_CARVEOUT -1  // -1: driver default
#endif

// Shared-memory carve-out preference for the graph kernels: they use < 1 KB
// of shared memory (TC's 16 KB hash is the exception), so the rest can be
// L1 for the random dist probes.
template <class K>
void prefer_l1(K kernel) {
  if (DP_L1_CARVEOUT >= 0)
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         DP_L1_CARVEOUT);
}

template <class App, int AGG, bool CDP>
void launch_parent_inst(const App& app, int grid, int pb, const Knobs& k,
                        const AggTables<App>& t, DevState* ds, long long base,
                        cudaStream_t s) {
  static bool once = [] {
    prefer_l1(parent_kernel<App, AGG, CDP>);
    prefer_l1(child_kernel<App>);
    prefer_l1(child_agg_kernel<App>);
    prefer_l1(child_agg_lb_kernel<App>);
    return true;
  }();
  (void)once;
  parent_kernel<App, AGG, CDP><<<grid, pb, 0, s>>>(app, k, t, ds, base);
}

// Parents per host launch such that the policy's worst-case number of
// pending device launches fits the pool (see ensure_pending_limit).
long long wave_parents(const dp_config* c, long long nparents,
                       long long launchers) {
  if (c->variant != DP_VARIANT_CDP) return nparents;
  if (launch_bound(c, nparents, launchers) <= kMaxPending) return nparents;
  long long per_launch = 1;  // parents that share one potential launch
  if (c->cf_wave <= 0) switch (c->agg) {
    case DP_AGG_WARP: per_launch = 32; break;
    case DP_AGG_BLOCK:
      per_launch = c->agg_threshold > 0 ? 1 : c->parent_block;
      break;
    case DP_AGG_MULTIBLOCK:
      per_launch = (long long)c->parent_block * c->group_size;
      break;
    default: break;
  }
  const long long align = (long long)c->parent_block *
                          (c->agg == DP_AGG_MULTIBLOCK ? c->group_size : 1);
  long long w = kMaxPending * per_launch;
  w = std::max(align, w / align * align);
  return std::min(w, nparents);
}

// Aggregation tables for a parent grid of `grid` x `pb` threads.
template <class App>
int prepare_tables(const dp_config* c, int grid, int pb, Workspace* w,
                   cudaStream_t s, AggTables<App>* t) {
  if (c->variant == DP_VARIANT_CDP && c->agg != DP_AGG_NONE) {
    const size_t rows = (size_t)grid * pb;
    size_t groups = 1;
    if (c->agg == DP_AGG_BLOCK) groups = grid;
    if (c->agg == DP_AGG_MULTIBLOCK)
      groups = dp::ceil_div_ll(grid, c->group_size);
    int r;
    if ((r = grow(&w->tab, &w->tab_bytes, rows * sizeof(typename App::Args))))
      return r;
    size_t scan_bytes = w->scan_rows * sizeof(int);
    void* scan = w->scan;
    if ((r = grow(&scan, &scan_bytes, rows * sizeof(int)))) return r;
    w->scan = (int*)scan;
    w->scan_rows = scan_bytes / sizeof(int);
    if (groups > w->groups) {
      if (w->ctr) cudaFree(w->ctr);
      if (w->done) cudaFree(w->done);
      w->ctr = nullptr;
      w->done = nullptr;
      w->groups = 0;
      DP_CUDA(cudaMalloc(&w->ctr, groups * sizeof(unsigned long long)));
      DP_CUDA(cudaMalloc(&w->done, groups * sizeof(int)));
      DP_CUDA(cudaMemsetAsync(w->ctr, 0, groups * sizeof(unsigned long long), s));
      DP_CUDA(cudaMemsetAsync(w->done, 0, groups * sizeof(int), s));
      w->groups = groups;
    }
    t->args = (typename App::Args*)w->tab;
    t->scan = w->scan;
    t->ctr = w->ctr;
    t->done = w->done;
  }
  return 0;
}

#if DP_CHECK_PUBLISH
// Checker builds, before every parent grid: stamps cleared, rows poisoned
// with 0xff bytes, the device-side table base set (common.cuh).
int arm_checker(Workspace* w, size_t rows, size_t row_bytes, cudaStream_t s) {
  int r;
  if ((r = grow(&w->pub, &w->pub_bytes, rows * sizeof(int)))) return r;
  DP_CUDA(cudaMemsetAsync(w->pub, 0, rows * sizeof(int), s));
  DP_CUDA(cudaMemsetAsync(w->tab, 0xff, rows * row_bytes, s));
  const int* stamp = (const int*)w->pub;
  const char* tab = (const char*)w->tab;
  DP_CUDA(cudaMemcpyToSymbolAsync(g_pub_stamp, &stamp, sizeof(stamp), 0,
                                  cudaMemcpyHostToDevice, s));
  DP_CUDA(cudaMemcpyToSymbolAsync(g_pub_tab, &tab, sizeof(tab), 0,
                                  cudaMemcpyHostToDevice, s));
  return 0;
}

// $DYNPAR_CHECK_TRAP=0: count unpublished reads without trapping (the
// reference's checked=False run of the mutated program)
bool checker_traps() {
  static const bool on = [] {
    const char* e = std::getenv("DYNPAR_CHECK_TRAP");
    return !(e && e[0] == '0');
  }();
  return on;
}
#endif

// One host launch of the parent grid over parents [base, base + nparents)
// (+ the grid-granularity glue).
template <class App>
int launch_wave(const App& app, long long base, long long nparents,
                const dp_config* c, Workspace* w, cudaStream_t s,
                RunCounters* rc) {
  if (nparents <= 0) return 0;  // empty host launch: suppressed (machine.py:172)
  const int pb = c->parent_block;
  const long long grid_ll = dp::ceil_div_ll(nparents, pb);
  if (grid_ll > 0x7fffffffLL)
    return fail(DP_ERR_INVALID, "parent grid too large");
  const int grid = (int)grid_ll;
  AggTables<App> t{nullptr, nullptr, nullptr, nullptr};
  const bool cdp = c->variant == DP_VARIANT_CDP;
  if (int r = prepare_tables(c, grid, pb, w, s, &t)) return r;
#if DP_CHECK_PUBLISH
  if (t.args) {
    if (int r = arm_checker(w, (size_t)grid * pb, sizeof(typename App::Args),
                            s))
      return r;
  }
#endif
  const Knobs k = knobs_of(c);
  const bool single_group =
      c->agg == DP_AGG_GRID ||
      (c->agg == DP_AGG_MULTIBLOCK && (long long)c->group_size >= grid);
  if constexpr (App::kPureExpand) {
    if (cdp && c->persistent > 0 && single_group && !c->frontier) {
      int sms = 148, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const long long pgrid =
          std::min<long long>(grid, (long long)sms * c->persistent);
      if (c->agg == DP_AGG_GRID)
        parent_persistent_kernel<App, kAggGrid><<<(int)pgrid, pb, 0, s>>>(
            app, k, t, w->ds, base, nparents);
      else
        parent_persistent_kernel<App, kAggMulti><<<(int)pgrid, pb, 0, s>>>(
            app, k, t, w->ds, base, nparents);
      DP_CUDA(cudaGetLastError());
      rc->host_launches += 1;
      rc->host_blocks += pgrid;
      rc->kernel_launches += 1;
      goto glue;
    }
  }
  if (!cdp) {
    launch_parent_inst<App, kAggNone, false>(app, grid, pb, k, t, w->ds, base, s);
  } else {
    switch (c->agg) {
      case DP_AGG_NONE:
        launch_parent_inst<App, kAggNone, true>(app, grid, pb, k, t, w->ds, base, s);
        break;
      case DP_AGG_WARP:
        launch_parent_inst<App, kAggWarp, true>(app, grid, pb, k, t, w->ds, base, s);
        break;
      case DP_AGG_BLOCK:
        launch_parent_inst<App, kAggBlock, true>(app, grid, pb, k, t, w->ds, base, s);
        break;
      case DP_AGG_MULTIBLOCK:
        launch_parent_inst<App, kAggMulti, true>(app, grid, pb, k, t, w->ds, base, s);
        break;
      default:
        launch_parent_inst<App, kAggGrid, true>(app, grid, pb, k, t, w->ds, base, s);
        break;
    }
  }
  DP_CUDA(cudaGetLastError());
  rc->host_launches += 1;
  rc->host_blocks += grid;
  rc->kernel_launches += 1;
glue:
  if (cdp && c->agg == DP_AGG_GRID) {
    // completion hook (common.py:144-164): read the fused counter, launch
    // the aggregated child from the host, re-arm the counter
    DP_CUDA(cudaMemcpyAsync(w->h_ctr, w->ctr, sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
    DP_CUDA(cudaStreamSynchronize(s));
    const unsigned long long cv = w->h_ctr[0];
    const int np = (int)(cv >> 32);
    const int total = (int)(cv & 0xffffffffull);
    if (total > 0) {
      child_agg_kernel<App><<<total, c->child_block, 0, s>>>(
          app, t.args, t.scan, np, c->cfactor, 0, w->ds, 0ull);
      DP_CUDA(cudaGetLastError());
      rc->host_launches += 1;
      rc->host_blocks += total;
      rc->kernel_launches += 1;
      DP_CUDA(cudaMemsetAsync(w->ctr, 0, sizeof(unsigned long long), s));
    }
  }
  return 0;
}

// One logical host launch = one or more waves (more only when the policy's
// pending-launch bound exceeds the pool; the reference would trap there).
template <class App>
int launch_parent(const App& app, long long nparents, long long launchers,
                  const dp_config* c, Workspace* w, cudaStream_t s,
                  RunCounters* rc) {
  const long long wave = wave_parents(c, nparents, launchers);
  // step time = parent grid(s) + every child they spawned (a CDP2 parent
  // grid completes only after its children) + the grid-glue launch
  DP_CUDA(cudaEventRecord(w->evk0, s));
  for (long long b = 0; b < nparents; b += wave) {
    int r = launch_wave(app, b, std::min(wave, nparents - b), c, w, s, rc);
    if (r) return r;
  }
  DP_CUDA(cudaEventRecord(w->evk1, s));
  return 0;
}

// after the stream has been synchronised
// per-step device times of the calling thread's last run (dp_step_times)
thread_local std::vector<double> g_step_ms;

int account_step(Workspace* w, RunCounters* rc) {
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->evk0, w->evk1));
  if (rc->ms_kernel_sum == 0.0 && rc->ms_kernel_max == 0.0) g_step_ms.clear();
  g_step_ms.push_back(ms);
  rc->ms_kernel_sum += ms;
  rc->ms_kernel_max = std::max<double>(rc->ms_kernel_max, ms);
  return 0;
}

#ifndef DP_BFS_SPREAD
#define DP_BFS_SPREAD 12  // log2 of the spread block (0: vertex order)
#endif

// spread block of dp_bfs*: DP_BFS_SPREAD, or $DYNPAR_SPREAD_BITS (A/B)
int spread_bits() {
  static const int b = [] {
    const char* e = std::getenv("DYNPAR_SPREAD_BITS");
    return e ? std::max(0, std::min(30, std::atoi(e))) : DP_BFS_SPREAD;
  }();
  return b;
}

// counts[v] = work[spread_slot(v)] (common.cuh)
__global__ void unspread_kernel(const int* __restrict__ work, unsigned mask,
                                int* counts, int n) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) counts[v] = __ldcg(work + spread_slot((unsigned)v, mask));
}

__global__ void init_dist_kernel(int* dist, int n, int src) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dist[i] = i == src ? 0 : kUnreached;
}

template <class T>
__global__ void fill_kernel(T* p, long long n, T v) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

int begin_run(Workspace* w, cudaStream_t s) {
  DP_CUDA(cudaMemsetAsync(w->ds, 0, sizeof(DevState), s));
  if (w->groups) {
    DP_CUDA(cudaMemsetAsync(w->ctr, 0, w->groups * sizeof(unsigned long long), s));
    DP_CUDA(cudaMemsetAsync(w->done, 0, w->groups * sizeof(int), s));
  }
  return 0;
}

// publication checker: an unpublished read traps like the reference's
// checked machine (sim/machine.py:559-574); always 0 in default builds
int check_published(Workspace* w) {
#if DP_CHECK_PUBLISH
  if (w->h_ds->unpublished && checker_traps())
    return fail(DP_ERR_UNPUBLISHED,
                "unpublished-read: " + std::to_string(w->h_ds->unpublished) +
                    " aggregated child block(s) read a table row written by "
                    "another block without an intervening fence");
#else
  (void)w;
#endif
  return 0;
}

__global__ void signal_kernel(const DevState* ds, Workspace::Signal* sig,
                              unsigned seq,
                              const unsigned long long* __restrict__ aux) {
  sig->ds = *ds;
  sig->aux = *aux;
  __threadfence_system();
  *(volatile unsigned*)&sig->seq = seq;
}

// Same result as read_state, lower latency: a one-thread kernel queued after
// the level's work publishes DevState into mapped host memory and the host
// spins on the sequence number (no cudaMemcpyAsync + stream synchronise).
int post_signal(Workspace* w, cudaStream_t s, unsigned* seq_out) {
  const unsigned seq = ++w->seq;
  signal_kernel<<<1, 1, 0, s>>>(w->ds, w->d_sig, seq, w->d_scratch + 1);
  DP_CUDA(cudaGetLastError());
  *seq_out = seq;
  return 0;
}

// wait until signal `seq` has landed; h_ds then holds the state after every
// kernel queued before that signal
int wait_signal(Workspace* w, cudaStream_t s, unsigned seq) {
  volatile unsigned* flag = &w->h_sig->seq;
  auto landed = [&] { return *flag == seq; };
  for (unsigned spin = 1; !landed(); ++spin) {
    if ((spin & 1023) == 0) {
      const cudaError_t e = cudaStreamQuery(s);
      if (e != cudaSuccess && e != cudaErrorNotReady)
        return fail(DP_ERR_CUDA, std::string("cuda-error: ") +
                                     cudaGetErrorString(e));
      if (e == cudaSuccess && !landed()) break;  // drained: re-check below
    }
  }
  __atomic_thread_fence(__ATOMIC_ACQUIRE);
  if (!landed()) {  // stream drained without the signal: fall back
    DP_CUDA(cudaStreamSynchronize(s));
  }
  std::memcpy((void*)w->h_ds, (const void*)&w->h_sig->ds, sizeof(DevState));
  if (w->h_ds->err) return map_device_error(w->h_ds->err);
  return check_published(w);
}

int read_state_fast(Workspace* w, cudaStream_t s) {
  unsigned seq = 0;
  int r;
  if ((r = post_signal(w, s, &seq))) return r;
  return wait_signal(w, s, seq);
}

int read_state(Workspace* w, cudaStream_t s) {
  DP_CUDA(cudaMemcpyAsync(w->h_ds, w->ds, sizeof(DevState),
                          cudaMemcpyDeviceToHost, s));
  DP_CUDA(cudaStreamSynchronize(s));
  if (w->h_ds->err) return map_device_error(w->h_ds->err);
  return check_published(w);
}

void finish_stats(Workspace* w, const RunCounters& rc, float ms,
                  dp_stats* st) {
  if (!st) return;
  st->num_launches = w->h_ds->launches;
  st->host_launches = rc.host_launches;
  st->blocks_scheduled = w->h_ds->blocks + rc.host_blocks;
  st->max_pending_depth = (unsigned long long)std::max(w->h_ds->max_pending, 0);
  st->ns_device = (double)ms * 1e6;
  st->ns_kernel_max = rc.ms_kernel_max * 1e6;
  st->ns_kernel_sum = rc.ms_kernel_sum * 1e6;
  st->kernel_launches = rc.kernel_launches;
  st->launch_lat_ns_mean =
      w->h_ds->lat_cnt ? (double)w->h_ds->lat_sum / (double)w->h_ds->lat_cnt
                       : 0.0;
  st->remote_ops = w->h_ds->remote;
  st->unpublished_reads = w->h_ds->unpublished;
  st->poisoned_reads = w->h_ds->poisoned;
  // DP_PROFILE builds: summed warp-cycles per phase -> warp-ns at the SM
  // clock rate the device reports (zero, and no query, in the default build)
  bool any = false;
  for (int i = 0; i < 5; ++i) any |= w->h_ds->phase[i] != 0;
  if (any) {
    int dev = 0, khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    for (int i = 0; i < 5; ++i)
      st->ns_phase[i] =
          khz > 0 ? (double)w->h_ds->phase[i] * 1e6 / (double)khz : 0.0;
  }
}

void clear_stats(dp_stats* st) {
  if (st) std::memset(st, 0, sizeof(*st));
}

double now_ns() {
  return (double)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// ---------------------------------------------------------------------------
// level/round-loop apps
// ---------------------------------------------------------------------------

// Levels/rounds chained on the device (round_controller, sched.cuh): one
// host launch per chain of kChain rounds; the host only checks done_round.
template <class App>
int device_loop(Workspace* w, const dp_config* c, long long nparents,
                int max_iter, cudaStream_t s, const App& app0,
                RunCounters* rc, int* it, bool* converged) {
  constexpr int kChain = 16;
  const int pb = c->parent_block;
  const int grid = (int)dp::ceil_div_ll(nparents, pb);
  AggTables<App> t{nullptr, nullptr, nullptr, nullptr};
  int r;
  if ((r = prepare_tables(c, grid, pb, w, s, &t))) return r;
  const Knobs k = knobs_of(c);
  for (int first = 0; first <= max_iter; first += kChain) {
    const int last = std::min(first + kChain - 1, max_iter);
    switch (c->agg) {
      case DP_AGG_NONE:
        round_controller<App, kAggNone><<<1, 1, 0, s>>>(
            app0, k, t, w->ds, grid, pb, first, first, last);
        break;
      case DP_AGG_WARP:
        round_controller<App, kAggWarp><<<1, 1, 0, s>>>(
            app0, k, t, w->ds, grid, pb, first, first, last);
        break;
      case DP_AGG_BLOCK:
        round_controller<App, kAggBlock><<<1, 1, 0, s>>>(
            app0, k, t, w->ds, grid, pb, first, first, last);
        break;
      default:
        round_controller<App, kAggMulti><<<1, 1, 0, s>>>(
            app0, k, t, w->ds, grid, pb, first, first, last);
        break;
    }
    DP_CUDA(cudaGetLastError());
    rc->host_launches += 1;
    rc->host_blocks += 1;
    rc->kernel_launches += 1;
    if ((r = read_state(w, s))) return r;
    if (w->h_ds->done_round > 0) {
      *it = w->h_ds->done_round;
      *converged = true;
      return 0;
    }
    *it = last + 1;
  }
  return 0;
}

// Host-buffer calls that overlap the H2D copy of the edge arrays with the
// rounds: chunks [0, nchunks) land in order; chunk_ev[k] completes when
// chunk k has (the device counter says the same to the kernels).
struct Arrival {
  int nchunks = 0;
  int waited = 0;  // chunks the host has already waited for
  // speculative readback of the result (dp_sssp): once every chunk has
  // landed, after each round that still lowered something the result is
  // copied device -> host on the copy stream while the next round runs; a
  // next round that lowers nothing writes nothing, so that copy is the
  // result and the call skips its final D2H
  void* host_out = nullptr;
  const void* dev_out = nullptr;
  size_t out_bytes = 0;
  int spec_after = -1;      // round whose state the last copy holds
  bool spec_final = false;  // that copy is the result
  uint64_t spec_d2h = 0;    // bytes of every speculative copy
};

struct NoFinish {
  void operator()() const {}
};
// which levels need the launching parent variant (default: all of them)
struct AlwaysCdp {
  bool operator()(int, const DevState*) const { return true; }
};

template <class MakeApp, class Finish = NoFinish, class Pick = AlwaysCdp>
int iterate(Workspace* w, const dp_config* c, long long nparents,
            long long launchers, int max_iter, cudaStream_t s, MakeApp make,
            dp_stats* st, Arrival* arr = nullptr, Finish finish = Finish(),
            Pick pick = Pick(), long long lazy_bound = -1) {
  // a level in which no parent can reach the threshold runs the launch-free
  // parent variant: same serial arm, same outputs and counters, but without
  // the ~11 us a CDP-capable parent grid costs even when it launches nothing
  // (profiles/r02/floor_probe_r02.txt)
  dp_config c_flat = *c;
  c_flat.variant = DP_VARIANT_NOCDP;
  RunCounters rc;
  int r;
  // lazy_bound >= 0 (count_launchers_lazy): `launchers` is an upper bound,
  // the pool bound is lazy_bound (one wave), and the exact count arrives
  // with round 0's readback; until then round 0 keeps the launching variant
  // (same outputs and counters either way)
  long long exact = lazy_bound >= 0 ? -1 : launchers;
  const long long wave_launchers = lazy_bound >= 0 ? 0 : launchers;
  if ((r = ensure_pending_limit(w, c,
                                lazy_bound >= 0
                                    ? lazy_bound
                                    : launch_bound(c, nparents, launchers))))
    return r;
  if ((r = begin_run(w, s))) return r;
  DP_CUDA(cudaEventRecord(w->ev0, s));
  int it = 0;
  bool converged = false;
  bool fresh = false;  // h_ds holds the state after the last kernel
  if (c->device_loop && c->variant == DP_VARIANT_CDP && !arr &&
      c->agg != DP_AGG_GRID &&
      wave_parents(c, nparents, wave_launchers) == nparents) {
    if ((r = device_loop(w, c, nparents, max_iter, s, make(0, w->ds), &rc,
                         &it, &converged)))
      return r;
  }
  for (; !converged && it <= max_iter; ++it) {
    auto app = make(it, w->ds);
    // no parent can ever reach the threshold (an exact launcher count of 0,
    // e.g. road graphs below T): every level runs launch-free
    const dp_config* cl = c->variant == DP_VARIANT_CDP &&
                                  (exact == 0 || !pick(it, w->h_ds))
                              ? &c_flat
                              : c;
    // chunks known to have landed before this round starts (it sees them)
    while (arr && arr->waited < arr->nchunks) {
      const cudaError_t q = cudaEventQuery(w->chunk_ev[arr->waited]);
      if (q == cudaSuccess) {
        ++arr->waited;
        continue;
      }
      if (q != cudaErrorNotReady) DP_CUDA(q);
      if (cudaPeekAtLastError() == cudaErrorNotReady) (void)cudaGetLastError();
      break;
    }
    if ((r = launch_parent(app, nparents, wave_launchers, cl, w, s, &rc)))
      return r;
    if ((r = read_state_fast(w, s))) return r;
    fresh = true;
    if (exact < 0) exact = (long long)w->h_sig->aux;
    if ((r = account_step(w, &rc))) return r;
    if (w->h_ds->flag[it & 1] == 0 &&
        (!arr || w->h_ds->skipped[it & 1] == 0)) {
      converged = true;
      if (arr && it > 0 && arr->spec_after == it - 1) arr->spec_final = true;
      ++it;
      break;
    }
    if (arr && arr->host_out &&
        (arr->nchunks == 0 ||
         cudaEventQuery(w->chunk_ev[arr->nchunks - 1]) == cudaSuccess)) {
      if (!w->ev_spec)
        DP_CUDA(cudaEventCreateWithFlags(&w->ev_spec, cudaEventDisableTiming));
      DP_CUDA(cudaEventRecord(w->ev_spec, s));
      DP_CUDA(cudaStreamWaitEvent(w->copy_stream, w->ev_spec, 0));
      DP_CUDA(cudaMemcpyAsync(arr->host_out, arr->dev_out, arr->out_bytes,
                              cudaMemcpyDeviceToHost, w->copy_stream));
      arr->spec_after = it;
      arr->spec_d2h += arr->out_bytes;
    }
    if (cudaPeekAtLastError() == cudaErrorNotReady) (void)cudaGetLastError();
    // edges still landing: the next round starts when the next chunk has
    // (rounds re-scanning unchanged data would only compete with the DMA
    // for L2: measured 13.2 vs 12.1 ms with back-to-back rounds)
    // (waiting only after a round that lowered nothing measured no better:
    // 7.95-8.03 vs 7.89-7.91 ms, profiles/r02/e2e_eager_r02.txt)
    if (arr && arr->waited < arr->nchunks && w->h_ds->skipped[it & 1])
      DP_CUDA(cudaEventSynchronize(w->chunk_ev[arr->waited++]));
  }
  finish();  // run epilogue kernels (inside the timed region)
  DP_CUDA(cudaEventRecord(w->ev1, s));
  DP_CUDA(cudaEventSynchronize(w->ev1));
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  // the epilogue kernels never touch DevState: the last round's readback
  // is already the final state (saves a copy + synchronise per call)
  if (!fresh && (r = read_state(w, s))) return r;
  if (rc.ms_kernel_sum == 0.0) {  // device loop: no per-level host events
    rc.ms_kernel_sum = ms;
    rc.ms_kernel_max = ms;
  }
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = it;
  if (!converged)
    return fail(DP_ERR_ITERATIONS, "used more iterations than vertices");
  return 0;
}

// bit v = 1 iff row v would launch under threshold t (cnt > 0 and (t == 0
// or cnt >= t), sched.cuh parent_kernel); one warp per 32 words
__global__ void launch_bits_kernel(const int* __restrict__ rowptr, int n,
                                   int t, unsigned* bits) {
  const long long words = (n + 31) / 32;
  for (long long wd = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
       wd * 32 < (long long)n + 0 && wd < words;
       wd += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long v = wd * 32 + lane_id();
    bool go = false;
    if (v < n) {
      const int d = __ldg(rowptr + v + 1) - __ldg(rowptr + v);
      go = d > 0 && (t == 0 || d >= t);
    }
    const unsigned m = __ballot_sync(DP_FULL, go);
    if (lane_id() == 0) bits[wd] = m;
  }
}

int bfs_dev_impl(const int32_t* rowptr, const int32_t* col, int32_t n,
                 int32_t src, const dp_config* c, int32_t* dist,
                 int32_t* counts, cudaStream_t s, dp_stats* st,
                 int64_t m = -1) {
  int r;
  if ((r = validate(c))) return r;
  if (n < 1) return fail(DP_ERR_INVALID, "graph must have at least 1 vertex");
  if (src < 0 || src >= n) return fail(DP_ERR_INVALID, "source out of range");
  Workspace* w = workspace(&r);
  if (!w) return r;
  init_dist_kernel<<<dp::ceil_div(n, 256), 256, 0, s>>>(dist, n, src);
  // counts accumulate in the spread layout (common.cuh spread_slot) and are
  // gathered into vertex order after the last level
  unsigned cmask = 0;
  int* cw = counts;
  const int sb = spread_bits();
  if (sb > 0 && n >= 1024) {
    const size_t blk = (size_t)1 << sb;
    const size_t slots = (n + blk - 1) / blk * blk;
    if ((r = grow(&w->cwork, &w->cwork_bytes, slots * sizeof(int)))) return r;
    cw = (int*)w->cwork;
    cmask = (unsigned)(blk - 1);
    DP_CUDA(cudaMemsetAsync(cw, 0, slots * sizeof(int), s));
  } else {
    DP_CUDA(cudaMemsetAsync(counts, 0, (size_t)n * sizeof(int), s));
  }
  long long launchers = 0, lazy = -1;
  if (c->variant == DP_VARIANT_CDP &&
      (r = count_launchers_lazy(w, c, rowptr, n, m, s, &launchers, &lazy)))
    return r;
  // launch bits: the host picks each level's parent variant from whether the
  // previous level discovered any vertex whose row would launch
  const unsigned* lbits = nullptr;
  const bool per_level = c->variant == DP_VARIANT_CDP && !c->device_loop;
  if (per_level) {
    if ((r = grow(&w->lbits, &w->lbits_bytes,
                  (size_t)(n + 31) / 32 * sizeof(unsigned))))
      return r;
    lbits = (const unsigned*)w->lbits;
    launch_bits_kernel<<<std::min(dp::ceil_div(dp::ceil_div(n, 32), 8), 148 * 8),
                         256, 0, s>>>(rowptr, n, effective_threshold(c),
                                      (unsigned*)w->lbits);
    DP_CUDA(cudaGetLastError());
  }
  // bench/benchmarks.py:157-168: one launch per level until nothing changes
  return iterate(w, c, n, launchers, n, s,
                 [&](int level, DevState* ds) {
                   BfsApp a;
                   a.rowptr = rowptr;
                   a.col = col;
                   a.dist = dist;
                   a.counts = cw;
                   a.changed = &ds->flag[level & 1];
                   a.changed_next = &ds->flag[(level + 1) & 1];
                   a.lbits = lbits;
                   a.big_next = &ds->big[(level + 1) & 1];
                   a.big_after = &ds->big[level & 1];
                   a.n = n;
                   a.level = level;
                   a.cmask = cmask;
                   a.pad_ = 0;
                   return a;
                 },
                 st, nullptr, [&] {
                   if (cmask)
                     unspread_kernel<<<dp::ceil_div(n, 256), 256, 0, s>>>(
                         cw, cmask, counts, n);
                 },
                 [&](int level, const DevState* h) {
                   // level 0 (the source alone) keeps the launching variant
                   return !per_level || level == 0 || h->big[level & 1] != 0;
                 },
                 lazy);
}

// Pack int32 weights into nibbles (w - 1, 8 per word); *bad = 1 if any
// weight lies outside [1, 16].  One thread per output word, two 16-byte loads.
__global__ void pack_weights_kernel(const int* __restrict__ w, long long m,
                                    unsigned* __restrict__ out, int* bad) {
  const long long words = (m + 7) >> 3;
  unsigned any = 0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
       k < words; k += (long long)gridDim.x * blockDim.x) {
    int x[8];
    if (k * 8 + 8 <= m) {
      const int4 a = __ldg(reinterpret_cast<const int4*>(w) + 2 * k);
      const int4 b = __ldg(reinterpret_cast<const int4*>(w) + 2 * k + 1);
      x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
      x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = k * 8 + j < m ? w[k * 8 + j] : 1;
    }
    unsigned word = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const unsigned v = (unsigned)(x[j] - 1);
      any |= v > 15u;
      word |= (v & 15u) << (4 * j);
    }
    out[k] = word;
  }
  if (__any_sync(DP_FULL, any) && lane_id() == 0) *bad = 1;
}

// Host twin for slots [lo, lo + len) (lo a multiple of 8); false if any
// weight lies outside [1, 16].  OpenMP over the host cores.
bool pack_weights_host(const int32_t* w, long long lo, long long len,
                       unsigned* out) {
  const long long full = len / 8;  // whole words: fixed trip count (SIMD)
  unsigned bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
  for (long long k = 0; k < full; ++k) {
    const int32_t* x = w + lo + k * 8;
    unsigned word = 0, b = 0;
#pragma GCC unroll 8
    for (int j = 0; j < 8; ++j) {
      const unsigned v = (unsigned)(x[j] - 1);
      b |= v;
      word |= (v & 15u) << (4 * j);
    }
    bad |= b;
    out[(lo >> 3) + k] = word;
  }
  if (full * 8 < len) {  // tail word
    unsigned word = 0;
    for (long long e = lo + full * 8; e < lo + len; ++e) {
      const unsigned v = (unsigned)(w[e] - 1);
      bad |= v;
      word |= (v & 15u) << (4 * (e & 7));
    }
    out[(lo >> 3) + full] = word;
  }
  return bad <= 15u;  // the OR of every (w - 1) fits 4 bits
}

// dp_config.weight_bits = 4 with resident weights: pack them on the device;
// *wpack stays null when some weight lies outside [1, 16]
int pack_weights_dev(Workspace* w, const int32_t* weight, long long m,
                     cudaStream_t s, const unsigned** wpack) {
  int r;
  *wpack = nullptr;
  if (m <= 0) return 0;
  if ((r = grow(&w->wpack, &w->wpack_bytes,
                (size_t)((m + 7) / 8) * sizeof(unsigned))))
    return r;
  if (!w->d_bad) DP_CUDA(cudaMalloc(&w->d_bad, sizeof(int)));
  DP_CUDA(cudaMemsetAsync(w->d_bad, 0, sizeof(int), s));
  const int blocks = (int)std::max<long long>(
      1, std::min<long long>(dp::ceil_div_ll((m + 7) / 8, 256), 148 * 8));
  pack_weights_kernel<<<blocks, 256, 0, s>>>(weight, m, (unsigned*)w->wpack,
                                             w->d_bad);
  DP_CUDA(cudaGetLastError());
  int bad = 0;
  DP_CUDA(cudaMemcpyAsync(&bad, w->d_bad, sizeof(int), cudaMemcpyDeviceToHost,
                          s));
  DP_CUDA(cudaStreamSynchronize(s));
  if (!bad) *wpack = (const unsigned*)w->wpack;
  return 0;
}

int sssp_dev_impl(const int32_t* rowptr, const int32_t* col,
                  const int32_t* weight, int32_t n, int32_t src,
                  const dp_config* c, int32_t* dist, cudaStream_t s,
                  dp_stats* st, Arrival* arr = nullptr, int shift = 0,
                  const unsigned* wpack = nullptr, int64_t m = -1) {
  int r;
  if ((r = validate(c))) return r;
  if (n < 1) return fail(DP_ERR_INVALID, "graph must have at least 1 vertex");
  if (src < 0 || src >= n) return fail(DP_ERR_INVALID, "source out of range");
  Workspace* w = workspace(&r);
  if (!w) return r;
  init_dist_kernel<<<dp::ceil_div(n, 256), 256, 0, s>>>(dist, n, src);
  int* last = nullptr;
  if (c->frontier) {
    if ((r = grow(&w->io[5], &w->io_bytes[5], (size_t)n * sizeof(int))))
      return r;
    last = (int*)w->io[5];
    fill_kernel<int><<<dp::ceil_div(n, 256), 256, 0, s>>>(last, n, kUnreached);
  }
  long long launchers = 0, lazy = -1;
  if (c->variant == DP_VARIANT_CDP &&
      (r = count_launchers_lazy(w, c, rowptr, n, m, s, &launchers, &lazy)))
    return r;
  // bench/benchmarks.py:259-270: rounds until a full round changes nothing
  // (and, while edges are still landing, no parent was deferred)
  const int max_iter = n + (arr ? arr->nchunks + 1 : 0);

  auto run = [&](auto tag) {
    using App = decltype(tag);
    return iterate(w, c, n, launchers, max_iter, s,
                   [&](int round, DevState* ds) {
                     App a;
                     a.rowptr = rowptr;
                     a.col = col;
                     a.weight = weight;
                     a.wpack = wpack;
                     a.dist = dist;
                     a.changed = &ds->flag[round & 1];
                     a.changed_next = &ds->flag[(round + 1) & 1];
                     a.last = last;
                     a.arrived = arr ? w->d_arrived : nullptr;
                     a.skipped = &ds->skipped[round & 1];
                     a.skipped_next = &ds->skipped[(round + 1) & 1];
                     a.n = n;
                     a.shift = shift;
                     return a;
                   },
                   st, arr, NoFinish(), AlwaysCdp(), lazy);
  };
  return wpack ? run(SsspPackedApp{}) : run(SsspApp{});
}

__global__ void gc_key_kernel(const int* __restrict__ rowptr, int n,
                              unsigned long long* key) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x)
    key[v] = gc_key((int)v, rowptr[v + 1] - rowptr[v]);
}

// Vertices whose wait count is 0 after the count pass: the first worklist.
__global__ void gc_seed_kernel(const int* __restrict__ wait, int n, int* list,
                               int* count) {
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x -
                     lane_id();
       b < n; b += (long long)gridDim.x * blockDim.x) {
    const long long u = b + lane_id();
    const bool ready = u < n && __ldg(wait + u) == 0;
    const unsigned m = __ballot_sync(DP_FULL, ready);
    int base = 0;
    if (lane_id() == 0 && m) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(DP_FULL, base, 0);
    if (ready) list[base + __popc(m & lanemask_lt())] = (int)u;
  }
}

// mex pass of a colouring round: each ready vertex takes the smallest colour
// not marked in its bitmap [rowptr[u] + u, rowptr[u] + u + deg].  Thread 0
// also counts the round if it was not empty and clears the next round's
// worklist length.
__global__ void gc_mex_kernel(const int* __restrict__ rowptr,
                              const int* __restrict__ list, const int* count,
                              int* next_count, int* rounds, int* color,
                              const unsigned* __restrict__ used) {
  const int nr = __ldcg(count);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *next_count = 0;
    if (nr > 0) *rounds += 1;
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nr;
       i += (long long)gridDim.x * blockDim.x) {
    const int u = list[i];
    const long long b0 = (long long)rowptr[u] + u;
    const long long b1 = (long long)rowptr[u + 1] + u + 1;  // deg + 1 bits
    long long bit = b0;
    int mex = -1;
    while (bit < b1) {
      const long long wi = bit >> 5;
      unsigned free_bits = ~__ldcg(used + wi);
      free_bits &= ~0u << (bit & 31);  // bits before the range
      const long long wend = (wi + 1) << 5;
      if (wend > b1) free_bits &= (1u << (b1 & 31)) - 1;  // bits after
      if (free_bits) {
        mex = (int)((wi << 5) + __ffs(free_bits) - 1 - b0);
        break;
      }
      bit = wend;
    }
    color[u] = mex;  // always found: deg neighbours use at most deg colours
  }
}

int gc_dev_impl(const int32_t* rowptr, const int32_t* col, int32_t n,
                int64_t m, const dp_config* c, int32_t* color,
                cudaStream_t s, dp_stats* st) {
  int r;
  if ((r = validate(c))) return r;
  if (n < 0 || m < 0) return fail(DP_ERR_INVALID, "bad graph size");
  Workspace* w = workspace(&r);
  if (!w) return r;
  // keys[n] | used bitmap | wait[n] | two worklists[n] | counts[2] | rounds
  const size_t words = (size_t)((m + n + 31) / 32) + 1;
  const size_t nn = (size_t)std::max(n, 1);
  if ((r = grow(&w->io[5], &w->io_bytes[5],
                nn * 8 + words * sizeof(unsigned) +
                    (nn * 3 + 4) * sizeof(int))))
    return r;
  unsigned long long* keys = (unsigned long long*)w->io[5];
  unsigned* used = (unsigned*)(keys + nn);
  int* wait = (int*)(used + words);
  int* list[2] = {wait + nn, wait + 2 * nn};
  int* cnt = wait + 3 * nn;  // cnt[0], cnt[1]: worklist lengths
  int* d_rounds = cnt + 2;
  long long launchers = 0;
  if (c->variant == DP_VARIANT_CDP &&
      (r = count_launchers(w, c, rowptr, n, 0, s, &launchers)))
    return r;
  if ((r = ensure_pending_limit(w, c, launch_bound(c, n, launchers))))
    return r;
  if ((r = begin_run(w, s))) return r;
  RunCounters rc;
  DP_CUDA(cudaEventRecord(w->ev0, s));
  DP_CUDA(cudaMemsetAsync(used, 0, words * sizeof(unsigned), s));
  DP_CUDA(cudaMemsetAsync(wait, 0, nn * sizeof(int), s));
  DP_CUDA(cudaMemsetAsync(cnt, 0, 3 * sizeof(int), s));
  const int kb = std::max(1, std::min(dp::ceil_div(std::max(n, 1), 256),
                                      148 * 8));
  gc_key_kernel<<<kb, 256, 0, s>>>(rowptr, n, keys);
  DP_CUDA(cudaGetLastError());
  rc.kernel_launches += 1;
  if (n) DP_CUDA(cudaMemsetAsync(color, 0xff, (size_t)n * sizeof(int), s));
  GcCountApp ca;
  ca.rowptr = rowptr;
  ca.col = col;
  ca.key = keys;
  ca.wait = wait;
  ca.n = n;
  ca.pad = 0;
  if ((r = launch_parent(ca, n, launchers, c, w, s, &rc))) return r;
  const int fb = std::max(1, std::min(dp::ceil_div(std::max(n, 1), 256),
                                      148 * 8));
  gc_seed_kernel<<<fb, 256, 0, s>>>(wait, n, list[0], cnt);
  DP_CUDA(cudaGetLastError());
  rc.kernel_launches += 1;
  // Rounds are queued in batches without a host round trip each: parents
  // past the device-side worklist length exit, an empty round is a no-op.
  // Every vertex is coloured after at most n non-empty rounds.
  constexpr int kBatch = 8;
  int cur = 0;
  for (long long queued = 0;; queued += kBatch) {
    if (queued > (long long)n + kBatch)
      return fail(DP_ERR_ITERATIONS, "colouring made no progress");
    for (int b = 0; b < kBatch; ++b) {
      GcGatherApp ga;
      ga.rowptr = rowptr;
      ga.col = col;
      ga.key = keys;
      ga.ready = list[cur];
      ga.nready = cnt + cur;
      ga.color = color;
      ga.used = used;
      if ((r = launch_parent(ga, n, launchers, c, w, s, &rc))) return r;
      gc_mex_kernel<<<fb, 256, 0, s>>>(rowptr, list[cur], cnt + cur,
                                       cnt + (cur ^ 1), d_rounds, color, used);
      DP_CUDA(cudaGetLastError());
      rc.kernel_launches += 1;
      GcNotifyApp na;
      na.rowptr = rowptr;
      na.col = col;
      na.key = keys;
      na.ready = list[cur];
      na.nready = cnt + cur;
      na.wait = wait;
      na.next = list[cur ^ 1];
      na.next_count = cnt + (cur ^ 1);
      if ((r = launch_parent(na, n, launchers, c, w, s, &rc))) return r;
      cur ^= 1;
    }
    int h[3] = {0, 0, 0};
    DP_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    if ((r = read_state(w, s))) return r;  // syncs s
    if (h[cur] == 0) break;  // the next round's worklist is empty: done
  }
  DP_CUDA(cudaEventRecord(w->ev1, s));
  DP_CUDA(cudaEventSynchronize(w->ev1));
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  if ((r = read_state(w, s))) return r;
  int rounds = 0;
  DP_CUDA(cudaMemcpy(&rounds, d_rounds, sizeof(int), cudaMemcpyDeviceToHost));
  rc.ms_kernel_sum = rc.ms_kernel_max = ms;
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = rounds;
  return 0;
}

// ---------------------------------------------------------------------------
// MST (Boruvka): per round MSTF (nested find) -> flag readback -> MSTV (nested
// verify) -> hook -> pointer jumping.  Under the strict (weight, eid) order
// the chosen edges form a forest whose only cycles are mutual pairs.
// ---------------------------------------------------------------------------
__global__ void mst_init_kernel(int n, int* comp, unsigned long long* cmin) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    comp[v] = (int)v;
    cmin[v] = kNoEdge;
  }
}

// Roots with a chosen edge attach to their partner component; of a mutual
// pair the smaller root stays.  Each chosen edge's weight is counted once.
__global__ void mst_hook_kernel(int n, int* comp,
                                const unsigned long long* __restrict__ cmin,
                                const int* __restrict__ partner,
                                unsigned long long* sums /* [wsum, edges] */) {
  long long w = 0, c = 0;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    if (comp[v] != v) continue;  // only thread v writes a root's comp
    const unsigned long long k = cmin[v];
    if (k == kNoEdge) continue;
    const int p = partner[v];
    const bool mutual = cmin[p] == k;
    if (!mutual || v < p) {
      w += (long long)(int)((unsigned)(k >> 32) ^ 0x80000000u);
      c += 1;
    }
    if (!mutual || v > p) comp[v] = p;
  }
  w = (long long)warp_sum_u64((unsigned long long)w);
  c = (long long)warp_sum_u64((unsigned long long)c);
  if (lane_id() == 0 && c) {
    atomicAdd(sums, (unsigned long long)w);
    atomicAdd(sums + 1, (unsigned long long)c);
  }
}

// New roots after hooking: every vertex walks read-only to its root and
// stores it.  Roots are fixed during the kernel and only roots are stored,
// so concurrent walkers always see ancestors and every vertex ends at its
// root.  Measured faster than in-place path halving on both RMAT-22 (4.2 vs
// 5.0 ms per MST) and road graphs with long hook chains (1.56 vs 1.76 ms on
// road:2000000): halving's stores to shared lines cost more than the longer
// read-only walks (profiles/mst_ab_r01.txt).  The pass also re-arms cmin.
__global__ void mst_root_kernel(int n, int* comp, unsigned long long* cmin) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    int x = __ldcg(comp + v);
    for (int p; (p = __ldcg(comp + x)) != x;) x = p;
    __stcg(comp + v, x);
    cmin[v] = kNoEdge;
  }
}

int mst_dev_impl(const int32_t* rowptr, const int32_t* col,
                 const int32_t* weight, const int32_t* eid, int32_t n,
                 int64_t m, const dp_config* cf, const dp_config* cv,
                 uint8_t* in_mst, int64_t* total_weight, int64_t* nedges,
                 cudaStream_t s, dp_stats* st) {
  int r;
  if (!cv) cv = cf;
  if ((r = validate(cf)) || (r = validate(cv))) return r;
  if (n < 0 || m < 0) return fail(DP_ERR_INVALID, "bad graph size");
  Workspace* w = workspace(&r);
  if (!w) return r;
  // cmin[n] | comp[n] | partner[n]
  const size_t nn = (size_t)std::max(n, 1);
  if ((r = grow(&w->io[5], &w->io_bytes[5], nn * (8 + 4 + 4)))) return r;
  unsigned long long* cmin = (unsigned long long*)w->io[5];
  int* comp = (int*)(cmin + nn);
  int* partner = comp + nn;
  unsigned long long* sums = w->d_scratch;  // [0] weight, [1] edges
  const int blocks = std::max(1, std::min(dp::ceil_div(std::max(n, 1), 256),
                                          148 * 8));
  mst_init_kernel<<<blocks, 256, 0, s>>>(n, comp, cmin);
  DP_CUDA(cudaGetLastError());
  if (m) DP_CUDA(cudaMemsetAsync(in_mst, 0, (size_t)m, s));
  long long lf = 0, lv = 0;
  if (cf->variant == DP_VARIANT_CDP &&
      (r = count_launchers(w, cf, rowptr, n, 0, s, &lf)))
    return r;
  if (cv->variant == DP_VARIANT_CDP &&
      (r = count_launchers(w, cv, rowptr, n, 0, s, &lv)))
    return r;
  if ((r = ensure_pending_limit(
           w, cf->variant == DP_VARIANT_CDP ? cf : cv,
           std::max(launch_bound(cf, n, lf), launch_bound(cv, n, lv)))))
    return r;
  // after count_launchers, which uses d_scratch[1]
  DP_CUDA(cudaMemsetAsync(sums, 0, 2 * sizeof(unsigned long long), s));
  if ((r = begin_run(w, s))) return r;
  RunCounters rc;
  DP_CUDA(cudaEventRecord(w->ev0, s));
  int rounds = 0;
  for (;; ++rounds) {
    if (rounds > 64)  // components at least halve every round
      return fail(DP_ERR_ITERATIONS, "Boruvka did not converge");
    DP_CUDA(cudaMemsetAsync(&w->ds->flag[0], 0, sizeof(int), s));
    MstFindApp fa;
    fa.rowptr = rowptr;
    fa.col = col;
    fa.weight = weight;
    fa.eid = eid;
    fa.comp = comp;
    fa.cmin = cmin;
    fa.changed = &w->ds->flag[0];
    fa.n = n;
    fa.pad = 0;
    if ((r = launch_parent(fa, n, lf, cf, w, s, &rc))) return r;
    if ((r = read_state_fast(w, s))) return r;
    if (w->h_ds->flag[0] == 0) break;  // no edge leaves any component
    MstVerifyApp va;
    va.rowptr = rowptr;
    va.col = col;
    va.eid = eid;
    va.comp = comp;
    va.cmin = cmin;
    va.in_mst = in_mst;
    va.partner = partner;
    va.n = n;
    va.pad = 0;
    if ((r = launch_parent(va, n, lv, cv, w, s, &rc))) return r;
    mst_hook_kernel<<<blocks, 256, 0, s>>>(n, comp, cmin, partner, sums);
    mst_root_kernel<<<blocks, 256, 0, s>>>(n, comp, cmin);
    DP_CUDA(cudaGetLastError());
    rc.kernel_launches += 2;
  }
  DP_CUDA(cudaEventRecord(w->ev1, s));
  DP_CUDA(cudaEventSynchronize(w->ev1));
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  if ((r = read_state(w, s))) return r;
  unsigned long long h[2] = {0, 0};
  DP_CUDA(cudaMemcpyAsync(h, sums, sizeof(h), cudaMemcpyDeviceToHost, s));
  DP_CUDA(cudaStreamSynchronize(s));
  if (total_weight) *total_weight = (int64_t)h[0];
  if (nedges) *nedges = (int64_t)h[1];
  rc.ms_kernel_sum = rc.ms_kernel_max = ms;
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = rounds + 1;  // + the final find that saw no edge
  return 0;
}

// ---------------------------------------------------------------------------
// Survey propagation: sweeps of (reset products -> SpVarApp -> SpClauseApp)
// until max |eta' - eta| <= eps or max_sweeps, then the variable biases.
// ---------------------------------------------------------------------------
__global__ void sp_reset_kernel(int n, SpVarProd* prod) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    SpVarProd q;
    q.p[0] = q.p[1] = 1.0;
    q.z[0] = q.z[1] = 0;
    q.pad[0] = q.pad[1] = 0;
    prod[i] = q;
  }
}

// occs[t] = sp_tile(occ[t]) << 1 | negated (the variable side reads signs
// in order)
__global__ void sp_pack_kernel(long long ne, int k,
                               const int* __restrict__ occ,
                               const int* __restrict__ lits, int* occs) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < ne;
       t += (long long)gridDim.x * blockDim.x) {
    const int e = occ[t];
    occs[t] = (int)(sp_tile(e / k, e % k, k) << 1) | (lits[e] & 1);
  }
}

// clause-major <-> clause-tiled (sp_tile) copies of lit and eta
__global__ void sp_tile_kernel(long long ne, int k,
                               const int* __restrict__ lits,
                               const double* __restrict__ eta, int* lit_t,
                               double* eta_t) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (long long)gridDim.x * blockDim.x) {
    const long long d = sp_tile(e / k, (int)(e % k), k);
    lit_t[d] = lits[e];
    eta_t[d] = eta[e];
  }
}

__global__ void sp_untile_kernel(long long ne, int k,
                                 const double* __restrict__ eta_t,
                                 double* eta) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (long long)gridDim.x * blockDim.x)
    eta[e] = eta_t[sp_tile(e / k, (int)(e % k), k)];
}

// Interior window bounds of the variable pass: seg[(w-1) n + i] = first
// occurrence of variable i whose edge is >= w * wsize (lists sorted by edge;
// a list that is not sets *unsorted and the caller runs one window)
__global__ void sp_window_kernel(int n, int nwin, long long wsize,
                                 const int* __restrict__ occ_row,
                                 const int* __restrict__ occ, int* seg,
                                 int* unsorted) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = occ_row[i], e = occ_row[i + 1];
    bool ok = true;
    for (int t = s + 1; t < e; ++t) ok &= occ[t - 1] <= occ[t];
    if (!ok) atomicOr(unsorted, 1);
    int lo = s;
    for (int w = 1; w < nwin; ++w) {
      const long long b = (long long)w * wsize;
      int hi = e;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (occ[mid] < b) lo = mid + 1; else hi = mid;
      }
      seg[(long long)(w - 1) * n + i] = lo;
    }
  }
}

#ifndef DP_SP_WINDOW_MB
#define DP_SP_WINDOW_MB 0  // eta slice per variable pass (0: one pass; see apps.cuh)
#endif

// W+ = Pi+ / (Pi+ + Pi- + Pi0), W- likewise, with P+ / P- the products of
// (1 - eta) over the positive / negative occurrences:
// Pi+ = (1 - P+) P-, Pi- = (1 - P-) P+, Pi0 = P+ P-.
__global__ void sp_bias_kernel(int n, const SpVarProd* __restrict__ prod,
                               float* wpos, float* wneg) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const SpVarProd q = prod[i];
    const double pp = q.z[0] == 0 ? q.p[0] : 0.0;
    const double pn = q.z[1] == 0 ? q.p[1] : 0.0;
    const double ip = __dmul_rn(__dsub_rn(1.0, pp), pn);
    const double in = __dmul_rn(__dsub_rn(1.0, pn), pp);
    const double i0 = __dmul_rn(pp, pn);
    const double den = __dadd_rn(__dadd_rn(ip, in), i0);
    wpos[i] = den > 0.0 ? __double2float_rn(__ddiv_rn(ip, den)) : 0.f;
    wneg[i] = den > 0.0 ? __double2float_rn(__ddiv_rn(in, den)) : 0.f;
  }
}

int sp_dev_impl(const int32_t* lits, int32_t k, int32_t nclauses,
                const int32_t* occ_row, const int32_t* occ, int32_t nvars,
                int32_t max_sweeps, float eps, const dp_config* c,
                double* eta, float* wpos, float* wneg, int32_t* sweeps_done,
                float* last_delta, cudaStream_t s, dp_stats* st) {
  int r;
  if ((r = validate(c))) return r;
  if (k < 1 || k > 32 || nclauses < 0 || nvars < 0 || max_sweeps < 0)
    return fail(DP_ERR_INVALID, "bad formula size");
  Workspace* w = workspace(&r);
  if (!w) return r;
  const long long ne = (long long)nclauses * k;
  if (ne >= (1LL << 30)) return fail(DP_ERR_INVALID, "too many edges");
  // L2 windows of the variable pass's eta gather
  long long win_mb = DP_SP_WINDOW_MB;
  if (const char* env = std::getenv("DYNPAR_SP_WINDOW_MB"))  // A/B; 0: off
    win_mb = std::atoll(env);
  int nwin = win_mb > 0 ? (int)std::min<long long>(
                              16, std::max<long long>(
                                      1, dp::ceil_div_ll(ne * 8, win_mb << 20)))
                        : 1;
  // prod[nvars] | eta_t x 2 [nt] | ratio[nt] | lit_t[nt] | occs[ne] |
  // seg[nwin-1][nv]; nt = the clause-tiled size (clauses padded to 32)
  const size_t nv = (size_t)std::max(nvars, 1);
  const size_t nes = (size_t)std::max(ne, 1LL);
  const size_t nt = (size_t)std::max(
      dp::ceil_div_ll(std::max(nclauses, 1), 32) * 32 * k, 1LL);
  if ((r = grow(&w->io[5], &w->io_bytes[5],
                nv * sizeof(SpVarProd) + nt * (8 + 8 + 8 + 4) + nes * 4 +
                    (size_t)(nwin - 1) * nv * 4)))
    return r;
  SpVarProd* prod = (SpVarProd*)w->io[5];
  double* eta_a = (double*)(prod + nv);
  double* eta_b = eta_a + nt;
  double* ratio = eta_b + nt;
  int* lit_t = (int*)(ratio + nt);
  int* occs = lit_t + nt;
  int* seg = occs + nes;
  long long lv = 0;
  if (c->variant == DP_VARIANT_CDP &&
      (r = count_launchers(w, c, occ_row, nvars, 0, s, &lv)))
    return r;
  // clause children (k each) launch when k >= T
  const long long lc = effective_threshold(c) <= k ? nclauses : 0;
  if ((r = ensure_pending_limit(w, c,
                                std::max(launch_bound(c, nvars, lv),
                                         launch_bound(c, nclauses, lc)))))
    return r;
  if ((r = begin_run(w, s))) return r;
  const int vb = std::max(1, std::min(dp::ceil_div(std::max(nvars, 1), 256),
                                      148 * 8));
  RunCounters rc;
  DP_CUDA(cudaEventRecord(w->ev0, s));
  const int eb = (int)std::min<long long>(
      dp::ceil_div_ll(std::max(ne, 1LL), 256), 148 * 8);
  if (ne) {
    sp_pack_kernel<<<eb, 256, 0, s>>>(ne, k, occ, lits, occs);
    DP_CUDA(cudaGetLastError());
    sp_tile_kernel<<<eb, 256, 0, s>>>(ne, k, lits, eta, lit_t, eta_a);
    DP_CUDA(cudaGetLastError());
    rc.kernel_launches += 2;
  }
  // window bounds on 32-clause tile boundaries: edge e < w * wsize exactly
  // when its tiled index is below the window's tiled start
  const long long wsize =
      dp::ceil_div_ll(dp::ceil_div_ll(std::max(nclauses, 1), 32), nwin) * 32 *
      k;
  if (nwin > 1) {
    DP_CUDA(cudaMemsetAsync(&w->ds->flag[1], 0, sizeof(int), s));
    sp_window_kernel<<<vb, 256, 0, s>>>(nvars, nwin, wsize, occ_row, occ, seg,
                                        &w->ds->flag[1]);
    DP_CUDA(cudaGetLastError());
    rc.kernel_launches += 1;
    if ((r = read_state_fast(w, s))) return r;
    if (w->h_ds->flag[1]) nwin = 1;  // caller's lists not sorted by edge
  }
  double* cur = eta_a;
  double* nxt = eta_b;
  int sweeps = 0;
  float delta = 0.f;
  auto var_pass = [&](const double* e) -> int {
    sp_reset_kernel<<<vb, 256, 0, s>>>(nvars, prod);
    DP_CUDA(cudaGetLastError());
    rc.kernel_launches += 1;
    for (int win = 0; win < nwin; ++win) {
      SpVarApp va;
      va.seg_lo = win == 0 ? occ_row : seg + (size_t)(win - 1) * nv;
      va.seg_hi = win == nwin - 1 ? occ_row + 1 : seg + (size_t)win * nv;
      va.occs = occs;
      va.eta = e;
      va.prod = prod;
      va.nvars = nvars;
      va.pad = 0;
      const int r2 = launch_parent(va, nvars, lv, c, w, s, &rc);
      if (r2) return r2;
    }
    return 0;
  };
  while (sweeps < max_sweeps) {
    if ((r = var_pass(cur))) return r;
    SpRatioApp ra;
    ra.lit = lit_t;
    ra.eta = cur;
    ra.prod = prod;
    ra.ratio = ratio;
    ra.nclauses = nclauses;
    ra.k = k;
    if ((r = launch_parent(ra, nclauses, lc, c, w, s, &rc))) return r;
    DP_CUDA(cudaMemsetAsync(&w->ds->flag[0], 0, sizeof(int), s));
    SpClauseApp ca;
    ca.ratio = ratio;
    ca.eta = cur;
    ca.eta_next = nxt;
    ca.max_delta = (unsigned*)&w->ds->flag[0];
    ca.nclauses = nclauses;
    ca.k = k;
    if ((r = launch_parent(ca, nclauses, lc, c, w, s, &rc))) return r;
    if ((r = read_state_fast(w, s))) return r;
    std::swap(cur, nxt);
    ++sweeps;
    std::memcpy(&delta, &w->h_ds->flag[0], sizeof(float));
    if (delta <= eps) break;
  }
  // biases from the final surveys
  if ((r = var_pass(cur))) return r;
  sp_bias_kernel<<<vb, 256, 0, s>>>(nvars, prod, wpos, wneg);
  DP_CUDA(cudaGetLastError());
  rc.kernel_launches += 1;
  if (ne) {
    sp_untile_kernel<<<eb, 256, 0, s>>>(ne, k, cur, eta);
    DP_CUDA(cudaGetLastError());
    rc.kernel_launches += 1;
  }
  DP_CUDA(cudaEventRecord(w->ev1, s));
  DP_CUDA(cudaEventSynchronize(w->ev1));
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  if ((r = read_state(w, s))) return r;
  rc.ms_kernel_sum = rc.ms_kernel_max = ms;
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = sweeps;
  if (sweeps_done) *sweeps_done = sweeps;
  if (last_delta) *last_delta = delta;
  return 0;
}

// single host launch apps
template <class App>
int once(Workspace* w, const dp_config* c, const App& app, long long nparents,
         long long launchers, cudaStream_t s, dp_stats* st) {
  RunCounters rc;
  int r;
  if ((r = ensure_pending_limit(w, c, launch_bound(c, nparents, launchers))))
    return r;
  if ((r = begin_run(w, s))) return r;
  DP_CUDA(cudaEventRecord(w->ev0, s));
  if ((r = launch_parent(app, nparents, launchers, c, w, s, &rc))) return r;
  DP_CUDA(cudaEventRecord(w->ev1, s));
  DP_CUDA(cudaEventSynchronize(w->ev1));
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  if ((r = read_state(w, s))) return r;
  if ((r = account_step(w, &rc))) return r;
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = 1;
  return 0;
}

int manylaunch_dev_impl(const int32_t* sizes, int32_t n, const dp_config* c,
                        int32_t* out, int32_t* total, cudaStream_t s,
                        dp_stats* st) {
  int r;
  if ((r = validate(c))) return r;
  if (n < 0) return fail(DP_ERR_INVALID, "negative size");
  Workspace* w = workspace(&r);
  if (!w) return r;
  if (n) DP_CUDA(cudaMemsetAsync(out, 0, (size_t)n * sizeof(int), s));
  DP_CUDA(cudaMemsetAsync(total, 0, sizeof(int), s));
  ManyLaunchApp a;
  a.sizes = sizes;
  a.out = out;
  a.total = total;
  a.n = n;
  a.pad = 0;
  long long launchers = 0;
  if (c->variant == DP_VARIANT_CDP &&
      (r = count_launchers(w, c, sizes, n, 1, s, &launchers)))
    return r;
  return once(w, c, a, n, launchers, s, st);
}

// ---------------------------------------------------------------------------
// TC: the transpose of the oriented CSR+ (in-lists over the shard's edge
// range), built on the device at the start of every call: count, exclusive
// scan, scatter.  In-list order is the scatter's (irrelevant: in-lists are
// only iterated, the probed / merged out-lists stay sorted).
// ---------------------------------------------------------------------------
// In-degrees of the oriented graph.  Edges point to the higher-ranked
// (higher-degree) end, so the top ranks (the hubs) collect most of them and
// their counters serialise at one L2 slice each (1.35 ms of RMAT-22's TC
// for 63 M edges; merging equal heads within a warp did not help -- a row's
// heads are distinct).  Each block counts heads in the top kTcHub ranks in
// shared memory and adds them to the global counters once.
constexpr int kTcHub = 4096;

__global__ void tc_count_in_kernel(const int* __restrict__ col, long long lo,
                                   long long hi, int n, int* cnt) {
  __shared__ int hist[kTcHub];
  const int h0 = n > kTcHub ? n - kTcHub : 0;  // hub ranks [h0, n)
  for (int i = threadIdx.x; i < kTcHub; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (long long e = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
       e < hi; e += (long long)gridDim.x * blockDim.x) {
    const int v = ld_stream(col + e);
    if (v >= h0)
      atomicAdd(hist + (v - h0), 1);
    else
      atomicAdd(cnt + v, 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kTcHub; i += blockDim.x)
    if (hist[i]) atomicAdd(cnt + h0 + i, hist[i]);
}

// exclusive scan of x[0, n) into y[0, n] (y[n] = total), three passes
constexpr int kScanTile = 4096;  // 1024 threads x 4

__global__ void __launch_bounds__(1024)
    scan_tiles_kernel(const int* __restrict__ x, long long n, int* y,
                      long long* tile_sum) {
  __shared__ int wsum[32];
  const long long base = (long long)blockIdx.x * kScanTile + threadIdx.x * 4;
  int v[4], t = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[j] = base + j < n ? x[base + j] : 0;
    t += v[j];
  }
  const int incl = warp_incl_scan(t);
  if (lane_id() == 31) wsum[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int ws = wsum[threadIdx.x];
    const int wi = warp_incl_scan(ws);
    wsum[threadIdx.x] = wi - ws;
    if (threadIdx.x == 31) tile_sum[blockIdx.x] = wi;
  }
  __syncthreads();
  int run = wsum[threadIdx.x >> 5] + incl - t;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (base + j < n) y[base + j] = run;
    run += v[j];
  }
}

__global__ void __launch_bounds__(1024)
    scan_sums_kernel(long long* tile_sum, int ntiles, int* y, long long n) {
  // one block: exclusive scan of the tile sums in place, y[n] = total
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < ntiles; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const long long v = i < ntiles ? tile_sum[i] : 0;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(DP_FULL, x, o);
      if (lane_id() >= o) x += t;
    }
    __shared__ long long ws[32];
    if (lane_id() == 31) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      long long a = ws[threadIdx.x];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(DP_FULL, a, o);
        if (lane_id() >= o) a += t;
      }
      ws[threadIdx.x] = a;
    }
    __syncthreads();
    const long long before = (threadIdx.x >= 32 ? ws[(threadIdx.x >> 5) - 1] : 0);
    const long long c = carry;
    if (i < ntiles) tile_sum[i] = c + before + x - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c + before + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) y[n] = (int)carry;
}

__global__ void scan_add_kernel(int* y, int* y2, long long n,
                                const long long* tile_sum) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int v = y[i] + (int)tile_sum[i / kScanTile];
    y[i] = v;
    y2[i] = v;
  }
}

// warp per source vertex: its out-edges in [lo, hi) land in the in-lists.
// In-edge (u -> v) at slot i records the slots of N+(u) above v, [i + 1,
// rowptr[u + 1]) (the rank-ordered CSR+ keeps rows ascending, so these are
// exactly the w > v that can close a triangle at v)
// One in-edge per lane of the row's warp, placed with an atomic cursor.
// Measured alternatives (profiles/r02/ab_tc_transpose_r02.txt): privatising
// the hub cursors in shared memory (2.01 vs 1.77 ms) and edge-balanced
// warp-flattened rows (2.44 ms) were slower -- the kernel is bound by the
// 8-byte scattered in_rng writes, not by the cursor atomics -- and so was
// placing the heads in L2-sized passes (15.5-21.8 vs 14.05 ms for the whole
// TC, ab_tc_window_r02.txt: each pass re-reads col).
__global__ void tc_scatter_in_kernel(const int* __restrict__ rowptr,
                                     const int* __restrict__ col, int n,
                                     long long lo, long long hi, int* cursor,
                                     int2* in_rng) {
  const int lane = lane_id();
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
       u < n; u += warps) {
    const int end = __ldg(rowptr + u + 1);
    long long b = __ldg(rowptr + u), e = end;
    if (b < lo) b = lo;
    if (e > hi) e = hi;
    for (long long i = b + lane; i < e; i += 32)
      in_rng[atomicAdd(cursor + __ldg(col + i), 1)] =
          make_int2((int)i + 1, end);
  }
}

int tc_dev_impl(const int32_t* rowptr, const int32_t* col, int32_t n,
                int64_t m, int64_t lo, int64_t hi, const dp_config* c,
                uint64_t* tri, cudaStream_t s, dp_stats* st) {
  int r;
  if ((r = validate(c))) return r;
  if (n < 0 || m < 0) return fail(DP_ERR_INVALID, "negative size");
  if (lo < 0) lo = 0;
  if (hi > m) hi = m;
  if (hi < lo) hi = lo;
  Workspace* w = workspace(&r);
  if (!w) return r;
  // tile sums | in_rng[hi-lo] | in_rowptr[n+1] | cursor[n+1]
  const long long ntiles = std::max(1LL, dp::ceil_div_ll(n, kScanTile));
  const size_t need = (size_t)(n + 1) * 8 +
                      (size_t)std::max<long long>(hi - lo, 1) * 8 +
                      (size_t)ntiles * 8 + 16;
  if ((r = grow(&w->io[5], &w->io_bytes[5], need))) return r;
  long long* tile_sum = (long long*)w->io[5];
  int2* in_rng = (int2*)(tile_sum + ntiles);  // 8-byte aligned
  int* in_rowptr = (int*)(in_rng + std::max<long long>(hi - lo, 1));
  int* cursor = in_rowptr + (n + 1);
  RunCounters rc;
  DP_CUDA(cudaMemsetAsync(tri, 0, sizeof(uint64_t), s));
  DP_CUDA(cudaEventRecord(w->ev0, s));
  const int gb = 148 * 8;
  DP_CUDA(cudaMemsetAsync(cursor, 0, (size_t)(n + 1) * 4, s));
  if (hi > lo)
    tc_count_in_kernel<<<gb, 256, 0, s>>>(col, lo, hi, n, cursor);
  scan_tiles_kernel<<<(int)ntiles, 1024, 0, s>>>(cursor, n, in_rowptr,
                                                 tile_sum);
  scan_sums_kernel<<<1, 1024, 0, s>>>(tile_sum, (int)ntiles, in_rowptr, n);
  scan_add_kernel<<<gb, 256, 0, s>>>(in_rowptr, cursor, n, tile_sum);
  if (hi > lo)
    tc_scatter_in_kernel<<<gb, 256, 0, s>>>(rowptr, col, n, lo, hi, cursor,
                                            in_rng);
  DP_CUDA(cudaGetLastError());
  rc.kernel_launches += 5;
  TcApp a;
  a.rowptr = rowptr;
  a.col = col;
  a.in_rowptr = in_rowptr;
  a.in_rng = in_rng;
  a.total = (unsigned long long*)tri;
  a.n = n;
  a.pad = 0;
  long long launchers = 0;
  if (c->variant == DP_VARIANT_CDP &&
      (r = count_launchers(w, c, in_rowptr, n, 0, s, &launchers)))
    return r;
  if ((r = ensure_pending_limit(w, c, launch_bound(c, n, launchers))))
    return r;
  if ((r = begin_run(w, s))) return r;
  if ((r = launch_parent(a, n, launchers, c, w, s, &rc))) return r;
  DP_CUDA(cudaEventRecord(w->ev1, s));
  DP_CUDA(cudaEventSynchronize(w->ev1));
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  if ((r = read_state(w, s))) return r;
  if ((r = account_step(w, &rc))) return r;
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = 1;
  return 0;
}

int bt_dev_impl(const float* cp, int32_t ncurves, int32_t max_tess,
                float scale, const dp_config* c, int32_t* ntess,
                int64_t* offsets, float* verts, int64_t cap, int64_t* nverts,
                cudaStream_t s, dp_stats* st) {
  int r;
  if ((r = validate(c))) return r;
  if (ncurves < 0) return fail(DP_ERR_INVALID, "negative curve count");
  if (max_tess < 4) return fail(DP_ERR_INVALID, "max_tess must be >= 4");
  Workspace* w = workspace(&r);
  if (!w) return r;
  DP_CUDA(cudaMemsetAsync(w->d_scratch, 0, sizeof(unsigned long long), s));
  DP_CUDA(cudaMemsetAsync(w->d_flag, 0, sizeof(int), s));
  BtApp a;
  a.cp = (const float2*)cp;
  a.ntess = ntess;
  a.offsets = (long long*)offsets;
  a.verts = (float2*)verts;
  a.cursor = w->d_scratch;
  a.overflow = w->d_flag;
  a.cap = cap;
  a.ncurves = ncurves;
  a.max_tess = max_tess;
  a.scale = scale;
  a.pad = 0;
  // every curve owns 4..max_tess vertices
  const long long launchers = effective_threshold(c) <= max_tess ? ncurves : 0;
  if ((r = once(w, c, a, ncurves, launchers, s, st))) return r;
  int ovf = 0;
  unsigned long long used = 0;
  DP_CUDA(cudaMemcpyAsync(&used, w->d_scratch, sizeof(used),
                          cudaMemcpyDeviceToHost, s));
  DP_CUDA(cudaMemcpyAsync(&ovf, w->d_flag, sizeof(int), cudaMemcpyDeviceToHost,
                          s));
  DP_CUDA(cudaStreamSynchronize(s));
  if (nverts) *nverts = (int64_t)used;
  if (ovf)
    return fail(DP_ERR_INVALID, "vertex capacity exceeded: need " +
                                    std::to_string(used) + " vertices");
  return 0;
}

__global__ void bfs_part_apply_kernel(const int* __restrict__ recv,
                                      long long nrecv, int nparts, int level,
                                      int* dist, int* changed) {
  int c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
       i < nrecv; i += (long long)gridDim.x * blockDim.x) {
    const int lv = local_of(__ldg(recv + i), nparts);
    if (__ldcg(dist + lv) == kUnreached &&
        atomicCAS(dist + lv, kUnreached, level + 1) == kUnreached)
      c = 1;
  }
  if (__any_sync(DP_FULL, c) && lane_id() == 0) *changed = 1;
}

int bfs_part_level_impl(const int32_t* rowptr, const int32_t* col,
                        int32_t n_local, int32_t nparts, int32_t part,
                        int32_t level, const dp_config* c, int32_t* dist,
                        int32_t* counts, uint32_t* sent, int32_t* send_buf,
                        int64_t stride, int32_t* send_count, int32_t* changed,
                        cudaStream_t s, dp_stats* st,
                        int32_t* const* peer_dist = nullptr) {
  int r;
  if ((r = validate(c))) return r;
  if (nparts < 1 || part < 0 || part >= nparts || n_local < 0 || level < 0)
    return fail(DP_ERR_INVALID, "bad partition arguments");
  Workspace* w = workspace(&r);
  if (!w) return r;
  long long launchers = 0;
  if (c->variant == DP_VARIANT_CDP &&
      (r = count_launchers(w, c, rowptr, n_local, 0, s, &launchers)))
    return r;
  if ((r = ensure_pending_limit(w, c, launch_bound(c, n_local, launchers))))
    return r;
  if ((r = begin_run(w, s))) return r;
  if (peer_dist)  // fused exchange: the flag is this level's alone
    DP_CUDA(cudaMemsetAsync(changed, 0, sizeof(int), s));
  auto fill = [&](auto& a) {
    a.rowptr = rowptr;
    a.col = col;
    a.dist = dist;
    a.counts = counts;
    a.sent = sent;
    a.send_buf = send_buf;
    a.send_count = send_count;
    a.changed = changed;
    a.peer_dist = (int* const*)peer_dist;
    a.remote_ops = &w->ds->remote;
    a.stride = stride;
    a.n_local = n_local;
    a.nparts = nparts;
    a.part = part;
    a.level = level;
    a.cmask = c->counts_spread > 0 ? (unsigned)((1ull << c->counts_spread) - 1)
                                   : 0u;
    a.pad_ = 0;
  };
  RunCounters rc;
  DP_CUDA(cudaEventRecord(w->ev0, s));
  if (peer_dist) {
    BfsPeerApp a;
    fill(a);
    if ((r = launch_parent(a, n_local, launchers, c, w, s, &rc))) return r;
  } else {
    BfsPartApp a;
    fill(a);
    if ((r = launch_parent(a, n_local, launchers, c, w, s, &rc))) return r;
  }
  DP_CUDA(cudaEventRecord(w->ev1, s));
  if ((r = read_state_fast(w, s))) return r;
  if ((r = account_step(w, &rc))) return r;
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = 1;
  return 0;
}

__global__ void sssp_part_apply_kernel(const unsigned long long* __restrict__ recv,
                                       long long nrecv, int nparts, int* dist,
                                       int* changed) {
  int c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
       i < nrecv; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long p = __ldg(recv + i);
    const int lv = local_of((int)(p >> 32), nparts);
    const int alt = (int)(unsigned)(p & 0xffffffffull);
    if (alt < __ldcg(dist + lv) && atomicMin(dist + lv, alt) > alt) c = 1;
  }
  if (__any_sync(DP_FULL, c) && lane_id() == 0) *changed = 1;
}

// One round of the fused-exchange partitioned SSSP (SsspPeerApp).
int sssp_peer_round_impl(const int32_t* rowptr, const int32_t* col,
                         const int32_t* weight, int32_t n_local,
                         int32_t nparts, int32_t part, const dp_config* c,
                         int32_t* dist, int32_t* const* peer_dist,
                         int32_t* best, int32_t* changed, cudaStream_t s,
                         dp_stats* st) {
  int r;
  if ((r = validate(c))) return r;
  if (nparts < 1 || part < 0 || part >= nparts || n_local < 0 || !peer_dist ||
      !dist)
    return fail(DP_ERR_INVALID, "bad partition arguments");
  Workspace* w = workspace(&r);
  if (!w) return r;
  long long launchers = 0;
  if (c->variant == DP_VARIANT_CDP &&
      (r = count_launchers(w, c, rowptr, n_local, 0, s, &launchers)))
    return r;
  if ((r = ensure_pending_limit(w, c, launch_bound(c, n_local, launchers))))
    return r;
  if ((r = begin_run(w, s))) return r;
  SsspPeerApp a;
  a.rowptr = rowptr;
  a.col = col;
  a.weight = weight;
  a.peer_dist = (int* const*)peer_dist;
  a.my_dist = dist;
  a.best = best;
  a.changed = changed;
  a.remote_ops = &w->ds->remote;
  DP_CUDA(cudaMemsetAsync(changed, 0, sizeof(int), s));  // this round's flag
  a.n_local = n_local;
  a.nparts = nparts;
  a.part = part;
  a.pad = 0;
  RunCounters rc;
  DP_CUDA(cudaEventRecord(w->ev0, s));
  if ((r = launch_parent(a, n_local, launchers, c, w, s, &rc))) return r;
  DP_CUDA(cudaEventRecord(w->ev1, s));
  if ((r = read_state_fast(w, s))) return r;
  if ((r = account_step(w, &rc))) return r;
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = 1;
  return 0;
}

// ---------------------------------------------------------------------------
// Partitioned solves with the round loop in the library (one part per host
// thread or process).  Per round: the part's parent grid (+ children, the
// exchange fused in as remote atomics), then one warp ORs the round flags of
// all parts through their signal slots -- no NCCL call, no per-round Python:
// the host loop is the single-GPU iterate() plus one tiny kernel.
//
// Signal slots: part q owns uint64 slots[2 * nparts] in memory every part can
// address (torch symmetric memory across GPUs; plain device memory when the
// parts share a GPU); peer_sig[q] points at part q's.  Exchange index i (0:
// the barrier after the parts initialised their dist, round r: r + 1) stores
// tag(epoch, i, bit) into slot [(i & 1) * nparts + part] of every part
// (st.release.sys) and waits until its own row (i & 1) holds index i's tag
// from every part (ld.acquire.sys).  A part cannot get two indices ahead of
// another (it would need that part's tag for the index in between), so two
// rows suffice; the caller's epoch (equal on every part, unique per call, >
// 0) keeps an earlier call's tags from matching.  The release orders the
// round's remote atomics (fenced system-wide by the warps that issued them)
// before the tag, so once every tag is in, every lowering of the round is
// visible to its owner.
// ---------------------------------------------------------------------------
constexpr int kErrPeerTimeout = 0x7fff0001;  // DevState::err marker

__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p,
                                                   unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v)
               : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(
    const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];"
               : "=l"(v)
               : "l"(p)
               : "memory");
  return v;
}

// one warp; flag_slot < 0: a pure barrier.  Each tag carries two bits: the
// round's `changed` flag and (partitioned BFS) whether the part's next
// frontier holds a launching row; both are OR-ed over the parts.
__global__ void part_flag_or_kernel(unsigned long long* const* peer_sig,
                                    int nparts, int part, long long idx,
                                    unsigned long long epoch, DevState* ds,
                                    int flag_slot,
                                    unsigned long long timeout_ns) {
  const int lane = threadIdx.x;
  const unsigned bits =
      flag_slot >= 0
          ? (ds->flag[flag_slot] != 0 ? 1u : 0u) | (ds->big_local ? 2u : 0u)
          : 0u;
  const unsigned long long key =
      (epoch << 32) | (unsigned long long)(idx + 1);  // tag >> 2
  const long long row = (idx & 1) * nparts;
  for (int q = lane; q < nparts; q += 32)
    st_release_sys_u64(peer_sig[q] + row + part, (key << 2) | bits);
  unsigned any = 0;
  const unsigned long long t0 = globaltimer_ns();
  bool timed_out = false;
  for (int q = lane; q < nparts && !timed_out; q += 32) {
    unsigned long long v;
    while (((v = ld_acquire_sys_u64(peer_sig[part] + row + q)) >> 2) != key) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        timed_out = true;
        break;
      }
      __nanosleep(64);
    }
    any |= (unsigned)(v & 3);
  }
  if (timed_out) atomicCAS(&ds->err, 0, kErrPeerTimeout);
  any = __reduce_or_sync(DP_FULL, any);
  if (lane == 0 && flag_slot >= 0) {
    ds->flag[flag_slot] = any & 1;  // the OR over the parts: what the host reads
    ds->flag[flag_slot ^ 1] = 0;    // the next round's own flag
    ds->big[flag_slot ^ 1] = (any >> 1) & 1;  // the next level's variant
    ds->big_local = 0;
  }
}

// partitioned BFS: does this part's next frontier (owned u with dist[u] ==
// level) hold a row that would launch (degree >= t)?  -> DevState::big_local
__global__ void part_big_kernel(const int* __restrict__ rowptr,
                                const int* __restrict__ dist, int n_local,
                                int level, int t, DevState* ds) {
  // warp-uniform trip count; stops as soon as any warp has found one (the
  // levels that need the launching variant end the scan early)
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long u0 = (long long)blockIdx.x * blockDim.x + threadIdx.x -
                       lane_id();
  for (long long b = u0, i = 0; b < n_local; b += stride, ++i) {
    if ((i & 7) == 0 && __ldcg(&ds->big_local)) return;
    const long long u = b + lane_id();
    bool found = false;
    if (u < n_local && __ldcg(dist + u) == level) {
      const int d = __ldg(rowptr + u + 1) - __ldg(rowptr + u);
      found = d > 0 && d >= t;
    }
    if (__any_sync(DP_FULL, found)) {
      if (lane_id() == 0) ds->big_local = 1;
      return;
    }
  }
}

unsigned long long peer_timeout_ns() {
  static const unsigned long long t = [] {
    const char* e = std::getenv("DYNPAR_PEER_TIMEOUT_MS");
    const long long ms = e ? std::atoll(e) : 60000;
    return (unsigned long long)std::max<long long>(ms, 1) * 1000000ull;
  }();
  return t;
}

struct PartSync {
  unsigned long long* const* sig;
  int nparts, part;
  unsigned long long epoch;
};

// iterate() for one part: rounds until no part changed anything
template <class MakeApp>
int iterate_parts(Workspace* w, const dp_config* c, long long nparents,
                  long long launchers, int max_iter, cudaStream_t s,
                  const PartSync& ps, MakeApp make, dp_stats* st,
                  const int* big_rowptr = nullptr,
                  const int* big_dist = nullptr) {
  // big_rowptr / big_dist (partitioned BFS): after each level the part scans
  // its next frontier for a launching row; when no part has one, the next
  // level runs the launch-free parent variant (as iterate() does for BFS)
  const bool per_level = big_rowptr && c->variant == DP_VARIANT_CDP;
  dp_config c_flat = *c;
  c_flat.variant = DP_VARIANT_NOCDP;
  RunCounters rc;
  int r;
  if ((r = ensure_pending_limit(w, c, launch_bound(c, nparents, launchers))))
    return r;
  // grow every buffer a round can need BEFORE the barrier: the cudaFree in
  // grow() synchronises the device, i.e. would wait on parts that already
  // spin in the barrier for this one
  {
    using App = decltype(make(0, w->ds));
    const long long wave = std::min(wave_parents(c, nparents, launchers),
                                    nparents);
    AggTables<App> t{nullptr, nullptr, nullptr, nullptr};
    if ((r = prepare_tables<App>(
             c, (int)dp::ceil_div_ll(wave, c->parent_block), c->parent_block,
             w, s, &t)))
      return r;
  }
  if ((r = begin_run(w, s))) return r;
  DP_CUDA(cudaEventRecord(w->ev0, s));
  const unsigned long long tmo = peer_timeout_ns();
  // every part has initialised its dist before any remote write lands
  part_flag_or_kernel<<<1, 32, 0, s>>>(ps.sig, ps.nparts, ps.part, 0,
                                       ps.epoch, w->ds, -1, tmo);
  DP_CUDA(cudaGetLastError());
  int it = 0;
  bool converged = false;
  for (; !converged && it <= max_iter; ++it) {
    auto app = make(it, w->ds);
    const dp_config* cl =
        per_level && it > 0 && w->h_ds->big[it & 1] == 0 ? &c_flat : c;
    if ((r = launch_parent(app, nparents, launchers, cl, w, s, &rc))) return r;
    if (per_level) {
      part_big_kernel<<<148 * 4, 256, 0, s>>>(
          big_rowptr, big_dist, (int)nparents, it + 1, effective_threshold(c),
          w->ds);
      rc.kernel_launches += 1;
    }
    part_flag_or_kernel<<<1, 32, 0, s>>>(ps.sig, ps.nparts, ps.part, it + 1,
                                         ps.epoch, w->ds, it & 1, tmo);
    DP_CUDA(cudaGetLastError());
    rc.kernel_launches += 1;
    if ((r = read_state_fast(w, s))) return r;
    if ((r = account_step(w, &rc))) return r;
    if (w->h_ds->flag[it & 1] == 0) {
      converged = true;
      ++it;
      break;
    }
  }
  DP_CUDA(cudaEventRecord(w->ev1, s));
  DP_CUDA(cudaEventSynchronize(w->ev1));
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  if ((r = read_state(w, s))) return r;
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = it;
  if (!converged)
    return fail(DP_ERR_ITERATIONS, "used more iterations than vertices");
  return 0;
}

int check_part_args(const dp_config* c, int32_t n_local, int32_t n_global,
                    int32_t nparts, int32_t part, int32_t src,
                    const void* peer_dist, const void* peer_sig,
                    uint64_t epoch) {
  int r;
  if ((r = validate(c))) return r;
  if (nparts < 1 || part < 0 || part >= nparts || n_local < 0 ||
      n_global < 1 || src < 0 || src >= n_global || !peer_dist ||
      !peer_sig || epoch == 0 || epoch >= (1ull << 31) ||
      (long long)n_local != ((long long)n_global - part + nparts - 1) / nparts)
    return fail(DP_ERR_INVALID, "bad partition arguments");
  return 0;
}

__global__ void part_init_kernel(int* dist, int n_local, int src_local,
                                 int* best, int n_global) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
       i < n_global || i < n_local; i += (long long)gridDim.x * blockDim.x) {
    if (i < n_local) dist[i] = i == src_local ? 0 : kUnreached;
    if (best && i < n_global) best[i] = kUnreached;
  }
}

int sssp_part_solve_peer_impl(const int32_t* rowptr, const int32_t* col,
                              const int32_t* weight, int32_t n_local,
                              int32_t n_global, int32_t nparts, int32_t part,
                              int32_t src, const dp_config* c, int32_t* dist,
                              int32_t* const* peer_dist, int32_t* best,
                              uint64_t* const* peer_sig, uint64_t epoch,
                              cudaStream_t s, dp_stats* st) {
  int r;
  if ((r = check_part_args(c, n_local, n_global, nparts, part, src, peer_dist,
                           peer_sig, epoch)))
    return r;
  if (!dist || !best) return fail(DP_ERR_INVALID, "null buffer");
  Workspace* w = workspace(&r);
  if (!w) return r;
  const int src_local = src % nparts == part
                            ? src / nparts : -1;
  part_init_kernel<<<148 * 4, 256, 0, s>>>(dist, n_local, src_local, best,
                                           n_global);
  DP_CUDA(cudaGetLastError());
  // every part uses the same worst-case launcher count, so every part sizes
  // the device-wide launch pool alike (no part grows it while another waits
  // in the barrier); cf_wave's solo launches are off here: with that bound
  // they would split every round into waves
  const long long launchers = n_local;
  dp_config cs = *c;
  cs.cf_wave = 0;
  c = &cs;
  const PartSync ps{(unsigned long long* const*)peer_sig, nparts, part,
                    epoch};
  return iterate_parts(w, c, n_local, launchers, n_global, s, ps,
                       [&](int round, DevState* ds) {
                         SsspPeerApp a;
                         a.rowptr = rowptr;
                         a.col = col;
                         a.weight = weight;
                         a.peer_dist = (int* const*)peer_dist;
                         a.my_dist = dist;
                         a.best = best;
                         a.changed = &ds->flag[round & 1];
                         a.remote_ops = &ds->remote;
                         a.n_local = n_local;
                         a.nparts = nparts;
                         a.part = part;
                         a.pad = 0;
                         return a;
                       },
                       st);
}

int bfs_part_solve_peer_impl(const int32_t* rowptr, const int32_t* col,
                             int32_t n_local, int32_t n_global, int32_t nparts,
                             int32_t part, int32_t src, const dp_config* c,
                             int32_t* dist, int32_t* const* peer_dist,
                             int32_t* counts, int64_t counts_len,
                             uint32_t* sent, uint64_t* const* peer_sig,
                             uint64_t epoch, cudaStream_t s, dp_stats* st) {
  int r;
  if ((r = check_part_args(c, n_local, n_global, nparts, part, src, peer_dist,
                           peer_sig, epoch)))
    return r;
  const unsigned cmask = c->counts_spread > 0
                             ? (unsigned)((1ull << c->counts_spread) - 1)
                             : 0u;
  const long long need =
      cmask ? ((long long)n_global + cmask) / (cmask + 1) * (cmask + 1)
            : n_global;
  if (!dist || !counts || !sent || counts_len < need)
    return fail(DP_ERR_INVALID, "bad counts / sent buffers");
  Workspace* w = workspace(&r);
  if (!w) return r;
  const int src_local = src % nparts == part
                            ? src / nparts : -1;
  part_init_kernel<<<148 * 4, 256, 0, s>>>(dist, n_local, src_local, nullptr,
                                           0);
  DP_CUDA(cudaGetLastError());
  DP_CUDA(cudaMemsetAsync(counts, 0, (size_t)counts_len * sizeof(int), s));
  DP_CUDA(cudaMemsetAsync(sent, 0, (size_t)(n_global + 31) / 32 * 4, s));
  const long long launchers = n_local;
  dp_config cs = *c;  // as sssp_part_solve_peer_impl
  cs.cf_wave = 0;
  c = &cs;
  const PartSync ps{(unsigned long long* const*)peer_sig, nparts, part,
                    epoch};
  return iterate_parts(w, c, n_local, launchers, n_global, s, ps,
                       [&](int level, DevState* ds) {
                         BfsPeerApp a;
                         a.rowptr = rowptr;
                         a.col = col;
                         a.dist = dist;
                         a.counts = counts;
                         a.sent = sent;
                         a.send_buf = nullptr;
                         a.send_count = nullptr;
                         a.changed = &ds->flag[level & 1];
                         a.peer_dist = (int* const*)peer_dist;
                         a.remote_ops = &ds->remote;
                         a.stride = 0;
                         a.n_local = n_local;
                         a.nparts = nparts;
                         a.part = part;
                         a.level = level;
                         a.cmask = cmask;
                         a.pad_ = 0;
                         return a;
                       },
                       st, rowptr, dist);
}

int sssp_part_round_impl(const int32_t* rowptr, const int32_t* col,
                         const int32_t* weight, int32_t n_local,
                         int32_t nparts, int32_t part, const dp_config* c,
                         int32_t* dist, int32_t* best, uint64_t* send_buf,
                         const int64_t* send_off, int32_t* send_count,
                         int32_t* changed, cudaStream_t s, dp_stats* st) {
  int r;
  if ((r = validate(c))) return r;
  if (nparts < 1 || part < 0 || part >= nparts || n_local < 0)
    return fail(DP_ERR_INVALID, "bad partition arguments");
  Workspace* w = workspace(&r);
  if (!w) return r;
  long long launchers = 0;
  if (c->variant == DP_VARIANT_CDP &&
      (r = count_launchers(w, c, rowptr, n_local, 0, s, &launchers)))
    return r;
  if ((r = ensure_pending_limit(w, c, launch_bound(c, n_local, launchers))))
    return r;
  if ((r = begin_run(w, s))) return r;
  SsspPartApp a;
  a.rowptr = rowptr;
  a.col = col;
  a.weight = weight;
  a.dist = dist;
  a.best = best;
  a.send_buf = (unsigned long long*)send_buf;
  a.send_off = (const long long*)send_off;
  a.send_count = send_count;
  a.changed = changed;
  a.n_local = n_local;
  a.nparts = nparts;
  a.part = part;
  a.pad = 0;
  RunCounters rc;
  DP_CUDA(cudaEventRecord(w->ev0, s));
  if ((r = launch_parent(a, n_local, launchers, c, w, s, &rc))) return r;
  DP_CUDA(cudaEventRecord(w->ev1, s));
  if ((r = read_state_fast(w, s))) return r;
  if ((r = account_step(w, &rc))) return r;
  float ms = 0.f;
  DP_CUDA(cudaEventElapsedTime(&ms, w->ev0, w->ev1));
  finish_stats(w, rc, ms, st);
  if (st) st->iterations = 1;
  return 0;
}

// ---------------------------------------------------------------------------
// RMAT edge generation on the device: the same counter-based hash as the host
// generator (gen.cpp), so the CSR built from these keys is bit-identical.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long dmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void rmat_part_keys_kernel(unsigned long long key, long long m,
                                      int scale, int nparts, int part,
                                      unsigned long long* keys,
                                      unsigned long long* cursor) {
  const unsigned long long kA = 2448131358ull, kAB = 3264175144ull,
                           kABC = 4080218931ull;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // each warp takes 32 consecutive edges per trip (warp-uniform loop)
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x -
                     lane_id();
       b < m; b += stride) {
    const long long e = b + lane_id();
    unsigned s = 0, d = 0;
    if (e < m) {
      unsigned long long h = 0;
      for (int l = 0; l < scale; ++l) {
        unsigned r;
        if ((l & 1) == 0) {
          h = dmix64(key ^ ((unsigned long long)e * 16 + (unsigned)(l >> 1)));
          r = (unsigned)h;
        } else {
          r = (unsigned)(h >> 32);
        }
        s = (s << 1) | (r >= kAB);
        d = (d << 1) | ((r >= kA && r < kAB) || r >= kABC);
      }
    }
    const bool keep = e < m && (int)(s % nparts) == part;
    const unsigned mk = __ballot_sync(DP_FULL, keep);
    unsigned long long base = 0;
    if (lane_id() == 0 && mk) base = atomicAdd(cursor, (unsigned long long)__popc(mk));
    base = __shfl_sync(DP_FULL, base, 0);
    if (keep && keys)
      keys[base + __popc(mk & lanemask_lt())] =
          ((unsigned long long)(s / nparts) << 32) | d;
  }
}

__global__ void set_arrived_kernel(int* arrived, int k) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(arrived), "r"(k));
}

// Copy the edge arrays (same slot ranges of each) host -> device in chunks
// of 2^shift slots on the copy stream, after everything queued on s so far;
// chunk k's landing is published to the kernels (d_arrived = k + 1) and to
// the host (chunk_ev[k]).
int stage_chunked(Workspace* w, cudaStream_t s, int nsrc, const void* const* host,
                  void* const* dev, int64_t m, int shift, Arrival* arr,
                  uint64_t* h2d) {
  if (!w->copy_stream) {
    DP_CUDA(cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking));
    DP_CUDA(cudaMalloc(&w->d_arrived, sizeof(int)));
    for (int k = 0; k < kMaxChunks; ++k)
      DP_CUDA(cudaEventCreateWithFlags(&w->chunk_ev[k],
                                       cudaEventDisableTiming));
  }
  const int64_t chunk = 1LL << shift;
  arr->nchunks = (int)((m + chunk - 1) / chunk);
  arr->waited = 0;
  if (arr->nchunks > kMaxChunks)
    return fail(DP_ERR_INVALID, "too many copy chunks");
  DP_CUDA(cudaMemsetAsync(w->d_arrived, 0, sizeof(int), s));
  DP_CUDA(cudaEventRecord(w->evk0, s));
  DP_CUDA(cudaStreamWaitEvent(w->copy_stream, w->evk0, 0));
  for (int k = 0; k < arr->nchunks; ++k) {
    const int64_t lo = (int64_t)k * chunk;
    const int64_t len = std::min(chunk, m - lo);
    for (int i = 0; i < nsrc; ++i) {
      DP_CUDA(cudaMemcpyAsync((int32_t*)dev[i] + lo,
                              (const int32_t*)host[i] + lo, (size_t)len * 4,
                              cudaMemcpyHostToDevice, w->copy_stream));
      *h2d += (uint64_t)len * 4;
    }
    set_arrived_kernel<<<1, 1, 0, w->copy_stream>>>(w->d_arrived, k + 1);
    DP_CUDA(cudaGetLastError());
    DP_CUDA(cudaEventRecord(w->chunk_ev[k], w->copy_stream));
  }
  return 0;
}

// col_bits = 24: four col values travel as three 32-bit words (v0 | v1 << 24,
// v1 >> 8 | v2 << 16, v2 >> 16 | v3 << 8).  Host packer for slots [lo, lo +
// len) (lo a multiple of 4) into out + 3 * lo / 4; false if a value lies
// outside [0, 2^24) (the chunk then travels as int32).  OpenMP.
bool pack_col24_host(const int32_t* c, long long lo, long long len,
                     unsigned* out) {
  const long long groups = (len + 3) / 4;
  unsigned bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
  for (long long g = 0; g < groups; ++g) {
    const long long e = lo + g * 4;
    unsigned v[4];
    if (e + 4 <= lo + len) {
#pragma GCC unroll 4
      for (int j = 0; j < 4; ++j) v[j] = (unsigned)c[e + j];
    } else {
      for (int j = 0; j < 4; ++j) v[j] = e + j < lo + len ? (unsigned)c[e + j] : 0u;
    }
    bad |= v[0] | v[1] | v[2] | v[3];
    unsigned* o = out + (lo >> 2) * 3 + g * 3;
    o[0] = v[0] | v[1] << 24;
    o[1] = v[1] >> 8 | v[2] << 16;
    o[2] = v[2] >> 16 | v[3] << 8;
  }
  return (bad >> 24) == 0;
}

// Device twin: expand groups [g0, g0 + groups) of 3 words into 4 int32 slots
// (the last group may be partial: slots < m only).
__global__ void unpack_col24_kernel(const unsigned* __restrict__ in,
                                    long long g0, long long groups,
                                    long long m, int* __restrict__ col) {
  for (long long g = g0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
       g < g0 + groups; g += (long long)gridDim.x * blockDim.x) {
    const unsigned a = __ldg(in + g * 3), b = __ldg(in + g * 3 + 1),
                   c = __ldg(in + g * 3 + 2);
    const int4 v = make_int4((int)(a & 0xffffffu),
                             (int)((a >> 24) | ((b & 0xffffu) << 8)),
                             (int)((b >> 16) | ((c & 0xffu) << 16)),
                             (int)(c >> 8));
    if (g * 4 + 4 <= m) {
      reinterpret_cast<int4*>(col)[g] = v;
    } else {
      const int x[4] = {v.x, v.y, v.z, v.w};
      for (int j = 0; j < 4 && g * 4 + j < m; ++j) col[g * 4 + j] = x[j];
    }
  }
}

// dp_sssp's host-buffer staging with transfer codecs: as stage_chunked for
// (col, weight), and
//   pack_w (weight_bits = 4): each weight chunk is packed on the host
//     (OpenMP, into pinned staging) and copied as nibbles, 1/8 of the bytes.
//     At the first chunk holding a weight outside [1, 16] the call reverts to
//     int32 weights: the earlier chunks' int32 weights are copied and awaited
//     (before any round can read them), the rest stream as int32.
//     *packed_all: every weight chunk went packed (the rounds read nibbles)
//   pack_c (col_bits = 24): each col chunk is packed to 3-byte values on the
//     host, copied (3/4 of the bytes) and expanded into the int32 col on the
//     copy stream before the chunk is published; a chunk holding a value
//     outside [0, 2^24) travels as int32 (per chunk: the device col is int32
//     either way)
// The packing of chunk k + 1 overlaps the DMA of chunk k.
int stage_chunked_codec(Workspace* w, cudaStream_t s, const int32_t* col,
                        const int32_t* weight, int32_t* d_col,
                        int32_t* d_weight, unsigned* d_wpack, int64_t m,
                        int shift, bool pack_w, bool pack_c, Arrival* arr,
                        uint64_t* h2d, bool* packed_all) {
  int r;
  if (!w->copy_stream) {
    DP_CUDA(cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking));
    DP_CUDA(cudaMalloc(&w->d_arrived, sizeof(int)));
    for (int k = 0; k < kMaxChunks; ++k)
      DP_CUDA(cudaEventCreateWithFlags(&w->chunk_ev[k],
                                       cudaEventDisableTiming));
  }
  auto pinned = [](void** p, size_t* have, size_t need) -> int {
    if (need <= *have) return 0;
    if (*p) cudaFreeHost(*p);
    *p = nullptr;
    *have = 0;
    DP_CUDA(cudaMallocHost(p, need));
    *have = need;
    return 0;
  };
  if (pack_w &&
      (r = pinned(&w->h_wpack, &w->h_wpack_bytes,
                  (size_t)((m + 7) / 8) * sizeof(unsigned))))
    return r;
  const size_t cbytes = (size_t)((m + 3) / 4) * 3 * sizeof(unsigned);
  if (pack_c && ((r = pinned(&w->h_cpack, &w->h_cpack_bytes, cbytes)) ||
                 (r = grow(&w->cpack, &w->cpack_bytes, cbytes))))
    return r;
  unsigned* hp = (unsigned*)w->h_wpack;
  unsigned* hc = (unsigned*)w->h_cpack;
  const int64_t chunk = 1LL << shift;
  arr->nchunks = (int)((m + chunk - 1) / chunk);
  arr->waited = 0;
  if (arr->nchunks > kMaxChunks)
    return fail(DP_ERR_INVALID, "too many copy chunks");
  DP_CUDA(cudaMemsetAsync(w->d_arrived, 0, sizeof(int), s));
  DP_CUDA(cudaEventRecord(w->evk0, s));
  DP_CUDA(cudaStreamWaitEvent(w->copy_stream, w->evk0, 0));
  bool packed = pack_w;
  for (int k = 0; k < arr->nchunks; ++k) {
    const int64_t lo = (int64_t)k * chunk;
    const int64_t len = std::min(chunk, m - lo);
    if (pack_c && pack_col24_host(col, lo, len, hc)) {
      const int64_t g0 = lo >> 2, groups = (len + 3) / 4;
      DP_CUDA(cudaMemcpyAsync((unsigned*)w->cpack + g0 * 3, hc + g0 * 3,
                              (size_t)groups * 3 * sizeof(unsigned),
                              cudaMemcpyHostToDevice, w->copy_stream));
      *h2d += (uint64_t)groups * 3 * sizeof(unsigned);
      const int blocks = (int)std::max<int64_t>(
          1, std::min<int64_t>(dp::ceil_div_ll(groups, 256), 148 * 8));
      unpack_col24_kernel<<<blocks, 256, 0, w->copy_stream>>>(
          (const unsigned*)w->cpack, g0, groups, m, d_col);
      DP_CUDA(cudaGetLastError());
    } else {
      DP_CUDA(cudaMemcpyAsync(d_col + lo, col + lo, (size_t)len * 4,
                              cudaMemcpyHostToDevice, w->copy_stream));
      *h2d += (uint64_t)len * 4;
    }
    if (packed && !pack_weights_host(weight, lo, len, hp)) {
      packed = false;
      if (lo > 0) {  // chunks [0, k) arrived packed only: add their int32
        DP_CUDA(cudaMemcpyAsync(d_weight, weight, (size_t)lo * 4,
                                cudaMemcpyHostToDevice, w->copy_stream));
        *h2d += (uint64_t)lo * 4;
        DP_CUDA(cudaStreamSynchronize(w->copy_stream));
      }
    }
    if (packed) {
      const size_t words = (size_t)((len + 7) / 8);
      DP_CUDA(cudaMemcpyAsync(d_wpack + (lo >> 3), hp + (lo >> 3),
                              words * sizeof(unsigned),
                              cudaMemcpyHostToDevice, w->copy_stream));
      *h2d += words * sizeof(unsigned);
    } else {
      DP_CUDA(cudaMemcpyAsync(d_weight + lo, weight + lo, (size_t)len * 4,
                              cudaMemcpyHostToDevice, w->copy_stream));
      *h2d += (uint64_t)len * 4;
    }
    set_arrived_kernel<<<1, 1, 0, w->copy_stream>>>(w->d_arrived, k + 1);
    DP_CUDA(cudaGetLastError());
    DP_CUDA(cudaEventRecord(w->chunk_ev[k], w->copy_stream));
  }
  *packed_all = packed;
  return 0;
}

// the compute stream waits for every chunk (the call must not return while
// the DMA still reads the caller's buffers)
int join_chunked(Workspace* w, cudaStream_t s, const Arrival& arr) {
  if (arr.nchunks > 0)
    DP_CUDA(cudaStreamWaitEvent(s, w->chunk_ev[arr.nchunks - 1], 0));
  return 0;
}

// Chunks of the edge arrays: about four (one round per landed chunk; more
// rounds only add L2 contention with the DMA), at least 2^20 slots each.
int chunk_shift(int64_t m) {
  int shift = 20;
  while (shift < 40 && ((m + (1LL << shift) - 1) >> shift) > 4) ++shift;
  if (const char* e = std::getenv("DP_COPY_CHUNK_SHIFT"))  // tests, probes
    shift = std::max(2, std::min(40, std::atoi(e)));
  while (shift < 40 && ((m + (1LL << shift) - 1) >> shift) > kMaxChunks)
    ++shift;
  return shift;
}

// host-buffer staging
int stage(Workspace* w, int slot, const void* host, size_t bytes,
          cudaStream_t s, uint64_t* h2d) {
  int r;
  if ((r = grow(&w->io[slot], &w->io_bytes[slot], bytes))) return r;
  if (host && bytes) {
    DP_CUDA(cudaMemcpyAsync(w->io[slot], host, bytes, cudaMemcpyHostToDevice, s));
    *h2d += bytes;
  }
  return 0;
}

int unstage(Workspace* w, int slot, void* host, size_t bytes, cudaStream_t s,
            uint64_t* d2h) {
  if (host && bytes) {
    DP_CUDA(cudaMemcpyAsync(host, w->io[slot], bytes, cudaMemcpyDeviceToHost, s));
    *d2h += bytes;
  }
  return 0;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int dp_abi_version(void) { return DP_ABI_VERSION; }

const char* dp_last_error(void) { return g_err.c_str(); }

int dp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int dp_init(int32_t device) {
  int n = dp_device_count();
  if (n <= 0) return fail(DP_ERR_NO_DEVICE, "no CUDA device visible");
  if (device < 0 || device >= n) return fail(DP_ERR_INVALID, "bad device");
  DP_CUDA(cudaSetDevice(device));
  g_device = device;
  cudaDeviceProp p;
  DP_CUDA(cudaGetDeviceProperties(&p, device));
  if (p.major != 10)
    return fail(DP_ERR_NO_DEVICE, std::string("libdynpar is built for sm_100a; "
                                              "device is ") + p.name);
  int r;
  Workspace* w = workspace(&r);
  return w ? 0 : r;
}

#define DP_HOST_CALL_BEGIN                \
  clear_stats(stats);                     \
  const double t0_ = now_ns();            \
  int r_;                                 \
  Workspace* w_ = workspace(&r_);         \
  if (!w_) return r_;                     \
  cudaStream_t s_ = 0;                    \
  uint64_t h2d_ = 0, d2h_ = 0;

#define DP_HOST_CALL_END                                      \
  DP_CUDA(cudaStreamSynchronize(s_));                         \
  if (stats) {                                                \
    stats->ns_host = now_ns() - t0_;                          \
    stats->h2d_bytes = h2d_;                                  \
    stats->d2h_bytes = d2h_;                                  \
  }                                                           \
  return 0;

#define DP_TRY(x)       \
  do {                  \
    if ((r_ = (x))) return r_; \
  } while (0)

int dp_bfs(const int32_t* rowptr, const int32_t* col, int32_t n, int64_t m,
           int32_t src, const dp_config* cfg, int32_t* dist, int32_t* counts,
           dp_stats* stats) {
  DP_HOST_CALL_BEGIN
  if (n < 1 || m < 0) return fail(DP_ERR_INVALID, "bad graph size");
  DP_TRY(stage(w_, 0, rowptr, (size_t)(n + 1) * 4, s_, &h2d_));
  DP_TRY(stage(w_, 1, col, (size_t)m * 4, s_, &h2d_));
  DP_TRY(stage(w_, 2, nullptr, (size_t)n * 4, s_, &h2d_));
  DP_TRY(stage(w_, 3, nullptr, (size_t)n * 4, s_, &h2d_));
  DP_TRY(bfs_dev_impl((int*)w_->io[0], (int*)w_->io[1], n, src, cfg,
                      (int*)w_->io[2], (int*)w_->io[3], s_, stats, m));
  DP_TRY(unstage(w_, 2, dist, (size_t)n * 4, s_, &d2h_));
  DP_TRY(unstage(w_, 3, counts, (size_t)n * 4, s_, &d2h_));
  DP_HOST_CALL_END
}

int dp_bfs_dev(const int32_t* d_rowptr, const int32_t* d_col, int32_t n,
               int64_t m, int32_t src, const dp_config* cfg, int32_t* d_dist,
               int32_t* d_counts, void* stream, dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = bfs_dev_impl(d_rowptr, d_col, n, src, cfg, d_dist, d_counts,
                       (cudaStream_t)stream, stats, m);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_sssp(const int32_t* rowptr, const int32_t* col, const int32_t* weight,
            int32_t n, int64_t m, int32_t src, const dp_config* cfg,
            int32_t* dist, dp_stats* stats) {
  DP_HOST_CALL_BEGIN
  if (n < 1 || m < 0) return fail(DP_ERR_INVALID, "bad graph size");
  DP_TRY(stage(w_, 0, rowptr, (size_t)(n + 1) * 4, s_, &h2d_));
  DP_TRY(stage(w_, 2, nullptr, (size_t)n * 4, s_, &h2d_));
  if (cfg && cfg->device_loop) {  // device-chained rounds: copy first
    DP_TRY(stage(w_, 1, col, (size_t)m * 4, s_, &h2d_));
    DP_TRY(stage(w_, 4, weight, (size_t)m * 4, s_, &h2d_));
    DP_TRY(sssp_dev_impl((int*)w_->io[0], (int*)w_->io[1], (int*)w_->io[4],
                         n, src, cfg, (int*)w_->io[2], s_, stats, nullptr, 0,
                         nullptr, m));
  } else {
    // rounds start as soon as rowptr has landed; col / weight stream in
    // behind them in chunks and parents whose edges are still in flight
    // are deferred to a later round (same distances, the copy hides the
    // compute)
    DP_TRY(stage(w_, 1, nullptr, (size_t)m * 4, s_, &h2d_));
    DP_TRY(stage(w_, 4, nullptr, (size_t)m * 4, s_, &h2d_));
    Arrival arr;
    arr.host_out = dist;
    arr.dev_out = w_->io[2];
    arr.out_bytes = (size_t)n * 4;
    const int shift = chunk_shift(m);
    const unsigned* wpack = nullptr;
    const bool pack_w = cfg && cfg->weight_bits == 4;
    const bool pack_c = cfg && cfg->col_bits == 24;
    if (pack_w || pack_c) {
      if (pack_w)
        DP_TRY(stage(w_, 3, nullptr, (size_t)((m + 7) / 8 + 1) * 4, s_, &h2d_));
      bool all = false;
      DP_TRY(stage_chunked_codec(w_, s_, col, weight, (int32_t*)w_->io[1],
                                 (int32_t*)w_->io[4], (unsigned*)w_->io[3], m,
                                 shift, pack_w, pack_c, &arr, &h2d_, &all));
      if (all) wpack = (const unsigned*)w_->io[3];
    } else {
      const void* hsrc[2] = {col, weight};
      void* ddst[2] = {w_->io[1], w_->io[4]};
      DP_TRY(stage_chunked(w_, s_, 2, hsrc, ddst, m, shift, &arr, &h2d_));
    }
    const int rs = sssp_dev_impl((int*)w_->io[0], (int*)w_->io[1],
                                 (int*)w_->io[4], n, src, cfg,
                                 (int*)w_->io[2], s_, stats, &arr, shift,
                                 wpack, m);
    DP_TRY(join_chunked(w_, s_, arr));
    if (rs) {
      cudaStreamSynchronize(s_);
      cudaStreamSynchronize(w_->copy_stream);
      return rs;
    }
    d2h_ += arr.spec_d2h;
    if (arr.spec_final) {  // the copy that overlapped the last round
      DP_CUDA(cudaStreamSynchronize(w_->copy_stream));
      DP_HOST_CALL_END
    }
    DP_CUDA(cudaStreamSynchronize(w_->copy_stream));  // stale copies
  }
  DP_TRY(unstage(w_, 2, dist, (size_t)n * 4, s_, &d2h_));
  DP_HOST_CALL_END
}

int dp_sssp_dev(const int32_t* d_rowptr, const int32_t* d_col,
                const int32_t* d_weight, int32_t n, int64_t m, int32_t src,
                const dp_config* cfg, int32_t* d_dist, void* stream,
                dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  const unsigned* wpack = nullptr;
  int r = 0;
  if (cfg && cfg->weight_bits == 4) {
    Workspace* w = workspace(&r);
    if (!w) return r;
    if ((r = pack_weights_dev(w, d_weight, m, (cudaStream_t)stream, &wpack)))
      return r;
  }
  r = sssp_dev_impl(d_rowptr, d_col, d_weight, n, src, cfg, d_dist,
                    (cudaStream_t)stream, stats, nullptr, 0, wpack, m);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_manylaunch(const int32_t* sizes, int32_t n, const dp_config* cfg,
                  int32_t* out, int32_t* total, dp_stats* stats) {
  DP_HOST_CALL_BEGIN
  if (n < 0) return fail(DP_ERR_INVALID, "negative size");
  DP_TRY(stage(w_, 0, sizes, (size_t)n * 4, s_, &h2d_));
  DP_TRY(stage(w_, 1, nullptr, (size_t)n * 4 + 4, s_, &h2d_));
  DP_TRY(stage(w_, 2, nullptr, 4, s_, &h2d_));
  DP_TRY(manylaunch_dev_impl((int*)w_->io[0], n, cfg, (int*)w_->io[1],
                             (int*)w_->io[2], s_, stats));
  DP_TRY(unstage(w_, 1, out, (size_t)n * 4, s_, &d2h_));
  DP_TRY(unstage(w_, 2, total, 4, s_, &d2h_));
  DP_HOST_CALL_END
}

int dp_manylaunch_dev(const int32_t* d_sizes, int32_t n, const dp_config* cfg,
                      int32_t* d_out, int32_t* d_total, void* stream,
                      dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = manylaunch_dev_impl(d_sizes, n, cfg, d_out, d_total,
                              (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_tc(const int32_t* rowptr, const int32_t* col, int32_t n, int64_t m,
          int64_t edge_lo, int64_t edge_hi, const dp_config* cfg,
          uint64_t* triangles, dp_stats* stats) {
  DP_HOST_CALL_BEGIN
  if (n < 0 || m < 0) return fail(DP_ERR_INVALID, "bad graph size");
  DP_TRY(stage(w_, 0, rowptr, (size_t)(n + 1) * 4, s_, &h2d_));
  DP_TRY(stage(w_, 1, col, (size_t)m * 4, s_, &h2d_));
  DP_TRY(stage(w_, 2, nullptr, 8, s_, &h2d_));
  DP_TRY(tc_dev_impl((int*)w_->io[0], (int*)w_->io[1], n, m, edge_lo, edge_hi,
                     cfg, (uint64_t*)w_->io[2], s_, stats));
  DP_TRY(unstage(w_, 2, triangles, 8, s_, &d2h_));
  DP_HOST_CALL_END
}

int dp_tc_dev(const int32_t* d_rowptr, const int32_t* d_col, int32_t n,
              int64_t m, int64_t edge_lo, int64_t edge_hi,
              const dp_config* cfg, uint64_t* d_triangles, void* stream,
              dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = tc_dev_impl(d_rowptr, d_col, n, m, edge_lo, edge_hi, cfg,
                      d_triangles, (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_gc(const int32_t* rowptr, const int32_t* col, int32_t n, int64_t m,
          const dp_config* cfg, int32_t* color, dp_stats* stats) {
  DP_HOST_CALL_BEGIN
  if (n < 0 || m < 0) return fail(DP_ERR_INVALID, "bad graph size");
  DP_TRY(stage(w_, 0, rowptr, (size_t)(n + 1) * 4, s_, &h2d_));
  DP_TRY(stage(w_, 1, col, (size_t)m * 4, s_, &h2d_));
  DP_TRY(stage(w_, 2, nullptr, (size_t)n * 4 + 4, s_, &h2d_));
  DP_TRY(gc_dev_impl((int*)w_->io[0], (int*)w_->io[1], n, m, cfg,
                     (int*)w_->io[2], s_, stats));
  DP_TRY(unstage(w_, 2, color, (size_t)n * 4, s_, &d2h_));
  DP_HOST_CALL_END
}

int dp_gc_dev(const int32_t* d_rowptr, const int32_t* d_col, int32_t n,
              int64_t m, const dp_config* cfg, int32_t* d_color, void* stream,
              dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = gc_dev_impl(d_rowptr, d_col, n, m, cfg, d_color,
                      (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_mst(const int32_t* rowptr, const int32_t* col, const int32_t* weight,
           const int32_t* eid, int32_t n, int64_t m, const dp_config* cfg_find,
           const dp_config* cfg_verify, uint8_t* in_mst, int64_t* total_weight,
           int64_t* nedges, dp_stats* stats) {
  DP_HOST_CALL_BEGIN
  if (n < 0 || m < 0) return fail(DP_ERR_INVALID, "bad graph size");
  DP_TRY(stage(w_, 0, rowptr, (size_t)(n + 1) * 4, s_, &h2d_));
  DP_TRY(stage(w_, 1, col, (size_t)m * 4, s_, &h2d_));
  DP_TRY(stage(w_, 4, weight, (size_t)m * 4, s_, &h2d_));
  DP_TRY(stage(w_, 2, eid, (size_t)m * 4, s_, &h2d_));
  DP_TRY(stage(w_, 3, nullptr, (size_t)m + 1, s_, &h2d_));
  DP_TRY(mst_dev_impl((int*)w_->io[0], (int*)w_->io[1], (int*)w_->io[4],
                      (int*)w_->io[2], n, m, cfg_find, cfg_verify,
                      (uint8_t*)w_->io[3], total_weight, nedges, s_, stats));
  DP_TRY(unstage(w_, 3, in_mst, (size_t)m, s_, &d2h_));
  DP_HOST_CALL_END
}

int dp_mst_dev(const int32_t* d_rowptr, const int32_t* d_col,
               const int32_t* d_weight, const int32_t* d_eid, int32_t n,
               int64_t m, const dp_config* cfg_find,
               const dp_config* cfg_verify, uint8_t* d_in_mst,
               int64_t* total_weight, int64_t* nedges, void* stream,
               dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = mst_dev_impl(d_rowptr, d_col, d_weight, d_eid, n, m, cfg_find,
                       cfg_verify, d_in_mst, total_weight, nedges,
                       (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_sp(const int32_t* lits, int32_t k, int32_t nclauses,
          const int32_t* occ_row, const int32_t* occ, int32_t nvars,
          const double* eta0, int32_t max_sweeps, float eps,
          const dp_config* cfg, double* eta, float* wpos, float* wneg,
          int32_t* sweeps, float* delta, dp_stats* stats) {
  DP_HOST_CALL_BEGIN
  if (k < 1 || nclauses < 0 || nvars < 0)
    return fail(DP_ERR_INVALID, "bad formula size");
  const size_t ne = (size_t)nclauses * (size_t)k;
  DP_TRY(stage(w_, 0, lits, ne * 4, s_, &h2d_));
  DP_TRY(stage(w_, 1, occ_row, (size_t)(nvars + 1) * 4, s_, &h2d_));
  DP_TRY(stage(w_, 2, occ, ne * 4, s_, &h2d_));
  DP_TRY(stage(w_, 3, eta0, ne * 8, s_, &h2d_));
  DP_TRY(stage(w_, 4, nullptr, (size_t)nvars * 8 + 8, s_, &h2d_));
  float* d_wpos = (float*)w_->io[4];
  float* d_wneg = d_wpos + nvars;
  DP_TRY(sp_dev_impl((int*)w_->io[0], k, nclauses, (int*)w_->io[1],
                     (int*)w_->io[2], nvars, max_sweeps, eps, cfg,
                     (double*)w_->io[3], d_wpos, d_wneg, sweeps, delta, s_,
                     stats));
  DP_TRY(unstage(w_, 3, eta, ne * 8, s_, &d2h_));
  if (wpos && nvars)
    DP_CUDA(cudaMemcpyAsync(wpos, d_wpos, (size_t)nvars * 4,
                            cudaMemcpyDeviceToHost, s_));
  if (wneg && nvars)
    DP_CUDA(cudaMemcpyAsync(wneg, d_wneg, (size_t)nvars * 4,
                            cudaMemcpyDeviceToHost, s_));
  d2h_ += (uint64_t)nvars * 8;
  DP_HOST_CALL_END
}

int dp_sp_dev(const int32_t* d_lits, int32_t k, int32_t nclauses,
              const int32_t* d_occ_row, const int32_t* d_occ, int32_t nvars,
              int32_t max_sweeps, float eps, const dp_config* cfg,
              double* d_eta, float* d_wpos, float* d_wneg, int32_t* sweeps,
              float* delta, void* stream, dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = sp_dev_impl(d_lits, k, nclauses, d_occ_row, d_occ, nvars,
                      max_sweeps, eps, cfg, d_eta, d_wpos, d_wneg, sweeps,
                      delta, (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_bfs_part_level(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                      int32_t n_local, int32_t nparts, int32_t part,
                      int32_t level, const dp_config* cfg, int32_t* d_dist_p,
                      int32_t* d_counts, uint32_t* d_sent, int32_t* d_send_buf,
                      int64_t send_stride, int32_t* d_send_counts,
                      int32_t* d_changed, void* stream, dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = bfs_part_level_impl(d_rowptr_p, d_col_p, n_local, nparts, part,
                              level, cfg, d_dist_p, d_counts, d_sent,
                              d_send_buf, send_stride, d_send_counts,
                              d_changed, (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_bfs_part_level_peer(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                           int32_t n_local, int32_t nparts, int32_t part,
                           int32_t level, const dp_config* cfg,
                           int32_t* d_dist_p, int32_t* const* d_peer_dist,
                           int32_t* d_counts, uint32_t* d_sent,
                           int32_t* d_changed, void* stream,
                           dp_stats* stats) {
  clear_stats(stats);
  if (!d_peer_dist) return fail(DP_ERR_INVALID, "null peer table");
  const double t0 = now_ns();
  int r = bfs_part_level_impl(d_rowptr_p, d_col_p, n_local, nparts, part,
                              level, cfg, d_dist_p, d_counts, d_sent, nullptr,
                              0, nullptr, d_changed, (cudaStream_t)stream,
                              stats, d_peer_dist);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_unspread_dev(const int32_t* d_work, int32_t b, int32_t n,
                    int32_t* d_out, void* stream) {
  if (n < 0 || b < 0 || b > 30 || !d_work || (n > 0 && !d_out))
    return fail(DP_ERR_INVALID, "bad unspread arguments");
  if (n == 0) return 0;
  const unsigned mask = b > 0 ? (unsigned)((1u << b) - 1) : 0u;
  unspread_kernel<<<dp::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_work, mask, d_out, n);
  DP_CUDA(cudaGetLastError());
  return 0;
}

int dp_bfs_part_apply(const int32_t* d_recv, int64_t nrecv, int32_t nparts,
                      int32_t level, int32_t* d_dist_p, int32_t* d_changed,
                      void* stream) {
  if (nparts < 1 || nrecv < 0) return fail(DP_ERR_INVALID, "bad arguments");
  if (nrecv == 0) return 0;
  const int blocks =
      (int)std::min<long long>(dp::ceil_div_ll(nrecv, 256), 148 * 16);
  bfs_part_apply_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      d_recv, nrecv, nparts, level, d_dist_p, d_changed);
  DP_CUDA(cudaGetLastError());
  return 0;
}

int dp_sssp_part_round(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                       const int32_t* d_weight_p, int32_t n_local,
                       int32_t nparts, int32_t part, const dp_config* cfg,
                       int32_t* d_dist_p, int32_t* d_best, uint64_t* d_send_buf,
                       const int64_t* d_send_off, int32_t* d_send_counts,
                       int32_t* d_changed, void* stream, dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = sssp_part_round_impl(d_rowptr_p, d_col_p, d_weight_p, n_local,
                               nparts, part, cfg, d_dist_p, d_best, d_send_buf,
                               d_send_off, d_send_counts, d_changed,
                               (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_sssp_part_round_peer(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                            const int32_t* d_weight_p, int32_t n_local,
                            int32_t nparts, int32_t part,
                            const dp_config* cfg, int32_t* d_dist_p,
                            int32_t* const* d_peer_dist, int32_t* d_best,
                            int32_t* d_changed, void* stream,
                            dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = sssp_peer_round_impl(d_rowptr_p, d_col_p, d_weight_p, n_local,
                               nparts, part, cfg, d_dist_p, d_peer_dist,
                               d_best, d_changed, (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_sssp_part_solve_peer(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                            const int32_t* d_weight_p, int32_t n_local,
                            int32_t n_global, int32_t nparts, int32_t part,
                            int32_t src, const dp_config* cfg,
                            int32_t* d_dist_p, int32_t* const* d_peer_dist,
                            int32_t* d_best, uint64_t* const* d_peer_sig,
                            uint64_t epoch, void* stream, dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = sssp_part_solve_peer_impl(
      d_rowptr_p, d_col_p, d_weight_p, n_local, n_global, nparts, part, src,
      cfg, d_dist_p, d_peer_dist, d_best, d_peer_sig, epoch,
      (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int dp_bfs_part_solve_peer(const int32_t* d_rowptr_p, const int32_t* d_col_p,
                           int32_t n_local, int32_t n_global, int32_t nparts,
                           int32_t part, int32_t src, const dp_config* cfg,
                           int32_t* d_dist_p, int32_t* const* d_peer_dist,
                           int32_t* d_counts, int64_t counts_len,
                           uint32_t* d_sent, uint64_t* const* d_peer_sig,
                           uint64_t epoch, void* stream, dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = bfs_part_solve_peer_impl(
      d_rowptr_p, d_col_p, n_local, n_global, nparts, part, src, cfg,
      d_dist_p, d_peer_dist, d_counts, counts_len, d_sent, d_peer_sig, epoch,
      (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

int64_t dp_step_times(double* ms, int64_t cap) {
  const int64_t k = (int64_t)g_step_ms.size();
  for (int64_t i = 0; i < std::min(k, cap); ++i) ms[i] = g_step_ms[i];
  return k;
}

void dp_thread_release(void) {
  for (Workspace& w : g_ws) {
    if (!w.ready) continue;
    cudaFree(w.tab);
    cudaFree(w.scan);
    cudaFree(w.ctr);
    cudaFree(w.done);
    cudaFree(w.ds);
    cudaFreeHost(w.h_ds);
    cudaFreeHost(w.h_ctr);
    cudaFree(w.d_scratch);
    cudaFree(w.d_flag);
    cudaEventDestroy(w.ev0);
    cudaEventDestroy(w.ev1);
    cudaEventDestroy(w.evk0);
    cudaEventDestroy(w.evk1);
    cudaFreeHost(w.h_sig);
    for (void* p : w.io) cudaFree(p);
    if (w.copy_stream) cudaStreamDestroy(w.copy_stream);
    cudaFree(w.d_arrived);
    for (cudaEvent_t e : w.chunk_ev)
      if (e) cudaEventDestroy(e);
    if (w.ev_spec) cudaEventDestroy(w.ev_spec);
    cudaFree(w.cwork);
    cudaFree(w.pub);
    cudaFree(w.wpack);
    cudaFreeHost(w.h_wpack);
    cudaFree(w.d_bad);
    cudaFree(w.cpack);
    cudaFreeHost(w.h_cpack);
    cudaFree(w.lbits);
    w = Workspace();
  }
}

int dp_sssp_part_apply(const uint64_t* d_recv, int64_t nrecv, int32_t nparts,
                       int32_t* d_dist_p, int32_t* d_changed, void* stream) {
  if (nparts < 1 || nrecv < 0) return fail(DP_ERR_INVALID, "bad arguments");
  if (nrecv == 0) return 0;
  const int blocks =
      (int)std::min<long long>(dp::ceil_div_ll(nrecv, 256), 148 * 16);
  sssp_part_apply_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      (const unsigned long long*)d_recv, nrecv, nparts, d_dist_p, d_changed);
  DP_CUDA(cudaGetLastError());
  return 0;
}

int dp_rmat_part_keys_dev(int32_t scale, int32_t edge_factor, uint64_t seed,
                          int32_t nparts, int32_t part, uint64_t* d_keys,
                          int64_t capacity, int64_t* count, void* stream) {
  if (scale < 1 || scale > 30 || edge_factor < 1 || nparts < 1 || part < 0 ||
      part >= nparts || !count)
    return fail(DP_ERR_INVALID, "bad rmat arguments");
  int r;
  Workspace* w = workspace(&r);
  if (!w) return r;
  cudaStream_t s = (cudaStream_t)stream;
  const long long m = (long long)edge_factor << scale;
  // same seed mixing as gen.cpp
  unsigned long long z = seed ^ 0x524D4154ull;
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const unsigned long long key = z ^ (z >> 31);
  DP_CUDA(cudaMemsetAsync(w->d_scratch, 0, sizeof(unsigned long long), s));
  const int blocks = 148 * 16;
  rmat_part_keys_kernel<<<blocks, 256, 0, s>>>(
      key, m, scale, nparts, part,
      capacity > 0 ? (unsigned long long*)d_keys : nullptr, w->d_scratch);
  DP_CUDA(cudaGetLastError());
  unsigned long long got = 0;
  DP_CUDA(cudaMemcpyAsync(&got, w->d_scratch, sizeof(got),
                          cudaMemcpyDeviceToHost, s));
  DP_CUDA(cudaStreamSynchronize(s));
  *count = (int64_t)got;
  if (capacity > 0 && (long long)got > capacity)
    return fail(DP_ERR_INVALID, "key capacity exceeded");
  return 0;
}

int dp_bt(const float* cp, int32_t ncurves, int32_t max_tess, float curv_scale,
          const dp_config* cfg, int32_t* ntess, int64_t* offsets, float* verts,
          int64_t vert_capacity, int64_t* nverts, dp_stats* stats) {
  DP_HOST_CALL_BEGIN
  if (ncurves < 0 || vert_capacity < 0)
    return fail(DP_ERR_INVALID, "bad size");
  int64_t used = 0;
  DP_TRY(stage(w_, 0, cp, (size_t)ncurves * 24, s_, &h2d_));
  DP_TRY(stage(w_, 1, nullptr, (size_t)ncurves * 4, s_, &h2d_));
  DP_TRY(stage(w_, 2, nullptr, (size_t)ncurves * 8, s_, &h2d_));
  DP_TRY(stage(w_, 3, nullptr, (size_t)vert_capacity * 8, s_, &h2d_));
  DP_TRY(bt_dev_impl((float*)w_->io[0], ncurves, max_tess, curv_scale, cfg,
                     (int*)w_->io[1], (int64_t*)w_->io[2], (float*)w_->io[3],
                     vert_capacity, &used, s_, stats));
  if (nverts) *nverts = used;
  DP_TRY(unstage(w_, 1, ntess, (size_t)ncurves * 4, s_, &d2h_));
  DP_TRY(unstage(w_, 2, offsets, (size_t)ncurves * 8, s_, &d2h_));
  DP_TRY(unstage(w_, 3, verts, (size_t)used * 8, s_, &d2h_));
  DP_HOST_CALL_END
}

int dp_bt_dev(const float* d_cp, int32_t ncurves, int32_t max_tess,
              float curv_scale, const dp_config* cfg, int32_t* d_ntess,
              int64_t* d_offsets, float* d_verts, int64_t vert_capacity,
              int64_t* nverts, void* stream, dp_stats* stats) {
  clear_stats(stats);
  const double t0 = now_ns();
  int r = bt_dev_impl(d_cp, ncurves, max_tess, curv_scale, cfg, d_ntess,
                      d_offsets, d_verts, vert_capacity, nverts,
                      (cudaStream_t)stream, stats);
  if (stats) stats->ns_host = now_ns() - t0;
  return r;
}

}  // extern "C"
