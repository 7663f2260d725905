#!/usr/bin/env python
"""Benchmark of the nested-parallel hot path (BASELINE.json) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Headline workload (BASELINE.json metric "GTEPS (BFS/SSSP RMAT-22) ...",
config "SSSP on RMAT scale-22 integer weights, threshold/coarsening/
aggregation ... vs naive CDP and aggregation-only"): one step = one complete
SSSP (all Bellman-Ford rounds until no change, bench/benchmarks.py:259-270 of
the reference) from vertex 0 over RMAT-22 (n = 4,194,304, m = 67,108,864,
weights in [1, 9]) through libdynpar's CDP2 scheduler with the tuned
T + C + A policy.  GTEPS = E_reach / t with E_reach = sum of out-degrees of
reached vertices (schedule-independent).  Inputs (col + weight = 512 MiB)
exceed the 126 MB L2, so no flush is needed between steps.

The line also carries: e2e (same metric through the host-buffer C-ABI call
dp_sssp, H2D of the graph + D2H of dist inside the timed region), roofline
of the dominant kernel (the per-round parent grid incl. its CDP2 children),
cpu_baseline (the C oracle on the host cores), speed-ups over the naive-CDP
and aggregation-only (KLAP-style) builds, and the other BASELINE workloads
(BFS RMAT-22, TC RMAT-22, BT 25k curves) under "workloads".

N > 1: the same SSSP over a cyclic 1D vertex partition (one part per rank;
remote relaxations are atomicMin into the owner's dist through symmetric
memory, one NCCL max-reduction per round; --exchange a2a uses the NCCL
all-to-all instead);
--workload bfs26 / tc run the other partitioned configs (5 / 4).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

SCALE = 22
SEED = 1

# tuned policies (profiles/ + DESIGN.md); parity defaults elsewhere.
# sssp: profiles/tune_sssp_cf_r01.txt (T x C x child block x group size)
BEST = {
    # one aggregation group spanning the parent grid: the last parent block
    # issues ONE CDP2 launch per round (tools/tune.py, profiles/tune_*)
    # cf_wave: the source hub's child (160k edges at RMAT-22, 1,247 logical
    # blocks) runs uncoarsened: BFS level 0 80 -> 58 us, SSSP round 0
    # 72 -> 57 us (profiles/r02/ab_cfwave_r02.txt)
    "sssp": dict(threshold=1024, cfactor=16, agg="multiblock",
                 group_size=1 << 20, parent_block=128, child_block=128,
                 serial="warp", cf_wave=592),
    "bfs": dict(threshold=1024, cfactor=16, agg="multiblock",
                group_size=1 << 20, parent_block=256, child_block=128,
                serial="warp", cf_wave=592),
    # TC over the transposed CSR+ (profiles/tune_tc_rmat22_r01c.txt)
    "tc": dict(threshold=32, cfactor=4, agg="grid", parent_block=128,
               child_block=256, serial="warp"),
    # BT 25k is launch-latency-sized: every child launch costs more than the
    # 2.2 M vertices; T = infinity (children run in the parent warps,
    # load-balanced) wins (profiles/bt_policies_r01.txt: 46 vs 57-63 us)
    "bt": dict(threshold=2147483647, parent_block=64, serial="warp"),
    # MSTF (find) row; the verify kernel runs MST_OTHER_POLICY
    "mstf": dict(threshold=1024, cfactor=16, agg="multiblock",
                 group_size=1 << 20, parent_block=256, child_block=128,
                 serial="warp"),
    # tools/tune_sp.py (profiles/tune_sp_r01.txt): children run in the
    # parent thread below T, one aggregated launch per pass above it
    "sp": dict(threshold=128, cfactor=4, agg="multiblock", group_size=1 << 20,
               parent_block=128, child_block=128, serial="thread"),
}


def bt_stream_row(ncurves: int, quick: bool, policy=None) -> dict:
    """BT at a streaming size on one GPU (the 25k config is
    launch-sized): device time of the tessellation (CUDA events inside
    libdynpar), algorithmic bytes 36 B/curve + 8 B/vertex against HBM."""
    import torch
    from paper_2201_02789_b200 import _lib
    from paper_2201_02789_b200.bench.graphs import (BT_CURV_SCALE,
                                                    BT_MAX_TESS,
                                                    bezier_curves)
    lib = _lib.device()
    dev = torch.device("cuda", torch.cuda.current_device())
    cp_h = np.ascontiguousarray(bezier_curves(ncurves, 1), dtype=np.float32)
    cp = torch.from_numpy(cp_h).to(dev)
    cap = ncurves * 128 + (1 << 16)
    ntess = torch.empty(ncurves, dtype=torch.int32, device=dev)
    offs = torch.empty(ncurves, dtype=torch.int64, device=dev)
    verts = torch.empty((cap, 2), dtype=torch.float32, device=dev)
    used = ctypes.c_int64()
    policy = BEST["bt"] if policy is None else policy
    cfg = _cfg(policy)
    ts = []
    for _ in range(7):
        st = _lib.DpStats()
        _lib.check(lib.dp_bt_dev(cp.data_ptr(), ncurves, BT_MAX_TESS,
                                 BT_CURV_SCALE, ctypes.byref(cfg),
                                 ntess.data_ptr(), offs.data_ptr(),
                                 verts.data_ptr(), cap, ctypes.byref(used),
                                 None, ctypes.byref(st)))
        ts.append(st.ns_device / 1e6)
    ms = statistics.median(ts[2:])
    nv = int(used.value)
    alg = 36 * ncurves + 8 * nv
    peak, src = hbm_peak()
    row = {"curves": ncurves, "ms": ms, "curves_per_s": ncurves / ms * 1e3,
           "vertices": nv, "gbps_alg": alg / (ms * 1e6),
           "frac_hbm": alg / (ms * 1e6) / peak, "peak_source": src,
           "policy": policy}
    if not quick:
        from oracle import oracle
        want_nt, want_v = oracle.bt(cp_h, BT_MAX_TESS, BT_CURV_SCALE)
        cs = float(verts[:nv].double().sum().item())
        want_cs = float(np.asarray(want_v, dtype=np.float64).sum())
        ok = (np.array_equal(ntess.cpu().numpy(), want_nt)
              and abs(cs - want_cs) <= 1e-6 * max(1.0, abs(want_cs)))
        row["parity"] = ("vertex counts exact, fp64 checksum within 1e-6 of "
                         "the oracle" if ok else "MISMATCH")
    del verts
    torch.cuda.empty_cache()
    return row


def reference_cpu_bfs(rowptr, col) -> dict | None:
    """BASELINE.md §3 `cpu_ref_s`: the reference's own CPU path,
    `dynoptc.bench.run_reference` (BFS_NOCDP on its pure-Python simulator,
    one core), on our RMAT CSR injected through its Workload
    (tests/golden/make_golden.py does the same).  Runs the unmodified
    reference installed in baseline/_ref (pip --target, git-ignored, shipped
    to the box); None when it is not installed."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "dynoptc").is_dir():
        return None
    sys.path.insert(0, str(ref))
    try:
        from dynoptc.bench import get_benchmark, run_reference
        from dynoptc.bench.benchmarks import Workload
        from dynoptc.bench.graphs import UNREACHED, DatasetSpec, Graph
        rp = [int(x) for x in rowptr]
        cl = [int(x) for x in col]
        g = Graph(tuple(rp), tuple(cl))
        dist = [UNREACHED] * g.n
        dist[0] = 0
        bufs = {"rowptr": rp, "col": cl, "dist": dist, "counts": [0] * g.n,
                "changed": [0]}
        wl = Workload(DatasetSpec("rmat", 16, SEED, f"rmat:16:seed{SEED}"),
                      bufs, g.n, g)
        t0 = time.perf_counter()
        rep = run_reference(get_benchmark("bfs"), wl)
        dt = time.perf_counter() - t0
        return {"seconds": dt, "cores": 1, "kind": "reference",
                "dist": np.asarray(rep.buffers["dist"], dtype=np.int64),
                "counts": np.asarray(rep.buffers["counts"], dtype=np.int64)}
    finally:
        sys.path.remove(str(ref))


def matched_agg_only(pol: dict, time_ms) -> dict:
    """The aggregation-only (KLAP-style) build like-for-like with a tuned
    policy: T = 0, C = 1, the policy's own parent / child blocks and serial
    mode, each granularity including one-group multiblock; time_ms(policy)
    returns a device time.  {granularity: ms}."""
    base = {k: pol[k] for k in ("parent_block", "child_block", "serial")
            if k in pol}
    out = {}
    for a in ("warp", "block", "multiblock", "grid"):
        p = dict(base, agg=a)
        if a == "multiblock":
            p["group_size"] = 1 << 20
        out[a] = time_ms(p)
    return out


# the host-buffer (e2e) call: weights copied as packed nibbles
E2E_EXTRA = dict(weight_bits=4)


# SSSP with the B200 `frontier` knob (profiles/tune_sssp_frontier_r01.txt)
FRONTIER_POLICY = dict(threshold=1024, cfactor=8, agg="multiblock",
                       group_size=2048, parent_block=128, child_block=128,
                       serial="warp", frontier=True)


def peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:  # noqa: BLE001
        return {}


def hbm_peak():
    p = peaks()
    if "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,"
         "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up is driver-heavy: let it reach steady
            # state (first sample) before the timed region begins
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.02)
            time.sleep(0.2)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap")
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# workloads on the device (C-ABI *_dev entry points, torch for memory/streams)
# ---------------------------------------------------------------------------

def _cfg(d: dict):
    from paper_2201_02789_b200.bench import BenchConfig
    return BenchConfig(**d).to_c()


class DeviceGraph:
    """RMAT-22 CSR (+ weights) resident in HBM."""

    def __init__(self, scale: int, seed: int, weights: bool):
        import torch
        from paper_2201_02789_b200.bench import graphs
        self.g = graphs.rmat_graph(scale, seed)
        self.w = graphs.edge_weights(self.g, seed) if weights else None
        self.n, self.m = self.g.n, self.g.m
        dev = torch.device("cuda", torch.cuda.current_device())
        self.rowptr = torch.from_numpy(self.g.rowptr).to(dev)
        self.col = torch.from_numpy(self.g.col).to(dev)
        self.weight = (torch.from_numpy(self.w).to(dev)
                       if weights else None)
        self.dist = torch.empty(self.n, dtype=torch.int32, device=dev)
        self.counts = torch.empty(self.n, dtype=torch.int32, device=dev)


def headline_config(n: int, m: int, e_reach: int) -> dict:
    """The `config` both arms print (identical keys and values, so the
    driver's same-config check compares like with like); run details such as
    the policy and round count go under "details"."""
    return {"workload": f"sssp rmat-{SCALE} from vertex 0",
            "graph": f"rmat scale {SCALE}, edge factor 16, seed {SEED}",
            "weights": "U[1,9] (bench/graphs.py:184-187 rule)",
            "n": n, "m": m, "e_reach": e_reach,
            "l2": "inputs (col+weight 512 MiB) exceed L2; no flush"}


def run_dev(kind: str, G, cfg, stream, raw: bool = False):
    """One call of dp_sssp_dev / dp_bfs_dev on resident buffers.  raw: return
    the DpStats struct itself (timed loops convert it after the timed region,
    so no Python dict building sits between two calls)."""
    from paper_2201_02789_b200 import _lib
    lib = _lib.device()
    st = _lib.DpStats()
    p = _lib.ptr
    if kind == "sssp":
        rc = lib.dp_sssp_dev(p(G.rowptr), p(G.col), p(G.weight), G.n, G.m, 0,
                             ctypes.byref(cfg), p(G.dist), stream,
                             ctypes.byref(st))
    else:
        rc = lib.dp_bfs_dev(p(G.rowptr), p(G.col), G.n, G.m, 0,
                            ctypes.byref(cfg), p(G.dist), p(G.counts),
                            stream, ctypes.byref(st))
    _lib.check(rc)
    return st if raw else _lib.stats_dict(st)


def timed_steps(fn, steps: int, warmup: int, stream_obj):
    """W untimed steps, then K steps bracketed by sync + CUDA events on the
    launching stream.  Returns (total ms, per-step stats list)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if torch.distributed.is_initialized():
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    out = []
    e0.record(stream_obj)
    for _ in range(steps):
        out.append(fn())
    e1.record(stream_obj)
    torch.cuda.synchronize()
    from paper_2201_02789_b200 import _lib
    return e0.elapsed_time(e1), [
        _lib.stats_dict(o) if isinstance(o, _lib.DpStats) else o for o in out]


def graph_traffic(kind: str, G, dist: np.ndarray, rounds: int):
    from paper_2201_02789_b200.bench.benchmarks import (bfs_traffic,
                                                        sssp_traffic)
    from paper_2201_02789_b200.bench.graphs import UNREACHED
    reached = dist < UNREACHED
    deg = np.diff(G.g.rowptr.astype(np.int64))
    e_reach = int(deg[reached].sum())
    if kind == "sssp":
        return e_reach, sssp_traffic(G.n, int(reached.sum()), e_reach, rounds)
    return e_reach, bfs_traffic(int(reached.sum()), e_reach)


def cpu_baseline_sssp(G, threads: int) -> dict:
    """The oracle (C restatement of SSSP_NOCDP) on the host cores over the
    full RMAT-22 workload (a few seconds at most, so no sub-sampling)."""
    from oracle import oracle
    reps, t0 = 0, time.perf_counter()
    while True:
        dist, rounds = oracle.sssp(G.g.rowptr, G.g.col, G.w, nthreads=threads)
        reps += 1
        if time.perf_counter() - t0 > 2.0 or reps >= 5:
            break
    dt = (time.perf_counter() - t0) / reps
    e_reach, _ = graph_traffic("sssp", G, dist, rounds)
    return {"value": e_reach / dt / 1e9, "unit": "GTEPS", "cores": threads,
            "kind": "port", "seconds_per_run": dt,
            "sample": f"full SSSP rmat-{SCALE} from vertex 0 ({rounds} rounds)"
                      f", mean of {reps} runs, oracle/oracle.c OpenMP",
            "dist": dist}


def e2e_sssp(G, cfg, steps: int) -> dict:
    """Same metric through the host-buffer C-ABI call dp_sssp: pinned host
    inputs, H2D copies + D2H of dist inside the timed region."""
    import torch
    from paper_2201_02789_b200 import _lib
    lib = _lib.device()
    rp = torch.from_numpy(G.g.rowptr).pin_memory()
    col = torch.from_numpy(G.g.col).pin_memory()
    w = torch.from_numpy(G.w).pin_memory()
    dist = torch.empty(G.n, dtype=torch.int32).pin_memory()
    times, st = [], _lib.DpStats()
    for i in range(steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(lib.dp_sssp(rp.data_ptr(), col.data_ptr(), w.data_ptr(),
                               G.n, G.m, 0, ctypes.byref(cfg),
                               dist.data_ptr(), ctypes.byref(st)))
        dt = time.perf_counter() - t0
        if i:
            times.append(dt)
    # the box's PCIe floor for the same bytes: pinned H2D of the call's
    # h2d_bytes and D2H of one dist, plain copies (e2e varies by box with
    # this; the call overlaps the rounds with the copy)
    hb = torch.empty(int(st.h2d_bytes), dtype=torch.uint8).pin_memory()
    db = torch.empty_like(hb, device="cuda")
    dd = torch.empty(G.n, dtype=torch.int32, device="cuda")
    dh = torch.empty(G.n, dtype=torch.int32).pin_memory()
    fl = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        db.copy_(hb, non_blocking=True)
        dh.copy_(dd, non_blocking=True)
        torch.cuda.synchronize()
        fl.append(time.perf_counter() - t0)
    floor = statistics.median(fl)
    del hb, db, dd, dh
    return {"seconds": statistics.median(times), "h2d": st.h2d_bytes,
            "d2h": st.d2h_bytes, "dist": dist.numpy().copy(),
            "copy_floor_s": floor}


def extra_workloads(stream, quick: bool) -> dict:
    """Other BASELINE configs, measured the same way (median of runs)."""
    import torch
    from paper_2201_02789_b200 import _lib
    from paper_2201_02789_b200.bench import load, run_config, BenchConfig
    out = {}
    lib = _lib.device()
    # BASELINE config 1: BFS RMAT-16, T=128, block aggregation, the
    # reference's launch shapes (parent and child blocks of 32)
    G16 = DeviceGraph(16, SEED, weights=False)
    c1 = dict(threshold=128, agg="block")
    runs = [run_dev("bfs", G16, _cfg(c1), stream) for _ in range(6)][1:]
    ms = statistics.median(r["ns_device"] for r in runs) / 1e6
    e16 = int(G16.counts.to(torch.int64).sum().item())
    naive16 = run_dev("bfs", G16, _cfg(dict()), stream)
    out["config1_bfs_rmat16_t128_block"] = {
        "gteps": e16 / ms / 1e6, "ms": ms, "levels": runs[0]["iterations"],
        "device_launches": runs[0]["num_launches"],
        "blocks_scheduled": runs[0]["blocks_scheduled"],
        "launch_lat_us": runs[0]["launch_lat_ns_mean"] / 1e3,
        "vs_naive_cdp": naive16["ns_device"] / 1e6 / ms,
        "naive_cdp_launches": naive16["num_launches"],
        "policy": c1}
    ref = None if quick else reference_cpu_bfs(G16.g.rowptr, G16.g.col)
    row = out["config1_bfs_rmat16_t128_block"]
    if ref is None:
        row["cpu_baseline"] = {
            "value": None, "note": "reference not installed in baseline/_ref;"
            " BASELINE.md §2 measured 3.08 s (1 core) in the build container"}
    else:
        ok = (np.array_equal(ref["dist"], G16.dist.cpu().numpy())
              and np.array_equal(ref["counts"], G16.counts.cpu().numpy()))
        row["cpu_baseline"] = {
            "value": e16 / ref["seconds"] / 1e9, "unit": "GTEPS",
            "seconds": ref["seconds"], "cores": 1, "kind": "reference",
            "sample": "dynoptc.bench.run_reference (BFS_NOCDP on the "
                      "reference's simulator) on the same RMAT-16 CSR, "
                      "unmodified reference from baseline/_ref"}
        row["parity"] = ("dist and counts equal the reference's own run"
                         if ok else "MISMATCH vs the reference")
        row["vs_reference_cpu"] = ref["seconds"] * 1e3 / ms
    del G16
    # BFS RMAT-22
    G = DeviceGraph(SCALE, SEED, weights=False)
    cfg = _cfg(BEST["bfs"])
    runs = [run_dev("bfs", G, cfg, stream) for _ in range(5)]
    ms = statistics.median(r["ns_device"] for r in runs) / 1e6
    counts = G.counts.cpu().numpy()
    e_t = int(counts.astype(np.int64).sum())
    e_reach, alg = graph_traffic("bfs", G, G.dist.cpu().numpy(), 0)
    naive = run_dev("bfs", G, _cfg(dict(parent_block=32)), stream)
    agg_ms = {a: run_dev("bfs", G, _cfg(dict(agg=a)), stream)["ns_device"]
              / 1e6 for a in ("warp", "block", "grid")}
    matched = matched_agg_only(
        BEST["bfs"], lambda p: statistics.median(
            run_dev("bfs", G, _cfg(p), stream)["ns_device"]
            for _ in range(3)) / 1e6)
    ceil = read_ceilings()
    vs = ceil.get("visit_spread")
    l2c = None
    if vs and ceil.get("m"):
        # the same per-edge visit as a flat, perfectly balanced kernel over
        # all m edges (L2-atomic / probe bound): time for e_t edges
        flat_ms = vs["ms"] * e_t / ceil["m"]
        l2c = {"ceiling": "flat visit of every edge, spread counts + merged "
                          "RED + probe + CAS (tools/ceiling.cu visit_spread)",
               "ceiling_g_edges_per_s": ceil["m"] / vs["ms"] / 1e6,
               "frac": flat_ms / ms,
               "red_hashed_g_ops_per_s":
                   ceil.get("red_hashed", {}).get("g_ops_per_s"),
               "probe_g_ops_per_s":
                   ceil.get("probe_targets", {}).get("g_ops_per_s"),
               "source": "profiles/ceilings.json"}
    out["bfs_rmat22"] = {"gteps": e_t / ms / 1e6, "ms": ms,
                         "l2_ceiling": l2c,
                         "vs_agg_only_matched": min(matched.values()) / ms,
                         "agg_only_matched_ms": matched,
                         "levels": runs[0]["iterations"],
                         "launches": runs[0]["num_launches"],
                         "gbps_alg": alg / (ms * 1e6),
                         "vs_naive_cdp": naive["ns_device"] / 1e6 / ms,
                         "vs_agg_only": min(agg_ms.values()) / ms,
                         "policy": BEST["bfs"]}
    if not quick:
        from oracle import oracle
        threads = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        wd, wc, _ = oracle.bfs(G.g.rowptr, G.g.col, nthreads=threads)
        dt = time.perf_counter() - t0
        # G holds the outputs of the last device run (every policy above
        # computes the same dist / counts)
        out["bfs_rmat22"]["parity"] = (
            "bit-exact vs oracle (dist, counts)"
            if np.array_equal(G.dist.cpu().numpy(), wd)
            and np.array_equal(G.counts.cpu().numpy(), wc) else "MISMATCH")
        out["bfs_rmat22"]["cpu_baseline"] = {
            "value": e_t / dt / 1e9, "unit": "GTEPS", "cores": threads,
            "kind": "port", "seconds": dt,
            "sample": "full BFS rmat-22 from vertex 0, oracle/oracle.c"}
    del G
    torch.cuda.empty_cache()
    # TC RMAT-22
    bench, wl = load("tc", f"rmat:{SCALE}:seed{SEED}")
    dev = torch.device("cuda", torch.cuda.current_device())
    rp = torch.from_numpy(wl.buffers["rowptr"]).to(dev)
    col = torch.from_numpy(wl.buffers["col"]).to(dev)
    tri = torch.zeros(1, dtype=torch.int64, device=dev)
    m = int(wl.buffers["col"].shape[0])

    def tc_once(c):
        st = _lib.DpStats()
        _lib.check(lib.dp_tc_dev(rp.data_ptr(), col.data_ptr(), wl.n, m, 0, m,
                                 ctypes.byref(c), tri.data_ptr(), stream,
                                 ctypes.byref(st)))
        return _lib.stats_dict(st)
    c = _cfg(BEST["tc"])
    tc_once(c)
    runs = [tc_once(c) for _ in range(5)]
    ms = statistics.median(r["ns_device"] for r in runs) / 1e6
    from paper_2201_02789_b200.bench.benchmarks import tc_traffic
    alg = tc_traffic(wl.buffers["rowptr"], wl.buffers["col"])
    ntri = int(tri.item())
    # TC is bound by hash probes (instruction issue), not by HBM: the
    # probes of the rank-ordered CSR+ (the part of N+(u) above v for every
    # edge u -> v) per second, next to the SM throughput ncu measured
    deg = np.diff(wl.buffers["rowptr"].astype(np.int64))
    probes = int((deg * (deg - 1) // 2).sum())
    out["tc_rmat22"] = {"triangles": ntri, "ms": ms,
                        "triangles_per_s": ntri / (ms * 1e-3),
                        "edges_per_s": m / (ms * 1e-3),
                        "probes": probes,
                        "probes_per_s": probes / (ms * 1e-3),
                        "bound": "hash probes (SM issue; ncu child SM "
                                 "throughput 78 %, profiles/r02/"
                                 "ncu_full_tc_r02.json); gbps_alg is the "
                                 "§8(d) model, which counts L2-resident list "
                                 "reads as HBM bytes",
                        "gbps_alg": alg / (ms * 1e6), "policy": BEST["tc"]}
    if not quick:
        naive_ms = tc_once(_cfg(dict()))["ns_device"] / 1e6
        agg_ms = {a: tc_once(_cfg(dict(agg=a)))["ns_device"] / 1e6
                  for a in ("warp", "block", "grid")}
        from oracle import oracle
        threads = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        cpu_tri = oracle.tc(wl.buffers["rowptr"], wl.buffers["col"],
                            nthreads=threads)
        dt = time.perf_counter() - t0
        matched = matched_agg_only(
            BEST["tc"], lambda p: statistics.median(
                tc_once(_cfg(p))["ns_device"] for _ in range(2)) / 1e6)
        out["tc_rmat22"].update({
            "vs_agg_only_matched": min(matched.values()) / ms,
            "agg_only_matched_ms": matched,
            "vs_naive_cdp": naive_ms / ms,
            "vs_agg_only": min(agg_ms.values()) / ms,
            "parity": "exact vs oracle" if cpu_tri == ntri else "MISMATCH",
            "cpu_baseline": {"value": cpu_tri / dt, "unit": "triangles/s",
                             "cores": threads, "kind": "port",
                             "seconds": dt,
                             "sample": "full TC rmat-22, oracle/oracle.c"}})
    del rp, col
    # BT 25k curves.  Device time on device-resident buffers, calls back to
    # back (dp_bt_dev), for every policy compared: the host-buffer call idles
    # the GPU between runs and a ~30 us kernel then starts at lower clocks
    # (45-63 vs 28 us for the same kernel, profiles/r02/bt25k_paths_r02.txt)
    bench, wl = load("bt", "curves:25000:seed1")
    rep0 = run_config(bench, wl, BenchConfig(**BEST["bt"]))[0]
    nv = int(rep0.arrays["ntess"].astype(np.int64).sum())

    def bt_ms(p):
        row = bt_stream_row(25000, True, p)
        assert row["vertices"] == nv, (row["vertices"], nv)
        return row["ms"]
    ms = bt_ms(BEST["bt"])
    out["bt_25k"] = {"curves_per_s": 25000 / (ms * 1e-3), "ms": ms,
                     "vertices": nv, "gbps_alg": (36 * 25000 + 8 * nv) /
                     (ms * 1e6), "policy": BEST["bt"],
                     "ms_host_call": rep0.ns_device / 1e6}
    # BASELINE config 2 as written: coarsening + multi-block aggregation
    c2 = dict(threshold=64, cfactor=16, agg="multiblock", group_size=4,
              parent_block=256, child_block=32, serial="warp")
    ms2 = bt_ms(c2)
    naive_ms = bt_ms({})
    out["config2_bt_25k_c_multiblock"] = {
        "curves_per_s": 25000 / (ms2 * 1e-3), "ms": ms2,
        "device_launches": run_config(bench, wl,
                                      BenchConfig(**c2))[0].num_launches,
        "vs_naive_cdp": naive_ms / ms2, "policy": c2}
    agg_ms = {a: bt_ms(dict(agg=a)) for a in ("warp", "block", "grid")}
    matched = matched_agg_only(BEST["bt"], bt_ms)
    out["bt_25k"]["vs_agg_only_matched"] = min(matched.values()) / ms
    out["bt_25k"]["agg_only_matched_ms"] = matched
    out["bt_25k"]["vs_naive_cdp"] = naive_ms / ms
    out["bt_25k"]["vs_agg_only"] = min(agg_ms.values()) / ms
    out["bt_1m_streaming"] = bt_stream_row(1000000, quick)
    if quick:
        return out
    from oracle import oracle
    threads = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    for _ in range(10):
        oracle.bt(wl.buffers["cp"], int(wl.buffers["max_tess"]),
                  float(wl.buffers["scale"]), nthreads=threads)
    dt = (time.perf_counter() - t0) / 10
    out["bt_25k"]["cpu_baseline"] = {
        "value": 25000 / dt, "unit": "curves/s", "cores": threads,
        "kind": "port", "seconds": dt,
        "sample": "25k curves (fp64 vertices), oracle/oracle.c OpenMP over "
                  "curves"}
    from paper_2201_02789_b200.bench import run_reference
    from paper_2201_02789_b200.bench.benchmarks import Workload

    def med(bench, wl, pol, k=4):
        reps = [run_config(bench, wl, BenchConfig(**pol))[0]
                for _ in range(k)]
        return statistics.median(r.ns_device for r in reps[1:]) / 1e6, reps[-1]
    # MST (MSTF row) on the symmetrised RMAT-22
    bench, wl = load("mstf", f"rmat:{SCALE}:seed{SEED}")
    ms, rep = med(bench, wl, BEST["mstf"])
    naive_ms, _ = med(bench, wl, dict(), k=1 + 1)
    ref = run_reference(bench, wl)
    agg_ms = {a: med(bench, wl, dict(agg=a), k=2)[0]
              for a in ("warp", "block", "grid")}
    m = int(wl.buffers["col"].shape[0])
    b = wl.buffers
    t0 = time.perf_counter()
    cpu = oracle.mst(b["rowptr"], b["col"], b["weight"], b["eid"])
    dt = time.perf_counter() - t0
    out["mst_rmat22"] = {
        "ms": ms, "edge_slots": m, "edges_per_s": m / (ms * 1e-3),
        "forest_weight": int(rep.arrays["weight"][0]),
        "forest_edges": int(rep.arrays["weight"][1]),
        "rounds": rep.iterations, "vs_naive_cdp": naive_ms / ms,
        "vs_agg_only": min(agg_ms.values()) / ms,
        "vs_nocdp": ref.ns_device / 1e6 / ms, "policy": BEST["mstf"],
        "parity": ("bit-exact vs oracle"
                   if np.array_equal(rep.arrays["in_mst"], cpu[0])
                   and rep.arrays["weight"].tolist() == [cpu[1], cpu[2]]
                   else "MISMATCH"),
        "cpu_baseline": {"value": m / dt, "unit": "edge slots/s",
                         "cores": 1, "kind": "port", "seconds": dt,
                         "sample": "Kruskal over rmat-22 (symmetrised), "
                                   "oracle/oracle.c; one core: Kruskal's "
                                   "sorted union-find sweep is sequential "
                                   "(it is the checker's unique-forest "
                                   "definition, not a parallel MST)"}}
    del wl
    # SP: 20 synchronous sweeps of random 5-SAT
    bench, wl = load("sp", "ksat5:200000:seed1")
    wl = Workload(wl.spec, dict(wl.buffers, max_sweeps=20, eps=0.0), wl.n,
                  wl.payload)
    ms, rep = med(bench, wl, BEST["sp"])
    grid_ms, _ = med(bench, wl, dict(agg="grid"), k=2)
    ref = run_reference(bench, wl)
    ne = int(wl.buffers["lits"].shape[0])
    t0 = time.perf_counter()
    cpu = oracle.sp(wl.payload, wl.buffers["eta0"], 20, 0.0,
                    nthreads=threads)
    dt = time.perf_counter() - t0
    from paper_2201_02789_b200.bench.benchmarks import sp_traffic
    alg = sp_traffic(wl.payload.nvars, ne, wl.payload.k, rep.iterations)
    try:  # DRAM bytes of one sweep's three passes, committed ncu capture
        cap = json.loads((ROOT / "profiles" / "r02" /
                          "ncu_full_sp_final_r02.json").read_text())
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        dram = sum(float(l[m]) * scale[cap["units"][m]]
                   for l in cap["launches"]
                   for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except Exception:  # noqa: BLE001
        dram = None
    out["sp_ksat5_200k"] = {
        "ms": ms, "sweeps": rep.iterations, "edges": ne,
        "edge_updates_per_s": ne * rep.iterations / (ms * 1e-3),
        "gbps_alg": alg / (ms * 1e-3) / 1e9,
        "frac_hbm": alg / (ms * 1e-3) / 1e9 / hbm_peak()[0],
        "alg_bytes_per_sweep": sp_traffic(wl.payload.nvars, ne,
                                          wl.payload.k, 1) -
                               sp_traffic(wl.payload.nvars, ne,
                                          wl.payload.k, 0),
        "dram_bytes_per_sweep_ncu": dram,
        "bound": "latency of the random fp64 eta / product gathers "
                 "(profiles/r02/ncu_full_sp_final_r02.json)",
        "vs_agg_only_grid": grid_ms / ms,
        "vs_nocdp": ref.ns_device / 1e6 / ms, "policy": BEST["sp"],
        "parity": ("within 1e-5 of the oracle"
                   if np.allclose(rep.arrays["eta"], cpu[0], rtol=1e-5,
                                  atol=1e-7) else "MISMATCH"),
        "cpu_baseline": {"value": ne * 20 / dt, "unit": "edge updates/s",
                         "cores": threads, "kind": "port", "seconds": dt,
                         "sample": "20 sweeps of ksat5:200000, "
                                   "oracle/oracle.c (fp64, OpenMP over "
                                   "variables and clauses)"},
        "naive_cdp": "not timed (37 s, 88 M launches; profiles/sp_time_r01)"}
    return out


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------

def init_dist(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    launched = world > 1 or ("MASTER_ADDR" in os.environ
                             and "RANK" in os.environ)
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if launched and not torch.distributed.is_initialized():
        if args.impl == "ours":  # one process per GPU, bound to LOCAL_RANK
            torch.distributed.init_process_group(
                "nccl", device_id=torch.device("cuda", local))
        else:
            torch.distributed.init_process_group("gloo")
    return world, rank, local


def max_over_ranks(x: float) -> float:
    import torch
    if not torch.distributed.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64,
                     device="cuda" if torch.distributed.get_backend() ==
                     "nccl" else "cpu")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def exchange_self_check(kind: str, exchange: str, world: int, rank: int,
                        dev) -> tuple[bool, str]:
    """Run the partitioned `kind` ("sssp" | "bfs") on RMAT-16 through
    `exchange` ("peer" | "a2a") and compare the gathered result with the
    oracle; the verdict is agreed over ranks (min), so every rank takes the
    same branch.  Runs before a partitioned timed region: the fused
    symmetric-memory exchange is used only where it has just proved itself
    bit-exact on this box."""
    import torch
    from paper_2201_02789_b200 import dist as pdist
    from oracle import oracle
    collective = torch.distributed.is_initialized()
    rowptr, col = oracle.rmat(16, SEED)
    n = rowptr.shape[0] - 1
    ok, err = False, ""
    try:
        if kind == "sssp":
            w = oracle.edge_weights(n, col.shape[0], SEED)
            rp_p, col_p, w_p = pdist.partition_csr(rowptr, col, world, rank,
                                                   w)
            cfg = _cfg(BEST["sssp"])
            if exchange == "peer":
                ex = pdist.PeerCollective() if collective else \
                    pdist.PeerLocal()
                buf = ex.alloc(n, world, dev)
                part = pdist.SsspPeerPart(rp_p, col_p, w_p, n, world, rank, 0,
                                          buf, dev)
                ex.bind([part])
                got, _ = pdist.sssp_1d_peer_solve([part], cfg, ex)
            else:
                part = pdist.SsspPart(rp_p, col_p, w_p, n, world, rank, 0,
                                      dev)
                ex = pdist.CollectiveExchange() if collective else \
                    pdist.LocalExchange()
                got, _ = pdist.sssp_1d([part], pdist.DeviceSsspOps(cfg), ex)
            want, _ = oracle.sssp(rowptr, col, w, nthreads=0)
            ok = bool(np.array_equal(got.cpu().numpy(), want))
        else:
            rp_p, col_p = pdist.partition_csr(rowptr, col, world, rank)
            ops = pdist.DeviceBfsOps(_cfg(BEST["bfs"]))
            if exchange == "peer":
                ex = pdist.PeerCollective() if collective else \
                    pdist.PeerLocal()
                buf = ex.alloc(n, world, dev)
                part = pdist.BfsPart(rp_p, col_p, n, world, rank, 0, dev,
                                     dist=buf, spread=True)
                ex.bind([part])
                got_d, got_c, _ = pdist.bfs_1d_peer_solve(
                    [part], _cfg(BEST["bfs"]), ex)
            else:
                part = pdist.BfsPart(rp_p, col_p, n, world, rank, 0, dev,
                                     spread=True)
                ex = pdist.CollectiveExchange() if collective else \
                    pdist.LocalExchange()
                got_d, got_c, _ = pdist.bfs_1d([part], ops, ex)
            wd, wc, _ = oracle.bfs(rowptr, col, nthreads=0)
            ok = bool(np.array_equal(got_d.cpu().numpy(), wd)
                      and np.array_equal(got_c.cpu().numpy(), wc))
        if not ok:
            err = "result differs from the oracle"
    except Exception as e:  # noqa: BLE001 - reported, then the fallback
        err = f"{type(e).__name__}: {e}"
    if collective:
        t = torch.tensor([int(ok)], dtype=torch.int32, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
        ok = bool(int(t.item()))
        if not ok and not err:
            err = "another rank failed"
    torch.cuda.synchronize()
    return ok, err


def choose_exchange(kind: str, requested: str, world: int, rank: int,
                    dev) -> tuple[str, str]:
    """The exchange the timed region will use, after the RMAT-16 self-check
    (peer falls back to the NCCL all-to-all); returns (exchange, note)."""
    ok, err = exchange_self_check(kind, requested, world, rank, dev)
    if ok:
        return requested, f"{requested}: RMAT-16 self-check bit-exact"
    note = f"{requested} failed the RMAT-16 self-check ({err})"
    if requested == "peer":
        print(f"[bench] {note}; falling back to the all-to-all exchange",
              file=sys.stderr)
        ok2, err2 = exchange_self_check(kind, "a2a", world, rank, dev)
        return "a2a", note + ("; a2a: self-check bit-exact" if ok2 else
                              f"; a2a ALSO FAILED ({err2})")
    return requested, note


def arm_sssp_partitioned(args, world, rank, local):
    """N > 1: the headline SSSP over a cyclic 1D vertex partition, one part
    per rank, per-round NCCL all-to-all of improving remote relaxations
    (paper_2201_02789_b200/dist.py).  Same metric: E_reach / t."""
    import torch
    from paper_2201_02789_b200 import _lib
    from paper_2201_02789_b200 import dist as pdist
    from paper_2201_02789_b200.bench import graphs
    from paper_2201_02789_b200.bench.graphs import UNREACHED
    _lib.device()
    dev = torch.device("cuda", torch.cuda.current_device())
    g = graphs.rmat_graph(SCALE, SEED)
    w = graphs.edge_weights(g, SEED)
    rp_p, col_p, w_p = pdist.partition_csr(g.rowptr, g.col, world, rank, w)
    collective = torch.distributed.is_initialized()
    exchange, check = choose_exchange("sssp", args.exchange, world, rank, dev)
    part = ex = None
    if exchange == "peer":
        # fused exchange: remote relaxations are atomicMin into the owner's
        # dist through symmetric memory (NVLink peer addresses)
        try:
            ex = pdist.PeerCollective() if collective else pdist.PeerLocal()
            buf = ex.alloc(g.n, world, dev)
            part = pdist.SsspPeerPart(rp_p, col_p, w_p, g.n, world, rank, 0,
                                      buf, dev)
            ex.bind([part])
            ops = _cfg(BEST["sssp"])
            # rounds looped in the library, flags OR-ed on the device
            run_rounds = pdist.sssp_1d_peer_solve
        except Exception as e:  # noqa: BLE001 - fall back to the NCCL a2a
            print(f"[bench] symmetric memory unavailable ({e}); using the "
                  f"all-to-all exchange", file=sys.stderr)
            exchange = "a2a"
    if exchange == "a2a":
        part = pdist.SsspPart(rp_p, col_p, w_p, g.n, world, rank, 0, dev)
        ops = pdist.DeviceSsspOps(_cfg(BEST["sssp"]))
        ex = pdist.CollectiveExchange() if collective else \
            pdist.LocalExchange()
        run_rounds = pdist.sssp_1d
    stream_obj = torch.cuda.current_stream()

    def step():
        # peer: the solve initialises its own state, and each rank keeps its
        # owned distances (gathered once after the timed region)
        if exchange != "peer":
            part.reset(0)
            return run_rounds([part], ops, ex)
        return run_rounds([part], ops, ex, gather=False)
    with ClockSampler(local) as clk:
        total_ms, outs = timed_steps(step, args.steps, args.warmup,
                                     stream_obj)
    dist_t, rounds = outs[-1]
    if dist_t is None:
        dist_t = ex.dist([part])
    # peer: one stats entry per solve (= step); a2a: one per round of the
    # last step (reset() clears them)
    launches_timed = int(sum(s["kernel_launches"] + s["num_launches"]
                             for s in part.stats[-args.steps:])) \
        if exchange == "peer" else \
        int(sum(s["kernel_launches"] + s["num_launches"]
                for s in part.stats)) * args.steps
    remote_per_round = statistics.mean(
        s["remote_ops"] / max(s["iterations"], 1) for s in part.stats[-3:])
    t_max = max_over_ranks(total_ms)
    ms_step = t_max / args.steps
    dist_h = dist_t.cpu().numpy()
    deg = np.diff(g.rowptr.astype(np.int64))
    e_reach = int(deg[dist_h < UNREACHED].sum())
    # e2e: this rank's part copied from pinned host memory every step
    hp = [torch.from_numpy(x).pin_memory() for x in (rp_p, col_p, w_p)]
    out_h = torch.empty(part.n_local, dtype=torch.int32).pin_memory()
    e2e = []
    for i in range(3):
        torch.cuda.synchronize()
        if torch.distributed.is_initialized():
            torch.distributed.barrier()
        t0 = time.perf_counter()
        part.rowptr.copy_(hp[0], non_blocking=True)
        part.col.copy_(hp[1], non_blocking=True)
        part.weight.copy_(hp[2], non_blocking=True)
        if exchange != "peer":
            part.reset(0)
            run_rounds([part], ops, ex)
        else:
            run_rounds([part], ops, ex, gather=False)
        out_h.copy_(part.dist, non_blocking=True)
        torch.cuda.synchronize()
        if i:
            e2e.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(statistics.median(e2e))
    h2d = sum(x.numel() * 4 for x in hp)
    subs = None if args.quick else partitioned_workloads(args, world, rank,
                                                         local)
    if rank != 0:
        return
    from oracle import oracle
    want, _ = oracle.sssp(g.rowptr, g.col, w, nthreads=0)
    print(json.dumps({
        "metric": "GTEPS (SSSP RMAT-22, T+C+A CDP2)",
        "value": e_reach * args.steps / (t_max * 1e-3) / 1e9,
        "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic RMAT (Graph500 a,b,c=.57,.19,.19, seed 1, "
                "edge factor 16), weights U[1,9]",
        "config": {"workload": f"sssp rmat-{SCALE} from vertex 0",
                   "n": g.n, "m": g.m, "e_reach": e_reach, "rounds": rounds,
                   "policy": BEST["sssp"],
                   "parallelism": f"1d-cyclic-partition x{world}",
                   "exchange": ("fused: remote atomicMin into the owner's "
                                "dist via symmetric memory; round flags "
                                "OR-ed on the device through symmetric-memory "
                                "signal slots, rounds looped in the library "
                                "(dp_sssp_part_solve_peer)"
                                if exchange == "peer" else
                                "NCCL all-to-all of (v, alt) pairs + apply"),
                   "exchange_check": check,
                   "remote_atomics_per_round_rank0": remote_per_round,
                   "l2": "inputs exceed L2; no flush"},
        "parity": "bit-exact vs oracle" if np.array_equal(dist_h, want)
        else "MISMATCH",
        "e2e": {"value": e_reach / e2e_s / 1e9, "unit": "GTEPS",
                "h2d_bytes_per_step": h2d * world,
                "d2h_bytes_per_step": g.n * 4,
                "ms_per_step": e2e_s * 1e3},
        "gpu_launches": launches_timed,
        "clocks": clk.summary(),
        "partitioned_workloads": subs}), flush=True)


def arm_ours(args, world, rank, local):
    import torch
    if world > 1 or args.partitioned:
        return arm_sssp_partitioned(args, world, rank, local)
    from paper_2201_02789_b200 import _lib
    from oracle import oracle  # checker + cpu_baseline only
    _lib.device()
    stream_obj = torch.cuda.current_stream()
    stream = ctypes.c_void_p(stream_obj.cuda_stream)
    G = DeviceGraph(SCALE, SEED, weights=True)
    cfg = _cfg(BEST["sssp"])
    with ClockSampler(local) as clk:
        total_ms, stats = timed_steps(lambda: run_dev("sssp", G, cfg, stream,
                                                      raw=True),
                                      args.steps, args.warmup, stream_obj)
    lib_ms = statistics.mean(s["ns_device"] for s in stats) / 1e6
    if args.profile:  # ncu pass: the timed steps only
        print(json.dumps({"profile": True, "ms": total_ms / args.steps}))
        return
    dist = G.dist.cpu().numpy()
    rounds = int(stats[-1]["iterations"])
    e_reach, alg_run = graph_traffic("sssp", G, dist, rounds)
    t_max = max_over_ranks(total_ms)
    ms_step = t_max / args.steps
    value = world * e_reach * args.steps / (t_max * 1e-3) / 1e9
    line = {"metric": "GTEPS (SSSP RMAT-22, T+C+A CDP2)", "value": value,
            "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic RMAT (Graph500 a,b,c=.57,.19,.19, seed 1, "
                    "edge factor 16), weights U[1,9]",
            "config": headline_config(G.n, G.m, e_reach),
            "details": {"rounds": rounds, "policy": BEST["sssp"],
                        "parallelism": "single",
                        "lib_device_ms_per_step": lib_ms},
            "gpu_launches": int(sum(s["kernel_launches"] + s["num_launches"]
                                    for s in stats))}
    if rank != 0:
        return
    # parity of the timed run against the oracle (checker, not measured)
    want, _ = oracle.sssp(G.g.rowptr, G.g.col, G.w, nthreads=0)
    line["parity"] = "bit-exact vs oracle" if np.array_equal(dist, want) \
        else "MISMATCH"
    # roofline: the dominant kernel = per-round parent grid incl. children
    steps_ns = [s["ns_kernel_sum"] / max(s["iterations"], 1) for s in stats]
    per_round = statistics.mean(steps_ns)
    alg_round = alg_run / rounds
    peak, peak_src = hbm_peak()
    achieved = alg_round / per_round  # bytes/ns == GB/s
    line["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peak,
                        "unit": "GB/s", "frac": achieved / peak,
                        "traffic": read_traffic(), "peak_source": peak_src,
                        "kernel": "parent_kernel<SsspApp,multiblock> round "
                                  "(+CDP2 children)",
                        "alg_bytes_per_launch": alg_round,
                        "ms_per_launch": per_round / 1e6,
                        # the same round against its measured DRAM bytes
                        # (ncu, profiles/traffic.json): dist probes hit L1/L2
                        "achieved_dram": (read_traffic() or 0) / per_round,
                        "frac_dram": (read_traffic() or 0) / per_round / peak,
                        "share_of_step": sum(s["ns_kernel_sum"] for s in stats)
                        / (total_ms * 1e6)}
    line["clocks"] = clk.summary()
    # e2e through the host-buffer C-ABI; weights travel as packed nibbles
    # (weight_bits = 4: packed on the host chunk by chunk ahead of the copy,
    # 1/8 of the int32 bytes; the resident device path keeps int32, which
    # measured faster there: 1.66 vs 1.72 ms, profiles/r02/ab_wbits_r02.txt)
    e = e2e_sssp(G, _cfg(dict(BEST["sssp"], **E2E_EXTRA)),
                 max(2, min(args.steps, 5)))
    line["e2e"] = {"value": e_reach / e["seconds"] / 1e9, "unit": "GTEPS",
                   "h2d_bytes_per_step": int(e["h2d"]),
                   "d2h_bytes_per_step": int(e["d2h"]),
                   "ms_per_step": e["seconds"] * 1e3,
                   "policy_extra": E2E_EXTRA,
                   "copy_floor_ms": e["copy_floor_s"] * 1e3,
                   "copy_floor_note": "plain pinned H2D of h2d_bytes + D2H "
                   "of one dist on this box, no compute"}
    assert np.array_equal(e["dist"], want)
    # speed-ups over the naive-CDP and aggregation-only builds (same device)
    naive = run_dev("sssp", G, _cfg(dict()), stream)
    aggonly = {a: run_dev("sssp", G, _cfg(dict(agg=a)), stream)
               for a in ("warp", "block", "grid")}
    best_agg = min(aggonly, key=lambda a: aggonly[a]["ns_device"])
    line["vs_naive_cdp"] = naive["ns_device"] / 1e6 / ms_step
    line["vs_agg_only"] = aggonly[best_agg]["ns_device"] / 1e6 / ms_step
    line["baselines_ms"] = {"naive_cdp": naive["ns_device"] / 1e6,
                            "naive_cdp_launches": naive["num_launches"],
                            **{f"agg_only_{a}": r["ns_device"] / 1e6
                               for a, r in aggonly.items()}}
    matched = matched_agg_only(
        BEST["sssp"], lambda p: statistics.median(
            run_dev("sssp", G, _cfg(p), stream)["ns_device"]
            for _ in range(3)) / 1e6)
    line["vs_agg_only_matched"] = min(matched.values()) / ms_step
    line["baselines_ms"]["agg_only_matched"] = matched
    cpu = cpu_baseline_sssp(G, len(os.sched_getaffinity(0)))
    cpu.pop("dist")
    line["cpu_baseline"] = cpu
    # B200 work-efficient rounds (frontier knob): a vertex relaxes only when
    # its distance changed since its last relaxation.  Same distances; not
    # the headline, which keeps SSSP_CDP's every-reached-vertex rounds.
    fcfg = _cfg(FRONTIER_POLICY)
    f_ms, f_stats = timed_steps(lambda: run_dev("sssp", G, fcfg, stream,
                                                raw=True),
                                args.steps, args.warmup, stream_obj)
    f_ms = max_over_ranks(f_ms) / args.steps
    fdist = G.dist.cpu().numpy()
    line["sssp_frontier"] = {
        "value": e_reach / (f_ms * 1e-3) / 1e9, "unit": "GTEPS",
        "ms_per_step": f_ms, "rounds": int(f_stats[-1]["iterations"]),
        "speedup_vs_headline": ms_step / f_ms,
        "parity": "bit-exact vs oracle" if np.array_equal(fdist, want)
        else "MISMATCH", "policy": FRONTIER_POLICY}
    if not args.quick:
        del G
        torch.cuda.empty_cache()
        line["workloads"] = extra_workloads(stream, args.quick)
        torch.cuda.empty_cache()
        line["partitioned_workloads"] = partitioned_workloads(args, 1, 0,
                                                              local)
        wl = line["workloads"]
        ratios = {"sssp_rmat22": line["vs_agg_only_matched"],
                  **{k: wl[k]["vs_agg_only_matched"]
                     for k in ("bfs_rmat22", "tc_rmat22", "bt_25k")
                     if "vs_agg_only_matched" in wl.get(k, {})}}
        line["vs_agg_only_matched_geomean"] = {
            "value": float(np.exp(np.mean(np.log(list(ratios.values()))))),
            "over": ratios,
            "definition": "tuned T+C+A device time vs the best aggregation-"
                          "only build (T=0, C=1) with the same parent/child "
                          "blocks, over warp / block / one-group multiblock "
                          "/ grid"}
    print(json.dumps(line), flush=True)


def arm_bfs26(args, world, rank, local):
    """BASELINE config 5: BFS on RMAT-26 over a cyclic 1D vertex partition
    (one part per rank).  One step = one full BFS from vertex 0.  GTEPS =
    examined edges / t."""
    line = measure_bfs26(args, world, rank, local, parity=True)
    if rank == 0:
        print(json.dumps(line), flush=True)


def measure_bfs26(args, world, rank, local, parity: bool = True,
                  steps: int = 0):
    """The config-5 measurement (rank 0 gets the line, others None).
    parity: check dist / counts / levels against the oracle on the host
    (RMAT-26: ~25 s of OpenMP); the exchange itself is always verified on
    RMAT-16 first (choose_exchange)."""
    import torch
    from paper_2201_02789_b200 import _lib
    from paper_2201_02789_b200 import dist as pdist
    _lib.device()
    dev = torch.device("cuda", torch.cuda.current_device())
    scale = args.scale or 26
    collective = torch.distributed.is_initialized()
    exchange, check = choose_exchange("bfs", args.exchange, world, rank, dev)
    rp, col = pdist.rmat_part_device(scale, SEED, world, rank, dev)
    part = None
    if exchange == "peer":
        # fused exchange: remote discoveries are CAS'd into the owner's dist
        # through symmetric memory
        try:
            ex = pdist.PeerCollective() if collective else pdist.PeerLocal()
            buf = ex.alloc(1 << scale, world, dev)
            part = pdist.BfsPart(rp, col, 1 << scale, world, rank, 0, dev,
                                 dist=buf, spread=True)
            ex.bind([part])
            run_levels = pdist.bfs_1d_peer_solve
        except Exception as e:  # noqa: BLE001 - fall back to the NCCL a2a
            print(f"[bench] symmetric memory unavailable ({e}); using the "
                  f"all-to-all exchange", file=sys.stderr)
            exchange = "a2a"
    if exchange == "a2a":
        part = pdist.BfsPart(rp, col, 1 << scale, world, rank, 0, dev,
                             spread=True)
        ex = pdist.CollectiveExchange() if collective else \
            pdist.LocalExchange()
        run_levels = pdist.bfs_1d
    del rp, col
    ops = _cfg(BEST["bfs"]) if exchange == "peer" else \
        pdist.DeviceBfsOps(_cfg(BEST["bfs"]))
    stream_obj = torch.cuda.current_stream()

    def step():
        # peer: the solve initialises its own state, and each rank keeps its
        # part of dist / counts (combined once after the timed region)
        if exchange != "peer":
            part.reset(0)
            return run_levels([part], ops, ex)
        return run_levels([part], ops, ex, gather=False)
    steps = steps or args.steps
    with ClockSampler(local) as clk:
        total_ms, outs = timed_steps(step, steps, args.warmup, stream_obj)
    dist_t, counts_t, levels = outs[-1]
    if dist_t is None:
        dist_t = ex.dist([part])
        counts_t = part.natural_counts(ex.counts([part]))
    e_t = int(counts_t.to(torch.int64).sum().item())
    t_max = max_over_ranks(total_ms)
    ms_step = t_max / steps
    remote = statistics.mean(s["remote_ops"] / max(s["iterations"], 1)
                             for s in part.stats[-steps:]) \
        if part.stats and "remote_ops" in part.stats[-1] else 0
    if rank != 0:
        return None
    line = {"metric": f"GTEPS (BFS RMAT-{scale}, 1D partition, T+C+A CDP2)",
            "value": e_t / (ms_step * 1e-3) / 1e9, "unit": "GTEPS",
            "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic RMAT (Graph500, seed 1, edge factor 16)",
            "config": {"workload": f"bfs rmat-{scale} from vertex 0",
                       "levels": levels, "edges_examined": e_t,
                       "policy": BEST["bfs"],
                       "parallelism": f"1d-cyclic-partition x{world}",
                       "exchange": ("fused: remote CAS into the owner's dist "
                                    "via symmetric memory; level flags OR-ed "
                                    "on the device through symmetric-memory "
                                    "signal slots (dp_bfs_part_solve_peer)"
                                    if exchange == "peer" else
                                    "NCCL all-to-all of discovered ids + "
                                    "apply"),
                       "exchange_check": check,
                       "remote_atomics_per_level_rank0": remote},
            "clocks": clk.summary()}
    if not parity:
        line["parity"] = ("not checked at this scale here; the exchange "
                          "passed the RMAT-16 self-check (" + check + ")")
        return line
    # parity at every scale (RMAT-26: 1.07 G edges through the OpenMP oracle
    # on the host; the oracle's own generator, rows unsorted since BFS
    # outputs do not depend on the row order)
    from oracle import oracle
    got_d, got_c = dist_t.cpu().numpy(), counts_t.cpu().numpy()
    del dist_t, counts_t
    t0 = time.perf_counter()
    orp, ocol = oracle.rmat(scale, SEED, sort_rows=False)
    wd, wc, wl = oracle.bfs(orp, ocol, nthreads=0)
    del orp, ocol
    line["parity"] = ("bit-exact vs oracle (dist, counts, levels)"
                      if np.array_equal(got_d, wd)
                      and np.array_equal(got_c, wc) and wl == levels
                      else "MISMATCH")
    line["parity_check_s"] = time.perf_counter() - t0
    return line


def arm_tc(args, world, rank, local):
    """BASELINE config 4: triangle counting on RMAT-22, oriented-edge ranges
    balanced by merge work, one all_reduce(sum).  One step = one count."""
    line = measure_tc(args, world, rank, local)
    if rank == 0:
        print(json.dumps(line), flush=True)


def tc_graph(scale: int, world: int, rank: int):
    """The degree-oriented CSR+ of RMAT-`scale` (host orientation, ~10 s at
    scale 22): built once by rank 0 and shared through /tmp with the other
    ranks of this job, instead of every rank re-orienting on the same host
    cores."""
    import torch
    from paper_2201_02789_b200.bench import load
    if world == 1:
        _, wl = load("tc", f"rmat:{scale}:seed{SEED}")
        return wl.buffers["rowptr"], wl.buffers["col"], wl.n
    tag = os.environ.get("MASTER_PORT", "0")
    path = Path(f"/tmp/dynpar_tc_{scale}_{SEED}_{tag}_{os.getppid()}.npz")
    if rank == 0:
        _, wl = load("tc", f"rmat:{scale}:seed{SEED}")
        np.savez(path, rowptr=wl.buffers["rowptr"], col=wl.buffers["col"])
    torch.distributed.barrier()
    z = np.load(path)
    rp, col = z["rowptr"], z["col"]
    torch.distributed.barrier()
    if rank == 0:
        path.unlink(missing_ok=True)
    return rp, col, int(rp.shape[0]) - 1


def measure_tc(args, world, rank, local, parity: bool = True,
               steps: int = 0):
    import torch
    from paper_2201_02789_b200 import _lib
    from paper_2201_02789_b200 import dist as pdist
    from paper_2201_02789_b200.bench import load
    _lib.device()
    dev = torch.device("cuda", torch.cuda.current_device())
    rp_h, col_h, n = tc_graph(args.scale or SCALE, world, rank)
    rp = torch.from_numpy(rp_h).to(dev)
    col = torch.from_numpy(col_h).to(dev)
    counter = pdist.tc_device_counter(rp, col, n, int(col_h.shape[0]),
                                      _cfg(BEST["tc"]))
    stream_obj = torch.cuda.current_stream()
    rng = pdist.tc_shard(rp_h, col_h)  # host-side partitioning, untimed
    steps = steps or args.steps
    with ClockSampler(local) as clk:
        total_ms, outs = timed_steps(
            lambda: pdist.tc_count_range(rng, counter, dev),
            steps, args.warmup, stream_obj)
    tri = outs[-1]
    t_max = max_over_ranks(total_ms)
    ms_step = t_max / steps
    if rank != 0:
        return None
    line = {
        "metric": f"triangles/s (TC RMAT-{args.scale or SCALE}, edge-range "
                  f"partition)",
        "value": tri / (ms_step * 1e-3), "unit": "triangles/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic RMAT, symmetrised, degree-oriented",
        "config": {"workload": f"tc rmat-{args.scale or SCALE}",
                   "triangles": tri,
                   "oriented_edges": int(col_h.shape[0]),
                   "policy": BEST["tc"],
                   "parallelism": f"edge-range x{world}",
                   "reduce": "one NCCL all_reduce(sum) of the per-rank "
                             "counts per step (inside the timed region)"},
        "clocks": clk.summary()}
    if parity:
        from oracle import oracle
        want = oracle.tc(rp_h, col_h, nthreads=len(os.sched_getaffinity(0)))
        line["parity"] = "exact vs oracle" if want == tri else "MISMATCH"
    return line


def measure_bt(args, world, rank, local, ncurves: int, steps: int = 0):
    """Bezier tessellation partitioned by curve range (even ranges, one
    all_reduce(sum) of the vertex counts per step); BT's tuned policy.  The
    fp64 coordinate checksum and the exact vertex count are compared with
    the oracle after the timed region."""
    import torch
    from paper_2201_02789_b200 import _lib
    from paper_2201_02789_b200 import dist as pdist
    from paper_2201_02789_b200.bench.graphs import (BT_CURV_SCALE,
                                                    BT_MAX_TESS,
                                                    bezier_curves)
    lib = _lib.device()
    dev = torch.device("cuda", torch.cuda.current_device())
    cp_h = np.ascontiguousarray(bezier_curves(ncurves, 1), dtype=np.float32)
    lo, hi = pdist.even_ranges(ncurves, world)[rank]
    k = hi - lo
    cp = torch.from_numpy(cp_h[lo:hi]).to(dev)
    cap = k * 128 + (1 << 16)
    ntess = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    offs = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
    verts = torch.empty((cap, 2), dtype=torch.float32, device=dev)
    cfg = _cfg(BEST["bt"])
    stream_obj = torch.cuda.current_stream()
    used = ctypes.c_int64()
    nv_t = torch.zeros(1, dtype=torch.int64, device=dev)
    stats = []

    def step():
        st = _lib.DpStats()
        _lib.check(lib.dp_bt_dev(cp.data_ptr(), k, BT_MAX_TESS,
                                 BT_CURV_SCALE, ctypes.byref(cfg),
                                 ntess.data_ptr(), offs.data_ptr(),
                                 verts.data_ptr(), cap, ctypes.byref(used),
                                 None, ctypes.byref(st)))
        stats.append(_lib.stats_dict(st))
        nv_t.fill_(used.value)
        if torch.distributed.is_initialized():
            torch.distributed.all_reduce(nv_t)
        return nv_t
    steps = steps or args.steps
    with ClockSampler(local) as clk:
        total_ms, outs = timed_steps(step, steps, args.warmup, stream_obj)
    nv = int(outs[-1].item())
    t_max = max_over_ranks(total_ms)
    ms_step = t_max / steps
    cs = float(verts[:used.value].double().sum().item())
    cs_all = pdist.allreduce_sum_f64([cs], dev)[0] \
        if torch.distributed.is_initialized() else cs
    if rank != 0:
        return None
    from oracle import oracle
    want_nt, want_v = oracle.bt(cp_h, BT_MAX_TESS, BT_CURV_SCALE)
    want_cs = float(np.asarray(want_v, dtype=np.float64).sum())
    ok = int(want_nt.astype(np.int64).sum()) == nv and \
        abs(cs_all - want_cs) <= 1e-6 * max(1.0, abs(want_cs))
    alg = 36 * ncurves + 8 * nv
    return {
        "metric": f"curves/s (BT {ncurves} curves, curve-range partition)",
        "value": ncurves / (ms_step * 1e-3), "unit": "curves/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vertices": nv, "gbps_alg": alg / (ms_step * 1e6),
        "frac_hbm_aggregate": alg / (ms_step * 1e6) / (hbm_peak()[0] * world),
        "policy": BEST["bt"],
        "parallelism": f"curve-range x{world}",
        "reduce": "NCCL all_reduce(sum) of the vertex count per step "
                  "(inside the timed region)",
        "parity": ("vertex count exact, fp64 coordinate checksum within "
                   "1e-6 of the oracle" if ok else "MISMATCH"),
        "clocks": clk.summary()}


def partitioned_workloads(args, world, rank, local) -> dict | None:
    """The north-star's partitioned workloads at this N, measured in the
    same run as the headline so the driver's 1/2/4/8-GPU lines carry their
    scaling: TC RMAT-22 (edge ranges), BT 4 M curves (curve ranges) and BFS
    RMAT-26 (1D partition, fused exchange).  Every rank calls; rank 0 gets
    the dict."""
    import torch
    out = {}
    for name, fn in (
            ("tc_rmat22", lambda: measure_tc(args, world, rank, local,
                                             parity=True, steps=5)),
            # 4 M curves (350 M vertices, 0.7 ms on one B200): large enough
            # that the per-step all_reduce does not hide the 8-GPU scaling
            ("bt_4m_curves", lambda: measure_bt(args, world, rank, local,
                                                4000000, steps=10)),
            ("bfs_rmat26", lambda: measure_bfs26(args, world, rank, local,
                                                 parity=False, steps=3))):
        r = fn()
        torch.cuda.empty_cache()
        if rank == 0:
            out[name] = {k: v for k, v in r.items()
                         if k not in ("higher_is_better", "vs_baseline",
                                      "dtype", "warmup")}
    return out if rank == 0 else None


def arm_bt(args, world, rank, local):
    """BT partitioned by curve range (the north-star's near-linear TC / BT
    scaling target), 1 M curves by default (--scale: curves in millions
    ... or a count)."""
    n = args.scale if args.scale > 64 else (args.scale or 1) * 1000000
    line = measure_bt(args, world, rank, local, n)
    if rank == 0:
        print(json.dumps(line), flush=True)


def read_ceilings() -> dict:
    """Flat-kernel ceilings of the BFS / SSSP edge work measured on the same
    RMAT-22 target stream (tools/ceiling.py --write -> profiles/
    ceilings.json), or {}."""
    try:
        return json.loads((ROOT / "profiles" / "ceilings.json").read_text())
    except Exception:  # noqa: BLE001
        return {}


def read_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/), else null."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text()).get("sssp_round_dram_bytes")
    except Exception:  # noqa: BLE001
        return None


def arm_reference(args, world, rank, local):
    """The reference's CPU path for this workload: the oracle port of
    SSSP_NOCDP (oracle/oracle.c, OpenMP on every host core) — the reference
    itself is pure Python and cannot travel to the GPU box."""
    if rank != 0:
        return
    # the input comes from the oracle's own restatement of the generator:
    # nothing of the product package (nor its library) is loaded in this arm
    from oracle import oracle
    rowptr, col = oracle.rmat(SCALE, SEED)
    n, m = rowptr.shape[0] - 1, col.shape[0]
    w = oracle.edge_weights(n, m, SEED)
    threads = len(os.sched_getaffinity(0))
    for _ in range(args.warmup):
        oracle.sssp(rowptr, col, w, nthreads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        dist, rounds = oracle.sssp(rowptr, col, w, nthreads=threads)
    dt = (time.perf_counter() - t0) / args.steps
    deg = np.diff(rowptr.astype(np.int64))
    e_reach = int(deg[dist < (1 << 30)].sum())
    value = e_reach / dt / 1e9
    sample = (f"full SSSP rmat-{SCALE} from vertex 0 ({rounds} rounds) per "
              f"step, oracle/oracle.c OpenMP")
    print(json.dumps({
        "impl": "reference", "metric": "GTEPS (SSSP RMAT-22, T+C+A CDP2)",
        "value": value, "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic RMAT (Graph500 a,b,c=.57,.19,.19, seed 1, "
                "edge factor 16), weights U[1,9]",
        "config": headline_config(n, m, e_reach),
        "details": {"rounds": rounds, "threads": threads,
                    "input": "oracle.rmat + oracle.edge_weights "
                             "(product library not loaded)"},
        "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--quick", action="store_true",
                    help="headline only (skip the other workloads)")
    ap.add_argument("--exchange", choices=("peer", "a2a"), default="peer",
                    help="partitioned SSSP / BFS-26: fused peer-memory "
                         "relaxation / discovery (default) "
                         "or the NCCL all-to-all exchange")
    ap.add_argument("--workload", choices=("sssp", "bfs26", "tc", "bt"),
                    default="sssp",
                    help="sssp = headline (BASELINE config 3); bfs26 / tc = "
                         "the partitioned multi-GPU configs 5 / 4")
    ap.add_argument("--scale", type=int, default=0,
                    help="override the RMAT scale of bfs26 / tc")
    ap.add_argument("--partitioned", action="store_true",
                    help="run the headline through the 1D-partitioned path "
                         "even at N=1 (exercises the collective code)")
    ap.add_argument("--profile", action="store_true",
                    help="warm-up + timed steps only (for ncu passes)")
    args = ap.parse_args()
    if args.warmup < 3 and not args.profile:
        args.warmup = 3
    world, rank, local = init_dist(args)
    if args.impl == "reference":
        arm_reference(args, world, rank, local)
    elif args.workload == "bfs26":
        arm_bfs26(args, world, rank, local)
    elif args.workload == "tc":
        arm_tc(args, world, rank, local)
    elif args.workload == "bt":
        arm_bt(args, world, rank, local)
    else:
        arm_ours(args, world, rank, local)
    import torch
    if torch.distributed.is_initialized():
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
