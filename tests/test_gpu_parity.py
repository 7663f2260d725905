"""Parity of the sm_100a CUDA path against the reference (B200 only).

Three routes, all through the C-ABI (libdynpar.so):
  1. golden: outputs and memory digests recorded from dynoptc's own
     run_reference / run_config (tests/golden), for every dataset the
     reference's tests use plus RMAT graphs injected into the reference;
  2. counters: num_launches / host_launches / blocks_scheduled of the
     reference's simulator for 17 T/C/A configurations, reproduced by the
     device counters at parent block 32 (the counter oracles of
     tests/test_passes.py);
  3. oracle: the CPU restatement (oracle/) on the same inputs at sizes up
     to RMAT-22, plus size-independent properties of BFS/SSSP results.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle
from paper_2201_02789_b200 import _lib
from paper_2201_02789_b200.bench import (BenchConfig, EquivalenceError,
                                         INF_THRESHOLD, graphs, load,
                                         run_benchmark, run_config,
                                         run_reference, sweep, verify_outputs)
from paper_2201_02789_b200.bench.benchmarks import BENCHMARKS, Workload
from paper_2201_02789_b200.bench.graphs import DatasetSpec, UNREACHED

pytestmark = pytest.mark.gpu

GRAPH_SPECS = ["hand", "powerlaw:150:seed2", "road:180:seed3",
               "powerlaw:150:seed3", "road:160:seed4", "powerlaw:120:seed5",
               "powerlaw:2000:seed1", "road:1000:seed7"]
SIZE_SPECS = ["sizes:100:seed4", "sizes:1024:seed1", "sizes:40:seed3",
              "sizes:20:seed2"]

# B200-only knobs that must not change any output
B200_VARIANTS = [dict(), dict(parent_block=256), dict(child_block=128),
                 dict(serial="warp"), dict(parent_block=128, serial="warp",
                                           child_block=64),
                 dict(persistent=2, parent_block=128, serial="warp"),
                 dict(device_loop=True, parent_block=64),
                 # rows of >= cf_wave logical blocks run uncoarsened
                 dict(cf_wave=2), dict(cf_wave=1, child_block=64),
                 dict(weight_bits=4, serial="warp")]


def _cfg(d):
    return BenchConfig(**d)


def _golden_ref(golden, bench, spec):
    return next(r for r in golden["reference"]
                if r["bench"] == bench and r["dataset"] == spec)


# ---------------------------------------------------------------------------
# 1 + 2: golden outputs and counters from the reference
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("bench_name,spec",
                         [("bfs", s) for s in GRAPH_SPECS]
                         + [("sssp", s) for s in GRAPH_SPECS]
                         + [("manylaunch", s) for s in SIZE_SPECS])
def test_golden_digests_and_counters(bench_name, spec, golden):
    bench, wl = load(bench_name, spec)
    ref = _golden_ref(golden, bench_name, spec)
    nocdp = run_reference(bench, wl)
    assert nocdp.memory_digest == ref["digest"]
    assert nocdp.num_launches == 0
    rows = [r for r in golden["counters"]
            if r["bench"] == bench_name and r["dataset"] == spec]
    assert len(rows) == 17
    for row in rows:
        rep, _ = run_config(bench, wl, BenchConfig(**row["config"]))
        assert rep.memory_digest == ref["digest"], row["config"]
        if bench_name == "sssp":
            continue  # rounds depend on the (real) schedule; outputs do not
        assert (rep.num_launches, rep.host_launches, rep.blocks_scheduled) \
            == (row["num_launches"], row["host_launches"],
                row["blocks_scheduled"]), row["config"]


@pytest.mark.parametrize("knobs", B200_VARIANTS)
@pytest.mark.parametrize("policy", [
    dict(), dict(threshold=8), dict(agg="warp"), dict(agg="block"),
    dict(agg="multiblock", group_size=3), dict(agg="grid"),
    dict(threshold=4, cfactor=4, agg="multiblock", group_size=2),
    dict(cfactor=3, agg="block", agg_threshold=5),
    dict(threshold=INF_THRESHOLD)])
def test_b200_knobs_keep_outputs(policy, knobs, golden):
    for bench_name, spec in (("bfs", "powerlaw:2000:seed1"),
                             ("sssp", "powerlaw:2000:seed1"),
                             ("manylaunch", "sizes:1024:seed1")):
        bench, wl = load(bench_name, spec)
        rep, _ = run_config(bench, wl, BenchConfig(**policy, **knobs))
        assert rep.memory_digest == \
            _golden_ref(golden, bench_name, spec)["digest"], (policy, knobs)


def test_warp_aggregation_launch_count():
    bench, wl = load("manylaunch", "sizes:1024:seed1")
    sizes = wl.payload
    rep, _ = run_config(bench, wl, BenchConfig(agg="warp"))
    warps = {i // 32 for i in range(sizes.shape[0]) if sizes[i] > 0}
    assert rep.num_launches == len(warps)
    rep, _ = run_config(bench, wl, BenchConfig(threshold=32, agg="warp"))
    warps = {i // 32 for i in range(sizes.shape[0]) if sizes[i] >= 32}
    assert rep.num_launches == len(warps)


def test_manylaunch_threshold_launch_count_is_large_parent_count():
    # reference tests/test_bench.py:245-248
    bench, wl = load("manylaunch", "sizes:1024:seed1")
    rep, _ = run_config(bench, wl, BenchConfig(threshold=32))
    assert rep.num_launches == int((wl.payload >= 32).sum())
    assert rep.buffers["out"] == [s * (s + 1) // 2 for s in wl.payload.tolist()]


def _rmat_workload(bench_name, scale, seed):
    g = graphs.rmat_graph(scale, seed)
    spec = DatasetSpec("rmat", scale, seed, f"rmat:{scale}:seed{seed}")
    dist = np.full(g.n, UNREACHED, np.int32)
    dist[0] = 0
    bufs = {"rowptr": g.rowptr, "col": g.col, "dist": dist}
    if bench_name == "bfs":
        bufs["counts"] = np.zeros(g.n, np.int32)
        payload = g
    else:
        w = graphs.edge_weights(g, seed)
        bufs["weight"] = w
        payload = (g, w)
    return BENCHMARKS[bench_name], Workload(spec, bufs, g.n, payload)


@pytest.mark.parametrize("bench_name,scale,seed", [
    ("bfs", 10, 1), ("bfs", 12, 1), ("bfs", 14, 1), ("bfs", 16, 1),
    ("sssp", 10, 1), ("sssp", 12, 2), ("sssp", 14, 1)])
def test_rmat_golden_digests(bench_name, scale, seed, golden):
    rec = next(r for r in golden["rmat"] if r["bench"] == bench_name
               and r["scale"] == scale and r["seed"] == seed)
    bench, wl = _rmat_workload(bench_name, scale, seed)
    configs = [dict(), dict(threshold=128, agg="block"),
               dict(threshold=128, cfactor=8, agg="multiblock", group_size=4),
               dict(threshold=64, cfactor=4, agg="grid", parent_block=256,
                    serial="warp")]
    for cfg in configs:
        rep, _ = run_config(bench, wl, BenchConfig(**cfg))
        assert rep.memory_digest == rec["digest"], cfg
        for row in rec.get("counters", []):
            if row["config"] == cfg and bench_name == "bfs":
                assert (rep.num_launches, rep.host_launches,
                        rep.blocks_scheduled) == (
                    row["num_launches"], row["host_launches"],
                    row["blocks_scheduled"]), cfg
    assert run_reference(bench, wl).memory_digest == rec["digest"]


# ---------------------------------------------------------------------------
# 3: oracle at full sizes + size-independent properties
# ---------------------------------------------------------------------------

def _bfs_properties(g, dist, counts):
    """dist is a BFS labelling from 0 and counts = in-edges from reached."""
    assert dist[0] == 0
    src = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    reached_u = dist[src] < UNREACHED
    du, dv = dist[src][reached_u], dist[g.col][reached_u]
    assert np.all(dv <= du + 1)
    # every reached vertex except the source has a parent one level up
    has_parent = np.zeros(g.n, bool)
    tight = dv == du + 1
    has_parent[g.col[reached_u][tight]] = True
    reached = dist < UNREACHED
    assert np.all(has_parent[reached] | (np.arange(g.n)[reached] == 0))
    np.testing.assert_array_equal(
        counts, np.bincount(g.col[reached_u], minlength=g.n))


@pytest.mark.parametrize("scale", [18, 22])
def test_bfs_rmat_full_size_vs_oracle(scale):
    bench, wl = _rmat_workload("bfs", scale, 1)
    g = wl.payload
    dist, counts, levels = oracle.bfs(g.rowptr, g.col, nthreads=0)
    for cfg in (BenchConfig(threshold=128, agg="block"),
                BenchConfig(threshold=512, cfactor=8, agg="multiblock",
                            group_size=4, parent_block=256, serial="warp"),
                BenchConfig(threshold=256, cfactor=4, agg="grid",
                            parent_block=256, child_block=128)):
        rep, _ = run_config(bench, wl, cfg)
        np.testing.assert_array_equal(rep.arrays["dist"], dist)
        np.testing.assert_array_equal(rep.arrays["counts"], counts)
        assert rep.host_launches >= levels  # + grid-glue launches
    _bfs_properties(g, dist, counts)


@pytest.mark.parametrize("scale", [16, 22])
def test_sssp_rmat_full_size_vs_oracle(scale):
    bench, wl = _rmat_workload("sssp", scale, 1)
    g, w = wl.payload
    dist, _ = oracle.sssp(g.rowptr, g.col, w, nthreads=0)
    for cfg in (BenchConfig(threshold=128, agg="block"),
                BenchConfig(threshold=512, cfactor=8, agg="multiblock",
                            group_size=4, parent_block=256, serial="warp")):
        rep, _ = run_config(bench, wl, cfg)
        np.testing.assert_array_equal(rep.arrays["dist"], dist)
    # optimality certificate: no edge can still be relaxed
    src = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    ok = dist[src] < UNREACHED
    assert np.all(dist[g.col[ok]] <= dist[src[ok]] + w[ok])


def test_naive_cdp_rmat16_matches():
    bench, wl = _rmat_workload("bfs", 16, 1)
    g = wl.payload
    dist, counts, _ = oracle.bfs(g.rowptr, g.col, nthreads=0)
    rep, _ = run_config(bench, wl, BenchConfig())
    np.testing.assert_array_equal(rep.arrays["dist"], dist)
    np.testing.assert_array_equal(rep.arrays["counts"], counts)
    # one launch per reached vertex with out-edges (reference: 33,957 at
    # RMAT-16 with its own generator)
    deg = np.diff(g.rowptr)
    assert rep.num_launches == int(((dist < UNREACHED) & (deg > 0)).sum())


@pytest.mark.parametrize("spec", ["rmat:12:seed1", "rmat:16:seed1",
                                  "rmat:18:seed2"])
def test_tc_vs_oracle(spec):
    bench, wl = load("tc", spec)
    gp = wl.payload[1]
    want = oracle.tc(gp.rowptr, gp.col, nthreads=0)
    for cfg in (BenchConfig(), BenchConfig(threshold=64, agg="block"),
                BenchConfig(threshold=256, cfactor=4, agg="grid",
                            parent_block=256, serial="warp")):
        rep, _ = run_config(bench, wl, cfg)
        assert int(rep.arrays["triangles"][0]) == want, cfg
    assert int(run_reference(bench, wl).arrays["triangles"][0]) == want
    # edge-range shards sum to the total (multi-GPU partition)
    m = gp.m
    cuts = np.linspace(0, m, 4).astype(int)
    tot = 0
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        out, _ = bench.run(wl, BenchConfig(threshold=64, agg="block").to_c(),
                           lo=int(lo), hi=int(hi))
        tot += int(out["triangles"][0])
    assert tot == want


@pytest.mark.parametrize("cfg", [
    BenchConfig(), BenchConfig(threshold=4096),
    BenchConfig(cfactor=4, agg="multiblock", group_size=4),
    BenchConfig(threshold=64, cfactor=2, agg="block", parent_block=128),
    BenchConfig(agg="grid", child_block=64)])
def test_bt_vs_oracle(cfg):
    bench, wl = load("bt", "curves:25000:seed1")
    ntess, verts = oracle.bt(wl.buffers["cp"], graphs.BT_MAX_TESS,
                             graphs.BT_CURV_SCALE)
    rep, _ = run_config(bench, wl, cfg)
    np.testing.assert_array_equal(rep.arrays["ntess"], ntess)
    got = rep.arrays["verts"].astype(np.float64)
    assert got.shape == verts.shape
    # tolerance from north_star: 1e-5 (coordinates are in [0, 1))
    assert np.max(np.abs(got - verts)) <= 1e-5


def test_run_benchmark_and_sweep_on_device():
    rep = run_benchmark("bfs", "hand", BenchConfig(agg="block"))
    assert rep.buffers["dist"] == list(graphs.HAND_BFS_DISTANCES)
    rows = sweep("bfs", "hand")
    assert len(rows) == 12 and all(r["error"] == "" for r in rows)
    assert rows[0]["num_launches"] > rows[-1]["num_launches"] == 0


def test_queue_overflow_fails_fast():
    bench, wl = load("manylaunch", "sizes:1024:seed1")
    with pytest.raises(_lib.DeviceTrap) as e:
        run_config(bench, wl, BenchConfig(pending_launch_limit=16))
    assert e.value.kind == "queue-overflow"
    # the same run with aggregation fits
    rep, _ = run_config(bench, wl, BenchConfig(agg="block",
                                               pending_launch_limit=2048))
    assert rep.num_launches > 0


def test_verify_outputs_detects_corruption():
    bench, wl = load("bfs", "powerlaw:150:seed2")
    ref = run_reference(bench, wl)
    got, _ = run_config(bench, wl, BenchConfig(threshold=8, agg="block"))
    verify_outputs(bench, wl, got, ref)
    got.arrays["counts"][5] += 1
    with pytest.raises(EquivalenceError, match=r"'counts'\[5\]"):
        verify_outputs(bench, wl, got, ref)


@pytest.mark.parametrize("spread", [False, True])
@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("policy", [
    dict(threshold=128, agg="block"),
    dict(threshold=1024, cfactor=16, agg="multiblock", group_size=1 << 20,
         parent_block=256, child_block=128, serial="warp"),
    dict()])
def test_bfs_1d_partition_on_device(P, policy, spread):
    """P parts of a cyclic 1D partition run their device steps on one GPU
    (LocalExchange); dist/counts must equal the single-GPU oracle."""
    import torch
    from paper_2201_02789_b200 import dist as pdist
    scale = 16
    g = graphs.rmat_graph(scale, 1)
    want_d, want_c, want_lv = oracle.bfs(g.rowptr, g.col, nthreads=0)
    parts = [pdist.BfsPart(*pdist.rmat_part(scale, 1, P, p), g.n, P, p, 0,
                           torch.device("cuda", 0), spread=spread)
             for p in range(P)]
    ops = pdist.DeviceBfsOps(BenchConfig(**policy).to_c())
    d, c, levels = pdist.bfs_1d(parts, ops, pdist.LocalExchange())
    np.testing.assert_array_equal(d.cpu().numpy(), want_d)
    np.testing.assert_array_equal(c.cpu().numpy(), want_c)
    assert levels == want_lv


@pytest.mark.parametrize("P", [1, 3])
def test_rmat_device_generator_matches_host(P):
    import torch
    from paper_2201_02789_b200 import dist as pdist
    for p in range(P):
        rp_h, col_h = pdist.rmat_part(14, 5, P, p)
        rp_d, col_d = pdist.rmat_part_device(14, 5, P, p,
                                             torch.device("cuda", 0))
        np.testing.assert_array_equal(rp_d.cpu().numpy(), rp_h)
        np.testing.assert_array_equal(col_d.cpu().numpy(), col_h)


# ---------------------------------------------------------------------------
# edge cases
# ---------------------------------------------------------------------------

EDGE_POLICIES = [dict(), dict(threshold=INF_THRESHOLD), dict(agg="warp"),
                 dict(agg="block", agg_threshold=1000),
                 dict(threshold=1, cfactor=1000, agg="multiblock",
                      group_size=1), dict(agg="multiblock", group_size=10**6),
                 dict(threshold=2, cfactor=3, agg="grid", parent_block=256,
                      child_block=64, serial="warp"),
                 dict(threshold=2, agg="multiblock", group_size=1 << 20,
                      persistent=1, serial="warp"),
                 dict(threshold=3, agg="grid", persistent=3),
                 dict(threshold=2, agg="block", device_loop=True),
                 dict(agg="multiblock", group_size=1 << 20, device_loop=True)]


def _graph_workload(bench_name, rowptr, col, weight=None):
    rowptr = np.asarray(rowptr, np.int32)
    col = np.asarray(col, np.int32)
    n = rowptr.shape[0] - 1
    g = graphs.Graph(rowptr, col)
    spec = DatasetSpec("hand", n, 0, f"custom:{n}")
    dist = np.full(n, UNREACHED, np.int32)
    dist[0] = 0
    bufs = {"rowptr": rowptr, "col": col, "dist": dist,
            "counts": np.zeros(n, np.int32)}
    payload = g
    if bench_name == "sssp":
        bufs["weight"] = np.asarray(weight if weight is not None
                                    else np.ones(col.shape[0]), np.int32)
        payload = (g, bufs["weight"])
    return BENCHMARKS[bench_name], Workload(spec, bufs, n, payload)


@pytest.mark.parametrize("policy", EDGE_POLICIES)
@pytest.mark.parametrize("rowptr,col", [
    ([0, 0], []),                      # single vertex, no edges
    ([0, 0, 1], [0]),                  # source without out-edges
    ([0, 3, 3, 3], [0, 0, 0]),         # self-loop multi-edge only
    ([0, 2, 4, 4, 4], [1, 1, 3, 3]),   # duplicates, unreachable vertex 2
])
def test_bfs_sssp_degenerate_graphs(rowptr, col, policy):
    for bench_name in ("bfs", "sssp"):
        bench, wl = _graph_workload(bench_name, rowptr, col)
        g = wl.payload if bench_name == "bfs" else wl.payload[0]
        want = oracle.bfs(g.rowptr, g.col)
        rep, _ = run_config(bench, wl, BenchConfig(**policy))
        np.testing.assert_array_equal(rep.arrays["dist"], want[0])
        if bench_name == "bfs":
            np.testing.assert_array_equal(rep.arrays["counts"], want[1])
            assert rep.iterations == want[2]
            if not policy.get("device_loop"):
                assert rep.host_launches >= want[2]


def test_sssp_negative_cycle_hits_iteration_limit():
    bench, wl = _graph_workload("sssp", [0, 1, 2], [1, 0], weight=[-1, -1])
    with pytest.raises(RuntimeError) as e:
        run_config(bench, wl, BenchConfig(threshold=4, agg="block"))
    assert getattr(e.value, "kind", "") == "iteration-limit"


@pytest.mark.parametrize("policy", EDGE_POLICIES)
def test_manylaunch_zero_negative_and_large_sizes(policy):
    sizes = np.array([0, -5, 1, 31, 32, 33, 1024, 0, 5000, -1] * 7, np.int32)
    spec = DatasetSpec("sizes", sizes.shape[0], 0, "custom")
    wl = Workload(spec, {"sizes": sizes, "out": np.zeros_like(sizes),
                         "total": np.zeros(1, np.int32)}, sizes.shape[0],
                  sizes)
    bench = BENCHMARKS["manylaunch"]
    want_out, want_total = oracle.manylaunch(sizes)
    rep, _ = run_config(bench, wl, BenchConfig(**policy))
    np.testing.assert_array_equal(rep.arrays["out"], want_out)
    np.testing.assert_array_equal(rep.arrays["total"], want_total)
    ref = run_reference(bench, wl)
    np.testing.assert_array_equal(ref.arrays["out"], want_out)


def test_tc_empty_and_tiny():
    bench = BENCHMARKS["tc"]
    for rowptr, col, want in (([0] * 11, [], 0),
                              ([0, 2, 3, 3], [1, 2, 2], 1)):
        rowptr = np.asarray(rowptr, np.int32)
        col = np.asarray(col, np.int32)
        spec = DatasetSpec("rmat", 1, 0, "custom")
        wl = Workload(spec, {"rowptr": rowptr, "col": col}, rowptr.shape[0] - 1,
                      None)
        for policy in EDGE_POLICIES:
            rep, _ = run_config(bench, wl, BenchConfig(**policy))
            assert int(rep.arrays["triangles"][0]) == want, policy


@pytest.mark.parametrize("policy", EDGE_POLICIES)
def test_bt_degenerate_curves(policy):
    cp = np.zeros((5, 3, 2), np.float32)
    cp[1] = [[0.5, 0.5], [0.9, 0.1], [0.5, 0.5]]   # P0 == P2: curvature inf
    cp[2] = [[0.1, 0.1], [0.2, 0.2], [0.3, 0.3]]   # straight: 4 vertices
    cp[3] = [[0.0, 0.0], [0.0, 0.0], [0.0, 0.0]]   # 0/0: NaN -> max
    cp[4] = [[0.0, 0.0], [1.0, 1.0], [1.0, 0.0]]
    spec = DatasetSpec("curves", 5, 0, "custom")
    wl = Workload(spec, {"cp": cp, "max_tess": graphs.BT_MAX_TESS,
                         "scale": graphs.BT_CURV_SCALE}, 5, cp)
    bench = BENCHMARKS["bt"]
    ntess, verts = oracle.bt(cp, graphs.BT_MAX_TESS, graphs.BT_CURV_SCALE)
    rep, _ = run_config(bench, wl, BenchConfig(**policy))
    np.testing.assert_array_equal(rep.arrays["ntess"], ntess)
    assert ntess[1] == ntess[3] == graphs.BT_MAX_TESS and ntess[2] == 4
    assert np.max(np.abs(rep.arrays["verts"] - verts)) <= 1e-5


def test_bt_zero_curves():
    cp = np.zeros((0, 3, 2), np.float32)
    wl = Workload(DatasetSpec("curves", 1, 0, "custom"),
                  {"cp": cp, "max_tess": graphs.BT_MAX_TESS,
                   "scale": graphs.BT_CURV_SCALE}, 0, cp)
    rep, _ = run_config(BENCHMARKS["bt"], wl, BenchConfig(agg="block"))
    assert rep.arrays["ntess"].shape == (0,)


def test_naive_cdp_waves_rmat21():
    """~1.1 M launching parents exceed the 2^19 pending-launch cap: the
    parent grid runs in waves (dynpar.cu wave_parents) and stays exact."""
    bench, wl = _rmat_workload("bfs", 21, 3)
    g = wl.payload
    dist, counts, _ = oracle.bfs(g.rowptr, g.col, nthreads=0)
    rep, _ = run_config(bench, wl, BenchConfig(parent_block=256))
    np.testing.assert_array_equal(rep.arrays["dist"], dist)
    np.testing.assert_array_equal(rep.arrays["counts"], counts)
    deg = np.diff(g.rowptr)
    launchers = int(((dist < UNREACHED) & (deg > 0)).sum())
    assert rep.num_launches == launchers
    assert launchers > (1 << 19)


@pytest.mark.parametrize("policy", [
    dict(device_loop=True), dict(threshold=4, agg="block", device_loop=True),
    dict(threshold=4, cfactor=2, agg="multiblock", group_size=1 << 20,
         serial="warp", parent_block=128, device_loop=True)])
def test_device_loop_many_levels(policy, golden):
    """road graphs have long BFS chains: several 16-round device chains."""
    for bench_name in ("bfs", "sssp"):
        bench, wl = load(bench_name, "road:1000:seed7")
        ref = _golden_ref(golden, bench_name, "road:1000:seed7")
        rep, _ = run_config(bench, wl, BenchConfig(**policy))
        assert rep.memory_digest == ref["digest"]
        if bench_name == "bfs":
            assert rep.iterations == ref["host_launches"] > 16
            assert rep.host_launches == -(-rep.iterations // 16) or \
                rep.host_launches == -(-(rep.iterations + 1) // 16)


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("policy", [
    dict(threshold=128, agg="block"),
    dict(threshold=1024, cfactor=32, agg="multiblock", group_size=2048,
         parent_block=128, child_block=64, serial="warp"),
    dict()])
def test_sssp_1d_partition_on_device(P, policy):
    import torch
    from paper_2201_02789_b200 import dist as pdist
    g = graphs.rmat_graph(16, 2)
    w = graphs.edge_weights(g, 2)
    want, _ = oracle.sssp(g.rowptr, g.col, w, nthreads=0)
    parts = [pdist.SsspPart(*pdist.partition_csr(g.rowptr, g.col, P, p, w),
                            g.n, P, p, 0, torch.device("cuda", 0))
             for p in range(P)]
    ops = pdist.DeviceSsspOps(BenchConfig(**policy).to_c())
    d, rounds = pdist.sssp_1d(parts, ops, pdist.LocalExchange())
    np.testing.assert_array_equal(d.cpu().numpy(), want)
    # a second run on the same parts after reset gives the same answer
    for p in parts:
        p.reset(0)
    d2, _ = pdist.sssp_1d(parts, ops, pdist.LocalExchange())
    np.testing.assert_array_equal(d2.cpu().numpy(), want)


GC_FAST = (dict(threshold=64, agg="block"),
           dict(threshold=256, cfactor=8, agg="multiblock", group_size=1 << 20,
                parent_block=256, child_block=128, serial="warp"),
           dict(threshold=32, agg="grid", serial="warp"))


@pytest.mark.parametrize("spec", ["hand", "powerlaw:2000:seed1",
                                  "road:1000:seed7", "rmat:12:seed1"])
def test_gc_vs_oracle(spec):
    bench, wl = load("gc", spec)
    want, k = oracle.gc(wl.buffers["rowptr"], wl.buffers["col"])
    for policy in (dict(), dict(threshold=INF_THRESHOLD)) + GC_FAST:
        rep, _ = run_config(bench, wl, BenchConfig(**policy))
        np.testing.assert_array_equal(rep.arrays["color"], want)
    np.testing.assert_array_equal(run_reference(bench, wl).arrays["color"],
                                  want)


def test_gc_rmat18_vs_oracle():
    bench, wl = load("gc", "rmat:18:seed2")
    want, k = oracle.gc(wl.buffers["rowptr"], wl.buffers["col"])
    for policy in GC_FAST:
        rep, _ = run_config(bench, wl, BenchConfig(**policy))
        np.testing.assert_array_equal(rep.arrays["color"], want)
        assert int(rep.arrays["color"].max()) + 1 == k


MST_POLICIES = (dict(), dict(threshold=INF_THRESHOLD), dict(agg="warp"),
                dict(threshold=32, agg="block"),
                dict(threshold=64, cfactor=4, agg="multiblock", group_size=4,
                     serial="warp"),
                dict(threshold=256, cfactor=8, agg="multiblock",
                     group_size=1 << 20, parent_block=256, child_block=128,
                     serial="warp"),
                dict(threshold=32, agg="grid", serial="warp"))


def _mst_want(wl):
    b = wl.buffers
    return oracle.mst(b["rowptr"], b["col"], b["weight"], b["eid"])


@pytest.mark.parametrize("bench_name", ["mstf", "mstv"])
@pytest.mark.parametrize("spec", ["hand", "powerlaw:2000:seed1",
                                  "road:1000:seed7", "rmat:12:seed1"])
def test_mst_vs_oracle(bench_name, spec):
    bench, wl = load(bench_name, spec)
    in_mst, total, k = _mst_want(wl)
    for policy in MST_POLICIES:
        rep, _ = run_config(bench, wl, BenchConfig(**policy))
        np.testing.assert_array_equal(rep.arrays["in_mst"], in_mst)
        assert rep.arrays["weight"].tolist() == [total, k]
    ref = run_reference(bench, wl)
    np.testing.assert_array_equal(ref.arrays["in_mst"], in_mst)
    assert ref.arrays["weight"].tolist() == [total, k]


def test_mst_rmat18_and_long_chains_vs_oracle():
    # rmat: one giant component + isolated vertices; road:20000: long hook
    # chains (pointer jumping depth)
    for spec in ("rmat:18:seed2", "road:20000:seed1"):
        for name in ("mstf", "mstv"):
            bench, wl = load(name, spec)
            in_mst, total, k = _mst_want(wl)
            for policy in MST_POLICIES[3:]:
                rep, _ = run_config(bench, wl, BenchConfig(**policy))
                np.testing.assert_array_equal(rep.arrays["in_mst"], in_mst)
                assert rep.arrays["weight"].tolist() == [total, k]
                assert rep.iterations <= 64


SP_POLICIES = (dict(), dict(threshold=INF_THRESHOLD), dict(agg="warp"),
               dict(threshold=16, agg="block"),
               dict(threshold=32, cfactor=4, agg="multiblock", group_size=8,
                    serial="warp"),
               dict(threshold=8, agg="grid", serial="warp",
                    parent_block=128, child_block=64))


def _sp_close(got, want):
    # surveys: 1e-5 relative (north star), 1e-7 absolute for tiny surveys;
    # biases are fp32
    np.testing.assert_allclose(got["eta"], want[0], rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(got["wpos"], want[1], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(got["wneg"], want[2], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("spec", ["ksat3:2000:seed1", "ksat5:1000:seed2",
                                  "ksat3:30000:seed3"])
def test_sp_vs_oracle_fixed_sweeps(spec):
    bench, wl = load("sp", spec)
    b = dict(wl.buffers, max_sweeps=25, eps=0.0)
    wl = Workload(wl.spec, b, wl.n, wl.payload)
    want = oracle.sp(wl.payload, b["eta0"], 25, 0.0)
    for policy in SP_POLICIES:
        rep, _ = run_config(bench, wl, BenchConfig(**policy))
        assert rep.iterations == 25
        _sp_close(rep.arrays, want)
    _sp_close(run_reference(bench, wl).arrays, want)


@pytest.mark.parametrize("shuffle", [False, True])
def test_sp_windowed_variable_pass(shuffle, monkeypatch):
    """The variable pass runs once per L2 window of eta (1 MB windows: three
    passes here); occurrence lists that are not sorted by edge fall back to
    one window.  Surveys and biases stay within tolerance either way."""
    monkeypatch.setenv("DYNPAR_SP_WINDOW_MB", "1")
    bench, wl = load("sp", "ksat3:30000:seed3")
    b = dict(wl.buffers, max_sweeps=12, eps=0.0)
    if shuffle:
        occ, row = b["occ"].copy(), b["occ_row"]
        rng = np.random.default_rng(5)
        for i in range(0, len(row) - 1, 7):
            rng.shuffle(occ[row[i]:row[i + 1]])
        b["occ"] = occ
    wl = Workload(wl.spec, b, wl.n, wl.payload)
    want = oracle.sp(wl.payload, b["eta0"], 12, 0.0)
    for policy in SP_POLICIES:
        rep, _ = run_config(bench, wl, BenchConfig(**policy))
        assert rep.iterations == 12
        _sp_close(rep.arrays, want)


def test_sp_converges_like_oracle():
    bench, wl = load("sp", "ksat3:20000:seed1")
    want = oracle.sp(wl.payload, wl.buffers["eta0"],
                     wl.buffers["max_sweeps"], wl.buffers["eps"])
    rep, _ = run_config(bench, wl, BenchConfig(threshold=32, agg="grid",
                                               serial="warp"))
    assert rep.iterations == want[3]
    _sp_close(rep.arrays, want)
    run_benchmark("sp", "ksat5:800:seed1", BenchConfig(threshold=64,
                                                       agg="block"))


@pytest.mark.parametrize("spec", GRAPH_SPECS + ["rmat:14:seed1"])
def test_sssp_frontier_mode_same_distances(spec):
    """B200 work-efficient rounds (frontier=True): identical distances."""
    bench, wl = load("sssp", spec)
    b = wl.buffers
    want, _ = oracle.sssp(b["rowptr"], b["col"], b["weight"], nthreads=0)
    for policy in (dict(), dict(threshold=INF_THRESHOLD, serial="warp"),
                   dict(threshold=64, cfactor=4, agg="multiblock",
                        group_size=1 << 20, serial="warp"),
                   dict(threshold=32, agg="grid"),
                   dict(device_loop=True, parent_block=64),
                   dict(persistent=2, agg="grid", parent_block=128)):
        rep, _ = run_config(bench, wl, BenchConfig(frontier=True, **policy))
        np.testing.assert_array_equal(rep.arrays["dist"], want)


def test_sssp_frontier_rmat22_fewer_relaxations():
    bench, wl = load("sssp", "rmat:20:seed1")
    b = wl.buffers
    want, _ = oracle.sssp(b["rowptr"], b["col"], b["weight"], nthreads=0)
    pol = dict(threshold=1024, cfactor=32, agg="multiblock", group_size=2048,
               parent_block=128, child_block=64, serial="warp")
    full, _ = run_config(bench, wl, BenchConfig(**pol))
    fr, _ = run_config(bench, wl, BenchConfig(frontier=True, **pol))
    np.testing.assert_array_equal(fr.arrays["dist"], want)
    np.testing.assert_array_equal(full.arrays["dist"], want)
    assert fr.ns_device < full.ns_device


def _mst_workload(name, rowptr, col, weight):
    """A custom symmetric simple graph as an mstf / mstv workload."""
    g = graphs.Graph(np.asarray(rowptr, np.int32), np.asarray(col, np.int32))
    eid = np.minimum(np.arange(g.m, dtype=np.int32), graphs.edge_mirror(g))
    w = np.asarray(weight, np.int32)[eid] if g.m else np.zeros(0, np.int32)
    spec = DatasetSpec("hand", g.n, 0, f"custom:{g.n}")
    return BENCHMARKS[name], Workload(spec, {
        "rowptr": g.rowptr, "col": g.col, "weight": np.ascontiguousarray(w),
        "eid": np.ascontiguousarray(eid)}, g.n, g)


@pytest.mark.parametrize("policy", EDGE_POLICIES)
@pytest.mark.parametrize("rowptr,col,weight", [
    ([0, 0], [], []),                                  # one vertex
    ([0, 0, 0, 0], [], []),                            # no edges at all
    ([0, 1, 2], [1, 0], [5, 5]),                       # one edge
    ([0, 2, 4, 6], [1, 2, 0, 2, 0, 1], [3] * 6),       # triangle, all ties
    ([0, 1, 2, 3, 4], [1, 0, 3, 2], [-7, -7, 2**31 - 1, 2**31 - 1]),
    # two components, extreme signed weights
])
def test_mst_degenerate_graphs(rowptr, col, weight, policy):
    for name in ("mstf", "mstv"):
        bench, wl = _mst_workload(name, rowptr, col, weight)
        b = wl.buffers
        want = oracle.mst(b["rowptr"], b["col"], b["weight"], b["eid"])
        rep, _ = run_config(bench, wl, BenchConfig(**policy))
        np.testing.assert_array_equal(rep.arrays["in_mst"], want[0])
        assert rep.arrays["weight"].tolist() == [want[1], want[2]]


def test_sp_edge_cases():
    """One clause; zero and one surveys (the zero-factor bookkeeping);
    max_sweeps = 0 leaves eta0 and only computes biases."""
    bench = BENCHMARKS["sp"]
    for spec_text, eta_fill in (("ksat3:3:seed1", None),
                                ("ksat3:50:seed2", 1.0),
                                ("ksat5:60:seed3", 0.0),
                                ("ksat3:40:seed4", "mixed")):
        _, wl = load("sp", spec_text)
        eta0 = wl.buffers["eta0"].copy()
        if eta_fill == "mixed":
            eta0[::3] = 1.0
            eta0[1::5] = 0.0
        elif eta_fill is not None:
            eta0[:] = eta_fill
        for sweeps in (0, 1, 7):
            b = dict(wl.buffers, eta0=eta0, max_sweeps=sweeps, eps=0.0)
            w2 = Workload(wl.spec, b, wl.n, wl.payload)
            want = oracle.sp(wl.payload, eta0, sweeps, 0.0)
            for policy in EDGE_POLICIES[:4]:
                rep, _ = run_config(bench, w2, BenchConfig(**policy))
                # eps = 0 still stops at an exact fixed point (delta == 0)
                assert rep.iterations == want[3] <= sweeps
                _sp_close(rep.arrays, want)


@pytest.mark.parametrize("spec", ["powerlaw:2000:seed1", "road:1000:seed7",
                                  "rmat:14:seed1"])
def test_sssp_host_call_overlaps_copy_in_chunks(spec, monkeypatch):
    """dp_sssp streams col / weight in chunks while the rounds run (parents
    whose edges are in flight are deferred): tiny chunks force many
    deferrals; distances stay exact in both round modes."""
    bench, wl = load("sssp", spec)
    b = wl.buffers
    want, _ = oracle.sssp(b["rowptr"], b["col"], b["weight"], nthreads=0)
    for shift in ("4", "8", "30"):
        monkeypatch.setenv("DP_COPY_CHUNK_SHIFT", shift)
        for policy in (dict(), dict(threshold=64, cfactor=4, agg="multiblock",
                                    group_size=1 << 20, serial="warp"),
                       dict(threshold=32, agg="grid", frontier=True)):
            rep, _ = run_config(bench, wl, BenchConfig(**policy))
            np.testing.assert_array_equal(rep.arrays["dist"], want)
        ref = run_reference(bench, wl)
        np.testing.assert_array_equal(ref.arrays["dist"], want)


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("policy", [
    dict(threshold=128, agg="block"),
    dict(threshold=1024, cfactor=16, agg="multiblock", group_size=1 << 20,
         parent_block=128, child_block=128, serial="warp"),
    dict()])
def test_sssp_fused_peer_exchange_on_device(P, policy):
    """The fused-exchange partitioned SSSP (remote atomicMin into the
    owner's dist through the pointer table), P parts on one GPU."""
    import torch
    from paper_2201_02789_b200 import dist as pdist
    g = graphs.rmat_graph(16, 1)
    w = graphs.edge_weights(g, 1)
    want, _ = oracle.sssp(g.rowptr, g.col, w, nthreads=0)
    dev = torch.device("cuda", 0)
    ex = pdist.PeerLocal()
    parts = [pdist.SsspPeerPart(*pdist.partition_csr(g.rowptr, g.col, P, p, w),
                                g.n, P, p, 0, ex.alloc(g.n, P, dev), dev)
             for p in range(P)]
    ex.bind(parts)
    ops = pdist.DeviceSsspPeerOps(BenchConfig(**policy).to_c())
    d, rounds = pdist.sssp_1d_peer(parts, ops, ex)
    np.testing.assert_array_equal(d.cpu().numpy(), want)
    for p in parts:
        p.reset(0)
    d2, _ = pdist.sssp_1d_peer(parts, ops, ex)
    np.testing.assert_array_equal(d2.cpu().numpy(), want)


@pytest.mark.parametrize("spread", [False, True])
@pytest.mark.parametrize("P", [1, 2, 3])
def test_bfs_fused_peer_exchange_on_device(P, spread):
    """BFS over the 1D partition with remote discoveries CAS'd straight into
    the owner's dist (pointer table), P parts on one GPU."""
    import torch
    from paper_2201_02789_b200 import dist as pdist
    g = graphs.rmat_graph(16, 1)
    want_d, want_c, want_lv = oracle.bfs(g.rowptr, g.col, nthreads=0)
    dev = torch.device("cuda", 0)
    ex = pdist.PeerLocal()
    parts = [pdist.BfsPart(*pdist.rmat_part(16, 1, P, p), g.n, P, p, 0, dev,
                           dist=ex.alloc(g.n, P, dev), spread=spread)
             for p in range(P)]
    ex.bind(parts)
    for policy in (dict(threshold=128, agg="block"),
                   dict(threshold=1024, cfactor=16, agg="multiblock",
                        group_size=1 << 20, parent_block=256,
                        child_block=128, serial="warp")):
        for p in parts:
            p.reset(0)
        ops = pdist.DeviceBfsOps(BenchConfig(**policy).to_c())
        d, c, levels = pdist.bfs_1d_peer(parts, ops, ex)
        np.testing.assert_array_equal(d.cpu().numpy(), want_d)
        np.testing.assert_array_equal(c.cpu().numpy(), want_c)
        assert levels == want_lv


# ---------------------------------------------------------------------------
# pass order (pipeline.py:45-81): every permutation / subset of "TCA" on the
# golden configurations reproduces the reference's digest and counters,
# including "A before C" (coarsening of the aggregated grid, logical blocks
# spanning parents) and a threshold pass skipped after C or A
# ---------------------------------------------------------------------------

def _order_rows():
    import json
    from conftest import GOLDEN
    return json.loads((GOLDEN / "order_counters.json").read_text())


@pytest.mark.parametrize("bench_name,spec", [
    ("bfs", "powerlaw:2000:seed1"), ("bfs", "road:1000:seed7"),
    ("manylaunch", "sizes:1024:seed1"), ("sssp", "powerlaw:150:seed3")])
def test_order_permutations_match_reference(bench_name, spec):
    rows = [r for r in _order_rows()
            if r["bench"] == bench_name and r["dataset"] == spec]
    assert len(rows) == 80
    bench, wl = load(bench_name, spec)
    for row in rows:
        rep, _ = run_config(bench, wl,
                            BenchConfig(order=row["order"], **row["config"]))
        key = (row["order"], row["config"])
        assert rep.memory_digest == row["digest"], key
        if bench_name == "sssp":
            continue  # rounds depend on the real schedule
        assert (rep.num_launches, rep.host_launches, rep.blocks_scheduled) \
            == (row["num_launches"], row["host_launches"],
                row["blocks_scheduled"]), key


@pytest.mark.parametrize("serial", ["thread", "warp"])
def test_aggregated_grid_coarsening_rmat(serial):
    """A-before-C at scale: RMAT-16 BFS / SSSP under block and multiblock
    aggregation with the aggregated grid coarsened, bit-exact vs oracle."""
    bfs_b, bfs_wl = _rmat_workload("bfs", 16, 1)
    sssp_b, sssp_wl = _rmat_workload("sssp", 16, 1)
    g, w = sssp_wl.payload
    wd, wc, _ = oracle.bfs(g.rowptr, g.col, nthreads=0)
    sd, _ = oracle.sssp(g.rowptr, g.col, w, nthreads=0)
    for agg, gs in (("block", 4), ("multiblock", 4), ("multiblock", 1 << 20),
                    ("warp", 4)):
        cfg = BenchConfig(threshold=64, cfactor=4, agg=agg, group_size=gs,
                          order="TAC", parent_block=128, child_block=128,
                          serial=serial)
        assert cfg.to_c().agg_coarsen == 1
        rep, _ = run_config(bfs_b, bfs_wl, cfg)
        assert np.array_equal(rep.arrays["dist"], wd), agg
        assert np.array_equal(rep.arrays["counts"], wc), agg
        rep, _ = run_config(sssp_b, sssp_wl, cfg)
        assert np.array_equal(rep.arrays["dist"], sd), agg


def test_registered_benchmark_runs_everywhere():
    """A benchmark registered from Python (register_benchmark, the
    reference's plug-in point) -- here BFS from source 7 with its own
    prepare / drive over the existing device App -- runs through
    run_config, run_reference, verify_outputs and sweep, bit-exact vs the
    oracle."""
    import ctypes
    from paper_2201_02789_b200 import _lib
    from paper_2201_02789_b200.bench import (Benchmark, register_benchmark,
                                             sweep, verify_outputs)
    base = BENCHMARKS["bfs"]

    def prepare(spec):
        wl = base.prepare(spec)
        wl.buffers["dist"][:] = UNREACHED
        wl.buffers["dist"][7] = 0
        return wl

    def run(wl, cfg):
        b = wl.buffers
        dist = np.empty(wl.n, np.int32)
        counts = np.empty(wl.n, np.int32)
        st = _lib.DpStats()
        _lib.check(_lib.device().dp_bfs(
            _lib.ptr(b["rowptr"]), _lib.ptr(b["col"]), wl.n,
            b["col"].shape[0], 7, ctypes.byref(cfg), _lib.ptr(dist),
            _lib.ptr(counts), ctypes.byref(st)))
        return {"dist": dist, "counts": counts}, _lib.stats_dict(st)

    register_benchmark(Benchmark("bfs_src7", base.outputs, base.kinds,
                                 prepare, run, base.traffic, "BFS from 7"))
    try:
        bench, wl = load("bfs_src7", "powerlaw:2000:seed1")
        b = wl.buffers
        want_d, want_c, _ = oracle.bfs(b["rowptr"], b["col"], src=7)
        for pol in (dict(), dict(threshold=8, cfactor=2, agg="multiblock",
                                 group_size=3)):
            rep, _ = run_config(bench, wl, BenchConfig(**pol))
            np.testing.assert_array_equal(rep.arrays["dist"], want_d)
            np.testing.assert_array_equal(rep.arrays["counts"], want_c)
            verify_outputs(bench, wl, rep, run_reference(bench, wl))
        rows = sweep("bfs_src7", "powerlaw:2000:seed1")
        assert rows and all(r["error"] == "" for r in rows)
    finally:
        BENCHMARKS.pop("bfs_src7", None)
