"""Property tests on the device: random inputs x random T/C/A policies,
checked against the CPU oracle (bit-exact) and against the counter
invariants of the reference's passes.

The reference pins its disaggregation search with a hypothesis test over
random child-grid lists (tests/test_passes.py:514-538); here the same idea
runs end to end through libdynpar: random child sizes (manylaunch) and random
skewed graphs (BFS, SSSP, TC, GC, MSTF, MSTV) under random policies, with
derandomised examples so a failure reproduces."""
from __future__ import annotations

import math

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import oracle
from paper_2201_02789_b200.bench import BenchConfig, graphs, run_config
from paper_2201_02789_b200.bench.benchmarks import BENCHMARKS, Workload
from paper_2201_02789_b200.bench.graphs import DatasetSpec, UNREACHED

pytestmark = pytest.mark.gpu

SETTINGS = settings(max_examples=250, deadline=None, derandomize=True,
                    suppress_health_check=list(HealthCheck))

INF = (1 << 31) - 1


@st.composite
def policies(draw):
    agg = draw(st.sampled_from([None, "warp", "block", "multiblock", "grid"]))
    p = dict(threshold=draw(st.sampled_from([0, 1, 2, 7, 32, 33, 100, INF])),
             cfactor=draw(st.sampled_from([1, 2, 3, 8, 64])),
             agg=agg,
             parent_block=draw(st.sampled_from([32, 64, 128, 256])),
             child_block=draw(st.sampled_from([32, 64, 256])),
             serial=draw(st.sampled_from(["thread", "warp"])))
    if agg == "multiblock":
        p["group_size"] = draw(st.sampled_from([1, 2, 3, 5, 1 << 20]))
    if agg == "block":
        p["agg_threshold"] = draw(st.sampled_from([0, 0, 3, 40]))
    if agg == "grid" or (agg == "multiblock" and p["group_size"] == 1 << 20):
        p["persistent"] = draw(st.sampled_from([0, 0, 1, 4]))
    return p


sizes_st = st.lists(
    st.one_of(st.just(0), st.integers(-3, 40), st.integers(31, 300),
              st.integers(1000, 9000)),
    min_size=1, max_size=1500)


def _ml_workload(sizes):
    sizes = np.asarray(sizes, np.int32)
    spec = DatasetSpec("sizes", sizes.shape[0], 0, "custom")
    return BENCHMARKS["manylaunch"], Workload(
        spec, {"sizes": sizes, "out": np.zeros_like(sizes),
               "total": np.zeros(1, np.int32)}, sizes.shape[0], sizes)


def _launched(sizes, policy):
    t = policy["threshold"]
    s = np.asarray(sizes, np.int64)
    return (s > 0) & ((s >= t) if t > 0 else True)


@SETTINGS
@given(sizes=sizes_st, policy=policies())
def test_manylaunch_random_sizes_and_policies(sizes, policy):
    bench, wl = _ml_workload(sizes)
    want_out, want_total = oracle.manylaunch(wl.payload)
    rep, _ = run_config(bench, wl, BenchConfig(**policy))
    np.testing.assert_array_equal(rep.arrays["out"], want_out)
    np.testing.assert_array_equal(rep.arrays["total"], want_total)
    # coarsening sets the blocks (coarsen.py:65-144): each launched parent
    # contributes ceil(ceil(size / child_block) / C) whatever aggregates,
    # plus the one host-launched parent grid (every grid counts,
    # sim/machine.py:165-247)
    go = _launched(sizes, policy)
    cb, cf = policy["child_block"], policy["cfactor"]
    blocks = sum(math.ceil(math.ceil(s / cb) / cf)
                 for s, g in zip(sizes, go) if g)
    parent_grid = math.ceil(len(sizes) / policy["parent_block"])
    assert rep.blocks_scheduled == blocks + parent_grid
    if not go.any():
        assert rep.num_launches == 0 and rep.host_launches == 1
    elif policy["agg"] is None:
        assert rep.num_launches == int(go.sum())
    elif policy["agg"] == "warp":
        assert rep.num_launches == len({i // 32 for i in np.flatnonzero(go)})
    elif policy["agg"] == "grid":
        assert rep.num_launches == 0 and rep.host_launches == 2
    else:
        assert 1 <= rep.num_launches <= int(go.sum())


@st.composite
def graphs_st(draw):
    n = draw(st.integers(1, 400))
    m = draw(st.integers(0, 6 * n))
    rng = np.random.default_rng(draw(st.integers(0, 2**32 - 1)))
    # skewed destinations (hubs) plus a few long chains for depth
    src = rng.integers(0, n, m)
    dst = np.minimum((rng.pareto(1.2, m) * 3).astype(np.int64), n - 1)
    dst = np.where(rng.random(m) < 0.5, dst, rng.integers(0, n, m))
    if n > 1 and draw(st.booleans()):
        chain = np.arange(n - 1)
        src = np.concatenate([src, chain])
        dst = np.concatenate([dst, chain + 1])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    rowptr = np.zeros(n + 1, np.int64)
    np.add.at(rowptr, src + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.int32)
    weight = rng.integers(1, 10, src.shape[0]).astype(np.int32)
    return rowptr, dst.astype(np.int32), weight


def _graph_workload(bench_name, rowptr, col, weight):
    n = rowptr.shape[0] - 1
    g = graphs.Graph(rowptr, col)
    spec = DatasetSpec("hand", n, 0, f"custom:{n}")
    dist = np.full(n, UNREACHED, np.int32)
    dist[0] = 0
    bufs = {"rowptr": rowptr, "col": col, "dist": dist,
            "counts": np.zeros(n, np.int32)}
    payload = g
    if bench_name == "sssp":
        bufs["weight"] = weight
        payload = (g, weight)
    return BENCHMARKS[bench_name], Workload(spec, bufs, n, payload)


@SETTINGS
@given(graph=graphs_st(), policy=policies(),
       device_loop=st.booleans(), frontier=st.booleans(),
       codec=st.sampled_from([{}, dict(weight_bits=4), dict(col_bits=24),
                              dict(weight_bits=4, col_bits=24)]))
def test_bfs_sssp_random_graphs_and_policies(graph, policy, device_loop,
                                             frontier, codec):
    rowptr, col, weight = graph
    dist, counts, levels = oracle.bfs(rowptr, col)
    bench, wl = _graph_workload("bfs", rowptr, col, weight)
    rep, _ = run_config(bench, wl,
                        BenchConfig(**policy, device_loop=device_loop))
    np.testing.assert_array_equal(rep.arrays["dist"], dist)
    np.testing.assert_array_equal(rep.arrays["counts"], counts)
    assert rep.iterations == levels
    sdist, _ = oracle.sssp(rowptr, col, weight)
    bench, wl = _graph_workload("sssp", rowptr, col, weight)
    rep, _ = run_config(bench, wl, BenchConfig(
        **policy, device_loop=device_loop, frontier=frontier, **codec))
    np.testing.assert_array_equal(rep.arrays["dist"], sdist)


def _raw_graph(rowptr, col):
    return graphs.Graph(np.asarray(rowptr, np.int32), np.asarray(col, np.int32))


@SETTINGS
@given(graph=graphs_st(), policy=policies(), seed=st.integers(0, 1000))
def test_tc_gc_mst_random_graphs_and_policies(graph, policy, seed):
    rowptr, col, _ = graph
    g = _raw_graph(rowptr, col)
    spec = DatasetSpec("hand", g.n, seed, f"custom:{g.n}")
    # TC over the degree-oriented CSR+ 
    gp = graphs.tc_orient(g)
    wl = Workload(spec, {"rowptr": gp.rowptr, "col": gp.col,
                         "triangles": np.zeros(1, np.uint64)}, gp.n, (g, gp))
    rep, _ = run_config(BENCHMARKS["tc"], wl, BenchConfig(**policy))
    assert int(rep.arrays["triangles"][0]) == oracle.tc(gp.rowptr, gp.col)
    # GC over the symmetrised graph (LLF Jones-Plassmann == greedy order)
    gs = graphs.symmetrize(g)
    wl = Workload(spec, {"rowptr": gs.rowptr, "col": gs.col,
                         "color": np.full(gs.n, -1, np.int32)}, gs.n, gs)
    rep, _ = run_config(BENCHMARKS["gc"], wl, BenchConfig(**policy))
    want, _ = oracle.gc(gs.rowptr, gs.col)
    np.testing.assert_array_equal(rep.arrays["color"], want)
    # MST find / verify (Boruvka == Kruskal in (weight, eid) order)
    gm, w, eid = graphs.mst_inputs(g, seed)
    wl = Workload(spec, {"rowptr": gm.rowptr, "col": gm.col, "weight": w,
                         "eid": eid}, gm.n, gm)
    in_mst, total, k = oracle.mst(gm.rowptr, gm.col, w, eid)
    for name in ("mstf", "mstv"):
        rep, _ = run_config(BENCHMARKS[name], wl, BenchConfig(**policy))
        np.testing.assert_array_equal(rep.arrays["in_mst"], in_mst)
        assert rep.arrays["weight"].tolist() == [total, k]
