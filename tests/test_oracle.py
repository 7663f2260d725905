"""The CPU oracle and the input generators, pinned to the reference.

- generators: byte-identical to dynoptc.bench.graphs (golden arrays made by
  importing the reference, tests/golden/make_golden.py);
- oracle bfs/sssp/manylaunch: equal to dynoptc.bench.run_reference outputs
  and memory digests, including RMAT graphs injected into the reference;
- oracle tc/bt (no reference implementation): against independent
  brute-force restatements here.
"""

from __future__ import annotations

import heapq
from collections import deque

import numpy as np
import pytest

from oracle import oracle
from paper_2201_02789_b200.bench import graphs
from paper_2201_02789_b200.bench.graphs import (UNREACHED, make_graph,
                                                parse_spec)
from paper_2201_02789_b200.bench.report import memory_digest

GRAPH_SPECS = ["hand", "powerlaw:150:seed2", "road:180:seed3",
               "powerlaw:150:seed3", "road:160:seed4", "powerlaw:120:seed5",
               "powerlaw:2000:seed1", "road:1000:seed7"]
SIZE_SPECS = ["sizes:100:seed4", "sizes:1024:seed1", "sizes:40:seed3",
              "sizes:20:seed2"]


def _weights(spec, g):
    s = parse_spec(spec)
    return (np.ones(g.m, np.int32) if s.kind == "hand"
            else graphs.edge_weights(g, s.seed))


# ---------------------------------------------------------------------------
# generators == reference generators
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("spec", GRAPH_SPECS)
def test_graph_generators_match_reference(spec, golden_arrays):
    g = make_graph(parse_spec(spec))
    np.testing.assert_array_equal(g.rowptr, golden_arrays[f"gen/{spec}/rowptr"])
    np.testing.assert_array_equal(g.col, golden_arrays[f"gen/{spec}/col"])
    np.testing.assert_array_equal(
        graphs.edge_weights(g, parse_spec(spec).seed),
        golden_arrays[f"gen/{spec}/weights"])


@pytest.mark.parametrize("spec", SIZE_SPECS)
def test_child_sizes_match_reference(spec, golden_arrays):
    s = parse_spec(spec)
    np.testing.assert_array_equal(graphs.child_sizes(s.size, s.seed),
                                  golden_arrays[f"gen/{spec}/sizes"])


def test_hand_fixture():
    g = graphs.hand_graph()
    dist, _, _ = oracle.bfs(g.rowptr, g.col)
    assert tuple(dist.tolist()) == graphs.HAND_BFS_DISTANCES


# ---------------------------------------------------------------------------
# oracle == reference run_reference (No-CDP variant on the simulator)
# ---------------------------------------------------------------------------

def _ref(golden, bench, spec):
    return next(r for r in golden["reference"]
                if r["bench"] == bench and r["dataset"] == spec)


@pytest.mark.parametrize("nthreads", [1, 4])
@pytest.mark.parametrize("spec", GRAPH_SPECS)
def test_oracle_bfs_matches_reference(spec, nthreads, golden, golden_arrays):
    g = make_graph(parse_spec(spec))
    dist, counts, levels = oracle.bfs(g.rowptr, g.col, nthreads=nthreads)
    np.testing.assert_array_equal(dist, golden_arrays[f"ref/bfs/{spec}/dist"])
    np.testing.assert_array_equal(counts,
                                  golden_arrays[f"ref/bfs/{spec}/counts"])
    ref = _ref(golden, "bfs", spec)
    assert memory_digest({"dist": dist, "counts": counts},
                         {"dist": "int", "counts": "int"}) == ref["digest"]
    assert levels == ref["host_launches"]  # level-synchronous: deterministic


@pytest.mark.parametrize("nthreads", [1, 4])
@pytest.mark.parametrize("spec", GRAPH_SPECS)
def test_oracle_sssp_matches_reference(spec, nthreads, golden, golden_arrays):
    g = make_graph(parse_spec(spec))
    dist, _ = oracle.sssp(g.rowptr, g.col, _weights(spec, g),
                          nthreads=nthreads)
    np.testing.assert_array_equal(dist, golden_arrays[f"ref/sssp/{spec}/dist"])
    assert memory_digest({"dist": dist}, {"dist": "int"}) == \
        _ref(golden, "sssp", spec)["digest"]


@pytest.mark.parametrize("spec", SIZE_SPECS)
def test_oracle_manylaunch_matches_reference(spec, golden, golden_arrays):
    s = parse_spec(spec)
    out, total = oracle.manylaunch(graphs.child_sizes(s.size, s.seed), 4)
    np.testing.assert_array_equal(out,
                                  golden_arrays[f"ref/manylaunch/{spec}/out"])
    np.testing.assert_array_equal(
        total, golden_arrays[f"ref/manylaunch/{spec}/total"])


# ---------------------------------------------------------------------------
# python mirrors of the reference tests (tests/test_bench.py:35-74)
# ---------------------------------------------------------------------------

def python_bfs(g, src=0):
    dist = [UNREACHED] * g.n
    dist[src] = 0
    q = deque([src])
    while q:
        u = q.popleft()
        for v in g.neighbors(u).tolist():
            if dist[v] == UNREACHED:
                dist[v] = dist[u] + 1
                q.append(v)
    return dist


def python_dijkstra(g, w, src=0):
    dist = [UNREACHED] * g.n
    dist[src] = 0
    heap = [(0, src)]
    rp = g.rowptr.tolist()
    col = g.col.tolist()
    w = w.tolist()
    while heap:
        d, u = heapq.heappop(heap)
        if d > dist[u]:
            continue
        for e in range(rp[u], rp[u + 1]):
            alt = d + w[e]
            if alt < dist[col[e]]:
                dist[col[e]] = alt
                heapq.heappush(heap, (alt, col[e]))
    return dist


@pytest.mark.parametrize("spec", ["rmat:8:seed1", "rmat:10:seed3",
                                  "powerlaw:500:seed9", "road:400:seed2"])
def test_oracle_against_python_mirrors(spec):
    g = make_graph(parse_spec(spec))
    dist, counts, _ = oracle.bfs(g.rowptr, g.col, nthreads=4)
    want = python_bfs(g)
    assert dist.tolist() == want
    reached = np.array(want) < UNREACHED
    exp_counts = np.bincount(
        g.col[np.repeat(reached, np.diff(g.rowptr))], minlength=g.n)
    np.testing.assert_array_equal(counts, exp_counts)
    w = _weights(spec, g)
    sd, _ = oracle.sssp(g.rowptr, g.col, w, nthreads=4)
    assert sd.tolist() == python_dijkstra(g, w)


# ---------------------------------------------------------------------------
# RMAT generator (builder-defined) and its parity through the reference
# ---------------------------------------------------------------------------

def test_rmat_generator_pinned(golden):
    g = graphs.rmat_graph(10, 1)
    gold = golden["rmat_generator"]
    assert int(g.rowptr.astype(np.int64).sum()) == \
        gold["scale10_seed1_rowptr_sum"]
    assert int(g.col.astype(np.int64).sum()) == gold["scale10_seed1_col_sum"]
    assert g.col[:16].tolist() == gold["scale10_seed1_col_head"]


def test_rmat_generator_shape_and_determinism():
    g = graphs.rmat_graph(12, 7)
    n, m = 1 << 12, 16 << 12
    assert g.n == n and g.m == m
    assert g.rowptr[0] == 0 and g.rowptr[-1] == m
    assert np.all(np.diff(g.rowptr) >= 0)
    assert g.col.min() >= 0 and g.col.max() < n
    rows_sorted = all(np.all(np.diff(g.neighbors(u)) >= 0)
                      for u in range(0, n, 97))
    assert rows_sorted
    g2 = graphs.rmat_graph(12, 7)
    np.testing.assert_array_equal(g.col, g2.col)
    assert not np.array_equal(graphs.rmat_graph(12, 8).col, g.col)
    # RMAT skew: vertex 0 is the heaviest source, (a+b)^scale of the edges
    deg = np.diff(g.rowptr)
    assert deg.argmax() == 0
    assert abs(deg[0] / m - 0.76 ** 12) < 0.01


@pytest.mark.parametrize("bench,scale,seed", [("bfs", 10, 1), ("bfs", 12, 1),
                                              ("bfs", 14, 1), ("bfs", 16, 1),
                                              ("sssp", 10, 1),
                                              ("sssp", 12, 2),
                                              ("sssp", 14, 1)])
def test_oracle_rmat_matches_reference_digest(bench, scale, seed, golden):
    rec = next(r for r in golden["rmat"] if r["bench"] == bench
               and r["scale"] == scale and r["seed"] == seed)
    g = graphs.rmat_graph(scale, seed)
    if bench == "bfs":
        dist, counts, levels = oracle.bfs(g.rowptr, g.col, nthreads=8)
        arrays = {"dist": dist, "counts": counts}
        assert levels == rec["host_launches"]
    else:
        dist, _ = oracle.sssp(g.rowptr, g.col, graphs.edge_weights(g, seed),
                              nthreads=8)
        arrays = {"dist": dist}
    assert memory_digest(arrays, {k: "int" for k in arrays}) == rec["digest"]


# ---------------------------------------------------------------------------
# triangle counting (parity unpinned by the reference: brute force here)
# ---------------------------------------------------------------------------

def _simple_undirected(g):
    src = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    dst = g.col.astype(np.int64)
    keep = src != dst
    a = np.concatenate([src[keep], dst[keep]])
    b = np.concatenate([dst[keep], src[keep]])
    key = np.unique(a * g.n + b)
    return key // g.n, key % g.n


def brute_triangles(g) -> int:
    a, b = _simple_undirected(g)
    adj = [set() for _ in range(g.n)]
    for x, y in zip(a.tolist(), b.tolist()):
        adj[x].add(y)
    t = 0
    for x in range(g.n):
        for y in adj[x]:
            if y > x:
                t += sum(1 for z in adj[x] & adj[y] if z > y)
    return t


def test_tc_orient_matches_numpy_restatement():
    """Rank-ordered CSR+: vertices relabelled by ascending (degree, id),
    u -> v iff rank u < rank v, rows ascending in the new ids."""
    g = graphs.rmat_graph(10, 2)
    gp = graphs.tc_orient(g)
    a, b = _simple_undirected(g)
    deg = np.bincount(a, minlength=g.n)
    rank = np.empty(g.n, np.int64)
    rank[np.lexsort((np.arange(g.n), deg))] = np.arange(g.n)
    ra, rb = rank[a], rank[b]
    keep = ra < rb
    ra, rb = ra[keep], rb[keep]
    order = np.lexsort((rb, ra))
    rowptr = np.concatenate(([0], np.cumsum(np.bincount(ra, minlength=g.n))))
    np.testing.assert_array_equal(gp.rowptr, rowptr)
    np.testing.assert_array_equal(gp.col, rb[order])
    assert gp.m * 2 == len(_simple_undirected(g)[0])
    src = np.repeat(np.arange(g.n), np.diff(gp.rowptr))
    assert (src < gp.col).all()


@pytest.mark.parametrize("spec", ["rmat:8:seed1", "rmat:9:seed4",
                                  "powerlaw:300:seed2", "road:300:seed1"])
def test_oracle_tc_matches_brute_force(spec):
    g = make_graph(parse_spec(spec))
    gp = graphs.tc_orient(g)
    want = brute_triangles(g)
    assert oracle.tc(gp.rowptr, gp.col, nthreads=1) == want
    assert oracle.tc(gp.rowptr, gp.col, nthreads=4) == want
    # edge-range shards add up (the multi-GPU partition)
    cuts = np.linspace(0, gp.m, 5).astype(int)
    assert sum(oracle.tc(gp.rowptr, gp.col, lo, hi)
               for lo, hi in zip(cuts[:-1], cuts[1:])) == want


# ---------------------------------------------------------------------------
# Bezier tessellation (parity unpinned by the reference)
# ---------------------------------------------------------------------------

def test_oracle_bt_counts_and_vertices():
    cp = graphs.bezier_curves(500, 1)
    ntess, verts = oracle.bt(cp, graphs.BT_MAX_TESS, graphs.BT_CURV_SCALE)
    p0, p1, p2 = (cp[:, i, :].astype(np.float32) for i in range(3))
    mid = np.float32(0.5) * (p0 + p2)
    d = p1 - mid
    ln = p2 - p0
    curv = (np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1])
            / np.sqrt(ln[:, 0] * ln[:, 0] + ln[:, 1] * ln[:, 1]))
    t = (curv * np.float32(graphs.BT_CURV_SCALE)).astype(np.float32)
    want = np.where(t < graphs.BT_MAX_TESS,
                    np.clip(t, 0, graphs.BT_MAX_TESS).astype(np.int32),
                    graphs.BT_MAX_TESS)
    np.testing.assert_array_equal(ntess, np.maximum(want, 4))
    assert verts.shape == (int(ntess.sum()), 2)
    # endpoints reproduce P0 and P2; all vertices inside the hull's box
    starts = np.concatenate(([0], np.cumsum(ntess)[:-1]))
    np.testing.assert_allclose(verts[starts], p0, atol=1e-7)
    np.testing.assert_allclose(verts[starts + ntess - 1], p2, atol=1e-7)
    assert verts.min() >= -1e-9 and verts.max() <= 1 + 1e-9


# ---------------------------------------------------------------------------
# graph colouring (no reference implementation: brute-force checks here)
# ---------------------------------------------------------------------------

def _py_gc_key(v, deg):
    """largest-log-degree-first, hash tie-break, vertex id last"""
    x = (v * 0x9E3779B1) & 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x85EBCA6B) & 0xFFFFFFFF
    x ^= x >> 13
    x = (x * 0xC2B2AE35) & 0xFFFFFFFF
    x ^= x >> 16
    lg = (deg + 1).bit_length() - 1
    return (lg << 59) | ((x >> 5) << 32) | v


@pytest.mark.parametrize("spec", ["hand", "rmat:9:seed1", "powerlaw:400:seed2",
                                  "road:500:seed3"])
def test_oracle_gc_is_priority_greedy_and_proper(spec):
    g = graphs.symmetrize(make_graph(parse_spec(spec)))
    color, k = oracle.gc(g.rowptr, g.col)
    src = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    assert np.all(color[src] != color[g.col])          # proper
    assert color.max() + 1 == k
    want = [-1] * g.n                                   # greedy mirror
    deg = np.diff(g.rowptr).tolist()
    for u in sorted(range(g.n), key=lambda v: _py_gc_key(v, deg[v]),
                    reverse=True):
        used = {want[w] for w in g.neighbors(u).tolist() if want[w] >= 0}
        c = 0
        while c in used:
            c += 1
        want[u] = c
    assert color.tolist() == want


def test_symmetrize_matches_numpy():
    g = graphs.rmat_graph(10, 4)
    s = graphs.symmetrize(g)
    a, b = _simple_undirected(g)
    order = np.lexsort((b, a))
    np.testing.assert_array_equal(s.col, b[order])
    np.testing.assert_array_equal(
        s.rowptr, np.concatenate(([0], np.cumsum(np.bincount(a, minlength=g.n)))))


# ---------------------------------------------------------------------------
# minimum spanning forest (MSTF / MSTV; no reference implementation): the
# Kruskal oracle against scipy's MST weight and a pure-Python Kruskal
# ---------------------------------------------------------------------------

MST_SPECS = ["hand", "rmat:9:seed1", "powerlaw:400:seed2", "road:500:seed3",
             "powerlaw:2000:seed1"]


@pytest.mark.parametrize("spec", MST_SPECS)
def test_mst_inputs_are_symmetric_and_canonical(spec):
    s = parse_spec(spec)
    g, w, eid = graphs.mst_inputs(make_graph(s), s.seed)
    mirror = graphs.edge_mirror(g)
    src = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    np.testing.assert_array_equal(src[mirror], g.col)       # reverse slot
    np.testing.assert_array_equal(g.col[mirror], src)
    np.testing.assert_array_equal(eid, np.minimum(np.arange(g.m), mirror))
    np.testing.assert_array_equal(w, w[mirror])              # symmetric
    assert w.min() >= 1 and w.max() <= 9
    assert np.all(src[eid] < g.col[eid])                     # (min, max) copy


@pytest.mark.parametrize("spec", MST_SPECS)
def test_oracle_mst_weight_matches_scipy(spec):
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components, minimum_spanning_tree
    s = parse_spec(spec)
    g, w, eid = graphs.mst_inputs(make_graph(s), s.seed)
    in_mst, total, k = oracle.mst(g.rowptr, g.col, w, eid)
    a = csr_matrix((w.astype(np.float64), g.col, g.rowptr), shape=(g.n, g.n))
    assert total == int(minimum_spanning_tree(a).sum())
    ncomp, _ = connected_components(a, directed=False)
    assert k == g.n - ncomp == int(in_mst.sum())
    assert total == int(w[in_mst.astype(bool)].sum())
    assert np.all(eid[in_mst.astype(bool)] == np.flatnonzero(in_mst))


@pytest.mark.parametrize("spec", ["hand", "powerlaw:150:seed2",
                                  "road:180:seed3", "rmat:7:seed2"])
def test_oracle_mst_is_kruskal_in_key_order(spec):
    s = parse_spec(spec)
    g, w, eid = graphs.mst_inputs(make_graph(s), s.seed)
    in_mst, _, _ = oracle.mst(g.rowptr, g.col, w, eid)
    src = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    parent = list(range(g.n))

    def find(x):
        while parent[x] != x:
            x = parent[x]
        return x
    want = np.zeros(g.m, np.uint8)
    for e in sorted((e for e in range(g.m) if eid[e] == e),
                    key=lambda e: (int(w[e]), e)):
        a, b = find(int(src[e])), find(int(g.col[e]))
        if a != b:
            parent[max(a, b)] = min(a, b)
            want[e] = 1
    np.testing.assert_array_equal(in_mst, want)


# ---------------------------------------------------------------------------
# survey propagation (no reference implementation): the oracle against the
# textbook update written with explicit clause sets (no division trick)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("spec", ["ksat3:60:seed1", "ksat5:40:seed2"])
def test_ksat_formula_invariants(spec):
    f = graphs.make_formula(parse_spec(spec))
    k, ratio = graphs.SAT_KINDS[parse_spec(spec).kind]
    assert f.k == k and f.nclauses == round(ratio * f.nvars)
    var = (f.lits >> 1).reshape(-1, k)
    assert all(len(set(r)) == k for r in var.tolist())     # distinct vars
    assert var.min() >= 0 and var.max() < f.nvars
    for i in range(f.nvars):                               # occurrence CSR
        occ = f.occ[f.occ_row[i]:f.occ_row[i + 1]]
        np.testing.assert_array_equal(occ, np.flatnonzero(var.reshape(-1) == i))


def _py_sp(f, eta0, sweeps):
    """Braunstein-Mezard-Zecchina SP, synchronous, straight from the sets."""
    k = f.k
    var = (f.lits >> 1).tolist()
    neg = (f.lits & 1).tolist()
    eta = list(map(float, eta0))
    occ = [f.occ[f.occ_row[i]:f.occ_row[i + 1]].tolist()
           for i in range(f.nvars)]
    for _ in range(sweeps):
        new = [0.0] * len(eta)
        for a in range(f.nclauses):
            for t in range(k):
                v = 1.0
                for j in range(k):
                    if j == t:
                        continue
                    e = a * k + j
                    x = var[e]
                    same = [b for b in occ[x] if b != e and neg[b] == neg[e]]
                    opp = [b for b in occ[x] if neg[b] != neg[e]]
                    S = float(np.prod([1 - eta[b] for b in same]))
                    U = float(np.prod([1 - eta[b] for b in opp]))
                    pu, ps, p0 = (1 - U) * S, (1 - S) * U, S * U
                    den = pu + ps + p0
                    v *= pu / den if den > 0 else 0.0
                new[a * k + t] = v
        eta = new
    return np.array(eta)


@pytest.mark.parametrize("spec", ["ksat3:60:seed1", "ksat5:40:seed2",
                                  "ksat3:200:seed3"])
def test_oracle_sp_matches_textbook_update(spec):
    s = parse_spec(spec)
    f = graphs.make_formula(s)
    eta0 = graphs.sp_initial_surveys(f, s.seed)
    for sweeps in (1, 3, 8):
        got = oracle.sp(f, eta0, sweeps, 0.0)
        assert got[3] == sweeps
        np.testing.assert_allclose(got[0], _py_sp(f, eta0, sweeps),
                                   rtol=1e-9, atol=1e-12)


def test_oracle_sp_biases_and_convergence():
    s = parse_spec("ksat3:2000:seed1")
    f = graphs.make_formula(s)
    eta, wpos, wneg, sweeps, delta = oracle.sp(
        f, graphs.sp_initial_surveys(f, s.seed), 200, 1e-3)
    assert sweeps < 200 and delta <= 1e-3        # converged
    assert np.all((eta >= 0) & (eta <= 1))
    assert np.all((wpos >= 0) & (wneg >= 0) & (wpos + wneg <= 1 + 1e-6))
