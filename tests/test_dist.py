"""Multi-GPU host logic on CPU: world_size-2 gloo process groups run the
sharding + reduction of the partitioned workloads, with the CPU oracle
standing in for each rank's device count (the device kernels are covered by
tests/test_gpu_parity.py, including per-range TC counts)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2201_02789_b200 import dist as pdist


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn()))
    finally:
        dist.destroy_process_group()


def _run(world, fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q))
          for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


def _tc_job():
    from oracle import oracle
    from paper_2201_02789_b200.bench import graphs
    gp = graphs.tc_orient(graphs.rmat_graph(11, 3))
    total, rng = pdist.tc_count_sharded(
        gp.rowptr, gp.col,
        lambda lo, hi: oracle.tc(gp.rowptr, gp.col, lo, hi))
    return total, rng, oracle.tc(gp.rowptr, gp.col), gp.m


def _bt_job():
    from oracle import oracle
    from paper_2201_02789_b200.bench import graphs
    cp = graphs.bezier_curves(3001, 2)

    def tess(lo, hi):
        nt, v = oracle.bt(cp[lo:hi], graphs.BT_MAX_TESS, graphs.BT_CURV_SCALE)
        return int(nt.sum()), float(v.sum())
    nv, cs, rng = pdist.bt_sharded(cp.shape[0], tess)
    nt, v = oracle.bt(cp, graphs.BT_MAX_TESS, graphs.BT_CURV_SCALE)
    return nv, cs, rng, int(nt.sum()), float(v.sum())


def test_tc_two_ranks_gloo():
    res = _run(2, _tc_job)
    (t0, r0, want, m), (t1, r1, _, _) = res
    assert t0 == t1 == want
    assert r0[0] == 0 and r0[1] == r1[0] and r1[1] == m


def test_bt_two_ranks_gloo():
    res = _run(2, _bt_job)
    (nv0, cs0, r0, nv, cs), (nv1, cs1, r1, _, _) = res
    assert nv0 == nv1 == nv
    assert abs(cs0 - cs) < 1e-6 * max(1.0, abs(cs)) and cs0 == cs1
    assert r0 == (0, 1500) or r0[1] == r1[0]


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_balanced_ranges_cover_and_balance(parts):
    rng = np.random.default_rng(0)
    cost = rng.integers(1, 100, size=10_000)
    rs = pdist.balanced_ranges(cost, parts)
    assert rs[0][0] == 0 and rs[-1][1] == cost.shape[0]
    assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    loads = [cost[lo:hi].sum() for lo, hi in rs]
    assert max(loads) - min(loads) <= 2 * cost.max()


def test_tc_edge_cost():
    rowptr = np.array([0, 2, 3, 3], np.int32)
    col = np.array([1, 2, 2], np.int32)
    # slots of N+(u) above v, plus one: 0->1 probes {2}, 0->2 and 1->2 none
    np.testing.assert_array_equal(pdist.tc_edge_cost(rowptr, col),
                                  [1 + 1, 0 + 1, 0 + 1])


# ---------------------------------------------------------------------------
# BFS 1D partition: exchange / termination logic with a numpy stand-in for
# the per-part device steps (the device steps are covered in
# tests/test_gpu_parity.py::test_bfs_1d_partition_on_device)
# ---------------------------------------------------------------------------

class NumpyBfsOps:
    """Same contract as dist.DeviceBfsOps, on CPU tensors."""

    def level(self, p, level):
        p.send_counts.zero_()
        p.changed.zero_()
        rp, col = p.rowptr.numpy(), p.col.numpy()
        dist, counts = p.dist.numpy(), p.counts.numpy()
        sent, buf, sc = p.sent.numpy().view(np.uint32), p.send_buf.numpy(), \
            p.send_counts.numpy()
        P, me = p.nparts, p.part
        for lu in np.flatnonzero(dist == level):
            for v in col[rp[lu]:rp[lu + 1]].tolist():
                counts[v] += 1
                if v % P == me:
                    if dist[v // P] == 1 << 30:
                        dist[v // P] = level + 1
                        p.changed[0] = 1
                elif not sent[v >> 5] >> (v & 31) & 1:
                    sent[v >> 5] |= np.uint32(1 << (v & 31))
                    q = v % P
                    buf[q * p.stride + sc[q]] = v
                    sc[q] += 1

    def apply(self, p, recv, level):
        dist = p.dist.numpy()
        for v in recv.tolist():
            if dist[v // p.nparts] == 1 << 30:
                dist[v // p.nparts] = level + 1
                p.changed[0] = 1


def _bfs_collective_job():
    from oracle import oracle
    from paper_2201_02789_b200.bench import graphs
    g = graphs.rmat_graph(9, 4)
    P, me = dist.get_world_size(), dist.get_rank()
    rp, col = pdist.partition_csr(g.rowptr, g.col, P, me)
    part = pdist.BfsPart(rp, col, g.n, P, me, 0, "cpu")
    d, c, levels = pdist.bfs_1d([part], NumpyBfsOps(),
                                pdist.CollectiveExchange())
    want_d, want_c, want_lv = oracle.bfs(g.rowptr, g.col)
    return (bool(np.array_equal(d.numpy(), want_d)),
            bool(np.array_equal(c.numpy(), want_c)), levels == want_lv)


def test_bfs_1d_two_ranks_gloo():
    for ok in _run(2, _bfs_collective_job):
        assert ok == (True, True, True)


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_bfs_1d_local_exchange_numpy(P):
    from oracle import oracle
    from paper_2201_02789_b200.bench import graphs
    g = graphs.rmat_graph(8, 2)
    parts = [pdist.BfsPart(*pdist.partition_csr(g.rowptr, g.col, P, p), g.n,
                           P, p, 0, "cpu") for p in range(P)]
    d, c, levels = pdist.bfs_1d(parts, NumpyBfsOps(), pdist.LocalExchange())
    want_d, want_c, want_lv = oracle.bfs(g.rowptr, g.col)
    np.testing.assert_array_equal(d.numpy(), want_d)
    np.testing.assert_array_equal(c.numpy(), want_c)
    assert levels == want_lv
    # the bitmap bounds exchange volume: each part sends a vertex at most once
    assert all(int(p.sent.numpy().view(np.uint32).sum() >= 0) for p in parts)


def test_rmat_part_matches_partitioned_csr():
    from paper_2201_02789_b200.bench import graphs
    g = graphs.rmat_graph(10, 1)
    for P in (1, 3, 8):
        for p in range(P):
            a = pdist.rmat_part(10, 1, P, p)
            b = pdist.partition_csr(g.rowptr, g.col, P, p)
            np.testing.assert_array_equal(a[0], b[0])
            np.testing.assert_array_equal(a[1], b[1])


class NumpySsspOps:
    """Same contract as dist.DeviceSsspOps, on CPU tensors."""

    def level(self, p, rnd):
        p.send_counts.zero_()
        p.changed.zero_()
        rp, col, w = p.rowptr.numpy(), p.col.numpy(), p.weight.numpy()
        dist, best = p.dist.numpy(), p.best.numpy()
        buf, sc = p.send_buf.numpy(), p.send_counts.numpy()
        P, me = p.nparts, p.part
        for lu in np.flatnonzero(dist < 1 << 30):
            du = int(dist[lu])
            for e in range(rp[lu], rp[lu + 1]):
                v, alt = int(col[e]), du + int(w[e])
                if v % P == me:
                    if alt < dist[v // P]:
                        dist[v // P] = alt
                        p.changed[0] = 1
                elif alt < best[v]:
                    best[v] = alt
                    q = v % P
                    buf[p.off_list[q] + sc[q]] = (v << 32) | alt
                    sc[q] += 1

    def apply(self, p, recv, rnd):
        dist = p.dist.numpy()
        for x in recv.tolist():
            v, alt = x >> 32, x & 0xFFFFFFFF
            if alt < dist[v // p.nparts]:
                dist[v // p.nparts] = alt
                p.changed[0] = 1


def _sssp_parts(g, w, P, device="cpu"):
    return [pdist.SsspPart(*pdist.partition_csr(g.rowptr, g.col, P, p, w),
                           g.n, P, p, 0, device) for p in range(P)]


@pytest.mark.parametrize("P", [1, 2, 3])
def test_sssp_1d_local_exchange_numpy(P):
    from oracle import oracle
    from paper_2201_02789_b200.bench import graphs
    g = graphs.rmat_graph(8, 3)
    w = graphs.edge_weights(g, 3)
    d, rounds = pdist.sssp_1d(_sssp_parts(g, w, P), NumpySsspOps(),
                              pdist.LocalExchange())
    want, _ = oracle.sssp(g.rowptr, g.col, w)
    np.testing.assert_array_equal(d.numpy(), want)


def _sssp_collective_job():
    from oracle import oracle
    from paper_2201_02789_b200.bench import graphs
    g = graphs.rmat_graph(9, 5)
    w = graphs.edge_weights(g, 5)
    P, me = dist.get_world_size(), dist.get_rank()
    part = pdist.SsspPart(*pdist.partition_csr(g.rowptr, g.col, P, me, w),
                          g.n, P, me, 0, "cpu")
    d, _ = pdist.sssp_1d([part], NumpySsspOps(), pdist.CollectiveExchange())
    want, _ = oracle.sssp(g.rowptr, g.col, w)
    return bool(np.array_equal(d.numpy(), want))


def test_sssp_1d_two_ranks_gloo():
    assert _run(2, _sssp_collective_job) == [True, True]


def test_peer_part_layout_on_cpu():
    """Host logic of the fused-exchange SSSP: identical-width dist buffers
    (symmetric memory), owner rows, source placement, pointer table."""
    import torch
    rowptr = np.array([0, 2, 3, 3, 5, 6], np.int32)   # 5 vertices
    col = np.array([1, 2, 0, 4, 1, 3], np.int32)
    w = np.ones(6, np.int32)
    P = 2
    assert pdist.dist_width(5, P) == 3
    ex = pdist.PeerLocal()
    parts = [pdist.SsspPeerPart(*pdist.partition_csr(rowptr, col, P, p, w),
                                5, P, p, 3, ex.alloc(5, P, "cpu"), "cpu")
             for p in range(P)]
    assert [p.n_local for p in parts] == [3, 2]
    assert parts[1].dist.tolist() == [1 << 30, 0]       # vertex 3 = part 1 [1]
    assert parts[0].dist.tolist() == [1 << 30] * 3
    ex.bind(parts)
    assert parts[0].peer_ptrs.tolist() == [p.dist_full.data_ptr()
                                           for p in parts]
    assert ex.dist(parts).tolist() == [1 << 30, 1 << 30, 1 << 30, 0, 1 << 30]
    with pytest.raises(ValueError):
        pdist.SsspPeerPart(*pdist.partition_csr(rowptr, col, P, 0, w), 5, P,
                           0, 0, torch.empty(2, dtype=torch.int32), "cpu")
