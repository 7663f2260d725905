"""Partitioned solves with the round loop in the library
(dp_sssp_part_solve_peer / dp_bfs_part_solve_peer): the fused exchange
(remote atomics into the owner's dist) plus a device-side OR of the parts'
round flags through signal slots, no host collective per round.  P parts on
one GPU run as P host threads with their own streams and workspaces
(dist.run_parts); results must equal the oracle bit for bit, and equal the
per-round Python-driven path (test_gpu_parity.py) on the same inputs."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle
from paper_2201_02789_b200.bench import BenchConfig, graphs

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

POLICIES = [
    dict(threshold=128, agg="block"),
    dict(threshold=1024, cfactor=16, agg="multiblock", group_size=1 << 20,
         parent_block=128, child_block=128, serial="warp"),
    dict(threshold=64, cfactor=4, agg="grid"),
]


def _sssp_parts(P, g, w, dev):
    from paper_2201_02789_b200 import dist as pdist
    ex = pdist.PeerLocal()
    parts = [pdist.SsspPeerPart(*pdist.partition_csr(g.rowptr, g.col, P, p, w),
                                g.n, P, p, 0, ex.alloc(g.n, P, dev), dev)
             for p in range(P)]
    ex.bind(parts)
    return ex, parts


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("pi", range(len(POLICIES)))
def test_sssp_part_solve_peer(P, pi):
    import torch
    from paper_2201_02789_b200 import dist as pdist
    g = graphs.rmat_graph(16, 1)
    w = graphs.edge_weights(g, 1)
    want, _ = oracle.sssp(g.rowptr, g.col, w, nthreads=0)
    dev = torch.device("cuda", 0)
    ex, parts = _sssp_parts(P, g, w, dev)
    cfg = BenchConfig(**POLICIES[pi]).to_c()
    for rep in range(3):  # later calls: new epoch over the same slots
        src = 0 if rep < 2 else 7
        d, rounds = pdist.sssp_1d_peer_solve(parts, cfg, ex, src=src)
        if src:
            want_s, _ = oracle.sssp(g.rowptr, g.col, w, src=src, nthreads=0)
        np.testing.assert_array_equal(d.cpu().numpy(),
                                      want if src == 0 else want_s)
        assert rounds >= 2
    remote = sum(p.stats[-1]["remote_ops"] for p in parts)
    assert (remote > 0) == (P > 1)


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("spread", [False, True])
def test_bfs_part_solve_peer(P, spread):
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
    for pol in POLICIES[:2]:
        d, c, levels = pdist.bfs_1d_peer_solve(parts, BenchConfig(**pol).to_c(),
                                               ex)
        np.testing.assert_array_equal(d.cpu().numpy(), want_d)
        np.testing.assert_array_equal(c.cpu().numpy(), want_c)
        assert levels == want_lv
        assert all(p.stats[-1]["iterations"] == want_lv for p in parts)


def test_solve_matches_per_round_driver():
    """Same rounds and distances as the per-round Python-driven path."""
    import torch
    from paper_2201_02789_b200 import dist as pdist
    g = graphs.rmat_graph(14, 1)
    w = graphs.edge_weights(g, 1)
    dev = torch.device("cuda", 0)
    ex, parts = _sssp_parts(1, g, w, dev)
    cfg = BenchConfig(**POLICIES[1]).to_c()
    d1, r1 = pdist.sssp_1d_peer(parts, pdist.DeviceSsspPeerOps(cfg), ex)
    d2, r2 = pdist.sssp_1d_peer_solve(parts, cfg, ex)
    np.testing.assert_array_equal(d1.cpu().numpy(), d2.cpu().numpy())
    assert r1 == r2


CHILD_TIMEOUT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2201_02789_b200 import dist as pdist
from paper_2201_02789_b200._lib import DeviceTrap
from paper_2201_02789_b200.bench import BenchConfig, graphs
g = graphs.rmat_graph(12, 1)
w = graphs.edge_weights(g, 1)
dev = torch.device("cuda", 0)
ex = pdist.PeerLocal()
parts = [pdist.SsspPeerPart(*pdist.partition_csr(g.rowptr, g.col, 2, p, w),
                            g.n, 2, p, 0, ex.alloc(g.n, 2, dev), dev)
         for p in range(2)]
ex.bind(parts)
try:  # only part 0 runs: its barrier never completes
    pdist.sssp_1d_peer_solve(parts[:1], BenchConfig().to_c(), ex)
    print("NO ERROR")
except DeviceTrap as e:
    print("TRAP", e.kind, e.message)
"""


def test_solve_times_out_without_peers():
    """A part whose peers never arrive fails after $DYNPAR_PEER_TIMEOUT_MS
    instead of hanging the GPU."""
    env = dict(os.environ, DYNPAR_PEER_TIMEOUT_MS="1500")
    r = subprocess.run([sys.executable, "-c", CHILD_TIMEOUT, str(ROOT)],
                       capture_output=True, text=True, env=env, timeout=300)
    assert "TRAP cuda-error" in r.stdout and "timed out" in r.stdout, \
        r.stdout + r.stderr[-2000:]
