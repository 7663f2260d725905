"""Parity at the BASELINE / bench sizes (B200 only): TC and MST on RMAT-22,
SP on the bench's 5-SAT formula, each against the CPU oracle, plus the
size-independent shard-sum property of the multi-GPU TC partition."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle
from paper_2201_02789_b200 import dist as pdist
from paper_2201_02789_b200.bench import BenchConfig, load, run_config
from paper_2201_02789_b200.bench.benchmarks import Workload

pytestmark = pytest.mark.gpu

TC_POLICY = dict(threshold=32, cfactor=4, agg="grid", parent_block=128,
                 child_block=256, serial="warp")
MST_POLICY = dict(threshold=1024, cfactor=16, agg="multiblock",
                  group_size=1 << 20, parent_block=256, child_block=128,
                  serial="warp")


def test_tc_rmat22_exact_and_shards_sum():
    bench, wl = load("tc", "rmat:22:seed1")
    gp = wl.payload[1]
    want = oracle.tc(gp.rowptr, gp.col, nthreads=0)
    rep, _ = run_config(bench, wl, BenchConfig(**TC_POLICY))
    assert int(rep.arrays["triangles"][0]) == want
    # the work-balanced edge-range shards of 4 GPUs add up to the total
    tot = 0
    for rank in range(4):
        lo, hi = pdist.balanced_ranges(pdist.tc_edge_cost(gp.rowptr, gp.col),
                                       4)[rank]
        out, _ = bench.run(wl, BenchConfig(**TC_POLICY).to_c(), lo=lo, hi=hi)
        tot += int(out["triangles"][0])
    assert tot == want


@pytest.mark.parametrize("name", ["mstf", "mstv"])
def test_mst_rmat22_bit_exact(name):
    bench, wl = load(name, "rmat:22:seed1")
    b = wl.buffers
    in_mst, total, k = oracle.mst(b["rowptr"], b["col"], b["weight"],
                                  b["eid"])
    rep, _ = run_config(bench, wl, BenchConfig(**MST_POLICY))
    np.testing.assert_array_equal(rep.arrays["in_mst"], in_mst)
    assert rep.arrays["weight"].tolist() == [total, k]


def test_sp_ksat5_bench_size_within_tolerance():
    bench, wl = load("sp", "ksat5:200000:seed1")
    wl = Workload(wl.spec, dict(wl.buffers, max_sweeps=20, eps=0.0), wl.n,
                  wl.payload)
    want = oracle.sp(wl.payload, wl.buffers["eta0"], 20, 0.0)
    rep, _ = run_config(bench, wl, BenchConfig(
        threshold=128, cfactor=4, agg="multiblock", group_size=1 << 20,
        parent_block=128, child_block=128, serial="thread"))
    assert rep.iterations == 20
    # north star: surveys within 1e-5 relative (1e-7 absolute floor)
    np.testing.assert_allclose(rep.arrays["eta"], want[0], rtol=1e-5,
                               atol=1e-7)
    np.testing.assert_allclose(rep.arrays["wpos"], want[1], rtol=1e-5,
                               atol=1e-6)
