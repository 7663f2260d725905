"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container (the reference is importable only there):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json + reference_arrays.npz:
  - generator outputs of dynoptc.bench.graphs (hand, powerlaw, road, sizes,
    weights) so our restated generators are pinned byte-for-byte;
  - dynoptc.bench.run_reference outputs + memory digests for bfs / sssp /
    manylaunch on the reference's own test datasets (tests/test_bench.py)
    and on RMAT graphs from our generator injected through Workload(...);
  - dynoptc.bench.run_config launch/block counters for a grid of T/C/A
    configurations (the counter oracles of tests/test_passes.py), which the
    B200 device counters must reproduce with parent block 32.
Nothing here runs on the GPU box; the committed files travel instead.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))

from dynoptc.bench import (BenchConfig, child_sizes, edge_weights,  # noqa: E402
                           get_benchmark, load, make_graph, parse_spec,
                           run_config, run_reference)
from dynoptc.bench.benchmarks import Workload  # noqa: E402
from dynoptc.passes import INF_THRESHOLD  # noqa: E402
from dynoptc.sim import CostParams  # noqa: E402

GRAPH_SPECS = ["hand", "powerlaw:150:seed2", "road:180:seed3",
               "powerlaw:150:seed3", "road:160:seed4", "powerlaw:120:seed5",
               "powerlaw:2000:seed1", "road:1000:seed7"]
SIZE_SPECS = ["sizes:100:seed4", "sizes:1024:seed1", "sizes:40:seed3",
              "sizes:20:seed2"]

CONFIGS = [
    dict(),
    dict(threshold=4),
    dict(threshold=32),
    dict(threshold=INF_THRESHOLD),
    dict(agg="block"),
    dict(agg="multiblock", group_size=2),
    dict(agg="multiblock", group_size=4),
    dict(agg="grid"),
    dict(cfactor=2),
    dict(cfactor=4, agg="block"),
    dict(threshold=8, agg="block"),
    dict(threshold=8, agg="multiblock"),
    dict(threshold=2, cfactor=2, agg="grid"),
    dict(cfactor=2, agg="multiblock", group_size=2),
    dict(threshold=4, cfactor=8, agg="multiblock", group_size=4),
    dict(agg="block", agg_threshold=3),
    dict(threshold=33, cfactor=2, agg="block", agg_threshold=3),
]

BIG_QUEUE = CostParams(queue_capacity=10 ** 8)


def rmat_csr(scale: int, seed: int):
    from paper_2201_02789_b200.bench.graphs import rmat_graph
    g = rmat_graph(scale, seed)
    return [int(x) for x in g.rowptr], [int(x) for x in g.col]


def rmat_workload(bench_name: str, scale: int, seed: int):
    """Our RMAT CSR injected into the reference's Workload."""
    from dynoptc.bench.graphs import DatasetSpec, Graph, UNREACHED
    rowptr, col = rmat_csr(scale, seed)
    g = Graph(tuple(rowptr), tuple(col))
    n = g.n
    spec = DatasetSpec("rmat", scale, seed, f"rmat:{scale}:seed{seed}")
    dist = [UNREACHED] * n
    dist[0] = 0
    if bench_name == "bfs":
        bufs = {"rowptr": rowptr, "col": col, "dist": dist,
                "counts": [0] * n, "changed": [0]}
        payload = g
    else:
        w = edge_weights(g, seed)
        bufs = {"rowptr": rowptr, "col": col, "weight": w, "dist": dist,
                "changed": [0]}
        payload = (g, w)
    return get_benchmark(bench_name), Workload(spec, bufs, n, payload)


def main() -> None:
    out: dict = {"generators": {}, "reference": [], "counters": [],
                 "rmat": []}
    arrays: dict = {}
    for spec in GRAPH_SPECS:
        g = make_graph(parse_spec(spec))
        arrays[f"gen/{spec}/rowptr"] = np.array(g.rowptr, dtype=np.int64)
        arrays[f"gen/{spec}/col"] = np.array(g.col, dtype=np.int64)
        arrays[f"gen/{spec}/weights"] = np.array(
            edge_weights(g, parse_spec(spec).seed), dtype=np.int64)
    for spec in SIZE_SPECS:
        s = parse_spec(spec)
        arrays[f"gen/{spec}/sizes"] = np.array(child_sizes(s.size, s.seed),
                                               dtype=np.int64)

    for bench_name, specs in (("bfs", GRAPH_SPECS), ("sssp", GRAPH_SPECS),
                              ("manylaunch", SIZE_SPECS)):
        for spec in specs:
            bench, wl = load(bench_name, spec)
            ref = run_reference(bench, wl)
            rec = {"bench": bench_name, "dataset": spec,
                   "digest": ref.memory_digest,
                   "host_launches": ref.host_launches}
            out["reference"].append(rec)
            for name in bench.outputs:
                arrays[f"ref/{bench_name}/{spec}/{name}"] = np.array(
                    ref.buffers[name], dtype=np.int64)
            for cfg in CONFIGS:
                rep, _ = run_config(bench, wl, BenchConfig(**cfg),
                                    cost=BIG_QUEUE)
                assert rep.memory_digest == ref.memory_digest, (spec, cfg)
                out["counters"].append({
                    "bench": bench_name, "dataset": spec, "config": cfg,
                    "num_launches": rep.num_launches,
                    "host_launches": rep.host_launches,
                    "blocks_scheduled": rep.blocks_scheduled})
            print(bench_name, spec, "ok", flush=True)

    for bench_name, scale, seed in (("bfs", 10, 1), ("bfs", 12, 1),
                                    ("bfs", 14, 1), ("bfs", 16, 1),
                                    ("sssp", 10, 1), ("sssp", 12, 2),
                                    ("sssp", 14, 1)):
        bench, wl = rmat_workload(bench_name, scale, seed)
        ref = run_reference(bench, wl)
        rec = {"bench": bench_name, "scale": scale, "seed": seed,
               "digest": ref.memory_digest,
               "host_launches": ref.host_launches,
               "sums": {k: int(sum(ref.buffers[k])) for k in bench.outputs}}
        if scale <= 12:
            for name in bench.outputs:
                arrays[f"rmat/{bench_name}/{scale}/{seed}/{name}"] = \
                    np.array(ref.buffers[name], dtype=np.int64)
            rows = []
            for cfg in (dict(), dict(threshold=128, agg="block"),
                        dict(threshold=128, cfactor=8, agg="multiblock",
                             group_size=4)):
                rep, _ = run_config(bench, wl, BenchConfig(**cfg),
                                    cost=BIG_QUEUE)
                assert rep.memory_digest == ref.memory_digest
                rows.append({"config": cfg,
                             "num_launches": rep.num_launches,
                             "host_launches": rep.host_launches,
                             "blocks_scheduled": rep.blocks_scheduled})
            rec["counters"] = rows
        out["rmat"].append(rec)
        print("rmat", bench_name, scale, "ok", flush=True)

    rp, col = rmat_csr(10, 1)
    out["rmat_generator"] = {
        "scale10_seed1_rowptr_sum": int(sum(rp)),
        "scale10_seed1_col_sum": int(sum(col)),
        "scale10_seed1_col_head": col[:16]}
    (HERE / "reference_golden.json").write_text(json.dumps(out, indent=1))
    np.savez_compressed(HERE / "reference_arrays.npz", **arrays)
    print("wrote", HERE / "reference_golden.json")


if __name__ == "__main__":
    main()
