"""Golden counters for the pass-order knob, from the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_order_golden.py

`dynoptc.pipeline.transform(order=...)` (pipeline.py:45-81) applies the
enabled passes in the given order.  This records, for every permutation and
subset of "TCA" on a few T / C / A configurations, the reference's
run_config counters, digest and pass manifest (which passes transformed and
which were skipped, e.g. a threshold pass placed after coarsening).  The
B200 `BenchConfig.order_effect` must reproduce the manifest and the device
counters must reproduce the numbers (tests/test_api.py,
tests/test_gpu_parity.py).  Writes tests/golden/order_counters.json.
"""

from __future__ import annotations

import itertools
import json
from pathlib import Path

from dynoptc.bench import BenchConfig, load, run_config, run_reference
from dynoptc.sim import CostParams

HERE = Path(__file__).resolve().parent
ORDERS = ["".join(p) for p in itertools.permutations("TCA")] + \
    ["TC", "CT", "TA", "AT", "CA", "AC", "T", "C", "A", ""]
CONFIGS = [
    dict(threshold=8, cfactor=3, agg="block"),
    dict(threshold=8, cfactor=3, agg="multiblock", group_size=4),
    dict(threshold=8, cfactor=3, agg="grid"),
    dict(threshold=4, cfactor=2, agg="multiblock", group_size=2),
    dict(cfactor=4, agg="block"),
]
DATASETS = [("bfs", "powerlaw:2000:seed1"), ("bfs", "road:1000:seed7"),
            ("manylaunch", "sizes:1024:seed1"), ("sssp", "powerlaw:150:seed3")]


def main() -> None:
    big = CostParams(queue_capacity=10 ** 8)
    rows = []
    for bench_name, spec in DATASETS:
        bench, wl = load(bench_name, spec)
        ref = run_reference(bench, wl)
        for cfg in CONFIGS:
            for order in ORDERS:
                rep, res = run_config(bench, wl, BenchConfig(order=order, **cfg),
                                      cost=big)
                assert rep.memory_digest == ref.memory_digest
                rows.append({
                    "bench": bench_name, "dataset": spec, "config": cfg,
                    "order": order, "digest": rep.memory_digest,
                    "num_launches": rep.num_launches,
                    "host_launches": rep.host_launches,
                    "blocks_scheduled": rep.blocks_scheduled,
                    "manifest": [e.render() for e in res.manifest]})
        print(bench_name, spec, "ok", flush=True)
    (HERE / "order_counters.json").write_text(json.dumps(rows, indent=0))
    print("wrote", len(rows), "rows")


if __name__ == "__main__":
    main()
