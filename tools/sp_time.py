"""Time SP sweeps on random k-SAT under several policies (vs the oracle)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402
from paper_2201_02789_b200.bench import (INF_THRESHOLD, BenchConfig,  # noqa
                                         load, run_config, run_reference)
from paper_2201_02789_b200.bench.benchmarks import Workload  # noqa: E402

for spec in sys.argv[1:] or ["ksat3:1000000:seed1", "ksat5:200000:seed1"]:
    t = time.time()
    bench, wl = load("sp", spec)
    b = dict(wl.buffers, max_sweeps=20, eps=0.0)
    wl = Workload(wl.spec, b, wl.n, wl.payload)
    print(spec, "prep s %.1f" % (time.time() - t), "edges",
          b["lits"].shape[0], flush=True)
    t = time.time()
    want = oracle.sp(wl.payload, b["eta0"], 20, 0.0)
    print("oracle s %.2f" % (time.time() - t), flush=True)
    for pol in [dict(threshold=INF_THRESHOLD, serial="warp"), dict(),
                dict(agg="block"), dict(agg="grid"),
                dict(threshold=32, agg="block", serial="warp"),
                dict(threshold=64, cfactor=8, agg="multiblock",
                     group_size=1 << 20, parent_block=256, child_block=128,
                     serial="warp"),
                dict(threshold=32, cfactor=4, agg="grid", parent_block=256,
                     child_block=64, serial="warp")]:
        try:
            for _ in range(2):
                rep, _ = run_config(bench, wl, BenchConfig(**pol))
            err = np.abs(rep.arrays["eta"] - want[0]).max()
            print(pol, "ms %.3f" % (rep.ns_device / 1e6), "sweeps",
                  rep.iterations, "launches", rep.num_launches,
                  "max abs err %.2e" % err, flush=True)
        except Exception as e:  # noqa: BLE001
            print(pol, "ERR", e, flush=True)
    rep = run_reference(bench, wl)
    print("nocdp ms %.3f" % (rep.ns_device / 1e6), flush=True)
