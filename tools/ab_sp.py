"""A/B an env toggle on SP (5-SAT 200k and 3-SAT 1M, 20 sweeps) + accuracy."""
import os
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from oracle import oracle  # noqa: E402
from bench import BEST  # noqa: E402
from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa
from paper_2201_02789_b200.bench.benchmarks import Workload  # noqa: E402
var, vals = sys.argv[1], sys.argv[2:4]
for spec in ("ksat5:200000:seed1", "ksat3:1000000:seed1"):
    bench, wl = load("sp", spec)
    wl = Workload(wl.spec, dict(wl.buffers, max_sweeps=20, eps=0.0), wl.n,
                  wl.payload)
    want = oracle.sp(wl.payload, wl.buffers["eta0"], 20, 0.0)
    for v in vals:
        os.environ[var] = v
        for pol in (BEST["sp"], dict(BEST["sp"], serial="warp"),
                    dict(threshold=2147483647, serial="thread")):
            reps = [run_config(bench, wl, BenchConfig(**pol))[0]
                    for _ in range(3)]
            ok = np.allclose(reps[-1].arrays["eta"], want[0], rtol=1e-5,
                             atol=1e-7)
            print(spec, var, v, "%.2f ms" % (statistics.median(
                r.ns_device for r in reps) / 1e6), "ok", ok, pol, flush=True)
