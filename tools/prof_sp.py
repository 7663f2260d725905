"""One SP run (fixed sweeps) on a random k-SAT formula under a policy, for ncu.

    python tools/prof_sp.py ksat5:200000:seed1 '{"threshold":32,...}' [sweeps]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa
from paper_2201_02789_b200.bench.benchmarks import Workload  # noqa

spec, policy = sys.argv[1], json.loads(sys.argv[2])
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
bench, wl = load("sp", spec)
wl = Workload(wl.spec, dict(wl.buffers, max_sweeps=sweeps, eps=0.0), wl.n,
              wl.payload)
rep, _ = run_config(bench, wl, BenchConfig(**policy))
print(json.dumps({"sweeps": rep.iterations, "ms": rep.ns_device / 1e6}))
