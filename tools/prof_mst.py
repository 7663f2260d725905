"""One MST run (mstf/mstv) on an RMAT graph under a policy, for ncu.

    python tools/prof_mst.py mstf 22 '{"threshold":1024,...}' [runs]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa

name, scale = sys.argv[1], int(sys.argv[2])
policy = json.loads(sys.argv[3])
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 2
bench, wl = load(name, f"rmat:{scale}:seed1")
for _ in range(runs):
    rep, _ = run_config(bench, wl, BenchConfig(**policy))
print(json.dumps({"iterations": rep.iterations, "launches": rep.num_launches,
                  "ms": rep.ns_device / 1e6}))
