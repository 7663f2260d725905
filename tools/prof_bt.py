"""One BT run (25k curves) under a policy (for ncu)."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa
bench, wl = load("bt", "curves:25000:seed1")
cfg = BenchConfig(**json.loads(sys.argv[1]))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    rep, _ = run_config(bench, wl, cfg)
print(rep.ns_device / 1e3)
