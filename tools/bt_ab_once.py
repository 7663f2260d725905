"""Median device time of the tuned BT policy and the config-2 policy (for
A/B of compile-time variants via DYNPAR_LIB)."""
import statistics
import sys
sys.path.insert(0, '.')
from bench import BEST  # noqa: E402
from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa

bench, wl = load("bt", "curves:25000:seed1")
c2 = dict(threshold=64, cfactor=16, agg="multiblock", group_size=4,
          parent_block=256, child_block=32, serial="warp")
for name, pol in (("best", BEST["bt"]), ("config2", c2)):
    ts = [run_config(bench, wl, BenchConfig(**pol))[0].ns_device / 1e3
          for _ in range(12)]
    print(name, "us %.1f" % statistics.median(ts[2:]))
