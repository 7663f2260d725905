"""TC RMAT-22 device time for a few policies (and exactness vs a count)."""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa
bench, wl = load("tc", "rmat:22:seed1")
for d in (dict(threshold=32, cfactor=4, agg="grid", parent_block=128,
               child_block=256, serial="warp"),
          dict(threshold=32, cfactor=4, agg="grid", parent_block=128,
               child_block=128, serial="warp"),
          dict(threshold=16, cfactor=8, agg="grid", parent_block=128,
               child_block=256, serial="warp"),
          dict(threshold=64, cfactor=4, agg="multiblock", group_size=1 << 20,
               parent_block=128, child_block=256, serial="warp")):
    reps = [run_config(bench, wl, BenchConfig(**d))[0] for _ in range(4)]
    print("%.3f ms" % (statistics.median(r.ns_device for r in reps[1:]) / 1e6),
          int(reps[-1].arrays["triangles"][0]), d, flush=True)
