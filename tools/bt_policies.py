"""BT 25k: device time of a few launch-heavy and launch-free policies."""
import itertools
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2201_02789_b200.bench import (INF_THRESHOLD, BenchConfig, load,  # noqa
                                         run_config)
bench, wl = load("bt", "curves:25000:seed1")
pols = [dict(threshold=INF_THRESHOLD, serial="warp", parent_block=64)]
for T, C, cb, agg, pb in itertools.product((4, 16, 64), (1, 2, 4),
                                           (64, 128, 256),
                                           ("multiblock", "grid"), (64, 256)):
    pols.append(dict(threshold=T, cfactor=C, agg=agg, group_size=1 << 20,
                     parent_block=pb, child_block=cb, serial="warp"))
res = []
for d in pols:
    ts = [run_config(bench, wl, BenchConfig(**d))[0].ns_device / 1e3
          for _ in range(6)]
    res.append((statistics.median(ts[1:]), d))
res.sort(key=lambda r: r[0])
for t, d in res[:12]:
    print("%.1f us" % t, d, flush=True)
print("launch-free:", [r for r in res if r[1].get("threshold") == INF_THRESHOLD])
