"""GC device time for a set of policies on one RMAT graph."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2201_02789_b200.bench import (INF_THRESHOLD, BenchConfig, load,  # noqa
                                         run_config)
bench, wl = load("gc", sys.argv[1] if len(sys.argv) > 1 else "rmat:20:seed1")
for d in (dict(threshold=256, cfactor=8, agg="multiblock", group_size=1 << 20,
               parent_block=256, child_block=128, serial="warp", persistent=1),
          dict(threshold=256, cfactor=8, agg="multiblock", group_size=1 << 20,
               parent_block=256, child_block=128, serial="warp", persistent=2),
          dict(threshold=128, cfactor=8, agg="multiblock", group_size=1 << 20,
               parent_block=256, child_block=128, serial="warp", persistent=2),
          dict(threshold=1024, cfactor=8, agg="multiblock", group_size=1 << 20,
               parent_block=256, child_block=128, serial="warp", persistent=2),
          dict(threshold=256, cfactor=8, agg="multiblock", group_size=1 << 20,
               parent_block=128, child_block=128, serial="warp", persistent=4),
          dict(threshold=INF_THRESHOLD, serial="warp", parent_block=256),
          dict(threshold=INF_THRESHOLD, serial="thread", parent_block=256),
          dict(threshold=256, agg="block", serial="warp", parent_block=256,
               child_block=128),
          dict(threshold=256, cfactor=8, agg="multiblock", group_size=64,
               parent_block=256, child_block=128, serial="warp"),
          dict(threshold=256, cfactor=8, agg="multiblock", group_size=1 << 20,
               parent_block=256, child_block=128, serial="warp"),
          dict(threshold=64, agg="grid", parent_block=256, child_block=128,
               serial="warp")):
    reps = [run_config(bench, wl, BenchConfig(**d))[0] for _ in range(2)]
    r = reps[-1]
    print(f"{r.ns_device / 1e6:9.2f} ms rounds={r.iterations} "
          f"launches={r.num_launches} {d}", flush=True)
