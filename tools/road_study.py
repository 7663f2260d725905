"""Low-parallelism study: on road-like
graphs (out-degree 1..8) child grids are tiny, so launches never pay; the
question is how close the CDP variants get to No-CDP once T/C/A remove the
launches, and what the mere presence of launch code costs."""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2201_02789_b200.bench import (BenchConfig, INF_THRESHOLD, load,
                                         run_config, run_reference)

args = [a for a in sys.argv[1:] if a != "--fast"]
spec = args[0] if args else "road:200000:seed1"
fast = "--fast" in sys.argv  # skip naive CDP and block aggregation (minutes)
for app in ("bfs", "sssp"):
    bench, wl = load(app, spec)
    ref = [run_reference(bench, wl) for _ in range(3)]
    print(f"{app} {spec} no-cdp: {statistics.median(r.ns_device for r in ref)/1e6:.3f} ms"
          f" iterations={ref[0].iterations}", flush=True)
    for d in (([] if fast else [dict(), dict(agg="block")]) + [dict(agg="grid"),
              dict(threshold=INF_THRESHOLD),
              dict(threshold=INF_THRESHOLD, parent_block=256, serial="warp"),
              dict(threshold=8, agg="grid", parent_block=256, serial="warp"),
              dict(threshold=INF_THRESHOLD, parent_block=256, serial="warp",
                   device_loop=True),
              dict(threshold=8, agg="block", parent_block=256, serial="warp",
                   device_loop=True)]):
        reps = [run_config(bench, wl, BenchConfig(**d))[0] for _ in range(3)]
        assert reps[0].memory_digest == ref[0].memory_digest
        print(f"  {statistics.median(r.ns_device for r in reps)/1e6:9.3f} ms"
              f" launches={reps[0].num_launches:9d}"
              f" lat={reps[0].launch_lat_ns/1e3:9.1f}us {d}", flush=True)
