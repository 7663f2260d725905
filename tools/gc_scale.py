"""GC rounds and time vs scale (good policies only; naive CDP is excluded:
every uncoloured vertex would launch twice per round)."""
import statistics, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2201_02789_b200.bench import BenchConfig, load, run_config, run_reference
for sc in [int(x) for x in sys.argv[1:]]:
    t0 = time.time(); bench, wl = load("gc", f"rmat:{sc}:seed1"); tl = time.time() - t0
    for d in (dict(threshold=64, agg="grid", parent_block=256, child_block=128, serial="warp"),
              dict(threshold=256, cfactor=8, agg="multiblock", group_size=1 << 20,
                   parent_block=256, child_block=128, serial="warp")):
        reps = [run_config(bench, wl, BenchConfig(**d))[0] for _ in range(2)]
        r = reps[-1]
        print(f"scale {sc} load {tl:.1f}s  {r.ns_device/1e6:9.2f} ms rounds={r.iterations} colors={int(r.arrays['color'].max())+1} launches={r.num_launches} {d}", flush=True)
    ref = run_reference(bench, wl)
    print(f"scale {sc} no-cdp {ref.ns_device/1e6:9.2f} ms", flush=True)
