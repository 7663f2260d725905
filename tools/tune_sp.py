"""Policy sweep for SP (fixed 20 sweeps): device ms per policy."""
import itertools
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2201_02789_b200.bench import (INF_THRESHOLD, BenchConfig,  # noqa
                                         load, run_config, run_reference)
from paper_2201_02789_b200.bench.benchmarks import Workload  # noqa: E402

for spec in sys.argv[1:] or ["ksat5:200000:seed1", "ksat3:1000000:seed1"]:
    bench, wl = load("sp", spec)
    wl = Workload(wl.spec, dict(wl.buffers, max_sweeps=20, eps=0.0), wl.n,
                  wl.payload)
    ref = [run_reference(bench, wl).ns_device / 1e6 for _ in range(2)][-1]
    print(spec, "nocdp ms %.2f" % ref, flush=True)
    rows = []
    for T, serial, agg, cf, cb, pb in itertools.product(
            (32, 128, INF_THRESHOLD), ("thread", "warp"),
            ("grid", "multiblock"), (1, 4), (64, 128), (128, 256)):
        if T == INF_THRESHOLD and (agg != "grid" or cf != 1 or cb != 64):
            continue
        pol = dict(threshold=T, serial=serial, agg=agg, cfactor=cf,
                   child_block=cb, parent_block=pb, group_size=1 << 20)
        ms = min(run_config(bench, wl, BenchConfig(**pol))[0].ns_device / 1e6
                 for _ in range(2))
        rows.append((ms, pol))
    rows.sort(key=lambda r: r[0])
    for ms, pol in rows[:8]:
        print("  %.2f ms" % ms, pol, flush=True)
