"""The paper's granularity preference on B200: device time of
the tuned T + C with each aggregation granularity (none / warp / block /
multiblock with one group / grid), per application."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import BEST  # noqa: E402
from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa
from paper_2201_02789_b200.bench.benchmarks import (MST_OTHER_POLICY,  # noqa
                                                    Workload)

APPS = (("sssp", "rmat:22:seed1", "sssp"), ("bfs", "rmat:22:seed1", "bfs"),
        ("tc", "rmat:22:seed1", "tc"), ("bt", "curves:25000:seed1", "bt"),
        ("mstf", "rmat:22:seed1", "mstf"), ("mstv", "rmat:22:seed1", "mstf"),
        ("sp", "ksat5:200000:seed1", "sp"))
PAPER = {"sp": "grid", "tc": "grid", "bfs": "multiblock", "sssp": "multiblock",
         "bt": "block", "mstf": "block", "mstv": "none"}
for name, spec, pol_of in APPS:
    bench, wl = load(name, spec)
    if name == "sp":
        wl = Workload(wl.spec, dict(wl.buffers, max_sweeps=20, eps=0.0),
                      wl.n, wl.payload)
    best = dict(BEST[pol_of] if name != "mstv" else MST_OTHER_POLICY)
    row = {}
    for agg in (None, "warp", "block", "multiblock", "grid"):
        pol = dict(best, agg=agg, group_size=1 << 20)
        try:
            row[agg or "none"] = min(
                run_config(bench, wl, BenchConfig(**pol))[0].ns_device
                for _ in range(3)) / 1e6
        except Exception as e:  # noqa: BLE001
            row[agg or "none"] = float("nan")
            print(name, agg, "ERROR", e, flush=True)
    winner = min(row, key=lambda k: row[k] if row[k] == row[k] else 1e30)
    print(f"{name:5s} " + " ".join(f"{k}={v:.3f}" for k, v in row.items())
          + f"  best={winner} paper={PAPER[name]}", flush=True)
