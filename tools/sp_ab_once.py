import sys, statistics
sys.path.insert(0, '.')
from paper_2201_02789_b200.bench import BenchConfig, load, run_config
from bench import BEST
bench, wl = load("sp", "ksat5:200000:seed1")
ts = []
for _ in range(5):
    rep, _ = run_config(bench, wl, BenchConfig(**BEST["sp"]))
    ts.append(rep.ns_device / 1e6)
print("ms %.3f" % statistics.median(ts[1:]), "sweeps", rep.iterations)
