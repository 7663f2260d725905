import numpy as np, sys
sys.path.insert(0, '.')
from paper_2201_02789_b200.bench import load, run_config, run_reference, BenchConfig, INF_THRESHOLD
from oracle import oracle
pols = [dict(), dict(threshold=INF_THRESHOLD), dict(agg="warp"), dict(threshold=32, agg="block"),
        dict(threshold=64, cfactor=4, agg="multiblock", group_size=4, serial="warp"),
        dict(threshold=32, agg="grid", serial="warp")]
for spec in ["road:1000:seed7", "rmat:21:seed1", "rmat:22:seed1"]:
    bench, wl = load("mstf", spec); b = wl.buffers
    want = oracle.mst(b["rowptr"], b["col"], b["weight"], b["eid"])
    for name in ("mstf", "mstv"):
        bench, _ = load(name, "hand")
        for pol in pols:
            for rep_i in range(2):
                rep, _ = run_config(bench, wl, BenchConfig(**pol))
                got = rep.arrays["in_mst"]
                d = np.flatnonzero(got != want[0])
                print(spec, name, pol, rep_i, "wt", rep.arrays["weight"].tolist(), "want", want[1:], "ndiff", d.size, d[:5], got.sum(), want[0].sum(), flush=True)
    rep = run_reference(bench, wl)
    print("ref", rep.arrays["weight"].tolist(), flush=True)
