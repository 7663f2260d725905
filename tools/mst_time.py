import time, numpy as np, sys
sys.path.insert(0, '.')
from paper_2201_02789_b200.bench import load, run_config, run_reference, BenchConfig, INF_THRESHOLD
from oracle import oracle
for spec in sys.argv[1:] or ["rmat:22:seed1"]:
    t=time.time(); bench, wl = load("mstf", spec); print(spec, "prep s", round(time.time()-t,1), "m", wl.buffers["col"].shape[0], flush=True)
    b=wl.buffers
    t=time.time(); want=oracle.mst(b["rowptr"], b["col"], b["weight"], b["eid"]); print("oracle s", round(time.time()-t,1), want[1:], flush=True)
    for name in ("mstf","mstv"):
        bench, _ = load(name, "hand")
        for pol in [dict(threshold=INF_THRESHOLD, serial="warp"), dict(), dict(agg="block"), dict(agg="grid"), dict(threshold=128, agg="block", serial="warp"),
                    dict(threshold=1024, cfactor=16, agg="multiblock", group_size=1<<20, parent_block=256, child_block=128, serial="warp"),
                    dict(threshold=256, cfactor=8, agg="grid", parent_block=256, child_block=128, serial="warp")]:
            try:
                for rep_i in range(2):
                    rep,_ = run_config(bench, wl, BenchConfig(**pol))
                ok = np.array_equal(rep.arrays["in_mst"], want[0]) and rep.arrays["weight"].tolist()==[want[1],want[2]]
                print(name, pol, "ms %.3f"%(rep.ns_device/1e6) if hasattr(rep,'ns_device') else rep.makespan, "rounds", rep.iterations, "launches", rep.num_launches, "ok", ok, flush=True)
            except Exception as e:
                print(name, pol, "ERR", e, flush=True)
    rep = run_reference(bench, wl); print("nocdp", rep.makespan, rep.iterations, flush=True)
