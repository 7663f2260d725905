"""A/B an environment toggle of libdynpar on the headline SSSP (and BFS):
    python tools/ab_env.py VAR v0 v1 [policy-json]
Alternates the two values, 5 runs each, prints medians and checks outputs."""
import ctypes
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import BEST, FRONTIER_POLICY, DeviceGraph, _cfg, run_dev  # noqa
from oracle import oracle  # noqa: E402

var, vals = sys.argv[1], sys.argv[2:4]
torch.cuda.set_device(0)
G = DeviceGraph(22, 1, weights=True)
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
want, _ = oracle.sssp(G.g.rowptr, G.g.col, G.w, nthreads=0)
for name, pol in (("sssp", BEST["sssp"]), ("frontier", FRONTIER_POLICY)):
    res = {v: [] for v in vals}
    for _ in range(5):
        for v in vals:
            os.environ[var] = v
            st = run_dev("sssp", G, _cfg(pol), stream)
            res[v].append(st["ns_device"] / 1e6)
            assert np.array_equal(G.dist.cpu().numpy(), want), (name, v)
    print(name, {v: round(statistics.median(t), 4) for v, t in res.items()},
          flush=True)
