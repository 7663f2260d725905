"""A/B the context's L2 fetch granularity (cudaLimitMaxL2FetchGranularity,
0-128 B) on the gather-heavy rows: SP 5-SAT (random fp64 eta gathers),
SSSP / BFS RMAT-22 (random dist probes), MST RMAT-22.
    python tools/ab_l2fetch.py [values...]      (default: 32 64 128)
Values alternate, 5 runs each; medians printed; outputs checked each run."""
import ctypes
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

from bench import BEST, DeviceGraph, _cfg, run_dev  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa

vals = [int(v) for v in sys.argv[1:]] or [32, 64, 128]
LIM = rt.cudaLimit.cudaLimitMaxL2FetchGranularity


def set_gran(v):
    torch.cuda.synchronize()
    err, = rt.cudaDeviceSetLimit(LIM, v)
    assert err == rt.cudaError_t.cudaSuccess, err
    err, got = rt.cudaDeviceGetLimit(LIM)
    return got


torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
err, dflt = rt.cudaDeviceGetLimit(LIM)
print("default L2 fetch granularity:", dflt, flush=True)
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

rows = []
G = DeviceGraph(22, 1, weights=True)
want_s, _ = oracle.sssp(G.g.rowptr, G.g.col, G.w, nthreads=0)
want_b, want_c, _ = oracle.bfs(G.g.rowptr, G.g.col, nthreads=0)


def sssp():
    st = run_dev("sssp", G, _cfg(BEST["sssp"]), stream)
    assert np.array_equal(G.dist.cpu().numpy(), want_s)
    return st["ns_device"] / 1e6


def bfs():
    st = run_dev("bfs", G, _cfg(BEST["bfs"]), stream)
    assert np.array_equal(G.dist.cpu().numpy(), want_b)
    return st["ns_device"] / 1e6


rows += [("sssp rmat-22", sssp), ("bfs rmat-22", bfs)]
sp_b, sp_wl = load("sp", "ksat5:200000:seed1")


def sp():
    rep, _ = run_config(sp_b, sp_wl, BenchConfig(**BEST["sp"]))
    return rep.ns_device / 1e6


mst_b, mst_wl = load("mstf", "rmat:22:seed1")


def mst():
    rep, _ = run_config(mst_b, mst_wl, BenchConfig(**BEST["mstf"]))
    return rep.ns_device / 1e6


rows += [("sp ksat5:200000 (20 sweeps)", sp), ("mst rmat-22", mst)]
for name, fn in rows:
    res = {v: [] for v in vals}
    fn()
    for _ in range(5):
        for v in vals:
            set_gran(v)
            res[v].append(fn())
    print(name, {v: round(statistics.median(t), 4) for v, t in res.items()},
          flush=True)
set_gran(dflt)
