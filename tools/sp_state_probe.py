import sys, statistics; sys.path.insert(0, '.')
import torch
from cuda.bindings import runtime as rt
from paper_2201_02789_b200.bench import BenchConfig, load, run_config
from bench import BEST
torch.cuda.set_device(0); torch.zeros(1, device="cuda")
b, wl = load("sp", "ksat5:200000:seed1")
def t():
    ts=[run_config(b, wl, BenchConfig(**BEST["sp"]))[0].ns_device/1e6 for _ in range(4)]
    return round(statistics.median(ts[1:]),3)
print("fresh", t(), flush=True)
rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, 64)
print("after setlimit 64", t(), flush=True)
from bench import DeviceGraph, _cfg, run_dev
import ctypes
G = DeviceGraph(22, 1, weights=True)
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
run_dev("sssp", G, _cfg(BEST["sssp"]), stream)
print("after sssp", t(), flush=True)
run_dev("bfs", G, _cfg(BEST["bfs"]), stream)
print("after bfs", t(), flush=True)
del G; torch.cuda.empty_cache()
print("after free", t(), flush=True)
