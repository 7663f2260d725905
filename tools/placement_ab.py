"""Does allocation order (library workspace before/after the graph) change
the device time of the same SSSP step?"""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import BEST, DeviceGraph, _cfg, run_dev, timed_steps
from paper_2201_02789_b200 import _lib
order = sys.argv[1]
torch.cuda.set_device(0)
if order == "lib-first":
    _lib.device()
G = DeviceGraph(22, 1, weights=True)
so = torch.cuda.current_stream()
stream = ctypes.c_void_p(so.cuda_stream)
cfg = _cfg(BEST["sssp"])
for _ in range(2):
    ms, st = timed_steps(lambda: run_dev("sssp", G, cfg, stream), 20, 3, so)
    dev = sum(s["ns_device"] for s in st) / 1e6 / 20
    print(f"{order:10s} step {ms/20:.3f} ms  lib.dev {dev:.3f}")
