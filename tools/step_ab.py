"""Back-to-back timed steps with / without the nvidia-smi sampler."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import BEST, ClockSampler, DeviceGraph, _cfg, run_dev, timed_steps
torch.cuda.set_device(0)
G = DeviceGraph(22, 1, weights=True)
so = torch.cuda.current_stream()
stream = ctypes.c_void_p(so.cuda_stream)
cfg = _cfg(BEST["sssp"])
for label in ("plain", "sampler", "plain", "sampler"):
    if label == "sampler":
        with ClockSampler(0):
            ms, st = timed_steps(lambda: run_dev("sssp", G, cfg, stream), 20, 3, so)
    else:
        ms, st = timed_steps(lambda: run_dev("sssp", G, cfg, stream), 20, 3, so)
    dev = sum(s["ns_device"] for s in st) / 1e6 / 20
    host = sum(s["ns_host"] for s in st) / 1e6 / 20
    print(f"{label:8s} step {ms/20:.3f} ms  lib.dev {dev:.3f}  lib.host {host:.3f}")
