"""Per-call breakdown of one headline step: torch-event step time vs the
library's device time, kernel time and host wall time."""
import ctypes, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import BEST, DeviceGraph, _cfg, run_dev
torch.cuda.set_device(0)
G = DeviceGraph(22, 1, weights=True)
so = torch.cuda.current_stream()
stream = ctypes.c_void_p(so.cuda_stream)
cfg = _cfg(BEST["sssp"])
for i in range(8):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(so)
    st = run_dev("sssp", G, cfg, stream)
    e1.record(so)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"event {e0.elapsed_time(e1):.3f} ms  wall {1e3*(t1-t0):.3f}  lib.host {st['ns_host']/1e6:.3f}  lib.dev {st['ns_device']/1e6:.3f}  kern {st['ns_kernel_sum']/1e6:.3f}  rounds {st['iterations']}")
