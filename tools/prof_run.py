"""One device-resident run of an app under a policy, for ncu captures.

    python tools/prof_run.py sssp 22 '{"threshold":512,...}' [runs]
"""
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import DeviceGraph, _cfg, run_dev  # noqa: E402

kind, scale = sys.argv[1], int(sys.argv[2])
policy = json.loads(sys.argv[3])
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 2
torch.cuda.set_device(0)
G = DeviceGraph(scale, 1, weights=(kind == "sssp"))
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(runs):
    st = run_dev(kind, G, _cfg(policy), stream)
print(json.dumps({k: st[k] for k in ("iterations", "num_launches",
                                     "host_launches", "blocks_scheduled",
                                     "ns_device", "ns_kernel_sum")}))
