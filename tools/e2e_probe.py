"""Where the host-buffer SSSP call spends its time: copy alone vs dp_sssp
(pipelined chunks of 2^shift slots) for a few chunk sizes and policies."""
import ctypes
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import BEST, FRONTIER_POLICY, _cfg  # noqa: E402
from paper_2201_02789_b200 import _lib  # noqa: E402
from paper_2201_02789_b200.bench import graphs  # noqa: E402

lib = _lib.device()
g = graphs.rmat_graph(22, 1)
w = graphs.edge_weights(g, 1)
rp = torch.from_numpy(g.rowptr).pin_memory()
col = torch.from_numpy(g.col).pin_memory()
wt = torch.from_numpy(w).pin_memory()
dist = torch.empty(g.n, dtype=torch.int32).pin_memory()
dcol = torch.empty_like(col, device="cuda")
dwt = torch.empty_like(wt, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dcol.copy_(col, non_blocking=True)
    dwt.copy_(wt, non_blocking=True)
    torch.cuda.synchronize()
print("copy col+weight alone ms %.3f" % ((time.perf_counter() - t0) * 1e3))
for name, pol in (("best", BEST["sssp"]), ("frontier", FRONTIER_POLICY)):
    for shift in ("21", "22", "23", "24", "25", "30"):
        os.environ["DP_COPY_CHUNK_SHIFT"] = shift
        cfg = _cfg(pol)
        st = _lib.DpStats()
        ts = []
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.check(lib.dp_sssp(rp.data_ptr(), col.data_ptr(), wt.data_ptr(),
                                   g.n, g.m, 0, ctypes.byref(cfg),
                                   dist.data_ptr(), ctypes.byref(st)))
            ts.append((time.perf_counter() - t0) * 1e3)
        print(name, "shift", shift, "host ms", ["%.2f" % t for t in ts[1:]],
              "rounds", st.iterations, "device ms %.2f" % (st.ns_device / 1e6),
              "kernel sum ms %.2f" % (st.ns_kernel_sum / 1e6), flush=True)
