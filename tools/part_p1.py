"""Partitioned SSSP / BFS at P=1 through the library solve drivers
(dp_*_part_solve_peer) vs the single-GPU path, same graph, device time
(CUDA events around the call).  For A/B builds: DYNPAR_LIB=... python
tools/part_p1.py [scale]"""
import ctypes
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2201_02789_b200 import dist as pdist  # noqa: E402


def timed(fn, k=8):
    ts = []
    for i in range(k + 2):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    G = bench.DeviceGraph(scale, 1, weights=True)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    out = {}
    for kind in ("sssp", "bfs"):
        cfg = bench._cfg(bench.BEST[kind])
        single = timed(lambda: bench.run_dev(kind, G, cfg, s))
        ex = pdist.PeerLocal()
        buf = ex.alloc(G.n, 1, dev)
        if kind == "sssp":
            part = pdist.SsspPeerPart(G.g.rowptr, G.g.col, G.w, G.n, 1, 0, 0,
                                      buf, dev)
            ex.bind([part])
            fn = lambda: pdist.sssp_1d_peer_solve([part], cfg, ex,  # noqa
                                                  gather=False)
        else:
            part = pdist.BfsPart(G.g.rowptr, G.g.col, G.n, 1, 0, 0, dev,
                                 dist=buf, spread=True)
            ex.bind([part])
            fn = lambda: pdist.bfs_1d_peer_solve([part], cfg, ex,  # noqa
                                                 gather=False)
        part_ms = timed(fn)
        st = part.stats[-1]
        out[kind] = {"single_ms": single, "partitioned_p1_ms": part_ms,
                     "ratio": part_ms / single,
                     "kernel_sum_ms": st["ns_kernel_sum"] / 1e6,
                     "rounds": st["iterations"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
