"""BFS on RMAT-`scale` through the single-GPU path (BfsApp, dp_bfs_dev) and
through the 1D-partitioned solve at P = 1 (BfsPartApp,
dp_bfs_part_solve_peer): device time and per-level step times of each, to
size what the partitioned kernels cost over the single-GPU ones.

    python tools/bfs26_compare.py [scale]
"""
import ctypes
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2201_02789_b200 import _lib  # noqa: E402
from paper_2201_02789_b200 import dist as pdist  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    cfg = bench._cfg(bench.BEST["bfs"])
    # partitioned P = 1 (device-generated graph, as bench --workload bfs26)
    rp, col = pdist.rmat_part_device(scale, bench.SEED, 1, 0, dev)
    ex = pdist.PeerLocal()
    part = pdist.BfsPart(rp, col, 1 << scale, 1, 0, 0, dev,
                         dist=ex.alloc(1 << scale, 1, dev), spread=True)
    ex.bind([part])
    ts, steps = [], []
    for _ in range(4):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        pdist.bfs_1d_peer_solve([part], cfg, ex, gather=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        steps.append(_lib.step_times())
    print(json.dumps({"path": "partitioned P=1", "ms": statistics.median(ts[1:]),
                      "step_ms": [round(x, 3) for x in steps[-1]]}), flush=True)
    # single-GPU path on the same device graph
    n = 1 << scale

    class G:
        pass
    g = G()
    g.rowptr, g.col, g.n, g.m = part.rowptr, part.col, n, int(part.col.numel())
    g.dist = torch.empty(n, dtype=torch.int32, device=dev)
    g.counts = torch.empty(n, dtype=torch.int32, device=dev)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ts, steps = [], []
    for _ in range(4):
        st = bench.run_dev("bfs", g, cfg, s)
        ts.append(st["ns_device"] / 1e6)
        steps.append(_lib.step_times())
    same = bool(torch.equal(g.dist, part.dist[:n]))
    print(json.dumps({"path": "single-GPU BfsApp", "ms": statistics.median(ts[1:]),
                      "step_ms": [round(x, 3) for x in steps[-1]],
                      "dist_equal": same}), flush=True)


if __name__ == "__main__":
    main()
