"""Focused re-tune of the BFS / SSSP policy on RMAT-`scale` with the round-2
mechanisms (cf_wave, launch-free levels): T x C x parent / child block,
one-group multiblock, warp serial arm.  Device ms (median of 5).

    python tools/tune_graph.py bfs|sssp [scale]
"""
import ctypes
import itertools
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    kind = sys.argv[1]
    scale = int(sys.argv[2]) if len(sys.argv) > 2 else 22
    torch.cuda.set_device(0)
    G = bench.DeviceGraph(scale, 1, weights=(kind == "sssp"))
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    res = []
    for T, C, pb, cb, wave in itertools.product(
            (512, 1024, 2048), (8, 16, 32), (128, 256), (128, 256),
            (0, 592)):
        pol = dict(threshold=T, cfactor=C, agg="multiblock",
                   group_size=1 << 20, parent_block=pb, child_block=cb,
                   serial="warp", cf_wave=wave)
        ts = [bench.run_dev(kind, G, bench._cfg(pol), s)["ns_device"] / 1e6
              for _ in range(6)]
        ms = statistics.median(ts[1:])
        res.append((ms, pol))
        print(json.dumps({"ms": round(ms, 4), "policy": pol}), flush=True)
    res.sort(key=lambda r: r[0])
    print("BEST", json.dumps({"ms": res[0][0], "policy": res[0][1]}))


if __name__ == "__main__":
    main()
