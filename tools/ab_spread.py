"""A/B the counts spread block (DYNPAR_SPREAD_BITS) on BFS RMAT-22
(dp_bfs_dev) and BFS RMAT-26 (1D partition, P=1, fused exchange), with
bit-exact checks at 22.

    python tools/ab_spread.py [bits ...]
"""
import ctypes
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD22 = r"""
import ctypes, statistics, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from bench import BEST, DeviceGraph, _cfg, run_dev
from oracle import oracle
torch.cuda.set_device(0)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
G = DeviceGraph(22, 1, weights=False)
ts = [run_dev('bfs', G, _cfg(BEST['bfs']), s)['ns_device'] / 1e6 for _ in range(9)]
wd, wc, _ = oracle.bfs(G.g.rowptr, G.g.col, nthreads=0)
ok = np.array_equal(G.dist.cpu().numpy(), wd) and np.array_equal(G.counts.cpu().numpy(), wc)
print('RESULT', statistics.median(ts[2:]), ok)
"""

CHILD26 = r"""
import statistics, sys, time
sys.path.insert(0, sys.argv[1])
import torch
from bench import BEST, _cfg
from paper_2201_02789_b200 import dist as pdist
torch.cuda.set_device(0)
dev = torch.device('cuda', 0)
scale = int(sys.argv[2])
rp, col = pdist.rmat_part_device(scale, 1, 1, 0, dev)
ex = pdist.PeerLocal()
part = pdist.BfsPart(rp, col, 1 << scale, 1, 0, 0, dev,
                     dist=ex.alloc(1 << scale, 1, dev), spread=True)
ex.bind([part])
ops = pdist.DeviceBfsOps(_cfg(BEST['bfs']))
ts = []
for _ in range(5):
    part.reset(0)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    d, c, lv = pdist.bfs_1d_peer([part], ops, ex)
    e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print('RESULT', statistics.median(ts[1:]), int(c.to(torch.int64).sum().item()))
"""


def run(code, bits, *extra):
    env = dict(os.environ, DYNPAR_SPREAD_BITS=str(bits))
    p = subprocess.run([sys.executable, "-c", code, str(ROOT), *extra],
                       env=env, capture_output=True, text=True, timeout=900)
    line = [x for x in p.stdout.splitlines() if x.startswith("RESULT")]
    return line[0][7:] if line else "FAILED " + p.stderr[-800:]


def main():
    bits = [int(b) for b in sys.argv[1:]] or [0, 8, 10, 12, 14, 16, 22]
    for rep in range(2):
        for b in bits:
            print(f"bits={b} rmat22 bfs ms, ok: {run(CHILD22, b)}", flush=True)
        for b in bits:
            print(f"bits={b} rmat26 part P=1 ms, edges: "
                  f"{run(CHILD26, b, '26')}", flush=True)


if __name__ == "__main__":
    main()
