"""A/B compile-time variants of libdynpar on BFS and SSSP RMAT-22 (BEST
policies), one subprocess per (library, pass), passes interleaved.

    python tools/ab_libs.py lib1.so lib2.so ... [--kinds bfs,sssp] [--scale 22]
"""
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import ctypes, json, statistics, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from bench import BEST, DeviceGraph, _cfg, run_dev
from oracle import oracle
kinds, scale = sys.argv[2].split(','), int(sys.argv[3])
torch.cuda.set_device(0)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
G = DeviceGraph(scale, 1, weights=True)
out = {}
import os
extra = json.loads(os.environ.get("AB_POLICY", "{}"))
for kind in kinds:
    cfg = _cfg(dict(BEST[kind], **extra))
    ts = []
    for _ in range(8):
        st = run_dev(kind, G, cfg, s)
        ts.append(st['ns_device'] / 1e6)
    d = G.dist.cpu().numpy()
    if kind == 'bfs':
        wd, wc, lv = oracle.bfs(G.g.rowptr, G.g.col, nthreads=0)
        ok = bool(np.array_equal(d, wd))
        okc = bool(np.array_equal(G.counts.cpu().numpy(), wc))
        out[kind] = dict(ms=statistics.median(ts[2:]), it=st['iterations'],
                         dist_ok=ok, counts_ok=okc, host_launches=st['host_launches'],
                         oracle_levels=lv)
    else:
        wd, rounds = oracle.sssp(G.g.rowptr, G.g.col, G.w, nthreads=0)
        out[kind] = dict(ms=statistics.median(ts[2:]), it=st['iterations'],
                         dist_ok=bool(np.array_equal(d, wd)))
print('RESULT', json.dumps(out))
"""


def main():
    args = sys.argv[1:]
    kinds, scale = "bfs,sssp", "22"
    libs = []
    i = 0
    while i < len(args):
        if args[i] == "--kinds":
            kinds = args[i + 1]
            i += 2
        elif args[i] == "--scale":
            scale = args[i + 1]
            i += 2
        else:
            libs.append(args[i])
            i += 1
    res = {lib: [] for lib in libs}
    for _ in range(2):
        for lib in libs:
            env = dict(os.environ, DYNPAR_LIB=str(Path(lib).resolve()),
                       DYNPAR_LIB_PARTIAL="1")
            p = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), kinds,
                                scale], env=env, capture_output=True, text=True,
                               timeout=600)
            line = [x for x in p.stdout.splitlines() if x.startswith("RESULT")]
            if not line:
                print(lib, "FAILED", p.stderr[-2000:], flush=True)
                continue
            r = json.loads(line[0][7:])
            res[lib].append(r)
            print(Path(lib).name, json.dumps(r), flush=True)
    print("== summary (median over passes of per-pass medians, ms)")
    for lib, rs in res.items():
        summ = {k: round(statistics.median(r[k]["ms"] for r in rs), 4)
                for k in (rs[0] if rs else {})}
        print(Path(lib).name, summ, flush=True)


if __name__ == "__main__":
    main()
