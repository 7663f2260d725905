"""Lazy launcher count + no epilogue readback vs the synchronous count
(DYNPAR_SYNC_COUNT=1), and rounds queued one ahead (SSSP; DYNPAR_NO_SPEC=1
turns them off): back-to-back timed steps as bench.py times them,
SSSP and BFS RMAT-22 with the bench policies; outputs compared."""
import ctypes
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from bench import BEST, DeviceGraph, _cfg, run_dev, timed_steps  # noqa: E402
torch.cuda.set_device(0)
G = DeviceGraph(22, 1, weights=True)
so = torch.cuda.current_stream()
stream = ctypes.c_void_p(so.cuda_stream)
ref = {}
for kind in ("sssp", "bfs"):
    cfg = _cfg(BEST[kind])
    for label in ("sync", "lazy", "spec") * 3:
        for var, on in (("DYNPAR_SYNC_COUNT", label == "sync"),
                        ("DYNPAR_NO_SPEC", label != "spec")):
            if on:
                os.environ[var] = "1"
            else:
                os.environ.pop(var, None)
        ms, st = timed_steps(lambda: run_dev(kind, G, cfg, stream), 20, 3, so)
        dev = sum(s["ns_device"] for s in st) / 1e6 / 20
        out = (G.dist.clone(), G.counts.clone() if kind == "bfs" else None)
        key = (kind,)
        if key not in ref:
            ref[key] = out
        same = torch.equal(ref[key][0], out[0]) and (
            kind == "sssp" or torch.equal(ref[key][1], out[1]))
        c = st[-1]
        print(f"{kind} {label:5s} step {ms / 20:.4f} ms  lib.dev {dev:.4f}  "
              f"it={c['iterations']} launches={c['num_launches']} "
              f"blocks={c['blocks_scheduled']} host={c['host_launches']} "
              f"kern={c['kernel_launches']} same={same}", flush=True)
