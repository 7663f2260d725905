"""Where the partitioned SSSP step spends its time at P = 1 (PeerLocal):
reset, per-round kernel device time (dp_stats.ns_device), per-round wall
time of the host loop, against the single-GPU headline round.

    python tools/peer_round_probe.py [exchange=peer|a2a]"""
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import BEST, SCALE, SEED, _cfg  # noqa: E402
from paper_2201_02789_b200 import _lib  # noqa: E402
from paper_2201_02789_b200 import dist as pdist  # noqa: E402
from paper_2201_02789_b200.bench import graphs  # noqa: E402


def main():
    exchange = sys.argv[1] if len(sys.argv) > 1 else "peer"
    torch.cuda.set_device(0)
    _lib.device()
    dev = torch.device("cuda", 0)
    g = graphs.rmat_graph(SCALE, SEED)
    w = graphs.edge_weights(g, SEED)
    rp, col, wp = pdist.partition_csr(g.rowptr, g.col, 1, 0, w)
    collective = "RANK" in os.environ
    if collective:
        torch.distributed.init_process_group(
            "nccl", device_id=torch.device("cuda", 0))
    if exchange == "peer":
        ex = pdist.PeerCollective() if collective else pdist.PeerLocal()
        buf = ex.alloc(g.n, 1, dev)
        part = pdist.SsspPeerPart(rp, col, wp, g.n, 1, 0, 0, buf, dev)
        ex.bind([part])
        ops = pdist.DeviceSsspPeerOps(_cfg(BEST["sssp"]))
        run = pdist.sssp_1d_peer
    else:
        part = pdist.SsspPart(rp, col, wp, g.n, 1, 0, 0, dev)
        ops = pdist.DeviceSsspOps(_cfg(BEST["sssp"]))
        ex = pdist.CollectiveExchange() if collective else \
            pdist.LocalExchange()
        run = pdist.sssp_1d
    for _ in range(3):
        part.reset(0)
        run([part], ops, ex)
    walls, resets, kern = [], [], []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        part.reset(0)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        part.stats.clear()
        _, rounds = run([part], ops, ex)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        resets.append((t1 - t0) * 1e3)
        walls.append((t2 - t1) * 1e3)
        kern.append([s["ns_device"] / 1e6 for s in part.stats])
    # the per-round collective alone
    t = torch.zeros(1, dtype=torch.int32, device=dev)
    ar = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if collective:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        int(t.item())
        ar.append((time.perf_counter() - t0) * 1e6)
    print(f"flag all_reduce + item: {statistics.median(ar):.1f} us "
          f"(collective={collective})")
    print(f"{exchange}: rounds {rounds}  reset ms {statistics.median(resets):.3f}"
          f"  rounds wall ms {statistics.median(walls):.3f}")
    print("  per-round device ms", [round(x, 3) for x in kern[-1]],
          "sum", round(sum(kern[-1]), 3))
    print("  per-round stats", {k: part.stats[-1][k] for k in
                                ("num_launches", "host_launches",
                                 "kernel_launches", "ns_kernel_sum",
                                 "ns_host")})


if __name__ == "__main__":
    main()
