"""Multi-process check of the fused exchange, one rank per GPU: torch
symmetric memory rendezvous, remote atomicMin / CAS into the other ranks'
dist over NVLink, flag reduction over NCCL; SSSP and BFS on RMAT-16 against
the oracle.

    torchrun --nproc-per-node N tools/peer2proc.py      (N GPUs)
Prints PASS / FAIL per workload on rank 0.  (Symmetric memory refuses two
ranks on one device, so this needs N GPUs; in-round gpurun has one.)"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2201_02789_b200 import dist as pdist  # noqa: E402
from paper_2201_02789_b200.bench import BenchConfig, graphs  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, world = dist.get_rank(), dist.get_world_size()
g = graphs.rmat_graph(16, 1)
w = graphs.edge_weights(g, 1)
cfg = BenchConfig(threshold=128, cfactor=4, agg="multiblock",
                  group_size=1 << 20, parent_block=128, child_block=128,
                  serial="warp").to_c()
ok = True
# SSSP
ex = pdist.PeerCollective()
buf = ex.alloc(g.n, world, dev)
part = pdist.SsspPeerPart(*pdist.partition_csr(g.rowptr, g.col, world, rank,
                                               w),
                          g.n, world, rank, 0, buf, dev)
ex.bind([part])
d, rounds = pdist.sssp_1d_peer([part], pdist.DeviceSsspPeerOps(cfg), ex)
want, _ = oracle.sssp(g.rowptr, g.col, w, nthreads=0)
res = np.array_equal(d.cpu().numpy(), want)
ok &= res
if rank == 0:
    print("sssp", "PASS" if res else "FAIL", "rounds", rounds, flush=True)
# BFS
ex2 = pdist.PeerCollective()
buf2 = ex2.alloc(g.n, world, dev)
bpart = pdist.BfsPart(*pdist.rmat_part(16, 1, world, rank), g.n, world, rank,
                      0, dev, dist=buf2)
ex2.bind([bpart])
d2, c2, lv = pdist.bfs_1d_peer([bpart], pdist.DeviceBfsOps(cfg), ex2)
wd, wc, wl = oracle.bfs(g.rowptr, g.col, nthreads=0)
res = (np.array_equal(d2.cpu().numpy(), wd)
       and np.array_equal(c2.cpu().numpy(), wc) and lv == wl)
ok &= res
if rank == 0:
    print("bfs", "PASS" if res else "FAIL", "levels", lv, flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
