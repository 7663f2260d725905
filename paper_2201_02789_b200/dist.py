"""Multi-GPU execution of the partitioned workloads.

One process per GPU, ``torch.distributed`` for the plumbing (``nccl`` on the
GPUs, ``gloo`` in the CPU tests).  The data path has no collective: each rank
runs the nested-parallel kernels on its own shard and ONE reduction combines
the per-rank results.

  tc   oriented-edge ranges of the CSR+ balanced by the per-edge work
       d+(u) + d+(v) (the merge lengths); CSR+ replicated on every rank;
       all_reduce(sum) of the uint64 triangle count.
  bt   curve ranges of equal size (curves are i.i.d., so vertex counts
       balance statistically); all_reduce(sum) of (vertex count, fp64
       coordinate checksum).

The reference is single-process (no collective code); these
are the BASELINE.json multi-GPU configurations.
"""

from __future__ import annotations

import ctypes
from typing import Callable

import numpy as np


# ---------------------------------------------------------------------------
# partitioning (pure host logic)
# ---------------------------------------------------------------------------

def tc_edge_cost(rowptr: np.ndarray, col: np.ndarray) -> np.ndarray:
    """Work of each oriented edge (u, v): d+(u) + d+(v) list elements."""
    deg = np.diff(rowptr.astype(np.int64))
    src = np.repeat(np.arange(deg.shape[0]), deg)
    return deg[src] + deg[col.astype(np.int64)]


def balanced_ranges(cost: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Contiguous [lo, hi) ranges over len(cost) items with near-equal total
    cost (prefix-sum cut points)."""
    n = int(cost.shape[0])
    if parts < 1:
        raise ValueError("parts must be >= 1")
    if n == 0:
        return [(0, 0)] * parts
    pref = np.cumsum(cost.astype(np.float64))
    targets = pref[-1] * np.arange(1, parts) / parts
    cuts = np.searchsorted(pref, targets, side="left") + 1
    cuts = np.clip(cuts, 0, n)
    bounds = np.concatenate(([0], np.maximum.accumulate(cuts), [n]))
    return [(int(bounds[i]), int(bounds[i + 1])) for i in range(parts)]


def even_ranges(n: int, parts: int) -> list[tuple[int, int]]:
    b = np.linspace(0, n, parts + 1).round().astype(np.int64)
    return [(int(b[i]), int(b[i + 1])) for i in range(parts)]


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------

def _group():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def allreduce_sum_i64(values: list[int], device) -> list[int]:
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(x) for x in t.tolist()]


def allreduce_sum_f64(values: list[float], device) -> list[float]:
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


# ---------------------------------------------------------------------------
# triangle counting
# ---------------------------------------------------------------------------

def tc_count_sharded(rowptr: np.ndarray, col: np.ndarray,
                     count_range: Callable[[int, int], int],
                     device="cpu") -> tuple[int, tuple[int, int]]:
    """This rank's share of the oriented edges is counted by
    ``count_range(lo, hi)``; returns (global count, this rank's range)."""
    rank, world = _group()
    lo, hi = balanced_ranges(tc_edge_cost(rowptr, col), world)[rank]
    local = int(count_range(lo, hi))
    return allreduce_sum_i64([local], device)[0], (lo, hi)


def tc_device_counter(rowptr_d, col_d, n: int, m: int, cfg, stream=None):
    """count_range on the local GPU through the C-ABI (dp_tc_dev)."""
    import torch
    from . import _lib
    lib = _lib.device()
    tri = torch.zeros(1, dtype=torch.int64, device=rowptr_d.device)

    def count(lo: int, hi: int) -> int:
        st = _lib.DpStats()
        _lib.check(lib.dp_tc_dev(rowptr_d.data_ptr(), col_d.data_ptr(), n, m,
                                 lo, hi, ctypes.byref(cfg), tri.data_ptr(),
                                 stream, ctypes.byref(st)))
        count.stats = _lib.stats_dict(st)
        return int(tri.item())
    count.stats = None
    return count


# ---------------------------------------------------------------------------
# Bezier tessellation
# ---------------------------------------------------------------------------

def bt_sharded(ncurves: int,
               tessellate: Callable[[int, int], tuple[int, float]],
               device="cpu") -> tuple[int, float, tuple[int, int]]:
    """``tessellate(lo, hi)`` -> (vertex count, fp64 coordinate sum) of this
    rank's curves; returns the global (count, checksum) and the range."""
    rank, world = _group()
    lo, hi = even_ranges(ncurves, world)[rank]
    nv, cs = tessellate(lo, hi)
    nv_all = allreduce_sum_i64([int(nv)], device)[0]
    cs_all = allreduce_sum_f64([float(cs)], device)[0]
    return nv_all, cs_all, (lo, hi)


def bt_device_tessellator(cp_d, max_tess: int, scale: float, cfg,
                          stream=None):
    """tessellate on the local GPU through the C-ABI (dp_bt_dev)."""
    import torch
    from . import _lib
    lib = _lib.device()
    dev = cp_d.device

    def tess(lo: int, hi: int):
        k = hi - lo
        cap = k * max_tess
        ntess = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
        offs = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
        verts = torch.empty((max(cap, 1), 2), dtype=torch.float32, device=dev)
        used = ctypes.c_int64()
        st = _lib.DpStats()
        sub = cp_d[lo:hi].contiguous()
        _lib.check(lib.dp_bt_dev(sub.data_ptr(), k, max_tess, scale,
                                 ctypes.byref(cfg), ntess.data_ptr(),
                                 offs.data_ptr(), verts.data_ptr(), cap,
                                 ctypes.byref(used), stream,
                                 ctypes.byref(st)))
        tess.stats = _lib.stats_dict(st)
        v = verts[:used.value].double()
        return int(used.value), float(v.sum().item())
    tess.stats = None
    return tess
