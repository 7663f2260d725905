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
    """Work of each oriented edge (u, v) at slot e in the transposed counter
    (csrc/apps.cuh TcApp): the elements of N+(u) above v, slots (e,
    rowptr[u+1]), probed into v's set, plus one unit for the edge itself
    (set setup is amortised per block)."""
    rp = rowptr.astype(np.int64)
    deg = np.diff(rp)
    end = np.repeat(rp[1:], deg)
    return end - np.arange(end.shape[0], dtype=np.int64)


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

def tc_shard(rowptr: np.ndarray, col: np.ndarray) -> tuple[int, int]:
    """This rank's oriented-edge range (work-balanced)."""
    rank, world = _group()
    return balanced_ranges(tc_edge_cost(rowptr, col), world)[rank]


def tc_count_range(rng: tuple[int, int],
                   count_range: Callable[[int, int], int],
                   device="cpu") -> int:
    """Count this rank's range, all_reduce(sum) -> the global count."""
    local = int(count_range(*rng))
    return allreduce_sum_i64([local], device)[0]


def tc_count_sharded(rowptr: np.ndarray, col: np.ndarray,
                     count_range: Callable[[int, int], int],
                     device="cpu") -> tuple[int, tuple[int, int]]:
    """This rank's share of the oriented edges is counted by
    ``count_range(lo, hi)``; returns (global count, this rank's range)."""
    rng = tc_shard(rowptr, col)
    return tc_count_range(rng, count_range, device), rng


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


# ---------------------------------------------------------------------------
# BFS over a cyclic 1D vertex partition with a per-level frontier exchange
# (BASELINE.json config 5)
# ---------------------------------------------------------------------------
#
# owner(v) = v % P, local index v // P.  Per level every part expands its
# owned frontier through the T/C/A scheduler (dp_bfs_part_level): local
# targets are discovered in place, remote ones are sent once per part for the
# whole run (bitmap) into per-owner buckets; the buckets are exchanged with an
# all-to-all, owners apply them (dp_bfs_part_apply), and an all-reduce(max)
# of the per-part `changed` flags ends the loop.  Per-part dense `counts` are
# summed at the end.  Levels are synchronous, so dist is bit-identical to the
# single-GPU run for any P.

def spread_bits() -> int:
    """log2 of the counts spread block (dp_config.counts_spread): 12 (4096
    vertices, 16 KiB), or $DYNPAR_SPREAD_BITS for A/B runs."""
    import os
    return max(0, min(30, int(os.environ.get("DYNPAR_SPREAD_BITS", "12"))))


class BfsPart:
    """One part's device state (tensors on ``device``)."""

    def __init__(self, rowptr, col, n_global: int, nparts: int, part: int,
                 src: int, device, dist=None, spread: bool = False):
        """``dist``: optional [>= n_local] int32 buffer the other parts can
        address (the fused exchange, bfs_1d_peer); default a private one.
        ``spread``: accumulate ``counts`` in the spread layout (2^k slots,
        dp_config.counts_spread; device ops only), gathered back into vertex
        order by ``natural_counts``."""
        import torch
        self.nparts, self.part, self.n = nparts, part, n_global
        self.rowptr = torch.as_tensor(rowptr).to(device=device,
                                                  dtype=torch.int32)
        self.col = torch.as_tensor(col).to(device=device, dtype=torch.int32)
        self.n_local = int(self.rowptr.shape[0]) - 1
        i32 = dict(dtype=torch.int32, device=device)
        if dist is None:
            dist = torch.empty(self.n_local, **i32)
        if dist.numel() < self.n_local:
            raise ValueError("dist buffer narrower than the part")
        self.dist_full = dist
        self.dist = dist[:self.n_local]
        self.dist_full.fill_(1 << 30)
        if src % nparts == part:
            self.dist[src // nparts] = 0
        self.peer_ptrs = None  # fused exchange: device int64[nparts]
        self.counts_log2 = spread_bits() if spread else 0
        blk = 1 << self.counts_log2
        self.counts = torch.zeros(-(-n_global // blk) * blk, **i32)
        self.sent = torch.zeros((n_global + 31) // 32, **i32)
        # a part sends each remote vertex at most once: bucket q never holds
        # more than the vertices q owns
        self.stride = max(1, -(-n_global // nparts))
        self.send_buf = torch.empty(nparts * self.stride, **i32)
        self.send_counts = torch.zeros(nparts, **i32)
        self.changed = torch.zeros(1, **i32)
        self.stats: list[dict] = []

    def reset(self, src: int) -> None:
        """Fresh BFS state (keeps the graph and buffers)."""
        self.dist_full.fill_(1 << 30)
        if src % self.nparts == self.part:
            self.dist[src // self.nparts] = 0
        self.counts.zero_()
        self.sent.zero_()
        self.stats = []

    def bucket(self, q: int, count: int):
        return self.send_buf[q * self.stride:q * self.stride + count]

    def natural_counts(self, counts):
        """Summed counts (this part's layout) in vertex order."""
        if not self.counts_log2:
            return counts
        import torch
        from . import _lib
        out = torch.empty(self.n, dtype=torch.int32, device=counts.device)
        _lib.check(_lib.device().dp_unspread_dev(
            counts.data_ptr(), self.counts_log2, self.n, out.data_ptr(),
            None))
        return out


class DeviceBfsOps:
    """The per-part steps on the local GPU through the C-ABI."""

    def __init__(self, cfg, stream=None):
        from . import _lib
        self.cfg = cfg
        self.stream = stream
        self.lib = _lib.device()

    def _cfg(self, p: BfsPart):
        c = type(self.cfg).from_buffer_copy(self.cfg)
        c.counts_spread = p.counts_log2
        return c

    def level(self, p: BfsPart, level: int) -> None:
        from . import _lib
        p.send_counts.zero_()
        p.changed.zero_()
        st = _lib.DpStats()
        _lib.check(self.lib.dp_bfs_part_level(
            p.rowptr.data_ptr(), p.col.data_ptr(), p.n_local, p.nparts,
            p.part, level, ctypes.byref(self._cfg(p)), p.dist.data_ptr(),
            p.counts.data_ptr(), p.sent.data_ptr(), p.send_buf.data_ptr(),
            p.stride, p.send_counts.data_ptr(), p.changed.data_ptr(),
            self.stream, ctypes.byref(st)))
        p.stats.append(_lib.stats_dict(st))

    def apply(self, p: BfsPart, recv, level: int) -> None:
        from . import _lib
        if recv.numel():
            _lib.check(self.lib.dp_bfs_part_apply(
                recv.data_ptr(), recv.numel(), p.nparts, level,
                p.dist.data_ptr(), p.changed.data_ptr(), self.stream))

    def level_peer(self, p: BfsPart, level: int) -> None:
        """The level with the exchange fused in (remote CAS through
        p.peer_ptrs, dp_bfs_part_level_peer; the call clears the flag)."""
        from . import _lib
        st = _lib.DpStats()
        _lib.check(self.lib.dp_bfs_part_level_peer(
            p.rowptr.data_ptr(), p.col.data_ptr(), p.n_local, p.nparts,
            p.part, level, ctypes.byref(self._cfg(p)), p.dist.data_ptr(),
            p.peer_ptrs.data_ptr(), p.counts.data_ptr(), p.sent.data_ptr(),
            p.changed.data_ptr(), self.stream, ctypes.byref(st)))
        p.stats.append(_lib.stats_dict(st))


class LocalExchange:
    """All parts live in this process (one device): the exchange is a
    gather of buckets.  Used to run P > 1 partitions on a single GPU."""

    def send_counts(self, parts):
        return [p.send_counts.tolist() for p in parts]

    def all_to_all(self, parts):
        import torch
        cnt = self.send_counts(parts)
        return [torch.cat([src.bucket(q, cnt[i][q])
                           for i, src in enumerate(parts)])
                for q in range(len(parts))]

    def any_changed(self, parts) -> bool:
        return any(int(p.changed.item()) for p in parts)

    def counts(self, parts):
        out = parts[0].counts.clone()
        for p in parts[1:]:
            out += p.counts
        return out

    def dist(self, parts):
        import torch
        n, P = parts[0].n, parts[0].nparts
        out = torch.empty(n, dtype=torch.int32, device=parts[0].dist.device)
        for p in parts:
            out[p.part::P] = p.dist
        return out


class CollectiveExchange:
    """One part per rank; torch.distributed collectives (NCCL on the GPUs,
    gloo in the CPU tests)."""

    def all_to_all(self, parts):
        import torch
        import torch.distributed as dist
        (p,) = parts
        sc = p.send_counts.to(torch.int64)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc)
        send_splits = sc.tolist()
        recv_splits = rc.tolist()
        packed = torch.cat([p.bucket(q, c) for q, c in enumerate(send_splits)])
        recv = torch.empty(sum(recv_splits), dtype=p.send_buf.dtype,
                           device=p.send_buf.device)
        dist.all_to_all_single(recv, packed, recv_splits, send_splits)
        return [recv]

    def any_changed(self, parts) -> bool:
        import torch.distributed as dist
        (p,) = parts
        flag = p.changed.clone()
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        return bool(int(flag.item()))

    def counts(self, parts):
        import torch.distributed as dist
        (p,) = parts
        out = p.counts.clone()
        dist.all_reduce(out, op=dist.ReduceOp.SUM)
        return out

    def dist(self, parts):
        import torch
        import torch.distributed as dist
        (p,) = parts
        P = p.nparts
        width = -(-p.n // P)
        pad = torch.full((width,), 1 << 30, dtype=torch.int32,
                         device=p.dist.device)
        pad[:p.n_local] = p.dist
        allp = [torch.empty_like(pad) for _ in range(P)]
        dist.all_gather(allp, pad)
        out = torch.empty(p.n, dtype=torch.int32, device=p.dist.device)
        for q in range(P):
            nq = len(range(q, p.n, P))
            out[q::P] = allp[q][:nq]
        return out


def bfs_1d(parts: list, ops, exchange, max_levels: int | None = None):
    """Level-synchronous BFS over the given parts (all P parts for
    LocalExchange, this rank's part for CollectiveExchange).
    Returns (dist, counts, levels) as device tensors; levels counts the host
    iterations including the final no-change one (like the reference's
    host_launches, bench/benchmarks.py:157-168)."""
    n = parts[0].n
    limit = n + 1 if max_levels is None else max_levels
    for level in range(limit):
        for p in parts:
            ops.level(p, level)
        recv = exchange.all_to_all(parts)
        for p, r in zip(parts, recv):
            ops.apply(p, r, level)
        if not exchange.any_changed(parts):
            return (exchange.dist(parts),
                    parts[0].natural_counts(exchange.counts(parts)), level + 1)
    raise RuntimeError("bfs used more levels than vertices")


def rmat_part(scale: int, seed: int, nparts: int, part: int,
              edge_factor: int = 16):
    """Rows of RMAT(scale, seed) owned by `part` (native generator)."""
    from . import _lib
    lib = _lib.load()
    n = 1 << scale
    n_local = len(range(part, n, nparts))
    rowptr = np.empty(n_local + 1, dtype=np.int32)
    m = ctypes.c_int64()
    _lib.check(lib.dp_rmat_csr_part(scale, edge_factor, seed, nparts, part,
                                    _lib.ptr(rowptr), None, 0,
                                    ctypes.byref(m), 0))
    col = np.empty(max(m.value, 1), dtype=np.int32)
    _lib.check(lib.dp_rmat_csr_part(scale, edge_factor, seed, nparts, part,
                                    _lib.ptr(rowptr), _lib.ptr(col),
                                    col.shape[0], ctypes.byref(m), 0))
    return rowptr, col[:m.value]


def rmat_part_device(scale: int, seed: int, nparts: int, part: int, device,
                     edge_factor: int = 16, stream=None):
    """Same rows as rmat_part, generated on the GPU: keys (local src << 32
    | dst) from the device hash, sorted, split into (rowptr, col) tensors."""
    import torch
    from . import _lib
    lib = _lib.device()
    n = 1 << scale
    n_local = len(range(part, n, nparts))
    cnt = ctypes.c_int64()
    _lib.check(lib.dp_rmat_part_keys_dev(scale, edge_factor, seed, nparts,
                                         part, None, 0, ctypes.byref(cnt),
                                         stream))
    keys = torch.empty(max(cnt.value, 1), dtype=torch.int64, device=device)
    _lib.check(lib.dp_rmat_part_keys_dev(scale, edge_factor, seed, nparts,
                                         part, keys.data_ptr(), cnt.value,
                                         ctypes.byref(cnt), stream))
    keys = keys[:cnt.value]
    keys, _ = torch.sort(keys)
    col = (keys & 0xFFFFFFFF).to(torch.int32)
    deg = torch.bincount(keys >> 32, minlength=n_local)
    del keys
    rowptr = torch.zeros(n_local + 1, dtype=torch.int64, device=device)
    torch.cumsum(deg, 0, out=rowptr[1:])
    return rowptr.to(torch.int32), col


def partition_csr(rowptr: np.ndarray, col: np.ndarray, nparts: int,
                  part: int, weight: np.ndarray | None = None):
    """Rows of an in-memory CSR owned by `part` (owner(v) = v % nparts):
    (rowptr_p, col_p) or, with `weight`, (rowptr_p, col_p, weight_p)."""
    rp = rowptr.astype(np.int64)
    own = np.arange(part, rp.shape[0] - 1, nparts)
    deg = rp[own + 1] - rp[own]
    lrp = np.concatenate(([0], np.cumsum(deg))).astype(np.int32)
    idx = (np.repeat(rp[own], deg)
           + np.arange(int(deg.sum())) - np.repeat(lrp[:-1].astype(np.int64),
                                                   deg))
    if weight is None:
        return lrp, col[idx].astype(np.int32)
    return lrp, col[idx].astype(np.int32), weight[idx].astype(np.int32)


# ---------------------------------------------------------------------------
# SSSP over the same 1D partition (SURVEY §8(e) row SSSP): per round each part
# relaxes its reached vertices' edges (dp_sssp_part_round); remote
# relaxations that strictly improve the part's best-sent value go to the
# owner as packed (v << 32 | alt) pairs, owners apply them with atomicMin
# (dp_sssp_part_apply); rounds end when no part changed anything.  dist is
# the exact shortest-path vector, identical to the single-GPU run.
# ---------------------------------------------------------------------------

class SsspPart:
    """One part's device state for the partitioned SSSP."""

    def __init__(self, rowptr, col, weight, n_global: int, nparts: int,
                 part: int, src: int, device):
        import torch
        self.nparts, self.part, self.n = nparts, part, n_global
        self.rowptr = torch.as_tensor(rowptr).to(device=device,
                                                  dtype=torch.int32)
        self.col = torch.as_tensor(col).to(device=device, dtype=torch.int32)
        self.weight = torch.as_tensor(weight).to(device=device,
                                                  dtype=torch.int32)
        self.n_local = int(self.rowptr.shape[0]) - 1
        i32 = dict(dtype=torch.int32, device=device)
        self.dist = torch.empty(self.n_local, **i32)
        self.best = torch.empty(n_global, **i32)
        # bucket q holds at most this part's edges into owner q per round
        owners = torch.remainder(self.col.to(torch.int64), nparts)
        cap = torch.bincount(owners, minlength=nparts).cpu()
        cap[part] = 0
        self.cap = cap.tolist()
        off = np.concatenate(([0], np.cumsum(self.cap)[:-1]))
        self.off_list = [int(x) for x in off]
        self.send_off = torch.as_tensor(off, dtype=torch.int64, device=device)
        self.send_buf = torch.empty(max(1, int(sum(self.cap))),
                                    dtype=torch.int64, device=device)
        self.send_counts = torch.zeros(nparts, **i32)
        self.changed = torch.zeros(1, **i32)
        self.stats: list[dict] = []
        self.reset(src)

    def reset(self, src: int) -> None:
        self.dist.fill_(1 << 30)
        if src % self.nparts == self.part:
            self.dist[src // self.nparts] = 0
        self.best.fill_(1 << 30)
        self.stats = []

    def bucket(self, q: int, count: int):
        return self.send_buf[self.off_list[q]:self.off_list[q] + count]


class DeviceSsspOps:
    """The per-part SSSP steps on the local GPU through the C-ABI."""

    def __init__(self, cfg, stream=None):
        from . import _lib
        self.cfg = cfg
        self.stream = stream
        self.lib = _lib.device()

    def level(self, p: SsspPart, rnd: int) -> None:
        from . import _lib
        p.send_counts.zero_()
        p.changed.zero_()
        st = _lib.DpStats()
        _lib.check(self.lib.dp_sssp_part_round(
            p.rowptr.data_ptr(), p.col.data_ptr(), p.weight.data_ptr(),
            p.n_local, p.nparts, p.part, ctypes.byref(self.cfg),
            p.dist.data_ptr(), p.best.data_ptr(), p.send_buf.data_ptr(),
            p.send_off.data_ptr(), p.send_counts.data_ptr(),
            p.changed.data_ptr(), self.stream, ctypes.byref(st)))
        p.stats.append(_lib.stats_dict(st))

    def apply(self, p: SsspPart, recv, rnd: int) -> None:
        from . import _lib
        if recv.numel():
            _lib.check(self.lib.dp_sssp_part_apply(
                recv.data_ptr(), recv.numel(), p.nparts, p.dist.data_ptr(),
                p.changed.data_ptr(), self.stream))


def sssp_1d(parts: list, ops, exchange, max_rounds: int | None = None):
    """Bellman-Ford rounds over the given parts.  Returns (dist, rounds)."""
    n = parts[0].n
    limit = n + 1 if max_rounds is None else max_rounds
    for rnd in range(limit):
        for p in parts:
            ops.level(p, rnd)
        recv = exchange.all_to_all(parts)
        for p, r in zip(parts, recv):
            ops.apply(p, r, rnd)
        if not exchange.any_changed(parts):
            return exchange.dist(parts), rnd + 1
    raise RuntimeError("sssp used more rounds than vertices")


# ---------------------------------------------------------------------------
# SSSP over the same partition with the exchange fused into the relaxation
# (csrc/apps.cuh SsspPeerApp): every part's dist is addressable from every
# part — torch symmetric memory (peer-mapped over NVLink / NVSwitch) across
# ranks, plain allocations when all parts share one GPU — so a remote
# relaxation is an atomicMin into the owner's dist.  A round is one kernel
# per part plus the max-reduction of the changed flags; no all-to-all.
# ---------------------------------------------------------------------------

def dist_width(n: int, nparts: int) -> int:
    """Rows of the largest part (every part's dist is allocated this wide, as
    symmetric memory requires identical shapes)."""
    return -(-n // nparts)


class SsspPeerPart:
    """One part's device state for the fused-exchange partitioned SSSP.
    ``dist`` must be a [dist_width(n, nparts)] int32 tensor the other parts
    can address (see PeerLocal / PeerCollective)."""

    def __init__(self, rowptr, col, weight, n_global: int, nparts: int,
                 part: int, src: int, dist, device):
        import torch
        self.nparts, self.part, self.n = nparts, part, n_global
        self.rowptr = torch.as_tensor(rowptr).to(device=device,
                                                  dtype=torch.int32)
        self.col = torch.as_tensor(col).to(device=device, dtype=torch.int32)
        self.weight = torch.as_tensor(weight).to(device=device,
                                                  dtype=torch.int32)
        self.n_local = int(self.rowptr.shape[0]) - 1
        if dist.numel() < self.n_local:
            raise ValueError("dist buffer narrower than the part")
        self.dist_full = dist
        self.dist = dist[:self.n_local]
        i32 = dict(dtype=torch.int32, device=device)
        self.best = torch.empty(n_global, **i32)
        self.changed = torch.zeros(1, **i32)
        self.peer_ptrs = None  # device int64[nparts], set by the exchange
        self.stats: list[dict] = []
        self.reset(src)

    def reset(self, src: int) -> None:
        self.dist_full.fill_(1 << 30)
        if src % self.nparts == self.part:
            self.dist_full[src // self.nparts] = 0
        self.best.fill_(1 << 30)
        self.stats = []


class DeviceSsspPeerOps:
    """One fused round of a part on the local GPU through the C-ABI."""

    def __init__(self, cfg, stream=None):
        from . import _lib
        self.cfg = cfg
        self.stream = stream
        self.lib = _lib.device()

    def round(self, p: SsspPeerPart) -> None:
        from . import _lib
        st = _lib.DpStats()  # the call clears p.changed
        _lib.check(self.lib.dp_sssp_part_round_peer(
            p.rowptr.data_ptr(), p.col.data_ptr(), p.weight.data_ptr(),
            p.n_local, p.nparts, p.part, ctypes.byref(self.cfg),
            p.dist.data_ptr(), p.peer_ptrs.data_ptr(), p.best.data_ptr(),
            p.changed.data_ptr(),
            self.stream, ctypes.byref(st)))
        p.stats.append(_lib.stats_dict(st))


class PeerLocal:
    """All parts on one GPU: the pointer table is the parts' own dist
    buffers (plain device memory)."""

    @staticmethod
    def alloc(n: int, nparts: int, device):
        import torch
        return torch.empty(dist_width(n, nparts), dtype=torch.int32,
                           device=device)

    def bind(self, parts) -> None:
        import torch
        table = torch.tensor([p.dist_full.data_ptr() for p in parts],
                             dtype=torch.int64, device=parts[0].dist.device)
        for p in parts:
            p.peer_ptrs = table
        # the parts' round-flag signal slots (dp_*_part_solve_peer)
        dev = parts[0].dist.device
        self.sig = [torch.zeros(2 * len(parts), dtype=torch.int64, device=dev)
                    for _ in parts]
        self.sig_table = torch.tensor([t.data_ptr() for t in self.sig],
                                      dtype=torch.int64, device=dev)
        self.epoch = 0

    def next_epoch(self) -> int:
        self.epoch += 1
        return self.epoch

    def any_changed(self, parts) -> bool:
        return any(int(p.changed.item()) for p in parts)

    def dist(self, parts):
        import torch
        n, P = parts[0].n, parts[0].nparts
        out = torch.empty(n, dtype=torch.int32, device=parts[0].dist.device)
        for p in parts:
            out[p.part::P] = p.dist
        return out

    def counts(self, parts):
        return LocalExchange().counts(parts)


class PeerCollective:
    """One part per rank: dist lives in torch symmetric memory; the
    rendezvous maps every rank's buffer into every rank (NVLink peer
    addresses), the changed flags are max-reduced with NCCL."""

    def __init__(self):
        self.handle = None

    def alloc(self, n: int, nparts: int, device):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        try:  # older releases need the group enabled explicitly
            symm_mem.enable_symm_mem_for_group(dist.group.WORLD.group_name)
        except Exception:  # noqa: BLE001
            pass
        t = symm_mem.empty(dist_width(n, nparts), dtype=torch.int32,
                           device=device)
        self.handle = symm_mem.rendezvous(t, dist.group.WORLD)
        return t

    def bind(self, parts) -> None:
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        (p,) = parts
        p.peer_ptrs = torch.tensor(list(self.handle.buffer_ptrs),
                                   dtype=torch.int64, device=p.dist.device)
        # round-flag signal slots (dp_*_part_solve_peer), mapped like dist
        self.sig = symm_mem.empty(2 * p.nparts, dtype=torch.int64,
                                  device=p.dist.device)
        self.sig.zero_()
        self.sig_handle = symm_mem.rendezvous(self.sig, dist.group.WORLD)
        self.sig_table = torch.tensor(list(self.sig_handle.buffer_ptrs),
                                      dtype=torch.int64, device=p.dist.device)
        self.epoch = 0
        torch.cuda.synchronize()
        dist.barrier()  # every rank's slots are zero before any tag lands

    def next_epoch(self) -> int:
        self.epoch += 1  # the same sequence of calls on every rank
        return self.epoch

    def any_changed(self, parts) -> bool:
        import torch.distributed as dist
        (p,) = parts
        # in place: the next round's call clears the flag itself
        dist.all_reduce(p.changed, op=dist.ReduceOp.MAX)
        return bool(int(p.changed.item()))

    def dist(self, parts):
        return CollectiveExchange().dist(
            [_DistView(parts[0])])

    def counts(self, parts):
        return CollectiveExchange().counts(parts)


class _DistView:
    """Adapter exposing SsspPeerPart's fields to CollectiveExchange.dist."""

    def __init__(self, p):
        self.nparts, self.n, self.n_local, self.dist = (p.nparts, p.n,
                                                        p.n_local, p.dist)


def sssp_1d_peer(parts: list, ops, exchange, max_rounds: int | None = None):
    """Bellman-Ford rounds with the fused exchange.  Returns (dist, rounds):
    the same distances as sssp_1d (Bellman-Ford tolerates the remote
    lowerings landing while the owner's round runs)."""
    n = parts[0].n
    limit = n + 1 if max_rounds is None else max_rounds
    for rnd in range(limit):
        for p in parts:
            ops.round(p)
        if not exchange.any_changed(parts):
            return exchange.dist(parts), rnd + 1
    raise RuntimeError("sssp used more rounds than vertices")


def bfs_1d_peer(parts: list, ops, exchange, max_levels: int | None = None):
    """bfs_1d with the exchange fused into the level kernel: remote
    discoveries are CAS'd straight into the owner's dist (parts bound to a
    PeerLocal / PeerCollective pointer table); the only collective per level
    is the max of the changed flags.  Returns (dist, counts, levels)."""
    n = parts[0].n
    limit = n + 1 if max_levels is None else max_levels
    for level in range(limit):
        for p in parts:
            ops.level_peer(p, level)
        if not exchange.any_changed(parts):
            return (exchange.dist(parts),
                    parts[0].natural_counts(exchange.counts(parts)), level + 1)
    raise RuntimeError("bfs used more levels than vertices")


def run_parts(parts, fn, streams=None) -> None:
    """fn(part, stream) for every part: directly for one part, else one host
    thread per part, each on its own CUDA stream (the solve drivers block in
    their round loop until every part has finished the round, so parts that
    share a process must run concurrently).  Re-raises the first failure."""
    import threading
    import torch
    from . import _lib
    if len(parts) == 1:
        fn(parts[0], streams[0] if streams else None)
        return
    if streams is None:
        streams = [torch.cuda.Stream() for _ in parts]
    errs = [None] * len(parts)
    lib = _lib.device()
    torch.cuda.synchronize()  # part state written on the default stream

    def body(i):
        try:
            fn(parts[i], ctypes.c_void_p(streams[i].cuda_stream))
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errs[i] = e
        finally:
            lib.dp_thread_release()
    threads = [threading.Thread(target=body, args=(i,))
               for i in range(len(parts))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    torch.cuda.synchronize()
    for e in errs:
        if e is not None:
            raise e


def sssp_1d_peer_solve(parts: list, cfg, exchange, src: int = 0,
                       stream=None, gather: bool = True):
    """sssp_1d_peer with the round loop in the library
    (dp_sssp_part_solve_peer): per round one parent grid + one warp that ORs
    the parts' flags through the signal slots -- no host collective per
    round.  Returns (dist, rounds); dist is None when gather=False (each
    part keeps its owned distances in p.dist)."""
    from . import _lib
    lib = _lib.device()
    epoch = exchange.next_epoch()

    def one(p, s):
        st = _lib.DpStats()
        _lib.check(lib.dp_sssp_part_solve_peer(
            p.rowptr.data_ptr(), p.col.data_ptr(), p.weight.data_ptr(),
            p.n_local, p.n, p.nparts, p.part, src, ctypes.byref(cfg),
            p.dist.data_ptr(), p.peer_ptrs.data_ptr(), p.best.data_ptr(),
            exchange.sig_table.data_ptr(), epoch, s, ctypes.byref(st)))
        p.stats.append(_lib.stats_dict(st))
    run_parts(parts, one, [stream] if stream is not None and
              len(parts) == 1 else None)
    rounds = {int(p.stats[-1]["iterations"]) for p in parts}
    if len(rounds) != 1:
        raise RuntimeError(f"parts disagree on the round count: {rounds}")
    return (exchange.dist(parts) if gather else None), rounds.pop()


def bfs_1d_peer_solve(parts: list, cfg, exchange, src: int = 0,
                      stream=None, gather: bool = True):
    """bfs_1d_peer with the level loop in the library
    (dp_bfs_part_solve_peer).  Returns (dist, counts, levels); dist and
    counts are None when gather=False (p.dist, p.counts hold the parts')."""
    from . import _lib
    lib = _lib.device()
    epoch = exchange.next_epoch()

    def one(p, s):
        c = type(cfg).from_buffer_copy(cfg)
        c.counts_spread = p.counts_log2
        st = _lib.DpStats()
        _lib.check(lib.dp_bfs_part_solve_peer(
            p.rowptr.data_ptr(), p.col.data_ptr(), p.n_local, p.n, p.nparts,
            p.part, src, ctypes.byref(c), p.dist.data_ptr(),
            p.peer_ptrs.data_ptr(), p.counts.data_ptr(), p.counts.numel(),
            p.sent.data_ptr(), exchange.sig_table.data_ptr(), epoch, s,
            ctypes.byref(st)))
        p.stats.append(_lib.stats_dict(st))
    run_parts(parts, one, [stream] if stream is not None and
              len(parts) == 1 else None)
    levels = {int(p.stats[-1]["iterations"]) for p in parts}
    if len(levels) != 1:
        raise RuntimeError(f"parts disagree on the level count: {levels}")
    if not gather:
        return None, None, levels.pop()
    return (exchange.dist(parts),
            parts[0].natural_counts(exchange.counts(parts)), levels.pop())
