"""Packed SSSP weights (dp_config.weight_bits = 4): weights in [1, 16] are
read as nibbles; outside that range the device path falls back to int32 and
the host-buffer path keeps int32 for the first chunk holding such a weight
and every later one.  The 3-byte col transfer (dp_config.col_bits = 24):
chunks of col cross PCIe packed and are expanded on the device; a chunk with
a value outside [0, 2^24) travels as int32.  Distances must equal the
oracle's bit for bit in all cases, and the host path must copy fewer bytes
when it packs."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle
from paper_2201_02789_b200.bench import BenchConfig, load, run_config
from paper_2201_02789_b200.bench.benchmarks import Workload

pytestmark = pytest.mark.gpu

POLICIES = [
    dict(weight_bits=4),
    dict(threshold=64, cfactor=4, agg="multiblock", group_size=1 << 20,
         serial="warp", weight_bits=4),
    dict(threshold=1024, cfactor=16, agg="multiblock", group_size=1 << 20,
         parent_block=128, child_block=128, serial="warp", weight_bits=4),
    dict(threshold=32, agg="grid", frontier=True, weight_bits=4),
]


def _with_weights(wl, weight):
    return Workload(wl.spec, dict(wl.buffers, weight=weight), wl.n,
                    wl.payload)


def _device_dist(wl, policy):
    import ctypes
    import torch
    from paper_2201_02789_b200 import _lib
    b = wl.buffers
    dev = torch.device("cuda", 0)
    t = {k: torch.from_numpy(np.ascontiguousarray(b[k], np.int32)).to(dev)
         for k in ("rowptr", "col", "weight")}
    dist = torch.empty(wl.n, dtype=torch.int32, device=dev)
    st = _lib.DpStats()
    _lib.check(_lib.device().dp_sssp_dev(
        t["rowptr"].data_ptr(), t["col"].data_ptr(), t["weight"].data_ptr(),
        wl.n, int(b["col"].shape[0]), 0,
        ctypes.byref(BenchConfig(**policy).to_c()), dist.data_ptr(), None,
        ctypes.byref(st)))
    return dist.cpu().numpy()


@pytest.mark.parametrize("spec", ["powerlaw:2000:seed1", "road:1000:seed7",
                                  "rmat:16:seed1"])
@pytest.mark.parametrize("pi", range(len(POLICIES)))
def test_packed_weights_exact(spec, pi):
    bench, wl = load("sssp", spec)
    b = wl.buffers
    want, _ = oracle.sssp(b["rowptr"], b["col"], b["weight"], nthreads=0)
    np.testing.assert_array_equal(_device_dist(wl, POLICIES[pi]), want)
    rep, _ = run_config(bench, wl, BenchConfig(**POLICIES[pi]))  # dp_sssp
    np.testing.assert_array_equal(rep.arrays["dist"], want)


@pytest.mark.parametrize("where", ["first", "middle", "last", "none"])
def test_out_of_range_weights_fall_back(where, monkeypatch):
    """Weights > 16 (or < 1) in some chunk: that chunk and the later ones
    travel as int32, the earlier ones packed; the device path drops packing
    altogether."""
    monkeypatch.setenv("DP_COPY_CHUNK_SHIFT", "12")  # many small chunks
    bench, wl = load("sssp", "rmat:14:seed1")
    w = np.array(wl.buffers["weight"], dtype=np.int32)
    m = w.shape[0]
    if where != "none":
        at = {"first": 5, "middle": m // 2, "last": m - 1}[where]
        w[at] = 40
        w[(at * 7) % m] = 17
    wl2 = _with_weights(wl, w)
    want, _ = oracle.sssp(wl.buffers["rowptr"], wl.buffers["col"], w,
                          nthreads=0)
    for pol in POLICIES[:3]:
        np.testing.assert_array_equal(_device_dist(wl2, pol), want)
        rep, _ = run_config(bench, wl2, BenchConfig(**pol))
        np.testing.assert_array_equal(rep.arrays["dist"], want)


def test_host_packing_copies_fewer_bytes():
    bench, wl = load("sssp", "rmat:16:seed1")
    m = wl.buffers["col"].shape[0]
    r0, _ = run_config(bench, wl, BenchConfig())
    r4, _ = run_config(bench, wl, BenchConfig(weight_bits=4))
    np.testing.assert_array_equal(r0.arrays["dist"], r4.arrays["dist"])
    # int32 weights: 4 B per slot; packed: 0.5 B per slot
    assert r0.h2d_bytes - r4.h2d_bytes >= int(m * 3.4)


@pytest.mark.parametrize("spec", ["rmat:16:seed1", "road:1000:seed7",
                                  "powerlaw:2000:seed1"])
@pytest.mark.parametrize("shift", ["", "2", "5", "12"])
def test_col24_transfer_exact(spec, shift, monkeypatch):
    """Chunk sizes 4, 32, 4096 slots and the default, with and without the
    packed weights: ragged last chunks and partial 4-slot groups."""
    if shift:
        monkeypatch.setenv("DP_COPY_CHUNK_SHIFT", shift)
    bench, wl = load("sssp", spec)
    b = wl.buffers
    want, _ = oracle.sssp(b["rowptr"], b["col"], b["weight"], nthreads=0)
    m = b["col"].shape[0]
    r0, _ = run_config(bench, wl, BenchConfig())
    for extra in (dict(col_bits=24), dict(col_bits=24, weight_bits=4)):
        rep, _ = run_config(bench, wl, BenchConfig(**extra))
        np.testing.assert_array_equal(rep.arrays["dist"], want)
        # 4 B per col slot -> 3 B (whole 4-slot groups per chunk)
        saved = r0.h2d_bytes - rep.h2d_bytes
        if "weight_bits" in extra:
            saved -= int(m * 3.4)
        assert saved >= int(m * 0.9), (extra, saved, m)


def test_col24_out_of_range_chunk_travels_int32(monkeypatch):
    """n > 2^24: the chunks naming a vertex >= 2^24 go as int32, the others
    packed; distances still exact."""
    monkeypatch.setenv("DP_COPY_CHUNK_SHIFT", "6")
    rng = np.random.default_rng(3)
    n = (1 << 24) + 64
    hubs = np.array([0, 1, 2, 3, n - 1, n - 2, (1 << 24) + 5, 12345],
                    np.int64)
    src_of = np.repeat(np.arange(hubs.size), 96)
    dst = rng.choice(hubs, size=src_of.size)
    dst[::7] = rng.integers(0, n, size=dst[::7].size)
    rows = hubs[src_of]
    order = np.lexsort((dst, rows))
    rows, dst = rows[order], dst[order]
    rowptr = np.zeros(n + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.int32)
    col = dst.astype(np.int32)
    w = rng.integers(1, 17, size=col.size).astype(np.int32)
    want, _ = oracle.sssp(rowptr, col, w, nthreads=0)
    d0, h0 = _host_sssp(rowptr, col, w, n, BenchConfig())
    d24, h24 = _host_sssp(rowptr, col, w, n, BenchConfig(col_bits=24))
    np.testing.assert_array_equal(d0, want)
    np.testing.assert_array_equal(d24, want)
    assert (col >= (1 << 24)).any()
    assert 0 < h0 - h24 < col.size


def _host_sssp(rowptr, col, w, n, cfg):
    import ctypes
    from paper_2201_02789_b200 import _lib
    dist = np.empty(n, dtype=np.int32)
    st = _lib.DpStats()
    _lib.check(_lib.device().dp_sssp(
        _lib.ptr(rowptr), _lib.ptr(col), _lib.ptr(w), n, col.shape[0], 0,
        ctypes.byref(cfg.to_c()), _lib.ptr(dist), ctypes.byref(st)))
    return dist, int(st.h2d_bytes)


@pytest.mark.parametrize("shift", ["", "6"])
def test_speculative_readback_is_the_result(shift, monkeypatch):
    """dp_sssp copies dist back while the next round runs; the copy that
    overlapped a round which lowered nothing is the result (no final D2H).
    Every copy is counted in d2h_bytes."""
    if shift:
        monkeypatch.setenv("DP_COPY_CHUNK_SHIFT", shift)
    for spec in ("rmat:16:seed1", "road:1000:seed7"):
        bench, wl = load("sssp", spec)
        b = wl.buffers
        want, _ = oracle.sssp(b["rowptr"], b["col"], b["weight"], nthreads=0)
        for pol in POLICIES[:2]:
            d, _ = _host_sssp(b["rowptr"], b["col"], b["weight"], wl.n,
                              BenchConfig(**pol))
            np.testing.assert_array_equal(d, want)
            rep, _ = run_config(bench, wl, BenchConfig(**pol))
            assert rep.d2h_bytes % (wl.n * 4) == 0 and rep.d2h_bytes >= wl.n * 4


def test_host_sssp_source_without_edges():
    """The first round lowers nothing: no speculative copy exists, the call
    must still return dist (regression: it once skipped the final D2H)."""
    rowptr = np.array([0, 0, 2, 3], np.int32)
    col = np.array([2, 0, 1], np.int32)
    w = np.array([1, 2, 3], np.int32)
    want, _ = oracle.sssp(rowptr, col, w, nthreads=0)
    for pol in POLICIES[:2]:
        d, _ = _host_sssp(rowptr, col, w, 3, BenchConfig(**pol))
        np.testing.assert_array_equal(d, want)
