"""Policy sweep on the device: median device time per configuration.

    python tools/tune.py sssp 22 [--quick]
Prints one line per config: ms, rounds, launches, blocks, GTEPS.
"""

from __future__ import annotations

import ctypes
import itertools
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import DeviceGraph, _cfg, run_dev  # noqa: E402


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "sssp"
    scale = int(sys.argv[2]) if len(sys.argv) > 2 else 22
    grid = sys.argv[3] if len(sys.argv) > 3 else "wide"
    torch.cuda.set_device(0)
    G = DeviceGraph(scale, 1, weights=(kind == "sssp"))
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    deg = np.diff(G.g.rowptr.astype(np.int64))
    configs = []
    if grid == "wide":
        configs.append(dict(variant="nocdp", parent_block=256))
        configs.append(dict(variant="nocdp", parent_block=256, serial="warp"))
        for agg in (None, "warp", "block", "grid"):
            configs.append(dict(agg=agg))
        for T, C, agg, pb, cb, ser in itertools.product(
                (128, 512, 2048, 8192), (1, 8), ("block", "multiblock", "grid"),
                (256,), (32, 128), ("thread", "warp")):
            configs.append(dict(threshold=T, cfactor=C, agg=agg,
                                group_size=4, parent_block=pb, child_block=cb,
                                serial=ser))
    elif grid == "best":
        from bench import BEST
        configs.append(dict(BEST[kind]))
        d = dict(BEST[kind]); d["agg"] = "grid"; d.pop("group_size", None)
        configs.append(d)
    elif grid == "dloop":
        from bench import BEST
        for dl in (False, True):
            d = dict(BEST[kind]); d["device_loop"] = dl
            configs.append(d)
            d = dict(d); d["group_size"] = 2048
            configs.append(d)
    elif grid == "persist":
        from bench import BEST
        for ps, T, C in itertools.product((0, 1, 2, 3, 4, 6), (512, 1024, 2048),
                                          (8, 32)):
            d = dict(BEST[kind]); d.update(persistent=ps, threshold=T,
                                           cfactor=C, group_size=1 << 20)
            configs.append(d)
    elif grid == "groups":
        from bench import BEST
        for gs in (8, 32, 128, 512, 2048, 1 << 20):
            d = dict(BEST[kind]); d["group_size"] = gs
            configs.append(d)
    elif grid == "top":
        for T, C, agg, cb in itertools.product(
                (512, 1024, 2048), (16, 32), ("grid", "mb-all", "mb16"),
                (64, 128)):
            d = dict(threshold=T, cfactor=C, parent_block=256, child_block=cb,
                     serial="warp")
            if agg == "grid":
                d["agg"] = "grid"
            elif agg == "mb-all":
                d.update(agg="multiblock", group_size=1 << 20)
            else:
                d.update(agg="multiblock", group_size=16)
            configs.append(d)
        for pb in (128, 512):
            configs.append(dict(threshold=1024, cfactor=32, agg="multiblock",
                                group_size=1 << 20, parent_block=pb,
                                child_block=64, serial="warp"))
    elif grid == "focus":
        configs.append(dict(variant="nocdp", parent_block=256, serial="warp"))
        configs.append(dict(agg="grid", parent_block=256))
        for T, C, agg, cb in itertools.product(
                (128, 256, 512, 1024, 2048, 4096), (4, 8, 16, 32),
                ("grid", "mb-all", "mb16"), (64, 128, 256)):
            d = dict(threshold=T, cfactor=C, parent_block=256, child_block=cb,
                     serial="warp")
            if agg == "grid":
                d["agg"] = "grid"
            elif agg == "mb-all":
                d.update(agg="multiblock", group_size=1 << 20)
            else:
                d.update(agg="multiblock", group_size=16)
            configs.append(d)
        for pb in (64, 128, 512, 1024):
            configs.append(dict(threshold=512, cfactor=8, agg="grid",
                                parent_block=pb, child_block=128,
                                serial="warp"))
    elif grid in ("cf", "frontier"):
        for T, C, cb, gs in itertools.product(
                (512, 1024, 2048), (4, 8, 16, 32), (64, 128),
                (512, 2048, 1 << 20)):
            configs.append(dict(threshold=T, cfactor=C, agg="multiblock",
                                group_size=gs, parent_block=128,
                                child_block=cb, serial="warp",
                                frontier=grid == "frontier"))
    elif grid == "cf2":
        # re-tune after the hub children's unroll changed (kChildUnroll)
        for T, C, cb, pb in itertools.product(
                (256, 512, 1024, 2048), (4, 8, 16, 32, 64), (64, 128, 256),
                (128, 256)):
            configs.append(dict(threshold=T, cfactor=C, agg="multiblock",
                                group_size=1 << 20, parent_block=pb,
                                child_block=cb, serial="warp"))
    from paper_2201_02789_b200 import _lib
    for d in configs:
        d = dict(d)
        variant = d.pop("variant", "cdp")
        c = _cfg(d)
        if variant == "nocdp":
            c.variant = _lib.VARIANT_NOCDP
        try:
            runs = [run_dev(kind, G, c, stream) for _ in range(3)]
        except Exception as e:  # noqa: BLE001
            print(f"{variant} {d} ERROR {e}", flush=True)
            continue
        ms = statistics.median(r["ns_device"] for r in runs) / 1e6
        ks = statistics.median(r["ns_kernel_sum"] for r in runs) / 1e6
        reached = G.dist.cpu().numpy() < (1 << 30)
        e = int(deg[reached].sum())
        print(f"{ms:9.3f} ms  kern {ks:9.3f}  it={runs[0]['iterations']:3d} "
              f"launches={runs[0]['num_launches']:9d} "
              f"blocks={runs[0]['blocks_scheduled']:10d} "
              f"GTEPS={e / ms / 1e6:7.2f} lat={runs[0]['launch_lat_ns_mean']:8.0f}ns"
              f"  {variant} {d}", flush=True)


if __name__ == "__main__":
    main()
