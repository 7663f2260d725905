"""The paper's ablation (Fig. 9) on one B200: device time
of No-CDP, CDP, and CDP with each subset of T / C / A, for SSSP, BFS, TC
(RMAT-22) and BT (25k curves).  A = best of warp / block / multiblock(one
group) / grid aggregation for that combination; T and C use the tuned
values of bench.BEST.  Prints a table of ms and the geomean ratios the paper
reports."""
import ctypes
import math
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import BEST, DeviceGraph, _cfg, run_dev  # noqa: E402
from paper_2201_02789_b200 import _lib  # noqa: E402
from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa

AGGS = ("warp", "block", "multiblock", "grid")


# BT's tuned policy runs every curve in the parent (T = INF, no launches);
# its ablation uses the config-2 policy's T and C instead
T_C_OVERRIDE = {"bt": (64, 16)}


def variants(best, kind=None):
    T, C = T_C_OVERRIDE.get(kind, (best["threshold"], best.get("cfactor", 1)))
    base = dict(parent_block=best.get("parent_block", 32),
                child_block=best.get("child_block", 32),
                serial=best.get("serial", "thread"))
    out = {"CDP": [dict(base)], "CDP+T": [dict(base, threshold=T)],
           "CDP+C": [dict(base, cfactor=C)],
           "CDP+T+C": [dict(base, threshold=T, cfactor=C)]}
    for name, extra in (("CDP+A", {}), ("CDP+T+A", dict(threshold=T)),
                        ("CDP+C+A", dict(cfactor=C)),
                        ("CDP+T+C+A", dict(threshold=T, cfactor=C))):
        out[name] = [dict(base, agg=a, group_size=1 << 20, **extra)
                     for a in AGGS]
    return out


def main():
    torch.cuda.set_device(0)
    lib = _lib.device()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    table = {}
    for kind in ("sssp", "bfs"):
        G = DeviceGraph(22, 1, weights=(kind == "sssp"))

        def t(pol, variant=_lib.VARIANT_CDP):
            c = _cfg(pol)
            c.variant = variant
            run_dev(kind, G, c, stream)
            return statistics.median(run_dev(kind, G, c, stream)["ns_device"]
                                     for _ in range(3)) / 1e6
        row = {"No CDP": t(dict(parent_block=256), _lib.VARIANT_NOCDP)}
        for name, pols in variants(BEST[kind], kind).items():
            row[name] = min(t(p) for p in pols)
        table[kind] = row
        del G
        torch.cuda.empty_cache()
        print(kind, {k: round(v, 3) for k, v in row.items()}, flush=True)
    for kind, spec in (("tc", "rmat:22:seed1"), ("bt", "curves:25000:seed1")):
        bench, wl = load(kind, spec)

        def t(pol, nocdp=False):
            from paper_2201_02789_b200.bench import run_reference
            if nocdp:
                return min(run_reference(bench, wl).ns_device
                           for _ in range(2)) / 1e6
            return min(run_config(bench, wl, BenchConfig(**pol))[0].ns_device
                       for _ in range(3)) / 1e6
        row = {"No CDP": t({}, nocdp=True)}
        for name, pols in variants(BEST[kind], kind).items():
            row[name] = min(t(p) for p in pols)
        table[kind] = row
        print(kind, {k: round(v, 3) for k, v in row.items()}, flush=True)

    def geo(a, b):
        return math.exp(statistics.mean(math.log(table[k][a] / table[k][b])
                                         for k in table))
    paper = {("CDP", "CDP+T+C+A"): 43.0, ("No CDP", "CDP+T+C+A"): 8.7,
             ("CDP+A", "CDP+T+C+A"): 3.6, ("CDP", "CDP+A"): 12.1,
             ("No CDP", "CDP+A"): 2.4, ("CDP", "CDP+T"): 13.4,
             ("CDP+A", "CDP+T+A"): 2.9, ("CDP+C+A", "CDP+T+C+A"): 3.1,
             ("CDP", "CDP+C"): 1.01, ("CDP+T", "CDP+T+C"): 1.09,
             ("CDP+A", "CDP+C+A"): 1.16, ("CDP+T+A", "CDP+T+C+A"): 1.22}
    print("\nspeed-up (geomean over sssp, bfs, tc, bt)   B200   paper (V100)")
    for (a, b), p in paper.items():
        print(f"  {b:>10} vs {a:<10}  {geo(a, b):8.2f}x   {p:6.2f}x")


if __name__ == "__main__":
    main()
