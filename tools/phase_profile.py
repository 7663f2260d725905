"""Per-phase device clocks (DP_PROFILE build) for SSSP and BFS on RMAT-22:
the measured counterpart of the reference's SimReport.phase_time
(sim/report.py:12-28) over the ablation's policy ladder (CDP, CDP+T,
CDP+T+C, CDP+T+C+A, No CDP).

Run with the profiled library:
  DYNPAR_LIB=paper_2201_02789_b200/csrc/libdynpar_prof.so \
      python tools/phase_profile.py
Phases are summed warp-cycles converted at the reported SM clock (warp-ms),
so they measure where warps spend time, not wall time; ns_device of a
profiled run includes the clock64/atomic overhead and is not a bench
number."""
import ctypes
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import BEST, DeviceGraph, _cfg, run_dev  # noqa: E402
from paper_2201_02789_b200 import _lib  # noqa: E402

PHASES = ("parent", "launch", "agg", "disagg", "child")


def ladder(best):
    T, C = best["threshold"], best["cfactor"]
    base = dict(parent_block=best["parent_block"],
                child_block=best["child_block"], serial=best["serial"])
    return {"CDP": dict(base), "CDP+T": dict(base, threshold=T),
            "CDP+T+C": dict(base, threshold=T, cfactor=C),
            "CDP+T+C+A": dict(best)}


def main():
    assert "prof" in os.environ.get("DYNPAR_LIB", ""), \
        "run with DYNPAR_LIB=.../libdynpar_prof.so"
    torch.cuda.set_device(0)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    out = {}
    for kind in ("sssp", "bfs"):
        G = DeviceGraph(22, 1, weights=(kind == "sssp"))
        rows = {}
        pols = dict(ladder(BEST[kind]))
        pols["No CDP"] = dict(parent_block=256)
        for name, pol in pols.items():
            c = _cfg(pol)
            if name == "No CDP":
                c.variant = _lib.VARIANT_NOCDP
            run_dev(kind, G, c, stream)
            runs = [run_dev(kind, G, c, stream) for _ in range(3)]
            st = min(runs, key=lambda s: s["ns_device"])
            ph = {p: st["ns_phase"][i] / 1e6 for i, p in enumerate(PHASES)}
            tot = sum(ph.values()) or 1.0
            rows[name] = dict(
                ms_device=round(statistics.median(
                    r["ns_device"] for r in runs) / 1e6, 3),
                launches=int(st["num_launches"]),
                warp_ms={p: round(v, 2) for p, v in ph.items()},
                share={p: round(v / tot, 3) for p, v in ph.items()})
            print(kind, name, json.dumps(rows[name]), flush=True)
        out[kind] = rows
        del G
        torch.cuda.empty_cache()
    dst = Path(os.environ.get("PHASE_OUT", "gpurun_out/phase_profile.json"))
    dst.parent.mkdir(parents=True, exist_ok=True)
    dst.write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
