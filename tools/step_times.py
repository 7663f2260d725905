"""Per-level / per-round device times (dp_step_times) of BFS and SSSP on
RMAT-`scale` under the BEST policies (or a JSON policy override).

    python tools/step_times.py [scale] ['{"cfactor": 4}']
"""
import ctypes
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2201_02789_b200 import _lib  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
    extra = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    torch.cuda.set_device(0)
    G = bench.DeviceGraph(scale, 1, weights=True)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    nocdp = extra.pop("nocdp", False)
    for kind in ("bfs", "sssp"):
        pol = dict(bench.BEST[kind], **extra)
        from paper_2201_02789_b200.bench import BenchConfig
        cfg = (BenchConfig(**pol).to_c(_lib.VARIANT_NOCDP) if nocdp
               else bench._cfg(pol))
        runs = []
        for _ in range(6):
            st = bench.run_dev(kind, G, cfg, s)
            runs.append((st["ns_device"] / 1e6, _lib.step_times()))
        runs = runs[1:]
        steps = [statistics.median(r[1][i] for r in runs)
                 for i in range(len(runs[0][1]))]
        print(json.dumps({"kind": kind, "policy": pol, "nocdp": nocdp,
                          "ms": statistics.median(r[0] for r in runs),
                          "step_ms": [round(x, 4) for x in steps],
                          "sum_steps": round(sum(steps), 4)}), flush=True)


if __name__ == "__main__":
    main()
