"""BT (Bezier tessellation) at the config-2 size and a streaming size:
device time per policy through dp_bt_dev with device-resident buffers,
achieved GB/s of the algorithmic bytes (36 B/curve + 8 B/vertex) against the
HBM peak, and parity of the timed policy against the oracle.

    python tools/bt_study.py [ncurves ...] [--profile NCURVES POLICY_JSON]
"""
import ctypes
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_02789_b200 import _lib  # noqa: E402
from paper_2201_02789_b200.bench import BenchConfig, INF_THRESHOLD  # noqa
from paper_2201_02789_b200.bench.graphs import (BT_CURV_SCALE,  # noqa: E402
                                                BT_MAX_TESS, bezier_curves)

POLICIES = [
    dict(threshold=INF_THRESHOLD, serial="warp", parent_block=32),
    dict(threshold=INF_THRESHOLD, serial="warp", parent_block=128),
    dict(threshold=256, cfactor=1, agg="multiblock", group_size=1 << 20,
         parent_block=64, child_block=256, serial="warp"),
    dict(threshold=512, cfactor=1, agg="multiblock", group_size=1 << 20,
         parent_block=64, child_block=256, serial="warp"),
    dict(threshold=512, cfactor=2, agg="multiblock", group_size=1 << 20,
         parent_block=64, child_block=128, serial="warp"),
    dict(threshold=1024, cfactor=1, agg="multiblock", group_size=1 << 20,
         parent_block=64, child_block=256, serial="warp"),
    dict(threshold=512, cfactor=1, agg="multiblock", group_size=64,
         parent_block=64, child_block=256, serial="warp"),
    dict(threshold=INF_THRESHOLD, serial="warp", parent_block=64),
    dict(threshold=INF_THRESHOLD, serial="warp", parent_block=256),
    dict(threshold=INF_THRESHOLD, serial="thread", parent_block=64),
    dict(threshold=64, cfactor=16, agg="multiblock", group_size=4,
         parent_block=256, child_block=32, serial="warp"),  # config 2
    dict(threshold=64, cfactor=4, agg="multiblock", group_size=1 << 20,
         parent_block=128, child_block=32, serial="warp"),
    dict(threshold=32, cfactor=1, agg="multiblock", group_size=1 << 20,
         parent_block=256, child_block=256, serial="warp"),
    dict(threshold=128, cfactor=8, agg="multiblock", group_size=1 << 20,
         parent_block=256, child_block=128, serial="warp"),
    dict(threshold=0, cfactor=1, agg="multiblock", group_size=1 << 20,
         parent_block=256, child_block=128, serial="warp"),
    dict(threshold=0, cfactor=4, agg="grid", parent_block=256,
         child_block=128, serial="warp"),
]


class Bt:
    def __init__(self, n: int):
        self.n = n
        cp = bezier_curves(n, 1)
        self.cp_h = np.ascontiguousarray(cp, dtype=np.float32)
        dev = torch.device("cuda", 0)
        self.cp = torch.from_numpy(self.cp_h).to(dev)
        self.cap = n * 160
        self.ntess = torch.empty(n, dtype=torch.int32, device=dev)
        self.offs = torch.empty(n, dtype=torch.int64, device=dev)
        self.verts = torch.empty((self.cap, 2), dtype=torch.float32,
                                 device=dev)
        self.stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        self.lib = _lib.device()

    def run(self, pol: dict):
        used = ctypes.c_int64()
        st = _lib.DpStats()
        _lib.check(self.lib.dp_bt_dev(
            self.cp.data_ptr(), self.n, BT_MAX_TESS, BT_CURV_SCALE,
            ctypes.byref(BenchConfig(**pol).to_c()), self.ntess.data_ptr(),
            self.offs.data_ptr(), self.verts.data_ptr(), self.cap,
            ctypes.byref(used), self.stream, ctypes.byref(st)))
        return int(used.value), _lib.stats_dict(st)

    def check(self, nv: int) -> str:
        from oracle import oracle
        from paper_2201_02789_b200.bench.benchmarks import canonical_vertices
        nt, want = oracle.bt(self.cp_h, BT_MAX_TESS, BT_CURV_SCALE)
        got_nt = self.ntess.cpu().numpy()
        if not np.array_equal(got_nt, nt):
            return "MISMATCH (ntess)"
        v = canonical_vertices(self.verts[:nv].cpu().numpy(), got_nt,
                               self.offs.cpu().numpy())
        ok = np.allclose(v, want, rtol=1e-5, atol=1e-6)
        return "within 1e-5 of the oracle" if ok else "MISMATCH (verts)"


def main():
    args = sys.argv[1:]
    torch.cuda.set_device(0)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    if args and args[0] == "--profile":
        bt = Bt(int(args[1]))
        pol = json.loads(args[2])
        for _ in range(3):
            bt.run(pol)
        torch.cuda.synchronize()
        return
    sizes = [int(a) for a in args] or [25000, 1000000]
    for n in sizes:
        bt = Bt(n)
        res = []
        for pol in POLICIES:
            ts = []
            for _ in range(7):
                nv, st = bt.run(pol)
                ts.append(st["ns_device"] / 1e3)
            t = statistics.median(ts[2:])
            alg = 36 * n + 8 * nv
            res.append((t, pol, nv, st))
            print(json.dumps({"ncurves": n, "us": round(t, 2),
                              "vertices": nv,
                              "gbps_alg": round(alg / (t * 1e3), 1),
                              "frac_hbm": round(alg / (t * 1e3) / hbm, 3),
                              "launches": st["num_launches"],
                              "launch_lat_us": round(
                                  st["launch_lat_ns_mean"] / 1e3, 2),
                              "policy": pol}), flush=True)
        best = min(res, key=lambda r: r[0])
        bt.run(best[1])
        print(json.dumps({"ncurves": n, "best_us": best[0],
                          "best_policy": best[1],
                          "parity": bt.check(best[2])}), flush=True)


if __name__ == "__main__":
    main()
