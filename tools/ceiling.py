"""Ceilings that bind the BFS / SSSP edge work (tools/ceiling.cu), measured
on the RMAT-22 target stream, next to the nested kernels' own times.

    python tools/ceiling.py [scale]   -> JSON lines (profiles/ceiling_*.txt)
"""
import ctypes
import json
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

SO = ROOT / "tools" / "libceiling.so"


def build():
    if not SO.exists() or SO.stat().st_mtime < (
            ROOT / "tools" / "ceiling.cu").stat().st_mtime:
        subprocess.run(["nvcc", "-O3", "-lineinfo", "-gencode",
                        "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
                        "-shared", "-o", str(SO),
                        str(ROOT / "tools" / "ceiling.cu")], check=True)
    L = ctypes.CDLL(str(SO))
    P = ctypes.c_void_p
    L.ceil_run.argtypes = [ctypes.c_int, P, P, ctypes.c_longlong, P, P,
                           ctypes.c_uint32, ctypes.c_int, ctypes.c_int, P, P]
    return L


NAMES = {0: "stream_col", 1: "stream_col_int4", 2: "red_uniform",
         3: "red_targets", 4: "red_merged", 5: "probe_targets",
         6: "visit_flat", 7: "relax_flat", 8: "cas_uniform", 9: "red_hashed",
         10: "red_single_address", 11: "red_one_line", 12: "visit_spread",
         13: "visit_hubrep", 14: "visit_nocount",
         15: "visit_fused64", 16: "visit_fused64_spread"}


def main():
    argv = [a for a in sys.argv[1:] if a != "--write"]
    scale = int(argv[0]) if argv else 22
    only = [int(x) for x in argv[1].split(",")] if len(argv) > 1 \
        else list(NAMES)
    L = build()
    from bench import BEST, DeviceGraph, _cfg, run_dev
    torch.cuda.set_device(0)
    G = DeviceGraph(scale, 1, weights=True)
    n, m = G.n, G.m
    s = torch.cuda.current_stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    scratch = torch.zeros(4, dtype=torch.int32, device="cuda")
    nmask = n - 1
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    out = {"scale": scale, "n": n, "m": m, "sms": sms, "hbm_gbs": hbm}
    hubrep = [int(x) for x in __import__("os").environ.get(
        "HUBREP", "3:4").split(":")]  # kmax : log2 replicas
    for which in only:
        best = None
        for blocks_per_sm, block in ((8, 256), (16, 128), (4, 512)):
            grid = sms * blocks_per_sm
            ts = []
            for it in range(6):
                G.counts.zero_()
                if which in (6, 12, 13, 14):
                    G.dist.fill_(1 << 30)
                    G.dist[0] = 0
                elif which == 7:
                    G.dist.fill_(1 << 30)
                else:
                    G.dist.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s)
                rc = L.ceil_run(which, p(G.col), p(G.weight), m, p(G.dist),
                                p(G.counts),
                                (hubrep[0] << 8 | hubrep[1]) if which == 13
                                else nmask, grid, block, p(scratch), sp)
                e1.record(s)
                torch.cuda.synchronize()
                assert rc == 0, rc
                if it:
                    ts.append(e0.elapsed_time(e1))
            t = statistics.median(ts)
            if best is None or t < best[0]:
                best = (t, grid, block)
        t, grid, block = best
        ops = m if which != 1 else m
        r = {"kernel": NAMES[which] + (f" k<={hubrep[0]} R={1 << hubrep[1]}"
                                       if which == 13 else ""), "ms": t, "grid": grid, "block": block,
             "g_ops_per_s": ops / t / 1e6}
        if which in (0, 1):
            r["gbps"] = 4 * m / t / 1e6
            r["frac_hbm"] = r["gbps"] / hbm
        if which == 3:
            r["red_atomics_per_s"] = m / t / 1e6
        out[NAMES[which]] = r
        print(json.dumps(r), flush=True)
    # the nested kernels on the same graph
    for kind in (("bfs", "sssp") if 6 in only and 7 in only else ()):
        cfg = _cfg(BEST[kind])
        ts, st = [], None
        for _ in range(6):
            st = run_dev(kind, G, cfg, sp)
            ts.append(st["ns_device"] / 1e6)
        r = {"kernel": f"nested {kind} (BEST policy)",
             "ms": statistics.median(ts[1:]),
             "iterations": st["iterations"]}
        if kind == "bfs":
            e_t = int(G.counts.to(torch.int64).sum().item())
            r["edges"] = e_t
            r["g_edges_per_s"] = e_t / r["ms"] / 1e6
            r["frac_of_visit_flat"] = (
                out["visit_flat"]["ms"] * e_t / m) / r["ms"]
            if "visit_spread" in out:
                r["frac_of_visit_spread"] = (
                    out["visit_spread"]["ms"] * e_t / m) / r["ms"]
        else:
            r["ms_per_round"] = st["ns_kernel_sum"] / 1e6 / st["iterations"]
            r["frac_of_relax_flat_per_round"] = (
                out["relax_flat"]["ms"] / r["ms_per_round"])
        out[r["kernel"]] = r
        print(json.dumps(r), flush=True)
    if "--write" in sys.argv:  # the summary bench.py reports against
        (ROOT / "profiles" / "ceilings.json").write_text(
            json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
