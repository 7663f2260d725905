"""Policy sweep for TC (RMAT-22) and BT (25k curves) through the Python API."""
import itertools
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2201_02789_b200.bench import BenchConfig, load, run_config  # noqa
from paper_2201_02789_b200 import _lib  # noqa

kind = sys.argv[1]
spec = {"tc": "rmat:22:seed1", "gc": "rmat:22:seed1"}.get(
    kind, "curves:25000:seed1")
bench, wl = load(kind, spec)
configs = [dict(), dict(agg="grid", parent_block=256)]
for T, C, agg, pb, cb in itertools.product(
        (8, 16, 32, 64, 128) if kind in ("tc", "gc") else (64, 256, 1024, 4096),
        (1, 4, 16), ("grid", "mb-all"), (128, 256), (64, 128, 256)):
    d = dict(threshold=T, cfactor=C, parent_block=pb, child_block=cb,
             serial="warp")
    if agg == "mb-all":
        d.update(agg="multiblock", group_size=1 << 20)
    else:
        d["agg"] = agg
    configs.append(d)
ref = None
for d in configs:
    try:
        reps = [run_config(bench, wl, BenchConfig(**d))[0] for _ in range(3)]
    except Exception as e:  # noqa: BLE001
        print("ERROR", d, e, flush=True)
        continue
    ms = statistics.median(r.ns_device for r in reps) / 1e6
    key = reps[0].memory_digest
    ref = ref or key
    print(f"{ms:9.3f} ms it={reps[0].iterations} launches={reps[0].num_launches:8d} "
          f"blocks={reps[0].blocks_scheduled:9d} same={key == ref} {d}",
          flush=True)
