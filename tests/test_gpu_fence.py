"""The multiblock protocol's fence is load-bearing: the reference's
publication checker and its fence-deletion mutation
(tests/test_passes.py:541-554, tests/conftest.py:13-28 `strip_fences`,
sim/machine.py:543-649) on hardware.

Two extra builds of the library (csrc/Makefile `check`):
  libdynpar_check.so    DP_CHECK_PUBLISH: every aggregation-table row carries
                        a stamp that only its publication sets (the
                        multiblock fence; the launch for warp/block rows; the
                        parent grid's end for grid rows), child blocks verify
                        it, rows are poisoned with 0xff bytes before every
                        parent grid; an unpublished read traps with kind
                        "unpublished-read" (the reference's SimTrap kind)
  libdynpar_nofence.so  the same with the protocol's fences deleted
Each build runs in a child process (DYNPAR_LIB), as in test_gpu_profile.py.

The reference asserts three things; so do these tests:
  intact program, checker on      -> clean, outputs equal the golden digests
  fences deleted, checker on      -> SimTrap("unpublished-read")
  fences deleted, checker off     -> (the quiet run) the bytes still come out
                                     right, which is why the checker exists;
                                     here also: no poisoned row was observed
                                     or the outputs would have diverged
Block, warp and grid aggregation need no fence (test_passes.py:557-562), so
the mutation leaves them clean."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2201_02789_b200" / "csrc"
CHECK_LIB = CSRC / "libdynpar_check.so"
NOFENCE_LIB = CSRC / "libdynpar_nofence.so"

# name -> (bench, dataset, policy); group_size=3 is the reference test's
MULTI = {
    "bfs_multi_g3": ("bfs", "powerlaw:2000:seed1",
                     dict(threshold=8, agg="multiblock", group_size=3)),
    "sssp_multi_g3": ("sssp", "powerlaw:2000:seed1",
                      dict(threshold=8, cfactor=2, agg="multiblock",
                           group_size=3)),
    "ml_multi_g2": ("manylaunch", "sizes:1024:seed1",
                    dict(agg="multiblock", group_size=2)),
    "bfs_rmat_multi_g1": ("bfs", "rmat:16:seed1",
                          dict(threshold=32, cfactor=2, agg="multiblock",
                               group_size=1, parent_block=128,
                               child_block=128, serial="warp")),
    "bfs_act_multi": ("bfs", "powerlaw:2000:seed1",
                      dict(threshold=8, cfactor=3, agg="multiblock",
                           group_size=3, order="ACT")),
}
NO_FENCE_NEEDED = {
    "bfs_block": ("bfs", "powerlaw:2000:seed1",
                  dict(threshold=8, agg="block")),
    "bfs_warp": ("bfs", "powerlaw:2000:seed1",
                 dict(threshold=8, agg="warp")),
    "sssp_grid": ("sssp", "powerlaw:2000:seed1",
                  dict(threshold=8, cfactor=2, agg="grid")),
}

CHILD = r"""
import json, sys
from paper_2201_02789_b200._lib import DeviceTrap
from paper_2201_02789_b200.bench import (BenchConfig, load, run_config,
                                         run_reference)
out = {}
for name, (b, ds, pol) in json.loads(sys.argv[1]).items():
    bench, wl = load(b, ds)
    ref = run_reference(bench, wl)
    try:
        rep, _ = run_config(bench, wl, BenchConfig(**pol))
        out[name] = dict(digest=rep.memory_digest, ref=ref.memory_digest,
                         unpublished=rep.unpublished_reads,
                         poisoned=rep.poisoned_reads,
                         launches=rep.num_launches)
    except DeviceTrap as e:
        out[name] = dict(trap=e.kind, msg=str(e), ref=ref.memory_digest)
print(json.dumps(out))
"""


def _run(lib: Path, cases: dict, trap: bool = True) -> dict:
    assert lib.exists(), f"{lib.name} not built (make -C csrc check)"
    env = dict(os.environ, DYNPAR_LIB=str(lib),
               DYNPAR_CHECK_TRAP="1" if trap else "0")
    r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(cases)],
                       capture_output=True, text=True, env=env, cwd=ROOT,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def _golden(golden, bench, ds):
    for r in golden["reference"]:
        if r["bench"] == bench and r["dataset"] == ds:
            return r["digest"]
    return None


def _assert_outputs(golden, cases, out):
    for name, (b, ds, _) in cases.items():
        o = out[name]
        assert o["digest"] == o["ref"], f"{name}: differs from No-CDP"
        want = _golden(golden, b, ds)
        if want is not None:
            assert o["digest"] == want, f"{name}: differs from the reference"


def test_checked_build_is_clean(golden):
    cases = {**MULTI, **NO_FENCE_NEEDED}
    out = _run(CHECK_LIB, cases)
    for name in cases:
        assert "trap" not in out[name], out[name]
        assert out[name]["unpublished"] == 0, (name, out[name])
        assert out[name]["poisoned"] == 0, (name, out[name])
        if cases[name][2]["agg"] != "grid":  # grid: host-launched child
            assert out[name]["launches"] > 0, name
    _assert_outputs(golden, cases, out)


def test_fence_deletion_is_caught():
    out = _run(NOFENCE_LIB, MULTI)
    for name in MULTI:
        assert out[name].get("trap") == "unpublished-read", (name, out[name])


def test_fence_deletion_spares_block_warp_grid(golden):
    out = _run(NOFENCE_LIB, NO_FENCE_NEEDED)
    for name in NO_FENCE_NEEDED:
        assert "trap" not in out[name], out[name]
        assert out[name]["unpublished"] == 0, (name, out[name])
    _assert_outputs(golden, NO_FENCE_NEEDED, out)


def test_fence_deletion_quiet_run(golden):
    """checked=False: the mutated program still counts its unpublished
    reads; the outputs are right exactly when no child observed a poisoned
    (not yet visible) row."""
    out = _run(NOFENCE_LIB, MULTI, trap=False)
    for name, (b, ds, _) in MULTI.items():
        o = out[name]
        assert "trap" not in o, o
        assert o["unpublished"] > 0, (name, o)
        if o["poisoned"] == 0:
            assert o["digest"] == o["ref"], (name, o)
            want = _golden(golden, b, ds)
            if want is not None:
                assert o["digest"] == want, name


def test_default_build_has_no_checker():
    from paper_2201_02789_b200.bench import BenchConfig, load, run_config
    bench, wl = load("bfs", "powerlaw:2000:seed1")
    rep, _ = run_config(bench, wl, BenchConfig(threshold=8, agg="multiblock",
                                               group_size=3))
    assert rep.unpublished_reads == 0 and rep.poisoned_reads == 0
