"""DP_PROFILE build (libdynpar_prof.so): the per-phase device clocks that
stand in for SimReport.phase_time (reference sim/report.py:12-28; folded
from per-thread costs at sim/machine.py:657-666).

The profiled library is loaded in a child process (DYNPAR_LIB), so the
default library of this process is untouched.  Outputs must be bit-identical
to the golden digests, and each phase must be populated exactly where the
policy has that phase."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

from paper_2201_02789_b200.bench import BenchConfig, load, run_config

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
PROF_LIB = ROOT / "paper_2201_02789_b200" / "csrc" / "libdynpar_prof.so"

POLICIES = {
    "nocdp": dict(threshold=1 << 30),
    "naive": dict(),
    "warp": dict(threshold=8, agg="warp"),
    "multiblock": dict(threshold=8, cfactor=2, agg="multiblock",
                       group_size=2),
}

CHILD = r"""
import json, sys
from paper_2201_02789_b200.bench import BenchConfig, load, run_config
out = {}
for name, pol in json.loads(sys.argv[1]).items():
    bench, wl = load("bfs", "powerlaw:2000:seed1")
    rep, _ = run_config(bench, wl, BenchConfig(**pol))
    out[name] = dict(digest=rep.memory_digest, phase=rep.phase_time,
                     launches=rep.num_launches)
print(json.dumps(out))
"""


def _golden_digest(golden):
    return next(r for r in golden["reference"]
                if r["bench"] == "bfs"
                and r["dataset"] == "powerlaw:2000:seed1")["digest"]


def test_default_build_reports_no_phase_time():
    bench, wl = load("bfs", "powerlaw:2000:seed1")
    rep, _ = run_config(bench, wl, BenchConfig(threshold=8, agg="warp"))
    assert all(v == 0 for v in rep.phase_time.values())


def test_profiled_build_phases(golden):
    assert PROF_LIB.exists(), "libdynpar_prof.so not built (make -C csrc prof)"
    env = dict(os.environ, DYNPAR_LIB=str(PROF_LIB))
    r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(POLICIES)],
                       cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    want = _golden_digest(golden)
    for name, rec in res.items():
        ph = rec["phase"]
        assert rec["digest"] == want, name
        assert ph["parent"] > 0 and ph["child"] > 0, (name, ph)
        if rec["launches"] == 0:
            assert ph["launch"] == 0 and ph["disagg"] == 0, (name, ph)
    # T = INF still runs the launch decision (agg phase), never a launch
    assert res["nocdp"]["launches"] == 0
    for name in ("naive", "warp", "multiblock"):
        assert res[name]["launches"] > 0
        assert res[name]["phase"]["launch"] > 0, name
    for name in ("warp", "multiblock"):
        assert res[name]["phase"]["disagg"] > 0, name
    assert res["naive"]["phase"]["disagg"] == 0


def test_max_pending_depth():
    # SimReport.max_pending_depth (sim/machine.py:237-244): the launch
    # queue's high-water mark; none without device launches, at most one
    # per level with a single aggregated launch, bounded by the launches
    bench, wl = load("bfs", "powerlaw:2000:seed1")
    rep, _ = run_config(bench, wl, BenchConfig(threshold=1 << 30))
    assert rep.num_launches == 0 and rep.max_pending_depth == 0
    rep, _ = run_config(bench, wl, BenchConfig())
    assert 1 <= rep.max_pending_depth <= rep.num_launches
    rep, _ = run_config(bench, wl, BenchConfig(agg="multiblock",
                                               group_size=1 << 20))
    assert rep.max_pending_depth == 1
