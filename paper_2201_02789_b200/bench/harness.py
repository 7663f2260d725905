"""Benchmark runner: policy selection, device run, dual-route verification.

Drop-in for ``dynoptc.bench.harness`` (pkg/src/dynoptc/bench/harness.py):
same names, same argument meaning, same errors.  Where the reference
transforms mini-language source (pipeline.transform) and simulates it,
``run_config`` hands the knobs to the policy-templated scheduler in
libdynpar.so and runs the real kernels; ``run_reference`` runs the serial
(No-CDP) variant on the same device.  Outputs are schedule-invariant, so the
dual-route check (harness.py:83-96) is an exact comparison.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .. import _lib
from .benchmarks import BLOCK, Benchmark, Workload, get_benchmark
from .report import Report

CANONICAL_ORDER = "TCA"  # pipeline.py:32
GRANULARITIES = ("warp", "block", "multiblock", "grid")  # + reference's three
INF_THRESHOLD = _lib.INF_THRESHOLD
BT_ABS_TOL = 1e-5  # vertex coordinates lie in [0,1): 1e-5 absolute == relative


@dataclass(frozen=True)
class BenchConfig:
    """One point in the transformation space (harness.py:21-34).

    Reference knobs: threshold, cfactor, agg, group_size, agg_threshold,
    order.  B200 knobs (defaults reproduce the reference's launch shapes):
    parent_block / child_block (threads per parent / child block; the
    reference uses 32 for both), serial ("thread": below-threshold children
    run in the parent thread as threshold.py:60-83 does; "warp": the parent
    warp shares them), pending_launch_limit (CDP2 pool, 0 = auto),
    persistent (blocks per SM of a persistent parent grid for single-group
    aggregation: record every launch first, then the serial arms),
    device_loop (chain BFS levels / SSSP rounds on the device with CDP2 tail
    launches instead of a host launch + flag readback per level), frontier
    (SSSP: a vertex relaxes only when its distance changed since its last
    relaxation; same distances, fewer relaxations)."""
    threshold: int = 0
    cfactor: int = 1
    agg: str | None = None
    group_size: int = 4
    agg_threshold: int = 0
    order: str = CANONICAL_ORDER
    parent_block: int = BLOCK
    child_block: int = 32
    serial: str = "thread"
    pending_launch_limit: int = 0
    persistent: int = 0
    device_loop: bool = False
    frontier: bool = False
    weight_bits: int = 0
    cf_wave: int = 0
    col_bits: int = 0

    def describe(self) -> str:
        return (f"threshold={self.threshold} cfactor={self.cfactor} "
                f"agg={self.agg or 'none'} group_size={self.group_size} "
                f"agg_threshold={self.agg_threshold}")

    def validate(self) -> None:
        """The reference's knob errors (aggregate.py:174-179,
        pipeline.py:79) plus the B200 knobs' ranges."""
        for step in self.order.upper():
            if step not in "TCA":
                raise ValueError(f"unknown pass step {step!r} in order")
        if self.agg is not None and self.agg not in GRANULARITIES:
            raise ValueError(f"unknown aggregation granularity {self.agg!r}")
        if self.agg is not None:
            if self.agg_threshold > 0 and self.agg != "block":
                raise ValueError(
                    "aggregation threshold requires block granularity")
            if self.agg == "multiblock" and self.group_size < 1:
                raise ValueError("group size must be at least 1")
        for name in ("parent_block", "child_block"):
            v = getattr(self, name)
            if v < 32 or v > 256 or v % 32:
                raise ValueError(
                    f"{name} must be a multiple of 32 in [32, 256]")
        if not 0 <= self.persistent <= 8:
            raise ValueError("persistent must be in [0, 8] blocks per SM")
        if self.persistent and self.order_effect(
                self.threshold, self.cfactor, self.agg)[2]:
            raise ValueError("a persistent parent cannot coarsen the "
                             "aggregated grid (order with A before C)")
        if self.serial not in _lib.SERIAL_MODES:
            raise ValueError(f"unknown serial mode {self.serial!r}")
        if self.weight_bits not in (0, 4):
            raise ValueError("weight_bits must be 0 (int32) or 4 (packed)")
        if self.cf_wave < 0:
            raise ValueError("cf_wave must be >= 0")
        if self.col_bits not in (0, 24):
            raise ValueError("col_bits must be 0 (int32) or 24 (3-byte "
                             "transfer)")

    def to_c(self, variant: int = _lib.VARIANT_CDP) -> _lib.DpConfig:
        self.validate()
        c = _lib.DpConfig()
        # threshold 0 (or any T <= 0) disables the pass: every non-empty
        # child launches (pipeline.py:59-61; `_threads >= T` always holds)
        c.threshold = max(int(self.threshold), 0)
        c.cfactor = max(int(self.cfactor), 1)  # cfactor <= 1: pass disabled
        agg_on = self.agg is not None and "A" in self.order.upper()
        c.agg = _lib.AGG_CODES[self.agg if agg_on else None]
        c.group_size = int(self.group_size)
        c.agg_threshold = int(self.agg_threshold) if agg_on else 0
        c.variant = variant
        c.parent_block = int(self.parent_block)
        c.child_block = int(self.child_block)
        c.serial_mode = _lib.SERIAL_MODES[self.serial]
        c.pending_launch_limit = int(self.pending_launch_limit)
        c.persistent = int(self.persistent)
        c.device_loop = int(bool(self.device_loop))
        c.frontier = int(bool(self.frontier))
        c.weight_bits = int(self.weight_bits)
        c.cf_wave = int(self.cf_wave)
        c.col_bits = int(self.col_bits)
        c.threshold, c.cfactor, c.agg_coarsen = self.order_effect(
            c.threshold, c.cfactor, self.agg if agg_on else None)
        return c

    def order_effect(self, threshold: int, cfactor: int,
                     agg: str | None) -> tuple[int, int, int]:
        """What the reference's `transform(order=...)` (pipeline.py:45-81)
        does to the knobs, measured by running it (tests/golden/
        order_counters.json): a disabled pass (T=0, C<=1, no agg) is a no-op
        wherever it sits; an absent step never runs; the threshold pass only
        recognises the original launch, so it is skipped when an active
        coarsen or aggregate step precedes it; a coarsen step after an active
        aggregate step rewrites the aggregated clone instead of the child
        (its logical blocks span parents) -- except at grid granularity,
        whose clone is host-launched, so nothing is coarsened.
        Returns (threshold, cfactor, agg_coarsen)."""
        order = self.order.upper()
        pos = {s: order.index(s) for s in "TCA" if s in order}
        t_on = threshold != 0 and "T" in pos
        c_on = cfactor > 1 and "C" in pos
        a_on = agg is not None and "A" in pos
        if t_on and ((c_on and pos["C"] < pos["T"])
                     or (a_on and pos["A"] < pos["T"])):
            t_on = False
        agg_coarsen = 0
        if c_on and a_on and pos["A"] < pos["C"]:
            if agg == "grid":
                c_on = False
            else:
                agg_coarsen = 1
        return (threshold if t_on else 0, cfactor if c_on else 1,
                agg_coarsen)


class EquivalenceError(AssertionError):
    pass


@dataclass
class ManifestEntry:
    site: str
    pass_name: str
    action: str

    def render(self) -> str:
        return f"site={self.site} pass={self.pass_name} action={self.action}"

    @property
    def transformed(self) -> bool:
        return self.action.startswith("transformed")


@dataclass
class TransformResult:
    """What the reference's pipeline.transform returns, restated as the
    policy the B200 scheduler applied (no source is generated)."""
    config: BenchConfig
    manifest: list = field(default_factory=list)

    def manifest_text(self) -> str:
        return "\n".join(e.render() for e in self.manifest)


def _manifest(bench: Benchmark, cfg: BenchConfig) -> TransformResult:
    site = f"{bench.name}:parent"
    res = TransformResult(cfg)
    order = cfg.order.upper()
    for step in order:
        if step == "T" and cfg.threshold != 0:
            res.manifest.append(ManifestEntry(site, "threshold",
                                              "transformed"))
        elif step == "C" and cfg.cfactor > 1:
            res.manifest.append(ManifestEntry(
                f"{bench.name}:child", "coarsen",
                f"transformed (factor={cfg.cfactor})"))
        elif step == "A" and cfg.agg is not None:
            detail = (f"granularity=multiblock, group={cfg.group_size}"
                      if cfg.agg == "multiblock"
                      else f"granularity={cfg.agg}")
            if cfg.agg_threshold > 0:
                detail += f", direct-launch threshold={cfg.agg_threshold}"
            res.manifest.append(ManifestEntry(site, "aggregate",
                                              f"transformed ({detail})"))
    return res


def load(bench_name: str, dataset: str) -> tuple[Benchmark, Workload]:
    bench = get_benchmark(bench_name)
    return bench, bench.workload(dataset)


def _report(bench: Benchmark, wl: Workload, out: dict, st: dict) -> Report:
    units, alg = bench.traffic(wl, out, st)
    st = dict(st)
    st["work_units"] = units
    st["bytes_alg"] = alg
    kinds = {k: bench.kinds[k] for k in bench.outputs}
    return Report.from_stats(st, {k: out[k] for k in bench.outputs}, kinds)


def run_reference(bench: Benchmark, wl: Workload, cost=None,
                  checked: bool = False) -> Report:
    """Run the serial (No-CDP) variant on the device (harness.py:57-62).

    ``cost``/``checked`` belong to the simulator and are accepted for
    signature compatibility; hardware has no cost model to override."""
    cfg = BenchConfig().to_c(_lib.VARIANT_NOCDP)
    out, st = bench.run(wl, cfg)
    return _report(bench, wl, out, st)


def run_config(bench: Benchmark, wl: Workload, cfg: BenchConfig, cost=None,
               checked: bool = False, schedule_seed: int | None = None
               ) -> tuple[Report, TransformResult]:
    """Run the dynamic (CDP) variant under ``cfg`` (harness.py:65-80).

    ``schedule_seed`` selected a simulated interleaving; on hardware every
    run is a real interleaving and outputs are schedule-invariant."""
    ccfg = cfg.to_c(_lib.VARIANT_CDP)
    out, st = bench.run(wl, ccfg)
    return _report(bench, wl, out, st), _manifest(bench, cfg)


def verify_outputs(bench: Benchmark, wl: Workload, got: Report, ref: Report,
                   label: str = "") -> None:
    """Raise EquivalenceError at the first divergent output element
    (harness.py:83-96).  Floating-point outputs compare within the
    benchmark's tolerance (bt vertices: BT_ABS_TOL absolute; sp surveys:
    1e-5 relative); everything else bit-exactly."""
    for name in bench.outputs:
        g = np.asarray(got.arrays[name])
        r = np.asarray(ref.arrays[name])
        if g.shape[0] != r.shape[0]:
            raise EquivalenceError(
                f"{bench.name}/{wl.spec.text}{label}: buffer '{name}' has "
                f"{g.shape[0]} elements, reference has {r.shape[0]}")
        if g.dtype.kind == "f" or r.dtype.kind == "f":
            rtol, atol = bench.tol
            bad = ~np.isclose(g, r, rtol=rtol, atol=atol)
            if bad.ndim > 1:
                bad = bad.any(axis=tuple(range(1, bad.ndim)))
        else:
            bad = g != r
        idx = np.flatnonzero(bad)
        if idx.size:
            i = int(idx[0])
            gv, rv = g[i].tolist(), r[i].tolist()
            raise EquivalenceError(
                f"{bench.name}/{wl.spec.text}{label}: '{name}'[{i}] = "
                f"{gv} differs from reference {rv}")


def run_benchmark(bench_name: str, dataset: str,
                  cfg: BenchConfig = BenchConfig(), cost=None,
                  checked: bool = False, verify: bool = True) -> Report:
    """One-shot: run ``cfg`` and verify against the serial variant
    (harness.py:99-109)."""
    bench, wl = load(bench_name, dataset)
    report, _ = run_config(bench, wl, cfg, cost=cost, checked=checked)
    if verify:
        ref = run_reference(bench, wl, cost=cost)
        verify_outputs(bench, wl, report, ref, label=f" ({cfg.describe()})")
    return report
