"""Host-side logic and the C-ABI boundary (no GPU needed).

Mirrors the reference's own API tests (tests/test_bench.py) for everything
that does not execute a kernel: dataset specs, knob validation with the
reference's error messages, the sweep schema and fault isolation, the memory
digest formula, and that libdynpar.so loads and exports every symbol the
header declares.
"""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2201_02789_b200 import _lib
from paper_2201_02789_b200.bench import (CSV_COLUMNS, BenchConfig,
                                         EquivalenceError, INF_THRESHOLD,
                                         default_grid, get_benchmark, load,
                                         parse_spec, render_csv, sweep,
                                         verify_outputs)
from paper_2201_02789_b200.bench.report import Report, memory_digest
from paper_2201_02789_b200.bench.sweep import REFERENCE_COLUMNS

from conftest import ROOT


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "dynpar.h").read_text()
    declared = set(re.findall(
        r"^(?:int|int64_t|void|const char\*)\s+(dp_[a-z0-9_]+)\(", header,
        re.M))
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTED)
    assert lib.dp_abi_version() == _lib.ABI_VERSION == 2
    assert f"#define DP_ABI_VERSION {_lib.ABI_VERSION}" in header


_C_TYPES = {"int32_t": ctypes.c_int32, "uint32_t": ctypes.c_uint32,
            "int64_t": ctypes.c_int64, "uint64_t": ctypes.c_uint64,
            "double": ctypes.c_double, "float": ctypes.c_float}


def header_struct(name: str) -> list[tuple[str, object]]:
    """(field, ctypes type) list of `typedef struct name {...} name;` parsed
    from include/dynpar.h (comments stripped; arrays as ctypes arrays)."""
    text = (ROOT / "include" / "dynpar.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), text,
                     re.S).group(1)
    fields = []
    for decl in body.split(";"):
        decl = " ".join(decl.split())
        if not decl:
            continue
        m = re.fullmatch(r"(\w+) (\w+)(?:\[(\d+)\])?", decl)
        assert m, decl
        t = _C_TYPES[m.group(1)]
        fields.append((m.group(2), t * int(m.group(3)) if m.group(3) else t))
    return fields


def same_layout(struct, fields) -> bool:
    got = [(n, t) for n, t in struct._fields_]
    if [n for n, _ in got] != [n for n, _ in fields]:
        return False
    for (_, a), (_, b) in zip(got, fields):
        if ctypes.sizeof(a) != ctypes.sizeof(b) or \
                getattr(a, "_type_", a) != getattr(b, "_type_", b):
            return False
    return True


@pytest.mark.parametrize("name,binding", [("dp_config", "DpConfig"),
                                          ("dp_stats", "DpStats")])
def test_struct_layouts_match_header(name, binding):
    fields = header_struct(name)
    struct = getattr(_lib, binding)
    assert same_layout(struct, fields), (name, struct._fields_, fields)
    # the size the library clears / writes
    class H(ctypes.Structure):
        _fields_ = fields
    assert ctypes.sizeof(struct) == ctypes.sizeof(H)


def test_integration_binding_matches_header():
    """The structs INTEGRATION.md tells a maintainer to paste are the
    header's (a short dp_stats would let the library write past it)."""
    doc = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", doc, re.S)
    abi = [b for b in blocks if "class dp_stats" in b]
    assert len(abi) == 1
    ns: dict = {}
    exec(abi[0], ns)  # noqa: S102 - the documented snippet itself
    for name in ("dp_config", "dp_stats"):
        assert same_layout(ns[name], header_struct(name)), name


def test_no_device_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except ImportError:
        pass
    with pytest.raises(_lib.DeviceTrap) as e:
        _lib.device()
    assert e.value.kind in ("no-device", "cuda-error")


def test_parse_spec_fields():
    s = parse_spec("powerlaw:500:seed3")
    assert (s.kind, s.size, s.seed) == ("powerlaw", 500, 3)
    assert parse_spec("rmat:22:seed1").size == 22
    assert parse_spec("hand").kind == "hand"


@pytest.mark.parametrize("bad,needle", [
    ("zzz:10:seed1", "unknown dataset kind"),
    ("powerlaw", "kind:size:seedN"),
    ("powerlaw:ten:seed1", "size"),
    ("powerlaw:10:7", "seed"),
    ("powerlaw:0:seed1", "size"),
    ("hand:10:seed1", "hand"),
    ("rmat:31:seed1", "scale"),
])
def test_parse_spec_rejects(bad, needle):
    with pytest.raises(ValueError, match=needle):
        parse_spec(bad)


@pytest.mark.parametrize("cfg,needle", [
    (BenchConfig(agg="multiblock", agg_threshold=2),
     "aggregation threshold requires block granularity"),
    (BenchConfig(agg="tile"), "unknown aggregation granularity"),
    (BenchConfig(agg="multiblock", group_size=0),
     "group size must be at least 1"),
    (BenchConfig(threshold=5, order="TXA"), "unknown pass step"),
    (BenchConfig(parent_block=48), "parent_block"),
    (BenchConfig(child_block=16), "child_block"),
    (BenchConfig(serial="lane"), "serial mode"),
    # round-2 B200 knobs
    (BenchConfig(weight_bits=3), "weight_bits"),
    (BenchConfig(cf_wave=-1), "cf_wave"),
    (BenchConfig(col_bits=16), "col_bits"),
    (BenchConfig(persistent=9), "persistent"),
])
def test_knob_validation_matches_reference_errors(cfg, needle):
    with pytest.raises(ValueError, match=needle):
        cfg.to_c()


def test_knob_encoding():
    c = BenchConfig(threshold=128, cfactor=8, agg="multiblock",
                    group_size=4).to_c()
    assert (c.threshold, c.cfactor, c.agg, c.group_size) == (128, 8, 3, 4)
    assert (c.parent_block, c.child_block, c.variant) == (32, 32, 1)
    # disabled passes (pipeline.py:59-73): T<=0, C<=1, agg None
    c = BenchConfig(threshold=-3, cfactor=0).to_c(_lib.VARIANT_NOCDP)
    assert (c.threshold, c.cfactor, c.agg, c.variant) == (0, 1, 0, 0)
    assert BenchConfig(threshold=INF_THRESHOLD).to_c().threshold == 2**31 - 1
    # order without a step disables that step
    c = BenchConfig(threshold=9, cfactor=4, agg="block", order="A").to_c()
    assert (c.threshold, c.cfactor, c.agg) == (0, 1, 2)


def test_default_grid_and_schema():
    grid = default_grid()
    assert len(grid) == 12
    assert [c.agg for c in grid[:4]] == [None, "block", "multiblock", "grid"]
    assert CSV_COLUMNS[:len(REFERENCE_COLUMNS)] == REFERENCE_COLUMNS
    assert REFERENCE_COLUMNS == (
        "bench", "dataset", "threshold", "cfactor", "agg", "group_size",
        "agg_threshold", "num_launches", "host_launches", "blocks_scheduled",
        "instructions", "makespan", "t_parent", "t_launch", "t_agg",
        "t_disagg", "t_child", "error")


def test_sweep_isolates_invalid_rows_without_device():
    rows = sweep("manylaunch", "sizes:40:seed3",
                 configs=[BenchConfig(agg="multiblock", agg_threshold=4)],
                 verify=False)
    assert "aggregation threshold requires block granularity" in \
        rows[0]["error"]
    assert rows[0]["makespan"] == ""
    text = render_csv(rows)
    assert text.splitlines()[0] == ",".join(CSV_COLUMNS)


def test_unknown_benchmark():
    with pytest.raises(ValueError, match="unknown benchmark"):
        get_benchmark("mst")


def test_memory_digest_matches_reference_formula(golden, golden_arrays):
    rec = next(r for r in golden["reference"]
               if r["bench"] == "bfs" and r["dataset"] == "powerlaw:150:seed2")
    arrays = {k: golden_arrays[f"ref/bfs/powerlaw:150:seed2/{k}"]
              for k in ("dist", "counts")}
    assert memory_digest(arrays, {"dist": "int", "counts": "int"}) == \
        rec["digest"]


def _fake_report(arrays):
    st = {k: 0 for k, _ in _lib.DpStats._fields_}
    st["ns_phase"] = [0.0] * 5
    return Report.from_stats(st, arrays, {k: "int" for k in arrays})


def test_verify_outputs_names_first_divergent_element():
    bench, wl = load("manylaunch", "sizes:20:seed2")
    ref = _fake_report({"out": np.arange(20, dtype=np.int32),
                        "total": np.array([7], np.int32)})
    got = _fake_report({"out": np.arange(20, dtype=np.int32),
                        "total": np.array([7], np.int32)})
    verify_outputs(bench, wl, got, ref)
    got.arrays["out"][3] += 1
    with pytest.raises(EquivalenceError, match=r"'out'\[3\]") as exc:
        verify_outputs(bench, wl, got, ref)
    assert "differs from reference" in str(exc.value)
    assert "manylaunch/sizes:20:seed2" in str(exc.value)


def test_report_text_and_lists():
    r = _fake_report({"dist": np.array([0, 1, 1 << 30], np.int32)})
    assert r.buffers["dist"] == [0, 1, 1 << 30]
    text = r.to_text(include_buffers=True)
    assert "buffer dist = 0 1 1073741824" in text
    assert text.splitlines()[0] == "num_launches=0"


def test_report_phase_times_and_pending_depth():
    # dp_stats.ns_phase -> SimReport.phase_time / t_* lines (sim/report.py:
    # 12-50); max_pending_depth passes through
    st = {k: 0 for k, _ in _lib.DpStats._fields_}
    st["ns_phase"] = [10.0, 20.4, 30.0, 40.0, 50.0]
    st["max_pending_depth"] = 3
    r = Report.from_stats(st, {"x": np.zeros(1, np.int32)}, {"x": "int"})
    assert r.phase_time == {"parent": 10, "launch": 20, "agg": 30,
                            "disagg": 40, "child": 50}
    assert r.max_pending_depth == 3
    text = r.to_text()
    assert "t_launch=20" in text and "max_pending_depth=3" in text


def test_profiled_build_target_exists():
    mk = (Path(__file__).resolve().parents[1] / "paper_2201_02789_b200" /
          "csrc" / "Makefile").read_text()
    assert "libdynpar_prof.so" in mk and "-DDP_PROFILE=1" in mk


def _order_rows():
    import json
    return json.loads((ROOT / "tests" / "golden" /
                       "order_counters.json").read_text())


def test_order_effect_matches_reference_manifest():
    """BenchConfig.order reproduces what the reference's transform(order=)
    did (pipeline.py:45-81), pass by pass, on every golden row: which
    threshold pass transformed or was skipped, and whether coarsening hit
    the child, the aggregated clone, or nothing."""
    rows = _order_rows()
    assert len(rows) == 320
    for row in rows:
        cfg = BenchConfig(order=row["order"], **row["config"])
        c = cfg.to_c()
        man = row["manifest"]
        t_done = any("pass=threshold action=transformed" in e for e in man)
        coarse = [e.split()[0] for e in man
                  if "pass=coarsen action=transformed" in e]
        assert (c.threshold > 0) == t_done, (row["order"], row["config"], man)
        if not coarse:
            assert c.cfactor == 1 and c.agg_coarsen == 0, (row, c.cfactor)
        else:
            assert c.cfactor == row["config"]["cfactor"]
            assert bool(c.agg_coarsen) == coarse[0].endswith("_agg"), row


def test_order_rejects_unknown_step():
    # pipeline.py:79 / tests/test_passes.py:672-674
    with pytest.raises(ValueError, match="unknown pass step"):
        BenchConfig(threshold=5, order="TXA").to_c()


def test_register_benchmark_plugin_contract():
    """register_benchmark (the reference's Benchmark registration,
    bench/benchmarks.py:56-68): validation, then every harness entry point
    serves the new name."""
    from paper_2201_02789_b200.bench import (BENCHMARKS, Benchmark,
                                             register_benchmark)
    base = BENCHMARKS["bfs"]
    with pytest.raises(ValueError, match="already registered"):
        register_benchmark(base)
    with pytest.raises(ValueError, match="element kind"):
        register_benchmark(Benchmark("bfs_x", ("dist", "zz"), {"dist": "int"},
                                     base.prepare, base.run, base.traffic))
    b = Benchmark("bfs_copy", base.outputs, base.kinds, base.prepare,
                  base.run, base.traffic, "plug-in test")
    try:
        register_benchmark(b)
        bench, wl = load("bfs_copy", "hand")
        assert bench is b and wl.n > 0
    finally:
        BENCHMARKS.pop("bfs_copy", None)
