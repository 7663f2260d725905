"""Command line: ``python -m paper_2201_02789_b200 sweep ...``.

Flag-compatible with the ``sweep`` subcommand of ``dynoptc``
(pkg/src/dynoptc/cli.py:139-165 flags, 345-367 behaviour): the same list
flags and spellings (``inf`` thresholds, ``none`` granularity), the same CSV
(reference columns first, measured B200 columns after), the CSV on stdout or
in ``--report``, one line per failed row on stderr and exit status 1 when any
row failed.  The compiler subcommands (``emit`` / ``run``) are out of scope
(DESIGN.md §1): the kernels here are written, not emitted.

    python -m paper_2201_02789_b200 sweep --bench bfs \\
        --dataset rmat:16:seed1 --thresholds 0,128,inf --aggs none,block
"""

from __future__ import annotations

import argparse
import sys
from typing import Callable

from .bench import BenchConfig, INF_THRESHOLD, render_csv, sweep, write_csv
from .bench.harness import GRANULARITIES

PROG = "paper_2201_02789_b200"


class CliError(Exception):
    """A usage problem reported as ``PROG: error: ...`` with status 1."""


def _threshold(token: str) -> int:
    word = token.strip().lower()
    if word in ("inf", "infinity"):
        return INF_THRESHOLD
    if not word.lstrip("-").isdigit():
        raise argparse.ArgumentTypeError(
            f"threshold must be an integer or 'inf', got {token!r}")
    if int(word) < 0:
        raise argparse.ArgumentTypeError("threshold must be >= 0")
    return int(word)


def _granularity(token: str):
    word = token.strip().lower()
    if word in ("", "none"):
        return None
    if word in GRANULARITIES:
        return word
    raise argparse.ArgumentTypeError(
        f"aggregation granularity must be one of {', '.join(GRANULARITIES)} "
        f"or 'none', got {token!r}")


def _listed(item: Callable) -> Callable[[str], list]:
    """Comma-separated list of ``item`` values (empty entries skipped)."""
    return lambda text: [item(t) for t in text.split(",") if t.strip()]


# grid axes (one BenchConfig per combination) and per-sweep knobs:
# (flag, type, default, metavar, help)
_AXES = (
    ("--thresholds", _listed(_threshold), [0, 32, INF_THRESHOLD], "N,...",
     "thresholds T (integers or inf)"),
    ("--cfactors", _listed(_threshold), [1], "F,...", "coarsening factors C"),
    ("--aggs", _listed(_granularity), [None, "block", "multiblock", "grid"],
     "G,...", "aggregation granularities A (or none)"),
)
_KNOBS = (
    ("--group-size", int, 4, "G", "multiblock group size"),
    ("--agg-threshold", int, 0, "N", "aggregation threshold (block only)"),
)
_B200_KNOBS = (
    ("--parent-block", int, 32, "B", "parent grid block size"),
    ("--child-block", int, 32, "B", "child grid block size"),
)


def build_parser() -> argparse.ArgumentParser:
    top = argparse.ArgumentParser(
        prog=PROG, description="Sweep the nested-parallel (CDP2 + T/C/A) "
                               "kernels on a B200.")
    cmds = top.add_subparsers(dest="command", required=True)
    p = cmds.add_parser("sweep", help="run a benchmark across a grid of "
                                      "configurations")
    p.add_argument("--bench", required=True,
                   help="benchmark name (bfs, sssp, manylaunch, tc, bt, ...)")
    p.add_argument("--dataset", required=True, metavar="SPEC",
                   help="dataset spec, e.g. rmat:16:seed1")
    p.add_argument("--report", metavar="CSV", default=None,
                   help="write the CSV here instead of stdout")
    for flag, typ, default, metavar, help_ in _AXES + _KNOBS:
        p.add_argument(flag, type=typ, default=default, metavar=metavar,
                       help=help_)
    p.add_argument("--cost", metavar="K=V,...", default="",
                   help="accepted for compatibility (hardware has no cost "
                        "model)")
    p.add_argument("--no-verify", action="store_true",
                   help="do not check outputs against the serial variant")
    b200 = p.add_argument_group("B200 knobs")
    for flag, typ, default, metavar, help_ in _B200_KNOBS:
        b200.add_argument(flag, type=typ, default=default, metavar=metavar,
                          help=help_)
    b200.add_argument("--serial", choices=("thread", "warp"),
                      default="thread", help="serial arm mode")
    return top


def _grid(args) -> list[BenchConfig]:
    shared = dict(group_size=args.group_size,
                  agg_threshold=args.agg_threshold,
                  parent_block=args.parent_block,
                  child_block=args.child_block, serial=args.serial)
    return [BenchConfig(threshold=t, cfactor=c, agg=a, **shared)
            for t in args.thresholds for c in args.cfactors
            for a in args.aggs]


def _emit(args, rows: list[dict]) -> None:
    if args.report is None:
        sys.stdout.write(render_csv(rows))
        return
    try:
        write_csv(args.report, rows)
    except OSError as e:
        raise CliError(f"cannot write '{args.report}': {e.strerror or e}") \
            from None
    print(f"wrote {args.report} ({len(rows)} rows)", file=sys.stderr)


def run_sweep(args) -> int:
    try:
        rows = sweep(args.bench, args.dataset, configs=_grid(args),
                     verify=not args.no_verify)
    except ValueError as e:  # unknown benchmark / bad dataset spec
        raise CliError(str(e)) from None
    _emit(args, rows)
    status = 0
    for row in rows:
        if row["error"]:
            status = 1
            print(f"row {row['threshold']}/{row['cfactor']}/{row['agg']}: "
                  f"{row['error']}", file=sys.stderr)
    return status


COMMANDS = {"sweep": run_sweep}


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as e:  # argparse already printed the usage error
        return int(e.code or 0)
    try:
        return COMMANDS[args.command](args)
    except (CliError, ValueError) as e:
        print(f"{PROG}: error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
