"""``sweep`` command line, compatible with ``dynoptc sweep``
(pkg/src/dynoptc/cli.py:139-165, 345-367): same flags, same CSV (the
reference's 18 columns first, measured B200 columns after), exit code 1 when
any row failed.  B200 knobs: --parent-block, --child-block, --serial.

    python -m paper_2201_02789_b200.cli sweep --bench bfs \\
        --dataset rmat:16:seed1 --thresholds 0,128,inf --aggs none,block
"""

from __future__ import annotations

import argparse
import sys

from .bench import (BenchConfig, INF_THRESHOLD, render_csv, write_csv)
from .bench import sweep as bench_sweep
from .bench.harness import GRANULARITIES


class CliError(Exception):
    pass


def _threshold_value(text: str) -> int:
    t = text.strip().lower()
    if t in ("inf", "infinity"):
        return INF_THRESHOLD
    try:
        v = int(t)
    except ValueError:
        raise argparse.ArgumentTypeError(
            f"threshold must be an integer or 'inf', got {text!r}") from None
    if v < 0:
        raise argparse.ArgumentTypeError("threshold must be >= 0")
    return v


def _int_list(text: str) -> list[int]:
    return [_threshold_value(t) for t in text.split(",") if t.strip()]


def _agg_value(text: str):
    t = text.strip().lower()
    if t in ("", "none"):
        return None
    if t not in GRANULARITIES:
        raise argparse.ArgumentTypeError(
            f"aggregation granularity must be one of "
            f"{', '.join(GRANULARITIES)} or 'none', got {text!r}")
    return t


def _agg_list(text: str) -> list:
    return [_agg_value(t) for t in text.split(",") if t.strip()]


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="paper_2201_02789_b200",
        description="Sweep the nested-parallel (CDP2 + T/C/A) kernels on a "
                    "B200.")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("sweep",
                       help="run a benchmark across a configuration grid")
    p.add_argument("--bench", required=True,
                   help="benchmark name (bfs, sssp, manylaunch, tc, bt)")
    p.add_argument("--dataset", required=True, metavar="SPEC",
                   help="dataset spec, e.g. rmat:16:seed1")
    p.add_argument("--report", metavar="CSV", default=None,
                   help="write the CSV here instead of stdout")
    p.add_argument("--thresholds", type=_int_list,
                   default=[0, 32, INF_THRESHOLD], metavar="N,...")
    p.add_argument("--cfactors", type=_int_list, default=[1],
                   metavar="F,...")
    p.add_argument("--aggs", type=_agg_list,
                   default=[None, "block", "multiblock", "grid"],
                   metavar="G,...")
    p.add_argument("--group-size", type=int, default=4, metavar="G")
    p.add_argument("--agg-threshold", type=int, default=0, metavar="N")
    p.add_argument("--cost", metavar="K=V,...", default="",
                   help="accepted for compatibility; hardware has no cost "
                        "model")
    p.add_argument("--no-verify", action="store_true",
                   help="skip checking outputs against the serial variant")
    g = p.add_argument_group("B200 knobs")
    g.add_argument("--parent-block", type=int, default=32)
    g.add_argument("--child-block", type=int, default=32)
    g.add_argument("--serial", choices=("thread", "warp"), default="thread")
    return parser


def _cmd_sweep(args) -> int:
    configs = [BenchConfig(threshold=t, cfactor=c, agg=a,
                           group_size=args.group_size,
                           agg_threshold=args.agg_threshold,
                           parent_block=args.parent_block,
                           child_block=args.child_block, serial=args.serial)
               for t in args.thresholds for c in args.cfactors
               for a in args.aggs]
    try:
        rows = bench_sweep(args.bench, args.dataset, configs=configs,
                           verify=not args.no_verify)
    except ValueError as e:
        raise CliError(str(e)) from None
    if args.report is not None:
        try:
            write_csv(args.report, rows)
        except OSError as e:
            raise CliError(f"cannot write '{args.report}': "
                           f"{e.strerror or e}") from None
        print(f"wrote {args.report} ({len(rows)} rows)", file=sys.stderr)
    else:
        sys.stdout.write(render_csv(rows))
    failed = [r for r in rows if r["error"]]
    for r in failed:
        print(f"row {r['threshold']}/{r['cfactor']}/{r['agg']}: "
              f"{r['error']}", file=sys.stderr)
    return 1 if failed else 0


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0)
    try:
        return {"sweep": _cmd_sweep}[args.command](args)
    except (CliError, ValueError) as e:
        print(f"paper_2201_02789_b200: error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
