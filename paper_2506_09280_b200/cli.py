"""`check` front end with the reference CLI's contract (cli.py:100-111, 276-293).

    python -m paper_2506_09280_b200.cli check --ref R --cand C --tol T [--k 3.0] [--json|--text]

Traces are read straight into HBM (read_trace(device="cuda")), compared on
the GPU, and the report is printed byte-identically to the reference's.
Exit codes: 0 clean, 1 usage/config/file errors, 2 tolerance flags,
3 replica or merge failures, 4 trace-format or run-compatibility errors.
The emulator commands (simulate, estimate-tol, sweep) are out of scope: on
B200 traces come from the real run (torchtap) and tolerances from
checker.estimate_tolerance with runner.torch_runner.
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

from .checker import ToleranceMap, check, render_report
from .errors import ConfigInvalid, DigestMismatch, FormatError, TraindiffError
from .tensor import POLICIES


def _resolve(path: str) -> Path:
    base = os.environ.get("TRAINDIFF_OUT")
    p = Path(path)
    return Path(base) / p if base and not p.is_absolute() else p


def _format_of(trace):
    model = trace.header.get("model")
    precision = model.get("precision") if isinstance(model, dict) else None
    if precision not in POLICIES:
        raise FormatError(f"trace header lacks a known model precision (got {precision!r})")
    return POLICIES[precision].storage


def _hbm_fits(paths) -> bool:
    """Reading a file to HBM holds its image and its unpacked payload arena
    (about the file size each) until the unpack ends; the first trace's
    arena stays while the second is read.  Peak ~ sum(sizes) + max(size)."""
    import torch
    if not torch.cuda.is_available():
        return False
    sizes = [p.stat().st_size for p in paths]
    free, _ = torch.cuda.mem_get_info()
    return sum(sizes) + max(sizes) + (256 << 20) <= free


def _cmd_check(args) -> int:
    from .tracestore import read_trace
    paths = [_resolve(args.ref), _resolve(args.cand)]
    # device reads unless asked otherwise or the traces would not fit in HBM
    # (then the host path: payloads are staged to the device by check())
    device = None if args.host or not _hbm_fits(paths) else "cuda"
    ref = read_trace(paths[0], device=device)
    cand = read_trace(paths[1], device=device)
    try:
        blob = _resolve(args.tol).read_bytes()
    except OSError as exc:
        raise ConfigInvalid(f"--tol: {exc}")
    tol = ToleranceMap.from_json(blob)
    report = check(ref, cand, tol, kappa=args.k, fmt=_format_of(cand))
    out = render_report(report, "json" if args.json else "text")
    sys.stdout.write(out if out.endswith("\n") else out + "\n")
    return report.exit_code()


class _Parser(argparse.ArgumentParser):
    def error(self, message):          # 2 means "flags" here, so usage errors exit 1
        self.exit(1, f"{self.prog}: error: {message}\n")


def _parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="traindiff-b200",
                     epilog="exit codes: 0 clean, 1 usage/config, 2 flags, "
                            "3 replica/merge failures, 4 format errors")
    sub = parser.add_subparsers(metavar="command")
    chk = sub.add_parser("check", help="compare a candidate trace to the reference")
    chk.add_argument("--ref", required=True)
    chk.add_argument("--cand", required=True)
    chk.add_argument("--tol", required=True)
    chk.add_argument("--k", type=float, default=3.0)
    chk.add_argument("--host", action="store_true",
                     help="read payloads to host memory first (they are uploaded during check); "
                          "the default reads them straight to HBM when both traces fit there "
                          "(peak ~ ref + cand + the larger file), else falls back to this")
    view = chk.add_mutually_exclusive_group()
    view.add_argument("--json", action="store_true")
    view.add_argument("--text", action="store_true")
    chk.set_defaults(func=_cmd_check)
    return parser


def main(argv=None) -> int:
    parser = _parser()
    args = parser.parse_args(argv)
    if not hasattr(args, "func"):
        parser.print_help()
        return 1
    try:
        return args.func(args)
    except (FormatError, DigestMismatch) as exc:
        print(f"traindiff: {exc}", file=sys.stderr)
        return 4
    except TraindiffError as exc:
        print(f"traindiff: {exc}", file=sys.stderr)
        return 1
    except OSError as exc:
        print(f"traindiff: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
