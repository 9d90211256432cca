"""``python -m paper_2601_17091_b200 transform`` — the reference's
``gridrocket transform`` subcommand (cli.py:138-168, flags cli.py:84-94 and
299-310) on the CUDA backend, streaming through rk_transform_stream
(paper_2601_17091_b200.stream).  The output feature file is byte-identical
to the reference's for the same dataset, bank and precision (mode "exact").
Exit codes follow cli.py:365-377: 3 on CapacityError, 2 on parse / format /
value / OS errors.

Only the transform subcommand is provided; the reference's gen-kernels, fit,
predict, bench, report and synth commands are outside the hot path
(DESIGN.md §6).
"""

import argparse
import sys
import time

from .binio import FormatError
from .data import ParseError
from .engine import CapacityError, GridLimits
from .features import FeatureMatrix
from .kernels import GenOptions, KernelBank, generate_bank
from .stream import transform_file

# key = value config file keys and their types (cli.py:24-34)
CONFIG_KEYS = {
    "precision": str,
    "workers_per_cell": int,
    "max_x": int,
    "max_y": int,
    "memory_budget_bytes": int,
    "devices": int,
}


def load_config(path) -> dict:
    """``key = value`` lines, '#' comments (cli.py:36-53)."""
    config = {}
    with open(path) as f:
        for lineno, raw in enumerate(f, start=1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ParseError(f"expected key = value, got {line!r}", lineno)
            key, value = (part.strip() for part in line.split("=", 1))
            if key not in CONFIG_KEYS:
                raise ParseError(f"unknown config key {key!r}", lineno)
            try:
                config[key] = CONFIG_KEYS[key](value)
            except ValueError:
                raise ParseError(f"bad value for {key!r}: {value!r}", lineno) from None
    return config


def engine_settings(args) -> dict:
    """Defaults, then the config file, then explicit flags (cli.py:56-72)."""
    settings = {
        "precision": "single",
        "workers_per_cell": 1024,
        "max_x": 2**31 - 1,
        "max_y": 65535,
        "memory_budget_bytes": 1 << 30,
        "devices": 1,
    }
    if getattr(args, "config", None):
        settings.update(load_config(args.config))
    for key in settings:
        value = getattr(args, key, None)
        if value is not None:
            settings[key] = value
    return settings


def _dataset_dims(path, csv_labels):
    from .data import cache_layout, load_dataset
    from .stream import _is_cache_path

    if _is_cache_path(path):
        layout = cache_layout(path)
        return layout.n_channels, layout.l_series, path
    ds = load_dataset(path, csv_labels=csv_labels)
    return ds.n_channels, ds.l_series, ds


def cmd_transform(args) -> int:
    settings = engine_settings(args)
    n_channels, l_series, source = _dataset_dims(args.data, args.csv_labels)
    if args.bank:
        bank = KernelBank.load(args.bank)
    else:
        if args.kernels is None:
            raise ValueError("either --bank or --kernels is required")
        bank = generate_bank(l_series, n_channels, args.kernels,
                             GenOptions(center_weights=not args.no_center, seed=args.seed))
    limits = GridLimits(max_x=settings["max_x"], max_y=settings["max_y"],
                        workers_per_cell=settings["workers_per_cell"],
                        memory_budget_bytes=settings["memory_budget_bytes"])
    start = time.perf_counter()
    transform_file(source, bank, args.out, limits=limits, include_mpv=args.mpv, precision=settings["precision"],
                   mode=args.mode, device=args.device, devices=settings["devices"])
    elapsed = time.perf_counter() - start
    if args.csv:
        FeatureMatrix.load(args.out).to_csv(args.csv)
    fpk = 3 if args.mpv else 2
    print(
        f"transformed {_count_rows(args.out)} instances x {bank.count * fpk} features "
        f"({settings['precision']}) in {elapsed:.3f}s -> {args.out}"
    )
    return 0


def _count_rows(path) -> int:
    from .binio import read_header, read_values
    from .features import FEATURE_HEADER_FMT, FEATURE_MAGIC, FEATURE_VERSION

    with open(path, "rb") as f:
        read_header(f, FEATURE_MAGIC, FEATURE_VERSION)
        return int(read_values(f, FEATURE_HEADER_FMT)[0])


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2601_17091_b200", description="B200 ROCKET transform")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("transform", help="extract features from a dataset")
    p.add_argument("--data", required=True, help="binary dataset cache (RKDS) or .npy array path")
    p.add_argument("--csv-labels", action="store_true", help=argparse.SUPPRESS)  # reference flag; text input is out of scope
    p.add_argument("--bank", help="load kernels from this bank file")
    p.add_argument("--kernels", type=int, help="generate this many kernels instead")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-center", action="store_true")
    p.add_argument("--mpv", action="store_true", help="add the mean-of-positives feature")
    p.add_argument("--out", required=True, help="feature matrix output path")
    p.add_argument("--csv", help="also export features as CSV")
    p.add_argument("--config", help="key = value config file")
    p.add_argument("--precision", choices=["single", "double"], default=None)
    p.add_argument("--workers", dest="workers_per_cell", type=int, default=None)
    p.add_argument("--max-x", dest="max_x", type=int, default=None)
    p.add_argument("--max-y", dest="max_y", type=int, default=None)
    p.add_argument("--memory-budget", dest="memory_budget_bytes", type=int, default=None)
    p.add_argument("--devices", type=int, default=None)
    p.add_argument("--backend", choices=["cuda"], default="cuda", help="compute backend (CUDA only)")
    p.add_argument("--mode", choices=["exact", "fast"], default="exact",
                   help="exact: byte-identical to the reference; fast: FFMA2 within 1e-5")
    p.add_argument("--device", type=int, default=0, help="first GPU")
    p.set_defaults(func=cmd_transform)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except CapacityError as exc:
        print(f"capacity error: {exc}", file=sys.stderr)
        return 3
    except (ParseError, FormatError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
