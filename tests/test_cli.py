"""CLI host logic (no GPU): config-file parsing and flag precedence as in the
reference's cli (cli.py:36-72), argument surface of `transform`
(cli.py:299-310), and the exit codes for errors raised before any device
work (cli.py:365-377)."""

import argparse
import os

import pytest

from paper_2601_17091_b200.cli import build_parser, engine_settings, load_config, main
from paper_2601_17091_b200.data import ParseError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "formats")


def test_load_config(tmp_path):
    p = tmp_path / "c.conf"
    p.write_text("# comment\nprecision = double\nmax_x = 7  # trailing\n\ndevices=2\n")
    assert load_config(p) == {"precision": "double", "max_x": 7, "devices": 2}


@pytest.mark.parametrize("text,line", [("bogus\n", 1), ("a = 1\n", 1), ("\nmax_x = seven\n", 2)])
def test_load_config_errors(tmp_path, text, line):
    p = tmp_path / "c.conf"
    p.write_text(text)
    with pytest.raises(ParseError) as err:
        load_config(p)
    assert err.value.line == line


def test_settings_precedence(tmp_path):
    p = tmp_path / "c.conf"
    p.write_text("precision = double\nmax_y = 99\n")
    args = build_parser().parse_args(["transform", "--data", "x", "--out", "y", "--config", str(p), "--max-y", "5"])
    s = engine_settings(args)
    assert s["precision"] == "double" and s["max_y"] == 5 and s["devices"] == 1
    args = argparse.Namespace(config=None, precision=None)
    assert engine_settings(args)["precision"] == "single"


def test_transform_flags():
    args = build_parser().parse_args(["transform", "--data", "d.ts", "--kernels", "10", "--out", "o", "--mpv",
                                      "--mode", "fast", "--devices", "2", "--backend", "cuda"])
    assert args.kernels == 10 and args.mpv and args.mode == "fast" and args.devices == 2
    with pytest.raises(SystemExit):
        build_parser().parse_args(["transform", "--data", "d", "--out", "o", "--backend", "cpu"])


def test_exit_codes_before_device_work(tmp_path, capsys):
    # text datasets are out of scope -> ValueError -> 2
    (tmp_path / "bad.ts").write_text("@data\n1,2,x\n")
    assert main(["transform", "--data", str(tmp_path / "bad.ts"), "--kernels", "2", "--out",
                 str(tmp_path / "o")]) == 2
    assert "not read by this package" in capsys.readouterr().err
    # neither --bank nor --kernels -> 2
    assert main(["transform", "--data", os.path.join(GOLDEN, "two_class.rkds"), "--out", str(tmp_path / "o")]) == 2
    # missing file -> 2 (OSError)
    assert main(["transform", "--data", str(tmp_path / "nope.rkds"), "--kernels", "2", "--out",
                 str(tmp_path / "o")]) == 2


def test_capacity_error_exits_3(tmp_path, capsys):
    """The reference's test_capacity_error_exits_3: a memory budget smaller
    than one series is a CapacityError (plan_batches, engine.py:111-115),
    exit code 3, raised before any device work (so it holds without a GPU)."""
    out = tmp_path / "o.rkfm"
    assert main(["transform", "--data", os.path.join(GOLDEN, "two_class.rkds"), "--kernels", "4",
                 "--memory-budget", "16", "--out", str(out)]) == 3
    assert "capacity error" in capsys.readouterr().err
    assert not out.exists()
