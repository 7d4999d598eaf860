"""Experiment CLI against the reference CLI's own CSVs.

``tests/golden/cli/*.csv`` were written by the reference's ``sincfft.cli.main``
(``tests/golden/make_cli_golden.py``) with the arguments in ``CASES`` below.
The B200 CLI must reproduce the schema, the row order, every parameter and
bound column (host scalars: 1e-12 relative) and the measured errors (GPU
transforms and GPU exact sums vs the reference's CPU ones: both measure the
same approximation error of the same draws, so they agree to rounding noise
of order 1e-15 relative to ||f||_1).  The contract tests mirror the
reference's ``tests/test_cli.py``: byte determinism, the optional time
column, the direct-oracle cap, and exit codes.
"""

import csv
import os

import pytest

from paper_2107_02671_b200.cli import main

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli")

CASES = {
    "nnfft_error": ["nnfft-error", "--N", "64", "--M1", "16", "--M2", "16", "--m1", "2", "4",
                    "--sigma1", "1.5", "2.0", "--reps", "3", "--seed", "5"],
    "nnfft_error_m2": ["nnfft-error", "--N", "32", "--M1", "40", "--M2", "24", "--m1", "3",
                       "--m2", "5", "--sigma1", "1.25", "--reps", "2", "--seed", "99"],
    "sinc_approx": ["sinc-approx", "--N", "16", "32", "--nu", "4", "5", "--R", "2000"],
    "sinc_transform": ["sinc-transform", "--N", "32", "64", "--nu", "4", "--reps", "2",
                       "--seed", "11"],
    "bounds_small": ["bounds", "--N", "128", "--m1", "4", "6", "--sigma1", "2.0",
                     "--nu", "4", "6"],
    "bounds_default": ["bounds"],
}
MEASURED = {"measured"}


def _read(path):
    lines = open(path, encoding="utf-8").read().splitlines()
    assert lines[0] == "# schema=1"
    return lines[1].split(","), list(csv.DictReader(lines[1:]))


def _compare(name, tmp_path):
    out = tmp_path / f"{name}.csv"
    assert main(CASES[name] + ["--out", str(out)]) == 0
    hdr, rows = _read(out)
    ghdr, grows = _read(os.path.join(GOLD, f"{name}.csv"))
    assert hdr == ghdr
    assert len(rows) == len(grows)
    for row, gold in zip(rows, grows):
        for col in hdr:
            a, b = row[col], gold[col]
            if a == b:
                continue
            assert a != "" and b != "", (name, col, a, b)
            fa, fb = float(a), float(b)
            if col in MEASURED:
                assert abs(fa - fb) <= 1e-14 + 1e-3 * abs(fb), (name, col, fa, fb)
            else:
                assert abs(fa - fb) <= 1e-12 * abs(fb), (name, col, fa, fb)
    return out


# ---------------------------------------------------------------- host only
@pytest.mark.parametrize("name", ["bounds_small", "bounds_default"])
def test_bounds_table_matches_reference(name, tmp_path):
    _compare(name, tmp_path)


def test_bounds_deterministic_bytes(tmp_path):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert main(CASES["bounds_small"] + ["--out", str(a)]) == 0
    assert main(CASES["bounds_small"] + ["--out", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()


def test_usage_error_exits_two():
    with pytest.raises(SystemExit) as info:
        main(["no-such-command"])
    assert info.value.code == 2


def test_bounds_parameter_error_exits_two(tmp_path):
    # sigma outside the sinh range is a ParameterError -> exit code 2
    assert main(["bounds", "--sigma1", "3.0", "--out", str(tmp_path / "x.csv")]) == 2


# ---------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["nnfft_error", "nnfft_error_m2", "sinc_approx",
                                  "sinc_transform"])
def test_cli_matches_reference(name, tmp_path):
    _compare(name, tmp_path)


@pytest.mark.gpu
def test_nnfft_error_deterministic_bytes_and_bound(tmp_path):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    args = ["nnfft-error", "--N", "32", "--M1", "10", "--M2", "12", "--m1", "3",
            "--sigma1", "2.0", "--reps", "1", "--seed", "99"]
    assert main(args + ["--out", str(a)]) == 0
    assert main(args + ["--out", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()
    _, rows = _read(a)
    assert float(rows[0]["measured"]) <= float(rows[0]["bound"])


@pytest.mark.gpu
def test_seed_changes_measurement(tmp_path):
    args = ["nnfft-error", "--N", "64", "--M1", "16", "--M2", "16", "--m1", "4",
            "--sigma1", "2.0", "--reps", "3"]
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    main(args + ["--seed", "5", "--out", str(a)])
    main(args + ["--seed", "6", "--out", str(b)])
    assert _read(a)[1][0]["measured"] != _read(b)[1][0]["measured"]


@pytest.mark.gpu
def test_time_column_optional(tmp_path):
    out = tmp_path / "t.csv"
    main(["nnfft-error", "--N", "32", "--M1", "8", "--M2", "8", "--m1", "3", "--sigma1", "2.0",
          "--reps", "1", "--time", "--out", str(out)])
    hdr, rows = _read(out)
    assert hdr[-1] == "time_s" and float(rows[0]["time_s"]) > 0.0


@pytest.mark.gpu
def test_sinc_transform_direct_cap(tmp_path):
    out = tmp_path / "capped.csv"
    assert main(["sinc-transform", "--N", "64", "--nu", "4", "--reps", "1", "--direct-cap", "32",
                 "--out", str(out)]) == 0
    row = _read(out)[1][0]
    assert row["measured"] == ""  # exact sum skipped above the cap
    assert row["assump_ok"] == "1" and float(row["epsilon"]) <= float(row["bound_full"])


@pytest.mark.gpu
def test_exit_codes_on_gpu_paths(tmp_path):
    # sigma outside the sinh range and (B200 deviation) non-sinh windows -> 2
    assert main(["nnfft-error", "--N", "32", "--M1", "4", "--M2", "4", "--m1", "3",
                 "--sigma1", "3.0", "--reps", "1", "--out", str(tmp_path / "x.csv")]) == 2
    assert main(["nnfft-error", "--N", "32", "--M1", "8", "--M2", "8", "--m1", "4",
                 "--sigma1", "2.0", "--window1", "bspline", "--window2", "bspline",
                 "--reps", "1", "--out", str(tmp_path / "y.csv")]) == 2
