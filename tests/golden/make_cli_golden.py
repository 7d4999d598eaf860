"""Golden CSVs for the experiment CLI, produced by the REFERENCE's own CLI.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cli_golden.py

Each case runs ``sincfft.cli.main`` (reference ``pkg/src/sincfft/cli.py``) with
small arguments and stores the CSV under ``tests/golden/cli/<name>.csv``;
``tests/test_cli.py`` runs the B200 CLI with the same arguments and compares
(bound columns to 1e-12 relative, measured errors to the GPU/CPU rounding
noise).  Tests never import the reference.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
from sincfft.cli import main  # noqa: E402  (the reference itself)

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

if __name__ == "__main__":
    out_dir = os.path.join(HERE, "cli")
    os.makedirs(out_dir, exist_ok=True)
    for name, args in CASES.items():
        rc = main(args + ["--out", os.path.join(out_dir, name + ".csv")])
        assert rc == 0, (name, rc)
