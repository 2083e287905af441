"""The C oracle under AddressSanitizer + UndefinedBehaviorSanitizer (CPU).

tests/csrc/oracle_sanitize.c drives oracle/nrmf_oracle.c over every length
0..300 (ragged tails, the empty input), both dtypes and both tops, a
multi-tile input, the tile API, ragged / padded / empty column sets and the
exact reference, with a few closed-form checks; any out-of-bounds access,
leak or undefined behaviour aborts the run (-fno-sanitize-recover)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_oracle_clean_under_asan_ubsan(tmp_path):
    exe = tmp_path / "oracle_sanitize"
    cmd = ["gcc", "-std=c11", "-O1", "-g", "-ffp-contract=off", "-fsanitize=address,undefined",
           "-fno-sanitize-recover=all", "-o", str(exe), os.path.join(ROOT, "tests", "csrc", "oracle_sanitize.c"),
           os.path.join(ROOT, "oracle", "nrmf_oracle.c"), "-lm"]
    try:
        subprocess.run(cmd, check=True, capture_output=True, text=True)
    except (FileNotFoundError, subprocess.CalledProcessError) as e:
        pytest.skip(f"no gcc sanitizer runtime: {e}")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "ASAN_OPTIONS": "detect_leaks=1"})
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok" in r.stdout
