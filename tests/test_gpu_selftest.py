"""The GPU selftest verb (tests/selftest.py): the reference's 144-instance
oracle-equivalence grid with the B200 kernels, CSV schema and exit codes of
the reference CLI (main.cpp:144-164,223-226)."""
import io
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import selftest  # noqa: E402


def test_usage_errors_exit_2():
    assert selftest.main(["--seq-lens", "0"]) == 2
    assert selftest.main(["--bogus"]) == 2


@pytest.mark.gpu
def test_selftest_grid_passes():
    buf = io.StringIO()
    rep = selftest.run_selftest(csv=buf)
    rows = buf.getvalue().strip().splitlines()
    assert rows[0] == ("config,seq_len,block_size,head_dim,num_heads,stride,comparison,tolerance,"
                       "max_rel_error,status")
    print("\n".join(r for r in rows if r.endswith("FAIL")))
    assert rep["instances"] == 144
    assert rep["failures"] == 0, rep


@pytest.mark.gpu
def test_selftest_detects_injected_corruption():
    r = subprocess.run([sys.executable, os.path.join(HERE, "selftest.py"), "--inject-corruption",
                        "--seq-lens", "64", "--csv", os.devnull], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 1, r.stderr
