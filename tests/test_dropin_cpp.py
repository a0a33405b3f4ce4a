"""Run the C++ drop-in KAT binary (tests/cpp/test_dropin.cpp) against libnulpa.so."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_cpp_dropin_kats():
    from paper_2411_11468_b200 import build
    exe = build.build_cpp_tests()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_dropin_compiles():
    """The reference-style C++ suite compiles and links against the drop-in (CPU)."""
    from paper_2411_11468_b200 import build
    exe = build.build_cpp_tests()
    assert exe.exists()
