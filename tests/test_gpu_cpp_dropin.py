"""Reference-style C++ tests of the C++ drop-in header (paper_1810_05628_b200/
cpp/ptycho_b200.hpp) over libptg, executed on the B200."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1810_05628_b200", "lib", "test_ptycho_b200")


def test_cpp_dropin_suite():
    assert os.path.exists(BIN), "build with python -m paper_1810_05628_b200._build"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed checks: 0" in r.stdout
