"""The C++ drop-in (paper_1810_05628_b200/cpp/include/ptycho: the reference's
public API, namespace ptycho, over libptg) on the B200:

* ref_tests_dropin: the reference's OWN unit tests -- proj/tests/
  test_objectives.cpp, test_solvers.cpp, test_multigrid.cpp, unmodified --
  compiled against the drop-in headers with a doctest shim (built where the
  reference sources exist; the binary ships with lib/);
* test_dropin_ext: the additive surface (patch-model probe, complex64 plans,
  GPU-resident solvers with callbacks / warm starts, coarse V-cycles)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1810_05628_b200", "lib")


def _run(name):
    path = os.path.join(LIB, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (python -m paper_1810_05628_b200._build)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:])
    return r


def test_reference_unit_tests_against_dropin():
    r = _run("ref_tests_dropin")
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
    assert "failed: 0; checks:" in r.stdout and ", failed: 0" in r.stdout.splitlines()[-1]


def test_dropin_extensions():
    r = _run("test_dropin_ext")
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
