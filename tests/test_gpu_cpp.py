"""Runs the C++ drop-in parity suite (tests/cpp/test_dropin.cpp) on the GPU."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "paper_2511_18871_b200", "build", "test_dropin")


def test_cpp_dropin_suite():
    from paper_2511_18871_b200 import _build

    _build.build_cpp_tests()  # rebuilds only when a source is newer than the binary
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
