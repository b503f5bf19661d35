"""Run the C++ drop-in tests (tests/cpp) on the GPU: the reference's scheduler
tests restated through include/janus_moesim_compat.hpp, and the same header on
the reference's own types against the reference library itself."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BUILD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build")


def run(name):
    exe = os.path.join(BUILD, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C tests/cpp)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert " 0 failures" in p.stdout


def test_aebs_compat_header():
    run("test_aebs_compat")


def test_dropin_on_reference_types():
    run("test_dropin")
