"""The C++ drop-in header (include/ib_b200/ib.hpp) over the C ABI.

CPU: the shim compiles against the reference's call pattern and links
libibcuda.so (the binary exits 77 = skipped without a device).
GPU: the same binary runs the reference-style coupling cases and checks them
against the C oracle (keys/perm/run_count bit-exact, values <= 1e-12).
"""
import subprocess

import pytest

from paper_2012_06646_b200 import _build


def _binary():
    return _build.build_cpp_tests()


def test_shim_builds_and_links():
    exe = _binary()
    assert exe is not None and exe.exists()


@pytest.mark.gpu
def test_shim_runs_reference_call_pattern_on_device():
    exe = _binary()
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim ok" in out.stdout
