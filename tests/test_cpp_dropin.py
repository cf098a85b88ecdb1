"""The C++ drop-in (include/dsplat_b200) against the reference C++ API.

tests/cpp/dropin_parity.cpp calls the reference (CPU) and dsplat::b200
(libdsg.so, GPU) with the same reference types; it is compiled where the
reference headers exist and the binary travels with the tree.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "_build", "dropin_parity")


@pytest.mark.gpu
def test_cpp_dropin_parity():
    if not os.path.exists(EXE):
        pytest.skip("dropin_parity not built (needs the reference headers at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
