"""GPU: the drop-in C++ API (include/i8t/*.hpp -> libi8t.so -> C-ABI) passes
the reference unit tests' known answers (tests/cpp/test_shim.cpp)."""
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_cpp_drop_in_api_known_answers():
    from paper_1912_12607_b200 import _build
    r = subprocess.run([_build.SHIM_TEST], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
