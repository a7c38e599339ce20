"""GPU: the C++ drop-in header (include/tsdg/gpu_search.hpp) against the reference
library in one C++ program (tests/cpp/test_gpu_api.cpp, built by build() where the
reference sources exist; the prebuilt binary travels with the repo snapshot)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_gpu_api")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/_build/test_gpu_api not built")
def test_cpp_dropin_matches_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "checks passed" in r.stdout
