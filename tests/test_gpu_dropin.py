"""The C++ drop-in (include/rdkv/cuda.hpp) against the unmodified reference
library on a B200: runs tests/cpp/_build/test_dropin (built here by
__graft_entry__.build(), see tests/cpp/Makefile) and requires every check to
pass. The binary prints one PASS/FAIL line per check."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "_build", "test_dropin")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference(cuda):
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} missing: build it with __graft_entry__.build() where /root/reference exists")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " 0 failed" in r.stdout
