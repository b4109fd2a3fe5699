"""The reference's C++ call sites against the paro::gpu drop-in adapter
(integration/paro_gpu.cpp over the C ABI), cross-checked with the CPU
reference in the same binary (integration/dropin_test.cpp)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "dropin_test"


def test_dropin_binary_passes():
    if not BIN.exists():
        pytest.skip("oracle/_ref/dropin_test not built (make -C oracle dropin)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
