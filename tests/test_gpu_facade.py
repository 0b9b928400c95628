"""The C++ drop-in facade (include/tsgm_gpu.hpp, tsgm::gpu::step and the
sub-stage functions) against the reference's own tsgm::step on the same
frames: oracle/_ref/facade_parity (built here by `make -C oracle facade`
from the reference sources, it travels to the GPU box prebuilt)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "facade_parity")

pytestmark = pytest.mark.gpu


def test_facade_matches_reference_step():
    if not os.path.exists(BIN):
        pytest.skip("facade_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade parity: ok" in r.stdout
