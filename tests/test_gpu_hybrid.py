"""Drop-in check: the reference's own sembox::pcg (compiled from
/root/reference) driving the B200 operators through include/sbx_sembox.hpp
reproduces the all-CPU run bit for bit; the fused device solver matches it.
The binary is built here (oracle/Makefile `hybrid`) and travels to the GPU box."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
BIN = os.path.join(ROOT, "oracle", "_ref", "hybrid_pcg")


def test_reference_pcg_with_b200_operators(cuda):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/hybrid_pcg not built (needs /root/reference at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "HYBRID PASS" in out.stdout
