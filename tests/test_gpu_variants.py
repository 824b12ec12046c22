"""Every kernel variant of the FAST path reaches the same parity bar: the FAST
PCG and operator tests re-run in a subprocess with the switches that select
the alternative kernels (stored-geometry K1 instead of the trilinear metric, the FMA K1 instead of
the DMMA one at n = 8,
the non-TMA K1/K2/Ax kernels, a one-iteration graph body)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = [{"SBX_STORED_GEOMETRY": "1"}, {"SBX_NO_TMA": "1"}, {"SBX_CG_UNROLL": "1"},
            {"SBX_K2_COLUMN": "1"}, {"SBX_K1_FMA": "1"}]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(e))
def test_fast_variants(cuda, env):
    full = dict(os.environ, **env)
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           "tests/test_gpu_pcg.py", "tests/test_gpu_ops.py", "tests/test_gpu_k1.py", "-k",
           "fast or axhelm or k1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=full)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
