"""Multi-GPU parity on real devices (skipped with fewer than 2 GPUs): runs
tools/dist_check.py under torchrun -- distributed gather-scatter bitwise equal
to the single-process reference, operator within 1e-12, PCG same iteration
count and solution within 1e-10."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ranks", [2, 4])
def test_dist_check(cuda, ranks):
    if cuda.cuda.device_count() < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    for _attempt in range(3):  # (a rendezvous port taken meanwhile: pick another)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={ranks}", "--master-addr", "127.0.0.1", "--master-port",
               str(_port()), os.path.join(ROOT, "tools", "dist_check.py")]
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
        if out.returncode == 0 or "EADDRINUSE" not in out.stderr:
            break
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert out.stdout.count("ALL OK") == ranks


def test_dist_check_8_ranks_oversubscribed(cuda):
    """The 8-rank limit (kMaxRanks) with 8 processes on the available GPUs (two
    or more per device): the exchange plan, mailboxes and flags of every rank
    pair at the largest supported world size."""
    if cuda.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    if not os.environ.get("SBX_TEST_OVERSUB"):
        # several ranks per GPU run spin-waiting exchange kernels as separate
        # processes on one device: nothing guarantees they are co-scheduled
        # (B200 driver 580 raised context-switch timeouts for such setups), so
        # this case runs only on request
        pytest.skip("set SBX_TEST_OVERSUB=1 to run ranks oversubscribed on the GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "dist_check.py")]
    env = dict(os.environ, SBX_OVERSUB="1")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert out.stdout.count("ALL OK") == 8
