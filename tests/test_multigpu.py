"""Multi-GPU path on real GPUs (-m gpu): 2 (or more) ranks over NCCL must reproduce the
1-GPU run bit-for-bit (tests/mgpu_run.py).  Skipped when fewer than 2 GPUs are visible."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case,redecomp", [("patch", 1), ("jitter", 1), ("weak", 1), ("evrard", 1),
                                           ("cloud_sym", 1), ("jitter", 3)])
def test_multigpu_bit_identical_to_one_gpu(case, redecomp):
    n = _ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    env = dict(os.environ, MGPU_CASE=case, MGPU_STEPS="4", MGPU_REDECOMP=str(redecomp))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mgpu_run.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert '"ok": true' in r.stdout
