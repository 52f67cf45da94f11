"""Multi-GPU paths (N >= 2): cross-process NVLink chain replication, NCCL
gradient reduction and the per-GPU swimlane loop.  Runs the worker under
torch.distributed.run on every visible GPU; skipped (not passed) on boxes
with fewer than two GPUs."""

import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def test_multigpu_worker():
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(here, "mp", "multigpu_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    for tag in ("SHARDED_LOSS_OK", "ZERO1_OK", "EXCHANGE_TIMEOUT_OK", "SWIMLANE_WEIGHTS_EQUAL_OK",
                "PEER_CHANNEL_OK",
                "MULTIGPU_OK"):
        assert tag in res.stdout, tag


def test_disaggregated_worker():
    """Learner ranks + rollout ranks with NVLink weight replication inside the
    RL loop (tests/mp/disagg_worker.py), on up to 4 GPUs."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = 4 if n >= 4 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(here, "mp", "disagg_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "DISAGG_OK" in res.stdout and "DISAGG_QUARANTINE_OK" in res.stdout
