"""Multi-GPU parity: one process per GPU, peer arenas mapped over CUDA IPC
(handles exchanged with torch.distributed), every pattern vs the oracle."""

from __future__ import annotations

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(nproc: int) -> subprocess.CompletedProcess:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "tests" / "_mgpu_worker.py")]
    env = dict(os.environ, CARAMEL_WATCHDOG_MS="3000")
    return subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))


def test_two_gpus_all_patterns():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    r = _run(2)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "failures=0" in r.stdout


def test_all_gpus_all_patterns():
    import torch

    n = torch.cuda.device_count()
    if n < 3:
        pytest.skip("needs >= 3 GPUs")
    r = _run(n)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "failures=0" in r.stdout
