"""Real multi-GPU parity (CUDA-IPC collectives over NVLink, one process per
GPU): runs tests/mp_worker.py under torchrun on 2 or 4 GPUs."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_multigpu_parity():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(HERE, "mp_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    res = json.loads(lines[-1])
    assert res["ok"] and res["raw_collectives"] == "bit-exact"


def test_multigpu_cli_verify():
    """`verify`: sharded fp32 training vs an unsharded torch.optim.Adam copy."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           "-m", "paper_2304_11277_b200", "verify", "--steps", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(HERE))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    last = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    assert json.loads(last)["verify"] == "PASS"
