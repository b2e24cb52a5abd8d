"""The row-partitioned path over a real NCCL communicator with one process per GPU
(torchrun, world size 2): Y, Z and t_k bitwise equal to the single-device run (SURVEY.md
§8(e) determinism claim).  Skips when fewer than 2 GPUs are visible (the in-process rank
group of tests/test_gpu_dist.py covers G = 2..8 on one device)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_torchrun_world2_bitwise():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one process per GPU)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(ROOT, "tests", "_nccl_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, (p.stdout[-3000:], p.stderr[-3000:])
    assert "bitwise equal to G=1: True" in p.stdout
