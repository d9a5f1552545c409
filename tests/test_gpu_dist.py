"""Real multi-GPU parity: one rank per GPU over NCCL (tools/dist_parity.py under torchrun).

Runs on boxes with >= 2 GPUs (P = 2, and P = 4 when 4 are visible); on a
single-GPU box the same kernels/buffers are covered by the LocalWorld parity
tests and the NCCL message plans by tests/test_world_gloo.py.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_parity(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (have {torch.cuda.device_count()})")
    # one retry on a fresh port: the rendezvous port from _free_port can be taken before torchrun
    # binds it (a parity mismatch is deterministic and fails both attempts)
    for attempt in range(2):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               str(ROOT / "tools" / "dist_parity.py")]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=dict(os.environ))
        if res.returncode == 0:
            break
        print(f"attempt {attempt}: rc={res.returncode}\n{res.stdout[-2000:]}\n{res.stderr[-2000:]}")
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert f"DIST PARITY OK (P={world}" in res.stdout


@pytest.mark.parametrize("world", [2, 4])
def test_fullsize_peer_equals_nccl(world):
    """Bench-size S1 step (tools/dist_fullsize.py): slice routing bit-exact against the oracle gate,
    and the fused NVLink transport bit-identical to the NCCL transport."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (have {torch.cuda.device_count()})")
    for attempt in range(2):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               str(ROOT / "tools" / "dist_fullsize.py")]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=dict(os.environ))
        if res.returncode == 0:
            break
        print(f"attempt {attempt}: rc={res.returncode}\n{res.stdout[-2000:]}\n{res.stderr[-2000:]}")
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert f"FULLSIZE OK (P={world}" in res.stdout
