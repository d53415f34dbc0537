"""The multi-rank code path on hardware: 2 ranks (torchrun, gloo) sharing the one GPU run the
row-sharded MLWE PCMM (words identical to one rank) and the sharded Rhombus PCMv (row shards
identical; column shards decrypt to the same values).  NCCL needs one GPU per rank, so the
collectives here are gloo's; the data path and the per-rank kernels are the real ones."""
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_on_one_gpu():
    root = Path(__file__).resolve().parents[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(root / "tests" / "_mp_gpu_worker.py")]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "multirank ok 2 fused ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
