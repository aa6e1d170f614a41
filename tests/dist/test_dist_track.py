"""Multi-GPU time slabs with a real NCCL communicator (torchrun, one process per GPU):
labels and records bit-identical to the single-GPU track for every world size the box offers (2..8),
and a failure on one slab reported as the same status on every rank.  Skips with fewer than 2 GPUs."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sorted(a):
    return a[np.argsort(a["face_id"], kind="stable")]


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_nccl_slabs_match_single_gpu(world, tmp_path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(HERE, "worker.py"),
           str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for name in ("woven2d", "woven3d", "c2_crop"):
        got = np.concatenate([np.load(tmp_path / f"{name}_rank{k}.npy") for k in range(world)])
        single = np.load(tmp_path / f"{name}_single.npy")
        assert _sorted(got).tobytes() == _sorted(single).tobytes(), name
    for k in range(world):
        st = [int(x) for x in open(tmp_path / f"status_rank{k}.txt").read().split()]
        assert st == [2] * world, st  # FTK_ERR_RANGE everywhere
