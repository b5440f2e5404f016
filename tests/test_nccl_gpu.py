"""NCCL transport: one process per GPU (torchrun), the drivers vs the oracle.

Needs >= 2 GPUs (gpurun --gpus 2/4); skipped on a single-GPU box, where the
same drivers are covered with virtual ranks by test_dist_gpu.py."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world,force_miss", [(2, False), (4, False), (2, True)])
def test_nccl_drivers(world, force_miss):
    """force_miss: BT_GATHER_SPEC_TEST=1 makes every speculative B gather miss
    (capacities halved after each exact one), so the redo path runs."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(29500 + world + 10 * force_miss), os.path.join(HERE, "nccl_worker.py")]
    env = dict(os.environ, BT_GATHER_SPEC_TEST="1" if force_miss else "0")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    print(p.stdout[-4000:])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert p.stdout.count(": OK") >= 8


@pytest.mark.parametrize("world", [2, 4])
def test_c3_case1_vs_oracle(world):
    """BASELINE c3 (10 %) through case 1 on `world` GPUs against the oracle."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(29600 + world), os.path.join(HERE, "c3_case1_worker.py"), "--occ", "0.10"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    print(p.stdout[-4000:])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert ": OK" in p.stdout or "] OK" in p.stdout
