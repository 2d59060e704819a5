"""Multi-GPU tests (``-m gpu``; need >= 2 GPUs, e.g. ``gpurun --gpus 2``): launches
tests/mp_worker.py under torchrun, one rank per GPU, and checks its report."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # pragma: no cover
        return 0


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_state_against_oracle(world, tmp_path):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    report = tmp_path / "report.json"
    env = dict(os.environ, PS_MP_REPORT=str(report))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world), os.path.join(ROOT, "tests", "mp_worker.py")]
    proc = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert report.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    rep = json.loads(report.read_text())
    assert rep["ok"], json.dumps(rep, indent=1)[-4000:]
    assert proc.returncode == 0, proc.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.slow
@pytest.mark.parametrize("world,n", [(2, 33), (4, 35)])
def test_large_sharded_coset_oracle(world, n, tmp_path):
    """a JW-shaped Trotter step at 33q on 2 GPUs / 35q on 4 GPUs (128 GiB of fp64 state
    per GPU, the 36q-on-8 footprint) checked on whole cosets by the coset oracle at 1e-10."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    report = tmp_path / "report.json"
    env = dict(os.environ, PS_MP_REPORT=str(report), PS_MP_LARGE=str(n), PS_MP_ONLY_LARGE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), os.path.join(ROOT, "tests", "mp_worker.py")]
    proc = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1800)
    assert report.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    rep = json.loads(report.read_text())
    assert rep["ok"], json.dumps(rep, indent=1)[-4000:]
