"""Multi-process NCCL path on the GPU box: one rank per visible GPU (the
driver gives this run one), through torch.distributed.run."""
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_sharded_accumulate_matches_single_process():
    n = max(1, torch.cuda.device_count())
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           str(ROOT / "tests" / "dist_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("sharded == single: True") == n


@pytest.mark.parametrize("nproc", [1, 2, 3])
def test_driver_collective_bit_identical_across_world_sizes(nproc):
    """run_mlmc + accumulate_samples with one all-gather per accumulate call:
    identical bits on every rank and to the single-process run, for 1, 2 and
    3 processes (ranks beyond the GPU count share a GPU over gloo)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port",
           str(free_port()), str(ROOT / "tests" / "dist_mlmc_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("collective == single-process: True") == nproc


def test_bench_collective_path_runs():
    """bench.py's NCCL all-gather path (forced at world size 1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           str(ROOT / "bench.py"), "--gpus", "1", "--force-dist", "--steps", "1", "--warmup", "3",
           "--paths", str(1 << 22), "--level", "4", "--no-extras", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    import json
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["value"] > 0 and line["n_gpus"] == 1
