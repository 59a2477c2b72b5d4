"""bench.py under torchrun with 2 ranks (SURVEY 8(e) plumbing on the GPU): both ranks share the
one visible GPU, so the collective backend is gloo (QEFT_DIST_BACKEND; NCCL refuses duplicate
devices). Checks the contract the driver relies on at N > 1: one JSON line from rank 0,
n_gpus = 2, whole-job values, and the data-parallel fine-tune step's single weak-gradient
all-reduce."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, QEFT_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29547", "bench.py", "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--blocks", "2", "--no-dstep", "--no-sweep", "--no-cpu", "--ft-blocks", "2",
           "--ft-seq", "256", "--ft-steps", "1", "--ft-warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["parallelism"] == "replicas2"
    ft = line["finetune"]
    assert ft["value"] > 0 and ft["config"]["parallelism"] == "dp2"
    assert ft["config"]["allreduce_bytes"] == 4 * ft["config"]["weak_params"]
