"""`finetune` data-parallel on the GPU: torchrun with 2 and 3 ranks sharing the one
visible GPU (gloo; NCCL refuses duplicate devices). grad_accum = 2, so world 2 splits whole
micro-batches and world 3 deals the 4 windows round-robin (tuning.rank_micro_batches). The
per-block bucket all-reduces are launched during the last backward (WeakTrainer.arm_overlap).
Each world's losses, pre-clip gradient norms and tuned weak blocks must equal world 1's (same
math, different summation order: <= 1e-4 relative) and the reference's (finetune.npz, the
bars of tests/test_finetune_gpu.py)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(world, out, mi, port):
    cmd = [sys.executable, os.path.join(ROOT, "scripts", "ft_dp_check.py"), out, str(mi)]
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
               "--master-addr", "127.0.0.1", "--master-port", str(port)] + cmd[1:]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


@pytest.mark.parametrize("mi", [0, 1])
def test_finetune_world_2_and_3_equal_world_1(mi, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    z = load_golden("finetune")
    w1 = _run(1, str(tmp_path / "w1.npz"), mi, 0)
    for world, port in ((2, 29611 + mi), (3, 29621 + mi)):
        wn = _run(world, str(tmp_path / f"w{world}.npz"), mi, port)
        assert _rel(wn["loss"], w1["loss"]) <= 1e-4, world
        assert _rel(wn["gnorm"], w1["gnorm"]) <= 1e-4, world
        worst = max(_rel(wn[k], w1[k]) for k in w1.files if k.startswith("w_"))
        print(f"model {mi} world {world}: worst weak rel vs world 1 {worst:.2e}")
        assert worst <= 1e-3, world
        assert rel_err(wn["loss"], z[f"m{mi}_log_loss"]) <= 1e-2
        assert _rel(wn["gnorm"], z[f"m{mi}_log_gnorm"]) <= 2e-2
        worst_ref = max(_rel(wn["w_" + n], z[f"m{mi}_tuned_{n}"]) for n in (k[2:] for k in w1.files if k.startswith("w_")))
        assert worst_ref <= 2e-2, world
