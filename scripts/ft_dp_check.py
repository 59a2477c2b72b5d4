"""Run the reference-parity fine-tune (tests/golden/finetune.npz, model mi) under torchrun with
the gloo backend (every rank on the one visible GPU) and write rank 0's log + tuned weak blocks.
usage: torchrun --nproc-per-node W scripts/ft_dp_check.py OUT.npz MI"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from tests.conftest import load_golden
from tests.test_finetune_gpu import _qmodel

out, mi = sys.argv[1], int(sys.argv[2])
ws = int(os.environ.get("WORLD_SIZE", "1"))
if ws > 1:
    dist.init_process_group("gloo")
from paper_2410_08661_b200.tuning import TuneConfig, finetune  # noqa: E402

z = load_golden("finetune")
tc = TuneConfig(steps=3, lr=1e-3, batch=2, grad_accum=2, seq_len=32, seed=2, log_every=1)
tuned, log = finetune(_qmodel(z, mi), z["ids"], tc)
if ws == 1 or dist.get_rank() == 0:
    d = {"loss": np.array([r["loss"] for r in log]), "gnorm": np.array([r["grad_norm"] for r in log])}
    for name, q in tuned.layer_items():
        d["w_" + name] = q.weak
    np.savez(out, **d)
if ws > 1:
    dist.destroy_process_group()
