"""Data-parallel host logic of the fine-tuning step on CPU (gloo, world_size 2).

The DP step of `finetune` (tuning.py in this package; reference semantics
pkg/src/qeft/tuning.py:201-236) needs: (1) ranks draw the reference's window
stream in lockstep and keep disjoint micro-batches whose union is the whole
accumulation group; (2) one all-reduce of the flat weak-gradient bucket (and
the loss sum) turns per-rank partial sums into the single-process totals.
The gradient here is a plain torch least-squares gradient on CPU, so the test
exercises exactly the partition + collective, not the CUDA kernels."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_08661_b200.tuning import TuneConfig, dp_allreduce_, rank_micro_batches, sample_windows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_micro_batch_partition_matches_reference_stream(world):
    ids = np.arange(5000) % 251
    cfg = TuneConfig(batch=3, grad_accum=5, seq_len=16, seed=4)
    ref_rng = np.random.default_rng(cfg.seed)
    rngs = [np.random.default_rng(cfg.seed) for _ in range(world)]
    for _ in range(3):  # three optimizer steps: generators must stay in lockstep
        ref = [sample_windows(ref_rng, ids, cfg.batch, cfg.seq_len) for _ in range(cfg.grad_accum)]
        got = {}
        for r in range(world):
            for i, xb, yb, wgt in rank_micro_batches(rngs[r], ids, cfg, r, world):
                assert i % world == r and i not in got and wgt == 1.0
                got[i] = (xb, yb)
        assert sorted(got) == list(range(cfg.grad_accum))
        for i, (xb, yb) in enumerate(ref):
            np.testing.assert_array_equal(got[i][0], xb)
            np.testing.assert_array_equal(got[i][1], yb)


@pytest.mark.parametrize("world,batch,accum", [(6, 3, 5), (8, 4, 4), (16, 2, 4), (8, 1, 2)])
def test_more_ranks_than_micro_batches_split_windows(world, batch, accum):
    """world > grad_accum: the accumulation group's windows are dealt round-robin, so every rank
    works (as long as there are >= world windows) and the weighted chunks cover the group once."""
    ids = np.arange(5000) % 251
    cfg = TuneConfig(batch=batch, grad_accum=accum, seq_len=16, seed=4)
    ref_rng = np.random.default_rng(cfg.seed)
    rngs = [np.random.default_rng(cfg.seed) for _ in range(world)]
    for _ in range(2):
        ref = [sample_windows(ref_rng, ids, cfg.batch, cfg.seq_len) for _ in range(cfg.grad_accum)]
        ref_x = np.concatenate([r[0] for r in ref])
        seen, wsum = [], 0.0
        for r in range(world):
            work = rank_micro_batches(rngs[r], ids, cfg, r, world)
            assert work or r >= ref_x.shape[0]
            for _, xb, yb, wgt in work:
                assert xb.shape[0] <= cfg.batch and wgt == xb.shape[0] / cfg.batch
                seen.append(xb)
                wsum += wgt
        got = np.concatenate(seen)
        assert sorted(map(bytes, got)) == sorted(map(bytes, ref_x))  # every window exactly once
        assert abs(wsum - cfg.grad_accum) < 1e-12


def _grad_of(W, xb, yb):
    """d/dW mean((W x - y)^2) for a toy 'weak block' W (8 x 4) fed by token ids."""
    x = torch.from_numpy((xb[:, :4] % 7).astype(np.float32))
    y = torch.from_numpy((yb[:, :8] % 5).astype(np.float32))
    r = x @ W.T - y
    return (2.0 / r.numel()) * r.T @ x, float((r ** 2).mean())


def _worker(rank, world, port, q, accum=4):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids = np.arange(3000) % 113
        cfg = TuneConfig(batch=2, grad_accum=accum, seq_len=12, seed=9)
        W = torch.linspace(-1, 1, 32).reshape(8, 4)
        rng = np.random.default_rng(cfg.seed)
        bucket = torch.zeros(32, dtype=torch.float32)
        loss_sum = torch.zeros((), dtype=torch.float64)
        for _, xb, yb, wgt in rank_micro_batches(rng, ids, cfg, rank, world):
            g, l = _grad_of(W, xb, yb)
            bucket += wgt * g.reshape(-1)
            loss_sum += wgt * l
        dp_allreduce_(bucket, loss_sum, dist.group.WORLD)
        q.put((rank, bucket.numpy().copy(), float(loss_sum)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,accum", [(2, 4), (3, 1)])
def test_gloo_two_ranks_bucket_allreduce_equals_single_process(world, accum):
    """world 2 (micro-batch split) and world 3 > grad_accum 1 (window split, weighted)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, accum)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: all grad_accum micro-batches on one rank
    ids = np.arange(3000) % 113
    cfg = TuneConfig(batch=2, grad_accum=accum, seq_len=12, seed=9)
    W = torch.linspace(-1, 1, 32).reshape(8, 4)
    rng = np.random.default_rng(cfg.seed)
    ref_g = torch.zeros(32)
    ref_l = 0.0
    for _ in range(cfg.grad_accum):
        xb, yb = sample_windows(rng, ids, cfg.batch, cfg.seq_len)
        g, l = _grad_of(W, xb, yb)
        ref_g += g.reshape(-1)
        ref_l += l
    for _, g, l in res:
        np.testing.assert_allclose(g, ref_g.numpy(), rtol=1e-5, atol=1e-6)
        assert abs(l - ref_l) <= 1e-6 * max(1.0, abs(ref_l))
    np.testing.assert_array_equal(res[0][1], res[1][1])  # every rank holds the same sum
