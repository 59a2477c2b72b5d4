#!/usr/bin/env python
"""Benchmark driver (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): the LLaMA-2-7B-shaped decoder layer stack
(32 blocks x {q,k,v,o: 4096x4096; up,gate: 11008x4096; down: 4096x11008}),
4-bit QEFT, g=128, k=128 weak columns, decode GEMV at batch 1. One step = one
decode token through all 224 quantized linears, replayed as a CUDA graph.
Weights are synthetic, directly in the B200 tile layout, 3.70 GB per step
(far above the 126 MB L2, so no flush is needed between steps).

  value     algorithmic HBM GB/s of the stack, device-timed (CUDA events),
            max over ranks, summed over ranks (replicas: decode does not shard)
  e2e       same metric through the public API LinearStack.run(): pinned host
            x -> device, graph replay, all outputs -> pinned host, wall clock
  roofline  dominant GEMV shape timed alone with CUDA events, algorithmic bytes
            per launch / mean launch time vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the CPU oracle (numpy port of pkg/src/qeft/kernels.py
            matvec_structured) on one decoder block, rank 0, N=1

`--impl reference` times the reference algorithm on the host CPU (the oracle
port; the numpy reference cannot travel to the GPU box) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QEFT decode GEMV HBM GB/s (% peak); fine-tune tokens/s at 1/2/4/8 B200"
def workload(blocks=32, n_cols=1):
    return (f"LLaMA-2-7B-shaped decoder layer stack ({blocks} blocks x 7 linears = {7 * blocks} GEMVs), "
            f"4-bit QEFT g=128 k=128, decode GEMV batch {n_cols}")


WORKLOAD = workload()
BLOCK_SHAPES = [(4096, 4096), (4096, 4096), (4096, 4096), (4096, 4096),
                (11008, 4096), (11008, 4096), (4096, 11008)]


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_oracle_sample(seconds: float = 10.0, seed: int = 0):
    """Time the CPU oracle's matvec_structured over one synthetic 7B decoder block
    (7 layers, 4-bit g128 k128) until `seconds` elapse. Returns (GB/s, sample desc, cores)."""
    from oracle import qeft_oracle as O
    rng = np.random.default_rng(seed)
    layers = []
    for oc, ic in BLOCK_SHAPES:
        k, g, m = 128, 128, ic - 128
        packed = rng.integers(0, 256, size=oc * O.row_bytes(m, 4), dtype=np.uint8).tobytes()
        ng = O.n_groups(m, g)
        sc = (1e-3 + 0.01 * np.abs(rng.standard_normal((oc, ng)))).astype(np.float32)
        zr = (0.05 * rng.standard_normal((oc, ng))).astype(np.float32)
        weak = (0.02 * rng.standard_normal((oc, k))).astype(np.float32)
        layers.append(O.OracleLayer(oc=oc, ic=ic, k=k, bits=4, g=g, packed=packed, scales=sc,
                                    zeros=zr, weak=weak, weak_indices=np.arange(m, ic),
                                    layout="structured"))
    xs = {ic: rng.standard_normal(ic).astype(np.float32) for _, ic in BLOCK_SHAPES}
    # the same SURVEY 8(d) bytes as the GPU line (codes + 4 B per row and group + fp16 weak + x, y)
    nbytes = [O.row_bytes(q.m, 4) * q.oc + 4 * q.oc * q.n_groups + 2 * q.oc * q.k
              + 2 * (q.ic + q.oc) for q in layers]
    O.matvec_structured(layers[0], xs[layers[0].ic])  # warm
    done_b, calls, t0 = 0, 0, time.perf_counter()
    while True:
        for q, b in zip(layers, nbytes):
            O.matvec_structured(q, xs[q.ic])
            done_b += b
            calls += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    return done_b / dt / 1e9, f"{calls} matvec_structured calls over one 7B decoder block (7 layers), {dt:.1f} s", cores


def finetune_cpu_baseline(seconds: float = 12.0, T: int = 256):
    """CPU reference of the fine-tune step's linears: the oracle port of
    qlinear_forward_train + qlinear_backward (tuning.py:52-103; per-call dense dequant, BLAS
    fp32 GEMMs) on one layer of each 7B shape at T tokens, timed until `seconds` elapse, and
    EXTRAPOLATED to the 32-block step (per-token cost x 7 layers x 32 blocks). Attention, norms
    and the head are not included (they are not on the reference's quantized path)."""
    from oracle import qeft_oracle as O
    rng = np.random.default_rng(5)
    per_tok = {}
    t_end = time.perf_counter() + seconds
    for oc, ic in ((4096, 4096), (11008, 4096), (4096, 11008)):
        k, g, m = 128, 128, ic - 128
        q = O.OracleLayer(oc=oc, ic=ic, k=k, bits=4, g=g,
                          packed=rng.integers(0, 256, size=oc * O.row_bytes(m, 4), dtype=np.uint8).tobytes(),
                          scales=(1e-3 + 0.01 * np.abs(rng.standard_normal((oc, O.n_groups(m, g))))).astype(np.float32),
                          zeros=(0.05 * rng.standard_normal((oc, O.n_groups(m, g)))).astype(np.float32),
                          weak=(0.02 * rng.standard_normal((oc, k))).astype(np.float32),
                          weak_indices=np.arange(m, ic), layout="structured")
        x = rng.standard_normal((ic, T)).astype(np.float32)
        dy = rng.standard_normal((oc, T)).astype(np.float32)
        reps, t0 = 0, time.perf_counter()
        while True:
            _, xw = O.forward_train(q, x)
            O.backward(q, xw, dy)
            reps += 1
            if time.perf_counter() >= min(t_end, t0 + seconds / 3):
                break
        per_tok[(oc, ic)] = (time.perf_counter() - t0) / reps / T
    step_tok = 32 * sum(per_tok[(oc, ic)] for oc, ic in BLOCK_SHAPES)
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    return {"value": 1.0 / step_tok, "unit": "tokens/s", "cores": cores, "kind": "port",
            "extrapolated": True,
            "sample": "oracle qlinear_forward_train + qlinear_backward, one layer of each 7B shape at "
                      f"T={T}, {seconds:.0f} s; x 7 layers x 32 blocks (linears only)"}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (oracle port) on host cores."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import qeft_oracle as O  # noqa: F401
    per_step = []
    for i in range(args.warmup + args.steps):
        gbs, sample, cores = cpu_oracle_sample(seconds=2.0, seed=i)
        if i >= args.warmup:
            per_step.append(gbs)
    v = float(statistics.mean(per_step))
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "impl": "reference", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_cols": 1},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "port",
                             "sample": "per step: " + sample},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _time_graph(fn, iters, torch):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


# launch types of one decoder block: (name, layers in the launch as (oc, ic), launches per block)
LAUNCHES = [("qkv", [(4096, 4096)] * 3, 1), ("o", [(4096, 4096)], 1),
            ("gate_up", [(11008, 4096)] * 2, 1), ("down", [(4096, 11008)], 1)]


def kernel_roofline(torch, n_blocks, peak, n_cols, fuse=True):
    """Per-launch GEMV time of each launch type of the stack (CUDA events on the launching
    stream; a graph of n_blocks launches of that type, distinct weights, so they stream
    from HBM). Returns the per-launch table."""
    from paper_2410_08661_b200.decode import LinearStack, random_layer
    out = []
    for si, (name, shapes, _) in enumerate(LAUNCHES):
        if not fuse and len(shapes) > 1:
            shapes = shapes[:1]
        layers, groups = [], []
        for b in range(n_blocks):
            groups.append(list(range(len(layers), len(layers) + len(shapes))))
            layers += [random_layer(oc, ic, 128, 4, 128, "f16", seed=9000 + si * 100 + b * 3 + i)
                       for i, (oc, ic) in enumerate(shapes)]
        st = LinearStack(layers, n_cols=n_cols, groups=groups)
        for _ in range(3):
            st.step()
        reps = 20
        t = _time_graph(st.step, reps, torch)
        per_launch = t / (reps * n_blocks)
        nb = st.bytes_per_step() / n_blocks
        out.append({"launch": name, "shapes": [list(x) for x in shapes], "us_per_launch": per_launch * 1e6,
                    "bytes_per_launch": nb, "achieved_gbs": nb / per_launch / 1e9,
                    "frac": nb / per_launch / 1e9 / peak})
        del st, layers
    return out


def layout_bench(torch, peak):
    """The reference's three layouts on the 4096 x 4096 shape (OGR models keep W_O irregular,
    qmodel.py:117-131; online reordering gives every layer an input_perm, 132-141): the decode
    GEMV (N=1, 32 distinct layers per graph: HBM-resident) and the prefill/fine-tune GEMMs at
    T=2048. Structured layers read x in place; irregular / online ones gather x through the
    column map (in the GEMV's x staging; a gather pre-pass in the GEMM) and scatter dX."""
    from paper_2410_08661_b200.decode import LinearStack, random_layer
    from paper_2410_08661_b200.layer import DeviceLayer
    rng = np.random.default_rng(7)
    ic, k = 4096, 128

    def variant(dl, kind):
        if kind == "structured":
            return dl
        if kind == "irregular":
            weak = np.sort(rng.choice(ic, k, replace=False))
            keep = np.setdiff1d(np.arange(ic), weak)
            perm = np.concatenate([keep, weak])
        else:
            perm = rng.permutation(ic)
        colmap = np.full(dl.m_pad + dl.k_pad, -1, np.int32)
        colmap[:dl.m] = perm[:dl.m]
        colmap[dl.m_pad:dl.m_pad + k] = perm[dl.m:]
        return DeviceLayer(oc=dl.oc, ic=dl.ic, k=dl.k, bits=dl.bits, g=dl.g, qweight=dl.qweight, sz=dl.sz,
                           weak16=dl.weak16, colmap=torch.from_numpy(colmap).cuda(), dtype=dl.dtype,
                           weak32=dl.weak32, sz16=dl.sz16)

    out = []
    bpk = _bf16_peak(burst=True)
    for kind in ("structured", "irregular", "online"):
        layers = [variant(random_layer(4096, ic, k, 4, 128, "f16", seed=500 + i), kind) for i in range(32)]
        st = LinearStack(layers, n_cols=1)
        for _ in range(3):
            st.step()
        t = _time_graph(st.step, 20, torch) / (20 * 32)
        nb = st.bytes_per_step() / 32
        x = torch.randn(2048, ic, device="cuda", dtype=torch.float16)
        dy = torch.randn(2048, 4096, device="cuda", dtype=torch.float16)
        L0 = layers[0]
        for _ in range(3):
            L0.gemm_fwd(x)
            L0.gemm_dgrad(dy)
        tf = _time_graph(lambda: L0.gemm_fwd(x), 20, torch) / 20
        td = _time_graph(lambda: L0.gemm_dgrad(dy), 20, torch) / 20
        fl = 2.0 * 2048 * 4096 * ic
        out.append({"layout": kind, "gemv_us": t * 1e6, "gemv_gbs": nb / t / 1e9, "gemv_frac": nb / t / 1e9 / peak,
                    "gemm_fwd_tflops": fl / tf / 1e12, "gemm_dgrad_tflops": fl / td / 1e12,
                    "gemm_fwd_frac": fl / tf / 1e12 / bpk, "gemm_dgrad_frac": fl / td / 1e12 / bpk})
        del st, layers
    return out


def run_b200(args):
    import torch
    ws, rank, local = _dist()
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist
        # NCCL over NVLink; QEFT_DIST_BACKEND=gloo only to exercise the multi-rank logic with
        # several ranks on one GPU (NCCL refuses duplicate devices)
        backend = os.environ.get("QEFT_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    from paper_2410_08661_b200.decode import LinearStack, llama_launch_groups, llama_stack_layers
    peak, peak_kind = _peaks()
    n = args.n_cols

    layers = llama_stack_layers("7b", k=128, bits=4, g=128, dtype="f16", n_blocks=args.blocks)
    # q/k/v and gate/up read the same x: one launch each (qeft_gemv_multi), 4 launches per block
    groups = None if args.no_fuse else llama_launch_groups(args.blocks)
    stack = LinearStack(layers, n_cols=n, groups=groups)
    launches = stack.launches_per_step()
    for _ in range(args.warmup):
        stack.step()
    bytes_step = stack.bytes_per_step()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            stack.step()
        e1.record()
        torch.cuda.synchronize()
        # keep the GPU busy while the sampler collects enough samples
        t_extra = time.perf_counter()
        while time.perf_counter() - t_extra < 1.0:
            stack.step()
        torch.cuda.synchronize()
    barrier()
    t = e0.elapsed_time(e1) / 1e3
    if ws > 1:
        tt = torch.tensor([t], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    value = ws * bytes_step * args.steps / t / 1e9

    # e2e through the public API with pinned host buffers
    xh = {ic: torch.randn(n, ic).half() for ic in stack.ics}
    for _ in range(2):
        stack.run(xh)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        stack.run(xh)
    te = time.perf_counter() - t0
    if ws > 1:
        tt = torch.tensor([te], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        te = float(tt.item())
    e2e = ws * bytes_step * args.steps / te / 1e9

    roof = kernel_roofline(torch, min(args.blocks, 32), peak, n, fuse=not args.no_fuse) if rank == 0 else []
    # configs[1] is batch 1..16: the same stack at the other column counts (same layers, device
    # time of 10 graph replays each; the headline value stays at --n-cols)
    sweep = []
    if rank == 0 and not args.no_sweep:
        for nc in (1, 2, 4, 8, 16):
            if nc == n:
                continue
            st2 = LinearStack(layers, n_cols=nc, groups=groups)
            for _ in range(3):
                st2.step()
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            for _ in range(10):
                st2.step()
            s1.record()
            torch.cuda.synchronize()
            sec = s0.elapsed_time(s1) / 1e3 / 10
            gbs = st2.bytes_per_step() / sec / 1e9
            sweep.append({"n_cols": nc, "value": gbs, "unit": "GB/s", "frac": gbs / peak,
                          "ms_per_step": sec * 1e3})
            del st2
    n_layers = len(layers)
    del stack, layers
    torch.cuda.empty_cache()
    lay = layout_bench(torch, peak) if (rank == 0 and not args.no_sweep) else None
    ds = None if (args.no_dstep or rank != 0) else decode_step_bench(args, torch, dev)
    torch.cuda.empty_cache()
    ft = None if args.no_ft else finetune_bench(args, ws, rank, dev, torch)
    line = None
    if rank == 0:
        dom = max(roof, key=lambda r: r["us_per_launch"])  # one launch of each type per block
        traffic = None
        import glob
        tps = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "gemv_traffic.json")))
        if tps:  # dram__bytes_read + write per launch from the latest committed ncu capture
            traffic = json.load(open(tps[-1])).get(dom["launch"])
        cpu = None
        if ws == 1 and not args.no_cpu:
            gbs, sample, cores = cpu_oracle_sample(seconds=args.cpu_seconds)
            cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample}
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic",
            "config": {"workload": workload(args.blocks, n), "n_cols": n, "blocks": args.blocks,
                       "gemv_per_step": n_layers, "launches_per_step": launches,
                       "fused_launches": "q/k/v and gate/up share x: one qeft_gemv_multi launch each" if groups else None,
                       "bytes_per_step": bytes_step,
                       "l2": "inputs larger than L2 (%.2f GB of weights per step)" % (bytes_step / 1e9),
                       "parallelism": f"replicas{ws}"},
            "frac_of_peak": value / ws / peak, "peak_gbs": peak, "peak_kind": peak_kind,
            "roofline": {"bound": "hbm", "achieved": dom["achieved_gbs"], "peak": peak,
                         "unit": "GB/s", "frac": dom["frac"], "traffic": traffic,
                         "kernel": "gemv_kernel<4-bit, N=%d, g=128, fp16> launch %s %s (largest share of the step)"
                                   % (n, dom["launch"], dom["shapes"]),
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                         "per_shape": roof},
            "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "finetune": ft,
            "decode_step": ds,
            "batch_sweep": sweep or None,
            "layouts": lay,
        }
        if ft is not None and ws == 1 and not args.no_cpu:
            ft["cpu_baseline"] = finetune_cpu_baseline()
        line["e2e"]["h2d_bytes_per_step"] = sum(2 * n * ic for ic in sorted({s[1] for s in BLOCK_SHAPES}))
        line["e2e"]["d2h_bytes_per_step"] = sum(2 * n * oc for oc, _ in BLOCK_SHAPES) * args.blocks
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return line


def decode_step_bench(args, torch, dev):
    """Whole decode step around the GEMV: 7B-shaped QEFTDecoder, batch 1,
    KV cache at `--dstep-ctx` tokens. One CUDA graph per step covers norms, q/k/v and
    gate/up as fused GEMV launches, rotary, the cache write, attention, o/down, SiLU*mul, the
    dense head and residuals. Device-timed with CUDA events; the GEMV stack's share is the
    headline value's step time over this one."""
    from paper_2410_08661_b200.generate import KVDecoder
    from paper_2410_08661_b200.model import QEFTDecoder
    from paper_2410_08661_b200.qmodel import LLAMA2_7B
    model = QEFTDecoder.synthetic(LLAMA2_7B, k=128, bits=4, g=128, act_dtype="f16", compute_dtype="f16")
    for p in model.parameters():
        p.requires_grad_(False)
    ctx, steps = args.dstep_ctx, 128
    dec = KVDecoder(model, max_seq=ctx + steps + 1, capture=True)
    tok = torch.tensor([1])
    for p in range(ctx):  # fill the cache (untimed)
        dec.step(tok, p)
    torch.cuda.synchronize()
    # this latency-bound step is clock-sensitive: after an idle second the GPU can stay ~8%
    # slower for it (scripts/dstep_gap.py), so the clocks it ran at go into the record
    with ClockSampler(dev) as clk:
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for i in range(steps):
            dec.step(tok, ctx + i)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del dec, model
    return {"metric": "QEFT greedy decode tokens/s (batch 1)", "value": 1e3 / ms, "unit": "tokens/s",
            "ms_per_token": ms, "steps": steps,
            "config": {"workload": "LLaMA-2-7B-shaped QEFT decoder (4-bit g128 k=128, 32 blocks, fp16), "
                                   "KV cache, one CUDA graph per step",
                       "context": ctx, "batch": 1},
            "clocks": clk.summary(), "data": "synthetic", "dtype": "f16",
            # the paper's generation speed for this workload (QEFT 7B, k=128, 4-bit
            # g=128, batch 1) -- on an A100 80GB, so context, not a same-box ratio
            "vs_baseline": 1e3 / ms / 146.0,
            "baseline": {"value": 146.0, "unit": "tokens/s", "hardware": "A100 80GB", "source": "PAPER.md:227-228"}}


def finetune_bench(args, ws, rank, local, torch):
    """LLaMA-2-7B-shaped QEFT fine-tuning step (BASELINE.json configs[2]): seq 2048,
    micro-batch args.ft_mb per GPU, data parallel over the ranks: the flat fp32 weak-gradient
    bucket (174,063,616 params at k=128) is all-reduced with NCCL one decoder block at a time,
    each launched on the collective's stream as soon as that block's dW_weak lands during the
    backward (overlapped with the remaining blocks' backward), then the two-pass fused
    sqnorm -> clip + Adam + weak16 shadow kernels. Synthetic random-init weights in the B200 layout, fp16
    activations and residual stream with the exact power-of-two loss scale `finetune` uses
    (tuning.py here; the precision the model-level parity tests pass at,
    tests/test_finetune_gpu.py), synthetic tokens. value = tokens/s of the whole job
    (device-timed, max over ranks); e2e adds the per-step H2D token copy (pinned) and D2H
    loss read."""
    import numpy as np
    import torch.distributed as dist
    from paper_2410_08661_b200 import _lib
    from paper_2410_08661_b200.model import QEFTDecoder, cross_entropy_mean
    from paper_2410_08661_b200.qmodel import LLAMA2_7B, ModelConfig
    from paper_2410_08661_b200.tuning import TuneConfig, WeakTrainer, dp_allreduce_
    cfg = ModelConfig(**{**LLAMA2_7B.__dict__, "n_blocks": args.ft_blocks})
    model = QEFTDecoder.synthetic(cfg, k=128, bits=4, g=128, act_dtype="f16", compute_dtype="f16", seed=0)
    group = dist.group.WORLD if ws > 1 else None
    mb, seq, V = args.ft_mb, args.ft_seq, cfg.vocab_size
    loss_scale = float(2 ** math.ceil(math.log2(mb * seq)))  # as tuning.finetune does for fp16
    tr = WeakTrainer(model, TuneConfig(lr=5e-6, max_grad_norm=0.3), group=group, loss_scale=loss_scale)
    nsteps = args.ft_warmup + args.ft_steps
    rng = np.random.default_rng(1000 + rank)  # disjoint synthetic micro-batches per rank
    host = torch.from_numpy(rng.integers(0, V, size=(nsteps, mb, seq + 1))).pin_memory()
    dev = torch.empty((mb, seq + 1), dtype=torch.int64, device="cuda")
    loss_host = torch.empty((), dtype=torch.float64).pin_memory()

    def step(i, e2e=False):
        if e2e:
            dev.copy_(host[i], non_blocking=True)
        tr.zero_grad()
        tr.arm_overlap()  # N > 1: each block's weak-gradient bucket is all-reduced as its dW lands
        loss = cross_entropy_mean(model(dev[:, :-1]), dev[:, 1:])
        (loss * loss_scale).backward()
        loss_sum = loss.detach().double()
        dp_allreduce_(None, loss_sum, group)
        tr.step(ws, reduced=True)  # waits for the bucket all-reduces, then clip + Adam (2 passes)
        if e2e:
            loss_host.copy_(loss_sum)  # D2H read of the step's loss (synchronizes)

    dev.copy_(host[0])
    for i in range(args.ft_warmup):
        step(i)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    calls0 = _lib.CALLS[0]
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.ft_steps):
            step(i)
        e1.record()
        torch.cuda.synchronize()
    calls = (_lib.CALLS[0] - calls0) // args.ft_steps
    t = e0.elapsed_time(e1) / 1e3 / args.ft_steps
    if ws > 1:
        tt = torch.tensor([t], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.ft_steps):
        step(args.ft_warmup + i if args.ft_warmup + i < nsteps else i, e2e=True)
    te = (time.perf_counter() - t0) / args.ft_steps
    if ws > 1:
        tt = torch.tensor([te], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
    tokens = ws * mb * seq
    flops_tok = 28.39e9 * args.ft_blocks / 32  # 7B linears+attention+head per token
    tf_peak = _bf16_peak()
    gemm = gemm_roofline(torch, seq) if rank == 0 else None
    del model, tr
    torch.cuda.empty_cache()
    return {"metric": "QEFT fine-tune tokens/s", "value": tokens / t, "unit": "tokens/s",
            "ms_per_step": t * 1e3, "steps": args.ft_steps, "warmup": args.ft_warmup,
            "config": {"workload": "LLaMA-2-7B-shaped QEFT fine-tuning step (4-bit g128 k=128, "
                                   f"{args.ft_blocks} blocks), seq {seq}, micro-batch {mb}/GPU",
                       "global_batch_tokens": tokens, "parallelism": f"dp{ws}",
                       "weak_params": tr_params(cfg), "allreduce_bytes": 4 * tr_params(cfg),
                       "allreduce": f"{args.ft_blocks} per-block buckets, overlapped with the backward",
                       "l2": "activations and weights far above L2"},
            "dtype": "f16", "scaling": "weak", "data": "synthetic",
            "mfu": tokens / t * flops_tok / (ws * tf_peak * 1e12), "tflops_peak": tf_peak,
            "e2e": {"value": tokens / te, "unit": "tokens/s", "h2d_bytes_per_step": mb * (seq + 1) * 8,
                    "d2h_bytes_per_step": 8},
            "gpu_launches": calls * args.ft_steps, "gpu_launches_note": "libqeft_b200 C-ABI calls in the timed region (each launches 1-2 kernels)",
            "roofline": gemm, "clocks": clk.summary()}


def tr_params(cfg, k=128):
    """Weak-block parameters: k columns x output channels of every block linear."""
    return cfg.n_blocks * k * (4 * cfg.d_model + 2 * cfg.d_ff + cfg.d_model)


def _bf16_peak(burst: bool = False):
    """Dense bf16/fp16 tensor peak (equal rates): the sustained figure for a kernel timed inside
    a long step, the burst figure for a kernel timed alone (B200_PROFILING.md)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["bf16_tflops"]) if burst else float(d.get("bf16_tflops_sustained", d["bf16_tflops"]))
    return 1590.0 if burst else 1400.0


def gemm_roofline(torch, T):
    """Dominant kernel of the step: the tcgen05 forward GEMM (dequant producer + TMA
    activations), timed alone on the 7B shapes at T tokens with CUDA events."""
    from paper_2410_08661_b200.decode import random_layer
    peak = _bf16_peak(burst=True)  # timed alone: the burst figure
    out = []
    for oc, ic in ((4096, 4096), (11008, 4096), (4096, 11008)):
        dl = random_layer(oc, ic, 128, 4, 128, "f16", seed=5)
        x = torch.randn(T, ic, device="cuda", dtype=torch.float16)
        y = torch.empty(T, oc, device="cuda", dtype=torch.float16)
        for _ in range(3):
            dl.gemm_fwd(x, out=y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            dl.gemm_fwd(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 1e3 / reps
        fl = 2.0 * T * oc * ic
        out.append({"shape": [oc, ic], "T": T, "us": s * 1e6, "tflops": fl / s / 1e12,
                    "frac": fl / s / 1e12 / peak})
    dom = max(out, key=lambda r: r["us"] * (2 if r["shape"] == [11008, 4096] else 1))
    return {"bound": "tensor", "achieved": dom["tflops"], "peak": peak, "unit": "TFLOP/s",
            "frac": dom["frac"], "traffic": None,
            "kernel": "gemm_kernel<fwd, 4-bit, fp16> %dx%d T=%d" % (dom["shape"][0], dom["shape"][1], T),
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst; the kernel is timed alone)", "per_shape": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n-cols", type=int, default=1)
    ap.add_argument("--blocks", type=int, default=32)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ft", action="store_true", help="skip the fine-tune step measurement")
    ap.add_argument("--no-fuse", action="store_true", help="one GEMV launch per layer (no q/k/v, gate/up grouping)")
    ap.add_argument("--no-dstep", action="store_true", help="skip the end-to-end decode step measurement")
    ap.add_argument("--no-sweep", action="store_true", help="skip the n_cols 1..16 sweep of the decode stack")
    ap.add_argument("--dstep-ctx", type=int, default=512)
    ap.add_argument("--ft-blocks", type=int, default=32)
    ap.add_argument("--ft-seq", type=int, default=2048)
    ap.add_argument("--ft-mb", type=int, default=1)
    ap.add_argument("--ft-steps", type=int, default=5)
    ap.add_argument("--ft-warmup", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
