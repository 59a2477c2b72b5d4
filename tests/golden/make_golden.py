"""Generate golden parity fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `qeft` from /root/reference/pkg/src (read-only), runs the hot-path
functions on small seeded inputs and writes `tests/golden/*.npz`. The GPU box
has no /root/reference; tests there read only these committed fixtures.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("QEFT_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from qeft import calibration, kernels, packing, quantizer, reorder, tuning  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _layer_dict(prefix, q, d):
    d[prefix + "oc"] = q.oc
    d[prefix + "ic"] = q.ic
    d[prefix + "k"] = q.k
    d[prefix + "bits"] = q.bits
    d[prefix + "g"] = q.g
    d[prefix + "packed"] = np.frombuffer(q.packed, np.uint8)
    d[prefix + "scales"] = q.scales
    d[prefix + "zeros"] = q.zeros
    d[prefix + "weak"] = q.weak
    d[prefix + "weak_indices"] = q.weak_indices
    d[prefix + "layout"] = q.layout
    d[prefix + "fallback"] = q.optq_fallback


def gen_packing():
    d = {}
    cases = []
    for t in range(40):
        rng = np.random.default_rng(100 + t)
        bits = int(rng.choice([3, 4]))
        oc, m = int(rng.integers(1, 20)), int(rng.integers(1, 70))
        codes = rng.integers(0, 1 << bits, size=(oc, m)).astype(np.uint8)
        d[f"c{t}_codes"] = codes
        d[f"c{t}_bits"] = bits
        d[f"c{t}_packed"] = np.frombuffer(packing.pack_codes(codes, bits), np.uint8)
        cases.append(t)
    d["n"] = len(cases)
    np.savez_compressed(os.path.join(OUT, "packing.npz"), **d)


def _rand_structured(rng):
    # same family as pkg/tests/test_kernels.py:17-26
    oc = int(rng.integers(1, 48))
    ic = int(rng.integers(2, 80))
    k = int(rng.integers(0, min(8, ic)))
    g = int(rng.integers(1, 40))
    bits = int(rng.choice([3, 4]))
    w = (rng.standard_normal((oc, ic)) * rng.uniform(0.1, 3.0)).astype(np.float32)
    return w, dict(k=k, bits=bits, g=g)


def gen_quantizer():
    d = {}
    n = 0
    # structured RTN family (kernel test family), seeds 0..59
    for t in range(60):
        rng = np.random.default_rng(t)
        w, kw = _rand_structured(rng)
        q = quantizer.quantize_layer(w, mode="rtn", layout="structured", **kw)
        x = rng.standard_normal(q.ic).astype(np.float32)
        d[f"q{n}_w"] = w
        d[f"q{n}_mode"] = "rtn"
        _layer_dict(f"q{n}_", q, d)
        d[f"q{n}_x"] = x
        d[f"q{n}_y_struct"] = kernels.matvec_structured(q, x)
        d[f"q{n}_y_ref"] = kernels.matvec_reference(q, x)
        n += 1
    # grid-search params + OPTQ rounding, structured and irregular
    for t in range(12):
        rng = np.random.default_rng(700 + t)
        oc, ic = int(rng.integers(4, 24)), int(rng.integers(12, 48))
        k = int(rng.integers(0, 6))
        g = int(rng.choice([4, 8, 16]))
        bits = int(rng.choice([3, 4]))
        w = rng.standard_normal((oc, ic)).astype(np.float32)
        x = rng.standard_normal((ic, 32)).astype(np.float32)
        layout = "structured" if t % 2 == 0 else "irregular"
        extra = {}
        if layout == "irregular":
            extra["lam"] = np.abs(rng.standard_normal(ic))
        q = quantizer.quantize_layer(w, k=k, bits=bits, g=g, mode="optq",
                                     layout=layout, x=x, **extra)
        d[f"q{n}_w"] = w
        d[f"q{n}_mode"] = "optq"
        d[f"q{n}_xcal"] = x
        if "lam" in extra:
            d[f"q{n}_lam"] = extra["lam"]
        _layer_dict(f"q{n}_", q, d)
        xv = rng.standard_normal(ic).astype(np.float32)
        d[f"q{n}_x"] = xv
        d[f"q{n}_y_ref"] = kernels.matvec_reference(q, xv)
        if layout == "irregular":
            d[f"q{n}_y_irr"] = kernels.matvec_irregular(q, xv)
        else:
            d[f"q{n}_y_struct"] = kernels.matvec_structured(q, xv)
        n += 1
    # pure grid-search parameter cases (outlier group, grid_steps=1)
    d["grid_outlier_params"] = np.array(
        [quantizer.grid_search_group_params(np.array([0.0, 1.0, 2.0, 100.0]), 2).scale,
         quantizer.grid_search_group_params(np.array([0.0, 1.0, 2.0, 100.0]), 2).zero])
    rng = np.random.default_rng(42)
    segs = rng.standard_normal((30, 37))
    gp = [quantizer.grid_search_group_params(s, 4) for s in segs]
    d["grid_segs"] = segs
    d["grid_scale"] = np.array([p.scale for p in gp])
    d["grid_zero"] = np.array([p.zero for p in gp])
    # fp32-valued segments (what quantize_layer feeds the search), incl. ragged/odd lengths
    segs32 = (rng.standard_normal((40, 128)) * 0.05).astype(np.float32)
    segs32[3, :] = segs32[3, 0]                  # constant group
    segs32[5, 7] = 3.0                           # outlier
    gp32 = [quantizer.grid_search_group_params(s.astype(np.float64), 4) for s in segs32]
    gp32_3 = [quantizer.grid_search_group_params(s[:53].astype(np.float64), 3) for s in segs32]
    d["grid_segs32"] = segs32
    d["grid_scale32"] = np.array([np.float32(p.scale) for p in gp32])
    d["grid_zero32"] = np.array([np.float32(p.zero) for p in gp32])
    d["grid_scale32_b3_n53"] = \
        np.array([np.float32(p.scale) for p in gp32_3])
    d["grid_zero32_b3_n53"] = np.array([np.float32(p.zero) for p in gp32_3])
    d["n"] = n
    np.savez_compressed(os.path.join(OUT, "quantizer.npz"), **d)


def gen_training():
    d = {}
    for t in range(10):
        rng = np.random.default_rng(500 + t)
        oc, ic = int(rng.integers(4, 40)), int(rng.integers(8, 64))
        k = int(rng.integers(1, min(8, ic - 1)))
        g = int(rng.choice([8, 16, 32]))
        bits = int(rng.choice([3, 4]))
        w = rng.standard_normal((oc, ic)).astype(np.float32)
        layout = "structured" if t % 3 else "irregular"
        extra = {} if layout == "structured" else {"lam": np.abs(rng.standard_normal(ic))}
        q = quantizer.quantize_layer(w, k=k, bits=bits, g=g, mode="rtn",
                                     layout=layout, **extra)
        if t % 4 == 3:  # online variant: runtime input permutation
            q.input_perm = rng.permutation(ic).astype(np.int64)
        tt = int(rng.integers(2, 12))
        x = rng.standard_normal((ic, tt)).astype(np.float32)
        dy = rng.standard_normal((oc, tt)).astype(np.float32)
        y, st = tuning.qlinear_forward_train(q, x)
        c = tuning.CostCounters()
        dx, dw = tuning.qlinear_backward(st, dy, q, counters=c)
        _layer_dict(f"t{t}_", q, d)
        d[f"t{t}_input_perm"] = (q.input_perm if q.input_perm is not None
                                 else np.zeros(0, np.int64))
        d[f"t{t}_x"], d[f"t{t}_dy"] = x, dy
        d[f"t{t}_y"], d[f"t{t}_xw"] = y, st.x_weak
        d[f"t{t}_dx"], d[f"t{t}_dw"] = dx, dw
        d[f"t{t}_counters"] = np.array([c.wgrad_fma, c.full_fma, c.saved_elems, c.full_elems])
    d["n"] = 10
    # Adam trajectories
    for t in range(3):
        rng = np.random.default_rng(60 + t)
        w = rng.standard_normal((5, 3)).astype(np.float32)
        st = tuning.AdamState.like(w)
        gs = rng.standard_normal((6, 5, 3)).astype(np.float32)
        d[f"adam{t}_w0"] = w.copy()
        d[f"adam{t}_g"] = gs
        for s in range(6):
            tuning.adam_step(st, w, gs[s], lr=0.01 * (t + 1))
        d[f"adam{t}_w"] = w
        d[f"adam{t}_m"], d[f"adam{t}_v"] = st.m, st.v
    np.savez_compressed(os.path.join(OUT, "training.npz"), **d)


def gen_selection():
    d = {}
    for t in range(6):
        rng = np.random.default_rng(300 + t)
        dm, ff, nb, k = 24, 48, 2, int(rng.integers(1, 6))
        lam = {}
        for b in range(nb):
            for nm in ("wq", "wk", "wv", "wo", "w_up", "w_gate"):
                v = np.abs(rng.standard_normal(dm))
                if t % 2:
                    v[rng.integers(0, dm, 3)] = 5.0  # ties
                lam[f"b{b}.{nm}"] = v
            lam[f"b{b}.w_down"] = np.abs(rng.standard_normal(ff))
        lam["head"] = np.abs(rng.standard_normal(dm))
        hd = calibration.HessianDiag(lam=lam, sample_count=1)
        gwc = calibration.select_global(hd, k, n_blocks=nb)
        for nm, v in lam.items():
            d[f"s{t}_lam_{nm}"] = v
        d[f"s{t}_names"] = np.array(list(lam.keys()))
        d[f"s{t}_k"] = k
        d[f"s{t}_resid"] = gwc.resid_indices
        d[f"s{t}_sglobal"] = gwc.s_global
        for b in range(nb):
            d[f"s{t}_ffn{b}"] = gwc.ffn_indices[b]
            d[f"s{t}_wo{b}"] = gwc.wo_indices[b]
        d[f"s{t}_perm"] = reorder.weak_to_tail(dm, gwc.resid_indices).perm
        # streaming lambda accumulation
        run = None
        xs = [rng.standard_normal((7, 5)) for _ in range(3)]
        for x in xs:
            run = calibration.accumulate_hessian_diag(
                calibration.ForwardTrace({"l": x}, 5), run)
        d[f"s{t}_lx"] = np.stack(xs)
        d[f"s{t}_lam_stream"] = run.lam["l"]
    d["n"] = 6
    np.savez_compressed(os.path.join(OUT, "selection.npz"), **d)


def gen_finetune():
    """Whole-model weak-column fine-tuning on a toy model (reference SMALL_CONFIG shape,
    pkg/tests/conftest.py:23-24): one forward/backward through the reference engine with
    QuantLinearTrainOp (loss, logits, every layer's dW_weak) and a 3-step finetune log and
    final weak blocks, for reorder modes ogr (structured + irregular wo) and online."""
    from qeft import model as M
    from qeft import qmodel as Q
    d = {}
    cfg = M.ModelConfig(d_model=32, n_heads=4, head_dim=8, d_ff=64, n_blocks=2,
                        vocab_size=256, max_seq=64, seed=5)
    dense = M.init_model(cfg)
    ids = np.random.default_rng(77).integers(0, 256, size=4000).astype(np.int64)
    hess = calibration.collect_calibration(dense, ids, n_seq=4, seq_len=48, seed=0)
    d["cfg"] = np.array([cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.d_ff, cfg.n_blocks,
                         cfg.vocab_size, cfg.max_seq, cfg.seed])
    d["ids"] = ids
    for mi, reo in enumerate(("ogr", "online")):
        qm = Q.quantize_model(dense, hess, k=4, bits=4, g=16, mode="rtn", reorder=reo)
        pre = f"m{mi}_"
        d[pre + "embedding"] = qm.embedding
        d[pre + "final_gain"] = qm.final_gain
        d[pre + "head"] = qm.head
        for i, b in enumerate(qm.blocks):
            d[pre + f"b{i}_gain1"] = b.gain1
            d[pre + f"b{i}_gain2"] = b.gain2
        for name, q in qm.layer_items():
            _layer_dict(pre + name + "_", q, d)
            d[pre + name + "_input_perm"] = (q.input_perm if q.input_perm is not None
                                            else np.zeros(0, np.int64))
        # one traced forward/backward of the engine with the training op
        rng = np.random.default_rng(11)
        xb, yb = M.sample_windows(rng, ids, 2, 32)
        em = Q.quant_engine(qm, op_factory=lambda nm, q: tuning.QuantLinearTrainOp(nm, q))
        logits, _, cache = M.forward_batch(em, xb, want_cache=True)
        loss, dlogits = M.cross_entropy_with_grad(logits, yb)
        grads = M.backward_batch(em, cache, dlogits, param_grads=False)
        d[pre + "xb"], d[pre + "yb"] = xb, yb
        d[pre + "logits"] = logits
        d[pre + "loss"] = loss
        for name in grads:
            d[pre + "grad_" + name] = grads[name]
        # short fine-tune
        tc = tuning.TuneConfig(steps=3, lr=1e-3, batch=2, grad_accum=2, seq_len=32, seed=2,
                               log_every=1)
        tuned, log = tuning.finetune(qm, ids, tc)
        d[pre + "log_loss"] = np.array([r["loss"] for r in log])
        d[pre + "log_gnorm"] = np.array([r["grad_norm"] for r in log])
        d[pre + "log_counts"] = np.array([[r["wgrad_fma"], r["full_fma"], r["saved_elems"],
                                           r["full_elems"]] for r in log])
        for name, q in tuned.layer_items():
            d[pre + "tuned_" + name] = q.weak
    d["n_models"] = 2
    np.savez_compressed(os.path.join(OUT, "finetune.npz"), **d)


def gen_container():
    """.qeft files written by the reference's save_checkpoint (container.py:311-319) for the
    toy quantized models of gen_finetune (OGR with plan + GWC + irregular wo; online with
    input permutations), plus the reference engine's logits on a fixed batch."""
    from qeft import container as C
    from qeft import model as M
    from qeft import qmodel as Q
    cfg = M.ModelConfig(d_model=32, n_heads=4, head_dim=8, d_ff=64, n_blocks=2,
                        vocab_size=256, max_seq=64, seed=5)
    dense = M.init_model(cfg)
    ids = np.random.default_rng(77).integers(0, 256, size=4000).astype(np.int64)
    hess = calibration.collect_calibration(dense, ids, n_seq=4, seq_len=48, seed=0)
    d = {}
    for reo in ("ogr", "online"):
        qm = Q.quantize_model(dense, hess, k=4, bits=4, g=16, mode="rtn", reorder=reo)
        path = os.path.join(OUT, f"toy_{reo}.qeft")
        C.save_checkpoint(path, qm)
        xb, _ = M.sample_windows(np.random.default_rng(13), ids, 2, 24)
        em = Q.quant_engine(qm, op_factory=lambda nm, q: tuning.QuantLinearTrainOp(nm, q))
        logits, _, _ = M.forward_batch(em, xb, want_cache=False)
        d[f"{reo}_xb"], d[f"{reo}_logits"] = xb, logits
        # greedy generation through the reference harness (kernels.py:197-228) and the logits
        # of every position of the final sequence (what each decode step must reproduce)
        prompt = ids[100:106]
        gen = kernels.bench_generate(qm, prompt, 10)
        seq = np.concatenate([prompt, gen.tokens])[None, :-1]
        glog, _, _ = M.forward_batch(em, seq, want_cache=False)
        d[f"{reo}_prompt"], d[f"{reo}_gen_tokens"], d[f"{reo}_gen_logits"] = prompt, gen.tokens, glog
        # weak-delta merging (merging.py): a 2-step tuned descendant, its delta (container kind 3)
        # and the delta applied back onto the base
        from qeft import merging
        tc = tuning.TuneConfig(steps=2, lr=1e-3, batch=2, grad_accum=1, seq_len=32, seed=4, log_every=1)
        tuned, _ = tuning.finetune(qm, ids, tc)
        C.save_checkpoint(os.path.join(OUT, f"toy_{reo}_tuned.qeft"), tuned)
        delta = merging.extract_delta(tuned, qm)
        C.save_checkpoint(os.path.join(OUT, f"toy_{reo}.delta.qeft"), delta)
        merged = merging.apply_to_quantized(qm, delta)
        for name, q in merged.layer_items():
            d[f"{reo}_merged_{name}"] = q.weak
        d[f"{reo}_plan_digest"] = np.array(merging.plan_digest(qm))
    np.savez_compressed(os.path.join(OUT, "container.npz"), **d)


def gen_qmodel():
    """Whole-model quantization (qmodel.py:82-156) on the toy model of gen_finetune: the dense
    weights, the traced calibration activations of every window (what collect_calibration feeds
    accumulate_hessian_full, calibration.py:113-122, 234-244), the reference's full Hessians,
    its global weak-column selection and OGR plan, and the quantized models for reorder modes
    ogr / online / none (RTN, so codes are BLAS-independent)."""
    from qeft import model as M
    from qeft import qmodel as Q
    cfg = M.ModelConfig(d_model=32, n_heads=4, head_dim=8, d_ff=64, n_blocks=2,
                        vocab_size=256, max_seq=64, seed=5)
    dense = M.init_model(cfg)
    ids = np.random.default_rng(77).integers(0, 256, size=4000).astype(np.int64)
    d = {"cfg": np.array([cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.d_ff, cfg.n_blocks,
                          cfg.vocab_size, cfg.max_seq, cfg.seed])}
    d["embedding"], d["head"], d["final_gain"] = dense.embedding, dense.head, dense.final_gain
    for i, b in enumerate(dense.blocks):
        for f in ("gain1", "gain2", "wq", "wk", "wv", "wo", "w_up", "w_gate", "w_down"):
            d[f"b{i}_{f}"] = getattr(b, f)
    # calibration_windows + traced forwards, exactly as collect_calibration does
    em = M.dense_engine(dense) if hasattr(M, "dense_engine") else calibration.dense_engine(dense)
    windows = calibration.calibration_windows(ids, 4, min(48, cfg.max_seq), 0)
    names = None
    for w, row in enumerate(windows):
        _, trace, _ = M.forward_batch(em, row[None, :], want_trace=True)
        names = list(trace.activations)
        for nm, x in trace.activations.items():
            d[f"act{w}_{nm}"] = x
    d["n_windows"] = len(windows)
    d["layer_names"] = np.array(names)
    hess = calibration.collect_calibration(dense, ids, n_seq=4, seq_len=48, seed=0)
    for nm, h in hess.h.items():
        d["h_" + nm] = h
    for reo in ("ogr", "online", "none"):
        qm = Q.quantize_model(dense, hess, k=4, bits=4, g=16, mode="rtn", reorder=reo)
        pre = reo + "_"
        d[pre + "embedding"], d[pre + "head"], d[pre + "final_gain"] = qm.embedding, qm.head, qm.final_gain
        for i, b in enumerate(qm.blocks):
            d[pre + f"b{i}_gain1"], d[pre + f"b{i}_gain2"] = b.gain1, b.gain2
        for name, q in qm.layer_items():
            _layer_dict(pre + name + "_", q, d)
            d[pre + name + "_input_perm"] = (q.input_perm if q.input_perm is not None
                                            else np.zeros(0, np.int64))
        if reo == "ogr":
            d["gwc_resid"] = qm.gwc.resid_indices
            d["gwc_s_global"] = qm.gwc.s_global
            for i in range(cfg.n_blocks):
                d[f"gwc_ffn{i}"] = qm.gwc.ffn_indices[i]
                d[f"gwc_wo{i}"] = qm.gwc.wo_indices[i]
                d[f"plan_ffn{i}"] = qm.plan.p_ffn[i].perm
            d["plan_resid"] = qm.plan.p_resid.perm
            d["fingerprint"] = np.array(qm.fingerprint)
    np.savez_compressed(os.path.join(OUT, "qmodel.npz"), **d)


if __name__ == "__main__":
    # `make_golden.py [packing quantizer training selection finetune]` (default: all)
    gens = {"packing": gen_packing, "quantizer": gen_quantizer, "training": gen_training,
            "selection": gen_selection, "finetune": gen_finetune, "container": gen_container,
            "qmodel": gen_qmodel}
    for name in (sys.argv[1:] or list(gens)):
        gens[name]()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
