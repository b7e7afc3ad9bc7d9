"""Golden vectors of the training path from the UNMODIFIED reference (autodiff.py,
training.py).  Run in the build container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_train.py

train.npz holds, per case, the inputs, the forward value and the reverse-mode gradients
of the reference tape (`ops_*`), the solver-loss value and weight gradients of the
kernel-inference net graphs (`net_*`), and the loss records / final parameters of short
training runs (`run_*`).  The net fixtures net_conv.json / net_fc.json are the final
weights of the `run_net_*` cases (make_golden.py trains them with the same recipe).
"""
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from mgsmooth import autodiff as ad, grid as rg, problems as rp, smoothers as rs, training as rt   # noqa: E402
from mgsmooth.hierarchy import build_hierarchy, equip_classical, equip_conv_init                  # noqa: E402
from mgsmooth.transfer import coarsen_full                                                        # noqa: E402

out = {}


def grads_of(build, params):
    ad.zero_grads(params)
    root = build()
    ad.backward(root)
    return float(root.value), [np.zeros_like(p.value) if p.grad is None else p.grad.copy() for p in params]


def ops_case(tag, geometry, n):
    A = rp.ProblemSpec("rotated", n, geometry, angle=np.pi / 6, anisotropy=100.0).assemble()
    tp = coarsen_full(A.spec)
    rng = np.random.default_rng(7)
    m = A.spec.mask
    u0 = np.where(m, rng.standard_normal((n, n)), 0.0)
    kv = rng.standard_normal((3, 3)) * 0.3
    cv = np.where(tp.coarse.mask, rng.standard_normal(tp.coarse.mask.shape), 0.0)
    pk = rng.standard_normal((n, n, 3, 3)) * 0.2
    ck = rng.standard_normal((4, 3, 3)) * 0.5
    img = rng.standard_normal((6, 3, 3))
    ma, mb = rng.standard_normal((5, 4)), rng.standard_normal((4, 3))
    out[f"{tag}_mask"] = m
    out[f"{tag}_A"] = A.data
    for name, arr in (("u0", u0), ("kv", kv), ("cv", cv), ("pk", pk), ("ck", ck), ("img", img), ("ma", ma), ("mb", mb)):
        out[f"{tag}_{name}"] = arr

    def rec(name, build, params):
        val, gs = grads_of(build, params)
        out[f"{tag}_{name}_val"] = val
        for q, g in enumerate(gs):
            out[f"{tag}_{name}_g{q}"] = g

    k, u = ad.Var(kv.copy()), ad.Var(u0.copy())
    rec("conv2d", lambda: ad.norm2(ad.conv2d(k, u, A.spec)), [k, u])
    u = ad.Var(u0.copy())
    rec("stencil", lambda: ad.norm2(ad.stencil_apply(A, u)), [u])
    u = ad.Var(u0.copy())
    rec("restrict", lambda: ad.norm2(ad.do_restrict(tp, u)), [u])
    c = ad.Var(cv.copy())
    rec("prolong", lambda: ad.norm2(ad.do_prolong(tp, c)), [c])
    p, u = ad.Var(pk.copy()), ad.Var(u0.copy())
    rec("pconv", lambda: ad.norm2(ad.pointwise_conv(p, u, A.spec)), [p, u])
    a, b = ad.Var(ck.copy()), ad.Var(img.copy())
    rec("convbatch", lambda: ad.norm2(ad.sum_axis(ad.leaky(ad.conv_batch(a, b), 0.01), 1)), [a, b])
    a, b = ad.Var(ma.copy()), ad.Var(mb.copy())
    rec("matmul", lambda: ad.norm2(ad.leaky(ad.matmul(a, b), 0.01)), [a, b])


def net_case(variant):
    A = rp.ProblemSpec("variable", 7, kappa=1.0).assemble()
    h = build_hierarchy(A, 2)
    equip_classical(h, "jacobi")
    ds = rp.make_dataset(A, 2, seed=13)
    net = rs.inference_net(variant, k=1, seed=3)
    noise = np.random.default_rng(4)
    for w in net.weights:
        w += noise.standard_normal(w.shape) * 0.05
    net.bump()
    wvars = [ad.Var(w.copy()) for w in net.weights]
    fn = rt._net_graph(net, wvars, A)
    stack = rt._stack_for(h, 0, fn)
    val, gs = grads_of(lambda: rt._sample_loss(stack, ds[0], 2), wvars)
    out[f"net_{variant}_loss"] = val
    for q, (w, g) in enumerate(zip(net.weights, gs)):
        out[f"net_{variant}_w{q}"] = w
        out[f"net_{variant}_g{q}"] = g
    out[f"net_{variant}_K"] = fn(ad.Var(ds[0].f.values)).value


def run_cases():
    A31 = rp.assemble_rotated_laplacian(rg.full_spec(31), math.pi / 6, 0.01)
    cfg = rt.TrainConfig(samples=10, max_steps=2, batch_size=5, epochs=20, seed=0)
    for variant in ("conv", "fc"):
        t0 = time.time()
        net, _, recs = rt.train_inference_net(A31, variant, 4, cfg, k=1, seed_net=0)
        print(f"train_inference_net {variant}: {time.time() - t0:.1f}s")
        out[f"run_net_{variant}_records"] = np.array([r.epochs for r in recs])
        for q, w in enumerate(net.weights):
            out[f"run_net_{variant}_w{q}"] = w
    A15 = rp.ProblemSpec("rotated", 15, angle=np.pi / 6).assemble()
    cfg2 = rt.TrainConfig(samples=6, max_steps=2, batch_size=3, epochs=6, seed=42)
    for act in ("linear", "leaky"):
        hier, recs = rt.train_adaptive(A15, 3, cfg2, activation=act)
        out[f"run_adaptive_{act}_records"] = np.array([r.epochs for r in recs])
        for l, lev in enumerate(hier.levels[:-1]):
            out[f"run_adaptive_{act}_layers{l}"] = np.stack([k.weights for k in lev.smoother.layers])
            out[f"run_adaptive_{act}_skip{l}"] = lev.smoother.skip.weights
    sm, rec = rt.train_independent(A15, cfg2, form="rb")
    out["run_independent_records"] = np.array(rec.epochs)
    out["run_independent_layers"] = np.stack([k.weights for k in sm.layers])
    ops = [rp.ProblemSpec("rotated", 15, angle=t).assemble() for t in (np.pi / 6, np.pi / 4)]
    hiers, recs = rt.train_mixture(ops, 3, cfg2)
    out["run_mixture_records"] = np.array([r.epochs for r in recs])
    for l in range(2):
        out[f"run_mixture_layers{l}"] = np.stack([k.weights for k in hiers[1].levels[l].smoother.layers])
        out[f"run_mixture_skip{l}"] = hiers[1].levels[l].smoother.skip.weights
        out[f"run_mixture_gains{l}"] = np.array([h.levels[l].smoother.gain for h in hiers])
    hier, _ = rt.train_adaptive(A15, 3, cfg2)
    hier, recs = rt.retrain_with_injection(hier, cfg2, k_probe=2, probes=3)
    out["run_injection_records"] = np.array([r.epochs for r in recs])
    for l, lev in enumerate(hier.levels[:-1]):
        out[f"run_injection_layers{l}"] = np.stack([k.weights for k in lev.smoother.layers])
    # forward-loss values of frozen hierarchies (graph == production cycle)
    h3 = build_hierarchy(A15, 3)
    equip_conv_init(h3)
    ds = rp.make_dataset(A15, 2, seed=12)
    fn = rt.frozen_graph(h3.levels[0].smoother, A15.spec)
    out["fwd_conv3_losses"] = np.array([float(rt.forward_loss(h3, 0, fn, ds[1], k).value) for k in (0, 1, 2, 3)])


ops_case("ops_sq7", "square", 7)
ops_case("ops_l9", "lshape", 9)
net_case("conv")
net_case("fc")
run_cases()
np.savez_compressed(os.path.join(HERE, "train.npz"), **out)
print("wrote train.npz", len(out), "arrays")
