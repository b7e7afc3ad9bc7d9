"""GPU training path against the reference tape and trainers:
tests/golden/train.npz was written by the unmodified reference (make_golden_train.py).
Per-op values and reverse-mode gradients, the solver-loss gradient of the net graphs,
loss records and final parameters of short training runs, and the net fixtures themselves
(net_conv.json / net_fc.json are the final weights of the staged training recipe)."""
import math
import os

import numpy as np
import pytest

import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import problems as gen

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def G():
    return np.load(os.path.join(GOLD, "train.npz"))


def _close(got, want, tol=1e-11):
    got, want = np.asarray(got), np.asarray(want)
    scale = max(float(np.max(np.abs(want))), 1e-300)
    assert got.shape == want.shape
    assert float(np.max(np.abs(got - want))) <= tol * scale, float(np.max(np.abs(got - want))) / scale


@pytest.mark.parametrize("tag,geometry,n", [("ops_sq7", "square", 7), ("ops_l9", "lshape", 9)])
def test_op_values_and_gradients_match_the_reference_tape(G, tag, geometry, n):
    from paper_2102_12071_b200 import autodiff as ad, device as dv
    A = gen.ProblemSpec("rotated", n, geometry, angle=np.pi / 6, anisotropy=100.0).assemble()
    assert np.array_equal(A.data, G[f"{tag}_A"])
    tp = mg.coarsen_full(A.spec)
    g = lambda k: G[f"{tag}_{k}"]   # noqa: E731

    def check(name, build, params):
        ad.zero_grads(params)
        root = build()
        ad.backward(root)
        assert float(root.value) == pytest.approx(float(g(f"{name}_val")), rel=1e-12)
        for q, p in enumerate(params):
            _close(dv.host(p.grad), g(f"{name}_g{q}"))

    k, u = ad.Var(g("kv")), ad.Var(g("u0"))
    check("conv2d", lambda: ad.norm2(ad.conv2d(k, u, A.spec)), [k, u])
    u = ad.Var(g("u0"))
    check("stencil", lambda: ad.norm2(ad.stencil_apply(A, u)), [u])
    u = ad.Var(g("u0"))
    check("restrict", lambda: ad.norm2(ad.do_restrict(tp, u)), [u])
    c = ad.Var(g("cv"))
    check("prolong", lambda: ad.norm2(ad.do_prolong(tp, c)), [c])
    p, u = ad.Var(g("pk")), ad.Var(g("u0"))
    check("pconv", lambda: ad.norm2(ad.pointwise_conv(p, u, A.spec)), [p, u])
    a, b = ad.Var(g("ck")), ad.Var(g("img"))
    check("convbatch", lambda: ad.norm2(ad.sum_axis(ad.leaky(ad.conv_batch(a, b), 0.01), 1)), [a, b])
    a, b = ad.Var(g("ma")), ad.Var(g("mb"))
    check("matmul", lambda: ad.norm2(ad.leaky(ad.matmul(a, b), 0.01)), [a, b])


def test_tape_bookkeeping():
    """autodiff.py tests :71-102: unused parameters keep no gradient; a variable feeding two
    branches receives both gradients; the closed-form quadratic."""
    from paper_2102_12071_b200 import autodiff as ad, device as dv
    A = gen.ProblemSpec("rotated", 7, angle=np.pi / 6, anisotropy=100.0).assemble()
    rng = np.random.default_rng(1)
    kv, unused = ad.Var(rng.standard_normal((3, 3))), ad.Var(np.ones((3, 3)))
    ad.zero_grads([kv, unused])
    ad.backward(ad.norm2(ad.conv2d(kv, rng.standard_normal((7, 7)), A.spec)))
    assert kv.grad is not None and unused.grad is None
    x = ad.Var(np.array([2.0]))
    ad.backward(ad.norm2(ad.add(ad.scale(x, 3.0), ad.scale(x, 4.0))))
    assert dv.host(x.grad)[0] == pytest.approx(7.0)
    w = ad.Var(np.array([1.5, -2.0, 0.25]))
    root = ad.reshape(ad.matmul(ad.reshape(ad.scale(w, 3.0), (1, 3)), ad.reshape(ad.scale(w, 3.0), (3, 1))), (1,))
    ad.zero_grads([w])
    ad.backward(root)
    assert np.allclose(dv.host(w.grad), 18.0 * np.array([1.5, -2.0, 0.25]), rtol=1e-12)


def test_gradients_survive_a_central_difference_audit():
    """grad_check on the device tape itself (autodiff.py:404-430)."""
    from paper_2102_12071_b200 import autodiff as ad
    A = gen.ProblemSpec("rotated", 7, angle=np.pi / 6, anisotropy=100.0).assemble()
    rng = np.random.default_rng(7)
    pk, uv = ad.Var(rng.standard_normal((7, 7, 3, 3)) * 0.2), ad.Var(rng.standard_normal((7, 7)))
    assert ad.grad_check(lambda: ad.norm2(ad.pointwise_conv(pk, uv, A.spec)), [pk, uv], seed=5, limit=60) < 1e-6


@pytest.mark.parametrize("variant", ["conv", "fc"])
def test_net_graph_loss_and_weight_gradients(G, variant):
    """training.py:434-467 + the solver loss: kernels, loss value and every weight
    gradient of the reference (tests/test_training.py:108)."""
    from paper_2102_12071_b200 import autodiff as ad, device as dv, training as tr
    A = gen.ProblemSpec("variable", 7, kappa=1.0).assemble()
    h = mg.equip_classical(mg.build_hierarchy(A, 2), "jacobi")
    h.levels[0].smoother = mg.jacobi(A)      # host-side classical smoother object for the frozen graph
    ds = tr.make_dataset(A, 2, seed=13)
    nw = 4
    net = mg.KernelInferenceNet(variant, [G[f"net_{variant}_w{q}"].copy() for q in range(nw)], 1)
    wvars = [ad.Var(w.copy()) for w in net.weights]
    fn = tr._net_graph(net, wvars, A)
    _close(dv.host(fn(ad.Var(ds[0].f.values)).value), G[f"net_{variant}_K"], 1e-12)
    # deployment path == training graph (tests/test_training.py:121-123)
    want = mg.infer_kernels(net, A).apply(ds[0].f).values
    assert np.max(np.abs(dv.host(fn(ad.Var(ds[0].f.values)).value) - want)) < 1e-12
    stack = tr._stack_for(h, 0, fn)
    ad.zero_grads(wvars)
    loss = tr._sample_loss(stack, ds[0], 2)
    ad.backward(loss)
    assert float(loss.value) == pytest.approx(float(G[f"net_{variant}_loss"]), rel=1e-12)
    for q, v in enumerate(wvars):
        _close(dv.host(v.grad), G[f"net_{variant}_g{q}"], 1e-10)


def test_forward_loss_equals_the_production_cycle(G):
    """The differentiable graph reproduces the V-cycle (tests/test_training.py:35-57)."""
    from paper_2102_12071_b200 import training as tr
    A = gen.ProblemSpec("rotated", 15, angle=np.pi / 6).assemble()
    h3 = mg.equip_conv_init(mg.build_hierarchy(A, 3))
    ds = tr.make_dataset(A, 2, seed=12)
    fn = tr.frozen_graph(h3.levels[0].smoother, A.spec)
    got = [float(tr.forward_loss(h3, 0, fn, ds[1], k).value) for k in (0, 1, 2, 3)]
    assert np.allclose(got, G["fwd_conv3_losses"], rtol=1e-11, atol=0)
    u = ds[1].u0
    for _ in range(2):
        u = mg.v_cycle(h3, 0, ds[1].f, u)
    assert abs(got[2] - (u - ds[1].u_star).norm()) < 1e-12


@pytest.mark.parametrize("variant", ["conv", "fc"])
def test_train_inference_net_reproduces_the_fixture(G, variant):
    """The staged training recipe behind net_conv.json / net_fc.json on the
    GPU: loss records of every stage and the final weights of the reference run."""
    from paper_2102_12071_b200 import training as tr
    A31 = gen.assemble_rotated_laplacian(mg.full_spec(31), math.pi / 6, 0.01)
    cfg = tr.TrainConfig(samples=10, max_steps=2, batch_size=5, epochs=20, seed=0)
    net, hier, recs = tr.train_inference_net(A31, variant, 4, cfg, k=1, seed_net=0)
    want = G[f"run_net_{variant}_records"]
    got = np.array([r.epochs for r in recs])
    assert got.shape == want.shape and np.allclose(got, want, rtol=1e-8, atol=0), np.max(np.abs(got / want - 1))
    fixture = mg.load_model(os.path.join(GOLD, f"net_{variant}.json"))
    for q, w in enumerate(net.weights):
        _close(w, G[f"run_net_{variant}_w{q}"], 1e-7)
        _close(w, fixture.weights[q], 1e-7)
    assert all(lev.smoother is not None for lev in hier.levels[:-1])


@pytest.mark.parametrize("act", ["linear", "leaky"])
def test_train_adaptive_matches_the_reference(G, act):
    from paper_2102_12071_b200 import training as tr
    A15 = gen.ProblemSpec("rotated", 15, angle=np.pi / 6).assemble()
    cfg = tr.TrainConfig(samples=6, max_steps=2, batch_size=3, epochs=6, seed=42)
    hier, recs = tr.train_adaptive(A15, 3, cfg, activation=act)
    assert np.allclose(np.array([r.epochs for r in recs]), G[f"run_adaptive_{act}_records"], rtol=1e-9, atol=0)
    for l, lev in enumerate(hier.levels[:-1]):
        _close(np.stack([k.weights for k in lev.smoother.layers]), G[f"run_adaptive_{act}_layers{l}"], 1e-8)
        _close(lev.smoother.skip.weights, G[f"run_adaptive_{act}_skip{l}"], 1e-8)
    # the trained hierarchy solves on the device with its new smoothers
    f = mg.GridFunction(A15.spec, gen.uniform_rhs(15, 3))
    _, rep = mg.solve(hier, f, tol=1e-6, max_iter=200)
    assert rep.converged


def test_train_independent_matches_the_reference(G):
    from paper_2102_12071_b200 import training as tr
    A15 = gen.ProblemSpec("rotated", 15, angle=np.pi / 6).assemble()
    cfg = tr.TrainConfig(samples=6, max_steps=2, batch_size=3, epochs=6, seed=42)
    sm, rec = tr.train_independent(A15, cfg, form="rb")
    assert np.allclose(rec.epochs, G["run_independent_records"], rtol=1e-9, atol=0)
    _close(np.stack([k.weights for k in sm.layers]), G["run_independent_layers"], 1e-8)


def test_train_mixture_and_injection_match_the_reference(G):
    """training.py:330-437: kernels shared across two rotation angles (per-operator gains),
    and residual-injection retraining on top of an adaptively trained hierarchy."""
    from paper_2102_12071_b200 import training as tr
    cfg = tr.TrainConfig(samples=6, max_steps=2, batch_size=3, epochs=6, seed=42)
    ops = [gen.ProblemSpec("rotated", 15, angle=t).assemble() for t in (np.pi / 6, np.pi / 4)]
    hiers, recs = tr.train_mixture(ops, 3, cfg)
    assert np.allclose(np.array([r.epochs for r in recs]), G["run_mixture_records"], rtol=1e-9, atol=0)
    for l in range(2):
        _close(np.stack([k.weights for k in hiers[1].levels[l].smoother.layers]), G[f"run_mixture_layers{l}"], 1e-8)
        _close(hiers[1].levels[l].smoother.skip.weights, G[f"run_mixture_skip{l}"], 1e-8)
        assert np.allclose([h.levels[l].smoother.gain for h in hiers], G[f"run_mixture_gains{l}"], rtol=1e-13)
        assert hiers[0].levels[l].smoother.layers[0] is hiers[1].levels[l].smoother.layers[0]   # shared kernels
    A15 = ops[0]
    hier, _ = tr.train_adaptive(A15, 3, cfg)
    hier, recs = tr.retrain_with_injection(hier, cfg, k_probe=2, probes=3)
    assert np.allclose(np.array([r.epochs for r in recs]), G["run_injection_records"], rtol=1e-8, atol=0)
    for l, lev in enumerate(hier.levels[:-1]):
        _close(np.stack([k.weights for k in lev.smoother.layers]), G[f"run_injection_layers{l}"], 1e-7)


def test_training_contract_errors():
    from paper_2102_12071_b200 import training as tr
    with pytest.raises(mg.ConfigError):
        tr.TrainConfig(samples=4, batch_size=5)
    with pytest.raises(mg.ConfigError):
        tr.train_mixture([], 2, tr.TrainConfig())
    A = gen.ProblemSpec("rotated", 7, angle=0.3).assemble()
    h = mg.equip_classical(mg.build_hierarchy(A, 2), "jacobi")
    with pytest.raises(mg.ConfigError):
        tr.train_level(h, 0, tr.TrainConfig(samples=2, batch_size=1, epochs=1))   # no trainable conv smoother
