"""Generate golden vectors by running the UNMODIFIED reference (mgsmooth 0.1.0).

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed, small):
    net_conv.json, net_fc.json   seeded small-problem training runs:
        train_inference_net(A31, variant, 4, TrainConfig(samples=10, max_steps=2,
        batch_size=5, epochs=20, seed=0), k=1, seed_net=0), A31 = rotated FD
        31x31, theta=pi/6, anisotropy=0.01; saved with smoothers.save_model.
    net_conv_k2.json             fresh inference_net('conv', k=2, seed=5) with a
        seeded random final layer (exercises the k>1 leaky-stage path).
    ops.npz                      apply_stencil / restrict / prolong / galerkin /
        coarse LU on random per-point stencils, square / lshape / cylinder masks.
    case_<name>.npz              full hierarchies: per-level A, per-level K
        (small cases), f, residual history, u after N cycles.
    c1.npz                       config 1 (255^2, V(2,2), 20 cycles) history + u.
    krylov.npz                   fgmres / gmres (krylov.py) with grid_action and
        cycle_preconditioner: histories, iteration counts, solutions.
    conv.npz                     shared-kernel ConvSmoother (smoothers.py:105-178,
        hierarchy.py:164-204): convolve / apply / effective_kernel pins, V-cycles.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import mgsmooth as mg                                     # noqa: E402  (reference)
from mgsmooth import grid as rg, transfer as rt, hierarchy as rh, smoothers as rs  # noqa: E402
from mgsmooth import problems as rp, dense as rd, training as rtr              # noqa: E402
from mgsmooth.cli import RepeatedSmoother                  # noqa: E402

from paper_2102_12071_b200 import problems as gen          # noqa: E402  (input generators only)


def spec_of(mask, h):
    return rg.GridSpec(mask.shape[0], mask.shape[1], h, mask)


def make_nets():
    out = {}
    A31 = rp.assemble_rotated_laplacian(rg.full_spec(31), math.pi / 6, 0.01)
    for variant in ("conv", "fc"):
        path = os.path.join(HERE, f"net_{variant}.json")
        if os.path.exists(path):
            out[variant] = rs.load_model(path)
            continue
        t0 = time.time()
        cfg = rtr.TrainConfig(samples=10, max_steps=2, batch_size=5, epochs=20, seed=0)
        net, _, _ = rtr.train_inference_net(A31, variant, 4, cfg, k=1, seed_net=0)
        rs.save_model(path, net, {"fixture": "SURVEY G4", "operator": "rotated FD 31x31 pi/6 0.01"})
        print(f"trained {variant} net in {time.time() - t0:.1f}s")
        out[variant] = rs.load_model(path)
    # the same recipe at config 2's parameters (theta = pi/4, anisotropy = 1e-3): the bench net
    path = os.path.join(HERE, "net_conv_c2.json")
    if not os.path.exists(path):
        A31c2 = rp.assemble_rotated_laplacian(rg.full_spec(31), math.pi / 4, 1e-3)
        cfg = rtr.TrainConfig(samples=10, max_steps=2, batch_size=5, epochs=20, seed=0)
        net, _, _ = rtr.train_inference_net(A31c2, "conv", 4, cfg, k=1, seed_net=0)
        rs.save_model(path, net, {"fixture": "SURVEY G4 recipe at config-2 parameters"})
    out["conv_c2"] = rs.load_model(path)
    # config 5 parameters (theta = pi/3, anisotropy = 0.01)
    path = os.path.join(HERE, "net_conv_c5.json")
    if not os.path.exists(path):
        A31c5 = rp.assemble_rotated_laplacian(rg.full_spec(31), math.pi / 3, 0.01)
        cfg = rtr.TrainConfig(samples=10, max_steps=2, batch_size=5, epochs=20, seed=0)
        net, _, _ = rtr.train_inference_net(A31c5, "conv", 4, cfg, k=1, seed_net=0)
        rs.save_model(path, net, {"fixture": "SURVEY G4 recipe at config-5 parameters"})
    out["conv_c5"] = rs.load_model(path)
    # config 3 (GRF diffusion, 5-point): the recipe on a seeded 31^2 GRF (corr. length 1/4)
    path = os.path.join(HERE, "net_conv_c3.json")
    if not os.path.exists(path):
        Ag = gen.grf_diffusion_5pt(31, corr_len=0.25, seed=2)
        S = rg.StencilField(rg.GridSpec(31, 31, 1 / 31, np.ones((31, 31), bool)), Ag)
        cfg = rtr.TrainConfig(samples=10, max_steps=2, batch_size=5, epochs=20, seed=0)
        net, _, _ = rtr.train_inference_net(S, "conv", 4, cfg, k=1, seed_net=0)
        rs.save_model(path, net, {"fixture": "SURVEY G4 recipe on a config-3 GRF 31^2", "corr_len": 0.25})
    out["conv_c3"] = rs.load_model(path)
    path = os.path.join(HERE, "net_conv_k2.json")
    if not os.path.exists(path):
        net = rs.inference_net("conv", k=2, seed=5)
        rng = np.random.default_rng(6)
        net.weights[-1] = rng.standard_normal(net.weights[-1].shape) * 0.05
        rs.save_model(path, net, {"fixture": "random k=2 conv net, seed 5/6"})
    out["conv_k2"] = rs.load_model(path)
    return out


def make_ops():
    rng = np.random.default_rng(20240817)
    d = {}
    for geom in ("square", "lshape", "cylinder"):
        for n in (9, 10):
            mask = gen.geometry_mask(geom, n) if n == 9 else np.ones((n, n + 3), bool)
            if n == 10 and geom != "square":
                continue
            h = 1.0 / (n + 1)
            spec = spec_of(mask, h)
            A = rng.standard_normal(mask.shape + (3, 3))
            A[:, :, 1, 1] += 8.0
            u = np.where(mask, rng.standard_normal(mask.shape), 0.0)
            S = rg.StencilField(spec, A)
            U = rg.GridFunction(spec, u)
            key = f"{geom}{n}"
            d[f"{key}_mask"] = mask
            d[f"{key}_A"] = A
            d[f"{key}_u"] = u
            d[f"{key}_Au"] = rg.apply_stencil(S, U).values
            tp = rt.coarsen_full(spec)
            d[f"{key}_rc"] = rt.restrict(tp, U).values
            ec = np.where(tp.coarse.mask, rng.standard_normal(tp.coarse.mask.shape), 0.0)
            d[f"{key}_ec"] = ec
            d[f"{key}_Pe"] = rt.prolong(tp, rg.GridFunction(tp.coarse, ec)).values
            Ac = rt.galerkin_product(S, tp)
            d[f"{key}_Ac"] = Ac.data
            d[f"{key}_maskc"] = tp.coarse.mask
            lu, perm = rd.lu_factor(rg.materialize_stencil(Ac))
            d[f"{key}_lu"] = lu
            d[f"{key}_perm"] = perm
            b = rng.standard_normal(tp.coarse.n_active)
            d[f"{key}_lub"] = b
            d[f"{key}_lux"] = rd.lu_solve(lu, perm, b)
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **d)


def run_case(name, A, mask, levels, smoother, nu, cycles, f, h, store_levels=True):
    """Reference hierarchy + fixed-count V(nu, nu) cycle loop."""
    spec = spec_of(mask, h)
    S = rg.StencilField(spec, A)
    hier = rh.build_hierarchy(S, levels)
    if smoother == "jacobi":
        rh.equip_classical(hier, "jacobi")
    else:
        rh.equip_inferred(hier, smoother)
    if nu > 1:
        for lev in hier.levels[:-1]:
            lev.smoother = RepeatedSmoother(lev.smoother, lev.operator, nu)
    F = rg.GridFunction(spec, f)
    u = rg.zeros(spec)
    denom = F.norm() if F.norm() > 0 else 1.0
    hist = [(F - rg.apply_stencil(S, u)).norm() / denom]
    for _ in range(cycles):
        u = rh.v_cycle(hier, 0, F, u)
        hist.append((F - rg.apply_stencil(S, u)).norm() / denom)
    d = {"u": u.values, "history": np.array(hist),
         "levels": levels, "nu": nu, "cycles": cycles, "h": h}
    if store_levels:                       # large cases regenerate A0 / f from their seeds
        d.update({"A0": A, "mask": mask, "f": F.values})
    if store_levels:
        for l, lev in enumerate(hier.levels):
            d[f"A{l}"] = lev.operator.data
            d[f"mask{l}"] = lev.spec.mask
            sm = lev.smoother
            if sm is not None:
                inner = sm.inner if isinstance(sm, RepeatedSmoother) else sm
                if isinstance(inner, rs.InferredSmoother):
                    d[f"K{l}"] = inner.kernels
        d["coarse_lu"] = hier.coarse_lu
        d["coarse_perm"] = hier.coarse_perm
    else:
        for l, lev in enumerate(hier.levels):
            d[f"Asum{l}"] = np.array([lev.operator.data.sum(), np.abs(lev.operator.data).sum()])
            sm = lev.smoother
            if sm is not None:
                inner = sm.inner if isinstance(sm, RepeatedSmoother) else sm
                if isinstance(inner, rs.InferredSmoother):
                    K = inner.kernels
                    d[f"Ksum{l}"] = np.array([K.sum(), np.abs(K).sum()])
                    d[f"Kmid{l}"] = K[K.shape[0] // 2, K.shape[1] // 2]
                    d[f"Kcorner{l}"] = K[0, 0]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(f"{name}: hist[-1]={hist[-1]:.3e}")


def make_problem_pins():
    """Reference assembly tables that pin the host-side generators."""
    d = {}
    for i, (n, th, ep) in enumerate([(7, math.pi / 6, 100.0), (255, math.pi / 6, 0.01),
                                      (4095, math.pi / 4, 1e-3), (511, 1.234, 0.05)]):
        S = rp.assemble_rotated_laplacian(rg.full_spec(n), th, ep)
        d[f"rot{i}"] = S.data[0, 0]
        d[f"rot{i}_params"] = np.array([n, th, ep])
    np.savez_compressed(os.path.join(HERE, "problems.npz"), **d)


def make_krylov(nets):
    """krylov.npz: the reference's fgmres / gmres (krylov.py) with grid_action and
    cycle_preconditioner on small stencil problems."""
    from mgsmooth import krylov as rk
    d = {}
    n = 31
    A = gen.rotated_fd(n, math.pi / 6, 0.01)     # the conv net's training operator family
    full = np.ones((n, n), bool)
    lsh = gen.geometry_mask("lshape", n)
    Av = rp.assemble_variable_diffusion(rg.full_spec(n), 10.0).data
    cases = [
        # name, A, mask, smoother/net, nu (None = no preconditioner), method, tol, max_iter, restart
        ("fg_conv_v11", A, full, nets["conv"], 1, "fgmres", 1e-10, 30, None),
        ("fg_conv_v22", A, full, nets["conv"], 2, "fgmres", 1e-10, 30, None),
        ("fg_lshape_v11", A, lsh, nets["conv"], 1, "fgmres", 1e-10, 30, None),
        ("fg_var_v22", Av, full, nets["conv"], 2, "fgmres", 1e-10, 30, 6),
        ("fg_jacobi_v11", A, full, "jacobi", 1, "fgmres", 1e-9, 40, None),
        ("fg_none_restart", A, full, None, None, "fgmres", 1e-8, 60, 8),
        ("fg_maxiter", A, full, nets["conv"], 1, "fgmres", 1e-14, 3, None),
        ("gm_restart", A, full, None, None, "gmres", 1e-9, 80, 10),
        ("gm_lshape", A, lsh, None, None, "gmres", 1e-8, 50, None),
    ]
    for name, Ac, mask, sm, nu, method, tol, max_iter, restart in cases:
        spec = spec_of(mask, 1 / (n + 1))
        S = rg.StencilField(spec, Ac)
        f = np.where(mask, gen.uniform_rhs(n, 9), 0.0).ravel()
        cfg = rk.FgmresConfig(tol=tol, max_iter=max_iter, restart=restart)
        pc = None
        if nu is not None:
            hier = rh.build_hierarchy(S, 4)
            if sm == "jacobi":
                rh.equip_classical(hier, "jacobi")
            else:
                rh.equip_inferred(hier, sm)
            if nu > 1:
                for lev in hier.levels[:-1]:
                    lev.smoother = RepeatedSmoother(lev.smoother, lev.operator, nu)
            pc = rk.cycle_preconditioner(hier)
        if method == "fgmres":
            u, rep = rk.fgmres(rk.grid_action(S), f, precond=pc, cfg=cfg)
        else:
            u, rep = rk.gmres(rk.grid_action(S), f, cfg=cfg)
        d[f"{name}/A"] = Ac
        d[f"{name}/mask"] = mask
        d[f"{name}/f"] = f
        d[f"{name}/u"] = u
        d[f"{name}/history"] = np.array(rep.history)
        d[f"{name}/meta"] = np.array([-1 if nu is None else nu, 0 if method == "fgmres" else 1, tol, max_iter,
                                      0 if restart is None else restart, rep.iterations, int(rep.converged)])
        d[f"{name}/smoother"] = np.array("none" if sm is None else ("jacobi" if sm == "jacobi" else "conv"))
        print(f"krylov {name}: iters={rep.iterations} conv={rep.converged} hist[-1]={rep.history[-1]:.3e}")
    np.savez_compressed(os.path.join(HERE, "krylov.npz"), **d)


def _conv_params(sm):
    return {"form": np.array(sm.form), "activation": np.array(sm.activation), "slope": sm.slope, "gain": sm.gain,
            "layers": np.stack([k.weights for k in sm.layers]),
            "skip": sm.skip.weights if sm.skip is not None else np.zeros((0, 3, 3))}


def _random_conv(spec, A, form, activation, seed, scale=0.05, omega=2.0 / 3.0):
    """A 'trained-looking' conv smoother: the Jacobi-equivalent initialisation
    (smoothers.py:148-164) plus seeded perturbations of every kernel."""
    rng = np.random.default_rng(seed)
    base = rs.conv_smoother(rg.StencilField(spec, A.data) if isinstance(A, rg.StencilField) else A, form, omega,
                            activation)
    layers = [rg.ConvKernel(k.weights + scale * rng.standard_normal((3, 3))) for k in base.layers]
    skip = None if base.skip is None else rg.ConvKernel(base.skip.weights + scale * rng.standard_normal((3, 3)))
    return rs.ConvSmoother(base.spec, form, layers, skip, activation, base.slope, base.gain)


def make_conv():
    """conv.npz: convolve / ConvSmoother.apply / effective_kernel pins and V-cycles
    with shared-kernel conv smoothers (equip_conv_init, perturbed full / rb forms,
    leaky activation, masked domain, equip_trained transport)."""
    d = {}
    rng = np.random.default_rng(77)
    n = 23
    for gname in ("square", "lshape"):
        mask = gen.geometry_mask(gname, n) if gname != "square" else np.ones((n, n), bool)
        spec = spec_of(mask, 1 / (n + 1))
        u = rg.GridFunction(spec, np.where(mask, rng.standard_normal((n, n)), 0.0))
        w = rng.standard_normal((3, 3))
        w[0, 2] = 0.0
        w[1, 0] = 0.0
        d[f"convolve/{gname}/w"] = w
        d[f"convolve/{gname}/mask"] = mask
        d[f"convolve/{gname}/u"] = u.values
        d[f"convolve/{gname}/out"] = rg.convolve(rg.ConvKernel(w), u).values
        A = rg.StencilField(spec, gen.rotated_fd(n, 0.4, 0.05))
        for form, act in (("full", "linear"), ("full", "leaky"), ("rb", "linear"), ("rb", "leaky")):
            sm = _random_conv(spec, A, form, act, seed=len(d), scale=0.3)
            key = f"apply/{gname}/{form}_{act}"
            for k2, v in _conv_params(sm).items():
                d[f"{key}/{k2}"] = v
            d[f"{key}/r"] = u.values
            d[f"{key}/out"] = sm.apply(u).values
            if act == "linear":
                d[f"{key}/effective"] = rs.effective_kernel(sm).weights
    # V-cycles: rotated FD 31^2, 4 levels
    n = 31
    A = gen.rotated_fd(n, math.pi / 6, 0.01)
    f = gen.uniform_rhs(n, 12)
    cases = [("init_v11", None, "init", "linear", 1), ("full_lin_v22", None, "full", "linear", 2),
             ("full_leaky_v11", None, "full", "leaky", 1), ("rb_lin_v22", None, "rb", "linear", 2),
             ("lshape_full_v11", "lshape", "full", "linear", 1)]
    for name, geom, form, act, nu in cases:
        mask = np.ones((n, n), bool) if geom is None else gen.geometry_mask(geom, n)
        spec = spec_of(mask, 1 / (n + 1))
        S = rg.StencilField(spec, A)
        hier = rh.build_hierarchy(S, 4)
        if form == "init":
            rh.equip_conv_init(hier)
        else:
            for l, lev in enumerate(hier.levels[:-1]):
                lev.smoother = _random_conv(lev.spec, lev.operator, form, act, seed=100 + l)
        for l, lev in enumerate(hier.levels[:-1]):
            for k2, v in _conv_params(lev.smoother).items():
                d[f"cycle/{name}/L{l}/{k2}"] = v
            if nu > 1:
                lev.smoother = RepeatedSmoother(lev.smoother, lev.operator, nu)
        F = rg.GridFunction(spec, np.where(mask, f, 0.0))
        u = rg.zeros(spec)
        hist = [(F - rg.apply_stencil(S, u)).norm() / F.norm()]
        for _ in range(8):
            u = rh.v_cycle(hier, 0, F, u)
            hist.append((F - rg.apply_stencil(S, u)).norm() / F.norm())
        d[f"cycle/{name}/A0"] = A
        d[f"cycle/{name}/mask"] = mask
        d[f"cycle/{name}/f"] = F.values
        d[f"cycle/{name}/nu"] = nu
        d[f"cycle/{name}/history"] = np.array(hist)
        d[f"cycle/{name}/u"] = u.values
        print(f"conv {name}: hist[-1]={hist[-1]:.3e}")
    # transport: smoothers of a 15^2 source hierarchy into a 31^2 target (equip_trained)
    src = rh.build_hierarchy(rg.StencilField(rg.full_spec(15), gen.rotated_fd(15, math.pi / 6, 0.01)), 3)
    for l, lev in enumerate(src.levels[:-1]):
        lev.smoother = _random_conv(lev.spec, lev.operator, "full", "linear", seed=200 + l)
    tgt = rh.build_hierarchy(rg.StencilField(rg.full_spec(n), A), 4)
    rh.equip_trained(tgt, src)
    for l, lev in enumerate(src.levels[:-1]):
        for k2, v in _conv_params(lev.smoother).items():
            d[f"transport/src/L{l}/{k2}"] = v
    for l, lev in enumerate(tgt.levels[:-1]):
        d[f"transport/tgt/L{l}/gain"] = lev.smoother.gain
    F = rg.GridFunction(rg.full_spec(n), f)
    u = rg.zeros(F.spec)
    hist = [F.norm() / F.norm()]
    for _ in range(6):
        u = rh.v_cycle(tgt, 0, F, u)
        hist.append((F - rg.apply_stencil(rg.StencilField(F.spec, A), u)).norm() / F.norm())
    d["transport/history"] = np.array(hist)
    d["transport/u"] = u.values
    np.savez_compressed(os.path.join(HERE, "conv.npz"), **d)


def main():
    if "--only-conv" in sys.argv:
        make_conv()
        return
    if "--only-krylov" in sys.argv:
        make_krylov(make_nets())
        return
    make_problem_pins()
    nets = make_nets()
    make_ops()
    # small structural cases (all-level A and K stored)
    n = 15
    A = gen.rotated_fd(n, math.pi / 6, 0.01)
    f = gen.uniform_rhs(n, 0)
    run_case("case_rot15_conv_v22", A, np.ones((n, n), bool), 3, nets["conv"], 2, 10, f, 1 / (n + 1))
    run_case("case_rot15_jacobi_v11", A, np.ones((n, n), bool), 3, "jacobi", 1, 10, f, 1 / (n + 1))
    run_case("case_rot15_convk2_v11", A, np.ones((n, n), bool), 3, nets["conv_k2"], 1, 6, f, 1 / (n + 1))
    n = 31
    A = gen.rotated_fd(n, math.pi / 4, 0.001)
    f = gen.uniform_rhs(n, 1)
    run_case("case_rot31_fc_v22", A, np.ones((n, n), bool), 4, nets["fc"], 2, 8, f, 1 / (n + 1))
    mask = gen.geometry_mask("lshape", n)
    fm = np.where(mask, f, 0.0)
    run_case("case_lshape31_conv_v11", A, mask, 4, nets["conv"], 1, 8, fm, 1 / (n + 1))
    mask = gen.geometry_mask("cylinder", n)
    fm = np.where(mask, f, 0.0)
    run_case("case_cyl31_fc_v11", A, mask, 3, nets["fc"], 1, 6, fm, 1 / (n + 1))
    # variable coefficient (reference bilinear-FE assembly) and config-3 style 5-point GRF
    spec = rg.full_spec(31)
    Av = rp.assemble_variable_diffusion(spec, 10.0).data
    run_case("case_var31_conv_v22", Av, np.ones((31, 31), bool), 4, nets["conv"], 2, 8, gen.uniform_rhs(31, 2), spec.spacing)
    Ag = gen.grf_diffusion_5pt(63, seed=2)
    run_case("case_grf63_conv_v22", Ag, np.ones((63, 63), bool), 5, nets["conv"], 2, 8, gen.uniform_rhs(63, 2), 1 / 63)
    # non-square + even sizes
    Ar = gen.rotated_fd(20, math.pi / 3, 0.01, cols=27)
    run_case("case_rect20x27_conv_v11", Ar, np.ones((20, 27), bool), 3, nets["conv"], 1, 6,
             gen.uniform_rhs(20, 3, cols=27), 1 / 21)
    # config 1: 255^2 rotated FD eps=0.01 theta=pi/6, V(2,2), 20 cycles, conv net
    n = 255
    run_case("c1_fd_conv", gen.rotated_fd(n, math.pi / 6, 0.01), np.ones((n, n), bool), 7, nets["conv"], 2, 20,
             gen.uniform_rhs(n, 0), 1 / (n + 1), store_levels=False)
    run_case("c1_q1_conv", gen.rotated_q1(n, math.pi / 6, 0.01), np.ones((n, n), bool), 7, nets["conv"], 2, 20,
             gen.uniform_rhs(n, 0), 1 / (n + 1), store_levels=False)
    # config 4 sample: first two problems of the batch, 511^2, V(1,1), 10 cycles
    eps, theta = gen.batch_parameters(256, seed=3)
    n = 511
    for i in range(2):
        run_case(f"c4_p{i}", gen.rotated_fd(n, theta[i], eps[i]), np.ones((n, n), bool), 8, nets["conv"], 1, 10,
                 gen.uniform_rhs(n, [4, i]), 1 / (n + 1), store_levels=False)
    make_krylov(nets)
    make_conv()


if __name__ == "__main__":
    main()
