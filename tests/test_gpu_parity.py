"""GPU parity of the CUDA path (through the C-ABI via the facade) against the
golden vectors produced by the unmodified reference and against the CPU
oracle.  Tolerances:
  * stencil / transfer / Galerkin: bit-exact (same operation order, no FMA);
  * hierarchy operators: bit-exact; level sizes, masks, k: exact;
  * fp64 CNN kernels: max|dK| / max|K| <= 1e-13 per level;
  * V-cycle histories and u: 1e-10 relative (+1e-14 absolute on histories);
  * fp32 CNN inference: max|dK| / max|K| <= 1e-5 per level.
"""

import math
import threading

import numpy as np
import pytest

import paper_2102_12071_b200 as mg
from oracle import mg_oracle as mo
from paper_2102_12071_b200 import problems as gen

from cases import LARGE, SMALL, load
from conftest import rel_err

pytestmark = pytest.mark.gpu

KEYS = ["square9", "lshape9", "cylinder9", "square10"]
HIST_RTOL, HIST_ATOL = 1e-10, 1e-14


def spec_of(mask, h):
    return mg.GridSpec(mask.shape[0], mask.shape[1], h, mask)


def net_of(name, nets_dir=None):
    import os
    from conftest import GOLDEN
    return mg.load_model(os.path.join(GOLDEN, f"net_{name}.json"))


def assert_hist(h, g):
    h = np.asarray(h)
    g = np.asarray(g)
    assert h.shape == g.shape
    assert np.all(np.abs(h - g) <= HIST_RTOL * np.abs(g) + HIST_ATOL), (h, g)


# ---------------------------------------------------------------------------
# stateless ops: bit-exact against the reference

@pytest.mark.parametrize("key", KEYS)
def test_apply_stencil_bit_exact(ops_golden, key):
    g = ops_golden
    spec = spec_of(g[f"{key}_mask"], 0.1)
    out = mg.apply_stencil(mg.StencilField(spec, g[f"{key}_A"]), mg.GridFunction(spec, g[f"{key}_u"]))
    assert np.array_equal(out.values, g[f"{key}_Au"])


@pytest.mark.parametrize("key", KEYS)
def test_transfers_bit_exact(ops_golden, key):
    g = ops_golden
    spec = spec_of(g[f"{key}_mask"], 0.1)
    tp = mg.coarsen_full(spec)
    assert np.array_equal(tp.coarse.mask, g[f"{key}_maskc"])
    rc = mg.restrict(tp, mg.GridFunction(spec, g[f"{key}_u"]))
    assert np.array_equal(rc.values, g[f"{key}_rc"])
    pe = mg.prolong(tp, mg.GridFunction(tp.coarse, g[f"{key}_ec"]))
    assert np.array_equal(pe.values, g[f"{key}_Pe"])


@pytest.mark.parametrize("key", KEYS)
def test_galerkin_bit_exact(ops_golden, key):
    g = ops_golden
    spec = spec_of(g[f"{key}_mask"], 0.1)
    Ac = mg.galerkin_product(mg.StencilField(spec, g[f"{key}_A"]), mg.coarsen_full(spec))
    assert np.array_equal(Ac.data, g[f"{key}_Ac"])


def test_constant_prolongs_to_half():
    """tests/test_transfer.py:50 of the reference: P(1) = 0.5 at odd/odd points."""
    spec = mg.full_spec(15)
    tp = mg.coarsen_full(spec)
    pe = mg.prolong(tp, mg.GridFunction(tp.coarse, np.ones((7, 7))))
    assert np.all(pe.values[1::2, 1::2] == 0.5)


@pytest.mark.parametrize("key", KEYS)
def test_device_lu(ops_golden, key):
    import ctypes as C
    from paper_2102_12071_b200 import _lib, device as dv
    g = ops_golden
    M = mo.materialize(g[f"{key}_Ac"], g[f"{key}_maskc"])
    n = M.shape[0]
    lu = dv.to_dev(M)
    perm = dv.to_dev(np.zeros(n, np.int32))
    _lib.call("mgb_lu_factor", n, dv.ptr(lu), dv.ptr(perm), dv.stream(lu))
    assert np.array_equal(dv.host(perm), g[f"{key}_perm"])
    assert np.array_equal(dv.host(lu), g[f"{key}_lu"])
    b = dv.to_dev(g[f"{key}_lub"])
    x = dv.empty((n,))
    _lib.call("mgb_lu_solve", n, dv.ptr(lu), dv.ptr(perm), dv.ptr(b), dv.ptr(x), dv.stream(x))
    assert np.array_equal(dv.host(x), g[f"{key}_lux"])


def test_singular_coarsest_raises_with_pivot():
    from paper_2102_12071_b200 import _lib, device as dv
    M = np.array([[1.0, 2.0], [2.0, 4.0]])
    lu = dv.to_dev(M)
    perm = dv.to_dev(np.zeros(2, np.int32))
    with pytest.raises(mg.SingularMatrixError) as ei:
        _lib.call("mgb_lu_factor", 2, dv.ptr(lu), dv.ptr(perm), dv.stream(lu))
    assert ei.value.pivot_index == 1
    # a zero operator makes the hierarchy's coarsest LU singular
    spec = mg.full_spec(7)
    with pytest.raises(mg.SingularMatrixError):
        mg.build_hierarchy(mg.StencilField(spec, np.zeros((7, 7, 3, 3))), 2)


# ---------------------------------------------------------------------------
# hierarchies: operators, kernels, cycles

def _equip(h, smoother, precision=64):
    if smoother == "jacobi":
        return mg.equip_classical(h, "jacobi")
    return mg.equip_inferred(h, net_of(smoother), precision)


@pytest.mark.parametrize("name", sorted(SMALL))
def test_hierarchy_operators_and_kernels(name):
    c = load(name)
    g = c["golden"]
    spec = spec_of(c["mask"], float(g["h"]))
    h = mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"])
    assert h.depth == c["levels"]
    for l in range(h.depth):
        lev = h.levels[l]
        assert np.array_equal(lev.spec.mask, g[f"mask{l}"])
        assert np.array_equal(lev.operator.data, g[f"A{l}"]), f"level {l}"
    _equip(h, c["smoother"])
    for l in range(h.depth - 1):
        if f"K{l}" in g:
            assert rel_err(h.levels[l].smoother.kernels, g[f"K{l}"]) <= 1e-13


@pytest.mark.parametrize("name", sorted(SMALL) + sorted(LARGE))
def test_cycles_match_reference_history(name):
    c = load(name)
    g = c["golden"]
    spec = spec_of(c["mask"], float(g["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), c["smoother"])
    from paper_2102_12071_b200 import device as dv
    f = dv.to_dev(np.where(c["mask"], c["f"], 0.0))
    u = dv.zeros(f.shape)
    hist = h.run_cycles(f, u, c["cycles"], c["nu"], c["nu"], u_zero=True)
    assert_hist(dv.host(hist)[0], g["history"])
    assert rel_err(dv.host(u), g["u"]) <= 1e-10


def test_v_cycle_facade_with_repeated_smoother():
    """The reference's V(2,2) convention (RepeatedSmoother) maps to 2 device sweeps."""
    c = load("case_rot15_conv_v22")
    g = c["golden"]
    spec = spec_of(c["mask"], float(g["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), "conv")
    for lev in h.levels[:-1]:
        lev.smoother = mg.RepeatedSmoother(lev.smoother, lev.operator, 2)
    F = mg.GridFunction(spec, c["f"])
    u = mg.zeros(spec)
    for _ in range(c["cycles"]):
        u = mg.v_cycle(h, 0, F, u)
    assert rel_err(u.values, g["u"]) <= 1e-10


def test_solve_report_contract():
    """tests/test_hierarchy.py:68 of the reference: history[0] = 1 from u0 = 0,
    len = iterations + 1, certified residual, converged flag."""
    c = load("case_var31_conv_v22")
    spec = spec_of(c["mask"], float(c["golden"]["h"]))
    A = mg.StencilField(spec, c["A0"])
    h = _equip(mg.build_hierarchy(A, c["levels"]), "conv")
    F = mg.GridFunction(spec, c["f"])
    u, rep = mg.solve(h, F, tol=1e-8, max_iter=50)
    assert rep.converged and rep.residual_history[0] == 1.0
    assert len(rep.residual_history) == rep.iterations + 1
    r = (F - mg.apply_stencil(A, u)).norm() / F.norm()
    assert abs(r - rep.residual_history[-1]) <= 1e-12 * max(r, 1e-300) + 1e-15
    # oracle cross-check of the whole history (V(1,1), solve semantics)
    ho = mo.equip_inferred(mo.build_hierarchy(c["A0"], c["levels"]), mo.load_net_json(
        __import__("os").path.join(__import__("conftest").GOLDEN, "net_conv.json")))
    _, hist, it, conv = mo.solve(ho, c["f"], tol=1e-8, max_iter=50)
    assert it == rep.iterations and conv
    assert_hist(rep.residual_history, hist)
    # non-converged flag at a tiny max_iter
    _, rep2 = mg.solve(h, F, tol=1e-30, max_iter=2)
    assert rep2.iterations == 2 and not rep2.converged


def test_solve_divergence_raises():
    """hierarchy.py:142-144: history > 1e6 max(r0, tol) -> NonConvergedError.  An
    over-relaxed point smoother (3 / diag: Jacobi with omega = 3, which jacobi()
    itself rejects, installed as per-point kernels) diverges deterministically; the
    oracle (same guard) raises at the same iteration."""
    n = 63
    A = gen.rotated_fd(n, math.pi / 3, 0.01)
    spec = mg.full_spec(n)
    h = mg.build_hierarchy(mg.StencilField(spec, A), 5)
    for lev in h.levels[:-1]:
        K = mo.jacobi_kernels(lev.operator.data, lev.spec.mask, 3.0)
        lev.smoother = mg.InferredSmoother(lev.spec, K, 1)
    f = gen.uniform_rhs(n, 0)
    with pytest.raises(mg.NonConvergedError) as ei:
        mg.solve(h, mg.GridFunction(spec, f), tol=1e-12, max_iter=200)
    with pytest.raises(mo.OracleError) as eo:
        mo.solve(mo.equip_jacobi(mo.build_hierarchy(A, 5), omega=3.0), f, tol=1e-12, max_iter=200)
    assert "NonConvergedError" in str(eo.value)
    import re
    it = [re.search(r"iteration (\d+)", str(e.value)) for e in (ei, eo)]
    assert all(it) and it[0].group(1) == it[1].group(1), (str(ei.value), str(eo.value))


def test_coarse_solve_exact():
    c = load("case_rot15_conv_v22")
    spec = spec_of(c["mask"], float(c["golden"]["h"]))
    h = mg.build_hierarchy(mg.StencilField(spec, c["A0"]), 2)
    Ac = h.levels[1].operator
    rng = np.random.default_rng(0)
    b = rng.standard_normal(Ac.data.shape[:2])
    x = mg.coarse_solve(h, mg.GridFunction(Ac.spec, b))
    want = np.linalg.solve(mo.materialize(Ac.data, Ac.spec.mask), b.ravel())
    assert np.max(np.abs(x.values.ravel() - want)) < 1e-10


def test_batched_hierarchy_matches_single_problems():
    """Config 4 path: two 511^2 problems in one batched hierarchy."""
    from paper_2102_12071_b200 import device as dv
    cs = [load("c4_p0"), load("c4_p1")]
    A = np.stack([c["A0"] for c in cs])
    h = mg.build_hierarchy_batch(A, 8)
    mg.equip_inferred(h, net_of("conv"))
    f = dv.to_dev(np.stack([c["f"] for c in cs]))
    u = dv.zeros(f.shape)
    hist = dv.host(h.run_cycles(f, u, 10, 1, 1, u_zero=True))
    U = dv.host(u)
    for b, c in enumerate(cs):
        assert_hist(hist[b], c["golden"]["history"])
        assert rel_err(U[b], c["golden"]["u"]) <= 1e-10


def test_fp32_inference_within_tolerance():
    c = load("c1_fd_conv")
    spec = mg.full_spec(255)
    A = mg.StencilField(spec, c["A0"])
    h64 = _equip(mg.build_hierarchy(A, 7), "conv", 64)
    h32 = _equip(mg.build_hierarchy(A, 7), "conv", 32)
    for l in range(6):
        K64 = h64.levels[l].smoother.kernels
        K32 = h32.levels[l].smoother.kernels
        assert rel_err(K32, K64) <= 1e-5
    hf = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), 7), "fc", 32)
    hd = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), 7), "fc", 64)
    for l in range(6):
        assert rel_err(hf.levels[l].smoother.kernels, hd.levels[l].smoother.kernels) <= 1e-5


# ---------------------------------------------------------------------------
# oracle cross-checks at sizes without golden vectors (masks, rectangles, k>1)

@pytest.mark.parametrize("rows,cols,geom,nu,variant", [
    (48, 64, "square", 1, "fc"),
    (63, 63, "cylinder", 2, "conv"),
    (33, 45, "square", 2, "conv_k2"),
    (127, 127, "lshape", 1, "conv"),
])
def test_random_operators_vs_oracle(rows, cols, geom, nu, variant):
    from paper_2102_12071_b200 import device as dv
    rng = np.random.default_rng(rows * cols)
    mask = gen.geometry_mask(geom, rows) if rows == cols else np.ones((rows, cols), bool)
    A = gen.rotated_fd(rows, 0.7, 0.05, cols=cols)
    A = A * (1.0 + 0.3 * rng.random((rows, cols, 1, 1)))   # per-point variation
    f = np.where(mask, rng.uniform(-1, 1, (rows, cols)), 0.0)
    levels = 4
    spec = spec_of(mask, 1.0 / (rows + 1))
    net = net_of(variant)
    h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(spec, A), levels), net)
    fd = dv.to_dev(f)
    u = dv.zeros(f.shape)
    hist = dv.host(h.run_cycles(fd, u, 5, nu, nu, u_zero=True))[0]
    ho = mo.equip_inferred(mo.build_hierarchy(A, levels, mask), mo.load_net_json(
        __import__("os").path.join(__import__("conftest").GOLDEN, f"net_{variant}.json")))
    uo, ho_hist = mo.run_cycles(ho, f, 5, nu, nu)
    assert_hist(hist, ho_hist)
    assert rel_err(dv.host(u), uo) <= 1e-10


# ---------------------------------------------------------------------------
# properties at full benchmark size (config 2: 4095^2)

@pytest.mark.slow
def test_config2_properties_full_size():
    """Size-independent checks at 4095^2: (1) runs are bitwise reproducible,
    (2) the Jacobi-smoothed V-cycle is linear in f (V(f1+f2) = V(f1)+V(f2) from
    u = 0, to round-off), (3) the learned-smoother history decreases."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    n = 4095
    A = gen.rotated_fd(n, math.pi / 4, 1e-3)
    h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), 11), net_of("conv_c2"))
    f = dv.to_dev(gen.uniform_rhs(n, 1))
    u1, u2 = dv.zeros(f.shape), dv.zeros(f.shape)
    h1 = h.run_cycles(f, u1, 3, 2, 2, u_zero=True).clone()
    h2 = h.run_cycles(f, u2, 3, 2, 2, u_zero=True).clone()
    assert t.equal(u1, u2) and t.equal(h1, h2)
    hh = dv.host(h1)[0]
    assert np.all(np.diff(hh) < 0)
    hj = mg.equip_classical(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), 11), "jacobi")
    fa = dv.to_dev(gen.uniform_rhs(n, 5))
    fb = dv.to_dev(gen.uniform_rhs(n, 6))
    ua, ub, uab = dv.zeros(f.shape), dv.zeros(f.shape), dv.zeros(f.shape)
    hj.run_cycles(fa, ua, 1, 1, 1, u_zero=True)
    hj.run_cycles(fb, ub, 1, 1, 1, u_zero=True)
    hj.run_cycles(fa + fb, uab, 1, 1, 1, u_zero=True)
    err = (uab - ua - ub).abs().max().item() / uab.abs().max().item()
    assert err < 1e-12


def test_concurrent_solves_share_one_hierarchy():
    """a built hierarchy is immutable; concurrent solves are safe."""
    c = load("case_var31_conv_v22")
    spec = spec_of(c["mask"], float(c["golden"]["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), "conv")
    F = mg.GridFunction(spec, c["f"])
    ref = mg.solve(h, F, tol=1e-8)[1].residual_history
    out = {}

    def run(i):
        import torch
        with torch.cuda.stream(torch.cuda.Stream()):
            out[i] = mg.solve(h, F, tol=1e-8)[1].residual_history

    ts = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for i in range(4):
        assert out[i] == ref


@pytest.mark.parametrize("name", ["c1_fd_conv", "c1_q1_conv", "case_var31_conv_v22", "case_rot31_fc_v22"])
def test_storage_modes_bit_identical(name):
    """Band-class tables vs per-point planes: same values, bit-identical cycles."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    c = load(name)
    g = c["golden"]
    spec = spec_of(c["mask"], float(g["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), c["smoother"])
    info = [h.storage_info(l) for l in range(h.depth - 1)]
    if name.startswith("c1") or "rot31" in name:
        assert all(a and k for a, k in info), info      # constant-coefficient chain is class-compact
    if "var31" in name:
        assert not info[0][0]                            # variable coefficients stay per-point
    f = dv.to_dev(np.where(c["mask"], c["f"], 0.0))
    u1, u2 = dv.zeros(f.shape), dv.zeros(f.shape)
    h1 = h.run_cycles(f, u1, 4, c["nu"], c["nu"], u_zero=True).clone()
    h.set_storage("planes")
    assert not any(h.storage_info(l)[0] for l in range(h.depth))
    h2 = h.run_cycles(f, u2, 4, c["nu"], c["nu"], u_zero=True).clone()
    assert t.equal(u1, u2)
    assert np.allclose(dv.host(h1), dv.host(h2), rtol=1e-14, atol=0)


@pytest.mark.parametrize("name", ["c1_fd_conv", "case_var31_conv_v22", "case_lshape31_conv_v11", "c4_p0",
                                  "case_rect20x27_conv_v11"])
def test_fused_and_separate_passes_agree(name):
    """Row-streaming PRE/POST passes vs separate sweep/restrict/prolong passes."""
    from paper_2102_12071_b200 import device as dv
    c = load(name)
    g = c["golden"]
    spec = spec_of(c["mask"], float(g["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), c["smoother"])
    f = dv.to_dev(np.where(c["mask"], c["f"], 0.0))
    u1, u2 = dv.zeros(f.shape), dv.zeros(f.shape)
    h1 = dv.host(h.run_cycles(f, u1, c["cycles"], c["nu"], c["nu"], u_zero=True))[0]
    for mode in (1, 0):
        h.set_fused(mode)
        u2 = dv.zeros(f.shape)
        h2 = dv.host(h.run_cycles(f, u2, c["cycles"], c["nu"], c["nu"], u_zero=True))[0]
        assert_hist(h1, h2)
        assert rel_err(dv.host(u1), dv.host(u2)) <= 1e-12


@pytest.mark.parametrize("n,cols,variant,nu", [(255, 255, "conv", 2), (127, 127, "fc", 1), (20, 27, "conv", 1),
                                               (64, 48, "jacobi", 2)])
def test_classed_only_hierarchy_matches_per_point_build(n, cols, variant, nu):
    """A hierarchy held only as band-class tables equals the per-point build:
    operators and kernels on every level, and the cycle histories, bitwise."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    A = gen.rotated_fd(n, 0.9, 0.02, cols=cols)
    levels = gen.levels_for(min(n, cols))
    h1 = mg.build_hierarchy(mg.StencilField(mg.GridSpec(n, cols, 1.0 / (n + 1), np.ones((n, cols), bool)), A),
                            levels)
    h2 = mg.build_hierarchy_classed(n, cols, A[0, 0], levels)
    for l in range(h1.depth):
        assert np.array_equal(h1.operator_batch(l), h2.operator_batch(l)), l
    _equip(h1, variant)
    _equip(h2, variant)
    for l in range(h1.depth - 1):
        assert np.array_equal(h1.kernels_batch(l), h2.kernels_batch(l)), l
    f = dv.to_dev(gen.uniform_rhs(n, 7, cols=cols))
    u1, u2 = dv.zeros(f.shape), dv.zeros(f.shape)
    a = h1.run_cycles(f, u1, 5, nu, nu, u_zero=True).clone()
    b = h2.run_cycles(f, u2, 5, nu, nu, u_zero=True).clone()
    assert t.equal(u1, u2) and t.equal(a, b)


@pytest.mark.parametrize("n,nparts,nu", [(511, 2, 2), (511, 3, 1), (1023, 4, 2), (255, 2, 2)])
def test_virtual_domain_decomposition_matches_single_domain(n, nparts, nu, monkeypatch):
    """Row-block decomposition on one GPU (halos by device copies, agglomerated
    coarse levels): u is bitwise the single-domain result, histories agree to
    rounding (only the norm summation order differs)."""
    from paper_2102_12071_b200 import dd, device as dv
    monkeypatch.setenv("MGB_STREAM_MIN", "0")       # streaming passes on every level, as the decomposition
    t = dv.torch()
    table = gen.rotated_fd(1, math.pi / 3, 0.01, h=1.0 / (n + 1))[0, 0]
    levels = gen.levels_for(n)
    h = mg.equip_inferred(mg.build_hierarchy_classed(n, n, table, levels), net_of("conv"))
    f_full = dv.to_dev(gen.uniform_rhs(n, 11))
    u_ref = dv.zeros(f_full.shape)
    hist_ref = dv.host(h.run_cycles(f_full, u_ref, 4, nu, nu, u_zero=True))[0]
    agg = n // 4
    s = dd.DecomposedSolver(h, nparts, local=True, agglomerate_rows=agg)
    assert s.distributed_levels >= 1
    blocks = [s.rows(p) for p in range(nparts)]
    assert blocks == dd.partition_rows(n, nparts, s.distributed_levels)
    for p, (r0, r1) in enumerate(blocks):
        s.set_rhs(p, f_full[r0:r1].contiguous())
    hist = dv.host(s.run_cycles(4, nu, nu))
    u = t.cat([s.solution(p) for p in range(nparts)])
    assert t.equal(u, u_ref), float((u - u_ref).abs().max())
    assert np.allclose(hist, hist_ref, rtol=1e-13, atol=0)


def test_nccl_decomposition_single_rank(monkeypatch):
    """The NCCL backend of the decomposition (dlopen'd NCCL, communicator init,
    graph-captured all-gather / all-reduce) on a 1-rank communicator: identical to
    the single-domain solve.  Multi-rank halos need several GPUs."""
    import torch.distributed as dist
    from paper_2102_12071_b200 import dd, device as dv
    monkeypatch.setenv("MGB_STREAM_MIN", "0")
    t = dv.torch()
    n = 511
    table = gen.rotated_fd(1, math.pi / 3, 0.01, h=1.0 / (n + 1))[0, 0]
    h = mg.equip_inferred(mg.build_hierarchy_classed(n, n, table, gen.levels_for(n)), net_of("conv"))
    f = dv.to_dev(gen.uniform_rhs(n, 3))
    u_ref = dv.zeros(f.shape)
    hist_ref = dv.host(h.run_cycles(f, u_ref, 3, 2, 2, u_zero=True))[0]
    s = dd.DecomposedSolver(h, 1, 0, local=False, nccl_id=dd.nccl_unique_id(), agglomerate_rows=127)
    s.set_rhs(0, f)
    hist = dv.host(s.run_cycles(3, 2, 2))
    assert t.equal(s.solution(0), u_ref)
    assert np.allclose(hist, hist_ref, rtol=1e-13, atol=0)


@pytest.mark.parametrize("name", ["c1_fd_conv", "c1_q1_conv", "case_var31_conv_v22", "case_lshape31_conv_v11",
                                  "case_rot31_fc_v22", "c4_p0", "case_rect20x27_conv_v11", "case_grf63_conv_v22"])
def test_tile_and_stream_passes_bit_identical(name):
    """Tile-local fused passes (mid-size levels) vs row-streaming passes on every
    level: the same arithmetic, so u is bitwise equal; histories differ in the
    order of the norm's partial sums and in how the final entry's residual is
    evaluated (streamed FMA chain vs the reference-order residual kernel), so
    they are held to the reference tolerance."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    c = load(name)
    g = c["golden"]
    spec = spec_of(c["mask"], float(g["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), c["smoother"])
    f = dv.to_dev(np.where(c["mask"], c["f"], 0.0))
    runs = []
    for stream_min, tile in ((0, 1), (1 << 62, 1), (1 << 62, 0)):
        h.set_passes(stream_min, tile)
        u = dv.zeros(f.shape)
        hist = h.run_cycles(f, u, c["cycles"], c["nu"], c["nu"], u_zero=True).clone()
        runs.append((u, dv.host(hist)[0]))
    assert t.equal(runs[0][0], runs[1][0])
    assert_hist(runs[0][1], runs[1][1])
    assert_hist(runs[1][1], runs[2][1])                       # vs separate kernels: rounding only
    assert rel_err(dv.host(runs[1][0]), dv.host(runs[2][0])) <= 1e-12
    assert_hist(runs[1][1], g["history"])                     # and the reference


def test_five_point_operator_detected():
    """The GRF 5-point cell-centred operator (config 3's family) has zero corner planes
    on level 0 only (its Galerkin coarse operators are 9-point); the streaming passes
    then skip the corner reads, which the bitwise stream/tile test above covers."""
    c = load("case_grf63_conv_v22")
    spec = spec_of(c["mask"], float(c["golden"]["h"]))
    h = mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"])
    assert h.stencil_points(0) == 5
    assert h.stencil_points(1) == 9
    c = load("case_var31_conv_v22")
    h = mg.build_hierarchy(mg.StencilField(spec_of(c["mask"], float(c["golden"]["h"])), c["A0"]), c["levels"])
    assert h.stencil_points(0) in (0, 9)


@pytest.mark.parametrize("n,nu", [(1023, 2), (1023, 1), (600, 2)])
def test_tile_passes_large_tiles(n, nu):
    """The 32-point tile (levels of ~550^2 and more) against row streaming, bitwise."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    table = gen.rotated_fd(1, math.pi / 4, 1e-3, h=1.0 / (n + 1))[0, 0]
    h = mg.equip_inferred(mg.build_hierarchy_classed(n, n, table, gen.levels_for(n)), net_of("conv_c2"))
    f = dv.to_dev(gen.uniform_rhs(n, 2))
    out = []
    for stream_min in (0, 1 << 62):
        h.set_passes(stream_min, 1)
        u = dv.zeros(f.shape)
        out.append((u, dv.host(h.run_cycles(f, u, 3, nu, nu, u_zero=True))[0]))
    assert t.equal(out[0][0], out[1][0])
    assert np.allclose(out[0][1], out[1][1], rtol=1e-13, atol=0)


@pytest.mark.parametrize("name", ["c1_fd_conv", "case_lshape31_conv_v11", "c4_p0", "case_var31_conv_v22"])
def test_single_launch_coarse_cycle_agrees(name):
    """The single-CTA shared-memory coarse cycle (levels <= 32^2 in one launch)
    against the per-level tile passes: rounding-level agreement and the reference."""
    from paper_2102_12071_b200 import device as dv
    c = load(name)
    g = c["golden"]
    spec = spec_of(c["mask"], float(g["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), c["smoother"])
    f = dv.to_dev(np.where(c["mask"], c["f"], 0.0))
    out = []
    for coarse_max in (0, 32 * 32):
        h.set_passes(coarse_max=coarse_max)
        u = dv.zeros(f.shape)
        hist = dv.host(h.run_cycles(f, u, c["cycles"], c["nu"], c["nu"], u_zero=True))[0]
        out.append((dv.host(u), hist))
    assert_hist(out[0][1], out[1][1])
    assert rel_err(out[0][0], out[1][0]) <= 1e-12
    assert_hist(out[1][1], g["history"])


def test_pipelined_host_solves_equal_single_calls():
    """mgb_run_cycles_host_many (copies overlapping neighbouring solves) gives each
    solve exactly what a synchronous mgb_run_cycles_host call gives."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    c = load("case_lshape31_conv_v11")
    spec = spec_of(c["mask"], float(c["golden"]["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), "conv")
    fs = [t.from_numpy(np.where(c["mask"], gen.uniform_rhs(31, 20 + k), 0.0)).pin_memory().numpy()
          for k in range(5)]
    us = [t.zeros(31, 31, dtype=t.float64).pin_memory().numpy() for _ in range(5)]
    hs = h.run_cycles_host_many(fs, us, 6, 1, 1, u_zero=True)
    for k in range(5):
        u1 = np.zeros((31, 31))
        h1 = h.run_cycles_host(np.ascontiguousarray(fs[k]), u1, 6, 1, 1, u_zero=True)
        assert np.array_equal(us[k], u1) and np.array_equal(hs[k], h1)
    # warm start path (u read from the host buffers)
    us2 = [u.copy() for u in us]
    h.run_cycles_host_many(fs, us2, 2, 1, 1, u_zero=False)
    u1 = us[3].copy()
    h.run_cycles_host(np.ascontiguousarray(fs[3]), u1, 2, 1, 1, u_zero=False)
    assert np.array_equal(us2[3], u1)


def test_host_calls_history_staging_grows_safely():
    """Regression (advisor r01): run_cycles_host_many, then run_cycles_host with more
    cycles (grows the history staging), then run_cycles_host_many again with the
    larger count on the same pooled workspace: both staging sets must have grown,
    so every solve still equals the synchronous single call."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    c = load("case_rot15_conv_v22")
    spec = spec_of(c["mask"], float(c["golden"]["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), "conv")
    n = c["mask"].shape[0]
    fs = [t.from_numpy(gen.uniform_rhs(n, 40 + k)).pin_memory().numpy() for k in range(3)]

    def many(cycles):
        us = [t.zeros(n, n, dtype=t.float64).pin_memory().numpy() for _ in fs]
        return us, h.run_cycles_host_many(fs, us, cycles, 1, 1, u_zero=True)

    many(5)
    u1 = np.zeros((n, n))
    h.run_cycles_host(np.ascontiguousarray(fs[0]), u1, 10, 1, 1, u_zero=True)
    us, hs = many(10)
    for k in range(3):
        uk = np.zeros((n, n))
        hk = h.run_cycles_host(np.ascontiguousarray(fs[k]), uk, 10, 1, 1, u_zero=True)
        assert np.array_equal(us[k], uk) and np.array_equal(hs[k], hk)


def test_facade_rejects_bad_device_buffers():
    """Advisor r01: raw pointers go to the C-ABI only for C-contiguous fp64 CUDA
    tensors of the level-0 size on the hierarchy's device."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    c = load("case_rot15_conv_v22")
    spec = spec_of(c["mask"], float(c["golden"]["h"]))
    h = _equip(mg.build_hierarchy(mg.StencilField(spec, c["A0"]), c["levels"]), "conv")
    n = c["mask"].shape[0]
    f = dv.to_dev(gen.uniform_rhs(n, 1))
    u = dv.zeros(f.shape)
    for bad in (f.float(), f.t(), f[:-1], f.cpu()):
        with pytest.raises(mg.ContractError):
            h.run_cycles(bad, u, 2, 1, 1)
    with pytest.raises(mg.ContractError):
        h.run_cycles(f, u, 4, 1, 1, history=t.empty(3, dtype=t.float64, device=f.device))
    h.run_cycles(f, u, 2, 1, 1, u_zero=True)


@pytest.mark.parametrize("rows,cols,theta,nu,net", [
    (600, 600, math.pi / 4, 2, "conv_c2"),     # even sides
    (511, 511, math.pi / 6, 2, "conv"),        # odd sides, several strips
    (300, 777, math.pi / 3, 1, "conv"),        # rectangle, V(1,1)
    (1023, 1023, math.pi / 4, 2, "fc"),        # fc net: boundary band classes differ (non-uniform)
    (97, 1201, math.pi / 4, 2, "conv_c2"),     # short and wide: many strips, few rows
    (2047, 130, math.pi / 5, 2, "conv"),       # tall and narrow: two strips, long segments
    (40, 40, 0.3, 1, "fc"),                    # one strip, one segment
    (1023, 2047, math.pi / 4, 2, "conv_c2"),   # quasi-uniform coarse levels with several strips (modes 4 / 5)
    (767, 515, 1.1, 1, "conv_c5"),             # the same, sizes that are not 2^k - 1, V(1,1)
])
def test_warp_strip_stream_kernel_bit_identical(rows, cols, theta, nu, net):
    """The one-warp-per-strip kernel (k_stream3: four columns per lane, shuffle
    neighbours, no stage lag) against the column-pair kernel, forced on every level
    of a band-class hierarchy (uniform and non-uniform levels, edge strips, grid-edge
    rows, segment boundaries, PRE / POST / zero-start / residual-norm passes): u
    bitwise equal, histories to summation order."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    table = gen.rotated_fd(1, theta, 1e-2, h=1.0 / (max(rows, cols) + 1))[0, 0]
    levels = gen.levels_for(min(rows, cols))
    h = mg.equip_inferred(mg.build_hierarchy_classed(rows, cols, table, levels), net_of(net))
    h.set_passes(0, 1)
    if (rows, cols) == (1023, 2047):
        # level 0 uniform; the Galerkin levels with conv-net kernels quasi-uniform (an fc net's
        # kernels see the neighbours' tables: two boundary bands differ)
        assert [h.level_uniformity(l) for l in range(3)] == [1, 2, 2]
    if net == "fc" and rows == 1023:
        assert h.level_uniformity(1) == 0
    f = dv.to_dev(np.random.default_rng(9).uniform(-1, 1, (rows, cols)))
    out = []
    for kind in (2, 3):
        h.set_stream_kernel(kind)
        u = dv.zeros(f.shape)
        hh = h.run_cycles(f, u, 3, nu, nu, u_zero=True)
        u2 = u.clone()
        hw = h.run_cycles(f, u2, 2, nu, nu, u_zero=False)     # warm start: the non-zero-start PRE
        out.append((u, dv.host(hh)[0], u2, dv.host(hw)[0]))
    h.set_stream_kernel(0)
    (ua, ha, wa, hwa), (ub, hb, wb, hwb) = out
    assert t.equal(ua, ub), float((ua - ub).abs().max())
    assert t.equal(wa, wb), float((wa - wb).abs().max())
    assert np.allclose(ha, hb, rtol=1e-13, atol=0) and np.allclose(hwa, hwb, rtol=1e-13, atol=0)


@pytest.mark.parametrize("rows,cols,nu,cycles,net", [
    (1023, 1025, 2, 3, "conv_c2"),      # odd x odd, just above the 1 M point threshold
    (1024, 1301, 1, 2, "conv"),         # even rows, V(1,1)
    (2047, 1025, 2, 1, "conv_c5"),      # one cycle: the first PRE and the last POST are the same cycle's
    (1100, 1100, 2, 2, "conv_c2"),      # even x even (no quasi-uniform levels: the column bands sit on odd columns)
])
def test_default_path_padded_level0_direct_output(rows, cols, nu, cycles, net):
    """The default pass selection on levels of at least 1 M points — padded level-0 copies
    staged by the copy kernel, the last POST pass writing the caller's dense u directly, the
    quasi-uniform flavour below — against the column-pair kernel on the caller's arrays:
    u bitwise equal for zero and warm starts, histories to summation order."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    table = gen.rotated_fd(1, math.pi / 4, 1e-2, h=1.0 / (max(rows, cols) + 1))[0, 0]
    h = mg.equip_inferred(mg.build_hierarchy_classed(rows, cols, table, gen.levels_for(min(rows, cols))), net_of(net))
    assert "k_stream3" in h.pass_kernel(0, nu)
    f = dv.to_dev(np.random.default_rng(3).uniform(-1, 1, (rows, cols)))
    out = []
    for kind in (2, 0):
        h.set_stream_kernel(kind)
        u = dv.zeros(f.shape)
        hh = h.run_cycles(f, u, cycles, nu, nu, u_zero=True)
        u2 = u.clone()
        hw = h.run_cycles(f, u2, cycles, nu, nu, u_zero=False)
        out.append((u, dv.host(hh)[0], u2, dv.host(hw)[0]))
    h.set_stream_kernel(0)
    (ua, ha, wa, hwa), (ub, hb, wb, hwb) = out
    assert t.equal(ua, ub), float((ua - ub).abs().max())
    assert t.equal(wa, wb), float((wa - wb).abs().max())
    assert np.allclose(ha, hb, rtol=1e-13, atol=0) and np.allclose(hwa, hwb, rtol=1e-13, atol=0)


def test_warp_strip_kernel_batched_uniform_level():
    """Config 4's path: a batch of constant-coefficient problems, V(1,1).  Level 0 (uniform per
    problem) and level 1 (quasi-uniform per problem) run the warp-strip kernel's batched flavours — work items (problem, strip, segment),
    the problem's interior weights in registers — against the column-pair kernel: u bitwise
    equal for every problem, histories to summation order; V(2,2) stays on column pairs."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    rows, cols, nb = 303, 391, 5
    rng = np.random.default_rng(5)
    tabs = np.stack([np.broadcast_to(gen.rotated_fd(1, th, eps, h=1.0 / (cols + 1))[0, 0], (25, 3, 3))
                     for th, eps in zip(rng.uniform(0, math.pi, nb), 10.0 ** rng.uniform(-3, 0, nb))])
    h = mg.equip_inferred(mg.build_hierarchy_classed(rows, cols, tabs, gen.levels_for(rows)), net_of("conv"))
    h.set_passes(0, 1)
    f = dv.to_dev(rng.uniform(-1, 1, (nb, rows, cols)))
    out = []
    for kind in (2, 3):
        h.set_stream_kernel(kind)
        if kind == 3:
            assert "k_stream3" in h.pass_kernel(0, 1) and "k_stream2" in h.pass_kernel(0, 2)
            # the batch's first Galerkin level (151 x 195: quasi-uniform per problem, two strips): the
            # batched quasi-uniform flavour, class tables per problem in shared memory; the next one
            # (75 x 97: one strip) stays on column pairs
            assert [h.level_uniformity(l) for l in range(3)] == [1, 2, 2]
            assert "k_stream3" in h.pass_kernel(1, 1) and "k_stream2" in h.pass_kernel(2, 1)
        u = dv.zeros(f.shape)
        hh = h.run_cycles(f, u, 3, 1, 1, u_zero=True)
        u2 = u.clone()
        hw = h.run_cycles(f, u2, 2, 1, 1, u_zero=False)
        out.append((u, dv.host(hh), u2, dv.host(hw)))
    h.set_stream_kernel(0)
    (ua, ha, wa, hwa), (ub, hb, wb, hwb) = out
    assert t.equal(ua, ub), float((ua - ub).abs().max())
    assert t.equal(wa, wb), float((wa - wb).abs().max())
    assert np.allclose(ha, hb, rtol=1e-13, atol=0) and np.allclose(hwa, hwb, rtol=1e-13, atol=0)


def test_warp_strip_kernel_full_size_c2():
    """Config 2 at 4095^2 (uniform level 0, non-uniform levels 1-2): the warp-strip
    kernel equals the column-pair kernel bitwise over 3 V(2,2) cycles."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    n = 4095
    table = gen.rotated_fd(1, math.pi / 4, 1e-3, h=1.0 / (n + 1))[0, 0]
    h = mg.equip_inferred(mg.build_hierarchy_classed(n, n, table, gen.levels_for(n)), net_of("conv_c2"))
    f = dv.to_dev(gen.uniform_rhs(n, 1))
    out = []
    for kind in (2, 3):
        h.set_stream_kernel(kind)
        u = dv.zeros(f.shape)
        out.append((u, dv.host(h.run_cycles(f, u, 3, 2, 2, u_zero=True))[0]))
    h.set_stream_kernel(0)
    assert t.equal(out[0][0], out[1][0]), float((out[0][0] - out[1][0]).abs().max())
    assert np.allclose(out[0][1], out[1][1], rtol=1e-13, atol=0)


@pytest.mark.parametrize("n,nparts", [(1023, 2), (1023, 3), (2047, 4)])
def test_virtual_decomposition_warp_strip_kernel(n, nparts, monkeypatch):
    """Row-block decomposition with the warp-strip kernel on the distributed levels
    (owned row ranges, ghost bands): bitwise the single-domain result."""
    from paper_2102_12071_b200 import dd, device as dv
    monkeypatch.setenv("MGB_STREAM_MIN", "0")
    t = dv.torch()
    table = gen.rotated_fd(1, math.pi / 3, 0.01, h=1.0 / (n + 1))[0, 0]
    h = mg.equip_inferred(mg.build_hierarchy_classed(n, n, table, gen.levels_for(n)), net_of("conv"))
    h.set_stream_kernel(3)
    f_full = dv.to_dev(gen.uniform_rhs(n, 11))
    u_ref = dv.zeros(f_full.shape)
    hist_ref = dv.host(h.run_cycles(f_full, u_ref, 4, 2, 2, u_zero=True))[0]
    s = dd.DecomposedSolver(h, nparts, local=True, agglomerate_rows=n // 4)
    for p, (r0, r1) in enumerate(s.rows(p) for p in range(nparts)):
        s.set_rhs(p, f_full[r0:r1].contiguous())
    hist = dv.host(s.run_cycles(4, 2, 2))
    u = t.cat([s.solution(p) for p in range(nparts)])
    h.set_stream_kernel(0)
    assert t.equal(u, u_ref), float((u - u_ref).abs().max())
    assert np.allclose(hist, hist_ref, rtol=1e-13, atol=0)


@pytest.mark.parametrize("rows,cols,theta,nu,net", [
    (600, 600, math.pi / 4, 2, "conv_c2"),     # even sides
    (511, 511, math.pi / 6, 2, "conv"),        # odd sides, two strips
    (300, 777, math.pi / 3, 1, "conv"),        # rectangle, V(1,1)
    (1023, 1023, math.pi / 4, 2, "fc"),        # fc net: boundary band classes differ
    (97, 1201, math.pi / 4, 2, "conv_c2"),     # short and wide: many strips, few rows
])
def test_column_pair_stream_kernel_bit_identical(rows, cols, theta, nu, net):
    """The column-pair row-streaming kernel (push-form stage chains) against the
    one-column kernel, forced on every level of a band-class hierarchy: edge strips,
    uniform and non-uniform levels, odd and even sides, segment boundaries.  u and
    the histories are bitwise equal (the kernels share stencil_dot's FMA order)."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    table = gen.rotated_fd(1, theta, 1e-2, h=1.0 / (max(rows, cols) + 1))[0, 0]
    levels = gen.levels_for(min(rows, cols))
    h = mg.equip_inferred(mg.build_hierarchy_classed(rows, cols, table, levels), net_of(net))
    h.set_passes(0, 1)                                    # streaming passes on every level
    f = dv.to_dev(np.random.default_rng(7).uniform(-1, 1, (rows, cols)))
    out = []
    for kind in (1, 2):
        h.set_stream_kernel(kind)
        u = dv.zeros(f.shape)
        out.append((u, dv.host(h.run_cycles(f, u, 3, nu, nu, u_zero=True))[0]))
    h.set_stream_kernel(0)
    assert t.equal(out[0][0], out[1][0]), float((out[0][0] - out[1][0]).abs().max())
    assert np.allclose(out[0][1], out[1][1], rtol=1e-13, atol=0)


def test_column_pair_stream_kernel_full_size_c2():
    """Config-2 size (4095^2, where the automatic choice is the column-pair kernel
    on levels 0-1): bitwise equal to the one-column kernel over 3 V(2,2) cycles."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    n = 4095
    table = gen.rotated_fd(1, math.pi / 4, 1e-3, h=1.0 / (n + 1))[0, 0]
    h = mg.equip_inferred(mg.build_hierarchy_classed(n, n, table, gen.levels_for(n)), net_of("conv_c2"))
    f = dv.to_dev(gen.uniform_rhs(n, 1))
    out = []
    for kind in (1, 0):
        h.set_stream_kernel(kind)
        u = dv.zeros(f.shape)
        out.append((u, dv.host(h.run_cycles(f, u, 3, 2, 2, u_zero=True))[0]))
    assert t.equal(out[0][0], out[1][0]), float((out[0][0] - out[1][0]).abs().max())
    assert np.allclose(out[0][1], out[1][1], rtol=1e-13, atol=0)


@pytest.mark.parametrize("n,nparts", [(1023, 2), (1023, 3)])
def test_virtual_decomposition_column_pair_kernel(n, nparts, monkeypatch):
    """Row-block decomposition with the column-pair kernel on the distributed levels
    (owned row ranges, ghost bands): bitwise the single-domain result."""
    from paper_2102_12071_b200 import dd, device as dv
    monkeypatch.setenv("MGB_STREAM_MIN", "0")
    t = dv.torch()
    table = gen.rotated_fd(1, math.pi / 3, 0.01, h=1.0 / (n + 1))[0, 0]
    h = mg.equip_inferred(mg.build_hierarchy_classed(n, n, table, gen.levels_for(n)), net_of("conv"))
    h.set_stream_kernel(2)
    f_full = dv.to_dev(gen.uniform_rhs(n, 11))
    u_ref = dv.zeros(f_full.shape)
    hist_ref = dv.host(h.run_cycles(f_full, u_ref, 4, 2, 2, u_zero=True))[0]
    s = dd.DecomposedSolver(h, nparts, local=True, agglomerate_rows=n // 4)
    for p, (r0, r1) in enumerate(s.rows(p) for p in range(nparts)):
        s.set_rhs(p, f_full[r0:r1].contiguous())
    hist = dv.host(s.run_cycles(4, 2, 2))
    u = t.cat([s.solution(p) for p in range(nparts)])
    assert t.equal(u, u_ref), float((u - u_ref).abs().max())
    assert np.allclose(hist, hist_ref, rtol=1e-13, atol=0)


@pytest.mark.parametrize("n,theta,nu,net", [(255, math.pi / 6, 2, "conv"), (127, math.pi / 4, 1, "conv"),
                                            (63, math.pi / 3, 2, "fc")])
def test_coarse_tail_kernel_bitwise_equals_tile_passes(n, theta, nu, net):
    """k_coarse_tail (band-class levels of at most 1024 points in one launch: the same
    stencil_dot chains in the tile passes' stage order) against the per-level passes: u
    and histories bit for bit."""
    from paper_2102_12071_b200 import device as dv
    t = dv.torch()
    A = gen.rotated_fd(n, theta, 0.01)
    h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), gen.levels_for(n)), net_of(net))
    f = dv.to_dev(gen.uniform_rhs(n, 4))
    out = []
    for coarse_max in (0, 1024):
        h.set_passes(coarse_max=coarse_max)
        u = dv.zeros(f.shape)
        hist = h.run_cycles(f, u, 4, nu, nu, u_zero=True).clone()
        out.append((u, hist, h.last_launches))
    assert t.equal(out[0][0], out[1][0]) and t.equal(out[0][1], out[1][1])
    assert out[1][2] < out[0][2]          # fewer launches per solve
