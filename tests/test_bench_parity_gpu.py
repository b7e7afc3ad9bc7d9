"""Parity at the BENCHMARKED configurations against the unmodified reference.

The golden files come from tests/golden/make_golden_bench.py, which runs the
reference's build_hierarchy + equip_inferred + RepeatedSmoother V(2,2) cycles
(hierarchy.py:70-146, smoothers.py:302-322, cli.py:365-377) on bench.py's own
input generators:

* bench_c2_full   config 2 at its full 4095^2 (net_conv_c2, seed 1, 3 cycles);
* bench_c3_511 / bench_c3_1023   config 3's exp(GRF) 5-point family (net_conv_c3);
* bench_c5_2047   config 5's family (theta = pi/3, eps = 0.01, net_conv_c5), also
  through the band-class-only build (bench's c5 path) and virtual row-block
  decompositions (the multi-GPU schedule on one GPU).

Gates: histories and u within 1e-10 relative (+1e-14 absolute on
histories); operators bit-exact (per-level checksums and sample tables equal);
fp64 CNN kernels within 1e-13 of max|K|.  Where u is too large to store, its
checksums (sum, sum |u|, sum u^2), the strided subsample u[::64, ::64], three
rows and the two edge columns are compared.
"""
import math
import os

import numpy as np
import pytest

import bench
import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import problems as gen

from conftest import GOLDEN, rel_err

pytestmark = pytest.mark.gpu

HIST_RTOL, HIST_ATOL, U_RTOL = 1e-10, 1e-14, 1e-10


def _golden(name):
    p = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(p):
        pytest.fail(f"missing golden {p} (tests/golden/make_golden_bench.py)")
    return np.load(p)


def _net(cfg):
    return mg.load_model(os.path.join(bench.ROOT, "paper_2102_12071_b200", "data", cfg["net"]))


def _check_hist(h, g):
    h, g = np.asarray(h), np.asarray(g)
    assert h.shape == g.shape
    assert np.all(np.abs(h - g) <= HIST_RTOL * np.abs(g) + HIST_ATOL), (h, g)


def _check_u(U, g):
    """u against the stored reference samples (or the full array)."""
    scale = float(np.max(np.abs(g["u_stride64"])))
    if "u" in g.files:
        assert rel_err(U, g["u"]) <= U_RTOL
    assert np.max(np.abs(U[::64, ::64] - g["u_stride64"])) <= U_RTOL * scale
    n = U.shape[0]
    assert np.max(np.abs(U[[0, n // 2, n - 1]] - g["u_rows"])) <= U_RTOL * scale
    assert np.max(np.abs(U[:, [0, U.shape[1] - 1]].T - g["u_cols"])) <= U_RTOL * scale
    cs = np.array([U.sum(), np.abs(U).sum(), (U * U).sum()])
    ref = g["u_checksums"]
    # sum and sum|u|: each term within U_RTOL * max|u|; sum u^2 within 2 U_RTOL relative
    bound = U_RTOL * np.max(np.abs(U)) * U.size
    assert abs(cs[0] - ref[0]) <= bound and abs(cs[1] - ref[1]) <= bound, (cs, ref)
    assert abs(cs[2] - ref[2]) <= 2 * U_RTOL * ref[2] + 1e-300, (cs, ref)


def _check_levels(h, g, exact_ops=True):
    """Per-level operator / kernel checksums of the device hierarchy vs the reference."""
    for l in range(int(g["levels"])):
        A = h.operator_batch(l)[0]
        if exact_ops:
            assert np.array_equal(A[A.shape[0] // 2, A.shape[1] // 2], g[f"Amid{l}"]), l
            assert np.array_equal(A[0, 0], g[f"Acorner{l}"]), l
            assert np.allclose([A.sum(), np.abs(A).sum()], g[f"Asum{l}"], rtol=1e-13, atol=0), l
        if f"Ksum{l}" in g.files:
            K = h.kernels_batch(l)[0]
            kmax = np.max(np.abs(K))
            assert np.max(np.abs(K[K.shape[0] // 2, K.shape[1] // 2] - g[f"Kmid{l}"])) <= 1e-13 * kmax, l
            assert np.max(np.abs(K[0, 0] - g[f"Kcorner{l}"])) <= 1e-13 * kmax, l
            assert abs(np.abs(K).sum() - g[f"Ksum{l}"][1]) <= 1e-12 * g[f"Ksum{l}"][1], l


def _run(h, f, g):
    from paper_2102_12071_b200 import device as dv
    fd = dv.to_dev(f)
    u = dv.zeros(fd.shape)
    nu, cycles = int(g["nu"]), int(g["cycles"])
    hist = dv.host(h.run_cycles(fd, u, cycles, nu, nu, u_zero=True))[0]
    return hist, dv.host(u)


@pytest.mark.parametrize("n", [511, 1023])
def test_config3_family_matches_reference(n):
    """exp(GRF) 5-point cell-centred operator, per-point planes on every level
    (the c3 path: 5-point level-0 A, streamed per-point A and M)."""
    g = _golden(f"bench_c3_{n}")
    cfg = bench.CONFIGS["c3"]
    A = gen.grf_diffusion_5pt(n, seed=cfg["seed"])
    f = gen.uniform_rhs(n, cfg["seed"])
    spec = mg.GridSpec(n, n, 1.0 / n, np.ones((n, n), bool))
    h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(spec, A), int(g["levels"])), _net(cfg))
    assert h.stencil_points(0) == 5
    _check_levels(h, g)
    hist, U = _run(h, f, g)
    _check_hist(hist, g["history"])
    _check_u(U, g)


@pytest.mark.parametrize("build", ["per_point", "classed"])
def test_config5_family_matches_reference(build):
    """Config 5's operator family at 2047^2 through the per-point build and the
    band-class-only build bench.py uses for 32767^2."""
    g = _golden("bench_c5_2047")
    cfg = bench.CONFIGS["c5"]
    n = 2047
    levels = int(g["levels"])
    f = gen.uniform_rhs(n, cfg["seed"])
    if build == "per_point":
        A = gen.rotated_fd(n, cfg["theta"], cfg["eps"])
        h = mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), levels)
    else:
        table = gen.rotated_fd(1, cfg["theta"], cfg["eps"], h=1.0 / (n + 1))[0, 0]
        h = mg.build_hierarchy_classed(n, n, table, levels)
    mg.equip_inferred(h, _net(cfg))
    _check_levels(h, g)
    hist, U = _run(h, f, g)
    _check_hist(hist, g["history"])
    _check_u(U, g)


@pytest.mark.parametrize("nparts", [2, 4])
def test_config5_family_decomposed_matches_reference(nparts, monkeypatch):
    """The row-block decomposition (virtual parts on one GPU: the NCCL path's
    schedule with device-copy halos, agglomerated coarse levels) against the
    reference at 2047^2."""
    from paper_2102_12071_b200 import dd, device as dv
    monkeypatch.setenv("MGB_STREAM_MIN", "0")
    t = dv.torch()
    g = _golden("bench_c5_2047")
    cfg = bench.CONFIGS["c5"]
    n = 2047
    table = gen.rotated_fd(1, cfg["theta"], cfg["eps"], h=1.0 / (n + 1))[0, 0]
    h = mg.equip_inferred(mg.build_hierarchy_classed(n, n, table, int(g["levels"])), _net(cfg))
    f = dv.to_dev(gen.uniform_rhs(n, cfg["seed"]))
    s = dd.DecomposedSolver(h, nparts, local=True, agglomerate_rows=255)
    assert s.distributed_levels >= 2
    for p in range(nparts):
        r0, r1 = s.rows(p)
        s.set_rhs(p, f[r0:r1].contiguous())
    hist = dv.host(s.run_cycles(int(g["cycles"]), int(g["nu"]), int(g["nu"])))
    U = dv.host(t.cat([s.solution(p) for p in range(nparts)]))
    _check_hist(hist, g["history"])
    _check_u(U, g)


@pytest.mark.slow
def test_config2_full_size_matches_reference():
    """Config 2 exactly as bench.py builds it (4095^2, per-point build stored as
    exact band classes, net_conv_c2, b seed 1): 3 V(2,2) cycles against the
    reference run at the same size."""
    g = _golden("bench_c2_full")
    cfg = bench.CONFIGS["c2"]
    h, f, _ = bench.build_problem("c2", 0)
    assert int(g["levels"]) == cfg["levels"] and int(g["n"]) == cfg["n"]
    _check_levels(h, g)
    hist, U = _run(h, f[0], g)
    _check_hist(hist, g["history"])
    _check_u(U, g)


# ---------------------------------------------------------------------------
# reference test pins recomputed on the device

def test_scale_equivariance_of_inferred_kernels():
    """tests/test_smoothers.py:137 of the reference: K(2A) = K(A) / 2 (the
    diagonal normalisation in and out of the net, smoothers.py:311-317), on the
    device inference, conv and fc nets, fp64."""
    n = 31
    A = gen.rotated_fd(n, 0.8, 0.05)
    A = A * (1.0 + 0.2 * np.random.default_rng(4).random((n, n, 1, 1)))
    spec = mg.full_spec(n)
    for name in ("net_conv.json", "net_fc.json"):
        net = mg.load_model(os.path.join(GOLDEN, name))
        K1 = mg.infer_kernels(net, mg.StencilField(spec, A)).kernels
        K2 = mg.infer_kernels(net, mg.StencilField(spec, 2.0 * A)).kernels
        assert np.max(np.abs(K2 - 0.5 * K1)) <= 1e-12 * np.max(np.abs(K1)), name


def test_restriction_is_half_prolongation_transpose():
    """tests/test_transfer.py:26 of the reference: materialised R = P^T / 2, with
    R and P each built column by column from the device kernels (unit vectors)."""
    from paper_2102_12071_b200 import transfer as tr
    for n, geom in ((9, "square"), (11, "lshape"), (10, "square")):
        mask = gen.geometry_mask(geom, n) if geom != "square" else np.ones((n, n), bool)
        spec = mg.GridSpec(n, n, 1.0 / (n + 1), mask)
        tp = tr.coarsen_full(spec)
        fi = np.flatnonzero(mask.ravel())
        ci = np.flatnonzero(tp.coarse.mask.ravel())
        R = np.zeros((ci.size, fi.size))
        P = np.zeros((fi.size, ci.size))
        for k, p in enumerate(fi):
            e = np.zeros(n * n)
            e[p] = 1.0
            R[:, k] = tr.restrict(tp, mg.GridFunction(spec, e.reshape(n, n))).values.ravel()[ci]
        for k, p in enumerate(ci):
            e = np.zeros(tp.coarse.mask.size)
            e[p] = 1.0
            P[:, k] = tr.prolong(tp, mg.GridFunction(tp.coarse, e.reshape(tp.coarse.mask.shape))).values.ravel()[fi]
        assert np.max(np.abs(R - 0.5 * P.T)) <= 1e-15, (n, geom)
