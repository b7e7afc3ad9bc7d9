"""The reference's own numerical pins recomputed on the device path:
R = 1/2 P^T materialised (tests/test_transfer.py:26), P(1) flat (:50), Galerkin = R A P
(:61), full weighting on bilinear fields (:92), apply_stencil vs the dense operator
(tests/test_grid.py:49), the coarse solve vs a dense solve (tests/test_hierarchy.py:28),
the V-cycle vs its dense error-propagation matrix (:39), kernel-inference scale
equivariance K(2A) = K(A) / 2 and constant kernels for constant coefficients
(tests/test_smoothers.py:126-148), memoisation until bump (:151)."""
import numpy as np
import pytest

import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import problems as gen

pytestmark = pytest.mark.gpu


def materialize(action, src, dst):
    """Dense matrix of a grid action between active-point vectors (grid.py:269-288)."""
    M = np.zeros((dst.n_active, src.n_active))
    for c in range(src.n_active):
        e = np.zeros(src.n_active)
        e[c] = 1.0
        M[:, c] = mg.to_active(action(mg.from_active(src, e)))
    return M


def dense_op(A):
    return materialize(lambda v: mg.apply_stencil(A, v), A.spec, A.spec)


def dense_pair(tp):
    return (materialize(lambda v: mg.prolong(tp, v), tp.coarse, tp.fine),
            materialize(lambda v: mg.restrict(tp, v), tp.fine, tp.coarse))


def perturbed_net(variant, seed, k=1):
    net = mg.inference_net(variant, k=k, seed=seed)
    rng = np.random.default_rng(seed + 100)
    for w in net.weights:
        w += rng.standard_normal(w.shape) * 0.05
    net.bump()
    return net


@pytest.mark.parametrize("geometry,n", [("square", 9), ("lshape", 9), ("cylinder", 11)])
def test_restriction_is_half_prolongation_transpose(geometry, n):
    tp = mg.coarsen_full(gen.build_geometry(geometry, n))
    P, R = dense_pair(tp)
    assert np.max(np.abs(R - 0.5 * P.T)) < 1e-14


def test_transfers_on_smooth_fields():
    tp = mg.coarsen_full(mg.full_spec(15))
    up = mg.prolong(tp, mg.GridFunction(tp.coarse, np.ones((7, 7))))
    assert np.max(np.abs(up.values[2:-2, 2:-2] - 0.5)) < 1e-13
    i, j = np.arange(15.0)[:, None], np.arange(15.0)[None, :]
    down = mg.restrict(tp, mg.GridFunction(tp.fine, 0.25 * i + 0.5 * j + 1.0))
    want = 0.25 * (2 * np.arange(7.0)[:, None] + 1) + 0.5 * (2 * np.arange(7.0)[None, :] + 1) + 1.0
    assert np.max(np.abs(down.values - want)) < 1e-12


@pytest.mark.parametrize("theta", [0.0, np.pi / 6, np.pi / 4])
def test_galerkin_product_equals_dense_triple_product(theta):
    A = gen.assemble_rotated_laplacian(mg.full_spec(9), theta, 100.0)
    tp = mg.coarsen_full(A.spec)
    P, R = dense_pair(tp)
    assert np.max(np.abs(dense_op(mg.galerkin_product(A, tp)) - R @ dense_op(A) @ P)) < 1e-12


def test_apply_stencil_matches_dense_operator():
    A = gen.ProblemSpec("variable", 9, "lshape", kappa=2.0).assemble()
    Ad = dense_op(A)
    rng = np.random.default_rng(3)
    v = mg.from_active(A.spec, rng.standard_normal(A.spec.n_active))
    assert np.max(np.abs(mg.to_active(mg.apply_stencil(A, v)) - Ad @ mg.to_active(v))) < 1e-13 * np.max(np.abs(Ad))


def test_coarse_solve_and_v_cycle_match_dense_algebra():
    """Two-level Jacobi V(1,1) on 7 x 7: u1 - u* = E (u0 - u*) with
    E = S (I - P Ac^-1 R A) S, S = I - M A (tests/test_hierarchy.py:28-50)."""
    A = gen.assemble_rotated_laplacian(mg.full_spec(7), np.pi / 6, 100.0)
    h = mg.equip_classical(mg.build_hierarchy(A, 2), "jacobi")
    Ad, Ac = dense_op(A), dense_op(h.levels[1].operator)
    rng = np.random.default_rng(0)
    b = mg.GridFunction(h.levels[1].spec, rng.standard_normal((3, 3)))
    assert np.max(np.abs(mg.to_active(mg.coarse_solve(h, b)) - np.linalg.solve(Ac, mg.to_active(b)))) < 1e-10
    P, R = dense_pair(h.levels[0].transfer)
    M = np.diag((2.0 / 3.0) / np.diag(Ad))
    S = np.eye(49) - M @ Ad
    E = S @ (np.eye(49) - P @ np.linalg.solve(Ac, R @ Ad)) @ S
    u_star, u0 = rng.standard_normal((7, 7)), rng.standard_normal((7, 7))
    f = mg.apply_stencil(A, mg.GridFunction(A.spec, u_star))
    u1 = mg.v_cycle(h, 0, f, mg.GridFunction(A.spec, u0))
    assert np.max(np.abs((u1.values - u_star).ravel() - E @ (u0 - u_star).ravel())) < 1e-12


@pytest.mark.parametrize("variant", ["fc", "conv"])
def test_inferred_kernels_scale_equivariance_and_constancy(variant):
    A = gen.ProblemSpec("variable", 9, kappa=1.0).assemble()
    B = mg.StencilField(A.spec, 2.0 * A.data)
    net = perturbed_net(variant, 2)
    ka, kb = mg.infer_kernels(net, A).kernels, mg.infer_kernels(net, B).kernels
    assert np.max(np.abs(ka)) > 0.0 and np.max(np.abs(kb - 0.5 * ka)) < 1e-10
    C = gen.ProblemSpec("variable", 9, kappa=0.0).assemble()     # constant coefficients
    inner = mg.infer_kernels(perturbed_net(variant, 1), C).kernels[2:-2, 2:-2]
    assert np.max(np.abs(inner)) > 0.0 and np.max(np.abs(inner - inner[0, 0])) < 1e-8


def test_scale_equivariance_through_the_device_hierarchy():
    """equip_inferred on a hierarchy of 2A installs half the kernels of the hierarchy of A
    on every level (the Galerkin chain is linear in A)."""
    A = gen.ProblemSpec("variable", 31, kappa=1.0).assemble()
    net = perturbed_net("conv", 5)
    ha = mg.equip_inferred(mg.build_hierarchy(A, 3), net)
    hb = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(A.spec, 2.0 * A.data), 3), net)
    for l in range(2):
        ka, kb = ha.levels[l].smoother.kernels, hb.levels[l].smoother.kernels
        assert np.max(np.abs(kb - 0.5 * ka)) < 1e-10 * np.max(np.abs(ka))


def test_infer_kernels_memoized_until_bump():
    A = gen.ProblemSpec("variable", 9, kappa=1.0).assemble()
    net = perturbed_net("conv", 3)
    first = mg.infer_kernels(net, A)
    assert mg.infer_kernels(net, A) is first
    net.weights[-1] += 0.01
    net.bump()
    assert mg.infer_kernels(net, A) is not first
