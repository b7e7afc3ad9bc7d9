"""CPU oracle for the learned-smoother multigrid hot path — TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference (`mgsmooth` 0.1.0,
``/root/reference/pkg/src/mgsmooth``) for the path named by BASELINE.json's
north star: stencil residual, per-point (CNN-inferred) smoother, full-weighting
restriction, prolongation, Galerkin RAP, coarsest LU, the V(nu1, nu2) cycle and
the solve loop, plus the stencil -> smoother CNN forward.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import it, and only as the checker.  The product path
(``paper_2102_12071_b200``) never imports this file.

Parity pin: every function here is checked against golden vectors produced by
running the unmodified reference in this container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``, ``tests/golden/*.json``;
test: ``tests/test_oracle_golden.py``).

Data model (identical to the reference): fp64 arrays, grid values ``(rows, cols)``
with i = row = y and j = col = x; stencils ``(rows, cols, 3, 3)`` with entry
``[di + 1, dj + 1]`` multiplying ``u(i + di, j + dj)`` (cross-correlation,
grid.py:3-13); a boolean mask marks active points and every grid function is
zero at inactive points (grid.py:85-92).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

LEAKY_SLOPE = 0.01                      # smoothers.py:22
FW = np.array([[1.0, 2.0, 1.0],
               [2.0, 4.0, 2.0],
               [1.0, 2.0, 1.0]]) / 16.0  # transfer.py:28-30 (R = FW, P = 2 FW, transfer.py:60-61)


class OracleError(Exception):
    """Raised where the reference raises (ConfigError/ContractError/...)."""

    def __init__(self, kind: str, msg: str, pivot_index=None):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.pivot_index = pivot_index


# --------------------------------------------------------------------------
# grid core (grid.py)

def neighbor(v: np.ndarray, di: int, dj: int) -> np.ndarray:
    """s[i, j] = v[i+di, j+dj], zero outside the lattice (grid.py:27-35).

    Implemented with a zero-padded copy instead of the reference's windowed
    assignment; the values are identical."""
    rows, cols = v.shape[:2]
    pad = np.zeros((rows + 2 * abs(di) + 2, cols + 2 * abs(dj) + 2) + v.shape[2:])
    oi, oj = abs(di) + 1, abs(dj) + 1
    pad[oi:oi + rows, oj:oj + cols] = v
    return pad[oi + di:oi + di + rows, oj + dj:oj + dj + cols].copy()


def apply_stencil(A: np.ndarray, u: np.ndarray, mask: np.ndarray | None = None) -> np.ndarray:
    """out(p) = sum_o A(p)[o] u(p+o); inactive outputs zeroed (grid.py:216-226).

    Accumulation order follows the reference (di-major, dj-minor, starting
    from 0.0) so results are bit-identical to it."""
    k = A.shape[2]
    r = k // 2
    out = np.zeros(u.shape)
    for di in range(-r, r + 1):
        for dj in range(-r, r + 1):
            out += A[:, :, di + r, dj + r] * neighbor(u, di, dj)
    if mask is not None:
        out[~mask] = 0.0
    return out


def masked(v: np.ndarray, mask: np.ndarray | None) -> np.ndarray:
    """GridFunction invariant: zero at inactive points (grid.py:92)."""
    if mask is None:
        return v
    return np.where(mask, v, 0.0)


# --------------------------------------------------------------------------
# transfers (transfer.py)

def coarse_mask(mask_f: np.ndarray) -> np.ndarray:
    """Full coarsening: coarse c <-> fine 2c+1, rows_c = rows // 2
    (transfer.py:50-61).  Raises where coarsen_full raises."""
    rows_c, cols_c = mask_f.shape[0] // 2, mask_f.shape[1] // 2
    if rows_c < 1 or cols_c < 1:
        raise OracleError("ConfigError", "grid cannot be coarsened further")
    m = mask_f[1::2, 1::2][:rows_c, :cols_c].copy()
    if not m.any():
        raise OracleError("ConfigError", "coarsening left no active points")
    return m


def _fine_at(vf: np.ndarray, shape_c, si: int, sj: int) -> np.ndarray:
    """g[c] = vf[2c + 1 + s], zero where that index leaves the fine lattice
    (the reference's _gather with stride 2, offset 1; transfer.py:94-105)."""
    rows_c, cols_c = shape_c
    rf, cf = vf.shape[:2]
    ii = 2 * np.arange(rows_c) + 1 + si
    jj = 2 * np.arange(cols_c) + 1 + sj
    vi = (ii >= 0) & (ii < rf)
    vj = (jj >= 0) & (jj < cf)
    out = np.zeros((rows_c, cols_c) + vf.shape[2:])
    out[np.ix_(vi, vj)] = vf[np.ix_(ii[vi], jj[vj])]
    return out


def restrict(rf: np.ndarray, mask_c: np.ndarray) -> np.ndarray:
    """r_c(c) = sum_d FW[d] r(2c+1+d), terms accumulated di-major
    (transfer.py:108-121)."""
    shape_c = mask_c.shape
    out = np.zeros(shape_c)
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            out += FW[di + 1, dj + 1] * _fine_at(rf, shape_c, di, dj)
    out[~mask_c] = 0.0
    return out


def prolong(ec: np.ndarray, shape_f, mask_f: np.ndarray) -> np.ndarray:
    """Scatter form: u_f(2c+1+d) += 2 FW[d] e(c), offsets visited di-major
    (transfer.py:124-147)."""
    rows_c, cols_c = ec.shape
    rf, cf = shape_f
    out = np.zeros((rf + 2, cf + 2))          # one guard ring absorbs off-grid targets
    P = 2.0 * FW
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            i0 = 1 + 1 + di                   # guard offset + anchor 1 + di
            j0 = 1 + 1 + dj
            out[i0:i0 + 2 * rows_c:2, j0:j0 + 2 * cols_c:2] += P[di + 1, dj + 1] * ec
    out = out[1:1 + rf, 1:1 + cf].copy()
    out[~mask_f] = 0.0
    return out


def galerkin(A: np.ndarray, mask_f: np.ndarray, mask_c: np.ndarray) -> np.ndarray:
    """Coarse stencil R A P per coarse point (transfer.py:150-209, _trim :212-222).

    Entry dc of coarse point c sums R[u] A(2c+1+u)[v] P[w] over chains with
    u + v - w = 2 dc, weighted by the activity of the fine source 2c+1+u, the
    fine target 2c+1+u+v and the coarse target c+dc.  Loop order matches the
    reference (u, v, w) so sums are bit-identical."""
    if A.shape[2] != 3:
        raise OracleError("ContractError", "oracle Galerkin supports 3x3 stencils")
    shape_c = mask_c.shape
    rows_c, cols_c = shape_c
    fm = mask_f.astype(float)
    cm = mask_c.astype(float)
    P = 2.0 * FW
    K = 1                                     # (1 + 1 + 1) // 2, transfer.py:164
    out = np.zeros((rows_c, cols_c, 3, 3))
    for ui in (-1, 0, 1):
        for uj in (-1, 0, 1):
            rw = FW[ui + 1, uj + 1]
            src = _fine_at(fm, shape_c, ui, uj)
            if not src.any():
                continue
            for vi in (-1, 0, 1):
                for vj in (-1, 0, 1):
                    e = _fine_at(A[:, :, vi + 1, vj + 1], shape_c, ui, uj) * src
                    e *= _fine_at(fm, shape_c, ui + vi, uj + vj)
                    if not e.any():
                        continue
                    for wi in (-1, 0, 1):
                        di, remi = divmod(ui + vi - wi, 2)
                        if remi:
                            continue
                        for wj in (-1, 0, 1):
                            dj, remj = divmod(uj + vj - wj, 2)
                            if remj:
                                continue
                            tgt = neighbor(cm, di, dj)
                            out[:, :, di + K, dj + K] += rw * P[wi + 1, wj + 1] * e * tgt
    out[~mask_c] = 0.0
    out[~mask_c, 1, 1] = 1.0
    return out


# --------------------------------------------------------------------------
# dense LU (dense.py:21-63) and materialization (grid.py:269-292)

def materialize(A: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """Dense operator over active points, row-major mask order.  Entry
    (i, j) = A(p_i)[p_j - p_i] when the offset is inside the stencil."""
    pts = np.argwhere(mask)
    index = -np.ones(mask.shape, dtype=np.int64)
    index[mask] = np.arange(len(pts))
    n = len(pts)
    M = np.zeros((n, n))
    r = A.shape[2] // 2
    for a, (i, j) in enumerate(pts):
        for di in range(-r, r + 1):
            for dj in range(-r, r + 1):
                ii, jj = i + di, j + dj
                if 0 <= ii < mask.shape[0] and 0 <= jj < mask.shape[1] and mask[ii, jj]:
                    M[a, index[ii, jj]] = A[i, j, di + r, dj + r]
    return M


def lu_factor(M: np.ndarray):
    """PA = LU, partial pivoting, pivot <= 1e-12 * max|A| is singular
    (dense.py:21-47).  Returns (LU, perm) with perm[i] the source row."""
    a = np.array(M, dtype=float)
    n = a.shape[0]
    scale = np.abs(a).max() if a.size else 0.0
    if scale == 0.0:
        raise OracleError("SingularMatrixError", "zero matrix", 0)
    perm = np.arange(n)
    for k in range(n):
        p = k + int(np.argmax(np.abs(a[k:, k])))
        if abs(a[p, k]) <= 1e-12 * scale:
            raise OracleError("SingularMatrixError", f"pivot {k}", k)
        if p != k:
            a[[k, p]] = a[[p, k]]
            perm[[k, p]] = perm[[p, k]]
        a[k + 1:, k] /= a[k, k]
        a[k + 1:, k + 1:] -= np.outer(a[k + 1:, k], a[k, k + 1:])
    return a, perm


def lu_solve(lu: np.ndarray, perm: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Forward (unit L) then backward (U) substitution (dense.py:50-63)."""
    x = np.asarray(b, dtype=float)[perm].copy()
    n = lu.shape[0]
    for k in range(n):
        x[k + 1:] -= lu[k + 1:, k] * x[k]
    for k in range(n - 1, -1, -1):
        x[k] /= lu[k, k]
        x[:k] -= lu[:k, k] * x[k]
    return x


# --------------------------------------------------------------------------
# smoothers and the kernel-inference CNN (smoothers.py)

@dataclass
class Net:
    """KernelInferenceNet payload (smoothers.py:217-235)."""
    variant: str                 # "conv" | "fc"
    weights: list
    k: int = 1
    slope: float = LEAKY_SLOPE


def load_net_json(path) -> Net:
    """Model JSON, kind 'inference_net' (smoothers.py:384-414)."""
    import json
    with open(path) as fh:
        doc = json.load(fh)
    if doc.get("format_version") != 1 or doc.get("kind") != "inference_net":
        raise OracleError("ConfigError", "not an inference_net model")
    ws = [np.array(w["data"], dtype=float).reshape(w["shape"]) for w in doc["weights"]]
    return Net(doc["variant"], ws, int(doc["k"]), float(doc["slope"]))


def leaky(x: np.ndarray, slope: float) -> np.ndarray:
    return np.where(x > 0.0, x, slope * x)          # smoothers.py:25-26


def features(A: np.ndarray, mask: np.ndarray, variant: str) -> np.ndarray:
    """Network input (smoothers.py:184-210): conv = own 3x3 table; fc = the
    nine neighbour tables, block ((oi+1)*3 + (oj+1)), entry e; off-grid or
    inactive neighbours give zero blocks."""
    rows, cols = mask.shape
    t = A.reshape(rows, cols, 9).copy()
    t[~mask] = 0.0
    if variant == "conv":
        return t.reshape(rows, cols, 3, 3)
    if variant == "fc":
        f = np.zeros((rows, cols, 9, 9))
        for oi in (-1, 0, 1):
            for oj in (-1, 0, 1):
                f[:, :, (oi + 1) * 3 + (oj + 1), :] = neighbor(t, oi, oj)
        f[~mask] = 0.0
        return f.reshape(rows, cols, 81)
    raise OracleError("ConfigError", f"unknown variant {variant!r}")


def conv3x3_same(W: np.ndarray, img: np.ndarray) -> np.ndarray:
    """Zero-padded 3x3 correlation of each channel kernel with a batch of
    3x3 images: (c,3,3) x (n,3,3) -> (n,c,3,3) (smoothers.py:256-270)."""
    n = img.shape[0]
    pad = np.zeros((n, 5, 5))
    pad[:, 1:4, 1:4] = img
    out = np.zeros((n, W.shape[0], 3, 3))
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            win = pad[:, 1 + di:4 + di, 1 + dj:4 + dj]
            out += W[None, :, di + 1, dj + 1, None, None] * win[:, None, :, :]
    return out


def net_forward(net: Net, x: np.ndarray) -> np.ndarray:
    """Batched forward (smoothers.py:273-288) -> (n, k, 3, 3)."""
    if net.variant == "fc":
        h = x
        for w in net.weights[:-1]:
            h = leaky(h @ w, net.slope)
        out = h @ net.weights[-1]
    else:
        h = x
        acts = None
        for w in net.weights[:-1]:
            acts = leaky(conv3x3_same(w, h), net.slope)
            h = acts.sum(axis=1)
        out = acts.reshape(acts.shape[0], -1) @ net.weights[-1]
    return out.reshape(-1, net.k, 3, 3)


def infer_kernels(net: Net, A: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """Per-point smoother kernels (rows, cols, k, 3, 3): diagonal-normalised
    in and out, zero at inactive points (smoothers.py:302-322)."""
    rows, cols = mask.shape
    f = features(A, mask, net.variant)
    d = A[:, :, 1, 1].copy()
    d[~mask] = 1.0
    flat = f.reshape(rows * cols, *f.shape[2:])
    kern = net_forward(net, flat / d.reshape(-1, *([1] * (flat.ndim - 1))))
    kern = kern / d.reshape(-1, 1, 1, 1)
    kern = kern.reshape(rows, cols, net.k, 3, 3)
    kern[~mask] = 0.0
    return kern


def jacobi_kernels(A: np.ndarray, mask: np.ndarray, omega: float = 2.0 / 3.0) -> np.ndarray:
    """omega-Jacobi (smoothers.py:29-50) written as a centre-only per-point
    kernel so it runs through the same smoother path."""
    d = A[:, :, 1, 1]
    if np.any(d[mask] == 0.0):
        raise OracleError("ConfigError", "jacobi: zero diagonal")
    kern = np.zeros(mask.shape + (1, 3, 3))
    kern[:, :, 0, 1, 1] = np.where(mask, omega / np.where(mask, d, 1.0), 0.0)
    return kern


def smoother_apply(kern: np.ndarray, r: np.ndarray, mask: np.ndarray,
                   slope: float = LEAKY_SLOPE) -> np.ndarray:
    """M(r): k stages of per-point 3x3 correlation, leaky between stages
    (smoothers.py:325-343)."""
    v = r
    for s in range(kern.shape[2]):
        if s > 0:
            v = leaky(v, slope)
        v = apply_stencil(kern[:, :, s], v, mask)
    return v


# --------------------------------------------------------------------------
# hierarchy, cycle, solve (hierarchy.py; cli.py:365-377 for V(nu, nu))

@dataclass
class Hierarchy:
    ops: list                     # per-level (rows, cols, 3, 3)
    masks: list                   # per-level bool (rows, cols)
    lu: np.ndarray = None
    perm: np.ndarray = None
    kernels: list = field(default_factory=list)   # per-level (rows, cols, k, 3, 3), levels 0..L-1
    slope: float = LEAKY_SLOPE

    @property
    def depth(self) -> int:
        return len(self.ops)


def build_hierarchy(A: np.ndarray, levels: int, mask: np.ndarray | None = None) -> Hierarchy:
    """Galerkin chain + coarsest LU (hierarchy.py:70-88)."""
    if levels < 2:
        raise OracleError("ConfigError", "a hierarchy needs at least two levels")
    if mask is None:
        mask = np.ones(A.shape[:2], dtype=bool)
    ops, masks = [A], [mask]
    for step in range(levels - 1):
        mc = coarse_mask(masks[-1])
        if mc.sum() >= masks[-1].sum():
            raise OracleError("ConfigError", f"level {step}: coarsening does not shrink")
        ops.append(galerkin(ops[-1], masks[-1], mc))
        masks.append(mc)
    lu, perm = lu_factor(materialize(ops[-1], masks[-1]))
    return Hierarchy(ops, masks, lu, perm)


def equip_inferred(h: Hierarchy, net: Net) -> Hierarchy:
    """hierarchy.py:207-214."""
    h.kernels = [infer_kernels(net, h.ops[l], h.masks[l]) for l in range(h.depth - 1)]
    h.slope = net.slope
    return h


def equip_jacobi(h: Hierarchy, omega: float = 2.0 / 3.0) -> Hierarchy:
    """hierarchy.py:152-161 with kind='jacobi'."""
    h.kernels = [jacobi_kernels(h.ops[l], h.masks[l], omega) for l in range(h.depth - 1)]
    return h


def coarse_solve(h: Hierarchy, f: np.ndarray) -> np.ndarray:
    """hierarchy.py:91-93."""
    m = h.masks[-1]
    x = np.zeros(m.shape)
    x[m] = lu_solve(h.lu, h.perm, f[m])
    return x


def _smooth(h: Hierarchy, l: int, r: np.ndarray, nu: int) -> np.ndarray:
    """RepeatedSmoother(M, A, nu).apply(r) (cli.py:373-377): c = M r, then
    nu - 1 times c <- c + M(r - A c).  M: per-point kernels or a ConvSm."""
    K, m = h.kernels[l], h.masks[l]
    M = (lambda x: conv_apply(K, x, m)) if isinstance(K, ConvSm) else (lambda x: smoother_apply(K, x, m, h.slope))
    c = M(r)
    for _ in range(nu - 1):
        c = masked(c + M(masked(r - apply_stencil(h.ops[l], c, m), m)), m)
    return c


# --------------------------------------------------------------------------
# shared-kernel convolutional smoother (grid.py:229-266, smoothers.py:99-178)

def convolve(w: np.ndarray, u: np.ndarray, mask: np.ndarray | None = None) -> np.ndarray:
    """grid.py:229-239: out += w[o] * u(p + o) over the non-zero weights,
    di-major, zero padding, output re-masked."""
    r = w.shape[0] // 2
    out = np.zeros(u.shape)
    for di in range(-r, r + 1):
        for dj in range(-r, r + 1):
            wo = w[di + r, dj + r]
            if wo != 0.0:
                out += wo * neighbor(u, di, dj)
    if mask is not None:
        out[~mask] = 0.0
    return out


@dataclass
class ConvSm:
    """ConvSmoother (smoothers.py:105-130) parameters."""
    layers: list
    skip: np.ndarray | None
    activation: str = "linear"
    slope: float = LEAKY_SLOPE
    gain: float = 1.0


def conv_apply(s: ConvSm, r: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """ConvSmoother.apply (smoothers.py:133-145)."""
    v = convolve(s.layers[0], r, mask)
    for w in s.layers[1:]:
        if s.activation == "leaky":
            v = leaky(v, s.slope)
        v = convolve(w, v, mask)
    out = v
    if s.skip is not None:
        out = out + convolve(s.skip, r, mask)
    return s.gain * out


def representative_diagonal(A: np.ndarray, mask: np.ndarray) -> float:
    """smoothers.py:99-102."""
    return float(np.median(A[:, :, 1, 1][mask]))


def conv_init(A: np.ndarray, mask: np.ndarray, form: str = "full", omega: float = 2.0 / 3.0,
              activation: str = "linear") -> ConvSm:
    """conv_smoother (smoothers.py:148-164): Jacobi-equivalent initialisation."""
    jk = np.zeros((3, 3))
    jk[1, 1] = omega
    gain = 1.0 / representative_diagonal(A, mask)
    if form == "full":
        return ConvSm([np.zeros((3, 3)) for _ in range(5)], jk, activation, gain=gain)
    delta = np.zeros((3, 3))
    delta[1, 1] = 1.0
    return ConvSm([delta, jk], None, activation, gain=gain)


def compose(outer: np.ndarray, inner: np.ndarray) -> np.ndarray:
    """compose_kernels (grid.py:242-256)."""
    k1, k2 = outer.shape[0], inner.shape[0]
    out = np.zeros((k1 + k2 - 1, k1 + k2 - 1))
    for i in range(k1):
        for j in range(k1):
            if outer[i, j] != 0.0:
                out[i:i + k2, j:j + k2] += outer[i, j] * inner
    return out


def effective_kernel(s: ConvSm) -> np.ndarray:
    """smoothers.py:167-178 with pad_kernel (grid.py:259-266)."""
    acc = s.layers[0]
    for w in s.layers[1:]:
        acc = compose(w, acc)
    out = acc.copy()
    if s.skip is not None:
        off = (acc.shape[0] - s.skip.shape[0]) // 2
        pad = np.zeros(acc.shape)
        pad[off:off + s.skip.shape[0], off:off + s.skip.shape[0]] = s.skip
        out = out + pad
    return s.gain * out


def v_cycle(h: Hierarchy, l: int, f: np.ndarray, u: np.ndarray, nu1: int = 1, nu2: int = 1) -> np.ndarray:
    """hierarchy.py:96-111 with each smoother wrapped as RepeatedSmoother(nu)."""
    if l == h.depth - 1:
        return coarse_solve(h, f)
    A, m = h.ops[l], h.masks[l]
    u = masked(u + _smooth(h, l, masked(f - apply_stencil(A, u, m), m), nu1), m)
    rc = restrict(masked(f - apply_stencil(A, u, m), m), h.masks[l + 1])
    ec = v_cycle(h, l + 1, rc, np.zeros(h.masks[l + 1].shape), nu1, nu2)
    u = masked(u + prolong(ec, m.shape, m), m)
    return masked(u + _smooth(h, l, masked(f - apply_stencil(A, u, m), m), nu2), m)


def solve(h: Hierarchy, f: np.ndarray, u0: np.ndarray | None = None, tol: float = 1e-6,
          max_iter: int = 100, nu1: int = 1, nu2: int = 1, raise_on_divergence: bool = True):
    """hierarchy.py:119-146.  Returns (u, history, iterations, converged)."""
    if tol <= 0.0:
        raise OracleError("ConfigError", "tolerance must be positive")
    A, m = h.ops[0], h.masks[0]
    u = np.zeros(m.shape) if u0 is None else u0.copy()
    fn = float(np.linalg.norm(f))
    denom = fn if fn > 0.0 else 1.0

    def rel(res):
        n = float(np.linalg.norm(res))
        return 0.0 if n == 0.0 else n / denom

    r0 = rel(masked(f - apply_stencil(A, u, m), m))
    hist = [r0]
    it = 0
    while hist[-1] >= tol and it < max_iter:
        u = v_cycle(h, 0, f, u, nu1, nu2)
        it += 1
        rr = rel(masked(f - apply_stencil(A, u, m), m))
        hist.append(rr)
        if raise_on_divergence and (not math.isfinite(rr) or rr > 1e6 * max(r0, tol)):
            raise OracleError("NonConvergedError", f"diverged at iteration {it}")
    return u, hist, it, hist[-1] < tol


def run_cycles(h: Hierarchy, f: np.ndarray, cycles: int, nu1: int, nu2: int,
               u0: np.ndarray | None = None):
    """Explicit fixed-count cycle loop with the history residual after each
    cycle (the oracle drives v_cycle directly, not solve())."""
    A, m = h.ops[0], h.masks[0]
    u = np.zeros(m.shape) if u0 is None else u0.copy()
    fn = float(np.linalg.norm(f))
    denom = fn if fn > 0.0 else 1.0
    hist = [float(np.linalg.norm(masked(f - apply_stencil(A, u, m), m))) / denom]
    for _ in range(cycles):
        u = v_cycle(h, 0, f, u, nu1, nu2)
        hist.append(float(np.linalg.norm(masked(f - apply_stencil(A, u, m), m))) / denom)
    return u, np.array(hist)


# ---------------------------------------------------------------------------
# Krylov (krylov.py:60-270): flexible GMRES with the V-cycle as right
# preconditioner and plain GMRES, restated on flat vectors.

REORTH_TOL = 1e-8       # krylov.py:19
BREAKDOWN_TOL = 1e-14   # krylov.py:20


def _givens(a: float, b: float):
    """krylov.py:54-58."""
    r = math.hypot(a, b)
    if r == 0.0:
        return 1.0, 0.0
    return a / r, b / r


def _arnoldi(apply_a, f, precond, u0, steps, tol_abs, history, record_beta, early_exit):
    """One (F)GMRES cycle from u0: krylov.py:60-135 (fgmres: record_beta on the
    first cycle, early_exit) and the body of krylov.py:189-230 (gmres)."""
    r = f - apply_a(u0)
    beta = float(np.linalg.norm(r))
    if record_beta:
        history.append(beta)
    if early_exit and beta <= tol_abs:
        return u0, True, 0
    steps = min(steps, r.size)
    V, Z = [r / beta], []
    H = np.zeros((steps + 1, steps))
    cs, sn, g = np.zeros(steps), np.zeros(steps), np.zeros(steps + 1)
    g[0] = beta
    j = 0
    while j < steps:
        z = V[j] if precond is None else precond(V[j])
        w = apply_a(z)
        Z.append(z)
        wnorm0 = float(np.linalg.norm(w))
        for i in range(j + 1):
            H[i, j] = float(V[i] @ w)
            w = w - H[i, j] * V[i]
        wnorm = float(np.linalg.norm(w))
        if wnorm < REORTH_TOL * wnorm0 or any(abs(float(V[i] @ w)) > REORTH_TOL * max(wnorm, 1e-300)
                                              for i in range(j + 1)):
            for i in range(j + 1):
                c = float(V[i] @ w)
                H[i, j] += c
                w = w - c * V[i]
        hsub = float(np.linalg.norm(w))
        H[j + 1, j] = hsub
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        cs[j], sn[j] = _givens(H[j, j], H[j + 1, j])
        H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        res = abs(g[j + 1])
        history.append(res)
        j += 1
        if res <= tol_abs:
            break
        if hsub <= BREAKDOWN_TOL * max(wnorm0, 1.0):
            raise OracleError("NumericError", f"Arnoldi breakdown at step {j}")
        V.append(w / hsub)
    y = np.zeros(j)
    for i in range(j - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:j]) / H[i, i]
    u = u0.copy()
    for i in range(j):
        u = u + y[i] * Z[i]
    return u, abs(g[j]) <= tol_abs, j


def fgmres(apply_a, f, precond=None, tol=1e-6, max_iter=200, restart=None):
    """krylov.py:138-164.  Returns (u, iterations, history, converged)."""
    f = np.asarray(f, dtype=float)
    beta0 = float(np.linalg.norm(f))
    if beta0 == 0.0:
        return np.zeros_like(f), 0, [0.0], True
    tol_abs = tol * beta0
    history: list = []
    u = np.zeros_like(f)
    done, total = False, 0
    while total < max_iter and not done:
        steps = max_iter - total
        if restart is not None:
            steps = min(steps, restart)
        u, done, took = _arnoldi(apply_a, f, precond, u, steps, tol_abs, history, not history, True)
        total += took
        if took == 0:
            break
    return u, total, history, done


def gmres(apply_a, f, tol=1e-6, max_iter=200, restart=None):
    """krylov.py:167-236.  Returns (u, iterations, history, converged)."""
    f = np.asarray(f, dtype=float)
    beta0 = float(np.linalg.norm(f))
    if beta0 == 0.0:
        return np.zeros_like(f), 0, [0.0], True
    tol_abs = tol * beta0
    history = [beta0]
    u = np.zeros_like(f)
    if beta0 <= tol_abs:
        return u, 0, history, True
    budget = max_iter
    while budget > 0:
        steps = budget if restart is None else min(budget, restart)
        u, done, j = _arnoldi(apply_a, f, None, u, steps, tol_abs, history, False, False)
        budget -= j
        if done or j == 0:
            return u, max_iter - budget, history, done
    return u, max_iter, history, False


def grid_action(A: np.ndarray, mask: np.ndarray | None = None):
    """krylov.py:249-258."""
    shape = A.shape[:2]
    return lambda x: apply_stencil(A, x.reshape(shape), mask).ravel()


def cycle_preconditioner(h: Hierarchy, nu1: int = 1, nu2: int = 1):
    """krylov.py:261-270: one V(nu1, nu2)-cycle from zero on the masked vector."""
    m = h.masks[0]
    return lambda r: v_cycle(h, 0, r.reshape(m.shape) * m, np.zeros(m.shape), nu1, nu2).ravel()
