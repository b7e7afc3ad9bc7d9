"""Reverse-mode differentiation over the grid operations, on the GPU.

The reference's tape (autodiff.py:21-430) with device-resident values: a ``Var`` wraps
a float64 CUDA tensor and remembers how it was produced; ``backward`` walks the graph
once in reverse topological order.  Every forward and backward operation is a
hand-written kernel behind the C-ABI (``csrc/mgb_train.cu`` plus the stateless grid
kernels); torch only allocates the buffers and moves scalars.  Operations accept plain
arrays / tensors wherever an argument is constant.  The coarsest dense solve is a
constant linear operator whose adjoint is the transposed solve (dense.py:66-80).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, device as dv
from .errors import ContractError, NumericError
from .grid import GridSpec, StencilField

_scratch = {}


def _t():
    return dv.torch()


def dev(x):
    """float64 CUDA tensor of a constant (tensors pass through)."""
    t = _t()
    if isinstance(x, t.Tensor):
        return x
    return dv.to_dev(np.ascontiguousarray(np.asarray(x, dtype=float)))


def _scr(outputs: int):
    """Reduction scratch (grown on demand, one buffer per device)."""
    n = _lib.lib().mgb_ad_scratch_doubles(int(outputs))
    d = dv.current_device()
    buf = _scratch.get(d)
    if buf is None or buf.numel() < n:
        buf = dv.empty((max(n, 4096),))
        _scratch[d] = buf
    return buf


def _call(name, *args):
    _lib.call(name, *args, dv.stream())


def _ptr(x):
    return None if x is None else dv.ptr(x)


class Var:
    """autodiff.py:21-33: value, accumulated gradient, parents, backward closure."""
    __slots__ = ("value", "grad", "parents", "backward_fn")

    def __init__(self, value, parents=(), backward_fn=None):
        self.value = dev(value)
        self.grad = None
        self.parents = parents
        self.backward_fn = backward_fn

    def add_grad(self, g):
        g = dev(g)
        if self.grad is None:
            self.grad = _t().zeros_like(self.value)
        _call("mgb_ad_axpby", self.grad.numel(), 1.0, _ptr(self.grad), 1.0, _ptr(g.contiguous()), _ptr(self.grad))


def value_of(x):
    return x.value if isinstance(x, Var) else dev(x)


def _node(value, inputs, backward_fn) -> Var:
    return Var(value, tuple(p for p in inputs if isinstance(p, Var)), backward_fn)


def _axpby(a, x, b, y):
    x = x.contiguous()
    out = _t().empty_like(x)
    _call("mgb_ad_axpby", x.numel(), float(a), _ptr(x), float(b), None if y is None else _ptr(y.contiguous()), _ptr(out))
    return out


# ---------------------------------------------------------------------------
# elementwise and shape operations (autodiff.py:41-125)

def add(a, b) -> Var:
    av, bv = value_of(a), value_of(b)

    def back(g):
        for x in (a, b):
            if isinstance(x, Var):
                x.add_grad(g)
    return _node(_axpby(1.0, av, 1.0, bv), (a, b), back)


def sub(a, b) -> Var:
    av, bv = value_of(a), value_of(b)

    def back(g):
        if isinstance(a, Var):
            a.add_grad(g)
        if isinstance(b, Var):
            b.add_grad(_axpby(-1.0, g, 0.0, None))
    return _node(_axpby(1.0, av, -1.0, bv), (a, b), back)


def scale(a, s: float) -> Var:
    av, s = value_of(a), float(s)

    def back(g):
        if isinstance(a, Var):
            a.add_grad(_axpby(s, g, 0.0, None))
    return _node(_axpby(s, av, 0.0, None), (a,), back)


def _mul(x, c, repeat=0):
    x = x.contiguous()
    out = _t().empty_like(x)
    _call("mgb_ad_mul", x.numel(), _ptr(x), _ptr(c), int(repeat), _ptr(out))
    return out


def mul_const(a, c) -> Var:
    """Elementwise product with a constant array; a (n, 1) column against (n, m) values
    broadcasts over the rows, as the net graphs use it."""
    av, cv = value_of(a), dev(c).contiguous()
    repeat = 0
    if cv.numel() != av.numel():
        if av.dim() != 2 or cv.numel() != av.shape[0]:
            raise ContractError("mul_const: constant does not broadcast over the value")
        repeat = av.shape[1]

    def back(g):
        if isinstance(a, Var):
            a.add_grad(_mul(g, cv, repeat))
    return _node(_mul(av, cv, repeat), (a,), back)


def leaky(a, slope: float) -> Var:
    av = value_of(a).contiguous()
    out = _t().empty_like(av)
    _call("mgb_ad_leaky", av.numel(), _ptr(av), float(slope), None, _ptr(out))

    def back(g):
        if isinstance(a, Var):
            gz = _t().empty_like(av)
            _call("mgb_ad_leaky", av.numel(), _ptr(av), float(slope), _ptr(g.contiguous()), _ptr(gz))
            a.add_grad(gz)
    return _node(out, (a,), back)


def reshape(a, shape) -> Var:
    av = value_of(a)

    def back(g):
        if isinstance(a, Var):
            a.add_grad(g.reshape(av.shape))
    return _node(av.contiguous().reshape(shape), (a,), back)


def sum_axis(a, axis: int) -> Var:
    av = value_of(a).contiguous()
    if axis != 1 or av.dim() < 2:
        raise ContractError("sum_axis: the device tape sums over axis 1")
    n, c = av.shape[0], av.shape[1]
    inner = int(av.numel() // (n * c))
    out = _t().empty((n,) + tuple(av.shape[2:]), dtype=av.dtype, device=av.device)
    _call("mgb_ad_sum_axis1", n, c, inner, _ptr(av), _ptr(out))

    def back(g):
        if isinstance(a, Var):
            ga = _t().zeros_like(av)
            _call("mgb_ad_bcast_axis1", n, c, inner, _ptr(g.contiguous()), _ptr(ga))
            a.add_grad(ga)
    return _node(out, (a,), back)


def slice_cols(a, j0: int, j1: int) -> Var:
    av = value_of(a)

    def back(g):
        if isinstance(a, Var):
            da = _t().zeros_like(av)
            da[:, j0:j1].copy_(g)          # data movement only
            a.add_grad(da)
    return _node(av[:, j0:j1].contiguous(), (a,), back)


def _mm(A, ta, B, tb, M, K, N):
    out = _t().empty((M, N), dtype=A.dtype, device=A.device)
    _call("mgb_ad_matmul", M, K, N, _ptr(A.contiguous()), int(ta), _ptr(B.contiguous()), int(tb), 0, _ptr(out),
          _ptr(_scr(M * N)))
    return out


def matmul(a, b) -> Var:
    av, bv = value_of(a), value_of(b)
    M, K = av.shape
    N = bv.shape[1]

    def back(g):
        if isinstance(a, Var):
            a.add_grad(_mm(g, 0, bv, 1, M, N, K))      # g @ b^T
        if isinstance(b, Var):
            b.add_grad(_mm(av, 1, g, 0, K, M, N))      # a^T @ g
    return _node(_mm(av, 0, bv, 0, M, K, N), (a, b), back)


# ---------------------------------------------------------------------------
# grid operations

class _Masks:
    """Per-spec device masks: uint8 for the kernels (None when all active) and a 0/1
    float64 copy for masking a field before an unmasked operation."""
    _cache = {}

    @classmethod
    def of(cls, spec: GridSpec):
        key = (id(spec), dv.current_device())
        hit = cls._cache.get(key)
        if hit is None or hit[0] is not spec:
            m8 = dv.mask_dev(spec.mask)
            mf = None if m8 is None else dv.to_dev(spec.mask.astype(float))
            hit = (spec, m8, mf)
            cls._cache[key] = hit
        return hit[1], hit[2]


def _masked(v, mf):
    return v if mf is None else _mul(v, mf)


def _conv3(w_host, mask8, u, rows, cols):
    w = np.ascontiguousarray(w_host, dtype=float)
    out = _t().empty_like(u)
    _call("mgb_convolve", 1, rows, cols, w.ctypes.data_as(_lib.P), _ptr(mask8), _ptr(u.contiguous()), _ptr(out))
    return out


def conv2d(kernel, u, spec: GridSpec) -> Var:
    """Shared-kernel correlation on the grid, output zeroed off the mask (autodiff.py:139-168)."""
    kv, uv = value_of(kernel), value_of(u).contiguous()
    if tuple(kv.shape) != (3, 3):
        raise ContractError("the device tape takes 3x3 shared kernels")
    m8, mf = _Masks.of(spec)
    k_host = dv.host(kv)

    def back(g):
        gm = _masked(g.contiguous(), mf)
        if isinstance(kernel, Var):
            dk = _t().empty_like(kv)
            _call("mgb_ad_conv_kgrad", spec.rows, spec.cols, 3, None, _ptr(gm), _ptr(uv), _ptr(_scr(9)), 0, _ptr(dk))
            kernel.add_grad(dk)
        if isinstance(u, Var):
            u.add_grad(_conv3(k_host[::-1, ::-1], None, gm, spec.rows, spec.cols))
    return _node(_conv3(k_host, m8, uv, spec.rows, spec.cols), (kernel, u), back)


class _OpCache:
    """Device copies of constant stencil tables, keyed by the StencilField object."""
    _cache = {}

    @classmethod
    def of(cls, A: StencilField):
        key = (id(A), dv.current_device())
        hit = cls._cache.get(key)
        if hit is None or hit[0] is not A:
            hit = (A, dv.to_dev(np.ascontiguousarray(A.data)))
            cls._cache[key] = hit
        return hit[1]


def _apply9(T, mask8, u, rows, cols):
    out = _t().empty_like(u)
    _call("mgb_apply_stencil", 1, rows, cols, 3, _ptr(T.contiguous()), _ptr(mask8), _ptr(u.contiguous()), _ptr(out))
    return out


def _adjoint9(T, mask_in, mask_out, g, order, rows, cols):
    out = _t().empty_like(g)
    _call("mgb_ad_stencil_adjoint", rows, cols, _ptr(T.contiguous()), _ptr(mask_in), _ptr(mask_out),
          _ptr(g.contiguous()), int(order), _ptr(out))
    return out


def stencil_apply(A: StencilField, u) -> Var:
    """Operator application; A is always constant (autodiff.py:171-192)."""
    if A.k != 3:
        raise ContractError("the device tape takes 3x3 stencil fields")
    uv = value_of(u)
    spec = A.spec
    m8, mf = _Masks.of(spec)
    T = _OpCache.of(A)

    def back(g):
        if isinstance(u, Var):
            u.add_grad(_adjoint9(T, m8, m8, g, 0, spec.rows, spec.cols))
    return _node(_apply9(T, m8, _masked(uv, mf), spec.rows, spec.cols), (u,), back)


def _restrict(tp, v):
    m8, _ = _Masks.of(tp.coarse)
    out = _t().empty((tp.coarse.rows, tp.coarse.cols), dtype=v.dtype, device=v.device)
    _call("mgb_restrict", 1, tp.fine.rows, tp.fine.cols, _ptr(m8), _ptr(v.contiguous()), _ptr(out))
    return out


def _prolong(tp, v):
    m8, _ = _Masks.of(tp.fine)
    _, mfc = _Masks.of(tp.coarse)
    out = _t().empty((tp.fine.rows, tp.fine.cols), dtype=v.dtype, device=v.device)
    _call("mgb_prolong", 1, tp.fine.rows, tp.fine.cols, _ptr(m8), _ptr(_masked(v.contiguous(), mfc)), _ptr(out))
    return out


def do_restrict(tp, u) -> Var:
    """autodiff.py:234-241: backward is half the prolongation."""
    uv = value_of(u)

    def back(g):
        if isinstance(u, Var):
            u.add_grad(_axpby(0.5, _prolong(tp, g), 0.0, None))
    return _node(_restrict(tp, uv), (u,), back)


def do_prolong(tp, u) -> Var:
    """autodiff.py:244-251: backward is twice the restriction."""
    uv = value_of(u)

    def back(g):
        if isinstance(u, Var):
            u.add_grad(_axpby(2.0, _restrict(tp, g), 0.0, None))
    return _node(_prolong(tp, uv), (u,), back)


def pointwise_conv(kern, u, spec: GridSpec) -> Var:
    """Unshared per-point kernels, kern (rows, cols, 3, 3) (autodiff.py:254-280)."""
    kv, uv = value_of(kern).contiguous(), value_of(u).contiguous()
    m8, _ = _Masks.of(spec)

    def back(g):
        g = g.contiguous()
        if isinstance(kern, Var):
            dk = _t().empty_like(kv)
            _call("mgb_ad_pconv_kgrad", spec.rows, spec.cols, _ptr(m8), _ptr(g), _ptr(uv), 0, _ptr(dk))
            kern.add_grad(dk)
        if isinstance(u, Var):
            u.add_grad(_adjoint9(kv, m8, None, g, 1, spec.rows, spec.cols))
    return _node(_apply9(kv, m8, uv, spec.rows, spec.cols), (kern, u), back)


def conv_batch(kern, img) -> Var:
    """Batched 3x3 correlation on 3x3 images: kern (c, 3, 3), img (n, 3, 3) -> (n, c, 3, 3)
    (autodiff.py:283-325)."""
    kv, iv = value_of(kern).contiguous(), value_of(img).contiguous()
    n, c = iv.shape[0], kv.shape[0]
    out = _t().empty((n, c, 3, 3), dtype=iv.dtype, device=iv.device)
    _call("mgb_ad_conv_batch", n, c, _ptr(kv), _ptr(iv), _ptr(out))

    def back(g):
        dk = _t().empty_like(kv) if isinstance(kern, Var) else None
        di = _t().empty_like(iv) if isinstance(img, Var) else None
        _call("mgb_ad_conv_batch_bwd", n, c, _ptr(kv), _ptr(iv), _ptr(g.contiguous()), _ptr(_scr(c * 9)), 0, _ptr(dk), 0,
              _ptr(di))
        if dk is not None:
            kern.add_grad(dk)
        if di is not None:
            img.add_grad(di)
    return _node(out, (kern, img), back)


class CoarseSolve:
    """Device copy of the coarsest factorisation (lu, perm) and the active-point index."""

    def __init__(self, lu: np.ndarray, perm: np.ndarray, spec: GridSpec):
        t = _t()
        self.spec = spec
        self.n = int(lu.shape[0])
        self.lu = dv.to_dev(np.ascontiguousarray(lu, dtype=float))
        self.perm = t.from_numpy(np.ascontiguousarray(perm, dtype=np.int32)).to(self.lu.device)
        self.idx = t.from_numpy(np.flatnonzero(spec.mask.ravel())).to(self.lu.device)
        self.scratch = dv.empty((self.n,))

    def _run(self, name, b, *extra):
        t = _t()
        rhs = b.reshape(-1)[self.idx].contiguous()      # gather of the active points (data movement)
        x = t.empty_like(rhs)
        _call(name, self.n, _ptr(self.lu), _ptr(self.perm), _ptr(rhs), _ptr(x), *extra)
        out = t.zeros_like(b).reshape(-1)
        out[self.idx] = x
        return out.reshape(b.shape)

    def solve(self, b):
        return self._run("mgb_lu_solve", b)

    def solve_t(self, b):
        return self._run("mgb_lu_solve_t", b, _ptr(self.scratch))


def coarse_solve_const(cs: CoarseSolve, f) -> Var:
    """Exact coarsest solve as a constant linear operator (autodiff.py:328-344)."""
    fv = value_of(f)

    def back(g):
        if isinstance(f, Var):
            f.add_grad(cs.solve_t(g))
    return _node(cs.solve(fv), (f,), back)


# ---------------------------------------------------------------------------
# scalars (autodiff.py:347-372): held on the host

class Scalar(Var):
    """A scalar node: the value is a Python float."""
    __slots__ = ()

    def __init__(self, value, parents=(), backward_fn=None):
        self.value = float(value)
        self.grad = None
        self.parents = parents
        self.backward_fn = backward_fn

    def add_grad(self, g):
        self.grad = float(g) if self.grad is None else self.grad + float(g)


def norm2(a) -> Scalar:
    av = value_of(a).contiguous()
    out = dv.empty((1,))
    _call("mgb_ad_dot", av.numel(), _ptr(av), None, _ptr(_scr(1)), _ptr(out))
    n = float(np.sqrt(out.item()))

    def back(g):
        if isinstance(a, Var):
            if n == 0.0:
                raise NumericError("2-norm not differentiable at zero")
            a.add_grad(_axpby(float(g) / n, av, 0.0, None))
    return Scalar(n, (a,) if isinstance(a, Var) else (), back)


def mean_of(items: list) -> Scalar:
    if not items:
        raise ContractError("mean of an empty list")
    vals = np.array([float(x.value) if isinstance(x, Var) else float(x) for x in items])
    inv = 1.0 / len(items)

    def back(g):
        for x in items:
            if isinstance(x, Var):
                x.add_grad(float(g) * inv)
    return Scalar(vals.mean(), tuple(x for x in items if isinstance(x, Var)), back)


def backward(root: Var):
    """Reverse accumulation from a scalar root, each node visited once (autodiff.py:375-396)."""
    if not isinstance(root, Scalar) and root.value.numel() != 1:
        raise ContractError("backward needs a scalar root")
    order, seen, stack = [], set(), [(root, False)]
    while stack:
        node, done = stack.pop()
        if done:
            order.append(node)
            continue
        if id(node) in seen:
            continue
        seen.add(id(node))
        stack.append((node, True))
        for p in node.parents:
            if id(p) not in seen:
                stack.append((p, False))
    root.grad = 1.0 if isinstance(root, Scalar) else _t().ones_like(root.value)
    for node in reversed(order):
        if node.backward_fn is not None and node.grad is not None:
            node.backward_fn(node.grad)


def zero_grads(params: list):
    for p in params:
        p.grad = None


def grad_check(build_loss, params: list, step: float = 1e-5, limit: int = 200, seed: int = 0) -> float:
    """Max relative error of the reverse-mode gradients against central differences over
    up to `limit` randomly chosen parameter entries (autodiff.py:404-430)."""
    zero_grads(params)
    backward(build_loss())
    grads = [np.zeros(tuple(p.value.shape)) if p.grad is None else dv.host(p.grad).copy() for p in params]
    entries = [(i, idx) for i, p in enumerate(params) for idx in np.ndindex(tuple(p.value.shape))]
    rng = np.random.default_rng(seed)
    chosen = [entries[j] for j in rng.choice(len(entries), size=limit, replace=False)] if len(entries) > limit else entries
    worst = 0.0
    for i, idx in chosen:
        keep = float(params[i].value[idx].item())
        params[i].value[idx] = keep + step
        f_plus = float(build_loss().value)
        params[i].value[idx] = keep - step
        f_minus = float(build_loss().value)
        params[i].value[idx] = keep
        fd = (f_plus - f_minus) / (2.0 * step)
        ad_ = float(grads[i][idx])
        worst = max(worst, abs(fd - ad_) / max(abs(fd), abs(ad_), 1.0))
    return worst
