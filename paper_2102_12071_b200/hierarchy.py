"""Multigrid hierarchy, V-cycle and solve — facade over the B200 C-ABI.

Mirrors the reference's hierarchy.py:26-214 (same names, arguments, return
types and exceptions).  The hierarchy (Galerkin operators, smoother kernels,
coarsest LU) lives on the GPU; ``v_cycle`` / ``solve`` upload the right-hand
side, run the whole cycle on the device (one CUDA graph per cycle) and copy
the result back.  ``run_cycles`` / ``solve_device`` are the device-resident
entry points used for throughput measurements (torch CUDA tensors in/out).

V(nu1, nu2) follows the reference convention of wrapping every level's
smoother in ``RepeatedSmoother(inner, A, steps=nu)`` (cli.py:365-377):
``v_cycle`` reads ``steps`` from such wrappers, or takes ``nu1``/``nu2``.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib, device as dv
from .errors import ConfigError, ContractError, UnsupportedOperationError
from .grid import GridFunction, GridSpec, StencilField, apply_stencil, zeros
from .smoothers import (LEAKY_SLOPE, VARIANT_ID, ConvSmoother, InferredSmoother, JacobiSmoother, KernelInferenceNet,
                        conv_smoother, representative_diagonal)
from .transfer import TransferPair, coarsen_full


@dataclass
class SolveReport:
    """hierarchy.py:54-59."""
    iterations: int
    residual_history: list
    converged: bool
    wall_time: float


@dataclass
class RepeatedSmoother:
    """cli.py:365-377: `steps` sweeps of `inner` per smoothing application.
    On the device this is exactly `steps` fused sweeps u <- u + M(f - A u)."""
    inner: object
    operator: StencilField
    steps: int

    def apply(self, r: GridFunction) -> GridFunction:
        u = self.inner.apply(r)
        for _ in range(self.steps - 1):
            u = u + self.inner.apply(r - apply_stencil(self.operator, u))
        return u


class Level:
    """hierarchy.py:26-35; the operator is fetched from the device on first use."""

    def __init__(self, hier, index: int, spec: GridSpec, transfer: TransferPair | None,
                 operator: StencilField | None = None):
        self._hier = hier
        self.index = index
        self._spec = spec
        self.transfer = transfer
        self.smoother = None
        self.scheme = "full"
        self._operator = operator

    @property
    def spec(self) -> GridSpec:
        return self._spec

    @property
    def operator(self) -> StencilField:
        if self._operator is None:
            self._operator = self._hier._download_operator(self.index)
        return self._operator


class DeviceSmoother:
    """Smoother installed in a device hierarchy (per-point kernels on the GPU).
    ``kernels`` downloads the (rows, cols, k, 3, 3) table on first use."""

    def __init__(self, hier, level: int, k: int, slope: float, kind: str, omega: float | None = None):
        self._hier = hier
        self.level = level
        self.k = k
        self.slope = slope
        self.kind = kind
        self.omega = omega
        self._kernels = None

    @property
    def spec(self) -> GridSpec:
        return self._hier.levels[self.level].spec

    @property
    def kernels(self) -> np.ndarray:
        if self._kernels is None:
            self._kernels = self._hier._download_kernels(self.level, self.k)
        return self._kernels

    def apply(self, r: GridFunction) -> GridFunction:
        return InferredSmoother(self.spec, self.kernels, self.k, self.slope).apply(r)


class MultigridHierarchy:
    """hierarchy.py:38-51 backed by an mgb_hier handle on one GPU."""

    def __init__(self, handle: C.c_void_p, device: int, batch: int, specs: list, transfers: list,
                 A0: StencilField | None):
        self._h = handle
        self.device = device
        self.batch = batch
        self.scheme = "full"
        self.levels = [Level(self, l, specs[l], transfers[l], A0 if l == 0 else None)
                       for l in range(len(specs))]
        self._installed = [None] * len(specs)
        self._pool = []
        self._lock = threading.Lock()
        self.coarse_lu = None
        self.coarse_perm = None

    # -- lifetime ----------------------------------------------------------
    def __del__(self):
        try:
            for w in self._pool:
                _lib.lib().mgb_work_destroy(w)
            if self._h:
                _lib.lib().mgb_hier_destroy(self._h)
        except Exception:
            pass
        self._h = None

    @property
    def depth(self) -> int:
        return len(self.levels)

    @property
    def finest(self) -> Level:
        return self.levels[0]

    @property
    def handle(self):
        return self._h

    # -- workspaces: one per concurrent solve -----------------
    def acquire_work(self):
        with self._lock:
            if self._pool:
                return self._pool.pop()
        w = C.c_void_p()
        _lib.call("mgb_work_create", self._h, C.byref(w))
        return w

    def release_work(self, w):
        with self._lock:
            self._pool.append(w)

    # -- level data ----------------------------------------------------------
    def level_info(self, l: int):
        r, c, k, ks = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        h = C.c_double()
        _lib.call("mgb_hier_level_info", self._h, l, C.byref(r), C.byref(c), C.byref(k), C.byref(ks), C.byref(h))
        return r.value, c.value, k.value, ks.value, h.value

    def _download_operator(self, l: int) -> StencilField:
        rows, cols, k, _, _ = self.level_info(l)
        out = np.empty((self.batch, rows, cols, k, k))
        _lib.call("mgb_hier_get_operator", self._h, l, out.ctypes.data_as(_lib.P))
        return StencilField(self.levels[l].spec, out[0] if self.batch == 1 else out[0])

    def operator_batch(self, l: int) -> np.ndarray:
        rows, cols, k, _, _ = self.level_info(l)
        out = np.empty((self.batch, rows, cols, k, k))
        _lib.call("mgb_hier_get_operator", self._h, l, out.ctypes.data_as(_lib.P))
        return out

    def _download_kernels(self, l: int, k: int) -> np.ndarray:
        rows, cols, _, ks, _ = self.level_info(l)
        out = np.empty((self.batch, rows, cols, ks, 3, 3))
        _lib.call("mgb_hier_get_kernels", self._h, l, out.ctypes.data_as(_lib.P))
        return out[0]

    def kernels_batch(self, l: int) -> np.ndarray:
        rows, cols, _, ks, _ = self.level_info(l)
        out = np.empty((self.batch, rows, cols, ks, 3, 3))
        _lib.call("mgb_hier_get_kernels", self._h, l, out.ctypes.data_as(_lib.P))
        return out

    # -- table storage ---------------------------------------------------------
    def set_storage(self, mode: str = "auto"):
        """'auto': exact band-class tables where a level's table allows it (default);
        'planes': per-point planes everywhere.  Results are bit-identical."""
        _lib.call("mgb_hier_set_storage", self._h, {"auto": 0, "planes": 1}[mode], None)

    def set_fused(self, mode=2):
        """Pass structure: 2 (default) one streaming pass per smoothing phase, 1 one
        streaming pass per sweep, 0 / False separate sweep, restriction, prolongation."""
        _lib.call("mgb_hier_set_fused", self._h, int(mode))

    def set_passes(self, stream_min: int = -1, tile: int = -1, coarse_max: int = -1):
        """Levels with batch*rows*cols >= stream_min run row-streaming passes, smaller
        ones tile-local passes (tile=1) or separate kernels (tile=0); levels of at most
        coarse_max points run in the single-launch coarse kernel (0 = off); -1 keeps a
        setting."""
        _lib.call("mgb_hier_set_passes", self._h, int(stream_min), int(tile), int(coarse_max))

    def set_stream_kernel(self, kind: int = 0):
        """Row-streaming kernel: 0 auto, 1 one column per thread, 2 column pairs,
        3 one warp per 128-column strip (single-problem band-class levels);
        bit-identical results."""
        _lib.call("mgb_hier_set_stream_kernel", self._h, int(kind))

    def storage_info(self, l: int):
        """(A class-compact, M class-compact) for level l."""
        a, k = C.c_int(), C.c_int()
        _lib.call("mgb_hier_storage_info", self._h, l, C.byref(a), C.byref(k))
        return bool(a.value), bool(k.value)

    def stencil_points(self, l: int) -> int:
        """Operator entries per point the streaming passes read for level l's per-point
        A: 5 (zero corner planes), 9, or 0 when A is class-compact."""
        p = C.c_int()
        _lib.call("mgb_hier_stencil_points", self._h, l, C.byref(p))
        return p.value

    def level_uniformity(self, l: int) -> int:
        """1: level l's band classes all equal the interior one; 2: they differ only on the
        first / last row and column (A only in entries that point out of the grid); 0 neither."""
        p = C.c_int()
        _lib.call("mgb_hier_level_uniformity", self._h, l, C.byref(p))
        return p.value

    PASS_KERNELS = {0: "separate kernels", 1: "k_stream (one column per thread)", 2: "k_stream2 (column pairs)",
                    3: "k_stream3 (one warp per 128-column strip, four columns per lane)", 4: "k_tile (tile-local passes)"}

    def pass_kernel(self, l: int, nu: int) -> str:
        """Name of the kernel that runs level l's fused V(nu, nu) passes."""
        k = C.c_int()
        _lib.call("mgb_hier_pass_kernel", self._h, l, int(nu), C.byref(k))
        return self.PASS_KERNELS[k.value]

    # -- smoother bookkeeping ------------------------------------------------
    def _sweeps(self, nu1, nu2):
        """Resolve (nu1, nu2) and make sure the device holds each level's smoother."""
        steps = set()
        for lev in self.levels[:-1]:
            sm = lev.smoother
            if sm is None:
                raise ConfigError(f"level {lev.index} has no smoother installed")
            base = sm
            if hasattr(sm, "inner") and hasattr(sm, "steps"):
                steps.add(int(sm.steps))
                base = sm.inner
            else:
                steps.add(1)
            if base is not self._installed[lev.index]:
                self._install(lev.index, base)
        if nu1 is None or nu2 is None:
            if len(steps) != 1:
                raise ConfigError("levels use different sweep counts; pass nu1/nu2 explicitly")
            nu = steps.pop()
            nu1 = nu if nu1 is None else nu1
            nu2 = nu if nu2 is None else nu2
        return int(nu1), int(nu2)

    def _install(self, l: int, sm):
        """Upload an arbitrary per-point smoother (InferredSmoother / JacobiSmoother)."""
        if isinstance(sm, DeviceSmoother) and sm._hier is self:
            self._installed[l] = sm
            return
        if isinstance(sm, ConvSmoother):
            if sm.spec != self.levels[l].spec:
                raise ContractError(f"smoother on level {l} is bound to a different grid")
            layers, skip = sm.device_args()
            _lib.call("mgb_hier_set_conv_smoother", self._h, l, len(sm.layers), layers.ctypes.data_as(_lib.P),
                      None if skip is None else skip.ctypes.data_as(_lib.P), 1 if sm.activation == "leaky" else 0,
                      float(sm.slope), float(sm.gain))
            self._installed[l] = sm
            return
        if isinstance(sm, JacobiSmoother):
            K, k, slope = sm.kernels(), 1, LEAKY_SLOPE
        elif isinstance(sm, InferredSmoother) or hasattr(sm, "kernels"):
            K, k, slope = np.asarray(sm.kernels, dtype=float), int(sm.k), float(sm.slope)
        else:
            raise UnsupportedOperationError(
                f"smoother {type(sm).__name__} on level {l} has no per-point kernels for the B200 path")
        if sm.spec != self.levels[l].spec:
            raise ContractError(f"smoother on level {l} is bound to a different grid")
        K = np.ascontiguousarray(np.broadcast_to(K, (self.batch,) + K.shape))
        _lib.call("mgb_hier_set_kernels", self._h, l, k, K.ctypes.data_as(_lib.P), 0, slope, None)
        self._installed[l] = sm

    # -- device-resident entry points (torch CUDA tensors) -------------------
    def _check_dev(self, x, name: str, count: int | None = None):
        """The C-ABI takes raw pointers: refuse anything but a C-contiguous fp64
        CUDA tensor on this hierarchy's device holding exactly `count` values
        (default: one level-0 grid function per problem; histories: at least)."""
        t = dv.torch()
        if not isinstance(x, t.Tensor):
            raise ContractError(f"{name} must be a CUDA tensor")
        if x.dtype != t.float64:
            raise ContractError(f"{name} must be float64, got {x.dtype}")
        if not x.is_cuda or x.device.index != self.device:
            raise ContractError(f"{name} must live on cuda:{self.device}, got {x.device}")
        if not x.is_contiguous():
            raise ContractError(f"{name} must be contiguous")
        spec = self.levels[0].spec
        if count is None:
            want = self.batch * spec.rows * spec.cols
            shapes = [(self.batch, spec.rows, spec.cols)] + ([(spec.rows, spec.cols)] if self.batch == 1 else [])
            if x.numel() != want or tuple(x.shape) not in shapes:
                raise ContractError(f"{name} has shape {tuple(x.shape)}, expected {shapes[0]}")
        elif x.numel() < count:
            raise ContractError(f"{name} holds {x.numel()} values, needs {count}")

    def run_cycles(self, f, u, cycles: int, nu1: int | None = None, nu2: int | None = None,
                   history=None, u_zero: bool = False):
        """Fixed-count V(nu1, nu2) loop entirely on the device: f, u are
        (batch, rows, cols) or (rows, cols) fp64 CUDA tensors; returns the
        (batch, cycles + 1) relative-residual history tensor (no host sync)."""
        nu1, nu2 = self._sweeps(nu1, nu2)
        if cycles < 0:
            raise ConfigError("cycles must be non-negative")
        t = dv.torch()
        self._check_dev(f, "f")
        self._check_dev(u, "u")
        if history is None:
            history = t.empty((self.batch, cycles + 1), dtype=t.float64, device=f.device)
        self._check_dev(history, "history", self.batch * (cycles + 1))
        w = self.acquire_work()
        try:
            _lib.call("mgb_run_cycles", self._h, w, dv.ptr(f), dv.ptr(u), nu1, nu2, int(cycles),
                      1 if u_zero else 0, dv.ptr(history), dv.stream(f))
            self.last_launches = int(_lib.lib().mgb_last_launch_count(w))
        finally:
            self.release_work(w)
        return history

    def _check_host(self, fs, us, hs, cycles: int):
        if cycles < 0:
            raise ConfigError("cycles must be non-negative")
        spec = self.levels[0].spec
        want = self.batch * spec.rows * spec.cols
        if len(hs) != len(fs):
            raise ContractError("one history buffer per solve")
        for a in list(fs) + list(us) + list(hs):
            if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ContractError("host buffers must be C-contiguous float64")
        for a in list(fs) + list(us):
            if a.size != want:
                raise ContractError(f"host grid buffer holds {a.size} values, expected {want}")
        for a in hs:
            if a.size < self.batch * (cycles + 1):
                raise ContractError(f"history buffer holds {a.size} values, needs {self.batch * (cycles + 1)}")

    def run_cycles_host(self, f_host: np.ndarray, u_host: np.ndarray, cycles: int, nu1: int | None = None,
                        nu2: int | None = None, history_host: np.ndarray | None = None, u_zero: bool = False,
                        stream=None) -> np.ndarray:
        """Host-buffer cycle loop through mgb_run_cycles_host: f_host / u_host are
        C-contiguous fp64 arrays (pinned for full-speed copies); u_host is updated
        in place; returns the (batch, cycles + 1) history."""
        nu1, nu2 = self._sweeps(nu1, nu2)
        if history_host is None:
            history_host = np.empty((self.batch, cycles + 1))
        self._check_host([f_host], [u_host], [history_host], cycles)
        w = self.acquire_work()
        try:
            _lib.call("mgb_run_cycles_host", self._h, w, f_host.ctypes.data_as(_lib.P),
                      u_host.ctypes.data_as(_lib.P), nu1, nu2, int(cycles), 1 if u_zero else 0,
                      history_host.ctypes.data_as(_lib.P), stream)
            self.last_launches = int(_lib.lib().mgb_last_launch_count(w))
        finally:
            self.release_work(w)
        return history_host

    def run_cycles_host_many(self, f_hosts, u_hosts, cycles: int, nu1: int | None = None, nu2: int | None = None,
                             history_hosts=None, u_zero: bool = False, stream=None):
        """A stream of independent host-buffer solves (mgb_run_cycles_host_many):
        copies of neighbouring solves overlap each solve's cycles.  Lists of
        C-contiguous fp64 arrays (pinned for full-speed copies); u_hosts updated
        in place; returns the list of (batch, cycles + 1) histories."""
        nu1, nu2 = self._sweeps(nu1, nu2)
        count = len(f_hosts)
        if len(u_hosts) != count:
            raise ContractError("f_hosts and u_hosts differ in length")
        if history_hosts is None:
            history_hosts = [np.empty((self.batch, cycles + 1)) for _ in range(count)]
        self._check_host(f_hosts, u_hosts, history_hosts, cycles)
        arr = lambda xs: (C.c_void_p * max(count, 1))(*[x.ctypes.data for x in xs])  # noqa: E731
        fp, up, hp = arr(f_hosts), arr(u_hosts), arr(history_hosts)
        w = self.acquire_work()
        try:
            _lib.call("mgb_run_cycles_host_many", self._h, w, count, C.cast(fp, C.c_void_p), C.cast(up, C.c_void_p),
                      nu1, nu2, int(cycles), 1 if u_zero else 0, C.cast(hp, C.c_void_p), stream)
            self.last_launches = int(_lib.lib().mgb_last_launch_count(w))
        finally:
            self.release_work(w)
        return history_hosts

    def solve_device(self, f, u, tol: float = 1e-6, max_iter: int = 100, nu1=None, nu2=None) -> SolveReport:
        nu1, nu2 = self._sweeps(nu1, nu2)
        self._check_dev(f, "f")
        self._check_dev(u, "u")
        hist = np.zeros(max_iter + 1)
        nh, it, conv, secs = C.c_int(), C.c_int(), C.c_int(), C.c_double()
        w = self.acquire_work()
        try:
            _lib.call("mgb_solve", self._h, w, dv.ptr(f), dv.ptr(u), nu1, nu2, float(tol), int(max_iter),
                      hist.ctypes.data_as(_lib.PD), C.byref(nh), C.byref(it), C.byref(conv), C.byref(secs),
                      dv.stream(f))
        finally:
            self.release_work(w)
        return SolveReport(it.value, hist[:nh.value].tolist(), bool(conv.value), secs.value)


# ---------------------------------------------------------------------------
# module API (hierarchy.py:62-214)

def _level_specs(spec: GridSpec, levels: int):
    specs, transfers = [spec], []
    for step in range(levels - 1):
        try:
            tp = coarsen_full(specs[-1])
        except ConfigError as exc:
            raise ConfigError(f"level {step}: {exc}") from exc
        if tp.coarse.n_active >= specs[-1].n_active:
            raise ConfigError(f"level {step}: coarsening does not shrink the active set")
        transfers.append(tp)
        specs.append(tp.coarse)
    transfers.append(None)
    return specs, transfers


def build_hierarchy(A: StencilField, levels: int, scheme: str = "full", device: int | None = None) -> MultigridHierarchy:
    """hierarchy.py:70-88: Galerkin chain + coarsest LU, built on the GPU."""
    if levels < 2:
        raise ConfigError("a hierarchy needs at least two levels")
    if scheme == "redblack":
        raise UnsupportedOperationError("red-black coarsening is not on the B200 path")
    if scheme != "full":
        raise ConfigError(f"unknown coarsening scheme {scheme!r}")
    if A.k != 3:
        raise UnsupportedOperationError("the device hierarchy takes 3x3 fine-level stencils")
    specs, transfers = _level_specs(A.spec, levels)
    return _build(np.ascontiguousarray(A.data)[None], A.spec, levels, specs, transfers, A, device)


def build_hierarchy_batch(A_batch: np.ndarray, levels: int, spec: GridSpec | None = None,
                          device: int | None = None) -> MultigridHierarchy:
    """A batch of independent problems on one grid (config 4): A_batch is
    (batch, rows, cols, 3, 3); every kernel runs over the batch in one launch."""
    A_batch = np.ascontiguousarray(np.asarray(A_batch, dtype=float))
    if A_batch.ndim != 5 or A_batch.shape[3:] != (3, 3):
        raise ContractError("batched operators must be (batch, rows, cols, 3, 3)")
    if not np.isfinite(A_batch).all():
        from .errors import NumericError
        raise NumericError("non-finite stencil weights")
    if levels < 2:
        raise ConfigError("a hierarchy needs at least two levels")
    rows, cols = A_batch.shape[1:3]
    if spec is None:
        spec = GridSpec(rows, cols, 1.0 / (rows + 1), np.ones((rows, cols), bool))
    specs, transfers = _level_specs(spec, levels)
    return _build(A_batch, spec, levels, specs, transfers, None, device)


def build_hierarchy_classed(rows: int, cols: int, tables, levels: int, spacing: float | None = None,
                            device: int | None = None) -> MultigridHierarchy:
    """Constant-coefficient hierarchy held entirely as band-class tables (no
    per-point planes on any level): memory is O(grid functions), so config 5's
    32767^2 fits one GPU.  `tables` is one 3x3 stencil (a constant_stencil,
    grid.py:209), or (25, 3, 3) band-class tables, or (batch, 25, 3, 3); band
    classes are band(i) * 5 + band(j) with band = 0, 1 for the first two
    rows/cols, 2 inside, 3, 4 for the last two.  Results equal build_hierarchy
    on the expanded per-point operator."""
    t = np.asarray(tables, dtype=float)
    if t.shape == (3, 3):
        t = np.broadcast_to(t, (1, 25, 3, 3))
    elif t.shape == (25, 3, 3):
        t = t[None]
    if t.ndim != 4 or t.shape[1:] != (25, 3, 3):
        raise ContractError("band-class tables must be (3, 3), (25, 3, 3) or (batch, 25, 3, 3)")
    t = np.ascontiguousarray(t)
    if levels < 2:
        raise ConfigError("a hierarchy needs at least two levels")
    spec = GridSpec(rows, cols, 1.0 / (rows + 1) if spacing is None else spacing, np.ones((rows, cols), bool))
    specs, transfers = _level_specs(spec, levels)
    dev = dv.current_device() if device is None else device
    dv.require_cuda(dev)
    h = C.c_void_p()
    _lib.call("mgb_hier_build_classed", dev, t.shape[0], rows, cols, float(spec.spacing), t.ctypes.data_as(_lib.P),
              int(levels), None, C.byref(h))
    return MultigridHierarchy(h, dev, t.shape[0], specs, transfers, None)


def _build(A_host, spec, levels, specs, transfers, A0, device):
    dev = dv.current_device() if device is None else device
    dv.require_cuda(dev)
    mask = None if spec.all_active else np.ascontiguousarray(spec.mask.astype(np.uint8))
    h = C.c_void_p()
    _lib.call("mgb_hier_build", dev, A_host.shape[0], spec.rows, spec.cols, float(spec.spacing),
              A_host.ctypes.data_as(_lib.P), 0, None if mask is None else mask.ctypes.data_as(_lib.P),
              int(levels), None, C.byref(h))
    return MultigridHierarchy(h, dev, A_host.shape[0], specs, transfers, A0)


def coarse_solve(hier: MultigridHierarchy, f: GridFunction) -> GridFunction:
    """hierarchy.py:91-93 (LU solve on the device)."""
    x = dv.to_dev(f.values)
    out = dv.empty(x.shape)
    _lib.call("mgb_coarse_solve", hier.handle, dv.ptr(x), dv.ptr(out), dv.stream(out))
    return GridFunction(f.spec, dv.host(out))


def v_cycle(hier: MultigridHierarchy, level: int, f: GridFunction, u: GridFunction,
            nu1: int | None = None, nu2: int | None = None) -> GridFunction:
    """hierarchy.py:96-111; V(nu1, nu2) from RepeatedSmoother wrappers or the arguments."""
    if level < 0 or level >= hier.depth:
        raise ConfigError(f"v_cycle: level {level} out of range")
    lev = hier.levels[level]
    if f.spec != lev.spec or u.spec != lev.spec:
        raise ConfigError(f"v_cycle: data not on level-{level} spec")
    if level == hier.depth - 1:
        return coarse_solve(hier, f)
    nu1, nu2 = hier._sweeps(nu1, nu2)
    fd = dv.to_dev(f.values)
    ud = dv.to_dev(u.values)
    w = hier.acquire_work()
    try:
        _lib.call("mgb_vcycle", hier.handle, w, level, dv.ptr(fd), dv.ptr(ud), nu1, nu2, dv.stream(ud))
    finally:
        hier.release_work(w)
    return GridFunction(lev.spec, dv.host(ud))


def cycle_correction(hier: MultigridHierarchy, r: GridFunction) -> GridFunction:
    """hierarchy.py:114-116."""
    return v_cycle(hier, 0, r, zeros(hier.finest.spec))


def solve(hier: MultigridHierarchy, f: GridFunction, u0: GridFunction | None = None, tol: float = 1e-6,
          max_iter: int = 100, nu1: int | None = None, nu2: int | None = None):
    """hierarchy.py:119-146: returns (u, SolveReport); NonConvergedError on divergence."""
    if tol <= 0.0:
        raise ConfigError("tolerance must be positive")
    if hier.batch != 1:
        raise ContractError("solve() takes a single-problem hierarchy; use run_cycles for batches")
    spec = hier.finest.spec
    if f.spec != spec:
        raise ConfigError("solve: right-hand side not on the finest spec")
    fd = dv.to_dev(f.values)
    ud = dv.zeros(fd.shape) if u0 is None else dv.to_dev(u0.values)
    rep = hier.solve_device(fd, ud, tol, max_iter, nu1, nu2)
    return GridFunction(spec, dv.host(ud)), rep


def equip_classical(hier: MultigridHierarchy, kind: str = "jacobi", omega: float = 2.0 / 3.0) -> MultigridHierarchy:
    """hierarchy.py:152-161 (jacobi on the device)."""
    if kind == "gauss-seidel":
        raise UnsupportedOperationError("Gauss-Seidel (sequential sweep) is not on the B200 path")
    if kind != "jacobi":
        raise ConfigError(f"unknown classical smoother {kind!r}")
    _lib.call("mgb_hier_equip_jacobi", hier.handle, float(omega), None)
    for lev in hier.levels[:-1]:
        sm = DeviceSmoother(hier, lev.index, 1, LEAKY_SLOPE, "jacobi", omega)
        lev.smoother = sm
        hier._installed[lev.index] = sm
    return hier


def equip_conv_init(hier: MultigridHierarchy, omega: float = 2.0 / 3.0, activation: str = "linear") -> MultigridHierarchy:
    """hierarchy.py:164-172: Jacobi-equivalent five-layer conv smoothers (full
    coarsening) on every smoothed level, run on the GPU."""
    for lev in hier.levels[:-1]:
        lev.smoother = conv_smoother(lev.operator, "full", omega, activation)
        hier._install(lev.index, lev.smoother)
    return hier


def retarget(sm: ConvSmoother, source: StencilField, target: StencilField) -> ConvSmoother:
    """hierarchy.py:175-182: rebind a trained conv smoother to an operator of
    another scale (ratio of representative diagonals in the gain)."""
    gain = sm.gain * representative_diagonal(source) / representative_diagonal(target)
    return ConvSmoother(target.spec, sm.form, list(sm.layers), sm.skip, sm.activation, sm.slope, gain)


def equip_trained(target: MultigridHierarchy, source: MultigridHierarchy) -> MultigridHierarchy:
    """hierarchy.py:185-204: install another hierarchy's conv smoothers level by
    level (deeper targets reuse the deepest), re-scaled to the target operators."""
    for l, lev in enumerate(target.levels[:-1]):
        ls = min(l, source.depth - 2)
        src = source.levels[ls].smoother
        if src is None:
            raise ConfigError(f"source level {ls} has no trained smoother")
        if not isinstance(src, ConvSmoother):
            raise ConfigError("only convolutional smoothers can be transported")
        lev.smoother = retarget(src, source.levels[ls].operator, lev.operator)
        target._install(l, lev.smoother)
    return target


def equip_inferred(hier: MultigridHierarchy, net: KernelInferenceNet, precision: int = 64) -> MultigridHierarchy:
    """hierarchy.py:207-214: CNN inference of every smoothed level on the device."""
    for lev in hier.levels[:-1]:
        if hier.level_info(lev.index)[2] != 3:
            raise ConfigError("kernel inference needs 3x3 stencils on every level")
    W = net.flat_weights()
    _lib.call("mgb_hier_equip_inferred", hier.handle, VARIANT_ID[net.variant], int(net.k),
              W.ctypes.data_as(_lib.P), W.size, float(net.slope), int(precision), None)
    for lev in hier.levels[:-1]:
        sm = DeviceSmoother(hier, lev.index, net.k, net.slope, f"inferred-{net.variant}")
        lev.smoother = sm
        hier._installed[lev.index] = sm
    return hier
