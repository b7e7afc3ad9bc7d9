"""Flexible GMRES with the multigrid V-cycle as right preconditioner — facade
over the B200 C-ABI (``mgb_krylov``, csrc/mgb_krylov.cu).

Mirrors the reference's krylov.py:1-270 (same names, arguments, report and
exceptions).  The operator is a device stencil action (``grid_action``), the
preconditioner one V-cycle from zero on a device hierarchy
(``cycle_preconditioner``); the Arnoldi vectors live in HBM and every vector
operation is a CUDA kernel, with the scalar recurrences (Hessenberg, Givens
rotations, back substitution) on the host in the reference's order.

Only device operators run here: ``fgmres``/``gmres`` raise
UnsupportedOperationError for arbitrary Python callables (there is no CPU path).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib, device as dv
from .errors import ConfigError, ContractError, UnsupportedOperationError
from .grid import GridFunction, StencilField, apply_stencil, zeros


@dataclass
class FgmresConfig:
    """krylov.py:23-43: stopping rule and subspace budget (restart=None: one
    unrestarted cycle of up to max_iter Arnoldi steps)."""

    tol: float = 1e-6
    max_iter: int = 200
    restart: Optional[int] = None

    def __post_init__(self):
        if self.tol <= 0:
            raise ConfigError(f"tol must be positive, got {self.tol}")
        if self.max_iter < 1:
            raise ConfigError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.restart is not None and self.restart < 1:
            raise ConfigError(f"restart must be >= 1, got {self.restart}")


@dataclass
class KrylovReport:
    """krylov.py:46-51."""

    iterations: int
    history: list
    converged: bool
    preconditioner: str


class GridAction:
    """krylov.py:249-258: flat-vector view of a stencil operator.  Calling it on a
    flat NumPy vector applies the stencil on the GPU (grid.py:216)."""

    def __init__(self, A: StencilField):
        if A.k != 3:
            raise UnsupportedOperationError("the device Krylov path takes 3x3 stencils")
        self.A = A
        self.spec = A.spec
        self._dev = None
        self._mask = None

    def device_operator(self):
        if self._dev is None:
            self._dev = dv.to_dev(np.ascontiguousarray(self.A.data))
            self._mask = None if self.spec.all_active else dv.mask_dev(self.spec.mask)
        return self._dev, self._mask

    def __call__(self, x: np.ndarray) -> np.ndarray:
        shape = (self.spec.rows, self.spec.cols)
        return apply_stencil(self.A, GridFunction(self.spec, np.asarray(x, float).reshape(shape))).values.ravel()


class CyclePreconditioner:
    """krylov.py:261-270: one V(nu1, nu2)-cycle from a zero initial guess on the
    masked residual.  nu1 / nu2 default to the hierarchy's RepeatedSmoother steps
    (as v_cycle does)."""

    def __init__(self, hier, nu1: int | None = None, nu2: int | None = None):
        self.hier = hier
        self.spec = hier.finest.spec
        self.nu1, self.nu2 = nu1, nu2

    def sweeps(self):
        return self.hier._sweeps(self.nu1, self.nu2)

    def __call__(self, r: np.ndarray) -> np.ndarray:
        from .hierarchy import v_cycle
        shape = (self.spec.rows, self.spec.cols)
        f = GridFunction(self.spec, np.asarray(r, float).reshape(shape) * self.spec.mask)
        nu1, nu2 = self.sweeps()
        return v_cycle(self.hier, 0, f, zeros(self.spec), nu1, nu2).values.ravel()


def grid_action(A: StencilField) -> GridAction:
    return GridAction(A)


def cycle_preconditioner(hier, nu1: int | None = None, nu2: int | None = None) -> CyclePreconditioner:
    return CyclePreconditioner(hier, nu1, nu2)


def _run(method: int, apply_a, f, precond, cfg: FgmresConfig):
    if not isinstance(apply_a, GridAction):
        raise UnsupportedOperationError("the B200 Krylov path needs a device operator from grid_action(A)")
    if precond is not None and not isinstance(precond, CyclePreconditioner):
        raise UnsupportedOperationError("the B200 Krylov path needs cycle_preconditioner(hier) or None")
    spec = apply_a.spec
    n = spec.rows * spec.cols
    t = dv.torch()
    on_device = t.is_tensor(f)
    fd = f if on_device else dv.to_dev(np.ascontiguousarray(np.asarray(f, dtype=float)).ravel())
    if fd.numel() != n:
        raise ContractError(f"right-hand side has {fd.numel()} entries, the grid {n}")
    fd = fd.reshape(-1).contiguous()
    A, mask = apply_a.device_operator()
    u = dv.empty((n,), device=fd.device.index)
    pc, nu1, nu2, w = None, 0, 0, None
    if precond is not None:
        if not precond.spec.same_lattice(spec):
            raise ContractError("preconditioner hierarchy and operator live on different grids")
        nu1, nu2 = precond.sweeps()
        w = precond.hier.acquire_work()
        pc = w
    hist = np.zeros(cfg.max_iter + 1)
    nh, it, conv = C.c_int(), C.c_int(), C.c_int()
    try:
        _lib.call("mgb_krylov", method, spec.rows, spec.cols, dv.ptr(A), None if mask is None else dv.ptr(mask),
                  pc, int(nu1), int(nu2), dv.ptr(fd), dv.ptr(u), float(cfg.tol), int(cfg.max_iter),
                  int(cfg.restart or 0), hist.ctypes.data_as(_lib.PD), C.byref(nh), C.byref(it), C.byref(conv),
                  dv.stream(fd))
    finally:
        if w is not None:
            precond.hier.release_work(w)
    out = u if on_device else dv.host(u)
    return out, it.value, hist[:nh.value].tolist(), bool(conv.value)


def fgmres(apply_a, f, precond=None, cfg: Optional[FgmresConfig] = None, tag: Optional[str] = None):
    """krylov.py:138-164: right-preconditioned flexible GMRES.  Returns
    (u, KrylovReport); running out of iterations is a non-converged report."""
    cfg = cfg or FgmresConfig()
    if tag is None:
        tag = "none" if precond is None else "preconditioned"
    u, it, hist, conv = _run(0, apply_a, f, precond, cfg)
    return u, KrylovReport(it, hist, conv, tag)


def gmres(apply_a, f, cfg: Optional[FgmresConfig] = None):
    """krylov.py:167-236: plain GMRES, its own restart loop and history."""
    cfg = cfg or FgmresConfig()
    u, it, hist, conv = _run(1, apply_a, f, None, cfg)
    return u, KrylovReport(it, hist, conv, "none")
