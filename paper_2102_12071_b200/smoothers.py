"""Smoothers and the stencil -> smoother-kernel inference net — facade over the
B200 kernels (reference smoothers.py:1-414).

* ``infer_kernels`` runs the CNN on the GPU (``mgb_infer_kernels``; fp64 by
  default for parity, ``precision=32`` for the fp32 network).
* ``InferredSmoother.apply`` and ``JacobiSmoother.apply`` run the per-point
  3x3 smoother on the GPU (``mgb_smoother_apply``).
* Model files use the reference's JSON format (smoothers.py:349-414), so nets
  trained by the reference load unchanged.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib, device as dv
from .errors import ConfigError, ContractError, UnsupportedOperationError
from .grid import GridFunction, GridSpec, StencilField

LEAKY_SLOPE = 0.01
_FC_SIZES = (81, 40, 40, 40)
_CONV_CHANNELS = (7, 5, 3)
VARIANT_ID = {"conv": _lib.NET_CONV, "fc": _lib.NET_FC}


def _pointwise_apply(spec: GridSpec, kernels: np.ndarray, kst: int, slope: float, r: GridFunction,
                     kdev=None) -> GridFunction:
    K = kdev if kdev is not None else dv.to_dev(kernels)
    x = dv.to_dev(r.values)
    out = dv.empty(x.shape)
    m = dv.mask_dev(spec.mask)
    _lib.call("mgb_smoother_apply", 1, spec.rows, spec.cols, kst, dv.ptr(K), dv.ptr(m), float(slope),
              dv.ptr(x), dv.ptr(out), dv.stream(out))
    return GridFunction(spec, dv.host(out))


@dataclass
class JacobiSmoother:
    """smoothers.py:29-41: omega * r / diag, run as a centre-only per-point kernel."""
    spec: GridSpec
    diag: np.ndarray
    omega: float = 2.0 / 3.0

    def kernels(self) -> np.ndarray:
        k = np.zeros((self.spec.rows, self.spec.cols, 1, 3, 3))
        m = self.spec.mask
        k[:, :, 0, 1, 1] = np.where(m, self.omega / np.where(m, self.diag, 1.0), 0.0)
        return k

    def apply(self, r: GridFunction) -> GridFunction:
        if r.spec != self.spec:
            raise ContractError("jacobi: residual on a different spec")
        return _pointwise_apply(self.spec, self.kernels(), 1, LEAKY_SLOPE, r)


def jacobi(A: StencilField, omega: float = 2.0 / 3.0) -> JacobiSmoother:
    """smoothers.py:44-50."""
    if not 0.0 < omega < 2.0:
        raise ConfigError(f"jacobi weight out of range: {omega}")
    d = A.center()
    if np.any(d[A.spec.mask] == 0.0):
        raise ConfigError("jacobi: operator has zero diagonal entries")
    return JacobiSmoother(A.spec, d, omega)


def gauss_seidel(A: StencilField):
    raise UnsupportedOperationError("Gauss-Seidel (sequential sweep) is not on the B200 path")


@dataclass
class KernelInferenceNet:
    """smoothers.py:217-235: bias-free net shared by every grid point."""
    variant: str
    weights: list
    k: int = 1
    slope: float = LEAKY_SLOPE
    version: int = 0
    _memo: dict = field(default_factory=dict, repr=False)

    def parameter_count(self) -> int:
        return int(sum(np.asarray(w).size for w in self.weights))

    def bump(self):
        self.version += 1
        self._memo.clear()

    def flat_weights(self) -> np.ndarray:
        """Concatenated row-major weights in the order mgb_infer_kernels expects."""
        shapes = ([(a, b) for a, b in zip(_FC_SIZES[:-1], _FC_SIZES[1:])] + [(_FC_SIZES[-1], 9 * self.k)]
                  if self.variant == "fc" else
                  [(c, 3, 3) for c in _CONV_CHANNELS] + [(9 * _CONV_CHANNELS[-1], 9 * self.k)])
        if self.variant not in VARIANT_ID:
            raise ConfigError(f"unknown net variant {self.variant!r}")
        if len(self.weights) != len(shapes):
            raise ConfigError("weight list does not match the net architecture")
        for w, s in zip(self.weights, shapes):
            if tuple(np.asarray(w).shape) != s:
                raise ConfigError(f"weight shape {np.asarray(w).shape} != expected {s}")
        return np.ascontiguousarray(np.concatenate([np.asarray(w, dtype=float).ravel() for w in self.weights]))


def inference_net(variant: str, k: int = 1, seed: int = 0) -> KernelInferenceNet:
    """smoothers.py:238-253: He-scaled hidden layers, zero final layer."""
    rng = np.random.default_rng(seed)
    ws = []
    if variant == "fc":
        for a, b in zip(_FC_SIZES[:-1], _FC_SIZES[1:]):
            ws.append(rng.standard_normal((a, b)) * math.sqrt(2.0 / a))
        ws.append(np.zeros((_FC_SIZES[-1], 9 * k)))
    elif variant == "conv":
        for c in _CONV_CHANNELS:
            ws.append(rng.standard_normal((c, 3, 3)) * math.sqrt(2.0 / 9.0))
        ws.append(np.zeros((9 * _CONV_CHANNELS[-1], 9 * k)))
    else:
        raise ConfigError(f"unknown net variant {variant!r}")
    return KernelInferenceNet(variant, ws, k)


@dataclass
class InferredSmoother:
    """smoothers.py:291-299: per-point kernels (rows, cols, k, 3, 3)."""
    spec: GridSpec
    kernels: np.ndarray
    k: int
    slope: float = LEAKY_SLOPE

    def apply(self, r: GridFunction) -> GridFunction:
        if r.spec != self.spec:
            raise ContractError("inferred smoother: residual on a different spec")
        return _pointwise_apply(self.spec, self.kernels, self.k, self.slope, r)


def infer_kernels(net: KernelInferenceNet, A: StencilField, precision: int = 64) -> InferredSmoother:
    """smoothers.py:302-322 on the GPU; memoised per (operator, net version)."""
    key = (id(A), precision)
    hit = net._memo.get(key)
    if hit is not None and hit[0] is A and hit[1] == net.version:
        return hit[2]
    if A.k != 3:
        raise ContractError("feature map defined for 3x3 stencils only")
    W = net.flat_weights()
    Ad = dv.to_dev(A.data)
    m = dv.mask_dev(A.spec.mask)
    K = dv.empty((A.spec.rows, A.spec.cols, net.k, 3, 3))
    _lib.call("mgb_infer_kernels", 1, A.spec.rows, A.spec.cols, dv.ptr(Ad), dv.ptr(m), VARIANT_ID[net.variant],
              net.k, W.ctypes.data_as(_lib.P), W.size, float(net.slope), int(precision), dv.ptr(K),
              dv.stream(K))
    sm = InferredSmoother(A.spec, dv.host(K), net.k, net.slope)
    net._memo[key] = (A, net.version, sm)
    return sm


# ---------------------------------------------------------------------------
# model files (smoothers.py:349-414)

FORMAT_VERSION = 1


def model_to_dict(model, metadata: dict | None = None) -> dict:
    if not isinstance(model, KernelInferenceNet):
        raise ConfigError(f"cannot serialize {type(model).__name__}")
    return {"format_version": FORMAT_VERSION, "metadata": metadata or {}, "kind": "inference_net",
            "variant": model.variant, "k": model.k, "slope": model.slope,
            "weights": [{"shape": list(np.asarray(w).shape), "data": np.asarray(w).ravel().tolist()}
                        for w in model.weights]}


def model_from_dict(doc: dict, spec: GridSpec | None = None):
    if doc.get("format_version") != FORMAT_VERSION:
        raise ConfigError(f"unsupported model format {doc.get('format_version')!r}")
    kind = doc.get("kind")
    if kind == "inference_net":
        ws = [np.array(it["data"], dtype=float).reshape(it["shape"]) for it in doc["weights"]]
        return KernelInferenceNet(doc["variant"], ws, int(doc["k"]), float(doc["slope"]))
    if kind == "conv_smoother":
        raise UnsupportedOperationError("shared-kernel ConvSmoother is not on the B200 path yet")
    raise ConfigError(f"unknown model kind {kind!r}")


def save_model(path, model, metadata: dict | None = None):
    with open(path, "w") as fh:
        json.dump(model_to_dict(model, metadata), fh)


def load_model(path, spec: GridSpec | None = None):
    with open(path) as fh:
        return model_from_dict(json.load(fh), spec)
