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
from .grid import (ConvKernel, GridFunction, GridSpec, StencilField, compose_kernels, delta_kernel, pad_kernel)

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
# shared-kernel convolutional smoother (smoothers.py:99-178)

def representative_diagonal(A: StencilField) -> float:
    """smoothers.py:99-102: median active centre entry."""
    return float(np.median(A.center()[A.spec.mask]))


@dataclass
class ConvSmoother:
    """smoothers.py:105-145: form "full" = five chained 3x3 kernels plus a
    parallel skip kernel, "rb" = two chained kernels and no skip; optional leaky
    activation between chained layers; gain rescales the output.  ``apply`` and
    the V-cycle run it on the GPU (mgb_conv.cu), bit-identical to the reference."""
    spec: GridSpec
    form: str
    layers: list
    skip: ConvKernel | None
    activation: str = "linear"
    slope: float = LEAKY_SLOPE
    gain: float = 1.0

    def __post_init__(self):
        if self.form not in ("full", "rb"):
            raise ConfigError(f"unknown smoother form {self.form!r}")
        if self.form == "full" and (len(self.layers) != 5 or self.skip is None):
            raise ConfigError("full form takes five layers and a skip kernel")
        if self.form == "rb" and (len(self.layers) != 2 or self.skip is not None):
            raise ConfigError("rb form takes two layers and no skip")
        if self.activation not in ("linear", "leaky"):
            raise ConfigError(f"unknown activation {self.activation!r}")

    def device_args(self):
        if any(k.size != 3 for k in self.layers) or (self.skip is not None and self.skip.size != 3):
            raise UnsupportedOperationError("the device conv smoother takes 3x3 kernels")
        layers = np.ascontiguousarray(np.stack([k.weights for k in self.layers]))
        skip = None if self.skip is None else np.ascontiguousarray(self.skip.weights)
        return layers, skip

    def apply(self, r: GridFunction) -> GridFunction:
        if r.spec != self.spec:
            raise ContractError("conv smoother: residual on a different spec")
        layers, skip = self.device_args()
        x = dv.to_dev(r.values)
        m = dv.mask_dev(r.spec.mask)
        out = dv.empty(x.shape)
        _lib.call("mgb_conv_smoother_apply", 1, r.spec.rows, r.spec.cols, len(self.layers),
                  layers.ctypes.data_as(_lib.P), None if skip is None else skip.ctypes.data_as(_lib.P),
                  1 if self.activation == "leaky" else 0, float(self.slope), float(self.gain), dv.ptr(m),
                  dv.ptr(x), dv.ptr(out), dv.stream(out))
        return GridFunction(self.spec, dv.host(out))

    def is_linear(self) -> bool:
        return self.activation == "linear"


def conv_smoother(A: StencilField, form: str, omega: float = 2.0 / 3.0, activation: str = "linear") -> ConvSmoother:
    """smoothers.py:148-164: initialisation reproducing weighted Jacobi exactly
    (inverse representative diagonal in the gain)."""
    jk = delta_kernel(3, omega)
    gain = 1.0 / representative_diagonal(A)
    if form == "full":
        return ConvSmoother(A.spec, form, [ConvKernel(np.zeros((3, 3))) for _ in range(5)], jk, activation, gain=gain)
    if form == "rb":
        return ConvSmoother(A.spec, form, [delta_kernel(3), jk], None, activation, gain=gain)
    raise ConfigError(f"unknown smoother form {form!r}")


def effective_kernel(s: ConvSmoother) -> ConvKernel:
    """smoothers.py:167-178: the single kernel a linear smoother equals."""
    if s.activation != "linear":
        raise UnsupportedOperationError("effective kernel undefined for nonlinear activation")
    acc = s.layers[0]
    for kern in s.layers[1:]:
        acc = compose_kernels(kern, acc)
    w = acc.weights
    if s.skip is not None:
        w = w + pad_kernel(s.skip, acc.size).weights
    return ConvKernel(s.gain * w)


# ---------------------------------------------------------------------------
# model files (smoothers.py:349-414)

FORMAT_VERSION = 1


def _arrays_to_lists(ws):
    return [{"shape": list(np.asarray(w).shape), "data": np.asarray(w).ravel().tolist()} for w in ws]


def model_to_dict(model, metadata: dict | None = None) -> dict:
    if isinstance(model, ConvSmoother):
        return {"format_version": FORMAT_VERSION, "metadata": metadata or {}, "kind": "conv_smoother",
                "form": model.form, "activation": model.activation, "slope": model.slope, "gain": model.gain,
                "layers": _arrays_to_lists([k.weights for k in model.layers]),
                "skip": _arrays_to_lists([model.skip.weights]) if model.skip is not None else None,
                "spec": {"rows": model.spec.rows, "cols": model.spec.cols, "spacing": model.spec.spacing}}
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
        if spec is None:
            meta = doc["spec"]
            spec = GridSpec(meta["rows"], meta["cols"], meta["spacing"], np.ones((meta["rows"], meta["cols"]), bool))
        lists = lambda items: [np.array(it["data"], dtype=float).reshape(it["shape"]) for it in items]  # noqa: E731
        layers = [ConvKernel(w) for w in lists(doc["layers"])]
        skip = ConvKernel(lists(doc["skip"])[0]) if doc["skip"] is not None else None
        return ConvSmoother(spec, doc["form"], layers, skip, doc["activation"], doc["slope"], doc["gain"])
    raise ConfigError(f"unknown model kind {kind!r}")


def save_model(path, model, metadata: dict | None = None):
    with open(path, "w") as fh:
        json.dump(model_to_dict(model, metadata), fh)


def load_model(path, spec: GridSpec | None = None):
    with open(path) as fh:
        return model_from_dict(json.load(fh), spec)
