"""Host-side input generators for the benchmark configurations (BASELINE.json).

Input assembly is not on the hot path (`problems`); these run once
on the host and produce the same ``(rows, cols, 3, 3)`` fp64 stencil tables the
reference's ``StencilField`` holds (grid.py:163), which are then handed to the
device hierarchy.

* ``rotated_fd``  — the reference's finite-difference rotated anisotropic
  Laplacian, restated from problems.py:23-52 ((a Sxx + c Syy - b Sxy) / h^2).
* ``rotated_q1``  — bilinear (Q1) finite-element 9-point stencil of the same
  operator, scaled by 1/h^2 (BASELINE config 1 names this; the reference has
  no Q1 assembly).
* ``grf_diffusion_5pt`` — config 3: a = exp(g) with g a seeded Gaussian random
  field, cell-centred 5-point finite volumes.
* ``geometry_mask`` — square / lshape / cylinder masks (problems.py:98-120).
"""

from __future__ import annotations

import math

import numpy as np

_SXX = np.array([[0.0, 0.0, 0.0], [-1.0, 2.0, -1.0], [0.0, 0.0, 0.0]])
_SYY = _SXX.T.copy()
_SXY = np.array([[1.0, -1.0, 0.0], [-1.0, 2.0, -1.0], [0.0, -1.0, 1.0]])


def rotated_coefficients(theta: float, eps: float):
    """Diffusion tensor R(theta) diag(1, eps) R(theta)^T entries
    (kxx, kxy, kyy) (problems.py:34-42)."""
    co, si = math.cos(theta), math.sin(theta)
    a = co * co + eps * si * si
    c = si * si + eps * co * co
    b = co * si * (1.0 - eps)
    return a, b, c


def spacing(n: int) -> float:
    """h = 1 / (n + 1) for an n x n interior grid (grid.py:74-77)."""
    return 1.0 / (n + 1)


def rotated_fd(n: int, theta: float, eps: float, cols: int | None = None,
               h: float | None = None) -> np.ndarray:
    """Reference FD rotated Laplacian as a constant per-point table
    (problems.py:45-52 + grid.py:209-213)."""
    if eps <= 0.0:
        raise ValueError("anisotropy must be positive")
    cols = n if cols is None else cols
    h = spacing(n) if h is None else h
    a, b, c = rotated_coefficients(theta, eps)
    table = (a * _SXX + c * _SYY - b * _SXY) / (h * h)
    return np.broadcast_to(table, (n, cols, 3, 3)).copy()


def q1_table(theta: float, eps: float, h: float) -> np.ndarray:
    """Q1 element stencil of -div(K grad u), divided by h^2.

    Rows are y offsets (-1, 0, +1), columns x offsets.  kxx contributes
    (1/6)[[-1,2,-1],[-4,8,-4],[-1,2,-1]], kyy its transpose, and the mixed
    term -kxy/2 on the SW/NE corners and +kxy/2 on NW/SE."""
    kxx, kxy, kyy = rotated_coefficients(theta, eps)
    sxx = np.array([[-1.0, 2.0, -1.0], [-4.0, 8.0, -4.0], [-1.0, 2.0, -1.0]]) / 6.0
    syy = sxx.T.copy()
    sxy = np.array([[-0.5, 0.0, 0.5], [0.0, 0.0, 0.0], [0.5, 0.0, -0.5]])
    return (kxx * sxx + kyy * syy + kxy * sxy) / (h * h)


def rotated_q1(n: int, theta: float, eps: float) -> np.ndarray:
    """Config 1's bilinear-FE 9-point operator."""
    return np.broadcast_to(q1_table(theta, eps, spacing(n)), (n, n, 3, 3)).copy()


def gaussian_random_field(n: int, corr_len: float = 1.0 / 32.0, seed: int = 2) -> np.ndarray:
    """Seeded stationary GRF on the n x n cell centres of the unit square with
    squared-exponential covariance exp(-r^2 / (2 l^2)), standardised to zero
    mean and unit variance.  Spectral synthesis on a periodic box padded by
    4 correlation lengths so the periodic wrap does not couple opposite
    edges."""
    rng = np.random.default_rng(seed)
    pad = int(math.ceil(4.0 * corr_len * n))
    m = n + pad
    k = np.fft.fftfreq(m, d=1.0 / n)              # cycles per unit length
    kk = k[:, None] ** 2 + k[None, :] ** 2
    spec = np.exp(-2.0 * (math.pi ** 2) * (corr_len ** 2) * kk)   # SE covariance spectrum
    noise = rng.standard_normal((m, m))
    g = np.fft.ifft2(np.fft.fft2(noise) * np.sqrt(spec)).real[:n, :n]
    g = g - g.mean()
    return g / g.std()


def grf_diffusion_5pt(n: int, corr_len: float = 1.0 / 32.0, seed: int = 2,
                      g: np.ndarray | None = None) -> np.ndarray:
    """Config 3: -div(a grad u), a = exp(g), cell-centred 5-point finite
    volumes on n x n cells of width h = 1/n.  Interior faces use the harmonic
    mean of the two cell coefficients; a boundary face (zero Dirichlet half a
    cell away) contributes 2 a_P to the centre only, and the off-grid
    neighbour entry is 0."""
    if g is None:
        g = gaussian_random_field(n, corr_len, seed)
    a = np.exp(g)
    h2 = (1.0 / n) ** 2
    A = np.zeros((n, n, 3, 3))

    def harm(x, y):
        return 2.0 * x * y / (x + y)

    # faces: north (i+1), south (i-1), east (j+1), west (j-1)
    tn = np.empty((n, n)); ts = np.empty((n, n)); te = np.empty((n, n)); tw = np.empty((n, n))
    tn[:-1] = harm(a[:-1], a[1:]); tn[-1] = 2.0 * a[-1]
    ts[1:] = harm(a[1:], a[:-1]); ts[0] = 2.0 * a[0]
    te[:, :-1] = harm(a[:, :-1], a[:, 1:]); te[:, -1] = 2.0 * a[:, -1]
    tw[:, 1:] = harm(a[:, 1:], a[:, :-1]); tw[:, 0] = 2.0 * a[:, 0]
    A[:, :, 1, 1] = (tn + ts + te + tw) / h2
    A[:-1, :, 2, 1] = -tn[:-1] / h2
    A[1:, :, 0, 1] = -ts[1:] / h2
    A[:, :-1, 1, 2] = -te[:, :-1] / h2
    A[:, 1:, 1, 0] = -tw[:, 1:] / h2
    return A


def geometry_mask(kind: str, n: int) -> np.ndarray:
    """problems.py:98-120: square, lshape (upper-right ceil(n/2) block
    removed), cylinder (disk of radius n//4 about the centre removed)."""
    mask = np.ones((n, n), dtype=bool)
    if kind == "square":
        return mask
    if kind == "lshape":
        cut = (n + 1) // 2
        mask[n - cut:, n - cut:] = False
        return mask
    if kind == "cylinder":
        c = (n - 1) / 2.0
        r = n // 4
        ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        mask[(ii - c) ** 2 + (jj - c) ** 2 <= r * r] = False
        return mask
    raise ValueError(f"unknown geometry {kind!r}")


def uniform_rhs(n: int, seed, cols: int | None = None) -> np.ndarray:
    """b ~ U[-1, 1] from default_rng(seed)."""
    cols = n if cols is None else cols
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (n, cols))


def batch_parameters(count: int, seed: int = 3):
    """Config 4 draws: log10 eps ~ U[-3, 0], theta ~ U[0, pi)."""
    rng = np.random.default_rng(seed)
    eps = 10.0 ** rng.uniform(-3.0, 0.0, count)
    theta = rng.uniform(0.0, math.pi, count)
    return eps, theta


def levels_for(n: int, coarsest: int = 3) -> int:
    """Number of levels coarsening n -> n // 2 down to `coarsest`."""
    lv = 1
    while n > coarsest:
        n //= 2
        lv += 1
    return lv


# ---------------------------------------------------------------------------
# reference problem families as StencilField objects (problems.py:45-152): what the
# command-line front end assembles.  Host-side, once per run.

def build_geometry(kind: str, n: int, spacing: float | None = None):
    """problems.py:98-120: GridSpec of a named domain."""
    from .errors import ConfigError
    from .grid import GridSpec
    try:
        mask = geometry_mask(kind, n)
    except ValueError:
        raise ConfigError(f"unknown geometry {kind!r}") from None
    return GridSpec(n, n, 1.0 / (n + 1) if spacing is None else spacing, mask)


def assemble_rotated_laplacian(spec, angle: float, anisotropy: float):
    """problems.py:45-52: one constant table on every point of `spec`."""
    from .errors import ConfigError
    from .grid import constant_stencil
    if anisotropy <= 0.0:
        raise ConfigError(f"anisotropy must be positive, got {anisotropy}")
    a, b, c = rotated_coefficients(angle, anisotropy)
    return constant_stencil(spec, (a * _SXX + c * _SYY - b * _SXY) / (spec.spacing * spec.spacing))


def assemble_variable_diffusion(spec, kappa: float):
    """problems.py:62-95: bilinear elements for -div(g grad u), g = sin(kappa pi x y)
    + 1.1 sampled at the four cell midpoints around each node, scaled by 1 / h^2;
    identity rows at inactive points."""
    from .errors import NumericError
    from .grid import StencilField
    h = spec.spacing
    y = (np.arange(spec.rows, dtype=float)[:, None] + 1.0) * h
    x = (np.arange(spec.cols, dtype=float)[None, :] + 1.0) * h
    g = {(sy, sx): np.sin(kappa * math.pi * (x + 0.5 * sx * h) * (y + 0.5 * sy * h)) + 1.1
         for sy in (-1, 1) for sx in (-1, 1)}
    lo = min(float(q.min()) for q in g.values())
    if lo <= 0.0:
        raise NumericError(f"diffusion coefficient not elliptic, min sample {lo}")
    s = 1.0 / (3.0 * h * h)
    data = np.zeros((spec.rows, spec.cols, 3, 3))
    for (sy, sx), q in g.items():
        data[:, :, 1 + sy, 1 + sx] = -q * s                 # corner neighbours: one cell each
    for sy in (-1, 1):                                       # edge neighbours: two cells each
        data[:, :, 1 + sy, 1] = -(g[(sy, -1)] + g[(sy, 1)]) * 0.5 * s
    for sx in (-1, 1):
        data[:, :, 1, 1 + sx] = -(g[(-1, sx)] + g[(1, sx)]) * 0.5 * s
    data[:, :, 1, 1] = 2.0 * (g[(1, 1)] + g[(1, -1)] + g[(-1, -1)] + g[(-1, 1)]) * s   # ne + nw + sw + se
    data[~spec.mask] = 0.0
    data[~spec.mask, 1, 1] = 1.0
    return StencilField(spec, data)


class ProblemSpec:
    """problems.py:123-146: (family, n, geometry, angle, anisotropy, kappa)."""

    FIELDS = ("family", "n", "geometry", "angle", "anisotropy", "kappa")

    def __init__(self, family: str, n: int, geometry: str = "square", angle: float = 0.0,
                 anisotropy: float = 100.0, kappa: float = 1.0):
        self.family, self.n, self.geometry = family, int(n), geometry
        self.angle, self.anisotropy, self.kappa = float(angle), float(anisotropy), float(kappa)

    def asdict(self) -> dict:
        return {k: getattr(self, k) for k in self.FIELDS}

    def grid(self):
        return build_geometry(self.geometry, self.n)

    def assemble(self, spec=None):
        from .errors import ConfigError
        spec = self.grid() if spec is None else spec
        if self.family == "rotated":
            return assemble_rotated_laplacian(spec, self.angle, self.anisotropy)
        if self.family == "variable":
            return assemble_variable_diffusion(spec, self.kappa)
        raise ConfigError(f"unknown problem family {self.family!r}")
