"""Algorithmic-byte models of one V(nu1, nu2) cycle and the HBM peak
they are reported against.  Shared by bench.py and the command-line front end."""

from __future__ import annotations

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md's stated figure when MEASURED_PEAKS.json is absent


def level_sizes(rows: int, cols: int, levels: int):
    out = []
    for _ in range(levels):
        out.append(rows * cols)
        rows //= 2
        cols //= 2
    return out


def cycle_bytes(rows: int, cols: int, levels: int, nu1: int, nu2: int, compact: bool) -> float:
    """Bytes one cycle must move.  Per-point model (the reference data model: 72 B/pt
    operator and smoother tables): sweep 168 B, first pre-sweep on a coarse level 88 B,
    residual + restriction 88 B, prolongation 16 B per fine point, 8 B per coarse point
    written / read.  Compact model (kernels that read no per-point tables): sweep 24 B,
    first coarse pre-sweep 16 B, residual 16 B, prolongation 16 B."""
    sz = level_sizes(rows, cols, levels)
    sweep, first_cut, rest = (24, 8, 32) if compact else (168, 80, 104)
    tot = 0.0
    for l in range(levels - 1):
        tot += sz[l] * (sweep * (nu1 + nu2) - first_cut * (l >= 1) + rest) + 16 * sz[l + 1]
    return tot + 16 * sz[-1]


def hbm_peak_gbs():
    """(GB/s, 'measured' | 'fallback')."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"
