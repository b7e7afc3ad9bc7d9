"""Domain-decomposed V-cycles over several GPUs (or virtual parts on one GPU).

The fine levels of a band-class hierarchy (`build_hierarchy_classed`) are split
into row blocks; each streaming pass runs on a block with 6 ghost rows per edge
after a halo exchange; levels with at most `agglomerate_rows` rows are solved
redundantly on every part after an all-gather of the restricted residual.  With
one process per GPU the exchanges are NCCL operations captured in the solve's
CUDA graph; `nparts > 1` with `local=True` keeps all parts on this GPU (device
copies) — the single-GPU test of the decomposition.  SURVEY §8(e)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, device as dv


class DecomposedSolver:
    def __init__(self, hier, nparts: int, first_part: int = 0, local: bool = True, nccl_id: bytes | None = None,
                 agglomerate_rows: int = 1023):
        self.hier = hier
        self.nparts = nparts
        self.first = first_part
        self.nlocal = nparts if local else 1
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        d = C.c_void_p()
        _lib.call("mgb_dd_create", hier.handle, nparts, first_part, self.nlocal,
                  None if idbuf is None else C.cast(idbuf, C.c_void_p), int(agglomerate_rows), C.byref(d))
        self._d = d

    def __del__(self):
        try:
            if self._d:
                _lib.lib().mgb_dd_destroy(self._d)
        except Exception:
            pass
        self._d = None

    @property
    def local_parts(self):
        return list(range(self.first, self.first + self.nlocal))

    def rows(self, part: int):
        """Level-0 rows [r0, r1) owned by `part`."""
        r0, r1, nl = C.c_int(), C.c_int(), C.c_int()
        _lib.call("mgb_dd_info", self._d, part, C.byref(r0), C.byref(r1), C.byref(nl))
        return r0.value, r1.value

    @property
    def distributed_levels(self) -> int:
        r0, r1, nl = C.c_int(), C.c_int(), C.c_int()
        _lib.call("mgb_dd_info", self._d, self.first, C.byref(r0), C.byref(r1), C.byref(nl))
        return nl.value

    def set_rhs(self, part: int, f_block):
        """f_block: CUDA tensor of the part's owned rows (r1 - r0, cols)."""
        _lib.call("mgb_dd_set_rhs", self._d, part, dv.ptr(f_block), dv.stream(f_block))

    def solution(self, part: int, out=None):
        r0, r1 = self.rows(part)
        cols = self.hier.levels[0].spec.cols
        if out is None:
            out = dv.empty((r1 - r0, cols))
        _lib.call("mgb_dd_get_solution", self._d, part, dv.ptr(out), dv.stream(out))
        return out

    def run_cycles(self, cycles: int, nu1: int = 2, nu2: int = 2, u_zero: bool = True, history=None):
        t = dv.torch()
        if history is None:
            history = t.empty(cycles + 1, dtype=t.float64, device=dv.require_cuda(self.hier.device))
        _lib.call("mgb_dd_run_cycles", self._d, int(nu1), int(nu2), int(cycles), 1 if u_zero else 0,
                  dv.ptr(history), dv.stream(history))
        return history


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _lib.call("mgb_dd_nccl_unique_id", C.cast(buf, C.c_void_p))
    return buf.raw


def from_process_group(hier, agglomerate_rows: int = 1023) -> DecomposedSolver:
    """One part per torch.distributed rank (NCCL exchanges); rank 0's NCCL id is
    broadcast with the process group."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return DecomposedSolver(hier, world, rank, local=False, nccl_id=obj[0], agglomerate_rows=agglomerate_rows)


def partition_rows(rows: int, nparts: int, dist_levels: int):
    """Level-0 row blocks as the C++ driver cuts them: equal blocks rounded up to a
    multiple of 2^dist_levels (so every distributed level's block starts at an even
    row and coarse anchors 2c+1 never straddle parts); the last part takes the rest."""
    align = 1 << dist_levels
    blk = -(-rows // nparts)
    blk = -(-blk // align) * align
    return [(min(p * blk, rows), min((p + 1) * blk, rows) if p < nparts - 1 else rows) for p in range(nparts)]
