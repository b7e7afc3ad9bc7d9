"""Domain-decomposed V-cycles over several GPUs (or virtual parts on one GPU).

The fine levels of a hierarchy (band-class tables or per-point planes, masks
allowed; `build_hierarchy` / `build_hierarchy_classed`) are split into row blocks;
each streaming pass runs on a block with 6 ghost rows per edge, its interior rows
overlapping the halo exchange; levels with at most `agglomerate_rows` rows are
solved redundantly on every part after an all-gather of the restricted residual.
Exchange backends: NCCL operations captured in the solve's CUDA graph (one process
per GPU); device copies with all parts on this GPU (`local=True`, the single-GPU
test of the decomposition); a host callback per exchange (`set_exchange`, e.g.
`gloo_exchange`: host-staged torch.distributed transfers between processes that
may share one GPU — the test of the rank-local schedule).  SURVEY §8(e)."""

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
        self._xfn = None   # keeps the ctypes callback alive

    def set_exchange(self, fn):
        """Callback backend: fn(op, peer, send_ptr, recv_ptr, count) -> None is called for
        every exchange of the rank-local schedule (see mgb_dd_set_exchange; device
        pointers as ints); the cycles then run eagerly."""
        proto = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int64)

        def tramp(_ctx, op, peer, send, recv, count):
            try:
                fn(int(op), int(peer), send, recv, int(count))
                return 0
            except Exception as exc:   # surfaces as MGB_NCCL -> RuntimeError
                import traceback
                traceback.print_exc()
                self._xerr = exc
                return 1

        self._xfn = proto(tramp)
        _lib.call("mgb_dd_set_exchange", self._d, C.cast(self._xfn, C.c_void_p), None)

    def set_option(self, key: str, value: bool):
        """'overlap' (interior rows overlap the halo exchange, default on) or 'exchange'
        (off: skip all exchanges — timing of the exposed exchange cost only)."""
        _lib.call("mgb_dd_set_option", self._d, key.encode(), 1 if value else 0)

    def stats(self):
        """(bytes this process sent, exchange steps) of the last enqueued run."""
        b, n = C.c_int64(), C.c_int()
        _lib.call("mgb_dd_stats", self._d, C.byref(b), C.byref(n))
        return b.value, n.value

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


class _DevSpan:
    """Zero-copy torch view of `count` doubles at a raw device pointer."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (int(ptr), False), "version": 2}


def gloo_exchange(device: int, group=None):
    """Exchange callback over torch.distributed with host staging (works with the gloo
    backend, so the ranks may share one GPU): halos by isend / irecv pairs, the
    agglomeration by all_gather, the history sums by all_reduce."""
    import torch
    import torch.distributed as dist

    def view(ptr, count):
        return torch.as_tensor(_DevSpan(ptr, count), device=torch.device("cuda", device))

    def fn(op, peer, send, recv, count):
        if op == 0:
            out = view(send, count).cpu()
            inc = torch.empty(count, dtype=torch.float64)
            reqs = [dist.isend(out, peer, group=group), dist.irecv(inc, peer, group=group)]
            for r in reqs:
                r.wait()
            view(recv, count).copy_(inc)
        elif op == 1:
            world = dist.get_world_size(group)
            outs = [torch.empty(count, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(outs, view(send, count).cpu(), group=group)
            view(recv, count * world).copy_(torch.cat(outs))
        elif op == 2:
            h = view(recv, count).cpu()
            dist.all_reduce(h, group=group)
            view(recv, count).copy_(h)
        else:
            raise ValueError(f"unknown exchange op {op}")
        torch.cuda.synchronize(device)

    return fn


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _lib.call("mgb_dd_nccl_unique_id", C.cast(buf, C.c_void_p))
    return buf.raw


def from_process_group(hier, agglomerate_rows: int = 1023, backend: str = "nccl") -> DecomposedSolver:
    """One part per torch.distributed rank.  backend "nccl": NCCL exchanges (rank 0's
    NCCL id is broadcast with the process group); "host": gloo_exchange callbacks."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    if backend == "host":
        s = DecomposedSolver(hier, world, rank, local=False, nccl_id=None, agglomerate_rows=agglomerate_rows)
        s.set_exchange(gloo_exchange(hier.device))
        return s
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
