"""World-size-2 gloo tests of the multi-process host logic (CPU only): problem
sharding, max-over-ranks timing and history gathering used by bench.py under
torchrun, plus the oracle solving each rank's shard of a config-4-style batch."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2102_12071_b200 import dist as D


def test_shard_covers_every_problem_once():
    for count in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = D.shard(count, r, world)
                assert 0 <= lo <= hi <= count
                seen.extend(range(lo, hi))
            assert seen == list(range(count))
            sizes = [D.shard(count, r, world)[1] - D.shard(count, r, world)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    D.init("gloo")
    try:
        t = D.max_over_ranks(1.0 + rank)
        s = D.sum_over_ranks(10.0 * (rank + 1))
        # each rank solves its shard of a small batch with the oracle (stand-in for the GPU arm)
        import math
        from oracle import mg_oracle as mo
        from paper_2102_12071_b200 import problems as gen
        count, n = 5, 15
        eps, theta = gen.batch_parameters(count, seed=3)
        lo, hi = D.shard(count, rank, world)
        rows = []
        for i in range(lo, hi):
            h = mo.equip_jacobi(mo.build_hierarchy(gen.rotated_fd(n, theta[i], eps[i]), 3))
            _, hist = mo.run_cycles(h, gen.uniform_rhs(n, [4, i]), 3, 1, 1)
            rows.append(hist)
        g = D.gather_rows(np.array(rows).reshape(hi - lo, 4), count)
        q.put((rank, t, s, None if g is None else g.tolist()))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_gloo_world2_collectives_and_sharded_batch():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    out = [q.get(timeout=240) for _ in range(world)]
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    out.sort()
    assert out[0][1] == out[1][1] == 2.0           # max over ranks
    assert out[0][2] == out[1][2] == 30.0          # sum over ranks
    gathered = np.array(out[0][3])
    assert out[1][3] is None and gathered.shape == (5, 4)
    # the gathered histories equal a single-process solve of the whole batch
    from oracle import mg_oracle as mo
    from paper_2102_12071_b200 import problems as gen
    eps, theta = gen.batch_parameters(5, seed=3)
    for i in range(5):
        h = mo.equip_jacobi(mo.build_hierarchy(gen.rotated_fd(15, theta[i], eps[i]), 3))
        _, hist = mo.run_cycles(h, gen.uniform_rhs(15, [4, i]), 3, 1, 1)
        assert np.array_equal(gathered[i], hist)


def _halo_worker(rank, world, port, q):
    """The ghost-row exchange pattern of mgb_dd.cu (6 rows per block edge, blocks
    from dd.partition_rows) with torch.distributed send/recv on CPU tensors."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist
    from paper_2102_12071_b200 import dd
    D.init("gloo")
    try:
        G = 6
        rows, cols, dl = 200, 7, 2
        blocks = dd.partition_rows(rows, world, dl)
        r0, r1 = blocks[rank]
        glob = torch.arange(rows * cols, dtype=torch.float64).reshape(rows, cols)
        blk = torch.full((r1 - r0 + 2 * G, cols), -1.0, dtype=torch.float64)
        blk[G:G + r1 - r0] = glob[r0:r1]
        ops = []
        if rank > 0:
            ops += [dist.P2POp(dist.isend, blk[G:2 * G].contiguous(), rank - 1),
                    dist.P2POp(dist.irecv, blk[:G], rank - 1)]
        if rank + 1 < world:
            nb = min(G, rows - r1)
            send = blk[G + r1 - r0 - nb:G + r1 - r0].contiguous()
            ops += [dist.P2POp(dist.isend, send, rank + 1), dist.P2POp(dist.irecv, blk[G + r1 - r0:G + r1 - r0 + nb], rank + 1)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        lo, hi = max(0, r0 - G), min(rows, r1 + G)
        ok = bool(torch.equal(blk[lo - (r0 - G):hi - (r0 - G)], glob[lo:hi]))
        aligned = all(b[0] % (1 << dl) == 0 for b in blocks)
        q.put((rank, ok, aligned, blocks))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_gloo_world2_halo_exchange_pattern():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    out = sorted(q.get(timeout=240) for _ in range(world))
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok, aligned, blocks in out:
        assert ok and aligned
        assert blocks[0][0] == 0 and blocks[-1][1] == 200
        assert all(blocks[i][1] == blocks[i + 1][0] for i in range(len(blocks) - 1))
