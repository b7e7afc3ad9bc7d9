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
