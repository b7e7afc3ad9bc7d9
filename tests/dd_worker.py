"""One rank of the two-process decomposition test (launched by test_dd_gpu.py under
torch.distributed.run with the gloo backend; both ranks use cuda:0).  Solves the
problem named on the command line through the rank-local schedule of mgb_dd with the
host-staged exchange callback and writes this rank's rows of u and the history."""
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import paper_2102_12071_b200 as mg                                    # noqa: E402
from paper_2102_12071_b200 import dd, device as dv, problems as gen   # noqa: E402
from dd_problems import build                                         # noqa: E402

out_dir, name = sys.argv[1], sys.argv[2]
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
h, f_full, nu, cycles, agg = build(name)
s = dd.from_process_group(h, agglomerate_rows=agg, backend="host")
r0, r1 = s.rows(rank)
s.set_rhs(rank, dv.to_dev(np.ascontiguousarray(f_full[r0:r1])))
hist = s.run_cycles(cycles, nu, nu)
torch.cuda.synchronize()
sent, steps = s.stats()
np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=dv.host(s.solution(rank)), hist=dv.host(hist), rows=np.array([r0, r1]),
         sent=sent, steps=steps, dist_levels=s.distributed_levels)
dist.barrier()
dist.destroy_process_group()
