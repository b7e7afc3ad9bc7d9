"""One config-2 step (10 V(2,2) cycles + history) bracketed by cudaProfilerStart/Stop,
for `ncu --profile-from-start off` launch lists and single-kernel captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
h, f_host, info = bench.build_problem(cfg, 0)
if os.environ.get("MGB_KIND"):   # streaming kernel kind (0 auto, 1, 2, 3)
    h.set_stream_kernel(int(os.environ["MGB_KIND"]))
f = torch.from_numpy(f_host).cuda()
u = torch.zeros_like(f)
for _ in range(2):
    h.run_cycles(f, u, info["cycles"], info["nu"], info["nu"], u_zero=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
hist = h.run_cycles(f, u, info["cycles"], info["nu"], info["nu"], u_zero=True)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("history", hist.cpu().numpy()[0].tolist(), "launches", h.last_launches)
