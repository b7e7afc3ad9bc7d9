"""Time one config-2 step (10 V(2,2) cycles + history) for each pass structure."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
h, f_host, info = bench.build_problem(cfg, 0)
f = torch.from_numpy(f_host).cuda()
u = torch.zeros_like(f)
for mode in [int(m) for m in os.environ.get("MODES", "2,1,0").split(",")]:
    h.set_fused(mode)
    for _ in range(3):
        hist = h.run_cycles(f, u, info["cycles"], info["nu"], info["nu"], u_zero=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        hist = h.run_cycles(f, u, info["cycles"], info["nu"], info["nu"], u_zero=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"mode {mode}: {ms:.3f} ms/step  {info['n']**2 * info['cycles'] / ms / 1e6:.3e} unknowns/s  "
          f"launches {h.last_launches}  last {hist[0, -1].item():.6e}", flush=True)
