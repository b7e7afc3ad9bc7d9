"""Device time of a V-cycle started at each level (CUDA graph of mgb_vcycle), so
differences give the per-level cost of the config-2 cycle."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2102_12071_b200 import _lib, device as dv
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
h, f_host, info = bench.build_problem(cfg, 0)
if len(sys.argv) > 2:  # streaming kernel: 0 auto, 1 one column, 2 column pairs
    h.set_stream_kernel(int(sys.argv[2]))
if len(sys.argv) > 3:  # stream_min (points): levels below run tile passes (-1 keeps)
    h.set_passes(int(sys.argv[3]))
if len(sys.argv) > 5:  # tile: 1 tile-local fused passes below stream_min, 0 separate kernels
    h.set_passes(-1, int(sys.argv[5]), -1)
if len(sys.argv) > 4:  # coarse_max (points): levels up to this run in the single-CTA coarse kernel
    h.set_passes(-1, -1, int(sys.argv[4]))
nu = info["nu"]
w = h.acquire_work()
res = []
for l in range(h.depth - 1):
    rows, cols = h.level_info(l)[:2]
    f = torch.randn(h.batch, rows, cols, dtype=torch.float64, device="cuda")
    u = torch.zeros_like(f)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        _lib.call("mgb_vcycle", h.handle, w, l, dv.ptr(f), dv.ptr(u), nu, nu, C.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        _lib.call("mgb_vcycle", h.handle, w, l, dv.ptr(f), dv.ptr(u), nu, nu, C.c_void_p(s.cuda_stream))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res.append((l, rows, e0.elapsed_time(e1) / 20 * 1e3))
for i, (l, rows, us) in enumerate(res):
    nxt = res[i + 1][2] if i + 1 < len(res) else 0.0
    print(f"level {l:2d} {rows:5d}^2  cycle-from-here {us:9.1f} us   this level {us - nxt:8.1f} us")
