"""Where the end-to-end (host-buffer) time goes: pipelined solves for several stream
lengths (slope = steady-state cost per solve), and the raw copy bandwidth."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2102_12071_b200 import device as dv
h, f_host, info = bench.build_problem("c2", 0)
cyc, nu = info["cycles"], info["nu"]
f_pin = [torch.from_numpy(np.ascontiguousarray(f_host[0])).pin_memory() for _ in range(2)]
u_pin = [torch.zeros_like(f_pin[0]).pin_memory() for _ in range(2)]
fh, uh = [x.numpy() for x in f_pin], [x.numpy() for x in u_pin]
s = torch.cuda.current_stream()
def run(count):
    hist = [np.empty((1, cyc + 1)) for _ in range(count)]
    fl = [fh[k % 2] for k in range(count)]; ul = [uh[k % 2] for k in range(count)]
    h.run_cycles_host_many(fl, ul, cyc, nu, nu, history_hosts=hist, u_zero=True, stream=s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); h.run_cycles_host_many(fl, ul, cyc, nu, nu, history_hosts=hist, u_zero=True, stream=s.cuda_stream)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for c in (2, 5, 10, 20):
    print(f"count {c:3d}: {run(c):8.2f} ms, {run(c) / c:6.3f} ms per solve")
d = torch.empty(f_pin[0].shape, dtype=torch.float64, device="cuda")
d2 = torch.empty_like(d)
for name, fn in (("H2D", lambda: d.copy_(f_pin[0], non_blocking=True)),
                 ("D2H", lambda: u_pin[0].copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(5)]; e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {ms:.3f} ms for {d.numel() * 8 / 1e6:.0f} MB = {d.numel() * 8 / ms / 1e6:.1f} GB/s")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(sa): d.copy_(f_pin[0], non_blocking=True)
    with torch.cuda.stream(sb): u_pin[1].copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D+D2H concurrent: {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms per pair")
