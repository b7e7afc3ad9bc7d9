"""Small solves that drive every cycle kernel family once (for compute-sanitizer):
k_stream / k_stream2 / k_stream3 (forced on every level), k_tile, the single-CTA coarse
kernel, per-point planes, a masked domain, the batched hierarchy (column pairs and the
warp-strip kernel's batched flavour), the padded level-0 path of run_cycles and the padded
quasi-uniform levels below it.  Prints the final relative residuals (must be finite)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2102_12071_b200 as mg
from paper_2102_12071_b200 import device as dv, problems as gen

net = mg.load_model(os.path.join(os.path.dirname(mg.__file__), "data", "net_conv.json"))
n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 255
lv = gen.levels_for(n)


PAD = 4096   # sentinel doubles around the caller's u, f and history buffers


def fenced(shape, fill=None):
    """A contiguous tensor of `shape` carved out of a larger buffer with sentinels on both sides."""
    cnt = int(np.prod(shape))
    big = torch.full((cnt + 2 * PAD,), 1.25e300, dtype=torch.float64, device="cuda")
    view = big[PAD:PAD + cnt].view(*shape)
    if fill is not None:
        view.copy_(torch.as_tensor(fill, dtype=torch.float64))
    else:
        view.zero_()
    return big, view


def fences_intact(big):
    return bool((big[:PAD] == 1.25e300).all() and (big[-PAD:] == 1.25e300).all())


def run(tag, h, f, nu=2, cycles=2):
    bf, fd = fenced(f.shape, f)
    bu, u = fenced(f.shape)
    bh, hist = fenced((h.batch, cycles + 1))
    h.run_cycles(fd, u, cycles, nu, nu, history=hist, u_zero=True)
    torch.cuda.synchronize()
    assert fences_intact(bf) and fences_intact(bu) and fences_intact(bh), f"{tag}: caller buffer overrun"
    hh = hist.cpu().numpy()
    assert np.isfinite(hh).all() and np.isfinite(u.cpu().numpy()).all(), tag
    print(f"{tag:34s} history[-1] = {hh[..., -1].ravel()[:3]}")


A = gen.rotated_fd(n, math.pi / 6, 0.01)
f = gen.uniform_rhs(n, 0)
for kind in (1, 2, 3):
    h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), lv), net)
    h.set_stream_kernel(kind)
    h.set_passes(1, 1, 0)          # every level streamed
    run(f"stream kernel {kind}, all levels", h, f)
    run(f"stream kernel {kind}, V(1,1)", h, f, nu=1)
h = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(n), A), lv), net)
h.set_passes(1 << 40, 1, 0)        # every level tile passes
run("tile passes, all levels", h, f)
h.set_passes(1 << 40, 1, 1023)     # + single-CTA coarse kernel
run("tile + coarse kernel", h, f)
h.set_passes(1 << 40, 0, 0)        # separate kernels
run("separate kernels", h, f)
# auto dispatch at a size where level 0 is the padded warp-strip path (>= 1M points)
if n >= 255:
    m = 1023
    hb = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(m), gen.rotated_fd(m, math.pi / 4, 1e-3)),
                                              gen.levels_for(m)), mg.load_model(os.path.join(os.path.dirname(mg.__file__), "data", "net_conv_c2.json")))
    run("auto, 1023^2 (padded level 0)", hb, gen.uniform_rhs(m, 1), cycles=1)
# per-point planes (GRF 5-point) and a masked domain
Ag = gen.grf_diffusion_5pt(n, seed=2)
hg = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.GridSpec(n, n, 1.0 / n, np.ones((n, n), bool)), Ag), lv), net)
hg.set_passes(1, 1, 0)
run("per-point planes, streamed", hg, gen.uniform_rhs(n, 2))
mask = gen.geometry_mask("lshape", n)
Am = A.copy(); Am[~mask] = 0.0; Am[~mask, 1, 1] = 1.0
hm = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.GridSpec(n, n, 1.0 / (n + 1), mask), Am), lv - 2), net)
hm.set_passes(1, 1, 0)
run("L-shape mask, streamed", hm, f * mask)
hm.set_passes(1 << 40, 1, 0)
run("L-shape mask, tile", hm, f * mask)
# batched hierarchy (config-4 shape)
eps, theta = gen.batch_parameters(3, seed=3)
Ab = np.stack([gen.rotated_fd(n, theta[i], eps[i]) for i in range(3)])
hb = mg.equip_inferred(mg.build_hierarchy_batch(Ab, lv), net)
run("batch of 3, V(1,1)", hb, np.stack([gen.uniform_rhs(n, [4, i]) for i in range(3)]), nu=1)
hb.set_stream_kernel(3)               # the warp-strip kernel's batched flavour on the uniform level 0
hb.set_passes(1, 1, 0)
run("batch of 3, V(1,1), warp strips", hb, np.stack([gen.uniform_rhs(n, [4, i]) for i in range(3)]), nu=1)
# quasi-uniform Galerkin levels wider than one strip: the padded buffers below level 0 (a warp-strip
# parent restricting into / prolonging from them) and the aligned quasi-uniform flavour
if n >= 255:
    m = 2 * n + 1
    hq = mg.equip_inferred(mg.build_hierarchy(mg.StencilField(mg.full_spec(m), gen.rotated_fd(m, math.pi / 5, 0.02)),
                                              gen.levels_for(m)), net)
    hq.set_stream_kernel(3)
    hq.set_passes(1, 1, 0)
    assert hq.level_uniformity(0) == 1 and hq.level_uniformity(1) == 2
    run(f"warp strips, {m}^2, padded levels", hq, gen.uniform_rhs(m, 6))
    run(f"warp strips, {m}^2, V(1,1)", hq, gen.uniform_rhs(m, 7), nu=1, cycles=3)
if "--guard" in sys.argv:
    import ctypes as C
    from paper_2102_12071_b200 import _lib
    na, nc = C.c_int(), C.c_int()
    _lib.call("mgb_guard_check", C.byref(na), C.byref(nc))
    print(f"guard: {na.value} allocations, {nc.value} corrupted", _lib.lib().mgb_last_error().decode() if nc.value else "")
print("sanitize driver done")
