"""Experiment: per-CTA entry / loop start / end (globaltimer) of one warp-strip (k_stream3) PRE /
POST pass of a level (needs a -DMGB_CTA_PROF build of mgb_stream3.cu in MGB_LIB_PATH):
    python scripts/cta_prof3.py c2 LEVEL"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2102_12071_b200 import _lib, device as dv
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
h, f_host, info = bench.build_problem(cfg, 0)
rows, cols = h.level_info(level)[:2]
f = torch.randn(h.batch, rows, cols, dtype=torch.float64, device="cuda")
u = torch.zeros_like(f)
w = h.acquire_work()
ms = C.c_double()
lib = C.CDLL(_lib.LIB_PATH)
for pas in (0, 1):
    for _ in range(3):
        _lib.call("mgb_time_pass", h.handle, w, level, pas, info["nu"], dv.ptr(f), dv.ptr(u), 1, C.byref(ms), dv.stream(f))
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (4 * 8192))()
    lib.mgb_debug_cta_prof3(buf, 8192)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4).astype(np.int64)
    a = a[a[:, 3] > 0]
    np.save(f"gpurun_out/cta_prof3_l{level}_p{pas}.npy", a)
    wid = a[:, 0] >> 16
    a[:, 0] &= 0xFFFF
    t0 = a[:, 1].min()
    st, lp, en = (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3, (a[:, 3] - t0) / 1e3
    pro, loop = lp - st, en - lp
    q = lambda x: f"{x.min():.1f}/{np.median(x):.1f}/{x.max():.1f}"
    print(f"pass {pas} level {level}: {len(a)} CTAs, pass {ms.value * 1e3:.1f} us; entry {q(st)}; prologue {q(pro)}; loop {q(loop)}; end {q(en)}")
    order = np.argsort(-en)[:10]
    print("  last CTAs (id, sm, entry, prologue, loop):", [(int(i), int(a[i, 0]), round(st[i], 1), round(pro[i], 1), round(loop[i], 1)) for i in order])
    sms = np.bincount(a[:, 0].astype(int))
    by_sm = np.array([loop[a[:, 0] == m].mean() for m in range(len(sms)) if sms[m]])
    print("  mean loop time per SM: min/med/max", q(by_sm), " spread inside an SM (max-min), median over SMs:",
          round(float(np.median([np.ptp(loop[a[:, 0] == m]) for m in range(len(sms)) if sms[m]])), 1))
    print("  mean loop by warp slot % 4:", [round(float(loop[wid % 4 == k].mean()), 1) for k in range(4)],
          " warps per (SM, slot % 4) histogram:", np.bincount(np.bincount((a[:, 0] * 4 + wid % 4).astype(int))).tolist())
    print("  CTAs per SM histogram:", np.bincount(sms).tolist())
