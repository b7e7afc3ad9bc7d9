"""Experiment: per-CTA start/end (globaltimer) of one level-0 PRE / POST pass (needs a
-DMGB_CTA_PROF build in MGB_LIB_PATH)."""
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
    buf = (C.c_ulonglong * (3 * 8192))()
    lib.mgb_debug_cta_prof(buf, 8192)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 3).astype(np.int64)
    a = a[a[:, 2] > 0]
    t0 = a[:, 1].min()
    st, en = (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
    dur = en - st
    print(f"pass {pas} level {level}: {len(a)} CTAs, ms {ms.value:.3f}; start max {st.max():.1f} us; end min/med/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f}; dur min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f}")
    order = np.argsort(-dur)[:12]
    print("  slowest CTAs (id, sm, start, dur):", [(int(i), int(a[i, 0]), round(st[i], 1), round(dur[i], 1)) for i in order])
    # per-SM concurrency: CTAs per SM
    sms = np.bincount(a[:, 0].astype(int))
    print("  CTAs per SM histogram:", np.bincount(sms).tolist())
    np.save(f"gpurun_out/cta_prof_l{level}_p{pas}.npy", a)
