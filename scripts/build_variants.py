"""Experiment builds of libmgb.so that differ in one source's -D defines:
    python scripts/build_variants.py SOURCE.cu name1:-DA=1,-DB=2 name2:-DC=3 ...
Objects of the other sources are compiled once into experiments/obj/; each variant
recompiles SOURCE.cu and links experiments/libmgb_<name>.so (use with MGB_LIB_PATH)."""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12071_b200 import build as B
src, variants = sys.argv[1], [v.split(":", 1) for v in sys.argv[2:]]
obj_dir = os.path.join(B.ROOT, "experiments", "obj")
os.makedirs(obj_dir, exist_ok=True)
nvcc = B.nvcc_path()
def cc(s, out, defs=()):
    r = subprocess.run([nvcc, *B.flags(), *defs, "-Xptxas", "-v", "-c", os.path.join(B.CSRC, s), "-o", out],
                       capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return r.stderr
# sources that are compiled with the variant's defines: mgb_stream3b.cu is mgb_stream3.cu's second half
group = ["mgb_stream3.cu", "mgb_stream3b.cu"] if src == "mgb_stream3.cu" else [src]
others = [s for s in B.SOURCES if s not in group]
def base(s):
    o = os.path.join(obj_dir, s.replace(".cu", ".o"))
    if not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(os.path.join(B.CSRC, f)) for f in os.listdir(B.CSRC)):
        cc(s, o)
    return o
with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(base, others))
def variant(v):
    name, defs = v
    vobjs, log = [], ""
    for g in group:
        o = os.path.join(obj_dir, f"{g[:-3]}_{name}.o")
        log += cc(g, o, [d for d in defs.split(",") if d])
        vobjs.append(o)
    lib = os.path.join(B.ROOT, "experiments", f"libmgb_{name}.so")
    r = subprocess.run([nvcc, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, *vobjs, "-ldl"], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    regs = [l for l in log.splitlines() if "registers" in l]
    return name, lib, log
with ThreadPoolExecutor(8) as ex:
    for name, lib, log in ex.map(variant, variants):
        open(os.path.join(obj_dir, f"{name}.ptxas.log"), "w").write(log)
        print(name, lib)
