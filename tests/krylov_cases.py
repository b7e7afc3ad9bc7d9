"""Reference Krylov fixtures (tests/golden/krylov.npz, made by make_golden.py from
the unmodified reference's krylov.py)."""
import os

import numpy as np

from conftest import GOLDEN

_Z = None


def krylov_golden():
    global _Z
    if _Z is None:
        _Z = np.load(os.path.join(GOLDEN, "krylov.npz"), allow_pickle=False)
    return _Z


def krylov_names():
    return sorted({k.split("/")[0] for k in krylov_golden().files})


def krylov_case(name):
    z = krylov_golden()
    meta = z[f"{name}/meta"]
    return {
        "A": z[f"{name}/A"], "mask": z[f"{name}/mask"], "f": z[f"{name}/f"], "u": z[f"{name}/u"],
        "history": z[f"{name}/history"], "nu": int(meta[0]), "method": "fgmres" if meta[1] == 0 else "gmres",
        "tol": float(meta[2]), "max_iter": int(meta[3]), "restart": int(meta[4]) or None,
        "iterations": int(meta[5]), "converged": bool(meta[6]), "smoother": str(z[f"{name}/smoother"]),
    }
