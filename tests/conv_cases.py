"""Reference shared-kernel conv smoother fixtures (tests/golden/conv.npz, made by
make_golden.py from the unmodified reference)."""
import os

import numpy as np

from conftest import GOLDEN

_Z = None


def conv_golden():
    global _Z
    if _Z is None:
        _Z = np.load(os.path.join(GOLDEN, "conv.npz"), allow_pickle=False)
    return _Z


def params(prefix):
    """(form, layers (n, 3, 3), skip (3, 3) or None, activation, slope, gain)."""
    z = conv_golden()
    skip = z[f"{prefix}/skip"]
    return (str(z[f"{prefix}/form"]), z[f"{prefix}/layers"], None if skip.shape[0] == 0 else skip,
            str(z[f"{prefix}/activation"]), float(z[f"{prefix}/slope"]), float(z[f"{prefix}/gain"]))


def names(section):
    z = conv_golden()
    return sorted({"/".join(k.split("/")[1:3]) if section == "apply" else k.split("/")[1]
                   for k in z.files if k.startswith(section + "/")})
