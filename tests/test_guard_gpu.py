"""Bounds checks without compute-sanitizer (closed on this GPU pool): the kernel-family
driver scripts/sanitize.py runs with MGB_GUARD=1, which puts 4 KiB canaries around every
device allocation of the library, and with sentinels around the caller's u / f / history
buffers; no canary may change.  (Races are covered by the bitwise-reproducibility tests:
test_config2_properties_full_size, the stream == tile == DD bitwise comparisons.)"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [127, 255])
def test_no_write_outside_any_allocation(n):
    env = dict(os.environ, MGB_GUARD="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize.py"), str(n), "--guard"],
                       capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("guard:")]
    assert line and " 0 corrupted" in line[0] and int(line[0].split()[1]) > 20, r.stdout[-1500:]
