"""The reference arm of bench.py (--impl reference): the CPU oracle port on all host
cores, one JSON line with the contract's keys.  Small sample grid so it runs on CPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _run(args, n):
    env = dict(os.environ, MGB_CPU_SAMPLE_N=str(n))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                       capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_arm_line_uses_all_cores():
    d = _run(["--steps", "2", "--warmup", "1"], 63)
    assert d["impl"] == "reference"
    assert d["metric"] == "unknowns/sec per V-cycle (fp64)" and d["unit"] == "unknowns/s"
    assert d["higher_is_better"] is True and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] == d["value"]
    assert cb["cores"] == max(1, min(os.cpu_count() or 1, 32))
    assert d["e2e"] == {"value": d["value"], "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("c2:") and d["config"]["sample_n"] == 63


def test_reference_arm_other_ranks_exit_without_work():
    env = dict(os.environ, MGB_CPU_SAMPLE_N="63", RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                       capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


def test_full_size_oracle_hierarchy_equals_the_direct_build():
    """bench.oracle_hierarchy_constant (the same-size reference arm's setup shortcut for
    constant-coefficient configs) reproduces the oracle's own build: operators and the
    coarsest LU bit for bit, kernels to one ulp, hence the same V(2,2) history."""
    import math
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    from oracle import mg_oracle as mo
    from paper_2102_12071_b200 import problems as gen
    net = mo.load_net_json(os.path.join(ROOT, "paper_2102_12071_b200", "data", "net_conv_c2.json"))
    n, lv = 255, 7
    A = gen.rotated_fd(n, math.pi / 4, 1e-3)
    h1 = mo.equip_inferred(mo.build_hierarchy(A, lv), net)
    h2 = bench.oracle_hierarchy_constant(A[0, 0], n, lv, net)
    assert all(np.array_equal(a, b) for a, b in zip(h1.ops, h2.ops))
    assert np.array_equal(h1.lu, h2.lu) and np.array_equal(h1.perm, h2.perm)
    for a, b in zip(h1.kernels, h2.kernels):
        assert np.max(np.abs(a - b)) <= 4 * np.finfo(float).eps * np.max(np.abs(a))
    f = gen.uniform_rhs(n, 1)
    _, q1 = mo.run_cycles(h1, f, 3, 2, 2)
    _, q2 = mo.run_cycles(h2, f, 3, 2, 2)
    assert np.allclose(q1, q2, rtol=1e-12, atol=0)
