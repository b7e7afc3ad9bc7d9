"""Domain decomposition beyond band-class levels and beyond one process:
per-point planes and masks, the overlapped interior / edge schedule, and the rank-local
schedule run by two processes that exchange through the host (gloo) on one GPU.  The
decomposed u must equal the single-domain u bitwise; histories differ only in the
summation order of the norms."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from dd_problems import build

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
pytestmark = pytest.mark.gpu


def _single(h, f_full, nu, cycles):
    from paper_2102_12071_b200 import device as dv
    f = dv.to_dev(f_full)
    u = dv.zeros(f.shape)
    hist = dv.host(h.run_cycles(f, u, cycles, nu, nu, u_zero=True))[0]
    return dv.host(u), hist


@pytest.mark.parametrize("name,nparts", [("grf1023", 3), ("lshape511", 2), ("c2_1023", 4), ("classed511", 2)])
@pytest.mark.parametrize("overlap", [True, False])
def test_virtual_parts_match_single_domain(name, nparts, overlap, monkeypatch):
    from paper_2102_12071_b200 import dd, device as dv
    monkeypatch.setenv("MGB_STREAM_MIN", "0")   # the single domain streams every level too
    h, f_full, nu, cycles, agg = build(name)
    u_ref, hist_ref = _single(h, f_full, nu, cycles)
    s = dd.DecomposedSolver(h, nparts, local=True, agglomerate_rows=agg)
    s.set_option("overlap", overlap)
    for p in range(nparts):
        r0, r1 = s.rows(p)
        s.set_rhs(p, dv.to_dev(np.ascontiguousarray(f_full[r0:r1])))
    hist = dv.host(s.run_cycles(cycles, nu, nu))
    u = np.concatenate([dv.host(s.solution(p)) for p in range(nparts)])
    assert np.array_equal(u, u_ref), float(np.abs(u - u_ref).max())
    assert np.allclose(hist, hist_ref, rtol=1e-12, atol=0)
    sent, steps = s.stats()
    assert sent > 0 and steps > 0


def test_skipping_exchanges_changes_the_result(monkeypatch):
    """The 'exchange' option really removes the halos (it exists for timing only)."""
    from paper_2102_12071_b200 import dd, device as dv
    monkeypatch.setenv("MGB_STREAM_MIN", "0")
    h, f_full, nu, cycles, agg = build("classed511")
    u_ref, _ = _single(h, f_full, nu, cycles)
    s = dd.DecomposedSolver(h, 2, local=True, agglomerate_rows=agg)
    s.set_option("exchange", False)
    for p in range(2):
        r0, r1 = s.rows(p)
        s.set_rhs(p, dv.to_dev(np.ascontiguousarray(f_full[r0:r1])))
    s.run_cycles(cycles, nu, nu)
    u = np.concatenate([dv.host(s.solution(p)) for p in range(2)])
    assert not np.array_equal(u, u_ref)


@pytest.mark.parametrize("name", ["classed511", "grf1023"])
def test_two_processes_rank_local_schedule(name, tmp_path, monkeypatch):
    """Two processes, one part each (nlocal = 1: the code path a multi-GPU run takes),
    exchanging halos, the agglomeration all-gather and the norm all-reduce through the
    host-staged gloo callback; both share cuda:0."""
    monkeypatch.setenv("MGB_STREAM_MIN", "0")
    h, f_full, nu, cycles, agg = build(name)
    u_ref, hist_ref = _single(h, f_full, nu, cycles)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, MGB_STREAM_MIN="0", OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "dd_worker.py"), str(tmp_path), name],
                       capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    parts = [np.load(tmp_path / f"rank{q}.npz") for q in range(2)]
    assert parts[0]["rows"][1] == parts[1]["rows"][0] and parts[1]["rows"][1] == f_full.shape[0]
    u = np.concatenate([p["u"] for p in parts])
    assert np.array_equal(u, u_ref), float(np.abs(u - u_ref).max())
    for p in parts:
        assert np.allclose(p["hist"], hist_ref, rtol=1e-12, atol=0)
        assert int(p["sent"]) > 0 and int(p["steps"]) > 0
    assert np.array_equal(parts[0]["hist"], parts[1]["hist"])   # every rank holds the same history


def test_bench_multi_rank_path_runs(tmp_path):
    """bench.py --gpus 2 (the default config: c2 decomposed over the ranks) end to end with
    two processes on this one GPU: gloo control plane, host-staged exchanges.  Checks
    the JSON line's contract and that the decomposed history equals the single-GPU one;
    the numbers themselves are not measurements."""
    import json
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, MGB_BENCH_BACKEND="gloo", OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "1", "--warmup", "1", "--no-cpu"],
                       capture_output=True, text=True, env=env, timeout=1500, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["workload"].startswith("c2:")
    assert d["dd"]["sent_bytes_per_step_rank0"] > 0 and d["dd"]["exchange_steps_per_step"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * 4095 * 4095
    # the c2 history after 10 V(2,2) cycles (bench_c2_full.npz pins 3 cycles; the N = 1 bench line prints this value)
    assert abs(d["history_last"] - 0.09833263200964358) < 1e-12
