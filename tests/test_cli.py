"""Command-line front end: `solve` / `bench` on the B200 path
against rows the reference CLI produced (tests/golden/cli_rows.json, written by
make_golden_cli.py from the unmodified reference)."""
import csv
import json
import math
import os

import pytest

from paper_2102_12071_b200 import cli
from paper_2102_12071_b200.errors import ConfigError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = json.load(open(os.path.join(GOLD, "cli_rows.json")))


def _cfg(argv):
    ns = cli.build_parser().parse_args(argv)
    return ns.subcommand, cli.resolve_config(ns.subcommand, ns)


@pytest.mark.parametrize("name", sorted(k for k, c in CASES.items() if c["rows"]))
def test_config_hash_is_the_references(name):
    sub, cfg = _cfg(CASES[name]["argv"])
    assert cli.config_hash(sub, cfg) == CASES[name]["rows"][0]["config_hash"]


def test_extension_options_enter_the_hash_only_off_default():
    sub, base = _cfg(["solve", "--n", "31"])
    _, same = _cfg(["solve", "--n", "31", "--device", "b200", "--gpus", "1", "--sweeps", "1"])
    _, more = _cfg(["solve", "--n", "31", "--sweeps", "2"])
    assert cli.config_hash(sub, base) == cli.config_hash(sub, same) != cli.config_hash(sub, more)


def test_angles_and_config_files(tmp_path, monkeypatch):
    assert cli.parse_angle("pi/6") == math.pi / 6 and cli.parse_angle("5pi/12") == 5 * math.pi / 12
    assert cli.parse_angle("-0.5pi") == -0.5 * math.pi and cli.parse_angle("0.3") == 0.3
    with pytest.raises(ConfigError):
        cli.parse_angle("pi/0")
    sub, cfg = _cfg(["bench", "--ns", "15,31", "--thetas", "pi/6,0.45", "--matched-cost", "true"])
    path = str(tmp_path / "run.cfg")
    cli.write_config_file(sub, cfg, path)
    _, again = _cfg(["bench", "--config", path])
    assert again == cfg
    _, over = _cfg(["bench", "--config", path, "--ns", "63"])      # flags win over the file
    assert over["ns"] == [63] and over["thetas"] == cfg["thetas"]
    monkeypatch.setenv("MGSMOOTH_SEED", "7")
    assert _cfg(["solve"])[1]["seed"] == 7
    (tmp_path / "bad.cfg").write_text("nope = 1\n")
    with pytest.raises(ConfigError):
        _cfg(["solve", "--config", str(tmp_path / "bad.cfg")])


def test_exit_codes_without_running(capsys):
    assert cli.main(["analyze", "--n", "15"]) == 1                # not on the B200 path
    assert "not on the B200 path" in capsys.readouterr().err
    assert cli.main(["train", "--family", "variable", "--n", "15", "--thetas", "0.1,0.2", "--device", "cpu"]) == 1
    assert cli.main(["solve", "--device", "cpu"]) == 1            # no CPU fallback
    assert cli.main(["solve", "--n", "many"]) == 1
    assert cli.main([]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_rows_match_the_reference_cli(name, tmp_path, monkeypatch):
    case = CASES[name]
    monkeypatch.chdir(GOLD)   # model paths are the bare fixture names, as in make_golden_cli.py
    path = str(tmp_path / "out.csv")
    rc = cli.main(case["argv"] + ["--csv", path])
    assert rc == case["exit_code"]
    if case["rows"] is None:
        assert not os.path.exists(path)
        return
    rows = list(csv.DictReader(open(path)))
    assert len(rows) == len(case["rows"])
    for got, want in zip(rows, case["rows"]):
        for col, v in want.items():
            if col == "wall_time":
                assert float(got[col]) > 0.0
            elif col == "rel_residual" and v:
                assert float(got[col]) == pytest.approx(float(v), rel=1e-5)
            else:
                assert got[col] == v, (col, got[col], v)
        assert got["device"] == "b200" and got["gpus"] == "1" and float(got["unknowns_per_s"]) > 0.0
        if "krylov" in want and want["krylov"] == "none":
            assert 0.0 < float(got["roofline_frac"]) < 1.0 and float(got["achieved_GBps"]) > 0.0


@pytest.mark.gpu
def test_sweeps_extension_and_trial_dealing(tmp_path, monkeypatch):
    """--sweeps 2 (V(2,2) through RepeatedSmoother) converges in fewer cycles than V(1,1);
    --gpus beyond the visible devices is a ConfigError (exit 1)."""
    monkeypatch.chdir(GOLD)
    base = ["solve", "--n", "63", "--theta", "pi/6", "--xi", "0.01", "--levels", "5", "--model", "net_conv.json"]
    its = []
    for extra in ([], ["--sweeps", "2"]):
        path = str(tmp_path / f"s{len(its)}.csv")
        assert cli.main(base + extra + ["--csv", path]) == 0
        its.append(int(list(csv.DictReader(open(path)))[0]["iterations"]))
    assert its[1] < its[0]
    assert cli.main(base + ["--gpus", "64"]) == 1


TRAIN_ARGV = ["train", "--n", "15", "--theta", "pi/6", "--xi", "0.01", "--levels", "3", "--epochs", "2", "--samples", "4",
              "--batch-size", "2", "--max-steps", "2"]


def test_train_config_hash_is_the_references():
    sub, cfg = _cfg(TRAIN_ARGV)
    want = json.load(open(os.path.join(GOLD, "stack_model.json")))["metadata"]["config_hash"]
    assert cli.config_hash(sub, cfg) == want


@pytest.mark.gpu
def test_train_reproduces_the_reference_model_file(tmp_path):
    """`train` (adaptive strategy) on the GPU against stack_model.json, the model file the
    reference CLI wrote for the same flags (make_golden_cli.py): same structure and
    metadata, smoother weights to 1e-8; loss.csv and manifest.json are written."""
    import numpy as np
    assert cli.main(TRAIN_ARGV + ["--out", str(tmp_path)]) == 0
    got = json.load(open(tmp_path / "model.json"))
    want = json.load(open(os.path.join(GOLD, "stack_model.json")))
    assert got["kind"] == want["kind"] == "smoother_stack" and got["levels"] == want["levels"]
    assert got["metadata"] == want["metadata"] and got["problem"] == want["problem"]
    for a, b in zip(got["smoothers"], want["smoothers"]):
        assert a["form"] == b["form"] and a["activation"] == b["activation"] and a["gain"] == pytest.approx(b["gain"], rel=1e-13)
        for x, y in zip(a["layers"] + a["skip"], b["layers"] + b["skip"]):
            assert np.allclose(x["data"], y["data"], rtol=0, atol=1e-8 * max(1e-300, np.max(np.abs(y["data"]))))
    rows = list(csv.DictReader(open(tmp_path / "loss.csv")))
    assert len(rows) == 2 * 2 and rows[0]["config_hash"] == want["metadata"]["config_hash"]
    man = json.load(open(tmp_path / "manifest.json"))
    assert man["subcommand"] == "train" and man["parameters"] == want["metadata"]["parameters"]
    # the trained stack deploys through `solve --model`
    assert cli.main(["solve", "--n", "31", "--theta", "pi/6", "--xi", "0.01", "--levels", "4", "--model",
                     str(tmp_path / "model.json"), "--csv", str(tmp_path / "s.csv")]) == 0
