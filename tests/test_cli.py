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
    assert cli.main(["train", "--n", "15"]) == 1                  # not on the B200 path
    assert "not on the B200 path" in capsys.readouterr().err
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
