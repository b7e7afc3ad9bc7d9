"""`solve` and `bench` on the B200 path: the reference front end's run core
(cli.py:389-487 `_equip` / `_make_rhs` / `_solve_once` / `_solve_rows`, :605-617
`cmd_solve`, :709-766 `cmd_bench`) driven through the device hierarchy.

    python -m paper_2102_12071_b200.cli solve --n 1023 --levels 9 --theta pi/4 \
        --xi 1e-3 --model net.json --device b200 [--gpus 2 --trials 8]

Same flags, config files (flat key = value, flags win, MGSMOOTH_SEED overrides the
seed), exit codes and CSV rows as the reference.  `config_hash` is the reference's:
a run the reference can also do carries the same hash, so its rows line up with CPU
rows (the extension options below enter the hash only when they leave their defaults).

Extensions: `--device b200` (the only device: there is no CPU fallback), `--gpus N`
(trials of `solve` / cells of `bench` are dealt round-robin to N visible GPUs, one
hierarchy per GPU), `--sweeps NU` (V(NU, NU) through RepeatedSmoother, cli.py:365-377)
and `--precision 64|32` (CNN inference arithmetic).  Every CSV row gains `device`,
`gpus`, `unknowns_per_s` (active unknowns x iterations / wall_time),
`achieved_GBps` (x SURVEY 8(d)'s bytes per cycle: the per-point model, or the compact
one when level 0 holds band-class tables) and `roofline_frac` (of the HBM peak in
MEASURED_PEAKS.json, else the profiling recipe's fallback).

`train` (cli.py:489-587) runs the GPU trainers of training.py: `--variant conv|fc` the
staged kernel-inference-net training, else the adaptive / independent conv-smoother
strategies; it writes model.json, loss.csv and manifest.json as the reference does
(including the `--thetas` mixture and `--inject-k` retraining).  `analyze` is out of
scope: it exits 1 with the reference's UnsupportedOperationError message format.
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import json
import math
import os
import re
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import roofline
from .errors import (ConfigError, ContractError, NonConvergedError, NumericError, SingularMatrixError,
                     TrainingError, UnsupportedOperationError)

# ---------------------------------------------------------------------------
# option tables: name -> (kind, default, choices, where).  where: "hash" (a reference
# option that enters config_hash), "plain" (a reference option that does not: output
# locations), "ext" (ours: hashed only when it differs from its default).

_ANGLE = re.compile(r"^(-?)(\d*\.?\d*)pi(?:/(\d+\.?\d*))?$")


def parse_angle(text) -> float:
    """cli.py:49-64: radians as a float or a multiple of pi ("pi/12", "5pi/12", "0.5pi")."""
    s = str(text).strip().lower().replace(" ", "")
    m = _ANGLE.match(s)
    if m:
        den = float(m.group(3)) if m.group(3) else 1.0
        if den == 0.0:
            raise ConfigError(f"bad angle {text!r}")
        return (-1.0 if m.group(1) else 1.0) * (float(m.group(2)) if m.group(2) else 1.0) * math.pi / den
    try:
        return float(s)
    except ValueError:
        raise ConfigError(f"bad angle {text!r}") from None


def _bool(text) -> bool:
    s = str(text).strip().lower()
    if s in ("true", "1", "yes"):
        return True
    if s in ("false", "0", "no"):
        return False
    raise ConfigError(f"bad boolean {text!r}")


def _items(text):
    return [p.strip() for p in str(text).split(",") if p.strip()]


PARSE = {"str": str, "int": int, "float": float, "angle": parse_angle, "bool": _bool,
         "strs": _items, "ints": lambda s: [int(p) for p in _items(s)],
         "floats": lambda s: [float(p) for p in _items(s)], "angles": lambda s: [parse_angle(p) for p in _items(s)]}


def render(kind: str, v) -> str:
    """The text a value has in config files and in the hash (cli.py:94-105)."""
    if kind in ("strs", "ints"):
        return ",".join(str(x) for x in v)
    if kind in ("floats", "angles"):
        return ",".join(repr(float(x)) for x in v)
    if kind == "bool":
        return "true" if v else "false"
    if kind in ("float", "angle"):
        return repr(float(v))
    return str(v)


def _opts(*rows):
    return {r[0]: (r[1], r[2], r[3] if len(r) > 3 else None, r[4] if len(r) > 4 else "hash") for r in rows}


_GEOS, _KRY = ("square", "lshape", "cylinder"), ("none", "fgmres", "gmres")
_EXT = (("device", "str", "b200", ("b200",), "ext"), ("gpus", "int", 1, None, "ext"),
        ("sweeps", "int", 1, None, "ext"), ("precision", "int", 64, (64, 32), "ext"))
_OUT = (("out", "str", ".", None, "plain"), ("csv", "str", None, None, "plain"))
OPTIONS = {
    "train": _opts(
        ("family", "str", "rotated", ("rotated", "variable")), ("n", "int", 16), ("geometry", "str", "square", _GEOS),
        ("theta", "angle", 0.0), ("xi", "float", 100.0), ("kappa", "float", 1.0), ("levels", "int", 2),
        ("scheme", "str", "full", ("full", "redblack")),
        ("strategy", "str", "adaptive", ("adaptive", "independent")), ("variant", "str", None, ("fc", "conv")),
        ("net_k", "int", 1), ("form", "str", "full", ("full", "rb")), ("omega", "float", 2.0 / 3.0),
        ("activation", "str", "linear", ("linear", "leaky")), ("epochs", "int", 500), ("samples", "int", 50),
        ("batch_size", "int", 10), ("learning_rate", "float", 1e-3), ("max_steps", "int", 4), ("inject_k", "int", 0),
        ("thetas", "angles", None), ("seed", "int", 0), ("out", "str", ".", None, "plain"),
        ("device", "str", "b200", ("b200",), "ext")),
    "solve": _opts(
        ("family", "str", "rotated", ("rotated", "variable")), ("n", "int", 16), ("geometry", "str", "square", _GEOS),
        ("theta", "angle", 0.0), ("xi", "float", 100.0), ("kappa", "float", 1.0), ("levels", "int", 2),
        ("scheme", "str", "full", ("full", "redblack")),
        ("smoother", "str", "jacobi", ("jacobi", "gauss-seidel", "exact")), ("omega", "float", 2.0 / 3.0),
        ("model", "str", None), ("tol", "float", 1e-6), ("max_iter", "int", 1000), ("krylov", "str", "none", _KRY),
        ("precond", "str", "mg", ("mg", "none")), ("rhs", "str", "random", ("random", "zero", "ones")),
        ("trials", "int", 1), ("seed", "int", 0), *_OUT, *_EXT),
    "bench": _opts(
        ("family", "str", "rotated", ("rotated", "variable")), ("geometry", "str", "square", _GEOS),
        ("xi", "float", 100.0), ("thetas", "angles", [0.0]), ("kappas", "floats", [1.0]), ("ns", "ints", [16]),
        ("schemes", "strs", ["full"]), ("levels", "int", 2), ("smoothers", "strs", ["jacobi"]),
        ("omega", "float", 2.0 / 3.0), ("krylov", "str", "none", _KRY), ("precond", "str", "mg", ("mg", "none")),
        ("matched_cost", "bool", False), ("tol", "float", 1e-6), ("max_iter", "int", 1000),
        ("rhs", "str", "random", ("random", "zero", "ones")), ("trials", "int", 1), ("workers", "int", 4),
        ("seed", "int", 0), *_OUT, *_EXT),
}
EXT_COLUMNS = ["device", "gpus", "unknowns_per_s", "achieved_GBps", "roofline_frac"]
SOLVE_COLUMNS = ["config_hash", "seed", "family", "geometry", "n", "theta", "xi", "kappa", "levels", "scheme",
                 "smoother", "krylov", "trial", "iterations", "rel_residual", "wall_time", "converged"] + EXT_COLUMNS


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise ConfigError(message)


def build_parser():
    top = _Parser(prog="mgsmooth-b200", description="Multigrid with trained smoothers on B200.")
    subs = top.add_subparsers(dest="subcommand")
    for sub, table in OPTIONS.items():
        p = subs.add_parser(sub)
        p.add_argument("--config", default=None, help="flat key=value config file; flags win")
        for name, (kind, default, choices, _) in table.items():
            p.add_argument("--" + name.replace("_", "-"), dest=name, default=None, type=PARSE[kind],
                           metavar=kind.upper(), help=f"default {default!r}" + (f", one of {choices}" if choices else ""))
    return top


def read_config_file(path: str, table: dict) -> dict:
    """cli.py:239-264: key = value lines with # comments; unknown keys are errors."""
    try:
        with open(path) as fh:
            lines = fh.read().splitlines()
    except OSError as exc:
        raise ConfigError(f"cannot read config {path}: {exc}") from None
    out = {}
    for no, raw in enumerate(lines, 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        key, eq, value = (s.strip() for s in line.partition("="))
        if not eq:
            raise ConfigError(f"{path}:{no}: expected key=value")
        if key not in table:
            raise ConfigError(f"{path}:{no}: unknown config key {key!r}")
        try:
            out[key] = PARSE[table[key][0]](value)
        except (ValueError, ConfigError) as exc:
            raise ConfigError(f"{path}:{no}: bad value for {key}: {exc}") from None
    return out


def write_config_file(sub: str, cfg: dict, path: str):
    with open(path, "w") as fh:
        for name in sorted(cfg):
            if cfg[name] is not None:
                fh.write(f"{name} = {render(OPTIONS[sub][name][0], cfg[name])}\n")


def resolve_config(sub: str, ns) -> dict:
    """cli.py:276-297: flag, else file value, else default; MGSMOOTH_SEED wins over both."""
    table = OPTIONS[sub]
    filed = read_config_file(ns.config, table) if getattr(ns, "config", None) else {}
    cfg = {}
    for name, (_, default, choices, _) in table.items():
        v = getattr(ns, name, None)
        v = filed.get(name, default) if v is None else v
        if v is not None and choices and v not in choices:
            raise ConfigError(f"{name} must be one of {', '.join(str(c) for c in choices)}, got {v!r}")
        cfg[name] = v
    env = os.environ.get("MGSMOOTH_SEED")
    if env is not None:
        try:
            cfg["seed"] = int(env)
        except ValueError:
            raise ConfigError(f"bad MGSMOOTH_SEED {env!r}") from None
    return cfg


def config_hash(sub: str, cfg: dict) -> str:
    """cli.py:300-308: sha256 over the sorted hashed options, 12 hex digits."""
    lines = [f"subcommand={sub}"]
    for name in sorted(cfg):
        kind, default, _, where = OPTIONS[sub][name]
        if cfg[name] is None or where == "plain" or (where == "ext" and cfg[name] == default):
            continue
        lines.append(f"{name}={render(kind, cfg[name])}")
    return hashlib.sha256("\n".join(lines).encode()).hexdigest()[:12]


# ---------------------------------------------------------------------------
# run core

def load_model_file(path: str):
    """cli.py:334-358: ("net", KernelInferenceNet) or ("stack", hierarchy with the
    file's conv smoothers on the operator it was trained on)."""
    from . import build_hierarchy, model_from_dict
    from .problems import ProblemSpec
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except OSError as exc:
        raise ConfigError(f"cannot read model {path}: {exc}") from None
    except json.JSONDecodeError as exc:
        raise ConfigError(f"model {path} is not valid JSON: {exc}") from None
    if doc.get("format_version") != 1:
        raise ConfigError(f"unsupported model format {doc.get('format_version')!r}")
    kind = doc.get("kind")
    if kind == "inference_net":
        return "net", model_from_dict(doc)
    if kind != "smoother_stack":
        raise ConfigError(f"model {path} has unknown kind {kind!r}")
    src = build_hierarchy(ProblemSpec(**doc["problem"]).assemble(), doc["levels"], scheme=doc["scheme"])
    if len(doc["smoothers"]) != src.depth - 1:
        raise ConfigError(f"model {path} smoother count does not match its hierarchy depth")
    for lev, sm in zip(src.levels[:-1], doc["smoothers"]):
        lev.smoother = model_from_dict(sm, spec=lev.spec)
    return "stack", src


def equip(hier, cfg: dict) -> str:
    """cli.py:389-401: install the run's smoother, return its CSV tag."""
    from . import equip_classical, equip_inferred, equip_trained
    if cfg.get("model"):
        kind, loaded = load_model_file(cfg["model"])
        if kind == "stack":
            equip_trained(hier, loaded)
        else:
            equip_inferred(hier, loaded, precision=cfg.get("precision", 64))
        return os.path.splitext(os.path.basename(cfg["model"]))[0]
    if cfg["smoother"] == "exact":
        raise ConfigError("the exact smoother is analysis-only")
    equip_classical(hier, cfg["smoother"], cfg["omega"])
    return cfg["smoother"]


def make_rhs(spec, kind: str, seed_parts):
    """cli.py:404-412."""
    from . import GridFunction, from_active, zeros
    if kind == "zero":
        return zeros(spec)
    if kind == "ones":
        return GridFunction(spec, np.where(spec.mask, 1.0, 0.0))
    vec = np.random.default_rng(seed_parts).standard_normal(spec.n_active)
    return from_active(spec, vec / np.linalg.norm(vec))


def solve_once(hier, A, cfg: dict, trial: int):
    """cli.py:415-441: (iterations, relative residual, wall seconds, converged)."""
    from . import FgmresConfig, cycle_preconditioner, fgmres, gmres, grid_action, solve
    f = make_rhs(A.spec, cfg["rhs"], [cfg["seed"], trial])
    if cfg["krylov"] == "none":
        _, rep = solve(hier, f, tol=cfg["tol"], max_iter=cfg["max_iter"])
        return rep.iterations, rep.residual_history[-1], rep.wall_time, rep.converged
    kcfg = FgmresConfig(tol=cfg["tol"], max_iter=cfg["max_iter"])
    action, fv = grid_action(A), f.values.ravel()
    t0 = time.perf_counter()
    if cfg["krylov"] == "gmres":
        _, rep = gmres(action, fv, cfg=kcfg)
    else:
        pc = cycle_preconditioner(hier) if cfg["precond"] == "mg" else None
        _, rep = fgmres(action, fv, precond=pc, cfg=kcfg, tag="mg" if pc is not None else "none")
    dt = time.perf_counter() - t0
    rel = rep.history[-1] / rep.history[0] if rep.history[0] > 0 else 0.0
    if cfg["krylov"] == "fgmres" and any(b > a * (1.0 + 1e-12) for a, b in zip(rep.history, rep.history[1:])):
        raise NumericError("FGMRES residual history is not monotone")
    return rep.iterations, rel, dt, rep.converged


def _visible_gpus(cfg: dict) -> int:
    from . import device as dv
    if cfg["device"] != "b200":
        raise ConfigError(f"device must be b200, got {cfg['device']!r}")
    if cfg["gpus"] < 1:
        raise ConfigError("gpus must be >= 1")
    t = dv.torch()
    have = t.cuda.device_count() if t.cuda.is_available() else 0
    if have < cfg["gpus"]:
        raise ConfigError(f"--gpus {cfg['gpus']} but {have} CUDA device(s) visible (the B200 path has no CPU fallback)")
    return cfg["gpus"]


def _prepare(cfg: dict, A, gpu: int):
    """Hierarchy of A on `gpu` with the run's smoother; (hier, tag, sweeps, bytes per cycle)."""
    from . import RepeatedSmoother, build_hierarchy
    hier = build_hierarchy(A, cfg["levels"], scheme=cfg["scheme"], device=gpu)
    tag = equip(hier, cfg)
    nu = int(cfg.get("sweeps") or 1)
    if cfg.get("matched_cost") and cfg.get("model") is None:
        nu = 6   # cli.py:380-383 (full coarsening)
    if nu < 1:
        raise ConfigError("sweeps must be >= 1")
    if nu > 1:
        for lev in hier.levels[:-1]:
            lev.smoother = RepeatedSmoother(lev.smoother, lev.operator, nu)
    compact = all(hier.storage_info(0))
    bytes_cycle = roofline.cycle_bytes(A.spec.rows, A.spec.cols, cfg["levels"], nu, nu, compact)
    return hier, tag, nu, bytes_cycle


def _throughput(n_active: int, iters, dt: float, bytes_cycle: float, krylov: str):
    """Extension columns of one row: unknowns/s per cycle; bytes only for plain cycles
    (a Krylov iteration moves the Arnoldi vectors too)."""
    ups = n_active * float(iters) / dt if dt > 0 else 0.0
    if krylov != "none" or dt <= 0:
        return {"unknowns_per_s": f"{ups:.6e}", "achieved_GBps": "", "roofline_frac": ""}
    gbps = bytes_cycle * float(iters) / dt / 1e9
    return {"unknowns_per_s": f"{ups:.6e}", "achieved_GBps": f"{gbps:.3f}",
            "roofline_frac": f"{gbps / roofline.hbm_peak_gbs()[0]:.4f}"}


def solve_rows(cfg: dict, chash: str, devices=None):
    """cli.py:450-477.  `devices`: the GPUs this run may use (default: 0 .. gpus-1); one
    hierarchy is built per GPU in use and trial t runs on devices[t mod len]."""
    from . import device as dv
    from .problems import ProblemSpec
    if devices is None:
        devices = list(range(_visible_gpus(cfg)))
    devices = devices[:max(1, cfg["trials"])]
    A = ProblemSpec(cfg["family"], cfg["n"], cfg["geometry"], cfg["theta"], cfg["xi"], cfg["kappa"]).assemble()
    prepared = {}
    for g in devices:
        dv.torch().cuda.set_device(g)
        prepared[g] = _prepare(cfg, A, g)
    tag, bytes_cycle = prepared[devices[0]][1], prepared[devices[0]][3]
    fixed = {"config_hash": chash, "seed": cfg["seed"], "family": cfg["family"], "geometry": cfg["geometry"],
             "n": cfg["n"], "theta": repr(cfg["theta"]), "xi": cfg["xi"], "kappa": cfg["kappa"],
             "levels": cfg["levels"], "scheme": cfg["scheme"], "smoother": tag, "krylov": cfg["krylov"],
             "device": cfg["device"], "gpus": cfg["gpus"]}

    def one(trial):
        g = devices[trial % len(devices)]
        dv.torch().cuda.set_device(g)
        iters, rel, dt, ok = solve_once(prepared[g][0], A, cfg, trial)
        return {**fixed, "trial": trial, "iterations": iters, "rel_residual": f"{rel:.6e}", "wall_time": f"{dt:.6f}",
                "converged": ok, **_throughput(A.spec.n_active, iters, dt, bytes_cycle, cfg["krylov"])}

    if len(devices) > 1:
        with ThreadPoolExecutor(max_workers=len(devices)) as pool:
            rows = list(pool.map(one, range(cfg["trials"])))
    else:
        rows = [one(t) for t in range(cfg["trials"])]
    all_ok = all(r["converged"] for r in rows)
    if cfg["trials"] > 1:
        mean_it = sum(r["iterations"] for r in rows) / len(rows)
        mean_dt = sum(float(r["wall_time"]) for r in rows) / len(rows)
        rows.append({**fixed, "trial": "mean", "iterations": f"{mean_it:.2f}", "rel_residual": "",
                     "wall_time": f"{mean_dt:.6f}", "converged": all_ok,
                     **_throughput(A.spec.n_active, mean_it, mean_dt, bytes_cycle, cfg["krylov"])})
    return rows, all_ok


def write_csv(path: str, columns: list, rows: list):
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=columns)
        w.writeheader()
        w.writerows(rows)


# ---------------------------------------------------------------------------
# subcommands

def cmd_solve(cfg: dict) -> int:
    chash = config_hash("solve", cfg)
    rows, all_ok = solve_rows(cfg, chash)
    write_csv(cfg["csv"] or os.path.join(cfg["out"], "solve.csv"), SOLVE_COLUMNS, rows)
    for r in rows:
        print(f"trial {r['trial']}: {r['iterations']} iterations, residual {r['rel_residual']}, "
              f"converged {r['converged']}, {r['unknowns_per_s']} unknowns/s")
    if not all_ok:
        raise NonConvergedError(f"solve failed to reach tol {cfg['tol']} within {cfg['max_iter']} iterations")
    return 0


def cmd_bench(cfg: dict) -> int:
    """cli.py:709-766: the sweep over (theta | kappa) x n x scheme x smoother, cells on
    a thread pool; cell c runs on GPU c mod gpus."""
    chash = config_hash("bench", cfg)
    gpus = _visible_gpus(cfg)
    by_kappa = cfg["family"] == "variable"
    var_col = "kappa" if by_kappa else "theta"
    cells = [(v, n, sch, sm) for v in (cfg["kappas"] if by_kappa else cfg["thetas"]) for n in cfg["ns"]
             for sch in cfg["schemes"] for sm in cfg["smoothers"]]
    gpu_locks = [threading.Lock() for _ in range(gpus)]

    def run_cell(idx):
        value, n, scheme, sm_tag = cells[idx]
        is_model = sm_tag.endswith(".json") or os.path.sep in sm_tag
        sub = dict(cfg, n=n, scheme=scheme, theta=0.0 if by_kappa else value, kappa=value if by_kappa else 1.0,
                   model=sm_tag if is_model else None, smoother="jacobi" if is_model else sm_tag,
                   matched_cost=False if is_model else cfg["matched_cost"])
        with gpu_locks[idx % gpus]:   # one cell at a time per GPU: wall times stay per-cell
            rows, ok = solve_rows(sub, chash, devices=[idx % gpus])
        s = rows[-1]
        return {"cell": idx, "config_hash": chash, "seed": cfg["seed"], "family": cfg["family"],
                "geometry": cfg["geometry"], "n": n, "scheme": scheme, var_col: repr(float(value)),
                "smoother": s["smoother"], "krylov": cfg["krylov"], "iterations": s["iterations"],
                "wall_time": s["wall_time"], "converged": ok, "device": cfg["device"], "gpus": gpus,
                **{k: s[k] for k in EXT_COLUMNS[2:]}}, ok

    workers = max(1, cfg["workers"])
    if workers == 1 or len(cells) == 1:
        results = [run_cell(i) for i in range(len(cells))]
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            results = list(pool.map(run_cell, range(len(cells))))
    columns = ["cell", "config_hash", "seed", "family", "geometry", "n", "scheme", var_col, "smoother", "krylov",
               "iterations", "wall_time", "converged"] + EXT_COLUMNS
    write_csv(cfg["csv"] or os.path.join(cfg["out"], "bench.csv"), columns, [r for r, _ in results])
    for r, _ in results:
        print(f"{var_col}={r[var_col]} n={r['n']} scheme={r['scheme']} {r['smoother']}: {r['iterations']} iterations, "
              f"{r['unknowns_per_s']} unknowns/s")
    if not all(ok for _, ok in results):
        raise NonConvergedError("at least one sweep cell failed to converge")
    return 0


def _not_on_path(name: str):
    def run(_cfg):
        raise UnsupportedOperationError(f"`{name}` is not on the B200 path; run the reference's `mgsmooth {name}` "
                                        "and pass its model file to `solve --model`")
    return run


def stack_to_dict(problem, hier, metadata: dict) -> dict:
    """cli.py:317-331: a hierarchy's conv smoothers with the problem they were trained on."""
    from . import model_to_dict
    return {"format_version": 1, "kind": "smoother_stack", "problem": problem.asdict(), "scheme": hier.scheme,
            "levels": hier.depth, "metadata": metadata,
            "smoothers": [model_to_dict(lev.smoother) for lev in hier.levels[:-1]]}


def _stack_params(hier) -> int:
    total = 0
    for lev in hier.levels[:-1]:
        sm = lev.smoother
        total += sum(k.weights.size for k in sm.layers) + (sm.skip.weights.size if sm.skip is not None else 0)
    return total


def cmd_train(cfg: dict) -> int:
    """cli.py:489-587 on the GPU trainers."""
    from . import build_hierarchy, model_to_dict, training as tr
    from .problems import ProblemSpec
    _visible_gpus(dict(cfg, gpus=1))
    chash = config_hash("train", cfg)
    problem = ProblemSpec(cfg["family"], cfg["n"], cfg["geometry"], cfg["theta"], cfg["xi"], cfg["kappa"])
    tc = tr.TrainConfig(samples=cfg["samples"], max_steps=cfg["max_steps"], batch_size=cfg["batch_size"],
                        learning_rate=cfg["learning_rate"], epochs=cfg["epochs"], seed=cfg["seed"])
    A = problem.assemble()
    meta = {"config_hash": chash, "seed": cfg["seed"], "epochs": cfg["epochs"]}
    notes = []
    t0 = time.perf_counter()
    if cfg["variant"] is not None:
        net, hier, records = tr.train_inference_net(A, cfg["variant"], cfg["levels"], tc, k=cfg["net_k"])
        params = net.parameter_count()
        doc = model_to_dict(net, {**meta, "parameters": params, "problem": problem.asdict()})
    elif cfg["thetas"] is not None:
        if cfg["family"] != "rotated":
            raise ConfigError("angle mixtures need the rotated family")
        ops = [ProblemSpec(cfg["family"], cfg["n"], cfg["geometry"], t, cfg["xi"], cfg["kappa"]).assemble()
               for t in cfg["thetas"]]
        hiers, records = tr.train_mixture(ops, cfg["levels"], tc, scheme=cfg["scheme"], omega=cfg["omega"],
                                          activation=cfg["activation"])
        hier = hiers[0]
        params = _stack_params(hier)
        notes.append("mixture model; kernels shared across angles, saved against the first angle's operator")
        doc = stack_to_dict(problem, hier, {**meta, "parameters": params})
    elif cfg["strategy"] == "independent":
        sm, record = tr.train_independent(A, tc, form=cfg["form"], omega=cfg["omega"], activation=cfg["activation"])
        hier = build_hierarchy(A, 2, scheme=cfg["scheme"])   # saved as a depth-2 stack (cli.py:527-531)
        hier.levels[0].smoother = sm
        records = [record]
        params = _stack_params(hier)
        doc = stack_to_dict(problem, hier, {**meta, "parameters": params})
    else:
        hier, records = tr.train_adaptive(A, cfg["levels"], tc, scheme=cfg["scheme"], omega=cfg["omega"],
                                          activation=cfg["activation"])
        if cfg["inject_k"] > 0:
            hier, more = tr.retrain_with_injection(hier, tc, cfg["inject_k"])
            records = records + more
            notes.append(f"retrained on residual probes after {cfg['inject_k']} cycles")
        params = _stack_params(hier)
        doc = stack_to_dict(problem, hier, {**meta, "parameters": params})
    wall = time.perf_counter() - t0
    if cfg["epochs"] < 500:
        notes.append("epochs below the 500 default")
    os.makedirs(cfg["out"], exist_ok=True)
    model_path = os.path.join(cfg["out"], "model.json")
    with open(model_path, "w") as fh:
        json.dump(doc, fh, sort_keys=True)
    loss_path = os.path.join(cfg["out"], "loss.csv")
    write_csv(loss_path, ["config_hash", "seed", "level", "epoch", "loss"],
              [{"config_hash": chash, "seed": cfg["seed"], "level": rec.level, "epoch": e, "loss": f"{v:.10e}"}
               for rec in records for e, v in enumerate(rec.epochs)])
    manifest = {"subcommand": "train",
                "config": {k: render(OPTIONS["train"][k][0], v) for k, v in cfg.items() if v is not None},
                "config_hash": chash, "seed": cfg["seed"], "problem": problem.asdict(), "parameters": params,
                "records": [{"level": r.level, "epochs": len(r.epochs), "initial": r.initial if r.epochs else None,
                             "final": r.final if r.epochs else None} for r in records],
                "wall_time": wall, "notes": notes, "device": cfg["device"],
                "outputs": {"model": model_path, "loss": loss_path}}
    with open(os.path.join(cfg["out"], "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=2, sort_keys=True)
    print(f"model: {model_path}")
    print(f"parameters: {params}")
    for r in records:
        print(f"level {r.level}: loss {r.initial:.6f} -> {r.final:.6f} ({len(r.epochs)} epochs)" if r.epochs
              else f"level {r.level}: initialization kept (0 epochs)")
    return 0


COMMANDS = {"train": cmd_train, "solve": cmd_solve, "bench": cmd_bench, "analyze": _not_on_path("analyze")}


def main(argv=None) -> int:
    """cli.py:774-793: exit codes 0 ok, 1 config / unsupported, 2 numeric failure, 3 not converged."""
    parser = build_parser()
    args = sys.argv[1:] if argv is None else list(argv)
    try:
        if args and args[0] == "analyze":
            return COMMANDS[args[0]]({})
        ns = parser.parse_args(args)
        if ns.subcommand is None:
            parser.print_help()
            return 1
        return COMMANDS[ns.subcommand](resolve_config(ns.subcommand, ns))
    except (ConfigError, UnsupportedOperationError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except NonConvergedError as exc:
        print(f"not converged: {exc}", file=sys.stderr)
        return 3
    except (NumericError, SingularMatrixError, TrainingError, ContractError) as exc:
        print(f"numeric failure: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
