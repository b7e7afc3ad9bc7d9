"""Golden rows of the reference command-line front end (cli.py `solve` / `bench`).

Run in the build container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cli.py

Runs the UNMODIFIED reference `mgsmooth.cli.main(argv)` from tests/golden/ (so model
paths are the bare fixture names) and writes cli_rows.json: for every case its argv,
exit code and the CSV rows the reference wrote.  stack_model.json is a `smoother_stack`
model file from a short reference `train` run (adaptive strategy, 15^2, 3 levels,
2 epochs, 4 samples, seed 0): the input of the equip_trained case.
"""
import csv
import json
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))

from mgsmooth import cli  # noqa: E402  (reference)

ROT31 = ["--n", "31", "--theta", "pi/6", "--xi", "0.01", "--levels", "4"]
CASES = {
    "solve_jacobi_trials2": ["solve", *ROT31, "--trials", "2", "--max-iter", "400"],
    "solve_variable": ["solve", "--family", "variable", "--n", "31", "--kappa", "3.0", "--levels", "4"],
    "solve_lshape_net": ["solve", *ROT31, "--geometry", "lshape", "--model", "net_conv.json", "--seed", "3"],
    "solve_cylinder_fc": ["solve", "--n", "31", "--theta", "pi/6", "--xi", "0.01", "--levels", "3", "--geometry",
                          "cylinder", "--model", "net_fc.json", "--rhs", "ones"],
    "solve_fgmres_mg": ["solve", *ROT31, "--model", "net_conv.json", "--krylov", "fgmres", "--tol", "1e-8"],
    "solve_fgmres_none": ["solve", "--n", "15", "--theta", "0.3", "--xi", "0.1", "--levels", "2", "--krylov", "fgmres",
                          "--precond", "none", "--max-iter", "300"],
    "solve_gmres": ["solve", "--n", "15", "--theta", "0.3", "--xi", "0.1", "--levels", "2", "--krylov", "gmres",
                    "--max-iter", "300"],
    "solve_stack": ["solve", "--n", "31", "--theta", "pi/6", "--xi", "0.01", "--levels", "4", "--model",
                    "stack_model.json"],
    "solve_not_converged": ["solve", *ROT31, "--max-iter", "3"],
    "bench_sweep": ["bench", "--ns", "15,31", "--thetas", "pi/6,0.45", "--xi", "0.01", "--levels", "3", "--smoothers",
                    "jacobi,net_conv.json", "--matched-cost", "true", "--trials", "2", "--workers", "1"],
    "bench_diverges": ["bench", "--ns", "15", "--thetas", "pi/3", "--xi", "0.01", "--levels", "3", "--smoothers",
                       "net_conv.json", "--workers", "1"],
    "bench_variable": ["bench", "--family", "variable", "--kappas", "1.0,4.0", "--ns", "31", "--levels", "4",
                       "--workers", "2"],
}


def main():
    os.chdir(HERE)
    tmp = tempfile.mkdtemp()
    if not os.path.exists("stack_model.json"):
        rc = cli.main(["train", "--n", "15", "--theta", "pi/6", "--xi", "0.01", "--levels", "3", "--epochs", "2",
                       "--samples", "4", "--batch-size", "2", "--max-steps", "2", "--out", tmp])
        assert rc == 0
        shutil.copy(os.path.join(tmp, "model.json"), "stack_model.json")
    out = {}
    for name, argv in CASES.items():
        path = os.path.join(tmp, name + ".csv")
        rc = cli.main(argv + ["--csv", path])
        rows = None   # an uncaught solver error (e.g. divergence) leaves no CSV
        if os.path.exists(path):
            with open(path) as fh:
                rows = list(csv.DictReader(fh))
        out[name] = {"argv": argv, "exit_code": rc, "rows": rows}
        print(name, rc, [(r.get("iterations"), r.get("rel_residual", "")) for r in rows or []])
    with open("cli_rows.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    sys.exit(main())
