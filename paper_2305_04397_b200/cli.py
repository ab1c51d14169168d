"""Command-line front end over the B200 path (mirrors the reference's `morap` verbs that
touch it: `solve`, `verify` and `bench`, cli.hpp:196-327).

    python -m paper_2305_04397_b200 solve  --instance FILE --thresholds a,b,... [--eps 0.01]
                                           [--norm FILE] [--max-iters 500] [--centralised] [--out FILE]
    python -m paper_2305_04397_b200 verify --instance FILE --thresholds a,b,... [--eps 0.01]
    python -m paper_2305_04397_b200 bench  --config FILE [--centralised] [--seed S] [--out FILE]

Negative bounds need the `=` form: `--thresholds=-20,-20,0.9,0.9`.
`solve` prints the reference's solveJson (cli.hpp:253-275): resultToJson plus converged,
eps, thresholds, iterationCount and the synthesis marginal. `bench` runs every warehouse
config of a {"runs": [...]} file and reports generate / solve seconds, verdict, iterations
and tUp/tDown per run like benchVerb (cli.hpp:277-327). Every solve runs on the GPU; there
is no CPU solver behind these verbs.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np


def _thresholds(text: str) -> list:
    try:
        return [float(v) for v in text.split(",") if v.strip()]
    except ValueError as e:
        raise SystemExit(f"bad --thresholds: {e}")


def _norm(path: str | None, inst):
    if path:
        return np.asarray(json.load(open(path)), np.float64)
    return inst.norm


def _solve_json(rep: dict, eps: float) -> dict:
    out = {k: rep[k] for k in ("feasible", "tUp", "tDown", "iterations") if k in rep}
    for k in ("lambda", "phi", "synthesis"):
        if k in rep:
            out[k] = rep[k]
    out["converged"] = rep["converged"]
    out["eps"] = eps
    out["thresholds"] = rep["thresholds"]
    out["iterationCount"] = len(rep["iterations"])
    if "marginal" in rep:
        out["marginal"] = rep["marginal"]
    return out


def cmd_solve(a) -> int:
    from .api import Centralised, Instance, Solver
    inst = Instance.from_json(open(a.instance).read(), os.path.dirname(os.path.abspath(a.instance)))
    thr = _thresholds(a.thresholds)
    solver = Solver(a.device)
    norm = _norm(a.norm, inst)
    if a.centralised:
        rep = solver.centralised_pareto(Centralised(inst), thr, eps=a.eps, norm=norm, iteration_cap=a.max_iters)
    else:
        rep = solver.pareto(inst, thr, eps=a.eps, norm=norm, iteration_cap=a.max_iters)
    out = _solve_json(rep, a.eps)
    text = json.dumps(out, indent=2)
    print(text)
    if a.out:
        open(a.out, "w").write(text + "\n")
    return 0


def cmd_verify(a) -> int:
    from .api import Instance, Solver
    inst = Instance.from_json(open(a.instance).read(), os.path.dirname(os.path.abspath(a.instance)))
    v = Solver(a.device).verify(inst, _thresholds(a.thresholds), eps=a.eps, norm=_norm(a.norm, inst),
                                iteration_cap=a.max_iters)
    print(json.dumps({"verdict": v}))
    return 0


def cmd_bench(a) -> int:
    from .api import Centralised, Instance, Solver
    cfg = json.load(open(a.config))
    if not isinstance(cfg, dict) or "runs" not in cfg:
        raise SystemExit("bench config needs a runs array")
    solver = Solver(a.device)
    runs = []
    for run in cfg["runs"]:
        wc = dict(run["config"])
        if a.seed is not None:
            wc["seed"] = a.seed
        eps = run.get("eps", 0.01)
        t0 = time.perf_counter()
        inst = Instance.warehouse(wc)
        t1 = time.perf_counter()
        entry = {"config": wc, "agents": inst.n, "totalProductStates": inst.total_states,
                 "distinctProducts": inst.distinct, "generateSeconds": t1 - t0}
        t2 = time.perf_counter()
        if a.centralised:
            c = Centralised(inst)
            entry["centralisedStates"] = c.S
            rep = solver.centralised_pareto(c, run["thresholds"], eps=eps)
        else:
            solver.release()
            rep = solver.pareto(inst, run["thresholds"], eps=eps)
        entry["solveSeconds"] = time.perf_counter() - t2
        entry.update(feasible=rep["feasible"], converged=rep["converged"], iterations=len(rep["iterations"]),
                     tUp=rep["tUp"], tDown=rep["tDown"])
        runs.append(entry)
    text = json.dumps({"runs": runs}, indent=2)
    print(text)
    if a.out:
        open(a.out, "w").write(text + "\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2305_04397_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="verb", required=True)
    for verb in ("solve", "verify"):
        p = sub.add_parser(verb)
        p.add_argument("--instance", required=True)
        p.add_argument("--thresholds", required=True)
        p.add_argument("--eps", type=float, default=0.01)
        p.add_argument("--norm")
        p.add_argument("--max-iters", type=int, default=500)
        p.add_argument("--device", type=int, default=0)
        if verb == "solve":
            p.add_argument("--centralised", action="store_true")
            p.add_argument("--out")
    p = sub.add_parser("bench")
    p.add_argument("--config", required=True)
    p.add_argument("--centralised", action="store_true")
    p.add_argument("--seed", type=int)
    p.add_argument("--out")
    p.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        return {"solve": cmd_solve, "verify": cmd_verify, "bench": cmd_bench}[a.verb](a)
    except Exception as e:  # a library error exits 2 with its message
        from .errors import MorapError
        if isinstance(e, MorapError):
            print(f"error: {e}", file=sys.stderr)
            return 2
        raise


if __name__ == "__main__":
    sys.exit(main())
