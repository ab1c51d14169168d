"""Command-line front end over the B200 path: the reference's `morap` verbs that touch it
(cli.hpp:335-410) with the same options, output and exit codes.

    python -m paper_2305_04397_b200 pareto --instance FILE --thresholds a,b,... [--eps 0.01]
                                           [--norm FILE] [--max-iters 500] [--centralised] [--out CSV]
    python -m paper_2305_04397_b200 verify --instance FILE --thresholds a,b,... [--out JSON] ...
    python -m paper_2305_04397_b200 synth  --instance FILE --thresholds a,b,... [--out JSON] ...
    python -m paper_2305_04397_b200 bench  --config FILE [--centralised] [--seed S] [--out FILE]

(`solve` is kept as an alias of `pareto`.) Negative bounds need the `=` form:
`--thresholds=-20,-20,0.9,0.9`.

pareto / verify / synth print solveJson (cli.hpp:253-275): resultToJson plus converged, eps,
thresholds and iterationCount; synth adds the certificate (synthesis terms, marginal).
`pareto --out` writes the CSV trace of writeParetoCsv (cli.hpp:135-153, %.9g); verify and
synth write the JSON. Exit codes follow runCli / exitCodeFor (cli.hpp:185-195, 387-410):
0 feasible, 1 infeasible, 2 usage / Syntax / InvalidConfig / DimensionMismatch / Io errors,
3 any other error. `bench` runs every warehouse config of a {"runs": [...]} file and reports
generate / solve seconds, verdict, iterations and tUp/tDown per run like benchVerb
(cli.hpp:277-327). Every solve runs on the GPU; there is no CPU solver behind these verbs.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

from .errors import Errc, MorapError

USAGE_CODES = (Errc.Syntax, Errc.InvalidConfig, Errc.DimensionMismatch, Errc.Io)


class _Usage(Exception):
    """An argument error (CLI::ParseError in the reference): exit code 2."""


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _Usage(message)


def exit_code_for(e: Exception) -> int:
    """exitCodeFor (cli.hpp:185-195)."""
    if isinstance(e, MorapError):
        return 2 if e.code in USAGE_CODES else 3
    return 3


def _fail(code: Errc, msg: str):
    raise MorapError(int(code) + 1, msg)


def _thresholds(text: str) -> list:
    """parseThresholds (cli.hpp:164-183): comma-separated doubles, at least one."""
    out = []
    for tok in text.split(","):
        try:
            out.append(float(tok))
        except ValueError:
            _fail(Errc.InvalidConfig, f"bad threshold '{tok}'")
    if not out:
        _fail(Errc.InvalidConfig, "no thresholds given")
    return out


def _read(path: str) -> str:
    try:
        with open(path) as f:
            return f.read()
    except OSError as e:
        _fail(Errc.Io, f"cannot read {path}: {e.strerror}")


def _load_instance(path: str, solver=None):
    """instanceFromJson; with `solver`, the products are built on its GPU (--device-build)."""
    from .api import Instance
    if solver is not None:
        return Instance.from_json_device(_read(path), solver, os.path.dirname(os.path.abspath(path)))
    return Instance.from_json(_read(path), os.path.dirname(os.path.abspath(path)))


def _solve_json(rep: dict, eps: float, synth: bool) -> dict:
    """solveJson (cli.hpp:253-275)."""
    out = {k: rep[k] for k in ("feasible", "tUp", "tDown") if k in rep}
    out["iterations"] = [{"w": it["w"], "r": it["r"], "assignment": it["assignment"]} for it in rep["iterations"]]
    out["synthesis"] = rep.get("synthesis", []) if synth else []
    out["converged"] = rep["converged"]
    out["eps"] = eps
    out["thresholds"] = rep["thresholds"]
    out["iterationCount"] = len(rep["iterations"])
    if synth:
        if "marginal" not in rep:
            _fail(Errc.NoCertificate, "no certificate: the query did not converge")
        out["marginal"] = rep["marginal"]
    return out


def _g9(v: float) -> str:
    return "%.9g" % v


def pareto_csv(rep: dict) -> str:
    """writeParetoCsv (cli.hpp:135-153)."""
    dim = len(rep["thresholds"])
    lines = ["iter" + "".join(f",w_{k}" for k in range(1, dim + 1)) + "".join(f",r_{k}" for k in range(1, dim + 1))]
    for i, it in enumerate(rep["iterations"]):
        lines.append(str(i + 1) + "".join("," + _g9(v) for v in it["w"]) + "".join("," + _g9(v) for v in it["r"]))
    lines.append("tUp" + "".join("," + _g9(v) for v in rep["tUp"]))
    lines.append("tDown" + "".join("," + _g9(v) for v in rep["tDown"]))
    return "\n".join(lines) + "\n"


def _write(path: str, text: str):
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError as e:
        _fail(Errc.Io, f"cannot open {path} for writing: {e.strerror}")


def cmd_solve(a, verb: str) -> int:
    """runSolve + the pareto / verify / synth branch of runCli (cli.hpp:230-250, 387-405)."""
    from .api import Centralised, Solver
    device_build = getattr(a, "device_build", False)
    if device_build and getattr(a, "centralised", False):
        _fail(Errc.InvalidConfig, "--device-build keeps the products on the device; --centralised needs them on the host")
    solver = Solver(a.device) if device_build else None
    inst = _load_instance(a.instance, solver)
    thr = _thresholds(a.thresholds)
    if len(thr) != inst.objectives * inst.n:  # paretoPoint's dimension check, before any device work
        _fail(Errc.DimensionMismatch, f"{len(thr)} thresholds for {inst.objectives * inst.n} objectives")
    norm = np.asarray(json.loads(_read(a.norm)), np.float64) if a.norm else inst.norm
    solver = solver or Solver(a.device)
    if getattr(a, "centralised", False):
        rep = solver.centralised_pareto(Centralised(inst), thr, eps=a.eps, norm=norm, iteration_cap=a.max_iters)
    else:
        rep = solver.pareto(inst, thr, eps=a.eps, norm=norm, iteration_cap=a.max_iters)
    out = _solve_json(rep, a.eps, synth=(verb == "synth"))
    text = json.dumps(out, indent=2)
    print(text)
    if a.out:
        _write(a.out, pareto_csv(rep) if verb == "pareto" else text + "\n")
    return 0 if rep["feasible"] else 1


def cmd_bench(a) -> int:
    """benchVerb (cli.hpp:277-327)."""
    from .api import Centralised, Instance, Solver
    cfg = json.loads(_read(a.config))
    if not isinstance(cfg, dict) or "runs" not in cfg:
        _fail(Errc.InvalidConfig, "bench config needs a runs array")
    solver = Solver(a.device)
    runs = []
    for run in cfg["runs"]:
        wc = dict(run["config"])
        if a.seed is not None:
            wc["seed"] = a.seed
        eps = run.get("eps", 0.01)
        t0 = time.perf_counter()
        if a.device_build and not a.centralised:
            solver.release()
            inst = Instance.warehouse_device(wc, solver)  # products built on the GPU, resident
        else:
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
            if not a.device_build:
                solver.release()
            rep = solver.pareto(inst, run["thresholds"], eps=eps)
        entry["solveSeconds"] = time.perf_counter() - t2
        entry.update(feasible=rep["feasible"], converged=rep["converged"], iterations=len(rep["iterations"]),
                     tUp=rep["tUp"], tDown=rep["tDown"])
        runs.append(entry)
    text = json.dumps({"runs": runs}, indent=2)
    print(text)
    if a.out:
        _write(a.out, text + "\n")
    return 0


def _parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="paper_2305_04397_b200",
                 description="model checking toolkit for random task assignment and planning (B200 path)")
    sub = ap.add_subparsers(dest="verb", parser_class=_Parser)
    helps = {"verify": "decide whether thresholds are achievable",
             "pareto": "decide feasibility and report the sandwich points; --out writes the CSV trace",
             "solve": "alias of pareto",
             "synth": "solve and emit the random assignment certificate (decentralised only)"}
    for verb, h in helps.items():
        p = sub.add_parser(verb, help=h)
        p.add_argument("--instance", required=True)
        p.add_argument("--thresholds", required=True)
        p.add_argument("--eps", type=float, default=0.01)
        p.add_argument("--norm")
        p.add_argument("--max-iters", type=int, default=500)
        p.add_argument("--workers", type=int, default=0, help="accepted for compatibility (device batches)")
        p.add_argument("--device", type=int, default=0)
        p.add_argument("--device-build", action="store_true", help="build the products on the GPU")
        p.add_argument("--out")
        if verb != "synth":
            p.add_argument("--centralised", action="store_true")
    p = sub.add_parser("bench", help="run a warehouse suite and report measurements")
    p.add_argument("--config", required=True)
    p.add_argument("--centralised", action="store_true")
    p.add_argument("--seed", type=int)
    p.add_argument("--workers", type=int, default=0)
    p.add_argument("--out")
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--device-build", action="store_true", help="build the products on the GPU (decentralised runs)")
    return ap


def main(argv=None) -> int:
    ap = _parser()
    try:
        a = ap.parse_args(argv)
    except _Usage as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except SystemExit as e:  # --help
        return 0 if not e.code else 2
    if not a.verb:
        print("error: a subcommand is required", file=sys.stderr)
        return 2
    try:
        if a.verb == "bench":
            return cmd_bench(a)
        return cmd_solve(a, "pareto" if a.verb == "solve" else a.verb)
    except MorapError as e:
        print(f"error: {e}", file=sys.stderr)
        return exit_code_for(e)


if __name__ == "__main__":
    sys.exit(main())
