#!/usr/bin/env python
"""Benchmark of the MORAP hot path on B200 (BASELINE.json metric: nnz Bellman backups per
second + Pareto-query wall time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2]

A step is one point-oriented Pareto query (paretoPoint, solver.hpp:281) on the workload
-- default C2 of BASELINE.json configs[1]: 10x10 grid warehouse, 10 agents x 10 tasks,
2 objectives, thresholds (-20 x10, 0.99 x10), eps 0.01 (infeasible; 13 Alg.-1 iterations
of 100 optimize + 20 evaluate jobs each). Synthetic instance from the seeded warehouse
generator (warehouse.hpp:176), built on the host before timing.

  value    nnz backups of the query (sweeps x nnz of every job: the reference's work for the
           same results) / device time of the query, products resident in HBM; the optimize
           sweeps skip frozen tiles (bit-identical results), executed backups are reported too
  e2e      the same metric through the host API with HOST buffers: every step uploads the
           instance's product CSR (H2D) and reads back values/policies (D2H)
  roofline dominant kernel k_greedy_sweep_cmp (compact streams): algorithmic bytes
           (4 nnz + 4 R + 20 S per swept tile) / its CUDA-event time
           over a second pass of the timed steps; traffic from the committed ncu capture
  cpu_baseline  the reference's own engine (oracle/_ref, runBatch over all host threads)
           on one optimize phase of the same instance

Multi-GPU (torchrun, N > 1): products are sharded across ranks (distributed.py); every
rank runs the host loop, values are exchanged by all_gather over NCCL. Reported "weak":
the instance grows with N so that per-GPU work stays ~constant (n = round(10 sqrt(N))).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "transitions/sec (nnz Bellman backups) + Pareto-query wall time at 1/2/4/8 B200 vs CPU"
UNIT = "nnz-backups/s"


# Algorithm-1 iteration cap per workload: C3's 150-dimensional sandwich needs hundreds of
# iterations to close an eps = 0.01 gap, so it is timed per iteration (the paper's own
# metric) over the first 10 iterations.
ITER_CAP = {"c3": 10, "c4": 3, "cent": 5}
# Instances whose host copy does not fit (C4: ~1e4 products, 4.6e9 nnz) are built streamed:
# `chunk` products at a time, uploaded lean (compact alphabet only) and dropped on the host.
STREAMED = {"c4": 256}


def workload(name: str, world: int = 1):
    if name == "c2":
        n = 10 if world == 1 else int(round(10 * math.sqrt(world)))
        W = H = 10
        cfg = {"W": W, "H": H, "n": n, "slip": 0.05,
               "racks": [[W - 1 - (k % W), H - 1 - (k // W)] for k in range(n)], "feed": [0, 0], "seed": 42}
        return cfg, [-20.0] * n + [0.99] * n, 0.01, 2
    if name == "c1":
        cfg = {"W": 6, "H": 6, "n": 2, "slip": 0.05, "racks": [[5, 5], [0, 5], [5, 0]], "feed": [0, 0], "seed": 42}
        return cfg, [-30.0, -36.0, 0.95, 0.8], 0.01, 2
    if name == "c3":  # 50 x 50, 3 objectives, infeasible target
        n, W = 50, 8
        cfg = {"W": W, "H": W, "n": n, "slip": 0.05,
               "racks": [[W - 1 - (k % W), W - 1 - (k // W)] for k in range(n)], "feed": [0, 0], "seed": 42}
        return cfg, [-20.0] * (2 * n) + [0.99] * n, 0.01, 3
    if name == "c4":  # 100 x 100 on a 10 x 10 grid, every cell a rack (~9.4e4 S per product)
        n, W, H = 100, 10, 10
        cfg = {"W": W, "H": H, "n": n, "slip": 0.05,
               "racks": [[W - 1 - (k % W), H - 1 - (k // W)] for k in range(n)], "feed": [0, 0], "seed": 42}
        return cfg, [-20.0] * n + [0.99] * n, 0.01, 2
    if name == "cent":  # centralised model: 6x6 grid, n = 4 agents x 4 tasks
        n, W = 4, 6
        cfg = {"W": W, "H": W, "n": n, "slip": 0.05,
               "racks": [[W - 1 - (k % W), W - 1 - (k // W)] for k in range(n)], "feed": [0, 0], "seed": 42}
        return cfg, [-30.0] * n + [0.9] * n, 0.01, 2
    raise SystemExit(f"unknown workload {name}")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    """DRAM bytes / algorithmic bytes of one sweep launch of this workload, from the committed
    ncu --set full capture (profiles/ncu_traffic.json, one entry per workload)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(workload)
        if d:
            return d.get("traffic_over_algorithmic"), d
    return None, None


# ------------------------------------------------------------------------------------------
def cpu_sample(cfg):
    """Bounded CPU sample of a workload: the whole instance when the reference can hold it,
    else the first 4 agents x 4 tasks of the same grid / racks (the same (i, j < 4) products:
    start poses and tasks do not depend on n, warehouse.hpp:69-84,157-174)."""
    if cfg["n"] <= 50:
        return cfg, "the same instance"
    sub = dict(cfg, n=4)
    return sub, f"its 4 x 4 sub-instance (agents 0-3, tasks 0-3: the same products) of the {cfg['W']}x{cfg['H']} grid"


def cpu_baseline(cfg, thr, eps):
    """The reference's own paretoPoint (oracle/_ref, all host threads) on the same query: one
    whole query timed (solveSeconds), its backups counted on the reference engine."""
    import oracle
    if not oracle.ref_available():
        return None
    ref = oracle.ref()
    sub, what = cpu_sample(cfg)
    n = sub["n"]
    if n != cfg["n"]:
        thr = [thr[0]] * n + [thr[-1]] * n
    inst = ref.warehouse(sub)
    rep = inst.pareto(thr, eps=eps, workers=0)
    ob, eb = inst.query_backups(rep, workers=0)
    threads = ref.hardware_threads()
    return {"value": (ob + eb) / rep["seconds"], "unit": UNIT, "cores": threads, "kind": "reference",
            "pareto_query_ms": 1e3 * rep["seconds"], "pareto_iterations": len(rep["iterations"]),
            "sample": f"oracle/_ref paretoPoint (solver.hpp:281) on {what}, one whole query "
                      f"({len(rep['iterations'])} iterations, {rep['seconds']:.2f} s) on {threads} host threads; "
                      f"backups {ob + eb:.3e} counted on the reference engine"}


REF_BUDGET_S = float(os.environ.get("MORAP_REF_BUDGET_S", "150"))  # timed reference queries per run


def run_reference(args):
    """--impl reference: the reference's own paretoPoint (solver.hpp:281, oracle/_ref built
    from /root/reference) on the same instance and query as our arm, on all host threads.
    A step is one whole query (the reference bench verb's solveSeconds, cli.hpp:304-315:
    instance build excluded). value = the query's nnz backups (optimize sweeps x nnz +
    evaluate sweeps x states, counted once on the reference engine, untimed) / query
    seconds -- the same units as our arm. The run is bounded: one warm-up query, then as
    many of the --steps queries as fit in REF_BUDGET_S seconds (at least one)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg, thr, eps, K = workload(args.workload, world)
    line = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": args.gpus, "warmup": args.warmup,
            "higher_is_better": True}
    if not oracle.ref_available():
        line["unavailable"] = "oracle/_ref/libmorap_ref.so was not built (needs /root/reference at build time)"
        print(json.dumps(line))
        return
    if K != 2 or cfg["n"] > 50:
        line["unavailable"] = (f"the reference has no K={K} objectives" if K != 2 else
                               f"the reference cannot hold the {cfg['n']}x{cfg['n']} instance in host memory")
        print(json.dumps(line))
        return
    ref = oracle.ref()
    n = cfg["n"]
    t0 = time.time()
    inst = ref.warehouse(cfg)
    gen = time.time() - t0
    threads = ref.hardware_threads()
    rep = inst.pareto(thr, eps=eps, workers=0)  # warm-up query (its report gives the work count)
    first_s = rep["seconds"]
    ob, eb = inst.query_backups(rep, workers=0)
    backups = ob + eb
    steps = max(1, min(args.steps, int(REF_BUDGET_S // max(first_s, 1e-3))))
    secs = []
    for _ in range(steps):
        r = inst.pareto(thr, eps=eps, workers=0)
        assert r["tDown"] == rep["tDown"] and len(r["iterations"]) == len(rep["iterations"])
        secs.append(r["seconds"])
    q = sum(secs) / len(secs)
    value = backups / q
    line.update({
        "value": value, "steps": steps, "ms_per_step": 1e3 * q, "pareto_query_ms": 1e3 * q, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded warehouse generator, warehouse.hpp:176)",
        "config": {"workload": args.workload, "grid": [cfg["W"], cfg["H"]], "agents": n, "tasks": n, "objectives": K,
                   "eps": eps, "thresholds": f"costs {thr[0]} x{n}, probs {thr[-1]}",
                   "feasible": rep["feasible"], "pareto_iterations": len(rep["iterations"]),
                   "step": "one paretoPoint query (solver.hpp:281) on the reference's CPU engine, instance build "
                           "excluded (cli.hpp:304-315 solveSeconds)",
                   "steps_requested": args.steps, "bounded": f"{steps} timed queries within {REF_BUDGET_S:.0f} s",
                   "generate_s": round(gen, 3)},
        "backups_per_query": {"optimize": ob, "evaluate_states": eb},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{steps} whole paretoPoint queries ({len(rep['iterations'])} iterations of "
                                   f"{n * n} optimize + {2 * n} evaluate jobs) on {threads} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })
    print(json.dumps(line))


# ------------------------------------------------------------------------------------------
def run_centralised(args):
    """--workload cent: centralisedParetoPoint (centralised.hpp:216) on one large model, the
    first ITER_CAP iterations, against the reference's own centralised solver on the host."""
    import torch
    import oracle
    from paper_2305_04397_b200.api import Centralised, Instance, Solver
    cfg, thr, eps, K = workload("cent", 1)
    cap = ITER_CAP["cent"]
    t0 = time.time()
    inst = Instance.warehouse(cfg)
    cm = Centralised(inst)
    gen_s = time.time() - t0
    solver = Solver(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    solver.set_stream(stream.cuda_stream)
    for _ in range(max(args.warmup, 0)):
        rep = solver.centralised_pareto(cm, thr, eps=eps, iteration_cap=cap)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    backups = 0.0
    with ClockSampler(0) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            rep = solver.centralised_pareto(cm, thr, eps=eps, iteration_cap=cap)
            backups += rep["stats"]["optimize_backups"] + rep["stats"]["evaluate_state_backups"]
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    iters = len(rep["iterations"])
    cpu = None
    if oracle.ref_available() and not args.no_cpu_baseline:
        r = oracle.ref().warehouse(cfg).centralised_pareto(thr, eps=eps, iter_cap=cap)
        cpu = {"value": r["seconds"] / len(r["iterations"]) * 1e3, "unit": "ms per iteration", "cores": 1,
               "kind": "reference", "sample": f"oracle/_ref centralisedParetoPoint, same model, first {cap} iterations"}
        assert r["tDown"] == rep["tDown"], "centralised query differs from the reference"
    print(json.dumps({
        "metric": METRIC, "value": backups / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded warehouse generator, warehouse.hpp:176)",
        "config": {"workload": "cent", "grid": [cfg["W"], cfg["H"]], "agents": cfg["n"], "tasks": cfg["n"],
                   "model": {"states": cm.S, "rows": cm.R, "nnz": cm.nnz, "objectives": cm.objectives},
                   "pareto_iterations": iters, "ms_per_iteration": ms / args.steps / iters,
                   "step": f"centralisedParetoPoint, first {cap} iterations", "generate_s": round(gen_s, 3)},
        "cpu_baseline": cpu, "clocks": clk.summary()}))


def query_pass(solver, inst, thr, eps, cap, steps, stream, profiling=False):
    """`steps` paretoPoint queries with the products resident, device-timed on `stream`."""
    import torch
    solver.set_profiling(profiling)
    solver.reset_cuda_stats()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    backups, reps = 0.0, []
    phase = {"optimize_s": 0.0, "evaluate_s": 0.0, "host_s": 0.0}
    e0.record(stream)
    for _ in range(steps):
        rep = solver.pareto(inst, thr, eps=eps, iteration_cap=cap)
        st = rep["stats"]
        backups += st["optimize_backups"] + st["evaluate_state_backups"]
        for k in phase:
            phase[k] += st[k] / steps
        reps.append(rep)
    e1.record(stream)
    torch.cuda.synchronize()
    cs = solver.cuda_stats()
    solver.set_profiling(False)
    return {"ms": e0.elapsed_time(e1), "backups": backups, "reports": reps, "phase": phase, "cuda": cs}


def roofline(cs, prof_ms, workload_name, inst):
    """Roofline of the dominant kernel (k_greedy_sweep_cmp) from a profiling pass: algorithmic
    bytes of the swept tiles / the CUDA-event time of its launches."""
    peak, peak_src = peak_hbm()
    achieved = cs["opt_bytes"] / (cs["opt_ms"] * 1e-3) / 1e9 if cs["opt_ms"] > 0 else None
    N, R, S = inst.total_nnz, inst.total_rows, inst.total_states
    survey_ratio = (12 * N + 12 * R + 21 * S) / (4 * N + 4 * R + 20 * S)
    ratio, tsrc = ncu_traffic(workload_name)
    alg_per_launch = cs["opt_bytes"] / max(cs["opt_launches"], 1)
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None,
            "traffic": ratio * alg_per_launch if ratio else None,
            "kernel": "k_greedy_sweep_cmp", "workload": workload_name, "launches": cs["opt_launches"],
            "traffic_over_algorithmic": ratio, "traffic_source": tsrc and tsrc.get("source"),
            "avg_launch_us": 1e3 * cs["opt_ms"] / max(cs["opt_launches"], 1),
            "algorithmic_bytes_per_launch": alg_per_launch,
            "kernel_exec_backups_per_s": cs["opt_exec_backups"] / (cs["opt_ms"] * 1e-3) if cs["opt_ms"] else None,
            "skipped_fraction": 1.0 - cs["opt_exec_backups"] / max(cs["opt_backups"], 1.0),
            "peak_source": peak_src,
            "timing": "CUDA events around every sweep-kernel launch (k_select outside them), in a separate "
                      f"profiling pass ({prof_ms:.1f} ms per query with the events)",
            "share_of_step": cs["opt_ms"] / prof_ms if prof_ms else None,
            "survey_8d": {"bytes_per_backup": (12 * N + 12 * R + 21 * S) / N,
                          "frac": achieved * survey_ratio / peak if achieved else None,
                          "note": "the same launches counted with SURVEY.md §8(d)'s reference-layout bytes "
                                  "(12 nnz + 12 R + 21 S); > 1 means the compact layout moves fewer bytes than "
                                  "the reference layout would at this rate"}}


NS_ITERS = 8  # Algorithm-1 iterations of the C4 north-star leg timed inside the default run


def north_star(args, local):
    """BASELINE north_star: the point-oriented query on 100 agents x 100 tasks on one B200.
    Builds C4 with the device product builder, times its first NS_ITERS Algorithm-1 iterations with
    the products resident, and reports s/iteration, nnz-backups/s and the sweep kernel's
    roofline at C4; the full query to convergence is a committed run (profiles/)."""
    import torch
    from paper_2305_04397_b200.api import Instance, Solver
    cfg, thr, eps, K = workload("c4", 1)
    solver = Solver(local)
    solver.set_fingerprints(False)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    solver.set_stream(stream.cuda_stream)
    solver.set_lean(True)
    t0 = time.time()
    inst = Instance.warehouse_device(cfg, solver)  # device product builder
    build_s = time.time() - t0
    solver.pareto(inst, thr, eps=eps, iteration_cap=1)  # warm-up
    run = query_pass(solver, inst, thr, eps, NS_ITERS, 1, stream)
    prof = query_pass(solver, inst, thr, eps, NS_ITERS, 1, stream, profiling=True)
    rep = run["reports"][0]
    it = len(rep["iterations"])
    out = {"workload": "c4", "grid": [cfg["W"], cfg["H"]], "agents": cfg["n"], "tasks": cfg["n"],
           "products": inst.distinct, "states": inst.total_states, "nnz": inst.total_nnz,
           "build_s": round(build_s, 2), "builder": "device (morap_instance_warehouse_device)",
           "step": f"the first {it} Algorithm-1 iterations of paretoPoint (thresholds -20 x100, 0.99 x100, eps 0.01), "
                   "products resident (device-built lean compact models)",
           "s_per_iteration": run["ms"] * 1e-3 / it, "value": run["backups"] / (run["ms"] * 1e-3), "unit": UNIT,
           "phase_s_per_iteration": {k: v / it for k, v in run["phase"].items()},
           "roofline": roofline(prof["cuda"], prof["ms"], "c4", inst)}
    full = os.path.join(ROOT, "profiles", "r02_c4_full_query.json")
    if os.path.exists(full):
        out["full_query"] = json.load(open(full))
    solver.close()
    return out


def run_ours(args):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload == "cent":
        return run_centralised(args)
    if world > 1 or args.sharded:
        from paper_2305_04397_b200 import distributed
        return distributed.bench_main(args, rank, world, local)
    from paper_2305_04397_b200.api import Instance, Solver

    torch.cuda.set_device(local)
    cfg, thr, eps, K = workload(args.workload, 1)
    cap = ITER_CAP.get(args.workload, 500)
    streamed = STREAMED.get(args.workload)
    image_s = None
    solver = Solver(local)
    solver.set_fingerprints(False)  # scheduler hashes are test evidence, not part of paretoPoint
    stream = torch.cuda.Stream()  # the library launches on this stream; the CUDA events below are recorded on it
    torch.cuda.set_stream(stream)
    solver.set_stream(stream.cuda_stream)
    t0 = time.time()
    if streamed:  # C4: too large for a host copy -- the products are built on the device
        inst = Instance.warehouse_device(cfg, solver)
    else:
        inst = Instance.warehouse(cfg)
        if K > 2:
            inst.add_objectives(K, seed=7)
        t1 = time.time()
        solver.upload(inst)  # first upload: the product builder's packed image + its copy
        image_s = time.time() - t1
    gen_s = time.time() - t0
    for _ in range(max(args.warmup, 0)):
        solver.pareto(inst, thr, eps=eps, iteration_cap=cap)

    # ---- device-resident timed region (clocks sampled during it) -------------------------
    with ClockSampler(local) as clk:
        run = query_pass(solver, inst, thr, eps, cap, args.steps, stream)
    ms, cs = run["ms"], run["cuda"]
    kernels_timed = int(cs["kernels"])
    value = run["backups"] / (ms * 1e-3)
    first = run["reports"][0]
    assert all(r["tDown"] == first["tDown"] and r["records"] == first["records"] for r in run["reports"]), \
        "queries of the timed region differ"

    # ---- the same steps again with CUDA events around every sweep launch (roofline) -----
    prof = query_pass(solver, inst, thr, eps, cap, args.steps, stream, profiling=True)

    # ---- end to end through the host API with host buffers (every step) ------------------
    e2e = None
    if not streamed:  # a streamed instance has no host copy to re-upload
        solver.reset_cuda_stats()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_backups = 0.0
        e0.record(stream)
        for _ in range(args.steps):
            solver.release()
            solver.upload(inst)
            rep = solver.pareto(inst, thr, eps=eps, iteration_cap=cap)
            e_backups += rep["stats"]["optimize_backups"] + rep["stats"]["evaluate_state_backups"]
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        ecs = solver.cuda_stats()
        e2e = {"value": e_backups / (e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": ecs["upload_bytes"] / args.steps,
               "d2h_bytes_per_step": ecs["d2h_bytes"] / args.steps, "steps": args.steps,
               "ms_per_step": e_ms / args.steps, "pareto_query_ms": e_ms / args.steps,
               "what": "release + re-upload of the instance's products from host memory -- the product "
                       "builder's packed device image (validated, tiled, compact streams; built once per "
                       "instance on the host threads, pinned) in one H2D copy -- then the query and every "
                       "result read (D2H), per step; bytes counted by the library's copy calls",
               "first_upload_s": round(image_s, 4) if image_s is not None else None}
    else:
        e2e = {"value": None, "unit": UNIT, "note": f"products built on the device ({gen_s:.1f} s, "
                                                   f"morap_instance_warehouse_device); no host copy to re-upload"}

    iters = len(first["iterations"])
    rl = roofline(prof["cuda"], prof["ms"], args.workload, inst)
    cpu = None if args.no_cpu_baseline or K != 2 else cpu_baseline(cfg, thr, eps)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded warehouse generator, warehouse.hpp:176; built before timing)",
        "config": {"workload": args.workload, "grid": [cfg["W"], cfg["H"]], "agents": cfg["n"], "tasks": cfg["n"],
                   "objectives": K, "eps": eps, "thresholds": f"costs {thr[0]} x{(K - 1) * cfg['n']}, probs {thr[-1]}",
                   "feasible": first["feasible"], "converged": first["converged"], "pareto_iterations": iters,
                   "products": inst.distinct, "states": inst.total_states, "nnz": inst.total_nnz,
                   "step": "one paretoPoint query (Alg. 1, solver.hpp:281) with products resident in HBM",
                   "l2": "inputs larger than L2 (product streams > 126 MB)",
                   "generate_s": round(gen_s, 3), "parallelism": "single GPU"},
        "value_executed": cs["opt_exec_backups"] / (ms * 1e-3) + 0.0,
        "value_note": "value counts sweeps x nnz of every optimize job plus evaluate sweeps x states (the "
                      "reference's work for the same, bitwise-identical results); value_executed counts only "
                      "the optimize backups the device executed (frozen tiles are skipped) per second of query",
        "pareto_query_ms": ms / args.steps,
        "roofline": rl,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clk.summary(),
        "gpu_launches": kernels_timed,
        "phase_s_per_query": run["phase"],
        "kernel_stats": cs,
    }
    if not args.no_north_star and args.workload == "c2":
        line["north_star"] = north_star(args, local)
    if rank == 0:
        print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-north-star", action="store_true", help="skip the C4 north-star leg of the default run")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (sharded, NCCL) path even on one rank (testing)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
