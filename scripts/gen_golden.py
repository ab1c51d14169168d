"""Generate tests/golden/ from the reference itself (oracle/_ref, built from
/root/reference by oracle/Makefile). Run in the build container:

    python scripts/gen_golden.py              # everything
    python scripts/gen_golden.py --measured   # only the C2 / C4 goldens (c2.json, c4_sub4.json)

Everything written here is a reference OUTPUT (plus two copies of the reference's own data
fixtures, proj/data/fig2.json and warehouse_suite.json), so the GPU box -- which has no
/root/reference -- can check parity against it.
"""
import hashlib
import json
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
DATA = "/root/reference/proj/data"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def product_fp(p) -> dict:
    return {"S": p.S, "R": p.R, "nnz": p.nnz, "initial": p.initial, "rewardFinite": p.rewardFinite,
            **{k: sha(getattr(p, k)) for k in ["rowOffset", "trnOffset", "succ", "prob", "cost", "success", "done",
                                                "accept"]}}


def bench_cfg(name):
    sys.path.insert(0, ROOT)
    import bench
    return bench.workload(name)


def measured_configs():
    """Goldens at the configurations bench.py measures (BASELINE.json configs[1], [3]):
    C2 -- every product fingerprint plus the whole paretoPoint report of the bench query
    (10x10, n = 10, thresholds (-20 x10, 0.99 x10), eps 0.01: 13 iterations, infeasible);
    C4 -- the 4 x 4 sub-instance of the C4 grid (agents 0-3, tasks 0-3: the start poses and
    tasks do not depend on n, warehouse.hpp:69-84,157-174, so these are C4's (i, j < 4)
    products): product fingerprints, optimize / evaluate fingerprints at two weights, and
    the Pareto query with C4's thresholds."""
    ref = oracle.ref()
    cfg, thr, eps, K = bench_cfg("c2")
    I = ref.warehouse(cfg)
    out = {"config": cfg, "products": [[product_fp(I.product(i, j)) for j in range(I.n)] for i in range(I.n)]}
    rep = I.pareto(thr, eps=eps, workers=0)
    rep.pop("seconds")
    out["pareto"] = {"thresholds": thr, "eps": eps, "result": rep}
    json.dump(out, open(os.path.join(GOLD, "c2.json"), "w"), indent=0)

    cfg, thr, eps, K = bench_cfg("c4")
    sub = dict(cfg, n=4)
    I = ref.warehouse(sub)
    out = {"config": sub, "products": [[product_fp(I.product(i, j)) for j in range(4)] for i in range(4)]}
    jobs = []
    for i in range(4):
        for j in range(4):
            for (wc, ws) in [(0.125, 0.125), (0.03125, 0.21875)]:
                rc, v, p, sw, r, v0 = I.optimize(i, j, wc, ws)
                ev = []
                for which in (0, 1):
                    erc, evv, es, er, ev0 = I.evaluate(i, j, p, which)
                    ev.append({"value": ev0, "sweeps": es, "residual": er, "values": sha(evv)})
                jobs.append({"i": i, "j": j, "w": [wc, ws], "rc": rc, "value": v0, "sweeps": sw, "residual": r,
                             "values": sha(v), "policy": sha(p), "evaluate": ev})
    out["jobs"] = jobs
    t4 = [thr[0]] * 4 + [thr[-1]] * 4
    rep = I.pareto(t4, eps=eps, workers=0)
    rep.pop("seconds")
    out["pareto"] = {"thresholds": t4, "eps": eps, "result": rep}
    json.dump(out, open(os.path.join(GOLD, "c4_sub4.json"), "w"), indent=0)


def main():
    os.makedirs(GOLD, exist_ok=True)
    if "--measured" in sys.argv:
        measured_configs()
        print("golden (measured configs) written to", GOLD)
        return
    shutil.copy(os.path.join(DATA, "fig2.json"), os.path.join(GOLD, "fig2.json"))
    shutil.copy(os.path.join(DATA, "warehouse_suite.json"), os.path.join(GOLD, "warehouse_suite.json"))
    ref = oracle.ref()
    fig2 = open(os.path.join(DATA, "fig2.json")).read()
    suite = json.load(open(os.path.join(DATA, "warehouse_suite.json")))["runs"]

    # products: fig2 and the suite configs (the bench configurations: measured_configs)
    prods = {}
    inst = ref.from_json(fig2)
    prods["fig2"] = [[product_fp(inst.product(0, 0))]]
    configs = {}
    for run in suite:
        key = json.dumps(run["config"], sort_keys=True)
        configs[key] = run["config"]
    for key, cfg in configs.items():
        I = ref.warehouse(cfg)
        prods[key] = [[product_fp(I.product(i, j)) for j in range(I.n)] for i in range(I.n)]
    json.dump(prods, open(os.path.join(GOLD, "products.json"), "w"), indent=1)

    # optimize / evaluate results on the 6x6 n=2 products (bitwise fingerprints)
    cfg = suite[3]["config"]
    I = ref.warehouse(cfg)
    opt = []
    for i in range(2):
        for j in range(2):
            for (wc, ws) in [(1.0, 0.0), (0.0, 1.0), (0.3, 0.7), (0.5, 0.5), (0.125, 0.375)]:
                rc, v, p, s, r, v0 = I.optimize(i, j, wc, ws)
                ev = []
                for which in (0, 1):
                    erc, evv, es, er, ev0 = I.evaluate(i, j, p, which)
                    ev.append({"value": ev0, "sweeps": es, "residual": er, "values": sha(evv)})
                opt.append({"i": i, "j": j, "w": [wc, ws], "rc": rc, "value": v0, "sweeps": s, "residual": r,
                            "values": sha(v), "policy": sha(p), "evaluate": ev})
    json.dump({"config": cfg, "jobs": opt}, open(os.path.join(GOLD, "optimize_6x6_n2.json"), "w"), indent=1)

    # Pareto queries: fig2 worked example + the whole warehouse suite
    par = {"fig2": []}
    for thr, eps in [([-1.8, 0.9], 1e-4), ([-2.5, 0.7], 1e-3), ([-1e6, 0.0], 1e-3), ([-1.8, 0.9], 0.01)]:
        out = ref.from_json(fig2).pareto(thr, eps=eps, workers=2)
        out.pop("seconds")
        par["fig2"].append({"thresholds": thr, "eps": eps, "result": out})
    par["fig2_verify"] = []
    for thr in ([-2.5, 0.7], [-1.8, 0.9]):
        v = ref.from_json(fig2).pareto(thr, eps=1e-3, workers=2, verify=True)
        par["fig2_verify"].append({"thresholds": thr, "eps": 1e-3, "verdict": v["verdict"]})
    par["suite"] = []
    for run in suite:
        I = ref.warehouse(run["config"])
        out = I.pareto(run["thresholds"], eps=run.get("eps", 0.01), workers=0)
        out.pop("seconds")
        par["suite"].append({"config": run["config"], "thresholds": run["thresholds"], "eps": run.get("eps", 0.01),
                             "result": out})
    json.dump(par, open(os.path.join(GOLD, "pareto.json"), "w"), indent=1)
    measured_configs()
    print("golden written to", GOLD)


if __name__ == "__main__":
    main()
