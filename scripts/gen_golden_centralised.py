"""Golden vectors for the centralised model (centralised.hpp) from the reference itself.

    python scripts/gen_golden_centralised.py     # needs /root/reference (oracle/_ref)

Writes tests/golden/centralised.json: for fig2 and the warehouse-suite runs, sha256 of every
array buildCentralised produces (centralised.hpp:54-179) and the centralisedParetoPoint
report (:216-222) for the run's thresholds. Committed, so the GPU box needs no reference."""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fingerprint(c: dict) -> dict:
    out = {k: sha(c[k]) for k in ("rowOffset", "trnOffset", "succ", "prob", "done", "rewards")}
    out.update(S=int(c["rowOffset"].shape[0] - 1), R=int(c["trnOffset"].shape[0] - 1), nnz=int(c["succ"].shape[0]),
               rewardFinite=c["rewardFinite"])
    return out


def main():
    ref = oracle.ref()
    fig2 = open(os.path.join(GOLD, "fig2.json")).read()
    suite = json.load(open(os.path.join(GOLD, "warehouse_suite.json")))["runs"]
    out = {"fig2": [], "suite": []}
    I = ref.from_json(fig2)
    out["fig2_model"] = fingerprint(I.centralised())
    for thr, eps in [([-1.8, 0.9], 1e-4), ([-2.5, 0.7], 1e-3), ([-1.8, 0.9], 0.01)]:
        res = ref.from_json(fig2).centralised_pareto(thr, eps=eps)
        res.pop("seconds")
        out["fig2"].append({"thresholds": thr, "eps": eps, "result": res})
    for run in suite:
        if run["config"]["n"] > 2:
            continue
        I = ref.warehouse(run["config"])
        t0 = time.time()
        res = I.centralised_pareto(run["thresholds"], eps=run.get("eps", 0.01))
        sec = res.pop("seconds")
        out["suite"].append({"config": run["config"], "thresholds": run["thresholds"], "eps": run.get("eps", 0.01),
                             "model": fingerprint(I.centralised()), "result": res, "reference_seconds": sec})
        print(run["config"]["W"], run["config"]["n"], f"{time.time() - t0:.1f}s", flush=True)
    json.dump(out, open(os.path.join(GOLD, "centralised.json"), "w"), indent=1)
    print("written", os.path.join(GOLD, "centralised.json"))


if __name__ == "__main__":
    main()
