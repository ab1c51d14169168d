"""Dev probe: one full point-oriented query (to convergence or a cap) on a large workload,
printing per-iteration progress, the verdict and the phase split.

    python scripts/probe_full_query.py c4 [cap] [device]
(device: products built by the device product builder instead of the host)
"""
import json
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2305_04397_b200.api import Instance, Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 500
cfg, thr, eps, K = bench.workload(name)
s = Solver(0)
s.set_fingerprints(False)
t = time.time()
if len(sys.argv) > 3 and sys.argv[3] == "device":
    inst = Instance.warehouse_device(cfg, s)
elif name in bench.STREAMED:
    s.set_lean(True)
    inst = Instance.warehouse_streamed(cfg, s, chunk=bench.STREAMED[name])
else:
    inst = Instance.warehouse(cfg)
    if K > 2:
        inst.add_objectives(K, seed=7)
    s.upload(inst)
print("build+upload", round(time.time() - t, 2), "s", inst.distinct, "products", inst.total_nnz, "nnz", flush=True)
t = time.time()
r = s.pareto(inst, thr, eps=eps, iteration_cap=cap)
q = time.time() - t
it = r["iterations"]
print(json.dumps({"workload": name, "query_s": q, "iterations": len(it), "converged": r["converged"],
                  "feasible": r["feasible"], "s_per_iteration": q / max(len(it), 1), "stats": r["stats"],
                  }), flush=True)
# the supporting points of every iteration, for an offline replay of the sandwich loop
# (scripts/replay_sandwich.py: same weight sequence from the reference's geometry)
import numpy as np  # noqa: E402
import os  # noqa: E402
gold = f"tests/golden/replay/{name}_query.npz"  # the round-2 recording (GPU run, replayed on the reference)
if os.path.exists(gold):
    z = np.load(gold)
    same = {k: np.array(v).tobytes() == z[k].tobytes() for k, v in
            (("w", [x["w"] for x in it]), ("r", [x["r"] for x in it]), ("tUp", r["tUp"]), ("tDown", r["tDown"]),
             ("lambdaStar", r["lambdaStar"]))}
    print(json.dumps({"same_as_recorded_query": same, "builder": sys.argv[3] if len(sys.argv) > 3 else "host"}),
          flush=True)
np.savez_compressed(f"gpurun_out/report_{name}.npz", thresholds=np.array(r["thresholds"]),
                    w=np.array([x["w"] for x in it]), r=np.array([x["r"] for x in it]),
                    assignment=np.array([x["assignment"] for x in it], dtype=np.int32),
                    tUp=np.array(r["tUp"]), tDown=np.array(r["tDown"]), lambdaStar=np.array(r["lambdaStar"]),
                    eps=eps, n=cfg["n"], converged=r["converged"], feasible=r["feasible"])
