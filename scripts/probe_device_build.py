"""Dev probe: C4 (or another bench workload) built with the device product builder; prints the
build time and, optionally, the first iterations of the query (python scripts/probe_device_build.py c4 2)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2305_04397_b200.api import Instance, Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg, thr, eps, K = bench.workload(name)
s = Solver(0)
s.set_fingerprints(False)
t = time.time()
inst = Instance.warehouse_device(cfg, s)
build = time.time() - t
out = {"workload": name, "device_build_s": round(build, 3), "products": inst.distinct, "states": inst.total_states,
       "nnz": inst.total_nnz}
if iters:
    t = time.time()
    rep = s.pareto(inst, thr, eps=eps, iteration_cap=iters)
    out["iterations"] = len(rep["iterations"])
    out["query_s"] = round(time.time() - t, 3)
    out["w_last"] = rep["iterations"][-1].get("w", [])[:4]
print(json.dumps(out))
