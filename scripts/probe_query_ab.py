"""Dev probe: C2 bench query timing (run with MORAP_FLOW=0 / 1 for the A/B of the dataflow
optimize batch). Prints ms per query, phase split and the sweep kernel's achieved rate."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_04397_b200.api import Instance, Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg, thr, eps, K = bench.workload(name)
cap = bench.ITER_CAP.get(name, 500)
s = Solver(0)
if name in bench.STREAMED:
    s.set_lean(True)
    inst = Instance.warehouse_streamed(cfg, s, chunk=bench.STREAMED[name])
else:
    inst = Instance.warehouse(cfg)
    if K > 2:
        inst.add_objectives(K, seed=7)
    s.upload(inst)
rep = s.pareto(inst, thr, eps=eps, iteration_cap=cap)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(steps):
    rep = s.pareto(inst, thr, eps=eps, iteration_cap=cap)
torch.cuda.synchronize()
ms = (time.perf_counter() - t) * 1e3 / steps
s.set_profiling(True)
s.reset_cuda_stats()
rep2 = s.pareto(inst, thr, eps=eps, iteration_cap=cap)
cs = s.cuda_stats()
peak = 6553.9
print(json.dumps({"workload": name, "flow": os.environ.get("MORAP_FLOW", "1"), "ms_per_query": ms,
                  "iterations": len(rep["iterations"]), "stats": rep["stats"],
                  "opt_kernel_ms": cs["opt_ms"], "opt_launches": cs["opt_launches"],
                  "opt_GBps": cs["opt_bytes"] / max(cs["opt_ms"], 1e-9) / 1e6,
                  "frac": cs["opt_bytes"] / max(cs["opt_ms"], 1e-9) / 1e6 / peak,
                  "exec_backups": cs["opt_exec_backups"], "backups": cs["opt_backups"],
                  "same": rep2["tDown"] == rep["tDown"] and rep2["records"] == rep["records"]}), flush=True)
