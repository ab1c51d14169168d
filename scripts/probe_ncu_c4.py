"""Dev probe for the ncu capture of one compact optimize sweep in the middle of a C4 batch
(10 000 jobs of the 100 x 100 instance, uniform w), frozen-tile skipping on.

    python scripts/probe_ncu_c4.py bytes K   # algorithmic bytes / backups swept by sweep K
    MORAP_GRAPHS=0 ncu --kernel-name regex:k_greedy_sweep_cmp --launch-skip K-1 --launch-count 1 \\
        --set full ... python scripts/probe_ncu_c4.py run K
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2305_04397_b200.api import Instance, Solver  # noqa: E402
from paper_2305_04397_b200.cuda import CudaBackend  # noqa: E402

mode, K = sys.argv[1], int(sys.argv[2])
cfg, thr, eps, _ = bench.workload("c4")
solver = Solver(0)
solver.set_lean(True)
inst = Instance.warehouse_streamed(cfg, solver, chunk=bench.STREAMED["c4"])
be = CudaBackend.__new__(CudaBackend)  # a view of the solver's context (not owned)
be.lib = __import__("paper_2305_04397_b200.cuda", fromlist=["load_library"]).load_library()
be.h = solver.cuda_ctx
be.device = 0
be._models = []
nm = be.lib.morap_cuda_num_models(be.h)
ids = np.arange(nm, dtype=np.int32)
n = cfg["n"]
Wm = np.tile([0.5 / n, 0.5 / n], (nm, 1))
if mode == "run":
    be.optimize(ids, Wm, sweep_cap=K)
else:
    got = []
    for cap in (K - 1, K):
        be.reset_stats()
        be.optimize(ids, Wm, sweep_cap=cap)
        s = be.stats()
        got.append((s["opt_bytes"], s["opt_exec_backups"]))
    print(json.dumps({"workload": "c4", "sweep": K, "jobs": int(nm), "exec_bytes": got[1][0] - got[0][0],
                      "exec_backups": got[1][1] - got[0][1]}))
be.h = None  # the solver owns the context
