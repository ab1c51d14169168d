"""Dev probe for the ncu capture of one compact optimize sweep in the middle of a C2 batch
(100 jobs, w = (0.5, 0.5)), frozen-tile skipping on.

    python scripts/probe_ncu_sweep.py bytes K   # algorithmic bytes swept by sweep K (stats diff)
    MORAP_GRAPHS=0 ncu --kernel-name regex:k_greedy_sweep_cmp --launch-skip K-1 --launch-count 1 \\
        --set full ... python scripts/probe_ncu_sweep.py run K
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.cuda import CudaBackend

mode, K = sys.argv[1], int(sys.argv[2])
inst = Instance.warehouse(bench.workload("c2")[0])
prods = [inst.product(i, j) for i in range(10) for j in range(10)]
be = CudaBackend(0)
be.set_lean(True)
ids = be.upload(prods)
Wm = np.tile([0.5, 0.5], (len(ids), 1))
if mode == "run":
    be.optimize(ids, Wm, sweep_cap=K)
else:
    got = []
    for cap in (K - 1, K):
        be.reset_stats()
        be.optimize(ids, Wm, sweep_cap=cap)
        s = be.stats()
        got.append((s["opt_bytes"], s["opt_exec_backups"]))
    print(json.dumps({"sweep": K, "exec_bytes": got[1][0] - got[0][0], "exec_backups": got[1][1] - got[0][1]}))
