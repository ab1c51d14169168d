"""Dev probe: per-launch time of the optimize sweep kernel with every C2 job active.
Each optimize call runs exactly one sweep (sweep_cap=1) over all 100 products, timed with
CUDA events (profiling on); prints the mean over calls. MORAP_CUDA_SO picks a variant."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.cuda import CudaBackend

W = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
racks = [[W - 1 - (k % W), W - 1 - (k // W)] for k in range(n)]
inst = Instance.warehouse({"W": W, "H": W, "n": min(n, 10), "slip": 0.05, "racks": racks, "feed": [0, 0], "seed": 42})
m = min(n, 10)
prods = [inst.product(i, j) for i in range(m) for j in range(m)]
be = CudaBackend(0)
ids = be.upload(prods)
Wm = np.tile([0.5, 0.5], (len(ids), 1))
be.optimize(ids, Wm, sweep_cap=3)
be.set_profiling(True)
be.reset_stats()
for _ in range(reps):
    be.optimize(ids, Wm, sweep_cap=3)
s = be.stats()
nnz = sum(p.nnz for p in prods)
us = 1e3 * s["opt_ms"] / s["opt_launches"]
print(json.dumps({"so": os.path.basename(os.environ.get("MORAP_CUDA_SO", "default")), "dry": os.environ.get("MORAP_DEBUG_DRY", "0"),
                  "us_per_launch": us, "launches": s["opt_launches"], "nnz": nnz,
                  "backups_per_s": nnz / (us * 1e-6), "alg_GBps": s["opt_bytes"] / (s["opt_ms"] * 1e-3) / 1e9}))
