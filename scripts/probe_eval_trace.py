"""Dev probe: per-sweep timeline of the persistent evaluate kernel (k_eval_persistent) on the
C2 evaluate batch of one Pareto iteration (10 assigned products, 2 RHS), from globaltimer
stamps per CTA (morap_cuda_debug_cta_trace): compute span (first start -> last CTA done),
barrier (last CTA done -> last CTA through the barrier) and decision step."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2305_04397_b200.api import Instance  # noqa: E402
from paper_2305_04397_b200.cuda import CudaBackend  # noqa: E402

cfg = bench.workload("c2")[0]
inst = Instance.warehouse(cfg)
n = cfg["n"]
prods = [inst.product(i, j) for i in range(n) for j in range(n)]
be = CudaBackend(0)
be.set_lean(True)
ids = be.upload(prods)
W = np.tile([0.5, 0.5], (len(ids), 1))
be.optimize(ids, W)
pairs = [i * n + i for i in range(n)]  # the identity assignment: 10 optimize jobs' policies
be.evaluate_optimized(pairs, (0, 1))
lib = be.lib
slots, blocks = 128, 592
buf = np.zeros(slots * blocks * 4, np.uint64)
assert lib.morap_cuda_debug_cta_trace(be.h, 1, None, 0) == 0
ev, esw, eres, est = be.evaluate_optimized(pairs, (0, 1))
assert lib.morap_cuda_debug_cta_trace(be.h, -1, buf.ctypes.data_as(C.c_void_p), buf.size) == 0
lib.morap_cuda_debug_cta_trace(be.h, 0, None, 0)
nb = 148
sweeps = int(esw.max())
t = buf.reshape(slots, blocks, 4)[:, :nb, :].astype(np.int64)
rows = []
for k in range(min(sweeps, slots)):
    s = t[k]
    if s[:, 0].min() == 0:
        continue
    t0 = s[:, 0].min()
    rows.append(((s[:, 1].max() - t0), (s[:, 2].max() - s[:, 1].max()), (s[:, 3].max() - s[:, 2].max()),
                 (s[:, 3].max() - t0), np.median(s[:, 1] - s[:, 0])))
r = np.array(rows, np.float64) / 1e3
print(json.dumps({"sweeps": sweeps, "traced": len(rows),
                  "mean_us": {"compute_span": r[:, 0].mean(), "barrier": r[:, 1].mean(), "decide": r[:, 2].mean(),
                              "sweep_total": r[:, 3].mean(), "median_cta_compute": r[:, 4].mean()},
                  "first5": r[:5].round(2).tolist(), "last5": r[-5:].round(2).tolist()}))
