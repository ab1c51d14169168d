"""Dev probe: one C2 optimize batch (100 jobs at w = (0.5, 0.5), eps 1e-6) to convergence,
with and without frozen-tile skipping: wall ms of the call, event-timed sweep ms, executed
vs reference backups. Run under ncu for the per-launch split of k_select / the sweep."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.cuda import CudaBackend

import bench

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["skip", "full"]
cfg = bench.workload("c2")[0]
inst = Instance.warehouse(cfg)
prods = [inst.product(i, j) for i in range(10) for j in range(10)]
be = CudaBackend(0)
be.set_lean(True)
ids = be.upload(prods)
Wm = np.tile([0.5, 0.5], (len(ids), 1))
for mode in modes:
    be.set_skip(mode == "skip")
    be.optimize(ids, Wm)
    be.set_profiling(False)
    t0 = time.perf_counter()
    for _ in range(reps):
        val, sw, res, st = be.optimize(ids, Wm)
    wall = (time.perf_counter() - t0) / reps * 1e3
    be.set_profiling(True)
    be.reset_stats()
    for _ in range(reps):
        be.optimize(ids, Wm)
    s = be.stats()
    be.set_profiling(False)
    print(f"{mode}: wall {wall:.2f} ms/call, sweeps max {sw.max()}, launches {s['opt_launches'] / reps:.0f}, "
          f"event ms {s['opt_ms'] / reps:.2f} ({s['opt_ms'] / max(s['opt_launches'], 1) * 1e3:.1f} us/launch), "
          f"exec/ref backups {s['opt_exec_backups'] / s['opt_backups']:.3f}, "
          f"GB/s {s['opt_bytes'] / (s['opt_ms'] * 1e-3) / 1e9:.0f}", flush=True)
