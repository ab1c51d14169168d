"""Dev probe: persistent evaluate kernel time per sweep against the batch size (1-20 C2 jobs)."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.cuda import CudaBackend
from tests.helpers import warehouse_config
inst = Instance.warehouse(warehouse_config(10, 10, 10))
prods = [inst.product(i, j) for i in range(10) for j in range(10)]
be = CudaBackend(0)
ids = be.upload(prods)
W = np.tile([0.35, 0.65], (100, 1))
be.optimize(ids, W)
for nj in (1, 2, 5, 10, 20):
    jobs = list(range(0, 100, 100 // nj))[:nj]
    be.evaluate_optimized(jobs, (0, 1))
    be.set_profiling(True); be.reset_stats()
    ev = be.evaluate_optimized(jobs, (0, 1))
    s = be.stats(); be.set_profiling(False)
    sw = int(np.max(ev[1]))
    print(nj, "jobs: kernel ms %.3f, sweeps %d, us/sweep %.1f" % (s['eval_ms'], sw, 1e3 * s['eval_ms'] / sw))
