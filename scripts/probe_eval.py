"""Dev probe: time the pieces of one supporting-point query on C2 through the CUDA ABI."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.cuda import CudaBackend
from tests.helpers import warehouse_config

inst = Instance.warehouse(warehouse_config(10, 10, 10))
prods = [inst.product(i, j) for i in range(10) for j in range(10)]
be = CudaBackend(0)
ids = be.upload(prods)
W = np.tile([0.35, 0.65], (100, 1))
for rep in range(4):
    t0 = time.perf_counter(); val, sw, res, st = be.optimize(ids, W); t1 = time.perf_counter()
    jobs = list(range(0, 100, 11))[:10]
    ev = be.evaluate_optimized(jobs, (0, 1)); t2 = time.perf_counter()
    for j in jobs: be.fetch_policy(j)
    t3 = time.perf_counter()
    be.set_profiling(True); be.reset_stats()
    ev = be.evaluate_optimized(jobs, (0, 1)); t4 = time.perf_counter()
    s = be.stats(); be.set_profiling(False)
    print(json.dumps(dict(opt_ms=(t1-t0)*1e3, eval_ms=(t2-t1)*1e3, fetch_ms=(t3-t2)*1e3, eval_prof_ms=(t4-t3)*1e3,
          eval_kernel_ms=s['eval_ms'], eval_launches=s['eval_launches'], kernels=s['kernels'], eval_sweeps=int(ev[1].max()))), flush=True)
