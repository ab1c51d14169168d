"""Dev probe: centralised Pareto iterations (bench workload `cent`) with kernel stats."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2305_04397_b200.api import Centralised, Instance, Solver

cfg, thr, eps, K = bench.workload("cent")
inst = Instance.warehouse(cfg)
cm = Centralised(inst)
solver = Solver(0)
solver.centralised_pareto(cm, thr, eps=eps, iteration_cap=5)
solver.reset_cuda_stats()
solver.set_profiling(True)
t0 = time.perf_counter()
rep = solver.centralised_pareto(cm, thr, eps=eps, iteration_cap=5)
dt = time.perf_counter() - t0
cs = solver.cuda_stats()
print(f"S={cm.S} {dt / len(rep['iterations']) * 1e3:.1f} ms/iter; opt launches {cs['opt_launches']:.0f} "
      f"opt ms {cs['opt_ms']:.1f} exec/ref {cs['opt_exec_backups'] / max(cs['opt_backups'], 1):.3f} "
      f"eval ms {cs['eval_ms']:.1f} kernels {cs['kernels']:.0f}")
