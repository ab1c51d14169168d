"""Dev probe: C3 (50x50, K=3) with tracing and an iteration cap."""
import sys, time
sys.path.insert(0, '.')
from paper_2305_04397_b200.api import Instance, Solver
import bench
cap = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg, thr, eps, K = bench.workload('c3')
t = time.time(); inst = Instance.warehouse(cfg); print('build', time.time() - t, flush=True)
t = time.time(); inst.add_objectives(K, seed=7); print('objectives', time.time() - t, flush=True)
s = Solver(0)
t = time.time(); s.upload(inst); print('upload', time.time() - t, flush=True)
t = time.time(); r = s.pareto(inst, thr, eps=eps, iteration_cap=cap); print('query', time.time() - t, len(r['iterations']), r['converged'], r['feasible'], r['stats'], flush=True)
