import sys
sys.path.insert(0, '.')
from paper_2305_04397_b200.api import Instance, Solver
from tests.helpers import warehouse_config
inst = Instance.warehouse(warehouse_config(10, 10, 10))
s = Solver(0); s.upload(inst)
thr = [-20.0] * 10 + [0.99] * 10
s.pareto(inst, thr, eps=0.01)
print("---- traced run ----", file=sys.stderr, flush=True)
r = s.pareto(inst, thr, eps=0.01)
print(r["stats"], file=sys.stderr)
