"""Dev probe: supportingPoint phase timings on C2 through the host API."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
from paper_2305_04397_b200.api import Instance, Solver
from tests.helpers import warehouse_config
inst = Instance.warehouse(warehouse_config(10, 10, 10))
s = Solver(0); s.upload(inst)
for prof in (False, True):
    s.set_profiling(prof)
    for w in (np.full(20, 0.05), np.eye(20)[0]):
        for rep in range(3):
            t0 = time.perf_counter(); r, a = s.supporting_point(inst, w); t1 = time.perf_counter()
            st = s.last_stats
            print(json.dumps(dict(prof=prof, w0=float(w[0]), wall_ms=(t1-t0)*1e3, opt_ms=st[4]*1e3, eval_ms=st[5]*1e3, host_ms=st[6]*1e3)), flush=True)
thr = [-20.0]*10 + [0.99]*10
for rep in range(2):
    t0 = time.perf_counter(); rep_ = s.pareto(inst, thr, eps=0.01); t1 = time.perf_counter()
    print("pareto wall ms", (t1-t0)*1e3, rep_["stats"], flush=True)
