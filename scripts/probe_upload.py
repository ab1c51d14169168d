"""Dev probe: e2e step pieces (release, upload, query) through the host API on C2."""
import sys, time, json
sys.path.insert(0, '.')
from paper_2305_04397_b200.api import Instance, Solver
from tests.helpers import warehouse_config
inst = Instance.warehouse(warehouse_config(10, 10, 10))
s = Solver(0)
if len(sys.argv) > 1 and sys.argv[1] == "lean":
    s.set_lean(True)
thr = [-20.0] * 10 + [0.99] * 10
for rep in range(4):
    t0 = time.perf_counter(); s.release(); t1 = time.perf_counter(); s.upload(inst); t2 = time.perf_counter()
    r = s.pareto(inst, thr, eps=0.01); t3 = time.perf_counter()
    print(json.dumps(dict(release_ms=(t1-t0)*1e3, upload_ms=(t2-t1)*1e3, query_ms=(t3-t2)*1e3)), flush=True)
