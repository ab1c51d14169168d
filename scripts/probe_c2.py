"""Dev probe: C2 (10x10 warehouse, n=10) optimize-phase throughput of the GPU backend.
Products come from the reference generator (oracle/_ref) -- this is a kernel probe only."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2305_04397_b200.cuda import CudaBackend
from tests.helpers import warehouse_config

W = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
t = time.time()
inst = oracle.ref().warehouse(warehouse_config(W, W, n))
prods = [inst.product(i, j) for i in range(n) for j in range(n)]
print("generate", time.time() - t, "s", sum(p.nnz for p in prods), "nnz", flush=True)
be = CudaBackend(0)
t = time.time(); ids = be.upload(prods); print("upload", time.time() - t, flush=True)
peak = json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'] if __import__('os').path.exists('MEASURED_PEAKS.json') else 6553.9
for wname, w in [("uniform", np.full(2, 0.5)), ("cost", np.array([1.0, 0.0])), ("w3", np.array([0.35, 0.65]))]:
    Wm = np.tile(w, (len(ids), 1))
    for rep in range(3):
        be.reset_stats()
        be.set_profiling(rep == 2)
        t0 = time.perf_counter()
        val, sw, res, st = be.optimize(ids, Wm)
        t1 = time.perf_counter()
        s = be.stats()
        bk = float(np.sum(sw.astype(np.float64) * np.array([p.nnz for p in prods])))
        line = dict(w=wname, rep=rep, wall_ms=(t1 - t0) * 1e3, sweeps_max=int(sw.max()), sweeps_min=int(sw.min()),
                    backups=bk, backups_per_s=bk / (t1 - t0), status=int(st.max()))
        if rep == 2:
            line.update(kernel_ms=s['opt_ms'], launches=s['opt_launches'], bytes=s['opt_bytes'],
                        GBps=s['opt_bytes'] / (s['opt_ms'] * 1e-3) / 1e9,
                        frac=s['opt_bytes'] / (s['opt_ms'] * 1e-3) / 1e9 / peak,
                        kernel_backups_per_s=bk / (s['opt_ms'] * 1e-3))
        print(json.dumps(line), flush=True)
# parity spot check on 3 jobs against the reference
val, sw, res, st = be.optimize(ids, np.tile([0.35, 0.65], (len(ids), 1)))
for q in [0, 37, len(ids) - 1]:
    i, j = divmod(q, n)
    rc, v, p, s, r, v0 = inst.optimize(i, j, 0.35, 0.65)
    ok = (be.fetch_values(q).tobytes() == v.tobytes()) and (be.fetch_policy(q).tobytes() == p.tobytes()) and sw[q] == s
    print("parity job", q, ok, flush=True)
# CPU reference on this host, all threads
sec, bk = inst.optimize_phase(np.concatenate([np.full(n, 0.35 / n), np.full(n, 0.65 / n)]) * 1.0, 0)
print("cpu ref optimize phase", sec, "s", bk / sec, "backups/s", oracle.ref().hardware_threads(), "threads", flush=True)
