"""C5 scaling sweep (BASELINE.json configs[4]): single warehouse products from 3x3 to 32x32
grids (1e3 .. 1e7 transitions), K = 2, 3, 5 objectives; optimize throughput on the GPU vs
the reference engine on one host thread (the reference runs one job per worker thread).
Two GPU numbers per size: one job alone (a small model cannot fill a B200: launch/latency
bound) and a batch of jobs on the same model with different weights, enough to stream
~3e7 transitions per sweep (how the Pareto query uses the GPU: n^2 jobs per batch).
Writes one JSON line per (grid, K)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402  (CPU baseline only)
from paper_2305_04397_b200.api import Instance  # noqa: E402
from paper_2305_04397_b200.cuda import CudaBackend  # noqa: E402

be = CudaBackend(0)
be.set_profiling(True)
grids = [int(g) for g in sys.argv[1:]] or [3, 4, 6, 8, 12, 16, 24, 32]
for W in grids:
    cfg = {"W": W, "H": W, "n": 1, "slip": 0.05, "racks": [[W - 1, W - 1]], "feed": [0, 0], "seed": 42}
    for K in (2, 3, 5):
        inst = Instance.warehouse(cfg)
        if K > 2:
            inst.add_objectives(K, seed=3)
        p = inst.product(0, 0)
        p.objectives = [inst.objective(0, 0, k) for k in range(K)]
        be.release_models()
        ids = be.upload([p])
        w = np.full((1, K), 1.0 / K)
        for _ in range(2):
            be.optimize(ids, w)
        be.reset_stats()
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            val, sw, res, st = be.optimize(ids, w)
        wall = (time.perf_counter() - t0) / reps
        s = be.stats()
        line = {"grid": W, "K": K, "states": p.S, "nnz": p.nnz, "sweeps": int(sw[0]),
                "gpu_backups_per_s_wall": float(sw[0]) * p.nnz / wall,
                "gpu_kernel_backups_per_s": s["opt_backups"] / (s["opt_ms"] * 1e-3),
                "gpu_kernel_GBps": s["opt_bytes"] / (s["opt_ms"] * 1e-3) / 1e9, "wall_ms": wall * 1e3}
        # a batch of jobs on the same model, different weights, ~3e7 transitions per sweep
        nb = int(min(4096, max(1, round(3e7 / p.nnz))))
        wb = np.random.default_rng(K).dirichlet(np.ones(K), size=nb)
        be.optimize(np.repeat(ids, nb), wb)
        be.reset_stats()
        t0 = time.perf_counter()
        vb, swb, rb, stb = be.optimize(np.repeat(ids, nb), wb)
        wallb = time.perf_counter() - t0
        sb = be.stats()
        line.update(batch_jobs=nb, batch_backups_per_s_wall=float(np.sum(swb)) * p.nnz / wallb,
                    batch_kernel_backups_per_s=sb["opt_backups"] / (sb["opt_ms"] * 1e-3),
                    batch_kernel_GBps=sb["opt_bytes"] / (sb["opt_ms"] * 1e-3) / 1e9, batch_wall_ms=wallb * 1e3)
        if K == 2 and oracle.ref_available():
            ri = oracle.ref().warehouse(cfg)
            sec, bk = ri.optimize_phase(np.array([0.5, 0.5]), 1)
            line["cpu_ref_backups_per_s_1thread"] = bk / sec
        print(json.dumps(line), flush=True)
