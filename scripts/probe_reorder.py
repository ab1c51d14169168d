"""Dev probe: does a locality-improving state order speed up the compact sweeps at C4 scale?
(Measured: the BFS numbering's per-tile successor spans are already ~500 states; RCM widens
them -- DESIGN.md §8 "Next".)
Products of the C4 grid (10 x 10, 100 racks) for n agents x n tasks are uploaded twice -- in
the reference's BFS numbering and permuted by reverse Cuthill-McKee (scipy) -- and the same
batch of optimize jobs runs on both; values / sweeps must be identical (a permutation does not
change any state's arithmetic).   python scripts/probe_reorder.py [n] [jobs_per_product]"""
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_04397_b200.api import Instance, Product  # noqa: E402
from paper_2305_04397_b200.cuda import CudaBackend  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
per = int(sys.argv[2]) if len(sys.argv) > 2 else 200
racks = [[9 - (k % 10), 9 - (k // 10)] for k in range(100)]
inst = Instance.warehouse({"W": 10, "H": 10, "n": n, "slip": 0.05, "racks": racks, "feed": [0, 0], "seed": 42})
prods = [inst.product(i, j) for i in range(n) for j in range(n)]


def permuted(p):
    S = p.S
    rows_of = np.diff(p.rowOffset)
    owner = np.repeat(np.arange(S), rows_of)
    trn_owner = np.repeat(owner, np.diff(p.trnOffset))
    A = sp.csr_matrix((np.ones(p.nnz), (trn_owner, p.succ)), shape=(S, S))
    order = reverse_cuthill_mckee(A + A.T, symmetric_mode=True)  # new -> old
    inv = np.empty(S, np.int64)
    inv[order] = np.arange(S)
    ro = np.zeros(S + 1, np.int64)
    ro[1:] = np.cumsum(rows_of[order])
    row_old = np.concatenate([np.arange(p.rowOffset[s], p.rowOffset[s + 1]) for s in order])
    tcount = np.diff(p.trnOffset)[row_old]
    to = np.zeros(len(row_old) + 1, np.int64)
    to[1:] = np.cumsum(tcount)
    k_old = np.concatenate([np.arange(p.trnOffset[r], p.trnOffset[r + 1]) for r in row_old])
    return Product(rowOffset=ro.astype(np.int32), trnOffset=to.astype(np.int32),
                   succ=inv[p.succ[k_old]].astype(np.int32), prob=p.prob[k_old], cost=p.cost[row_old],
                   success=p.success[row_old], done=p.done[order], accept=p.accept[order],
                   initial=int(inv[p.initial]), rewardFinite=True)


t = time.time()
perm = [permuted(p) for p in prods]
print("permuted in", round(time.time() - t, 1), "s", flush=True)
rng = np.random.default_rng(5)
wc = rng.uniform(0.05, 0.95, size=len(prods) * per)
W = np.stack([wc, 1.0 - wc], axis=1)
out = {}
for name, models in (("bfs", prods), ("rcm", perm), ("bfs2", prods), ("rcm2", perm)):
    be = CudaBackend(0)
    be.set_lean(True)
    ids = be.upload(models)
    jobs = np.repeat(ids, per)
    be.optimize(jobs[: len(ids)], W[: len(ids)])  # warm-up
    t = time.time()
    val, sw, res, st = be.optimize(jobs, W)
    dt = time.time() - t
    out[name] = (dt, val, sw)
    print(name, "optimize", round(dt, 3), "s, sweeps max", int(sw.max()), flush=True)
    be.close()
same = out["bfs"][1].tobytes() == out["rcm"][1].tobytes() and out["bfs"][2].tobytes() == out["rcm"][2].tobytes()
print(json.dumps({"n": n, "jobs": int(len(W)), "bfs_s": [out["bfs"][0], out["bfs2"][0]],
                  "rcm_s": [out["rcm"][0], out["rcm2"][0]], "values_sweeps_identical": same}))
