"""Evaluations with more objectives than the policy-chain kernels take at once (> 4, e.g.
the 2n objectives of a centralised model) are split into sub-jobs of <= 4 RHS on the same
chain; every RHS has its own stop test (numerics.hpp:130-168), so the split batch returns
exactly what the RHS evaluated a few at a time return, in the caller's layout. The optimize
jobs on these K-objective products are checked against the oracle bit for bit."""
from types import SimpleNamespace

import numpy as np
import pytest

import oracle

from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.cuda import CudaBackend

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K", [5, 7, 8])
def test_wide_evaluation_matches_narrow_batches(K):
    inst = Instance.warehouse({"W": 6, "H": 6, "n": 2, "slip": 0.05, "racks": [[5, 5], [0, 5], [5, 0]],
                               "feed": [0, 0], "seed": 42})
    inst.add_objectives(K, seed=3)
    prods = []
    for i in range(2):
        for j in range(2):
            p = inst.product(i, j)
            prods.append(SimpleNamespace(rowOffset=p.rowOffset, trnOffset=p.trnOffset, succ=p.succ, prob=p.prob,
                                         done=p.done, initial=p.initial, rewardFinite=p.rewardFinite,
                                         objectives=[inst.objective(i, j, k) for k in range(K)]))
    be = CudaBackend(0)
    ids = be.upload(prods)
    rng = np.random.default_rng(K)
    W = rng.dirichlet(np.ones(K), size=len(ids))
    val, sw, res, st = be.optimize(ids, W, eps=1e-7)
    # K-objective products with more than 256 reward tuples take the compact path too (u16
    # reward classes): bitwise against the oracle
    vi = oracle.vi()
    for k, p in enumerate(prods):
        m = oracle.Csr(p.rowOffset, p.trnOffset, p.succ, p.prob, p.done, p.initial, p.objectives[0],
                       p.objectives[-1])
        rc, v, pol, s_, r, v0 = vi.optimize(m, vi.weighted_reward(p.objectives, W[k]), eps=1e-7)
        assert (sw[k], res[k], val[k]) == (s_, r, v0)
        assert be.fetch_values(k).tobytes() == v.tobytes()
        assert be.fetch_policy(k).tobytes() == pol.tobytes()
    jobs = list(range(len(ids)))
    wide = be.evaluate_optimized(jobs, tuple(range(K)), eps=1e-7)
    wide_vals = [[be.fetch_eval_values(q, o).tobytes() for o in range(K)] for q in jobs]
    groups = [tuple(range(a, min(K, a + 3))) for a in range(0, K, 3)]
    for g in groups:
        part = be.evaluate_optimized(jobs, g, eps=1e-7)
        for r_wide, r_part in zip(wide, part):
            got = np.asarray(r_wide).reshape(len(jobs), K)[:, list(g)]
            assert got.tobytes() == np.asarray(r_part).reshape(len(jobs), len(g)).tobytes()
        for q in jobs:
            for oi, o in enumerate(g):
                assert be.fetch_eval_values(q, oi).tobytes() == wide_vals[q][o]
