"""Parity of the sm_100a kernels (through the C ABI) with the CPU oracle, bit for bit.

Checker: oracle/ (the C restatement of numerics.hpp, pinned against the reference in
tests/test_oracle.py) and oracle/_ref (the reference itself) where present.
"""
import numpy as np
import pytest

import oracle
from tests.helpers import SUITE_6x6, random_done_model, random_scheduler

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def be():
    from paper_2305_04397_b200.cuda import CudaBackend
    b = CudaBackend(0)
    yield b
    b.close()


def _same(a, b):
    return np.asarray(a).tobytes() == np.asarray(b).tobytes()


def test_random_models_optimize_bitwise(be):
    rng = np.random.default_rng(424242)
    models = [random_done_model(rng, int(rng.integers(2, 60))) for _ in range(40)]
    be.release_models()
    ids = be.upload(models)
    vi = oracle.vi()
    W = np.array([[1.0, 0.0] for _ in models])
    val, sw, res, st = be.optimize(ids, W, eps=1e-8)
    for k, m in enumerate(models):
        rho = vi.weighted_reward([m.cost, m.success], W[k])
        rc, v, p, s, r, v0 = vi.optimize(m, rho, eps=1e-8)
        assert st[k] == rc == 0
        assert sw[k] == s and res[k] == r and val[k] == v0
        assert _same(be.fetch_values(k), v)
        assert _same(be.fetch_policy(k), p)


def test_warehouse_products_bitwise(be):
    ref = oracle.ref()
    inst = ref.warehouse(dict(SUITE_6x6, n=2))
    prods = [inst.product(i, j) for i in range(2) for j in range(2)]
    be.release_models()
    ids = be.upload(prods)
    weights = [(1.0, 0.0), (0.3, 0.7), (0.0, 1.0), (0.5, 0.5)]
    jobs, W = [], []
    for k in range(4):
        for w in weights:
            jobs.append(ids[k])
            W.append(w)
    val, sw, res, st = be.optimize(np.array(jobs), np.array(W))
    for q in range(len(jobs)):
        i, j = divmod(q // 4, 2)
        rc, v, p, s, r, v0 = inst.optimize(i, j, *W[q])
        assert rc == 0 and st[q] == 0
        assert (sw[q], res[q], val[q]) == (s, r, v0)
        assert _same(be.fetch_values(q), v)
        assert _same(be.fetch_policy(q), p)
    # fused cost+success evaluation of every job's own policy (solver.hpp:148-172)
    ev, esw, eres, est = be.evaluate_optimized(np.arange(len(jobs)), (0, 1))
    for q in range(len(jobs)):
        i, j = divmod(q // 4, 2)
        pol = be.fetch_policy(q)
        for o in range(2):
            rc, v, s, r, v0 = inst.evaluate(i, j, pol, o)
            assert est[q, o] == 0 and esw[q, o] == s and eres[q, o] == r and ev[q, o] == v0
            assert _same(be.fetch_eval_values(q, o), v)


def test_sweep_mechanics(be):
    rng = np.random.default_rng(7)
    m = random_done_model(rng, 12)
    bad = random_done_model(rng, 12)
    bad.rewardFinite = False
    be.release_models()
    ids = be.upload([m, bad])
    # at least one sweep even with a huge tolerance (test_numerics.cpp:61-64)
    val, sw, res, st = be.optimize(ids[:1], np.array([[1.0, 0.0]]), eps=1e9)
    assert sw[0] == 1 and st[0] == 0
    # sweep cap raises NonConvergence (test_numerics.cpp:66-68)
    val, sw, res, st = be.optimize(ids[:1], np.array([[1.0, 0.0]]), eps=1e-300, sweep_cap=3)
    assert st[0] == 7 and sw[0] == 3
    # models that can dodge the objective are refused (test_numerics.cpp:74-80)
    val, sw, res, st = be.optimize(ids[1:], np.array([[1.0, 0.0]]))
    assert st[0] == 6 and sw[0] == 0


def test_general_evaluate_random_policies(be):
    rng = np.random.default_rng(99)
    models = [random_done_model(rng, 20) for _ in range(30)]
    be.release_models()
    ids = be.upload(models)
    pols = [random_scheduler(rng, m) for m in models]
    val, sw, res, st = be.evaluate(ids, pols, [m.cost for m in models])
    vi = oracle.vi()
    for k, m in enumerate(models):
        rc, v, s, r, v0 = vi.evaluate(m, pols[k], m.cost)
        assert st[k] == rc and sw[k] == s and res[k] == r and val[k] == v0
        assert _same(be.fetch_eval_values(k, 0), v)
    # a foreign row is rejected (checkScheduler, numerics.hpp:58-59)
    p = pols[0].copy()
    p[0] = models[0].rowOffset[1] + 5 if models[0].R > models[0].rowOffset[1] + 5 else -1
    val, sw, res, st = be.evaluate(ids[:1], [p], [models[0].cost])
    assert st[0] == 5
