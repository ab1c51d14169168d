"""The reference's engine/numerics pins that are not about a single job, on the GPU
(SURVEY.md §8c):

* acceptance.cpp:439-497 (criterion 7): 64 optimize jobs over the 6x6 n=3 warehouse
  products with w_c = 0.2 + 0.6 * ((37 k) mod 64) / 64 -- here bitwise against the
  reference itself (oracle/_ref) and invariant under how the jobs are batched.
* test_numerics.cpp:82-97: with non-positive rewards every sweep is pointwise
  non-increasing (optimize and evaluate); read here as the values after a cap of k sweeps.
* test_numerics.cpp:100-110: iterative evaluation agrees with the exact linear solve
  within 100 eps.
* test_engine.cpp:239-283: failures stay contained to their job.
"""
import numpy as np
import pytest

import oracle
from paper_2305_04397_b200.api import Instance
from tests.helpers import GOLDEN, SUITE_6x6, random_done_model, random_scheduler

pytestmark = pytest.mark.gpu

MORAP_OK, MORAP_INVALID_MODEL, MORAP_NOT_REWARD_FINITE, MORAP_NON_CONVERGENCE = 0, 5, 6, 7


@pytest.fixture(scope="module")
def be():
    from paper_2305_04397_b200.cuda import CudaBackend
    b = CudaBackend(0)
    yield b
    b.close()


def _bits(a):
    return np.ascontiguousarray(a).tobytes()


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_criterion7_64_jobs_bitwise_and_batch_invariant(be):
    cfg = dict(SUITE_6x6, n=3)
    ref = oracle.ref().warehouse(cfg)
    ours = Instance.warehouse(cfg)
    slots = []  # distinct products in (i, j) order, as acceptance.cpp:452-455
    for i in range(3):
        for j in range(3):
            first = int(ours.product_dims(i, j)[0][5])
            if first == i * 3 + j:
                slots.append((i, j))
    prods = [ours.product(i, j) for i, j in slots]
    assert all(p.S >= 10000 for p in prods)
    be.release_models()
    ids = be.upload(prods)
    jobs = [k % len(prods) for k in range(64)]
    wc = [0.2 + 0.6 * ((k * 37) % 64) / 64.0 for k in range(64)]
    W = np.array([[w, 1.0 - w] for w in wc])
    val, sw, res, st = be.optimize(ids[jobs], W)
    full = [be.fetch_values(k) for k in range(64)]
    for k in range(64):
        i, j = slots[jobs[k]]
        rc, v, p, s, r, v0 = ref.optimize(i, j, wc[k], 1.0 - wc[k])
        assert rc == 0 and st[k] == MORAP_OK
        assert sw[k] == s and res[k] == r and val[k] == v0
        assert _bits(full[k]) == _bits(v)
        assert _bits(be.fetch_policy(k)) == _bits(p)
    # the same jobs in batches of 1 and 7 (the reference's 1/2/4/8-worker check)
    for size in (1, 7):
        for b0 in range(0, 64, size):
            ks = list(range(b0, min(64, b0 + size)))
            v2, s2, r2, t2 = be.optimize(ids[[jobs[k] for k in ks]], W[ks])
            for q, k in enumerate(ks):
                assert v2[q] == val[k] and s2[q] == sw[k] and r2[q] == res[k]
                assert _bits(be.fetch_values(q)) == _bits(full[k])


def test_nonpositive_rewards_give_nonincreasing_sweeps(be):
    rng = np.random.default_rng(7)
    models = [random_done_model(rng, 12, 0.08, 3, nonpositive=True) for _ in range(40)]
    scheds = [random_scheduler(rng, m) for m in models]
    be.release_models()
    ids = be.upload(models)
    W = np.array([[1.0, 0.0]] * len(models))
    _, sw_opt, _, _ = be.optimize(ids, W, eps=1e-8)
    _, sw_ev, _, _ = be.evaluate(ids, scheds, [m.cost for m in models], eps=1e-8)
    prev_o = [None] * len(models)
    prev_e = [None] * len(models)
    for k in range(1, int(max(sw_opt.max(), sw_ev.max())) + 1):
        be.optimize(ids, W, eps=1e-8, sweep_cap=k)
        for q in range(len(models)):
            x = be.fetch_values(q)
            if prev_o[q] is not None:
                assert np.all(x <= prev_o[q] + 1e-12)
            prev_o[q] = x
        be.evaluate(ids, scheds, [m.cost for m in models], eps=1e-8, sweep_cap=k)
        for q in range(len(models)):
            x = be.fetch_eval_values(q)
            if prev_e[q] is not None:
                assert np.all(x <= prev_e[q] + 1e-12)
            prev_e[q] = x


def _exact(m, mu, rho):
    """Exact value of the chain under mu: (I - P) v = rho on the non-done states."""
    S = m.S
    A = np.eye(S)
    b = np.zeros(S)
    for s in range(S):
        if m.done[s]:
            continue
        r = mu[s]
        b[s] = rho[r]
        for k in range(m.trnOffset[r], m.trnOffset[r + 1]):
            t = m.succ[k]
            if not m.done[t]:
                A[s, t] -= m.prob[k]
    return np.linalg.solve(A, b)


def test_iterative_and_exact_evaluation_agree(be):
    rng = np.random.default_rng(99)
    eps = 1e-6
    models = [random_done_model(rng, 20) for _ in range(60)]
    scheds = [random_scheduler(rng, m) for m in models]
    be.release_models()
    ids = be.upload(models)
    val, sw, res, st = be.evaluate(ids, scheds, [m.cost for m in models], eps=eps)
    for q, m in enumerate(models):
        assert st[q] == MORAP_OK
        ex = _exact(m, scheds[q], m.cost)[m.initial]
        assert abs(val[q] - ex) <= 100 * eps


def test_failures_stay_contained_to_their_job(be):
    inst = Instance.from_json(open(f"{GOLDEN}/fig2.json").read())
    p = inst.product(0, 0)
    fig2 = oracle.Csr(p.rowOffset, p.trnOffset, p.succ, p.prob, p.done, p.initial, p.cost, p.success, p.accept, True)
    # a model that can avoid its done state forever
    trap = oracle.Csr(np.array([0, 2, 3], np.int32), np.array([0, 1, 2, 3], np.int32), np.array([0, 1, 1], np.int32),
                      np.ones(3), np.array([0, 1], np.uint8), 0, np.array([-1.0, -1.0, 0.0]), np.zeros(3),
                      np.array([0, 1], np.uint8), False)
    be.release_models()
    ids = be.upload([fig2, trap])
    val, sw, res, st = be.optimize_rho([ids[0], ids[1], ids[0]], [fig2.cost, trap.cost, fig2.success])
    assert list(st) == [MORAP_OK, MORAP_NOT_REWARD_FINITE, MORAP_OK]
    assert abs(val[0] - (-1.0)) <= 1e-4 and abs(val[2] - 5.0 / 7.0) <= 1e-4
    rng = np.random.default_rng(1)
    good = random_scheduler(rng, fig2)
    foreign = good.copy()
    foreign[fig2.initial] = fig2.rowOffset[(fig2.initial + 1) % fig2.S]  # a row of another state
    val, sw, res, st = be.evaluate([ids[0], ids[0]], [good, foreign], [fig2.cost, fig2.cost])
    assert st[0] == MORAP_OK and st[1] == MORAP_INVALID_MODEL
    val, sw, res, st = be.evaluate([ids[0], ids[0]], [good, good], [fig2.cost, fig2.success], sweep_cap=1)
    assert st[0] == MORAP_NON_CONVERGENCE  # every action costs 1: one sweep never settles
