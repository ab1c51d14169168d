"""Edge cases of the device path, checked bit for bit against the CPU oracle:
oversized tiles (a state with more rows than a shared-memory stage holds, rows with more
transitions than a stage holds) that take the kernels' global-memory fallback, models
with a single state, all-done models, empty batches, a K = 3 objective instance."""
import numpy as np
import pytest

import oracle
from tests.helpers import random_done_model

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def be():
    from paper_2305_04397_b200.cuda import CudaBackend
    b = CudaBackend(0)
    yield b
    b.close()


def hub_model(rng, rows_at_hub=2000, fan_at_hub=3, wide_row=0):
    """Random done-model whose state 0 has `rows_at_hub` rows (> one stage) and, optionally,
    one row with `wide_row` transitions (> the per-stage transition cap)."""
    S = 60
    done = np.zeros(S, np.uint8)
    done[-2:] = 1
    ro, to, succ, prob, cost = [0], [0], [], [], []
    for s in range(S):
        nrows = 1 if done[s] else (rows_at_hub if s == 0 else int(rng.integers(1, 4)))
        for r in range(nrows):
            if done[s]:
                succ.append(s)
                prob.append(1.0)
                cost.append(0.0)
            else:
                fan = wide_row if (s == 1 and r == 0 and wide_row) else fan_at_hub
                esc = 0.1 + rng.uniform(0, 0.3)
                raw = rng.uniform(0.05, 1.0, fan)
                for k in range(fan):
                    succ.append(int(rng.integers(0, S)))
                    prob.append((1 - esc) * raw[k] / raw.sum())
                succ.append(S - 1 - int(rng.integers(0, 2)))
                prob.append(esc)
                cost.append(rng.uniform(-2, 0.5))
            to.append(len(succ))
        ro.append(len(to) - 1)
    R = len(to) - 1
    return oracle.Csr(np.array(ro, np.int32), np.array(to, np.int32), np.array(succ, np.int32), np.array(prob),
                      done, 0, np.array(cost), np.zeros(R), done.copy(), True)


def check_against_oracle(be, models, W, eps=1e-8):
    vi = oracle.vi()
    be.release_models()
    ids = be.upload(models)
    val, sw, res, st = be.optimize(ids, W, eps=eps)
    pols = []
    for k, m in enumerate(models):
        rc, v, p, s, r, v0 = vi.optimize(m, vi.weighted_reward([m.cost, m.success], W[k]), eps=eps)
        assert (st[k], sw[k], res[k], val[k]) == (rc, s, r, v0)
        assert be.fetch_values(k).tobytes() == v.tobytes()
        assert be.fetch_policy(k).tobytes() == p.tobytes()
        pols.append(p)
    ev, esw, eres, est = be.evaluate_optimized(np.arange(len(models)), (0, 1), eps=eps)
    for k, m in enumerate(models):
        for o, rho in ((0, m.cost), (1, m.success)):
            rc, v, s, r, v0 = vi.evaluate(m, pols[k], rho, eps=eps)
            assert (est[k, o], esw[k, o], eres[k, o], ev[k, o]) == (rc, s, r, v0)
            assert be.fetch_eval_values(k, o).tobytes() == v.tobytes()


def test_oversized_state_fallback(be):
    rng = np.random.default_rng(1)
    models = [hub_model(rng), random_done_model(rng, 40), hub_model(rng, rows_at_hub=900)]
    check_against_oracle(be, models, np.array([[1.0, 0.0]] * 3))


def test_wide_row_fallback(be):
    rng = np.random.default_rng(2)
    m = hub_model(rng, rows_at_hub=3, wide_row=1500)
    # force the wide row to be chosen: it is the only row of state 1 in this model
    check_against_oracle(be, [m, random_done_model(rng, 30)], np.array([[1.0, 0.0], [0.0, 1.0]]))


def test_tiny_and_done_models(be):
    one = oracle.Csr(np.array([0, 1], np.int32), np.array([0, 1], np.int32), np.array([0], np.int32),
                     np.array([1.0]), np.array([1], np.uint8), 0, np.array([0.0]), np.array([0.0]))
    rng = np.random.default_rng(3)
    check_against_oracle(be, [one, random_done_model(rng, 3), one], np.array([[1.0, 0.0]] * 3))


def test_empty_batches(be):
    be.release_models()
    be.upload([random_done_model(np.random.default_rng(4), 10)])
    val, sw, res, st = be.optimize(np.zeros(0, np.int32), np.zeros((0, 2)))
    assert val.shape == (0,)


def test_three_objectives_supporting_point():
    """K = 3 extension (not in the reference): r[g_k(f(j), j)] equals the
    oracle's evaluation of the chosen pair under each objective (parity unpinned by the
    reference; checked against the C restatement)."""
    from paper_2305_04397_b200.api import Instance, Solver
    inst = Instance.warehouse({"W": 5, "H": 5, "n": 2, "slip": 0.1, "racks": [[4, 4], [0, 4]], "feed": [2, 0],
                               "seed": 7})
    inst.add_objectives(3, seed=11)
    s = Solver(0)
    w = np.array([0.2, 0.1, 0.15, 0.05, 0.3, 0.2])
    r, a = s.supporting_point(inst, w)
    assert r.shape == (6,)
    vi = oracle.vi()
    n = 2
    # recompute every pair's weighted optimum and the assignment on the CPU
    from paper_2305_04397_b200.api import max_assignment
    c = np.zeros((n, n))
    pol = {}
    objs = {}
    for i in range(n):
        for j in range(n):
            p = inst.product(i, j)
            m = oracle.Csr(p.rowOffset, p.trnOffset, p.succ, p.prob, p.done, p.initial, p.cost, p.success)
            extra = _extra_objective(s, inst, i, j)
            parts = [p.cost, extra, p.success]
            rho = vi.weighted_reward(parts, [w[i], w[n + i], w[2 * n + j]])
            rc, v, pl, sw, res, v0 = vi.optimize(m, rho)
            c[i, j] = v0
            pol[(i, j)] = (m, pl)
            objs[(i, j)] = parts
    assert max_assignment(c).tolist() == a.tolist()
    for j in range(n):
        i = int(a[j])
        m, pl = pol[(i, j)]
        for k, g in enumerate((i, n + i, 2 * n + j)):
            assert vi.evaluate(m, pl, objs[(i, j)][k])[4] == r[g]


def _extra_objective(solver, inst, i, j):
    """Objective vector 1 of product (i, j) in device order [cost, extra, success]."""
    return inst.objective(i, j, 1)
