"""Frozen-tile skipping (k_select) is exact: the compact optimize sweeps
leave out tiles whose successor window and own states did not change bitwise in the
previous sweep, and every result -- values, policies, residuals, sweep counts, the
fused evaluations and whole Pareto queries -- is bit-for-bit the same as sweeping every
tile, and the same as the oracle (numerics.hpp:74-122)."""
import json

import numpy as np
import pytest

import oracle
from paper_2305_04397_b200.api import Instance, Solver
from paper_2305_04397_b200.cuda import CudaBackend
from tests.helpers import random_done_model

pytestmark = pytest.mark.gpu

GRID = {"W": 10, "H": 10, "n": 3, "slip": 0.05, "racks": [[9 - k, 9] for k in range(3)], "feed": [0, 0], "seed": 42}


def _run(be, ids, W, eps):
    val, sw, res, st = be.optimize(ids, W, eps=eps)
    vals = [be.fetch_values(k).tobytes() for k in range(len(ids))]
    pols = [be.fetch_policy(k).tobytes() for k in range(len(ids))]
    ev = be.evaluate_optimized(list(range(len(ids))), (0, 1), eps=eps)
    return (val.tobytes(), sw.tolist(), res.tobytes(), st.tolist(), vals, pols, [a.tobytes() for a in ev])


@pytest.mark.parametrize("eps", [1e-6, 1e-9])
def test_skipping_is_bitwise_neutral(eps):
    inst = Instance.warehouse(GRID)
    prods = [inst.product(i, j) for i in range(3) for j in range(3)]
    prods += [random_done_model(np.random.default_rng(11), 300) for _ in range(3)]
    be = CudaBackend(0)
    ids = be.upload(prods)
    W = np.array([[0.2 + 0.07 * k, 0.8 - 0.07 * k] for k in range(len(prods))])
    be.set_skip(False)
    be.reset_stats()
    full = _run(be, ids, W, eps)
    s_full = be.stats()
    be.set_skip(True)
    be.reset_stats()
    skip = _run(be, ids, W, eps)
    s_skip = be.stats()
    assert skip == full
    assert s_full["opt_exec_backups"] == s_full["opt_backups"]
    assert s_skip["opt_backups"] == s_full["opt_backups"]
    # warehouse products freeze layer by layer: a good share of the tile sweeps is skipped
    assert s_skip["opt_exec_backups"] < 0.8 * s_skip["opt_backups"]
    assert s_skip["opt_bytes"] < s_full["opt_bytes"]
    # and the oracle agrees on every job
    vi = oracle.vi()
    val, sw, res, st = be.optimize(ids, W, eps=eps)
    for k, p in enumerate(prods):
        m = oracle.Csr(p.rowOffset, p.trnOffset, p.succ, p.prob, p.done, p.initial, p.cost, p.success)
        rc, v, pol, s, r, v0 = vi.optimize(m, vi.weighted_reward([m.cost, m.success], W[k]), eps=eps)
        assert (sw[k], res[k], val[k]) == (s, r, v0)
        assert be.fetch_values(k).tobytes() == v.tobytes()
        assert be.fetch_policy(k).tobytes() == pol.tobytes()


def test_pareto_query_identical_with_and_without_skipping():
    from paper_2305_04397_b200.cuda import load_library
    inst = Instance.warehouse(GRID)
    thr = [-25.0] * 3 + [0.95] * 3
    reps = []
    for on in (False, True):
        solver = Solver(0)
        assert load_library().morap_cuda_set_skip(solver.cuda_ctx, int(on)) == 0
        rep = solver.pareto(inst, thr, eps=0.01)
        st = rep.pop("stats")
        reps.append(json.dumps(rep, sort_keys=True) + repr((st["optimize_backups"], st["evaluate_state_backups"])))
        solver.close()
    assert reps[0] == reps[1]


def _chain(n_states, fan):
    """A long chain to one done state (value reaches state s after n - s sweeps: almost every
    tile is frozen in almost every sweep), with `fan` extra rows on state 0 (> 768 rows:
    an oversized tile swept from the global arrays, never skipped)."""
    S = n_states + 1
    row_off, trn_off, succ, prob, cost = [0], [0], [], [], []
    for s in range(S):
        rows = [(s + 1, 1.0)] if s < n_states else [(s, 1.0)]
        if s == 0:
            rows += [(min(n_states, 1 + (r * 7919) % n_states), 1.0) for r in range(fan)]
        for t, p in rows:
            succ.append(t)
            prob.append(p)
            cost.append(-1.0 if s < n_states else 0.0)
            trn_off.append(len(succ))
        row_off.append(len(trn_off) - 1)
    done = np.zeros(S, np.uint8)
    done[n_states] = 1
    c = np.array(cost)
    return oracle.Csr(np.array(row_off, np.int32), np.array(trn_off, np.int32), np.array(succ, np.int32),
                      np.array(prob), done, 0, c, np.zeros_like(c), done.copy(), True)


def _compact_random(rng, n_states):
    """Random successors over the whole model (wide windows, out-of-window successors) with a
    compact alphabet: probabilities {0.375, 0.25}, costs {-1, -0.5, 0}."""
    S = n_states + 1
    row_off, trn_off, succ, prob, cost = [0], [0], [], [], []
    for s in range(S):
        if s == n_states:
            succ.append(s)
            prob.append(1.0)
            cost.append(0.0)
            trn_off.append(len(succ))
        else:
            for _ in range(int(rng.integers(1, 4))):
                for t in rng.integers(0, S, size=2):
                    succ.append(int(t))
                    prob.append(0.375)
                succ.append(n_states)
                prob.append(0.25)
                cost.append(float(rng.choice([-1.0, -0.5, 0.0])))
                trn_off.append(len(succ))
        row_off.append(len(trn_off) - 1)
    done = np.zeros(S, np.uint8)
    done[n_states] = 1
    c = np.array(cost)
    return oracle.Csr(np.array(row_off, np.int32), np.array(trn_off, np.int32), np.array(succ, np.int32),
                      np.array(prob), done, 0, c, np.zeros_like(c), done.copy(), True)


def test_skipping_on_chains_wide_windows_and_oversized_tiles():
    rng = np.random.default_rng(29)
    prods = [_compact_random(rng, 3000), _compact_random(rng, 20000), _chain(6000, 0), _chain(3000, 900)]
    be = CudaBackend(0)
    ids = be.upload(prods)
    W = np.array([[0.5, 0.5], [0.9, 0.1], [1.0, 0.0], [0.7, 0.3]])
    out = {}
    for on in (False, True):
        be.set_skip(on)
        be.reset_stats()
        out[on] = _run(be, ids, W, 0.0)  # eps 0: to the exact fixed point
        st = be.stats()
    assert out[True] == out[False]
    assert st["opt_exec_backups"] < st["opt_backups"]  # the chains freeze from the far end
    vi = oracle.vi()
    val, sw, res, stt = be.optimize(ids, W, eps=0.0)
    for k, p in enumerate(prods):
        rc, v, pol, s, r, v0 = vi.optimize(p, vi.weighted_reward([p.cost, p.success], W[k]), eps=0.0)
        assert (sw[k], res[k], val[k]) == (s, r, v0)
        assert be.fetch_values(k).tobytes() == v.tobytes()
        assert be.fetch_policy(k).tobytes() == pol.tobytes()
