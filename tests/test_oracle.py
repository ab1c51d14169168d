"""The oracle pinned before it is trusted (CPU only).

* vi_oracle.c against the known answers of proj/tests/test_numerics.cpp:18-80
* vi_oracle.c against the reference's own outputs: golden fingerprints written by
  scripts/gen_golden.py from oracle/_ref, and -- when oracle/_ref is present -- live,
  bit for bit, on random models.
"""
import hashlib

import numpy as np
import pytest

import oracle
from paper_2305_04397_b200.api import Instance
from tests.helpers import GOLDEN, load_golden, random_done_model, random_scheduler


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fig2_product():
    inst = Instance.from_json(open(f"{GOLDEN}/fig2.json").read())
    p = inst.product(0, 0)
    return oracle.Csr(p.rowOffset, p.trnOffset, p.succ, p.prob, p.done, p.initial, p.cost, p.success, p.accept, True)


def test_fig2_known_answers():
    vi = oracle.vi()
    m = fig2_product()
    rc, v, pol_c, sw, res, best_cost = vi.optimize(m, vi.weighted_reward([m.cost, m.success], [1.0, 0.0]))
    assert rc == 0 and abs(best_cost - (-1.0)) <= 1e-5
    rc, v, pol_s, sw, res, best_succ = vi.optimize(m, vi.weighted_reward([m.cost, m.success], [0.0, 1.0]))
    assert rc == 0 and abs(best_succ - 5.0 / 7.0) <= 1e-5
    assert pol_c[m.initial] != pol_s[m.initial]
    # cross-evaluation gives the hull corners (test_numerics.cpp:34-40)
    assert abs(vi.evaluate(m, pol_c, m.success)[4] - 0.1) <= 1e-5
    assert abs(vi.evaluate(m, pol_s, m.cost)[4] - (-15.0 / 7.0)) <= 1e-5
    # sweep mechanics (test_numerics.cpp:58-72)
    assert vi.optimize(m, m.cost, eps=1e9)[3] == 1
    assert vi.optimize(m, m.success, eps=1e-12, cap=3)[0] == 7  # NonConvergence


def test_chain_known_answer():
    # test_numerics.cpp:43-56: 0 -> 1 -> 2 (y), costs -1: optimum -2, success 1
    inst = Instance.from_json('{"agents": [{"states": 3, "initial": 0, "labels": {"2": ["y"]}, "actions": ['
                              '{"state": 0, "name": "go", "to": [{"s": 1, "p": 1.0}], "reward": -1},'
                              '{"state": 1, "name": "go", "to": [{"s": 2, "p": 1.0}], "reward": -1},'
                              '{"state": 2, "name": "stay", "to": [{"s": 2, "p": 1.0}], "reward": -1}]}],'
                              '"tasks": ["F y"]}')
    p = inst.product(0, 0)
    m = oracle.Csr(p.rowOffset, p.trnOffset, p.succ, p.prob, p.done, p.initial, p.cost, p.success)
    vi = oracle.vi()
    assert abs(vi.optimize(m, m.cost)[5] - (-2.0)) <= 1e-9
    assert abs(vi.optimize(m, m.success)[5] - 1.0) <= 1e-9


def test_not_reward_finite():
    rng = np.random.default_rng(3)
    m = random_done_model(rng, 8)
    m.rewardFinite = False
    assert oracle.vi().optimize(m, m.cost)[0] == 6


def test_oracle_matches_reference_golden_fingerprints():
    gold = load_golden("optimize_6x6_n2.json")
    inst = Instance.warehouse(gold["config"])
    vi = oracle.vi()
    for job in gold["jobs"]:
        p = inst.product(job["i"], job["j"])
        m = oracle.Csr(p.rowOffset, p.trnOffset, p.succ, p.prob, p.done, p.initial, p.cost, p.success)
        rc, v, pol, sw, res, v0 = vi.optimize(m, vi.weighted_reward([m.cost, m.success], job["w"]))
        assert (rc, sw, res, v0) == (job["rc"], job["sweeps"], job["residual"], job["value"])
        assert sha(v) == job["values"] and sha(pol) == job["policy"]
        for which, e in zip((0, 1), job["evaluate"]):
            erc, ev, es, er, ev0 = vi.evaluate(m, pol, m.cost if which == 0 else m.success)
            assert (es, er, ev0) == (e["sweeps"], e["residual"], e["value"]) and sha(ev) == e["values"]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_reference_live_random_models():
    vi = oracle.vi()
    lib = oracle.ref().lib
    import ctypes as C
    rng = np.random.default_rng(424242)
    for _ in range(60):
        m = random_done_model(rng, int(rng.integers(2, 40)), nonpositive=bool(rng.integers(0, 2)))
        w = rng.uniform(0, 1, 2)
        w /= w.sum()
        rho = vi.weighted_reward([m.cost, m.success], w)
        rc, v, pol, sw, res, v0 = vi.optimize(m, rho, eps=1e-8)
        rv = np.zeros(m.S)
        rp = np.zeros(m.S, np.int32)
        rs, rr = C.c_int(0), C.c_double(0)
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        lib.ref_optimize_csr.argtypes = [C.c_int] * 4 + [C.c_void_p] * 5 + [C.c_int, C.c_void_p, C.c_double, C.c_int] + [C.c_void_p] * 4
        rrc = lib.ref_optimize_csr(m.S, m.R, m.nnz, m.initial, p(m.rowOffset), p(m.trnOffset), p(m.succ), p(m.prob),
                                   p(m.done), 1, p(rho), 1e-8, 100000, p(rv), p(rp), C.byref(rs), C.byref(rr))
        assert rrc == rc == 0
        assert v.tobytes() == rv.tobytes() and pol.tobytes() == rp.tobytes() and sw == rs.value and res == rr.value
        mu = random_scheduler(rng, m)
        erc, ev, es, er, ev0 = vi.evaluate(m, mu, m.cost)
        lib.ref_evaluate_csr.argtypes = [C.c_int] * 4 + [C.c_void_p] * 7 + [C.c_double, C.c_int] + [C.c_void_p] * 3
        rv2 = np.zeros(m.S)
        rrc = lib.ref_evaluate_csr(m.S, m.R, m.nnz, m.initial, p(m.rowOffset), p(m.trnOffset), p(m.succ), p(m.prob),
                                   p(m.done), p(mu), p(m.cost), 1e-6, 100000, p(rv2), C.byref(rs), C.byref(rr))
        assert rrc == erc == 0 and ev.tobytes() == rv2.tobytes() and es == rs.value
        lib.ref_reward_finite_csr.argtypes = [C.c_int] * 3 + [C.c_void_p] * 5
        assert vi.reward_finite(m) == bool(lib.ref_reward_finite_csr(m.S, m.R, m.nnz, p(m.rowOffset), p(m.trnOffset),
                                                                      p(m.succ), p(m.prob), p(m.done)))
