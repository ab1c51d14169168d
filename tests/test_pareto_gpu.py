"""End-to-end parity of the Pareto-point query on the GPU (host C++ -> C ABI -> sm_100a)
against the reference's own runs (tests/golden/pareto.json from oracle/_ref): same
verdicts, same weight sequence, same supporting points, tUp/tDown, lambda*, schedulers
(FNV fingerprint of every recorded policy) and synthesis marginals -- bit for bit."""
import json

import numpy as np
import pytest

from paper_2305_04397_b200.errors import Errc, MorapError
from tests.helpers import GOLDEN, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def solver():
    from paper_2305_04397_b200.api import Solver
    s = Solver(0)
    yield s
    s.close()


def same(mine, theirs):
    for key in ("feasible", "converged", "tUp", "tDown", "lambdaStar", "thresholds", "iterations", "synthesis"):
        assert mine[key] == theirs[key], key
    assert mine["records"] == theirs["records"]
    assert mine.get("marginal") == theirs.get("marginal")


def test_fig2_queries(solver):
    from paper_2305_04397_b200.api import Instance
    inst = Instance.from_json(open(f"{GOLDEN}/fig2.json").read())
    gold = load_golden("pareto.json")
    for case in gold["fig2"]:
        same(solver.pareto(inst, case["thresholds"], eps=case["eps"]), case["result"])
    for case in gold["fig2_verify"]:
        assert solver.verify(inst, case["thresholds"], eps=case["eps"]) == case["verdict"]


def test_fig2_supporting_points(solver):
    # test_solver.cpp:47-66
    from paper_2305_04397_b200.api import Instance
    inst = Instance.from_json(open(f"{GOLDEN}/fig2.json").read())
    r, a = solver.supporting_point(inst, [1.0, 0.0])
    assert a.tolist() == [0] and abs(r[0] + 1.0) < 1e-4 and abs(r[1] - 0.1) < 1e-4
    r, a = solver.supporting_point(inst, [0.0, 1.0])
    assert abs(r[0] + 15.0 / 7.0) < 1e-4 and abs(r[1] - 5.0 / 7.0) < 1e-4
    for bad, code in (([1.0, 0.0, 0.0], Errc.DimensionMismatch), ([0.5, 0.2], Errc.InvalidConfig),
                      ([float("nan"), 0.0], Errc.InvalidConfig)):
        with pytest.raises(MorapError) as e:
            solver.supporting_point(inst, bad)
        assert e.value.code == code


def test_identical_pairs_collapse(solver):
    # test_solver.cpp:68-90: one deduplicated optimization (+ 2n evaluations); skewed agent
    # weights need two
    from paper_2305_04397_b200.api import Instance
    agent = json.load(open(f"{GOLDEN}/fig2.json"))["agents"][0]
    inst = Instance.from_json(json.dumps({"agents": [agent, agent], "tasks": ["!x U y", "!x U y"]}))
    assert inst.distinct == 1
    r, a = solver.supporting_point(inst, [0.25, 0.25, 0.25, 0.25])
    assert solver.last_stats[0] == 1 and solver.last_stats[2] == 4
    assert a.tolist() == [0, 1] and r[0] == r[1] and r[2] == r[3]
    r, a = solver.supporting_point(inst, [0.5, 0.25, 0.125, 0.125])
    assert solver.last_stats[0] == 2 and a.tolist() == [0, 1]


def test_warehouse_suite(solver):
    from paper_2305_04397_b200.api import Instance
    gold = load_golden("pareto.json")
    for case in gold["suite"]:
        inst = Instance.warehouse(case["config"])
        mine = solver.pareto(inst, case["thresholds"], eps=case["eps"])
        same(mine, case["result"])
        assert 2 <= len(mine["iterations"]) <= 16


def test_batching_does_not_change_results(solver):
    # engine determinism (test_engine.cpp:52-65, acceptance.cpp:439-497): results are the
    # same whether jobs run alone or in one batch
    from paper_2305_04397_b200.api import Instance
    from paper_2305_04397_b200.cuda import CudaBackend
    from tests.helpers import SUITE_6x6
    inst = Instance.warehouse(dict(SUITE_6x6, n=3))
    prods = [inst.product(i, j) for i in range(3) for j in range(3)]
    be = CudaBackend(0)
    ids = be.upload(prods)
    W = np.array([[0.2 + 0.6 * ((k * 37) % 64) / 64.0, 0.0] for k in range(64)])
    W[:, 1] = 1.0 - W[:, 0]
    jobs = np.array([ids[k % len(ids)] for k in range(64)])
    val, sw, res, st = be.optimize(jobs, W)
    batch = [be.fetch_values(k).tobytes() for k in range(64)]
    for k in (0, 17, 63):
        v1, s1, r1, t1 = be.optimize(jobs[k:k + 1], W[k:k + 1])
        assert v1[0] == val[k] and s1[0] == sw[k] and r1[0] == res[k]
        assert be.fetch_values(0).tobytes() == batch[k]
    be.close()
