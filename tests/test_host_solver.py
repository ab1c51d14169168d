"""Host side of the Pareto query on CPU: runParetoCore + projections + weight vectors +
Hungarian (libmorap_host.so) against the reference.

The supporting points are REPLAYED from the reference's own runs (tests/golden/pareto.json,
written from oracle/_ref), so the host loop is exercised without a GPU; every derived
quantity -- weight sequence, tUp/tDown, lambda*, verdict, synthesis marginals -- must come
out identical to the reference's.
"""
import numpy as np
import pytest

import oracle
from paper_2305_04397_b200.api import max_assignment, pareto_core
from paper_2305_04397_b200.errors import Errc, MorapError
from tests.helpers import load_golden


def replay(result):
    its = result["iterations"]
    calls = []

    def query(w):
        k = len(calls)
        calls.append(w.tolist())
        assert k < len(its), "more queries than the reference made"
        assert w.tolist() == its[k]["w"], f"weight vector {k} differs"
        return np.array(its[k]["r"]), np.array(its[k]["assignment"], np.int32)

    return query, calls


def check_same(mine, theirs):
    for key in ("feasible", "converged", "tUp", "tDown", "lambdaStar", "thresholds"):
        assert mine[key] == theirs[key], key
    assert [it["w"] for it in mine["iterations"]] == [it["w"] for it in theirs["iterations"]]
    assert [r["tUp"] for r in mine["records"]] == [r["tUp"] for r in theirs["records"]]
    assert [r["tDown"] for r in mine["records"]] == [r["tDown"] for r in theirs["records"]]
    if "marginal" in theirs:
        assert mine["marginal"] == theirs["marginal"]
        assert mine["synthesis"] == theirs["synthesis"]


def test_fig2_pareto_replay():
    gold = load_golden("pareto.json")
    for case in gold["fig2"]:
        q, calls = replay(case["result"])
        mine = pareto_core(case["result"]["thresholds"], 1, q, eps=case["eps"])
        check_same(mine, case["result"])
        assert len(calls) == len(case["result"]["iterations"])
    # the worked infeasible example: w3 = (0.349, 0.651), tDown (-1.9542975, 0.6129347) (test_cli.cpp:80-81)
    inf = gold["fig2"][0]["result"]
    assert abs(inf["iterations"][2]["w"][0] - 0.349) < 1e-3
    assert abs(inf["tDown"][0] + 1.9542975) < 1e-4 and abs(inf["tDown"][1] - 0.6129347) < 1e-4


def test_warehouse_suite_pareto_replay():
    gold = load_golden("pareto.json")
    for case in gold["suite"]:
        res = case["result"]
        n = len(res["iterations"][0]["assignment"])
        q, _ = replay(res)
        mine = pareto_core(res["thresholds"], n, q, eps=case["eps"])
        check_same(mine, res)
        assert 2 <= len(res["iterations"]) <= 16 and res["converged"]


def test_verify_mode_replay():
    gold = load_golden("pareto.json")
    res = gold["fig2"][0]["result"]  # infeasible thresholds
    q, calls = replay(res)
    out = pareto_core(res["thresholds"], 1, q, eps=1e-4, verify=True)
    assert out["verdict"] is False and len(calls) == 2  # stops at the first violation (test_solver.cpp:176-194: 6 jobs)


def test_bad_inputs():
    with pytest.raises(MorapError) as e:
        pareto_core([0.0, 0.0], 1, lambda w: (np.zeros(2), np.zeros(1, np.int32)), eps=-1.0)
    assert e.value.code == Errc.InvalidConfig
    with pytest.raises(MorapError) as e:
        pareto_core([0.0, 0.0], 1, lambda w: (np.zeros(2), np.zeros(1, np.int32)), norm=[[1.0, 2.0], [0.0, 1.0]])
    assert e.value.code == Errc.InvalidModel
    with pytest.raises(MorapError) as e:
        max_assignment(np.zeros((2, 3)))
    assert e.value.code == Errc.NonSquare


def test_assignment_lexicographic_ties():
    # all-equal values: every permutation is optimal -> identity (assignment.hpp:87-109)
    assert max_assignment(np.ones((4, 4))).tolist() == [0, 1, 2, 3]
    c = np.array([[1.0, 1.0], [1.0, 1.0]])
    assert max_assignment(c).tolist() == [0, 1]
    c = np.array([[0.0, 5.0], [5.0, 0.0]])
    assert max_assignment(c).tolist() == [1, 0]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_assignment_matches_reference_live():
    ref = oracle.ref()
    rng = np.random.default_rng(5)
    for _ in range(500):
        n = int(rng.integers(1, 8))
        c = np.round(rng.uniform(-3, 3, (n, n)) * float(rng.integers(1, 4))) / 2
        assert max_assignment(c).tolist() == ref.max_assignment(c).tolist()


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_pareto_core_with_reference_supporting_points_live():
    ref = oracle.ref()
    fig2 = open("tests/golden/fig2.json").read()
    inst = ref.from_json(fig2)
    rng = np.random.default_rng(11)
    for _ in range(20):
        t = [float(rng.uniform(-3.0, -0.5)), float(rng.uniform(0.0, 1.0))]
        eps = float(10 ** rng.uniform(-5, -2))
        mine = pareto_core(t, 1, lambda w: inst.supporting_point(w, 1)[:2], eps=eps)
        theirs = inst.pareto(t, eps=eps, workers=1)
        check_same(mine, theirs)
