"""Parity at the configurations bench.py measures (BASELINE.json configs[1] and [3]),
against reference outputs written by scripts/gen_golden.py --measured from oracle/_ref
(tests/golden/c2.json, tests/golden/c4_sub4.json):

* C2 (10x10 grid, 10 agents x 10 tasks): all 100 host-built products array for array, and
  the whole bench query -- paretoPoint with thresholds (-20 x10, 0.99 x10), eps 0.01,
  13 iterations, infeasible -- bit for bit on the GPU: weight sequence, supporting points,
  assignments, tUp / tDown per iteration, lambda*, verdict and every recorded scheduler's
  fingerprint; once from the in-memory instance, once streamed + lean (the C4 code path).
* C4 (10x10 grid, every cell a rack, 100 x 100): its (i, j < 4) products are the products of
  the 4 x 4 sub-instance (start poses and tasks do not depend on n, warehouse.hpp:69-84,
  157-174). Their fingerprints, optimize values / policies / sweeps / residuals at two
  weight pairs, the fused evaluations of those policies, and the 4 x 4 Pareto query with
  C4's thresholds, bit for bit.
"""
import hashlib

import numpy as np
import pytest

from paper_2305_04397_b200.api import Instance
from tests.helpers import load_golden

FIELDS = ["rowOffset", "trnOffset", "succ", "prob", "cost", "success", "done", "accept"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fingerprint(p):
    return {"S": p.S, "R": p.R, "nnz": p.nnz, "initial": p.initial, "rewardFinite": p.rewardFinite,
            **{k: sha(getattr(p, k)) for k in FIELDS}}


@pytest.fixture(scope="module")
def c2():
    return load_golden("c2.json")


@pytest.fixture(scope="module")
def c4():
    return load_golden("c4_sub4.json")


def _report(rep):
    keys = ("feasible", "converged", "tUp", "tDown", "lambdaStar", "thresholds", "iterations", "synthesis",
            "records", "marginal")
    return {k: rep.get(k) for k in keys}


def test_c2_products_match_reference(c2):
    inst = Instance.warehouse(c2["config"])
    assert inst.n == 10
    for i, row in enumerate(c2["products"]):
        for j, fp in enumerate(row):
            assert fingerprint(inst.product(i, j)) == fp, (i, j)


def test_c4_sub_products_match_reference(c4):
    inst = Instance.warehouse(c4["config"])
    for i, row in enumerate(c4["products"]):
        for j, fp in enumerate(row):
            assert fingerprint(inst.product(i, j)) == fp, (i, j)


@pytest.mark.gpu
def test_c2_bench_query_bitwise(c2):
    from paper_2305_04397_b200.api import Solver
    inst = Instance.warehouse(c2["config"])
    s = Solver(0)
    case = c2["pareto"]
    got = s.pareto(inst, case["thresholds"], eps=case["eps"])
    assert len(got["iterations"]) == 13 and not got["feasible"]
    assert _report(got) == _report(case["result"])
    s.close()


@pytest.mark.gpu
def test_c2_bench_query_streamed_lean_bitwise(c2):
    from paper_2305_04397_b200.api import Solver
    s = Solver(0)
    s.set_lean(True)
    inst = Instance.warehouse_streamed(c2["config"], s, chunk=16)
    case = c2["pareto"]
    assert _report(s.pareto(inst, case["thresholds"], eps=case["eps"])) == _report(case["result"])
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("lean", [False, True])
def test_c4_sub_jobs_bitwise(c4, lean):
    from paper_2305_04397_b200.cuda import CudaBackend
    inst = Instance.warehouse(c4["config"])
    be = CudaBackend(0)
    be.set_lean(lean)
    ids = be.upload([inst.product(i, j) for i in range(4) for j in range(4)])
    jobs = c4["jobs"]
    val, sw, res, st = be.optimize(np.array([ids[4 * jb["i"] + jb["j"]] for jb in jobs]),
                                   np.array([jb["w"] for jb in jobs]))
    for q, jb in enumerate(jobs):
        assert (st[q], val[q], sw[q], res[q]) == (jb["rc"], jb["value"], jb["sweeps"], jb["residual"]), q
        assert sha(be.fetch_values(q)) == jb["values"] and sha(be.fetch_policy(q)) == jb["policy"], q
    ev, esw, eres, est = be.evaluate_optimized(list(range(len(jobs))), (0, 1))
    for q, jb in enumerate(jobs):
        for o in range(2):
            e = jb["evaluate"][o]
            assert (est[q, o], ev[q, o], esw[q, o], eres[q, o]) == (0, e["value"], e["sweeps"], e["residual"]), (q, o)
    be.close()


@pytest.mark.gpu
def test_c4_sub_query_bitwise(c4):
    from paper_2305_04397_b200.api import Solver
    s = Solver(0)
    s.set_lean(True)
    inst = Instance.warehouse_streamed(c4["config"], s, chunk=8)
    case = c4["pareto"]
    assert _report(s.pareto(inst, case["thresholds"], eps=case["eps"])) == _report(case["result"])
    s.close()
