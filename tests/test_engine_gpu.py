"""runBatch (engine.hpp:370) through the host C ABI (morap_run_batch), on the GPU.

* test_engine.cpp:239-283 restated: failures stay contained to their job -- a reward of the
  wrong length (DimensionMismatch), a job without a model (InvalidModel), an evaluate job
  capped at one sweep (NonConvergence) -- while the good jobs answer -1 and 5/7.
* Explicit-reward jobs on products that a Pareto query uploaded lean get their own full
  device copy, and their results equal the reference's optimalScheduler bit for bit.
* Results do not depend on how jobs are batched (test_engine.cpp:52-65)."""
import numpy as np
import pytest

import oracle
from paper_2305_04397_b200.api import Instance, Solver
from paper_2305_04397_b200.errors import Errc
from tests.helpers import GOLDEN, SUITE_6x6

pytestmark = pytest.mark.gpu


def _st(e):
    return int(e) + 1


def test_failures_stay_contained_to_their_job():
    inst = Instance.from_json(open(f"{GOLDEN}/fig2.json").read())
    p = inst.product(0, 0)
    rng = np.random.default_rng(1)
    sched = np.array([int(rng.integers(p.rowOffset[s], p.rowOffset[s + 1])) for s in range(p.S)], np.int32)
    jobs = [
        {"id": 0, "product": (0, 0), "reward": p.cost},
        {"id": 1, "product": (0, 0), "reward": p.cost[:1]},  # wrong length
        {"id": 2, "product": None},  # no model
        {"id": 3, "kind": "evaluate", "product": (0, 0), "reward": p.cost, "scheduler": sched, "sweep_cap": 1},
        {"id": 4, "product": (0, 0), "reward": p.success},
    ]
    res = {r["id"]: r for r in Solver(0).run_batch(inst, jobs)}
    assert len(res) == 5
    assert res[0]["ok"] and abs(res[0]["value"] - (-1.0)) <= 1e-4
    assert not res[1]["ok"] and res[1]["status"] == _st(Errc.DimensionMismatch)
    assert not res[2]["ok"] and res[2]["status"] == _st(Errc.InvalidModel)
    assert not res[3]["ok"] and res[3]["status"] == _st(Errc.NonConvergence)
    assert res[4]["ok"] and abs(res[4]["value"] - 5.0 / 7.0) <= 1e-4


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_explicit_rewards_after_lean_query_match_reference_and_batching():
    cfg = dict(SUITE_6x6, n=2)
    inst = Instance.warehouse(cfg)
    solver = Solver(0)
    solver.pareto(inst, [-30.0, -36.0, 0.95, 0.8], eps=0.01)  # uploads the products lean
    ref = oracle.ref().warehouse(cfg)
    jobs = []
    for k, (i, j) in enumerate([(0, 0), (0, 1), (1, 0), (1, 1)]):
        p = inst.product(i, j)
        wc = 0.2 + 0.6 * ((k * 37) % 64) / 64.0
        rho = np.array([(0.0 + wc * c) + (1.0 - wc) * u for c, u in zip(p.cost, p.success)])
        jobs.append({"id": k, "product": (i, j), "reward": rho, "wc": wc})
    together = solver.run_batch(inst, jobs)
    alone = [solver.run_batch(inst, [j])[0] for j in jobs]
    for j, a, b in zip(jobs, together, alone):
        assert a["ok"] and b["ok"]
        assert a["values"].tobytes() == b["values"].tobytes() and a["policy"].tobytes() == b["policy"].tobytes()
        assert (a["sweeps"], a["residual"], a["value"]) == (b["sweeps"], b["residual"], b["value"])
        rc, v, pol, sw, res, v0 = ref.optimize(*j["product"], j["wc"], 1.0 - j["wc"])
        assert rc == 0 and a["values"].tobytes() == v.tobytes() and a["policy"].tobytes() == pol.tobytes()
        assert (a["sweeps"], a["residual"], a["value"]) == (sw, res, v0)
