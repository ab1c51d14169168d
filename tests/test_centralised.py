"""Centralised model (centralised.hpp), SURVEY.md §8(f) row 2.

CPU: buildCentralised's arrays equal the reference's -- against the committed golden
fingerprints (scripts/gen_golden_centralised.py) and live against oracle/_ref when present;
guards. GPU: centralisedParetoPoint through the device kernels gives the reference's report
bit for bit (same floats, weights, tUp/tDown, scheduler fingerprints)."""
import hashlib

import numpy as np
import pytest

import oracle
from paper_2305_04397_b200.api import Centralised, Instance
from paper_2305_04397_b200.errors import Errc, MorapError
from tests.helpers import GOLDEN, SUITE_5x5, SUITE_6x6, load_golden

GOLD = load_golden("centralised.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _fp(c: Centralised) -> dict:
    a = c.arrays()
    out = {k: sha(a[k]) for k in ("rowOffset", "trnOffset", "succ", "prob", "done", "rewards")}
    out.update(S=c.S, R=c.R, nnz=c.nnz, rewardFinite=c.reward_finite)
    return out


def _fig2():
    return Instance.from_json(open(f"{GOLDEN}/fig2.json").read())


def test_centralised_model_matches_golden():
    assert _fp(Centralised(_fig2())) == GOLD["fig2_model"]
    for run in GOLD["suite"]:
        assert _fp(Centralised(Instance.warehouse(run["config"]))) == run["model"]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_centralised_model_matches_reference_live():
    for cfg in (dict(SUITE_5x5, n=2, seed=11), dict(SUITE_6x6, n=2, slip=0.1)):
        ours = Centralised(Instance.warehouse(cfg)).arrays()
        ref = oracle.ref().warehouse(cfg).centralised()
        for k in ("rowOffset", "trnOffset", "succ", "prob", "done", "rewards"):
            assert np.asarray(ours[k]).tobytes() == np.asarray(ref[k]).tobytes(), k


def test_centralised_guards():
    with pytest.raises(MorapError) as e:
        Centralised(Instance.warehouse(dict(SUITE_6x6, n=2)), state_guard=1000)
    assert e.value.code == Errc.SizeGuard
    with pytest.raises(MorapError):
        Centralised(_fig2(), state_guard=0)


@pytest.mark.gpu
def test_centralised_pareto_matches_reference():
    from paper_2305_04397_b200.api import Solver
    solver = Solver(0)
    cases = [(_fig2(), g) for g in GOLD["fig2"]] + [(Instance.warehouse(g["config"]), g) for g in GOLD["suite"]]
    for inst, g in cases:
        rep = solver.centralised_pareto(Centralised(inst), g["thresholds"], eps=g["eps"])
        rep.pop("stats")
        want = g["result"]
        for key in ("feasible", "converged", "tDown", "tUp", "lambdaStar", "records"):
            assert rep[key] == want[key], key
        assert [(it["w"], it["r"]) for it in rep["iterations"]] == [(it["w"], it["r"]) for it in want["iterations"]]
