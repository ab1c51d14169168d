"""Host product builder (libmorap_host.so, CPU) == the reference's products, array for
array (model.hpp:230-321, instance.hpp:42-91, warehouse.hpp:88-198)."""
import hashlib
import json

import numpy as np
import pytest

import oracle
from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.errors import Errc, MorapError
from tests.helpers import GOLDEN, load_golden

FIELDS = ["rowOffset", "trnOffset", "succ", "prob", "cost", "success", "done", "accept"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fingerprint(p):
    return {"S": p.S, "R": p.R, "nnz": p.nnz, "initial": p.initial, "rewardFinite": p.rewardFinite,
            **{k: sha(getattr(p, k)) for k in FIELDS}}


def test_products_match_reference_golden():
    gold = load_golden("products.json")
    fig2 = Instance.from_json(open(f"{GOLDEN}/fig2.json").read())
    assert fingerprint(fig2.product(0, 0)) == gold["fig2"][0][0]
    for key, grid in gold.items():
        if key == "fig2":
            continue
        inst = Instance.warehouse(json.loads(key))
        for i, row in enumerate(grid):
            for j, fp in enumerate(row):
                assert fingerprint(inst.product(i, j)) == fp, (key, i, j)


def test_instance_dedup_and_padding():
    # identical agents/tasks share one product (instance.hpp:70-89; test_solver.cpp:68-75)
    agent = json.load(open(f"{GOLDEN}/fig2.json"))["agents"][0]
    two = Instance.from_json(json.dumps({"agents": [agent, agent], "tasks": ["!x U y", "!x U y"]}))
    assert two.distinct == 1
    # fewer tasks than agents pads with an immediately satisfied dummy task
    padded = Instance.from_json(json.dumps({"agents": [agent, agent], "tasks": ["!x U y"]}))
    assert padded.real_tasks == 1 and padded.n == 2


def test_loader_errors():
    with pytest.raises(MorapError) as e:
        Instance.from_json('{"agents": [{"states": 1, "actions": [{"state": 0, "to": [{"s": 0, "p": 0.5}]}]}], "tasks": ["F y"]}')
    assert e.value.code == Errc.InvalidModel
    with pytest.raises(MorapError) as e:
        Instance.from_json('{"agents": [{"states": 1, "actions": [{"state": 0, "to": [{"s": 0, "p": 1.0}]}]}], "tasks": ["G y"]}')
    assert e.value.code == Errc.NotCoSafe
    with pytest.raises(MorapError) as e:
        Instance.from_json('{"agents": [{"states": 1, "actions": [{"state": 0, "to": [{"s": 0, "p": 1.0}]}]}], "tasks": ["F (y"]}')
    assert e.value.code == Errc.Syntax
    with pytest.raises(MorapError) as e:  # can idle forever: NotRewardFinite (test_numerics.cpp:74-80)
        Instance.from_json('{"agents": [{"states": 1, "actions": [{"state": 0, "to": [{"s": 0, "p": 1.0}]}]}], "tasks": ["F y"]}')
    assert e.value.code == Errc.NotRewardFinite
    with pytest.raises(MorapError) as e:
        Instance.warehouse({"W": 3, "H": 3, "n": 2, "racks": [[0, 0]], "feed": [0, 0]})
    assert e.value.code == Errc.InvalidConfig


FORMULAS = ["F x", "F y", "x U y", "y U x", "F (x & F y)", "F (x & y)", "X x", "true", "F x | F y", "F x & F y",
            "!x U y", "X (x | y) U (y & !x)", "F (x & X X y)"]


def random_agent(rng, max_states=5):
    S = int(rng.integers(2, max_states + 1))
    labels, actions = {}, []
    for s in range(S):
        lab = [a for a in ("x", "y") if rng.integers(0, 3) == 0]
        if lab:
            labels[str(s)] = lab
        for a in range(int(rng.integers(1, 3))):
            tos = sorted(set(int(t) for t in rng.integers(0, S, size=int(rng.integers(1, 3)))))
            w = rng.uniform(0.2, 1.0, size=len(tos))
            actions.append({"state": s, "name": f"a{a}", "to": [{"s": t, "p": float(p)} for t, p in zip(tos, w / w.sum())],
                            "reward": float(rng.uniform(-2, 0))})
    return {"states": S, "initial": 0, "labels": labels, "actions": actions}


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_random_tiny_instances_match_reference_live():
    ref = oracle.ref()
    rng = np.random.default_rng(777001)
    checked = 0
    for _ in range(300):
        n = int(rng.integers(1, 3))
        doc = {"agents": [random_agent(rng) for _ in range(n)],
               "tasks": [FORMULAS[int(rng.integers(0, len(FORMULAS)))] for _ in range(int(rng.integers(1, n + 1)))]}
        text = json.dumps(doc)
        try:
            mine = Instance.from_json(text)
        except MorapError as e:
            with pytest.raises(oracle.RefError):
                ref.from_json(text)
            continue
        theirs = ref.from_json(text)
        assert mine.distinct == theirs.distinct
        for i in range(n):
            for j in range(n):
                assert fingerprint(mine.product(i, j)) == fingerprint(theirs.product(i, j))
        checked += 1
    assert checked > 50
