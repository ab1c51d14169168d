"""Test fixtures mirroring the reference's tests/helpers.hpp generators.

random_done_model follows helpers.hpp:156-205 (every action leaks >= min_escape to a
done state, so value iteration contracts); random_scheduler follows :312-316. They use
numpy's generator, so the draws differ from the C++ ones -- the oracle is the checker.
"""
from __future__ import annotations

import json
import os

import numpy as np

from oracle import Csr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def random_done_model(rng: np.random.Generator, max_states: int, min_escape=0.08, max_actions=3,
                      nonpositive=False) -> Csr:
    non_done = int(rng.integers(1, max(1, max_states - 1) + 1))
    n_done = int(rng.integers(1, 3))
    S = non_done + n_done
    row_off, trn_off, succ, prob, cost, success = [0], [0], [], [], [], []
    for s in range(S):
        is_done = s >= non_done
        acts = 1 if is_done else int(rng.integers(1, max_actions + 1))
        for _ in range(acts):
            if is_done:
                succ.append(s)
                prob.append(1.0)
                cost.append(0.0)
            else:
                fan = int(rng.integers(1, 4))
                escape = min_escape + rng.uniform(0.0, 0.4)
                raw = rng.uniform(0.05, 1.0, size=fan)
                tot = raw.sum()
                for k in range(fan):
                    succ.append(int(rng.integers(0, S)))
                    prob.append((1.0 - escape) * raw[k] / tot)
                succ.append(non_done + int(rng.integers(0, n_done)))
                prob.append(escape)
                cost.append(rng.uniform(-2.0, 0.0) if nonpositive else rng.uniform(-2.0, 1.0))
            trn_off.append(len(succ))
            success.append(0.0)
        row_off.append(len(trn_off) - 1)
    done = np.zeros(S, np.uint8)
    done[non_done:] = 1
    return Csr(np.array(row_off, np.int32), np.array(trn_off, np.int32), np.array(succ, np.int32),
               np.array(prob, np.float64), done, 0, np.array(cost), np.array(success), done.copy(), True)


def random_scheduler(rng: np.random.Generator, m: Csr) -> np.ndarray:
    ro = m.rowOffset
    return np.array([int(rng.integers(ro[s], ro[s + 1])) for s in range(m.S)], np.int32)


def load_golden(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def warehouse_config(W, H, n, racks=None, feed=(0, 0), slip=0.05, seed=42, deadline=None):
    """BASELINE configs: racks row-major from the top-right."""
    if racks is None:
        racks = [[W - 1 - (k % W), H - 1 - (k // W)] for k in range(n)]
    cfg = {"W": W, "H": H, "n": n, "slip": slip, "racks": [list(r) for r in racks], "feed": list(feed), "seed": seed}
    if deadline is not None:
        cfg["deadline"] = deadline
    return cfg


SUITE_6x6 = {"W": 6, "H": 6, "slip": 0.05, "racks": [[5, 5], [0, 5], [5, 0]], "feed": [0, 0], "seed": 42}
SUITE_5x5 = {"W": 5, "H": 5, "slip": 0.1, "racks": [[4, 4], [0, 4]], "feed": [2, 0], "seed": 7}
