"""The restated Pareto sandwich loop and its geometry QPs (csrc/solver.cpp runParetoCore,
csrc/geometry.cpp projectToLowerApprox / weightVector / projectToUpperApprox) against the
reference's own runParetoCore (solver.hpp:192-266, geometry.hpp:99-333, via oracle/_ref)
at the dimensions of the measured configurations: D = 20 (C2), 150 (C3, K = 3, n = 50) and
200 (C4). The supporting-point source is a synthetic convex point cloud shaped like
warehouse results (costs in [-20, 0], probabilities in [0, 1]); both sides call the same
Python callback, so every weight vector, tUp / tDown, lambda* and the verdict must agree bit
for bit. CPU-only: no Bellman work is involved."""
import numpy as np
import pytest

import oracle
from paper_2305_04397_b200 import api

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def cloud(K, n, m, seed):
    rng = np.random.default_rng(seed)
    d = K * n
    P = np.empty((m, d))
    P[:, :(K - 1) * n] = -20.0 * rng.random((m, (K - 1) * n))
    P[:, (K - 1) * n:] = rng.random((m, n))
    A = rng.integers(0, n, size=(m, n)).astype(np.int32)

    def query(w):
        k = int(np.argmax(P @ w))  # first maximum: identical on both sides
        return P[k], A[k]

    return query


CASES = [
    # (K, n, cost threshold, prob threshold, eps, norm seed or None)
    (2, 10, -20.0, 0.99, 0.01, None),   # C2 shape (D = 20), infeasible
    (2, 10, -12.0, 0.4, 0.01, None),    # C2 shape, feasible side
    (2, 10, -15.0, 0.8, 1e-3, 3),       # non-identity norm
    (3, 50, -4.0, 0.9, 0.01, None),     # C3 shape (D = 150)
    (2, 100, -4.0, 0.9, 0.01, None),    # C4 shape (D = 200)
]


@pytest.mark.parametrize("K,n,tc,tp,eps,nseed", CASES)
def test_sandwich_matches_reference(K, n, tc, tp, eps, nseed):
    q = cloud(K, n, 300, 11 * K + n)
    thr = np.array([tc] * ((K - 1) * n) + [tp] * n)
    norm = None
    if nseed is not None:
        rng = np.random.default_rng(nseed)
        B = rng.random((K * n, K * n)) * 0.1
        norm = B @ B.T + np.eye(K * n)
    want = oracle.ref().pareto_core(thr, n, q, eps=eps, norm=norm, iter_cap=40)
    got = api.pareto_core(thr, n, q, eps=eps, norm=norm, iteration_cap=40)
    assert len(want["iterations"]) >= 2
    for key in ("feasible", "converged", "tUp", "tDown", "lambdaStar", "thresholds", "iterations"):
        assert got[key] == want[key], key
    assert [r["tUp"] for r in got["records"]] == [r["tUp"] for r in want["records"]]
    assert [r["tDown"] for r in got["records"]] == [r["tDown"] for r in want["records"]]


def test_verify_mode_matches_reference():
    q = cloud(3, 50, 300, 5)
    for tc, tp in ((-4.0, 0.9), (-15.0, 0.2)):
        thr = np.array([tc] * 100 + [tp] * 50)
        want = oracle.ref().pareto_core(thr, 50, q, eps=0.01, iter_cap=60, verify=True)
        got = api.pareto_core(thr, 50, q, eps=0.01, iteration_cap=60, verify=True)
        assert got["verdict"] == want["verdict"]
        assert [it["w"] for it in got["iterations"]] == [it["w"] for it in want["iterations"]]
