"""Replay a recorded Pareto query's sandwich loop on the host (no GPU): the supporting
point of iteration t is the one the GPU query returned (tests/golden/replay/*.npz, written
by scripts/probe_full_query.py). The loop must ask for exactly the recorded weight vectors
-- bit for bit -- and end with the recorded tUp / tDown / lambda*.

    python scripts/replay_sandwich.py tests/golden/replay/c3_query.npz [ours|ref|both] [iters]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")


def replay(path, which="ours", iters=None):
    z = np.load(path)
    W, R, A = z["w"], z["r"], z["assignment"]
    n = int(z["n"])
    T = len(W) if iters is None else min(int(iters), len(W))
    state = {"t": 0, "bad": None}

    def query(w):
        t = state["t"]
        if t >= T:
            raise RuntimeError("more iterations than recorded")
        if w.tobytes() != W[t].tobytes() and state["bad"] is None:
            state["bad"] = t
        state["t"] = t + 1
        return R[t], A[t]

    cap = T + 1 if T == len(W) else T  # a full replay ends with the converging projection
    t0 = time.perf_counter()
    if which == "ref":
        import oracle
        rep = oracle.ref().pareto_core(z["thresholds"], n, query, eps=float(z["eps"]), iter_cap=cap)
    else:
        from paper_2305_04397_b200 import api
        rep = api.pareto_core(z["thresholds"], n, query, eps=float(z["eps"]), iteration_cap=cap)
    sec = time.perf_counter() - t0
    full = T == len(W)
    ok = state["bad"] is None and len(rep["iterations"]) == T
    diffs = []
    if full:
        if rep["converged"] != bool(z["converged"]) or rep["feasible"] != bool(z["feasible"]):
            diffs.append("verdict")
        for key in ("tUp", "tDown", "lambdaStar"):
            a, b = np.array(rep[key], np.float64), z[key]
            if a.shape != b.shape or a.tobytes() != b.tobytes():
                d = np.abs(a - b).max() if a.shape == b.shape else None
                diffs.append(f"{key} (max abs diff {d})")
    rep["diffs"] = diffs
    ok = ok and not diffs
    return ok, sec, state["bad"], rep


if __name__ == "__main__":
    path = sys.argv[1]
    which = sys.argv[2] if len(sys.argv) > 2 else "ours"
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else None
    for w in (["ours", "ref"] if which == "both" else [which]):
        ok, sec, bad, rep = replay(path, w, iters)
        print(f"{w}: match={ok} seconds={sec:.2f} first_mismatch={bad} iterations={len(rep['iterations'])} "
              f"diffs={rep['diffs']}", flush=True)
