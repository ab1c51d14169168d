"""The drop-in, proven with the reference's own code: oracle/_ref/ref_gpu_routed
is the reference's supportingPoint / paretoPoint (solver.hpp:103-294, compiled unmodified
from /root/reference) with its two runBatch calls routed to libmorap_cuda.so through the
plug-in integration/morap_gpu_runbatch.hpp (engine.hpp:370's contract). On the GPU its
reports must equal, bit for bit, the goldens the unmodified CPU reference wrote -- fig2, the
warehouse suite and the C2 bench query -- and gpu_runBatch must return runBatch's exact
JobResults. Without a GPU the plug-in must fail loudly (no CPU fallback)."""
import json
import os
import subprocess

import pytest

from tests.helpers import GOLDEN, ROOT, load_golden

BIN = os.path.join(ROOT, "oracle", "_ref", "ref_gpu_routed")
pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/ref_gpu_routed not built")


def _run(*args, timeout=900):
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=timeout)


def _report(rep):
    keys = ("feasible", "converged", "tUp", "tDown", "lambdaStar", "thresholds", "iterations", "synthesis",
            "records", "marginal")
    return {k: rep.get(k) for k in keys}


def test_plugin_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _run("jobs", json.dumps({"W": 6, "H": 6, "n": 2, "slip": 0.05, "racks": [[5, 5], [0, 5], [5, 0]],
                                 "feed": [0, 0], "seed": 42}), timeout=120)
    assert r.returncode == 3 and "GPU backend create" in r.stderr


@pytest.mark.gpu
def test_gpu_runbatch_equals_reference_runbatch():
    cfg = {"W": 6, "H": 6, "n": 3, "slip": 0.05, "racks": [[5, 5], [0, 5], [5, 0]], "feed": [0, 0], "seed": 42}
    r = _run("jobs", json.dumps(cfg))
    assert r.returncode == 0, r.stderr + r.stdout
    out = json.loads(r.stdout)
    assert out["optimize_jobs"] == 36 and out["evaluate_jobs"] == 72 and out["mismatches"] == 0


@pytest.mark.gpu
def test_reference_pareto_routed_to_gpu_fig2_and_suite():
    gold = load_golden("pareto.json")
    for case in gold["fig2"]:
        r = _run("pareto", "fig2", f"{GOLDEN}/fig2.json", ",".join(map(repr, case["thresholds"])), repr(case["eps"]))
        assert r.returncode == 0, r.stderr
        assert _report(json.loads(r.stdout)) == _report(case["result"])
    for case in gold["suite"]:
        r = _run("pareto", "warehouse", json.dumps(case["config"]), ",".join(map(repr, case["thresholds"])),
                 repr(case["eps"]))
        assert r.returncode == 0, r.stderr
        assert _report(json.loads(r.stdout)) == _report(case["result"])


@pytest.mark.gpu
def test_reference_pareto_routed_to_gpu_c2_bench_query():
    c2 = load_golden("c2.json")
    case = c2["pareto"]
    r = _run("pareto", "warehouse", json.dumps(c2["config"]), ",".join(map(repr, case["thresholds"])),
             repr(case["eps"]))
    assert r.returncode == 0, r.stderr
    assert _report(json.loads(r.stdout)) == _report(case["result"])
