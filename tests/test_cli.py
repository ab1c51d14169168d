"""The CLI verbs (cli.py, mirroring cli.hpp:196-327): argument handling on CPU; on the GPU,
`bench` over the warehouse suite and `solve` on fig2 reproduce the reference's golden
reports (verdict, iteration count, tUp/tDown bit for bit)."""
import json
import subprocess
import sys

import pytest

from tests.helpers import GOLDEN, ROOT, load_golden


def _run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2305_04397_b200", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=600)


def test_cli_help_and_bad_config(tmp_path):
    r = _run("--help")
    assert r.returncode == 0 and "solve" in r.stdout and "bench" in r.stdout
    bad = tmp_path / "bad.json"
    bad.write_text("{}")
    r = _run("bench", "--config", str(bad))
    assert r.returncode != 0 and "runs" in r.stderr


@pytest.mark.gpu
def test_cli_bench_suite_matches_reference():
    r = _run("bench", "--config", f"{GOLDEN}/warehouse_suite.json")
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout)["runs"]
    want = load_golden("pareto.json")["suite"]
    assert len(got) == len(want)
    for g, w in zip(got, want):
        res = w["result"]
        assert (g["feasible"], g["converged"], g["iterations"]) == (res["feasible"], res["converged"],
                                                                    len(res["iterations"]))
        assert g["tUp"] == res["tUp"] and g["tDown"] == res["tDown"]


@pytest.mark.gpu
def test_cli_solve_fig2_matches_reference(tmp_path):
    case = load_golden("pareto.json")["fig2"][0]
    out = tmp_path / "res.json"
    r = _run("solve", "--instance", f"{GOLDEN}/fig2.json", "--thresholds=" + ",".join(map(str, case["thresholds"])),
             "--eps", str(case["eps"]), "--out", str(out))
    assert r.returncode == 0, r.stderr
    got = json.loads(out.read_text())
    res = case["result"]
    assert got["tDown"] == res["tDown"] and got["feasible"] == res["feasible"]
    assert got["iterationCount"] == len(res["iterations"]) and got["eps"] == case["eps"]
    assert [it["w"] for it in got["iterations"]] == [it["w"] for it in res["iterations"]]
