"""The CLI verbs (cli.py, mirroring cli.hpp:135-410): argument handling and exit codes on CPU
(test_cli.cpp:86-108); on the GPU, verify / pareto / synth on fig2 (test_cli.cpp:65-84,
110-165) and `bench` over the warehouse suite reproduce the reference's golden reports
(verdict, iteration count, tUp/tDown bit for bit) with exit code 0 feasible / 1 infeasible."""
import json
import subprocess
import sys

import pytest

from tests.helpers import GOLDEN, ROOT, load_golden

FIG2 = f"{GOLDEN}/fig2.json"


def _run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2305_04397_b200", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=600)


def test_cli_help_and_bad_config(tmp_path):
    r = _run("--help")
    assert r.returncode == 0 and "verify" in r.stdout and "pareto" in r.stdout and "bench" in r.stdout
    bad = tmp_path / "bad.json"
    bad.write_text("{}")
    r = _run("bench", "--config", str(bad))
    assert r.returncode == 2 and "runs" in r.stderr


def test_cli_usage_and_input_errors_exit_two():
    """test_cli.cpp:86-108: every usage / input error exits 2 before any device work."""
    r = _run("verify", "--instance", "/nonexistent/nowhere.json", "--thresholds=-1,0.5")
    assert r.returncode == 2 and "error" in r.stderr
    assert _run("verify", "--instance", FIG2, "--thresholds=-1,zebra").returncode == 2
    assert _run("verify", "--instance", FIG2, "--thresholds=-1,-1,0.5,0.5").returncode == 2  # DimensionMismatch
    assert _run().returncode == 2
    assert _run("frobnicate").returncode == 2
    assert _run("verify", "--instance", FIG2).returncode == 2
    # synth has no --centralised flag (test_cli.cpp:299-301)
    assert _run("synth", "--instance", FIG2, "--thresholds=-2.5,0.7", "--centralised").returncode == 2


def test_cli_exit_code_mapping():
    from paper_2305_04397_b200.cli import exit_code_for, pareto_csv
    from paper_2305_04397_b200.errors import Errc, MorapError
    for code, rc in ((Errc.Syntax, 2), (Errc.InvalidConfig, 2), (Errc.DimensionMismatch, 2), (Errc.Io, 2),
                     (Errc.NonConvergence, 3), (Errc.NotCoSafe, 3), (Errc.NotRewardFinite, 3)):
        assert exit_code_for(MorapError(int(code) + 1, "")) == rc
    assert exit_code_for(MorapError(100, "cuda")) == 3
    csv = pareto_csv({"thresholds": [-1.8, 0.9], "iterations": [{"w": [1.0, 0.0], "r": [-1.0, 0.1]}],
                      "tUp": [-1.0, 5 / 7], "tDown": [-1.95429753, 0.612934689]})
    assert csv.splitlines() == ["iter,w_1,w_2,r_1,r_2", "1,1,0,-1,0.1", "tUp,-1,0.714285714",
                                "tDown,-1.95429753,0.612934689"]


@pytest.mark.gpu
def test_cli_verify_fig2_exit_codes():
    """test_cli.cpp:65-84."""
    ok = _run("verify", "--instance", FIG2, "--thresholds=-2.5,0.7")
    assert ok.returncode == 0, ok.stderr
    j = json.loads(ok.stdout)
    assert j["feasible"] and j["converged"] and j["iterationCount"] == 2 and j["thresholds"] == [-2.5, 0.7]
    bad = _run("verify", "--instance", FIG2, "--thresholds=-1.8,0.9")
    assert bad.returncode == 1, bad.stderr
    k = json.loads(bad.stdout)
    assert not k["feasible"]
    assert abs(k["tDown"][0] - -1.9542975) < 1e-4 and abs(k["tDown"][1] - 0.6129347) < 1e-4


@pytest.mark.gpu
def test_cli_pareto_csv_trace(tmp_path):
    """test_cli.cpp:110-148: the CSV trace carries one line per iteration plus tUp / tDown."""
    out = tmp_path / "trace.csv"
    r = _run("pareto", "--instance", FIG2, "--thresholds=-1.8,0.9", "--out", str(out))
    assert r.returncode == 1, r.stderr
    j = json.loads(r.stdout)
    lines = out.read_text().splitlines()
    assert lines[0] == "iter,w_1,w_2,r_1,r_2"
    assert len(lines) == 1 + j["iterationCount"] + 2
    assert lines[-1].startswith("tDown,") and lines[-2].startswith("tUp,")
    for i, it in enumerate(j["iterations"]):
        cells = [float(c) for c in lines[1 + i].split(",")[1:]]
        assert all(abs(a - b) <= 1e-8 * max(1.0, abs(b)) for a, b in zip(cells, it["w"] + it["r"]))


@pytest.mark.gpu
def test_cli_synth_certificate():
    """test_cli.cpp:150-166: a feasible fig2 query yields a certificate over assignments."""
    r = _run("synth", "--instance", FIG2, "--thresholds=-2.5,0.7")
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert j["synthesis"] and abs(sum(t["p"] for t in j["synthesis"]) - 1.0) < 1e-9
    for t in j["synthesis"]:
        assert t["assignment"] == [0]
    assert len(j["marginal"]) == 1 and abs(j["marginal"][0][0] - 1.0) < 1e-9


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
    r = _run("solve", "--instance", FIG2, "--thresholds=" + ",".join(map(str, case["thresholds"])),
             "--eps", str(case["eps"]))
    res = case["result"]
    assert r.returncode == (0 if res["feasible"] else 1), r.stderr
    got = json.loads(r.stdout)
    assert got["tDown"] == res["tDown"] and got["feasible"] == res["feasible"]
    assert got["iterationCount"] == len(res["iterations"]) and got["eps"] == case["eps"]
    assert [it["w"] for it in got["iterations"]] == [it["w"] for it in res["iterations"]]


@pytest.mark.gpu
def test_cli_device_build_same_output(tmp_path):
    case = load_golden("pareto.json")["fig2"][0]
    args = ["pareto", "--instance", FIG2, "--thresholds=" + ",".join(map(str, case["thresholds"])), "--eps",
            str(case["eps"])]
    host, dev = _run(*args), _run(*args, "--device-build")
    assert dev.returncode == host.returncode, dev.stderr
    assert dev.stdout == host.stdout
    b_host = _run("bench", "--config", f"{GOLDEN}/warehouse_suite.json")
    b_dev = _run("bench", "--config", f"{GOLDEN}/warehouse_suite.json", "--device-build")
    assert b_dev.returncode == 0, b_dev.stderr
    strip = ("generateSeconds", "solveSeconds")
    got = [{k: v for k, v in r.items() if k not in strip} for r in json.loads(b_dev.stdout)["runs"]]
    want = [{k: v for k, v in r.items() if k not in strip} for r in json.loads(b_host.stdout)["runs"]]
    assert got == want
