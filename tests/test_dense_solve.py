"""The host QP's dense solve (csrc/linalg.cpp): the blocked, multi-threaded elimination used
for KKT systems of dimension >= 128 (the C3/C4 sandwich QPs) must return exactly the bits of
the unblocked elimination (common.hpp:47-125 restated), on random systems and across host
thread counts. The replay tests (test_sandwich_replay.py) cover it inside the real QPs."""
import os
import subprocess

import pytest

from paper_2305_04397_b200 import build
from tests.helpers import ROOT


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    build.build_all()
    out = str(tmp_path_factory.mktemp("dense") / "dense_equiv")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"-I{build.CSRC}", f"-I{build.JSON_DIR}",
                    os.path.join(ROOT, "tests", "cpp", "dense_equiv.cpp"), f"-L{build.PKG}", "-lmorap_host",
                    "-lmorap_cuda", f"-Wl,-rpath,{build.PKG}", "-o", out], check=True)
    return out


@pytest.mark.parametrize("threads", ["1", "3", "8"])
def test_blocked_solve_bitwise_equal(exe, threads):
    r = subprocess.run([exe], env={**os.environ, "MORAP_HOST_THREADS": threads}, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
