"""Replays of the recorded C3 (D = 150) and C4 (D = 200) GPU queries on the host
(scripts/replay_sandwich.py; tests/golden/replay/*.npz hold each iteration's supporting
point as the B200 returned it): the reference's own runParetoCore (oracle/_ref) and the
product's restatement must ask for exactly the recorded weight vectors, bit for bit. The
full replays (230 / 232 iterations, ending with the recorded tUp / tDown / lambda*) are
logged in profiles/r02_replay_*.log; here the first iterations keep the CPU suite short."""
import os
import sys

import pytest

import oracle
from tests.helpers import GOLDEN, ROOT

sys.path.insert(0, os.path.join(ROOT, "scripts"))
from replay_sandwich import replay  # noqa: E402

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("name,iters", [("c3", 30), ("c4", 20)])
@pytest.mark.parametrize("which", ["ours", "ref"])
def test_replay_reproduces_weight_sequence(name, iters, which):
    ok, sec, bad, rep = replay(os.path.join(GOLDEN, "replay", f"{name}_query.npz"), which, iters)
    assert bad is None and ok, (name, which, bad, rep.get("diffs"))
