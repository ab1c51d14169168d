"""Every device code path produces the same bits. The kernel variant is chosen when a
CUDA context is created (environment), so each variant runs in its own process:

  default            compact streams, 5-stage TMA pipeline (k_greedy_sweep_cmp)
  MORAP_COMPACT=0    fp64 streams, 2-stage TMA pipeline (k_greedy_sweep_tma)
  MORAP_EVAL_INTERLEAVED=0    per-RHS value layout in the persistent evaluate kernel
  MORAP_GRAPHS=0     sweeps launched one by one instead of CUDA-graph batches
  MORAP_SKIP=0       every tile swept every sweep (no frozen-tile skipping)

Each process runs optimize + fused evaluate on 6x6 warehouse products and random models
and prints fingerprints; all variants must agree with each other and with the oracle."""
import hashlib
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import oracle
from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.cuda import CudaBackend
from tests.helpers import random_done_model
inst = Instance.warehouse({"W": 6, "H": 6, "n": 2, "slip": 0.05, "racks": [[5, 5], [0, 5], [5, 0]],
                           "feed": [0, 0], "seed": 42})
prods = [inst.product(i, j) for i in range(2) for j in range(2)]
rng = np.random.default_rng(5)
prods += [random_done_model(rng, 50) for _ in range(6)]
be = CudaBackend(0)
ids = be.upload(prods)
W = np.array([[0.3, 0.7], [1.0, 0.0], [0.0, 1.0], [0.5, 0.5]] + [[0.6, 0.4]] * 6)
val, sw, res, st = be.optimize(ids, W, eps=1e-7)
h = hashlib.sha256()
for k in range(len(prods)):
    h.update(be.fetch_values(k).tobytes()); h.update(be.fetch_policy(k).tobytes())
ev, esw, eres, est = be.evaluate_optimized(list(range(len(prods))), (0, 1), eps=1e-7)
for k in range(len(prods)):
    for o in range(2):
        h.update(be.fetch_eval_values(k, o).tobytes())
vi = oracle.vi()
ok = True
for k, p in enumerate(prods):
    m = oracle.Csr(p.rowOffset, p.trnOffset, p.succ, p.prob, p.done, p.initial, p.cost, p.success)
    rc, v, pol, s, r, v0 = vi.optimize(m, vi.weighted_reward([m.cost, m.success], W[k]), eps=1e-7)
    ok &= (sw[k], res[k], val[k]) == (s, r, v0) and be.fetch_policy(k).tobytes() == pol.tobytes()
print(json.dumps({"hash": h.hexdigest(), "sweeps": sw.tolist(), "eval": ev.tolist(), "oracle_ok": bool(ok)}))
"""

VARIANTS = {
    "default": {},
    "plain_tma": {"MORAP_COMPACT": "0"},
    "per_rhs_eval": {"MORAP_EVAL_INTERLEAVED": "0"},
    "no_graphs": {"MORAP_GRAPHS": "0"},
    "no_persistent_eval": {"MORAP_PERSISTENT": "0"},
    "no_skip": {"MORAP_SKIP": "0"},
}


def test_all_kernel_variants_agree():
    out = {}
    for name, env in VARIANTS.items():
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=e, capture_output=True, text=True, timeout=300,
                           cwd=ROOT)
        assert r.returncode == 0, (name, r.stderr[-2000:])
        out[name] = json.loads(r.stdout.strip().splitlines()[-1])
        assert out[name]["oracle_ok"], name
    hashes = {k: v["hash"] for k, v in out.items()}
    assert len(set(hashes.values())) == 1, hashes
