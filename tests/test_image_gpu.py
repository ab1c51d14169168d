"""The product builder's packed device image (morap_cuda_build_image / upload_image): the
same models uploaded through an image (and re-uploaded from it after a release) give the
same bits as the packing upload -- optimize values, policies, sweeps, residuals and the
fused evaluations -- on compact warehouse products (lean and full, whose queries never wait
for the image's segment B) and on non-compact random models (whose sweeps read segment B),
and both match the oracle. A warehouse query through the Solver (always via the cached
image) is covered by the golden Pareto tests."""
import numpy as np
import pytest

import oracle
from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.cuda import CudaBackend
from tests.helpers import random_done_model

pytestmark = pytest.mark.gpu


def _models():
    inst = Instance.warehouse({"W": 6, "H": 6, "n": 2, "slip": 0.05, "racks": [[5, 5], [0, 5], [5, 0]],
                               "feed": [0, 0], "seed": 42})
    prods = [inst.product(i, j) for i in range(2) for j in range(2)]
    rng = np.random.default_rng(11)
    return prods, [random_done_model(rng, 60) for _ in range(4)]


def _run(models, lean, image, skip=True):
    be = CudaBackend(0)
    be.set_lean(lean)
    be.set_skip(skip)
    ids = be.upload(models, image=image)
    W = np.tile([0.35, 0.65], (len(ids), 1))
    val, sw, res, st = be.optimize(ids, W, eps=1e-7)
    vals = [be.fetch_values(k).tobytes() for k in range(len(ids))]
    pols = [be.fetch_policy(k).tobytes() for k in range(len(ids))]
    ev = be.evaluate_optimized(list(range(len(ids))), (0, 1), eps=1e-7)
    evv = [be.fetch_eval_values(k, o).tobytes() for k in range(len(ids)) for o in range(2)]
    be.close()
    return (val.tobytes(), sw.tobytes(), res.tobytes(), st.tobytes(), vals, pols,
            [a.tobytes() for a in ev], evv)


@pytest.mark.parametrize("lean", [True, False])
def test_image_upload_equals_packing_upload_on_warehouse_products(lean):
    prods, _ = _models()
    assert _run(prods, lean, image=True) == _run(prods, lean, image=False)


def test_image_upload_equals_packing_upload_on_non_compact_models():
    _, rnd = _models()
    got = _run(rnd, False, image=True)
    assert got == _run(rnd, False, image=False)
    # and the oracle's bits (values / policies / sweeps of the optimize jobs)
    vi = oracle.vi()
    be = CudaBackend(0)
    ids = be.upload(rnd, image=True)
    W = np.tile([0.35, 0.65], (len(ids), 1))
    val, sw, res, st = be.optimize(ids, W, eps=1e-7)
    for k, m in enumerate(rnd):
        rc, v, pol, s, r, v0 = vi.optimize(m, vi.weighted_reward([m.cost, m.success], W[k]), eps=1e-7)
        assert (st[k], sw[k], res[k], val[k]) == (rc, s, r, v0)
        assert be.fetch_values(k).tobytes() == v.tobytes() and be.fetch_policy(k).tobytes() == pol.tobytes()
    be.close()


def test_image_upload_mixed_batch_without_skipping():
    prods, rnd = _models()
    assert _run(prods + rnd, False, image=True, skip=False) == _run(prods + rnd, False, image=False, skip=False)
