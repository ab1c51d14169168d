"""Streamed instances (C4 path): products built in chunks, uploaded -- optionally lean --
and dropped on the host must answer the Pareto query with exactly the bits of the
ordinary in-memory instance (morap.h: morap_instance_warehouse_streamed)."""
import pytest

from paper_2305_04397_b200.api import Instance, Solver
from paper_2305_04397_b200.errors import MorapError

pytestmark = pytest.mark.gpu

CFG = {"W": 6, "H": 6, "n": 3, "slip": 0.05, "racks": [[5, 5], [0, 5], [5, 0]], "feed": [0, 0], "seed": 42}
THR = [-25.0, -25.0, -25.0, 0.9, 0.9, 0.9]


def _strip(rep):
    rep = dict(rep)
    rep.pop("stats", None)
    return rep


@pytest.fixture(scope="module")
def reference_report():
    inst = Instance.warehouse(CFG)
    s = Solver(0)
    rep = s.pareto(inst, THR, eps=0.01, iteration_cap=40)
    return inst, _strip(rep)


@pytest.mark.parametrize("lean", [False, True])
@pytest.mark.parametrize("chunk", [1, 4, 9])
def test_streamed_query_bitwise(reference_report, lean, chunk):
    inst0, want = reference_report
    s = Solver(0)
    s.set_lean(lean)
    inst = Instance.warehouse_streamed(CFG, s, chunk=chunk)
    assert (inst.n, inst.distinct, inst.total_states, inst.total_rows, inst.total_nnz) == \
           (inst0.n, inst0.distinct, inst0.total_states, inst0.total_rows, inst0.total_nnz)
    for i in range(inst.n):
        for j in range(inst.n):
            assert inst.product_dims(i, j)[0].tolist() == inst0.product_dims(i, j)[0].tolist()
    got = _strip(s.pareto(inst, THR, eps=0.01, iteration_cap=40))
    assert got == want


def test_streamed_products_have_no_host_copy():
    s = Solver(0)
    inst = Instance.warehouse_streamed(CFG, s, chunk=4)
    with pytest.raises(MorapError):
        inst.product(0, 0)
    with pytest.raises(MorapError):
        inst.add_objectives(3, seed=1)
    # another solver cannot take the products: their only copy is on the first device context
    with pytest.raises(MorapError):
        Solver(0).pareto(inst, THR, eps=0.01, iteration_cap=2)
