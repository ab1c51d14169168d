"""The sharded multi-GPU query (distributed.py) through the real CUDA backend at world size 1
over NCCL (only one GPU is reachable here; world 2 runs on CPU over gloo in
test_distributed_cpu.py): the C2 bench query must equal the reference's golden run bit for
bit, and a K = 3 query must equal the single-GPU Solver's."""
import os
import socket

import numpy as np
import pytest

from tests.helpers import load_golden

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def pg():
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def _report(rep):
    return {k: rep.get(k) for k in ("feasible", "converged", "tUp", "tDown", "lambdaStar", "iterations")}


def test_sharded_c2_query_matches_reference(pg):
    from paper_2305_04397_b200.api import Instance
    from paper_2305_04397_b200.distributed import pareto_sharded
    c2 = load_golden("c2.json")
    inst = Instance.warehouse(c2["config"])
    case = c2["pareto"]
    rep, q = pareto_sharded(inst, case["thresholds"], case["eps"], 0, 1, 0)
    assert _report(rep) == _report(case["result"])
    assert q.stats["local_products"] == 100 and q.stats["optimize_backups"] > 0


def test_sharded_k3_matches_single_gpu(pg):
    from paper_2305_04397_b200.api import Instance, Solver
    from paper_2305_04397_b200.distributed import pareto_sharded
    cfg = {"W": 6, "H": 6, "n": 3, "slip": 0.05, "racks": [[5, 5], [0, 5], [5, 0]], "feed": [0, 0], "seed": 42}
    inst = Instance.warehouse(cfg)
    inst.add_objectives(3, seed=7)
    thr = [-20.0] * 6 + [0.9] * 3
    want = Solver(0).pareto(inst, thr, eps=0.01, iteration_cap=30)
    got, _ = pareto_sharded(inst, thr, 0.01, 0, 1, 0, iteration_cap=30)
    assert _report(got) == _report(want)
