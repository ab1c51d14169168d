"""The sharded multi-GPU query (paper_2305_04397_b200/distributed.py) on CPU: world_size 2
over gloo. The per-rank device backend is replaced by the CPU oracle (test
infrastructure) -- what is under test is the sharding, the bit-preserving exchange, the
identical Hungarian / host loop on every rank. Results must equal the reference's own
Pareto runs exactly (tests/golden/pareto.json)."""
import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from tests.helpers import load_golden


class OracleBackend:
    """CudaBackend stand-in backed by oracle/vi_oracle.c (tests only)."""

    def __init__(self):
        self.vi = oracle.vi()
        self.models = []

    def upload(self, prods):
        base = len(self.models)
        for p in prods:
            self.models.append(oracle.Csr(p.rowOffset, p.trnOffset, p.succ, p.prob, p.done, p.initial, p.cost,
                                          p.success, p.accept, p.rewardFinite))
        return np.arange(base, base + len(prods), dtype=np.int32)

    def optimize(self, ids, weights, eps=1e-6, cap=100000):
        self.last = []
        out = [np.zeros(len(ids)), np.zeros(len(ids), np.int32), np.zeros(len(ids)), np.zeros(len(ids), np.int32)]
        for q, (mid, w) in enumerate(zip(ids, weights)):
            m = self.models[mid]
            rc, v, pol, sw, res, v0 = self.vi.optimize(m, self.vi.weighted_reward([m.cost, m.success], w), eps, cap)
            self.last.append((m, pol))
            out[0][q], out[1][q], out[2][q], out[3][q] = v0, sw, res, rc
        return tuple(out)

    def evaluate_optimized(self, jobs, objectives, eps=1e-6, cap=100000):
        n, k = len(jobs), len(objectives)
        val, sw, res, st = np.zeros((n, k)), np.zeros((n, k), np.int32), np.zeros((n, k)), np.zeros((n, k), np.int32)
        for q, j in enumerate(jobs):
            m, pol = self.last[j]
            for o, obj in enumerate(objectives):
                rc, v, s, r, v0 = self.vi.evaluate(m, pol, m.cost if obj == 0 else m.success, eps, cap)
                val[q, o], sw[q, o], res[q, o], st[q, o] = v0, s, r, rc
        return val, sw, res, st


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_path, mode="full"):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_04397_b200.api import Instance
        from paper_2305_04397_b200.distributed import _Exchange, pareto_sharded

        if mode == "shard":  # every rank builds only its own products
            inst = Instance.warehouse_shard(case["config"], rank, world, chunk=3)
        else:
            inst = Instance.warehouse(case["config"])
        res, q = pareto_sharded(inst, case["thresholds"], case["eps"], rank, world, backend=OracleBackend(),
                                exchange=_Exchange(world, "cpu"))
        with open(f"{out_path}.{rank}", "w") as f:
            json.dump({"result": res, "local": q.stats["local_products"]}, f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("which,mode", [(3, "full"), (6, "full"), (6, "shard")])
def test_sharded_query_world2_matches_reference(which, mode):
    case = load_golden("pareto.json")["suite"][which]  # n = 2 and n = 3 warehouse runs
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res")
        mp.spawn(_worker, args=(2, _free_port(), case, out, mode), nprocs=2, join=True)
        got = [json.load(open(f"{out}.{r}")) for r in range(2)]
    n = case["config"]["n"]
    assert got[0]["local"] + got[1]["local"] == n * n and min(g["local"] for g in got) > 0
    for g in got:  # both ranks ran the same loop
        res, ref = g["result"], case["result"]
        for key in ("feasible", "converged", "tUp", "tDown", "lambdaStar", "iterations"):
            assert res[key] == ref[key], key


def test_lpt_partition_balances():
    from paper_2305_04397_b200.distributed import lpt_partition

    w = [5, 4, 3, 3, 2, 2, 1]
    own = lpt_partition(w, 3)
    loads = [sum(x for x, o in zip(w, own) if o == r) for r in range(3)]
    assert max(loads) - min(loads) <= 2 and sorted(set(own)) == [0, 1, 2]
