"""The multi-GPU Pareto query in the host library (csrc/shard.cpp) on a B200:

* one process driving several devices (MultiSolver / morap_multi_*): here two CUDA contexts
  on device 0 -- two shards whose batches never wait on each other, only the host joins them;
* one process per GPU (shard_pareto / morap_shard_pareto) at world size 2: two ranks as two
  host threads with their own contexts on device 0 exchanging through an in-process
  allgather, and as two processes over torch.distributed gloo.

Every variant must equal the reference's golden C2 run (tests/golden/c2.json) bit for bit:
the same weight sequence, supporting points, assignments, tUp / tDown / lambda*."""
import os
import socket
import tempfile
import threading
import json

import numpy as np
import pytest

from tests.helpers import load_golden

pytestmark = pytest.mark.gpu

KEYS = ("feasible", "converged", "tUp", "tDown", "lambdaStar", "iterations")


def _report(rep):
    return {k: rep.get(k) for k in KEYS}


@pytest.fixture(scope="module")
def c2():
    from paper_2305_04397_b200.api import Instance
    g = load_golden("c2.json")
    return g, Instance.warehouse(g["config"])


def test_multi_device_query_matches_reference(c2):
    from paper_2305_04397_b200.api import MultiSolver
    g, inst = c2
    case = g["pareto"]
    m = MultiSolver([0, 0])
    m.upload(inst)
    owners = {m.owner(i, j) for i in range(inst.n) for j in range(inst.n)}
    assert owners == {0, 1}, "both shards own products"
    rep = m.pareto(inst, case["thresholds"], eps=case["eps"])
    assert _report(rep) == _report(case["result"])
    assert rep["stats"]["optimize_jobs"] == 13 * 100
    m.close()


def test_sharded_ranks_in_process_match_reference(c2):
    """world 2, one host thread per rank, an in-process allgather (the exchange contract of
    morap_shard_pareto: recv[r * count + k] = rank r's send[k])."""
    from paper_2305_04397_b200.api import Solver, shard_pareto
    g, inst = c2
    case = g["pareto"]
    world = 2
    slots = [None] * world
    bar = threading.Barrier(world)

    def make_allgather(rank):
        def allgather(send):
            slots[rank] = send
            bar.wait()
            out = np.stack([slots[r] for r in range(world)])
            bar.wait()
            return out
        return allgather

    solvers = [Solver(0) for _ in range(world)]
    reps, errs = [None] * world, []

    def run(rank):
        try:
            reps[rank] = shard_pareto(solvers[rank], inst, rank, world, make_allgather(rank), case["thresholds"],
                                      eps=case["eps"])
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for rep in reps:
        assert _report(rep) == _report(case["result"])
    # the work is split: each rank optimized only its own products' jobs
    assert 0 < reps[0]["stats"]["optimize_jobs"] < 13 * 100
    assert reps[0]["stats"]["optimize_jobs"] + reps[1]["stats"]["optimize_jobs"] == 13 * 100
    for s in solvers:
        s.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    from paper_2305_04397_b200.api import Instance, Solver, shard_pareto
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = load_golden("c2.json")
    case = g["pareto"]
    inst = Instance.warehouse(g["config"])

    def allgather(send):
        t = torch.from_numpy(send)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return torch.stack(out).numpy()

    rep = shard_pareto(Solver(0), inst, rank, world, allgather, case["thresholds"], eps=case["eps"])
    with open(f"{out_path}.{rank}", "w") as f:
        json.dump({"report": _report(rep), "jobs": rep["stats"]["optimize_jobs"]}, f)
    dist.destroy_process_group()


def test_sharded_ranks_gloo_processes_match_reference():
    import torch.multiprocessing as mp
    g = load_golden("c2.json")
    world = 2
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "rep")
        mp.spawn(_gloo_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        got = [json.load(open(f"{out}.{r}")) for r in range(world)]
    want = _report(g["pareto"]["result"])
    assert all(x["report"] == want for x in got)
    assert sum(x["jobs"] for x in got) == 13 * 100 and all(x["jobs"] > 0 for x in got)
