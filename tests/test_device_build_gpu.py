"""Device product builder (morap_cuda_build_products): products built on the GPU
must be the very models the host path uploads -- every array of the device model (CSR,
done flags, probability indices, reward classes, tiles, successor windows, the compact
sweep streams, out-of-window lists) bit for bit against buildProduct (model.hpp:230-321)
+ the host upload preparation -- and the Pareto query on the device-built instance must
return the host-built instance's report exactly. Errors and seeded retries follow
generateInstance (warehouse.hpp)."""
import ctypes as C

import pytest

from paper_2305_04397_b200 import cuda
from paper_2305_04397_b200.api import Instance, Solver
from paper_2305_04397_b200.errors import Errc, MorapError
from tests.helpers import SUITE_5x5, SUITE_6x6, warehouse_config

pytestmark = pytest.mark.gpu

ARRAYS = ["rowOffset", "trnOffset", "succ", "done", "probIdx", "rclass", "tileStart", "tiles", "probDict",
          "classTable", "stW", "rowW", "trW", "tilePos", "outIdx", "outGrp", "outSucc"]

C4_RACKS = [[9 - (k % 10), 9 - (k // 10)] for k in range(100)]
CONFIGS = {
    "suite6x6_n3": {**SUITE_6x6, "n": 3},
    "suite5x5_n2": {**SUITE_5x5, "n": 2},
    "c2_10x10_n10": warehouse_config(10, 10, 10),
    "slip0_8x8_n4": warehouse_config(8, 8, 4, slip=0.0),
    "deadline7_6x6_n3": warehouse_config(6, 6, 3, deadline=7),
    # the (i, j < 4) products of C4 (10 x 10, 100 racks): ~9.5e4 states, ~4.6e5 transitions each
    "c4_sub_n4": {"W": 10, "H": 10, "n": 4, "slip": 0.05, "racks": C4_RACKS, "feed": [0, 0], "seed": 42},
}


def digests(solver):
    lib = cuda.load_library()
    ctx = solver.cuda_ctx
    out = []
    for m in range(lib.morap_cuda_num_models(ctx)):
        d = (C.c_uint64 * 17)()
        assert lib.morap_cuda_debug_model_digest(ctx, m, d) == 0, lib.morap_cuda_last_error(ctx)
        out.append(list(d))
    return out


def host_and_device(cfg):
    host = Instance.warehouse(cfg)
    hs = Solver(0)
    hs.set_lean(True)
    hs.upload(host)
    ds = Solver(0)
    dev = Instance.warehouse_device(cfg, ds)
    return host, hs, dev, ds


@pytest.mark.parametrize("name", list(CONFIGS))
def test_device_models_bitwise(name):
    host, hs, dev, ds = host_and_device(CONFIGS[name])
    assert (dev.n, dev.distinct, dev.total_states, dev.total_rows, dev.total_nnz) == \
           (host.n, host.distinct, host.total_states, host.total_rows, host.total_nnz)
    for i in range(host.n):
        for j in range(host.n):
            # S, R, nnz, initial, rewardFinite, first slot of the product (dedup)
            assert dev.product_dims(i, j)[0].tolist() == host.product_dims(i, j)[0].tolist(), (i, j)
    want, got = digests(hs), digests(ds)
    assert len(got) == len(want) == host.distinct
    for m, (a, b) in enumerate(zip(want, got)):
        bad = [ARRAYS[k] for k in range(17) if a[k] != b[k]]
        assert not bad, f"model {m}: {bad}"


def _strip(rep):
    rep = dict(rep)
    rep.pop("stats", None)
    return rep


@pytest.mark.parametrize("name,thr", [
    ("suite6x6_n3", [-25.0] * 3 + [0.9] * 3),
    ("c2_10x10_n10", [-20.0] * 10 + [0.99] * 10),
])
def test_device_built_query_bitwise(name, thr):
    cfg = CONFIGS[name]
    want = _strip(Solver(0).pareto(Instance.warehouse(cfg), thr, eps=0.01, iteration_cap=40))
    s = Solver(0)
    got = _strip(s.pareto(Instance.warehouse_device(cfg, s), thr, eps=0.01, iteration_cap=40))
    assert got == want


def test_device_build_errors_follow_generate_instance():
    # deadline 0: no product is reward-finite, 10 seeded attempts, GenerationFailure
    cfg = warehouse_config(6, 6, 2, deadline=0)
    with pytest.raises(MorapError) as host_err:
        Instance.warehouse(cfg)
    s = Solver(0)
    with pytest.raises(MorapError) as dev_err:
        Instance.warehouse_device(cfg, s)
    assert dev_err.value.code == host_err.value.code == Errc.GenerationFailure
    assert str(dev_err.value).split(": ", 1)[1] == str(host_err.value).split(": ", 1)[1]
    # the failed attempts left nothing registered on the solver
    assert cuda.load_library().morap_cuda_num_models(s.cuda_ctx) == 0


def test_device_products_have_no_host_copy():
    s = Solver(0)
    inst = Instance.warehouse_device(CONFIGS["suite6x6_n3"], s)
    with pytest.raises(MorapError):
        inst.product(0, 0)
    with pytest.raises(MorapError):
        Solver(0).pareto(inst, [-25.0] * 3 + [0.9] * 3, eps=0.01, iteration_cap=2)


def test_multi_device_build_matches_reference():
    """One process, two contexts on device 0: each builds the products it owns."""
    from paper_2305_04397_b200.api import MultiSolver
    from tests.helpers import load_golden
    g = load_golden("c2.json")
    case = g["pareto"]
    m = MultiSolver([0, 0])
    inst = m.warehouse_device(g["config"])
    owners = {m.owner(i, j) for i in range(inst.n) for j in range(inst.n)}
    assert owners == {0, 1}
    rep = m.pareto(inst, case["thresholds"], eps=case["eps"])
    keys = ("feasible", "converged", "tUp", "tDown", "lambdaStar", "iterations")
    assert {k: rep.get(k) for k in keys} == {k: case["result"].get(k) for k in keys}
    m.close()


def test_device_shard_ranks_match_reference():
    """world 2 as two host threads, each rank building only its own products on its GPU."""
    import threading

    import numpy as np

    from paper_2305_04397_b200.api import shard_pareto
    from tests.helpers import load_golden
    g = load_golden("c2.json")
    case = g["pareto"]
    world = 2
    slots = [None] * world
    bar = threading.Barrier(world)
    reps, errs = [None] * world, []

    def run(rank):
        try:
            s = Solver(0)
            inst = Instance.warehouse_device_shard(g["config"], s, rank, world)
            mine = sum(inst.product_owner(i, j) == rank for i in range(inst.n) for j in range(inst.n))
            assert 0 < mine < inst.n * inst.n

            def allgather(send):
                slots[rank] = send
                bar.wait()
                out = np.stack([slots[r] for r in range(world)])
                bar.wait()
                return out
            reps[rank] = shard_pareto(s, inst, rank, world, allgather, case["thresholds"], eps=case["eps"])
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    keys = ("feasible", "converged", "tUp", "tDown", "lambdaStar", "iterations")
    for rep in reps:
        assert {k: rep.get(k) for k in keys} == {k: case["result"].get(k) for k in keys}
    assert reps[0]["stats"]["optimize_jobs"] + reps[1]["stats"]["optimize_jobs"] == 13 * 100


def test_json_instance_built_on_device_matches_reference():
    """instanceFromJson with the device builder: the fig2 instance (hand-written agent MDP and
    formulas) answers every recorded query of the reference bit for bit, schedulers included."""
    from tests.helpers import GOLDEN, load_golden
    gold = load_golden("pareto.json")
    s = Solver(0)
    inst = Instance.from_json_device(open(f"{GOLDEN}/fig2.json").read(), s)
    host = Instance.from_json(open(f"{GOLDEN}/fig2.json").read())
    assert (inst.n, inst.distinct, inst.total_states, inst.total_nnz) == \
           (host.n, host.distinct, host.total_states, host.total_nnz)
    for case in gold["fig2"]:
        got = s.pareto(inst, case["thresholds"], eps=case["eps"])
        for key in ("feasible", "converged", "tUp", "tDown", "lambdaStar", "thresholds", "iterations", "synthesis",
                    "records"):
            assert got[key] == case["result"][key], key


def _chain_instance(nstates):
    """A chain agent whose every state has its own pair of probabilities: 2 * nstates distinct
    values -- no compact layout above 256 (the host path falls back to fp64 arrays)."""
    import json
    acts = []
    for s in range(nstates):
        p = 0.5 + 1e-4 * (s + 1)
        acts.append({"state": s, "name": "go", "to": [{"s": s + 1, "p": p}, {"s": s, "p": 1.0 - p}], "reward": -1})
    acts.append({"state": nstates, "name": "stay", "to": [{"s": nstates, "p": 1.0}], "reward": -1})
    agent = {"states": nstates + 1, "initial": 0, "labels": {str(nstates): ["goal"]}, "actions": acts}
    return json.dumps({"agents": [agent], "tasks": ["F goal"]})


@pytest.mark.parametrize("nstates,msg", [(200, "compact"), (600, "alphabet")])
def test_device_build_rejects_what_it_cannot_lay_out(nstates, msg):
    text = _chain_instance(nstates)
    host = Instance.from_json(text)  # the host path takes any product
    rep = Solver(0).pareto(host, [-2000.0, 0.5], eps=0.01)
    assert rep["converged"]
    with pytest.raises(MorapError) as err:
        Instance.from_json_device(text, Solver(0))
    assert err.value.code == Errc.InvalidConfig
    assert msg in str(err.value)


@pytest.mark.parametrize("seed", range(24 + 4))
def test_device_models_bitwise_random_configs(seed):
    """Random warehouse layouts (grid, racks, feed, slip, deadline, seed): the device models
    equal the host-prepared ones array for array (the last four at C4-like product sizes)."""
    import random
    rng = random.Random(1000 + seed)
    big = seed >= 24
    W, H = (rng.randint(9, 12), rng.randint(9, 12)) if big else (rng.randint(3, 8), rng.randint(3, 8))
    n = rng.randint(3, 5) if big else rng.randint(1, 4)
    cells = [[x, y] for x in range(W) for y in range(H)]
    rng.shuffle(cells)
    racks = cells[: max(n, rng.randint(n, n + 3))]
    cfg = {"W": W, "H": H, "n": n, "slip": rng.choice([0.0, 0.05, 0.1, 0.25]), "racks": racks,
           "feed": cells[-1], "seed": rng.randint(0, 10000)}
    if rng.random() < 0.5:
        cfg["deadline"] = rng.randint(W + H, 3 * (W + H))
    try:
        host, hs, dev, ds = host_and_device(cfg)
    except MorapError as e:  # the host path rejects it too (e.g. no reward-finite seed)
        with pytest.raises(MorapError) as err:
            Instance.warehouse(cfg)
        assert err.value.code == e.code
        return
    assert (dev.n, dev.distinct, dev.total_states, dev.total_nnz) == (host.n, host.distinct, host.total_states,
                                                                       host.total_nnz)
    want, got = digests(hs), digests(ds)
    for m, (a, b) in enumerate(zip(want, got)):
        bad = [ARRAYS[k] for k in range(17) if a[k] != b[k]]
        assert not bad, f"{cfg}: model {m}: {bad}"
