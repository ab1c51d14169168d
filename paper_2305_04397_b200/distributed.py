"""Multi-GPU Pareto query: the n^2 agent x task products sharded across ranks.

One process per GPU (torch.distributed; NCCL on GPUs, gloo in the CPU tests). The products
are independent, so each rank owns a subset -- assigned by LPT on nnz --
and keeps them resident on its GPU for the whole query. Per Algorithm-1 iteration
(solver.hpp:103-184, supportingPoint):

  1. every rank optimizes the (deduplicated) jobs of the pairs (i, j) it owns;
  2. the n^2 initial-state values are exchanged with ONE all_gather (values + ownership
     mask, so each entry keeps its exact bits);
  3. every rank runs the same host Hungarian (maxAssignment) -> identical assignment;
  4. the owner of each assigned pair evaluates its policy under all K objectives (fused
     multi-RHS device batch) and the K*n results are exchanged with a second all_gather.

The sandwich loop itself (runParetoCore, projections, weight vectors) runs redundantly on
every rank through morap_pareto_core with this query as the supporting-point source, so
all ranks see the same w sequence. There is no per-sweep communication.
"""
from __future__ import annotations

import os

import numpy as np

from .api import Instance, max_assignment, pareto_core
from .errors import MorapError


def lpt_partition(weights, world: int):
    """Longest-processing-time assignment of items (by weight) to `world` bins."""
    order = sorted(range(len(weights)), key=lambda k: (-weights[k], k))
    load = [0.0] * world
    owner = [0] * len(weights)
    for k in order:
        r = min(range(world), key=lambda b: (load[b], b))
        owner[k] = r
        load[r] += weights[k]
    return owner


class _Exchange:
    """all_gather of float64 arrays that preserves bits, over the default process group: one
    collective and one device-to-host copy per exchange."""

    def __init__(self, world: int, device):
        import torch

        self.torch = torch
        self.world = world
        self.device = device

    def gather(self, values: np.ndarray, mask: np.ndarray) -> np.ndarray:
        """values/mask: flat arrays; entry k is taken from the (unique) rank whose mask is set."""
        torch = self.torch
        import torch.distributed as dist

        m = values.shape[0]
        t = torch.from_numpy(np.concatenate([values.astype(np.float64), mask.astype(np.float64)])).to(self.device)
        out = torch.empty(self.world * 2 * m, dtype=torch.float64, device=self.device)
        dist.all_gather_into_tensor(out, t)
        a = out.cpu().numpy().reshape(self.world, 2 * m)
        sel = a[:, m:] > 0.5
        if not np.all(sel.sum(axis=0) == 1):
            raise MorapError(14, "sharded exchange: every entry needs exactly one owner")
        return np.take_along_axis(a[:, :m], np.argmax(sel, axis=0)[None, :], axis=0)[0]  # owner's exact bits


class ShardedQuery:
    """Supporting-point source (w -> (r, agent_of)) over products sharded across ranks.
    Per-iteration work on the host is vectorised (numpy) over the n^2 pairs."""

    def __init__(self, inst: Instance, rank: int, world: int, device: int = 0, backend=None, exchange=None,
                 eps: float = 1e-6, sweep_cap: int = 100000):
        self.inst, self.rank, self.world = inst, rank, world
        self.n, self.K = inst.n, inst.objectives
        self.eps, self.cap = eps, sweep_cap
        n = self.n
        # distinct products (slot of first occurrence) and their owners
        slot = np.zeros((n, n), np.int64)
        firsts, sizes, states = [], [], []
        for i in range(n):
            for j in range(n):
                dims, _ = inst.product_dims(i, j)
                first = int(dims[5])
                slot[i, j] = first
                if first == i * n + j:
                    firsts.append(first)
                    sizes.append(float(dims[2]))
                    states.append(int(dims[0]))
        if inst.product_owner(0, 0) >= 0:  # built per rank (Instance.warehouse_shard): its owners
            owner = {f: inst.product_owner(f // n, f % n) for f in firsts}
            if any(o < 0 or o >= world for o in owner.values()):
                raise MorapError(18, "instance was sharded for a different world size")
        else:
            owner = dict(zip(firsts, lpt_partition(sizes, world)))
        self.slot = slot
        self.local = [f for f in firsts if owner[f] == rank]
        self.owner_of_slot = owner
        self.nnz_of_slot = dict(zip(firsts, sizes))
        self.states_of_slot = dict(zip(firsts, states))
        if backend is None:
            from .cuda import CudaBackend

            backend = CudaBackend(device)
            backend.set_lean(True)  # the query needs weighted optimize + chain evaluate only
        self.be = backend
        self.upload()
        # per pair: owned here?, device model id
        own = np.vectorize(lambda f: owner[f] == rank)(slot) if n else np.zeros((0, 0), bool)
        self.mine = own.astype(bool)
        if exchange is None:
            import torch

            exchange = _Exchange(world, torch.device("cuda", device) if torch.cuda.is_available() else "cpu")
        self.ex = exchange
        self.stats = {"optimize_backups": 0.0, "evaluate_state_backups": 0.0, "local_products": len(self.local)}
        # objective coordinates g_k(i, j) (SURVEY.md §8a K-objective extension; K = 2: solver.hpp:118-119)
        ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        self.coords = np.stack([k * n + ii if k < self.K - 1 else (self.K - 1) * n + jj for k in range(self.K)], -1)

    def upload(self) -> int:
        """(Re-)upload this rank's products from their host arrays; returns the CSR bytes."""
        n = self.n
        if getattr(self, "model_of", None) is not None and hasattr(self.be, "release_models"):
            self.be.release_models()
        if getattr(self, "_prods", None) is None:  # host buffers of this rank's products, kept
            self._prods = [self.inst.product(f // n, f % n) for f in self.local]
            if self.K > 2:  # device objective order: cost, extras, success (weights w[g_k(i, j)])
                for f, p in zip(self.local, self._prods):
                    p.objectives = [self.inst.objective(f // n, f % n, k) for k in range(self.K)]
        prods = self._prods
        measured = hasattr(self.be, "stats")
        before = self.be.stats()["upload_bytes"] if measured else 0.0
        ids = self.be.upload(prods) if prods else []
        self.model_of = {f: int(m) for f, m in zip(self.local, ids)}
        self.model_nnz = np.array([self.nnz_of_slot[f] for f in self.local], np.float64)
        self.model_states = np.array([self.states_of_slot[f] for f in self.local], np.float64)
        self.model_index = {f: q for q, f in enumerate(self.local)}
        if measured:  # the bytes the upload actually copied (lean compact layout)
            return int(self.be.stats()["upload_bytes"] - before)
        return sum(4 * (p.S + 1) + 4 * (p.R + 1) + 12 * p.nnz + p.S + 16 * p.R for p in prods)

    def __call__(self, w):
        n, K = self.n, self.K
        w = np.asarray(w, dtype=np.float64)
        if w.shape[0] != K * n:
            raise MorapError(9, "weight vector must have one entry per objective")
        if not np.all(np.isfinite(w)) or abs(np.abs(w).sum() - 1.0) > 1e-6:
            raise MorapError(18, "weight vector must be finite with unit 1-norm")
        # 1. local optimize jobs, deduplicated on (product, weight bits) as solver.hpp:110-131
        pi, pj = np.nonzero(self.mine)
        wk = w[self.coords[pi, pj]]  # (pairs, K)
        vals = np.zeros(n * n)
        mask = np.zeros(n * n)
        job = np.zeros(pi.shape[0], np.int64)
        models = np.zeros(0, np.int32)
        if pi.size:
            key = np.concatenate([self.slot[pi, pj][:, None].astype(np.uint64), wk.view(np.uint64)], axis=1)
            uniq, first, job = np.unique(key, axis=0, return_index=True, return_inverse=True)
            job = job.reshape(-1)
            slots = self.slot[pi, pj][first]
            midx = np.array([self.model_index[int(f)] for f in slots], np.int64)
            models = np.array([self.model_of[int(f)] for f in slots], np.int32)
            v, sw, res, st = self.be.optimize(models, wk[first], self.eps, self.cap)
            if np.any(st != 0):
                raise MorapError(int(st[st != 0][0]), "weighted optimization failed")
            vals[pi * n + pj] = v[job]
            mask[pi * n + pj] = 1.0
            self.stats["optimize_backups"] += float(np.dot(sw.astype(np.float64), self.model_nnz[midx]))
        # 2. exchange the n^2 values, 3. identical Hungarian everywhere
        c = self.ex.gather(vals, mask).reshape(n, n)
        agent_of = max_assignment(c)
        # 4. owners evaluate their assigned pairs under all K objectives (fused multi-RHS)
        r = np.zeros(K * n)
        rmask = np.zeros(K * n)
        jobs_of_pair = {(int(a), int(b)): int(q) for a, b, q in zip(pi, pj, job)}
        mine = [(j, int(agent_of[j])) for j in range(n) if (int(agent_of[j]), j) in jobs_of_pair]
        if mine:
            qs = [jobs_of_pair[(i, j)] for j, i in mine]
            ev, esw, eres, est = self.be.evaluate_optimized(qs, tuple(range(K)), self.eps, self.cap)
            if np.any(est != 0):
                raise MorapError(int(est[est != 0][0]), "evaluation failed")
            for q, (j, i) in enumerate(mine):
                self.stats["evaluate_state_backups"] += float(np.sum(esw[q])) * \
                    self.states_of_slot[int(self.slot[i, j])]
                cc = self.coords[i, j]
                r[cc] = ev[q, :K]
                rmask[cc] = 1.0
        r = self.ex.gather(r, rmask)
        return r, agent_of


def torch_allgather(world: int, device):
    """allgather for shard_pareto over the default torch.distributed group (NCCL over
    NVLink with a CUDA device, gloo with "cpu"); float64 bits are carried unchanged."""
    import torch
    import torch.distributed as dist

    def allgather(send: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(send).to(device)
        out = torch.empty(world * t.numel(), dtype=torch.float64, device=device)
        dist.all_gather_into_tensor(out, t)
        return out.cpu().numpy().reshape(world, -1)

    return allgather


class _ShardRun:
    def __init__(self, rep, solver):
        st = rep["stats"]
        self.solver = solver
        self.stats = {"optimize_backups": st["optimize_backups"], "evaluate_state_backups": st["evaluate_state_backups"],
                      "optimize_jobs": st["optimize_jobs"], "local_products": 0}


def pareto_sharded(inst: Instance, thresholds, eps: float, rank: int, world: int, device: int = 0, backend=None,
                   exchange=None, iteration_cap: int = 500, verify: bool = False, solver=None):
    """paretoPoint (solver.hpp:281) over products sharded across ranks. On GPUs (no test
    backend given) this rank's part runs in the host library (morap_shard_pareto: shard
    optimize -> allgather -> Hungarian -> owner evaluate -> allgather, csrc/shard.cpp) with
    torch.distributed carrying the exchanges; a `backend` (the CPU oracle of the CPU tests)
    runs the same protocol in ShardedQuery."""
    t = np.asarray(thresholds, np.float64)
    if inst.real_tasks != inst.n or t.shape[0] != inst.objectives * inst.n:
        raise MorapError(9, "sharded query expects n real tasks and K*n thresholds (expandThresholds identity)")
    if backend is None and exchange is None and not verify:
        import torch

        from .api import Solver, shard_pareto
        if solver is None:
            solver = Solver(device)
            solver.set_fingerprints(False)
        dev = torch.device("cuda", device) if torch.cuda.is_available() else "cpu"
        rep = shard_pareto(solver, inst, rank, world, torch_allgather(world, dev), t, eps=eps,
                           iteration_cap=iteration_cap)
        run = _ShardRun(rep, solver)
        n = inst.n
        owners = [inst.product_owner(f // n, f % n) for f in range(n * n)]
        run.stats["local_products"] = len({inst.product_dims(f // n, f % n)[0][5] for f in range(n * n)
                                           if (owners[f] < 0 and world == 1) or owners[f] == rank})
        return rep, run
    q = ShardedQuery(inst, rank, world, device, backend, exchange)
    return pareto_core(t, inst.n, q, eps=eps, iteration_cap=iteration_cap, verify=verify), q


# ------------------------------------------------------------------------------------------
def bench_main(args, rank: int, world: int, local: int):
    """bench.py --gpus N under torchrun: sharded C2-family query, max-over-ranks timing.
    Every rank builds only its own products (Instance.warehouse_shard; for --workload c4 on its
    GPU, Instance.warehouse_device_shard -- then there is no host copy and no e2e leg)."""
    import json

    import torch
    import torch.distributed as dist

    import bench as B

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, thr, eps, K = B.workload(args.workload, world)
    threads = max(1, (os.cpu_count() or 1) // world)  # ranks share the host cores
    from .api import Solver, shard_pareto
    solver = Solver(local)
    solver.set_fingerprints(False)
    device_built = args.workload == "c4"  # C4 sharded: each rank builds its own products on its GPU
    if device_built:
        inst = Instance.warehouse_device_shard(cfg, solver, rank, world)
    else:
        inst = Instance.warehouse_shard(cfg, rank, world, threads=threads)
    stream = torch.cuda.current_stream()
    solver.set_stream(stream.cuda_stream)
    allgather = torch_allgather(world, torch.device("cuda", local))
    thr = np.array(thr, np.float64)
    cap = B.ITER_CAP.get(args.workload, 500)
    for _ in range(max(args.warmup, 0)):
        shard_pareto(solver, inst, rank, world, allgather, thr, eps=eps, iteration_cap=cap)

    def timed(steps, reupload):
        solver.reset_cuda_stats()
        backups = 0.0
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            if reupload:
                solver.release()  # the next query re-uploads this rank's products (host image)
            rep = shard_pareto(solver, inst, rank, world, allgather, thr, eps=eps, iteration_cap=cap)
            backups += rep["stats"]["optimize_backups"] + rep["stats"]["evaluate_state_backups"]
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        cs = solver.cuda_stats()
        ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        tot = torch.tensor([backups, float(cs["kernels"]), float(cs["upload_bytes"]), float(cs["d2h_bytes"])],
                           device="cuda", dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        return float(ms.item()), [float(x) for x in tot.tolist()], rep

    with B.ClockSampler(local) as clk:
        ms, (bk, kernels, _, _), rep = timed(args.steps, False)
    e2e_steps = max(1, args.steps)
    if device_built:  # no host copy of the products to re-upload: no end-to-end leg
        e_ms, e_bk, h2d, d2h = None, None, None, None
    else:
        e_ms, (e_bk, _, h2d, d2h), _ = timed(e2e_steps, True)
    if rank == 0:
        n = inst.n
        print(json.dumps({
            "metric": B.METRIC, "value": bk / (ms * 1e-3), "unit": B.UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded warehouse generator)",
            "config": {"workload": args.workload, "grid": [cfg["W"], cfg["H"]], "agents": n, "tasks": n,
                       "objectives": K, "parallelism": f"products sharded over {world} GPUs (greedy by nnz; "
                                                       "morap_shard_pareto, NCCL allgather of the n^2 values "
                                                       "and the K*n evaluations per iteration)",
                       "pareto_iterations": len(rep["iterations"]), "feasible": rep["feasible"],
                       "products": inst.distinct, "nnz": inst.total_nnz,
                       "value_counts": "optimize + evaluate backups summed over ranks / max-over-ranks device time"},
            "e2e": None if device_built else {
                "value": e_bk / (e_ms * 1e-3), "unit": B.UNIT, "h2d_bytes_per_step": h2d / e2e_steps,
                "d2h_bytes_per_step": d2h / e2e_steps, "steps": e2e_steps, "ms_per_step": e_ms / e2e_steps,
                "note": "every rank re-uploads its products from host memory each step (the library's "
                        "copy calls, summed over ranks); exchanges through NCCL allgather"},
            "gpu_launches": int(kernels),
            "clocks": clk.summary(),
        }))
    dist.destroy_process_group()
