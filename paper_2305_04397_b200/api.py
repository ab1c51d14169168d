"""Python face of the host library (libmorap_host.so, include/morap.h).

Mirrors the reference's user-level API (model loader, Pareto-point query):

    inst = Instance.warehouse({"W": 10, "H": 10, "n": 10, ...})   # generateInstance
    inst = Instance.from_json(text, base_dir)                      # instanceFromJson
    solver = Solver(device=0); solver.upload(inst)
    r, agent_of = solver.supporting_point(inst, w)                 # supportingPoint
    report = solver.pareto(inst, thresholds, eps=0.01)             # paretoPoint
    verdict = solver.verify(inst, thresholds, eps=0.01)            # verifyOnly

Errors raise MorapError carrying the reference's Errc (common.hpp:12-34).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from .cuda import load_library as _load_cuda
from .errors import MorapError

PKG = os.path.dirname(os.path.abspath(__file__))
HOST_SO = os.environ.get("MORAP_HOST_SO", os.path.join(PKG, "libmorap_host.so"))  # (A/B builds: scripts/)

QUERY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double),
                       C.POINTER(C.c_int32), C.c_int)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double))

_lib = None


def load_host_library() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(HOST_SO):
        raise FileNotFoundError(f"{HOST_SO} missing: run `python -m paper_2305_04397_b200.build` (no CPU fallback)")
    _load_cuda()  # libmorap_cuda.so first (rpath also finds it)
    lib = C.CDLL(HOST_SO)
    p, i32, f64, u64 = C.c_void_p, C.c_int, C.c_double, C.c_uint64
    sig = {
        "morap_last_error": (C.c_char_p, []),
        "morap_instance_warehouse": (i32, [C.c_char_p, i32, C.POINTER(p)]),
        "morap_instance_from_json": (i32, [C.c_char_p, C.c_char_p, C.POINTER(p), p, i32, C.POINTER(C.c_int)]),
        "morap_instance_from_json_device": (i32, [C.c_char_p, C.c_char_p, p, C.POINTER(p), p, i32,
                                                  C.POINTER(C.c_int)]),
        "morap_instance_free": (None, [p]),
        "morap_instance_info": (i32, [p, p]),
        "morap_instance_product_dims": (i32, [p, i32, i32, p, C.POINTER(u64)]),
        "morap_instance_product_export": (i32, [p, i32, i32, p, p, p, p, p, p, p, p]),
        "morap_instance_add_objectives": (i32, [p, i32, u64]),
        "morap_instance_product_objective": (i32, [p, i32, i32, i32, p]),
        "morap_solver_create": (i32, [i32, C.POINTER(p)]),
        "morap_solver_free": (None, [p]),
        "morap_solver_cuda": (p, [p]),
        "morap_solver_upload": (i32, [p, p]),
        "morap_solver_release": (i32, [p]),
        "morap_solver_set_lean": (i32, [p, i32]),
        "morap_solver_set_fingerprints": (i32, [p, i32]),
        "morap_instance_warehouse_shard": (i32, [C.c_char_p, i32, i32, i32, i32, C.POINTER(p)]),
        "morap_instance_product_owner": (i32, [p, i32, i32]),
        "morap_instance_warehouse_streamed": (i32, [C.c_char_p, i32, p, i32, C.POINTER(p)]),
        "morap_instance_warehouse_device": (i32, [C.c_char_p, p, C.POINTER(p)]),
        "morap_instance_warehouse_device_shard": (i32, [C.c_char_p, p, i32, i32, C.POINTER(p)]),
        "morap_multi_warehouse_device": (i32, [p, C.c_char_p, C.POINTER(p)]),
        "morap_supporting_point": (i32, [p, p, p, i32, p, p, p]),
        "morap_pareto": (i32, [p, p, p, i32, p, f64, i32, i32, C.c_char_p, i32, p]),
        "morap_pareto_core": (i32, [p, i32, i32, p, f64, i32, i32, QUERY_FN, p, C.c_char_p, i32]),
        "morap_max_assignment": (i32, [i32, p, p]),
        "morap_run_batch": (i32, [p, p, i32, p, p, p, p]),
        "morap_centralised_build": (i32, [p, C.c_int64, C.POINTER(p)]),
        "morap_centralised_free": (None, [p]),
        "morap_centralised_info": (i32, [p, p]),
        "morap_centralised_export": (i32, [p, p, p, p, p, p, p]),
        "morap_centralised_pareto": (i32, [p, p, p, i32, p, f64, i32, C.c_char_p, i32, p]),
        "morap_multi_create": (i32, [p, i32, C.POINTER(p)]),
        "morap_multi_free": (None, [p]),
        "morap_multi_upload": (i32, [p, p]),
        "morap_multi_owner": (i32, [p, i32, i32]),
        "morap_multi_pareto": (i32, [p, p, p, i32, p, f64, i32, C.c_char_p, i32, p]),
        "morap_shard_pareto": (i32, [p, p, i32, i32, ALLGATHER_FN, p, p, i32, p, f64, i32, C.c_char_p, i32, p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc != 0:
        raise MorapError(rc, f"{what}: {_lib.morap_last_error().decode()}")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Product:
    """Host copy of one product MDP (ProductMdp, model.hpp:143-157)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    @property
    def S(self):
        return self.rowOffset.shape[0] - 1

    @property
    def R(self):
        return self.trnOffset.shape[0] - 1

    @property
    def nnz(self):
        return self.succ.shape[0]


class Instance:
    """MorapInstance (instance.hpp:20-28) owned by the host library."""

    def __init__(self, handle, norm=None):
        self._lib = load_host_library()
        self.h = handle
        self.norm = norm
        info = np.zeros(8, np.int64)
        _check(self._lib.morap_instance_info(self.h, _ptr(info)), "instance_info")
        (self.n, self.real_tasks, self.distinct, self.objectives, self.total_states, self.total_rows,
         self.total_nnz, self.distinct_nnz) = (int(x) for x in info)

    @classmethod
    def warehouse(cls, config: dict, threads: int = 0) -> "Instance":
        lib = load_host_library()
        h = C.c_void_p()
        _check(lib.morap_instance_warehouse(json.dumps(config).encode(), threads, C.byref(h)), "generateInstance")
        return cls(h)

    @classmethod
    def warehouse_streamed(cls, config: dict, solver: "Solver", chunk: int = 256, threads: int = 0) -> "Instance":
        """Streamed generateInstance for instances too large for a host copy (C4): products
        are built `chunk` at a time, uploaded to `solver` and their host arrays dropped, so
        the instance only answers queries on that solver (morap.h)."""
        lib = load_host_library()
        h = C.c_void_p()
        _check(lib.morap_instance_warehouse_streamed(json.dumps(config).encode(), threads, solver.h, chunk,
                                                     C.byref(h)), "generateInstance (streamed)")
        inst = cls(h)
        inst.streamed = True
        return inst

    @classmethod
    def warehouse_device(cls, config: dict, solver: "Solver") -> "Instance":
        """generateInstance with the products built on `solver`'s GPU (morap.h,
        morap_cuda_build_products): the host never holds a product array, so the instance
        only answers queries on that solver, like a streamed one."""
        lib = load_host_library()
        h = C.c_void_p()
        _check(lib.morap_instance_warehouse_device(json.dumps(config).encode(), solver.h, C.byref(h)),
               "generateInstance (device)")
        inst = cls(h)
        inst.streamed = True
        return inst

    @classmethod
    def warehouse_device_shard(cls, config: dict, solver: "Solver", rank: int, world: int) -> "Instance":
        """Per-rank device build for shard_pareto: the owners warehouse_shard takes, only this
        rank's products built on `solver`'s GPU (morap.h)."""
        lib = load_host_library()
        h = C.c_void_p()
        _check(lib.morap_instance_warehouse_device_shard(json.dumps(config).encode(), solver.h, rank, world,
                                                         C.byref(h)), "generateInstance (device shard)")
        inst = cls(h)
        inst.streamed = True
        return inst

    @classmethod
    def warehouse_shard(cls, config: dict, rank: int, world: int, chunk: int = 256, threads: int = 0) -> "Instance":
        """Per-rank build for the sharded query: host arrays only for this rank's products
        (owners: least-loaded rank by nnz in first-occurrence order, see morap.h)."""
        lib = load_host_library()
        h = C.c_void_p()
        _check(lib.morap_instance_warehouse_shard(json.dumps(config).encode(), threads, rank, world, chunk,
                                                  C.byref(h)), "generateInstance (shard)")
        return cls(h)

    def product_owner(self, i, j) -> int:
        return int(self._lib.morap_instance_product_owner(self.h, i, j))

    @classmethod
    def from_json(cls, text: str, base_dir: str = ".") -> "Instance":
        lib = load_host_library()
        h = C.c_void_p()
        norm = np.zeros(4096, np.float64)
        has = C.c_int(0)
        _check(lib.morap_instance_from_json(text.encode(), base_dir.encode(), C.byref(h), _ptr(norm), norm.shape[0],
                                            C.byref(has)), "instanceFromJson")
        d = has.value
        return cls(h, norm[: d * d].reshape(d, d).copy() if d else None)

    @classmethod
    def from_json_device(cls, text: str, solver: "Solver", base_dir: str = ".") -> "Instance":
        """from_json with the products built on `solver`'s GPU (morap.h)."""
        lib = load_host_library()
        h = C.c_void_p()
        norm = np.zeros(4096, np.float64)
        has = C.c_int(0)
        _check(lib.morap_instance_from_json_device(text.encode(), base_dir.encode(), solver.h, C.byref(h), _ptr(norm),
                                                   norm.shape[0], C.byref(has)), "instanceFromJson (device)")
        d = has.value
        inst = cls(h, norm[: d * d].reshape(d, d).copy() if d else None)
        inst.streamed = True
        return inst

    def close(self):
        if getattr(self, "h", None):
            self._lib.morap_instance_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def add_objectives(self, K: int, seed: int = 0):
        _check(self._lib.morap_instance_add_objectives(self.h, K, seed), "add_objectives")
        self.objectives = K

    def objective(self, i, j, k) -> np.ndarray:
        """Objective vector k of product (i, j): 0 cost, 1..K-2 extras, K-1 success."""
        dims, _ = self.product_dims(i, j)
        out = np.zeros(int(dims[1]))
        _check(self._lib.morap_instance_product_objective(self.h, i, j, k, _ptr(out)), "product_objective")
        return out

    def product_dims(self, i, j):
        dims = np.zeros(6, np.int64)
        h = C.c_uint64(0)
        _check(self._lib.morap_instance_product_dims(self.h, i, j, _ptr(dims), C.byref(h)), "product_dims")
        return dims, h.value

    def product(self, i, j) -> Product:
        dims, h = self.product_dims(i, j)
        S, R, nnz, initial, fin, first = (int(x) for x in dims)
        p = Product(rowOffset=np.zeros(S + 1, np.int32), trnOffset=np.zeros(R + 1, np.int32),
                    succ=np.zeros(nnz, np.int32), prob=np.zeros(nnz), cost=np.zeros(R), success=np.zeros(R),
                    done=np.zeros(S, np.uint8), accept=np.zeros(S, np.uint8), initial=initial,
                    rewardFinite=bool(fin), first_slot=first, structural_hash=h)
        _check(self._lib.morap_instance_product_export(
            self.h, i, j, _ptr(p.rowOffset), _ptr(p.trnOffset), _ptr(p.succ), _ptr(p.prob), _ptr(p.cost),
            _ptr(p.success), _ptr(p.done), _ptr(p.accept)), "product_export")
        return p


class Job(C.Structure):
    """morap_job (include/morap.h): one Job of the reference's engine (engine.hpp:40-54)."""
    _fields_ = [("id", C.c_int64), ("kind", C.c_int32), ("agent", C.c_int32), ("task", C.c_int32),
                ("reward", C.c_void_p), ("reward_len", C.c_int32), ("scheduler", C.c_void_p),
                ("scheduler_len", C.c_int32), ("eps", C.c_double), ("sweep_cap", C.c_int32)]


class JobResult(C.Structure):
    _fields_ = [("id", C.c_int64), ("status", C.c_int32), ("sweeps", C.c_int32), ("value", C.c_double),
                ("residual", C.c_double)]


class Centralised:
    """Centralised model of an instance (buildCentralised, centralised.hpp:54-179)."""

    def __init__(self, inst: Instance, state_guard: int = 10000000):
        self._lib = load_host_library()
        h = C.c_void_p()
        _check(self._lib.morap_centralised_build(inst.h, state_guard, C.byref(h)), "buildCentralised")
        self.h = h
        self.n = inst.n
        info = np.zeros(6, np.int64)
        _check(self._lib.morap_centralised_info(self.h, _ptr(info)), "centralised_info")
        self.S, self.R, self.nnz, self.initial, fin, self.objectives = (int(x) for x in info)
        self.reward_finite = bool(fin)

    def arrays(self) -> dict:
        out = {"rowOffset": np.zeros(self.S + 1, np.int32), "trnOffset": np.zeros(self.R + 1, np.int32),
               "succ": np.zeros(self.nnz, np.int32), "prob": np.zeros(self.nnz), "done": np.zeros(self.S, np.uint8),
               "rewards": np.zeros((self.objectives, self.R))}
        rows = (C.c_void_p * max(1, self.objectives))(*[out["rewards"][k].ctypes.data for k in range(self.objectives)])
        _check(self._lib.morap_centralised_export(self.h, _ptr(out["rowOffset"]), _ptr(out["trnOffset"]),
                                                  _ptr(out["succ"]), _ptr(out["prob"]), _ptr(out["done"]),
                                                  C.cast(rows, C.c_void_p)), "centralised_export")
        return out

    def close(self):
        if getattr(self, "h", None):
            self._lib.morap_centralised_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Solver:
    """One CUDA context with the instance's products resident (GpuBackend)."""

    def __init__(self, device: int = 0):
        self._lib = load_host_library()
        h = C.c_void_p()
        _check(self._lib.morap_solver_create(device, C.byref(h)), "solver_create")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self._lib.morap_solver_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def cuda_ctx(self):
        return self._lib.morap_solver_cuda(self.h)

    def upload(self, inst: Instance):
        _check(self._lib.morap_solver_upload(self.h, inst.h), "upload")

    def release(self):
        _check(self._lib.morap_solver_release(self.h), "release")

    def set_fingerprints(self, on: bool):
        """Scheduler fingerprints in pareto()'s records (on by default; the benchmark turns
        them off: hashing the schedulers is test evidence, not part of paretoPoint)."""
        _check(self._lib.morap_solver_set_fingerprints(self.h, int(on)), "set_fingerprints")

    def set_lean(self, on: bool):
        """Store compact-alphabet products without fp64 prob/objective arrays (morap_cuda_set_lean)."""
        _check(self._lib.morap_solver_set_lean(self.h, int(on)), "set_lean")

    def cuda_stats(self) -> dict:
        from .cuda import load_library
        lib = load_library()
        out = np.zeros(12)
        lib.morap_cuda_stats(self.cuda_ctx, _ptr(out), 12)
        keys = ["opt_launches", "opt_ms", "opt_bytes", "opt_backups", "eval_launches", "eval_ms", "eval_bytes",
                "eval_state_backups", "kernels", "upload_bytes", "opt_exec_backups", "d2h_bytes"]
        return dict(zip(keys, out.tolist()))

    def reset_cuda_stats(self):
        from .cuda import load_library
        load_library().morap_cuda_reset_stats(self.cuda_ctx)

    def set_profiling(self, on: bool):
        from .cuda import load_library
        load_library().morap_cuda_set_profiling(self.cuda_ctx, int(on))

    def set_stream(self, cuda_stream):
        from .cuda import load_library
        load_library().morap_cuda_set_stream(self.cuda_ctx, cuda_stream or None)

    def supporting_point(self, inst: Instance, w):
        w = np.ascontiguousarray(w, np.float64)
        r = np.zeros(inst.objectives * inst.n)
        a = np.zeros(inst.n, np.int32)
        st = np.zeros(8)
        _check(self._lib.morap_supporting_point(self.h, inst.h, _ptr(w), w.shape[0], _ptr(r), _ptr(a), _ptr(st)),
               "supportingPoint")
        self.last_stats = st
        return r, a

    def pareto(self, inst: Instance, thresholds, eps=0.01, norm=None, iteration_cap=500, verify=False) -> dict:
        t = np.ascontiguousarray(thresholds, np.float64)
        nm = None if norm is None else np.ascontiguousarray(norm, np.float64)
        buf = self._json_buffer()
        st = np.zeros(8)
        _check(self._lib.morap_pareto(self.h, inst.h, _ptr(t), t.shape[0], None if nm is None else _ptr(nm), eps,
                                      iteration_cap, int(verify), buf, len(buf), _ptr(st)), "paretoPoint")
        out = json.loads(buf.value.decode())
        out["stats"] = dict(zip(["optimize_jobs", "optimize_backups", "evaluate_jobs", "evaluate_state_backups",
                                 "optimize_s", "evaluate_s", "host_s", "evaluate_batch_s"], st[:8].tolist()))
        return out

    def run_batch(self, inst: Instance, jobs: list) -> list:
        """runBatch (engine.hpp:370) on this GPU. jobs: dicts with id, kind ("optimize" |
        "evaluate"), product (agent, task) or None, reward, scheduler (evaluate), eps,
        sweep_cap. Returns dicts with id, ok, status, value, sweeps, residual, values
        (and policy for optimize jobs) -- failures contained per job (engine.hpp:140-150)."""
        n = len(jobs)
        arr = (Job * max(1, n))()
        keep, vals, pols = [], [], []
        for k, j in enumerate(jobs):
            a = arr[k]
            a.id = int(j["id"])
            a.kind = 1 if j.get("kind") == "evaluate" else 0
            prod = j.get("product")
            a.agent, a.task = (int(prod[0]), int(prod[1])) if prod is not None else (-1, -1)
            rw = np.ascontiguousarray(j.get("reward", []), np.float64)
            sc = np.ascontiguousarray(j.get("scheduler", []), np.int32)
            keep += [rw, sc]
            a.reward, a.reward_len = (rw.ctypes.data if rw.size else None), rw.size
            a.scheduler, a.scheduler_len = (sc.ctypes.data if sc.size else None), sc.size
            a.eps = float(j.get("eps", 1e-6))
            a.sweep_cap = int(j.get("sweep_cap", 100000))
            S = int(inst.product_dims(*prod)[0][0]) if prod is not None else 0
            vals.append(np.zeros(max(S, 1)))
            pols.append(np.zeros(max(S, 1), np.int32))
        res = (JobResult * max(1, n))()
        vp = (C.c_void_p * max(1, n))(*[v.ctypes.data for v in vals])
        pp = (C.c_void_p * max(1, n))(*[q.ctypes.data for q in pols])
        _check(self._lib.morap_run_batch(self.h, inst.h, n, arr, res, C.cast(vp, C.c_void_p), C.cast(pp, C.c_void_p)),
               "runBatch")
        out = []
        for k, j in enumerate(jobs):
            r = res[k]
            d = {"id": int(r.id), "ok": r.status == 0, "status": int(r.status), "value": r.value, "sweeps": r.sweeps,
                 "residual": r.residual}
            if r.status == 0 and j.get("product") is not None:
                d["values"] = vals[k]
                if j.get("kind") != "evaluate":
                    d["policy"] = pols[k]
            out.append(d)
        return out

    def centralised_pareto(self, c: Centralised, thresholds, eps=0.01, norm=None, iteration_cap=500) -> dict:
        """centralisedParetoPoint (centralised.hpp:216-222) on this solver's GPU."""
        t = np.ascontiguousarray(thresholds, np.float64)
        nm = None if norm is None else np.ascontiguousarray(norm, np.float64)
        buf = self._json_buffer()
        st = np.zeros(8)
        _check(self._lib.morap_centralised_pareto(self.h, c.h, _ptr(t), t.shape[0], None if nm is None else _ptr(nm),
                                                  eps, iteration_cap, buf, len(buf), _ptr(st)), "centralisedParetoPoint")
        out = json.loads(buf.value.decode())
        out["stats"] = dict(zip(["optimize_jobs", "optimize_backups", "evaluate_jobs", "evaluate_state_backups",
                                 "optimize_s", "evaluate_s", "host_s", "evaluate_batch_s"], st[:8].tolist()))
        return out

    def _json_buffer(self):
        if getattr(self, "_buf", None) is None:
            self._buf = C.create_string_buffer(1 << 24)
        return self._buf

    def verify(self, inst: Instance, thresholds, eps=0.01, norm=None, iteration_cap=500) -> bool:
        return bool(self.pareto(inst, thresholds, eps, norm, iteration_cap, verify=True)["verdict"])


_STAT_KEYS = ["optimize_jobs", "optimize_backups", "evaluate_jobs", "evaluate_state_backups", "optimize_s",
              "evaluate_s", "host_s", "evaluate_batch_s"]


class MultiSolver:
    """One process driving several GPUs (morap_multi_*): one CUDA context and one host
    thread per device, products sharded by LPT on nnz, results equal Solver.pareto's."""

    def __init__(self, devices):
        self._lib = load_host_library()
        devs = np.ascontiguousarray(list(devices), np.int32)
        h = C.c_void_p()
        _check(self._lib.morap_multi_create(_ptr(devs), devs.shape[0], C.byref(h)), "multi create")
        self.h = h
        self.devices = devs.tolist()

    def close(self):
        if getattr(self, "h", None):
            self._lib.morap_multi_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def upload(self, inst: Instance):
        _check(self._lib.morap_multi_upload(self.h, inst.h), "multi upload")

    def warehouse_device(self, config: dict) -> Instance:
        """generateInstance with every product built on the device that owns it (morap.h:
        morap_multi_warehouse_device); query it with pareto()."""
        h = C.c_void_p()
        _check(self._lib.morap_multi_warehouse_device(self.h, json.dumps(config).encode(), C.byref(h)),
               "generateInstance (multi device)")
        inst = Instance(h)
        inst.streamed = True
        return inst

    def owner(self, i, j) -> int:
        return int(self._lib.morap_multi_owner(self.h, i, j))

    def pareto(self, inst: Instance, thresholds, eps=0.01, norm=None, iteration_cap=500) -> dict:
        t = np.ascontiguousarray(thresholds, np.float64)
        nm = None if norm is None else np.ascontiguousarray(norm, np.float64)
        buf = C.create_string_buffer(1 << 24)
        st = np.zeros(8)
        _check(self._lib.morap_multi_pareto(self.h, inst.h, _ptr(t), t.shape[0], None if nm is None else _ptr(nm), eps,
                                            iteration_cap, buf, len(buf), _ptr(st)), "multi paretoPoint")
        out = json.loads(buf.value.decode())
        out["stats"] = dict(zip(_STAT_KEYS, st[:8].tolist()))
        return out


def shard_pareto(solver: "Solver", inst: Instance, rank: int, world: int, allgather, thresholds, eps=0.01, norm=None,
                 iteration_cap=500) -> dict:
    """This rank's part of the multi-GPU query (morap_shard_pareto): allgather(send) -> recv
    (numpy float64, recv.shape = (world, send.size)) carries the two exchanges per iteration
    (torch.distributed: NCCL on GPUs, gloo on CPU)."""
    lib = load_host_library()
    t = np.ascontiguousarray(thresholds, np.float64)
    nm = None if norm is None else np.ascontiguousarray(norm, np.float64)
    err = []

    def cb(user, sp, count, rp):
        try:
            send = np.ctypeslib.as_array(sp, shape=(count,)).copy()
            recv = np.asarray(allgather(send), np.float64).reshape(world * count)
            np.ctypeslib.as_array(rp, shape=(world * count,))[:] = recv
            return 0
        except Exception as e:  # noqa: BLE001
            err.append(e)
            return 14

    fn = ALLGATHER_FN(cb)
    buf = C.create_string_buffer(1 << 24)
    st = np.zeros(8)
    rc = lib.morap_shard_pareto(solver.h, inst.h, rank, world, fn, None, _ptr(t), t.shape[0],
                                None if nm is None else _ptr(nm), eps, iteration_cap, buf, len(buf), _ptr(st))
    if rc != 0 and err:
        raise err[0]
    _check(rc, "sharded paretoPoint")
    out = json.loads(buf.value.decode())
    out["stats"] = dict(zip(_STAT_KEYS, st[:8].tolist()))
    return out


def pareto_core(thresholds, n, query, eps=0.01, norm=None, iteration_cap=500, verify=False) -> dict:
    """runParetoCore (solver.hpp:192) over a Python supporting-point source
    query(w) -> (r, agent_of). Used by the multi-GPU driver (ranks own product shards)."""
    lib = load_host_library()
    t = np.ascontiguousarray(thresholds, np.float64)
    d = t.shape[0]
    nm = None if norm is None else np.ascontiguousarray(norm, np.float64)
    err = []

    def cb(user, wp, dd, rp, ap, nn):
        try:
            w = np.ctypeslib.as_array(wp, shape=(dd,)).copy()
            r, a = query(w)
            np.ctypeslib.as_array(rp, shape=(dd,))[:] = r
            np.ctypeslib.as_array(ap, shape=(nn,))[:] = a
            return 0
        except MorapError as e:
            err.append(e)
            return e.status
        except Exception as e:  # noqa: BLE001
            err.append(e)
            return 14

    fn = QUERY_FN(cb)
    buf = C.create_string_buffer(1 << 24)
    rc = lib.morap_pareto_core(_ptr(t), d, n, None if nm is None else _ptr(nm), eps, iteration_cap, int(verify), fn,
                               None, buf, len(buf))
    if rc != 0 and err and not isinstance(err[0], MorapError):
        raise err[0]
    _check(rc, "runParetoCore")
    return json.loads(buf.value.decode())


def max_assignment(c) -> np.ndarray:
    lib = load_host_library()
    c = np.ascontiguousarray(c, np.float64)
    if c.ndim != 2 or c.shape[0] != c.shape[1]:
        raise MorapError(10, "assignment needs a square value matrix")
    out = np.zeros(c.shape[0], np.int32)
    _check(lib.morap_max_assignment(c.shape[0], _ptr(c), _ptr(out)), "maxAssignment")
    return out
