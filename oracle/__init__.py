"""TEST INFRASTRUCTURE ONLY -- the checkers for the B200 hot path.

Two checkers live here, both CPU-only:

* ``vi`` -- ctypes bindings to ``oracle/libvi_oracle.so``, the plain-C restatement of the
  reference's value-iteration numerics (``vi_oracle.c``; numerics.hpp:74-168,224-234,
  model.hpp:163-206).
* ``ref`` -- ctypes bindings to ``oracle/_ref/libmorap_ref.so``, the UNMODIFIED reference
  headers (/root/reference/proj/include) compiled with a thin shim (``ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this package, and only as the checker / CPU baseline.
The product path (``paper_2305_04397_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
VI_SO = os.path.join(HERE, "libvi_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmorap_ref.so")

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile the C restatement and (when /root/reference exists) the reference shim."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


@dataclass
class Csr:
    """One product MDP in the reference CSR layout (model.hpp:19-34,143-157)."""

    rowOffset: np.ndarray
    trnOffset: np.ndarray
    succ: np.ndarray
    prob: np.ndarray
    done: np.ndarray
    initial: int
    cost: np.ndarray | None = None
    success: np.ndarray | None = None
    accept: np.ndarray | None = None
    rewardFinite: bool = True
    rewards: list = field(default_factory=list)  # extra objective vectors (K > 2 extension)

    @property
    def S(self) -> int:
        return int(self.rowOffset.shape[0] - 1)

    @property
    def R(self) -> int:
        return int(self.trnOffset.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.succ.shape[0])


class _Vi:
    def __init__(self) -> None:
        if not os.path.exists(VI_SO):
            build()
        lib = C.CDLL(VI_SO)
        lib.vo_optimize.restype = C.c_int
        lib.vo_optimize.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _i32p, _i32p, _i32p, _f64p, _u8p,
                                    C.c_int, _f64p, C.c_double, C.c_int, _f64p, _i32p,
                                    C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.vo_evaluate.restype = C.c_int
        lib.vo_evaluate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _i32p, _i32p, _i32p, _f64p, _u8p,
                                    _i32p, _f64p, C.c_double, C.c_int, _f64p,
                                    C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.vo_reward_finite.restype = C.c_int
        lib.vo_reward_finite.argtypes = [C.c_int, C.c_int, _i32p, _i32p, _i32p, _u8p]
        lib.vo_weighted_reward.restype = None
        lib.vo_weighted_reward.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_void_p), _f64p, _f64p]
        lib.vo_optimize_batch.restype = C.c_int
        self.lib = lib

    def weighted_reward(self, parts, w) -> np.ndarray:
        parts = [np.ascontiguousarray(p, dtype=np.float64) for p in parts]
        R = parts[0].shape[0]
        ptrs = (C.c_void_p * len(parts))(*[p.ctypes.data for p in parts])
        out = np.empty(R, dtype=np.float64)
        self.lib.vo_weighted_reward(R, len(parts), ptrs, np.ascontiguousarray(w, dtype=np.float64), out)
        return out

    def optimize(self, m: Csr, rho, eps=1e-6, cap=100000):
        """optimalSchedulerOn (numerics.hpp:74). Returns (rc, values, policy, sweeps, residual, value)."""
        vals = np.zeros(m.S, dtype=np.float64)
        pol = np.zeros(m.S, dtype=np.int32)
        sw, res, val = C.c_int(0), C.c_double(0), C.c_double(0)
        rc = self.lib.vo_optimize(m.S, m.R, m.nnz, m.initial, m.rowOffset, m.trnOffset, m.succ, m.prob,
                                  m.done, int(m.rewardFinite), np.ascontiguousarray(rho, dtype=np.float64),
                                  eps, cap, vals, pol, C.byref(sw), C.byref(res), C.byref(val))
        return rc, vals, pol, sw.value, res.value, val.value

    def evaluate(self, m: Csr, policy, rho, eps=1e-6, cap=100000):
        """evaluateSchedulerOn (numerics.hpp:130) for a deterministic policy."""
        vals = np.zeros(m.S, dtype=np.float64)
        sw, res, val = C.c_int(0), C.c_double(0), C.c_double(0)
        rc = self.lib.vo_evaluate(m.S, m.R, m.nnz, m.initial, m.rowOffset, m.trnOffset, m.succ, m.prob,
                                  m.done, np.ascontiguousarray(policy, dtype=np.int32),
                                  np.ascontiguousarray(rho, dtype=np.float64), eps, cap, vals,
                                  C.byref(sw), C.byref(res), C.byref(val))
        return rc, vals, sw.value, res.value, val.value

    def reward_finite(self, m: Csr) -> bool:
        return bool(self.lib.vo_reward_finite(m.S, m.R, m.rowOffset, m.trnOffset, m.succ, m.done))

    def optimize_batch(self, models, rhos, eps=1e-6, cap=100000, threads=1):
        """Multi-threaded batch of optimize jobs (cpu_baseline 'port'). Returns (rc, values, sweeps, backups)."""
        n = len(models)
        I = C.c_int * n
        P = C.c_void_p * n
        keep = [np.ascontiguousarray(r, dtype=np.float64) for r in rhos]
        vals = np.zeros(n, dtype=np.float64)
        sweeps = np.zeros(n, dtype=np.int32)
        backups = C.c_double(0)
        rc = self.lib.vo_optimize_batch(
            C.c_int(n), I(*[m.S for m in models]), I(*[m.R for m in models]), I(*[m.nnz for m in models]),
            I(*[m.initial for m in models]), P(*[m.rowOffset.ctypes.data for m in models]),
            P(*[m.trnOffset.ctypes.data for m in models]), P(*[m.succ.ctypes.data for m in models]),
            P(*[m.prob.ctypes.data for m in models]), P(*[m.done.ctypes.data for m in models]),
            P(*[r.ctypes.data for r in keep]), C.c_double(eps), C.c_int(cap), C.c_int(threads),
            vals.ctypes.data_as(C.c_void_p), sweeps.ctypes.data_as(C.c_void_p), C.byref(backups))
        return rc, vals, sweeps, backups.value


class RefInstance:
    """A MorapInstance built by the reference (instance.hpp:42 / warehouse.hpp:176)."""

    def __init__(self, lib, handle):
        self._lib = lib
        self._h = handle
        self.n = lib.ref_instance_n(handle)
        self.real_tasks = lib.ref_instance_real_tasks(handle)
        self.distinct = lib.ref_instance_distinct(handle)

    def __del__(self):
        try:
            self._lib.ref_instance_free(self._h)
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, self._lib.ref_last_error().decode())

    def product_dims(self, i, j):
        dims = np.zeros(5, dtype=np.int64)
        h = C.c_uint64(0)
        self._check(self._lib.ref_product_dims(self._h, i, j, dims.ctypes.data_as(C.c_void_p), C.byref(h)))
        return dims, h.value

    def product_slot(self, i, j) -> int:
        return int(self._lib.ref_product_slot(self._h, i, j))

    def product(self, i, j) -> Csr:
        dims, h = self.product_dims(i, j)
        S, R, nnz, initial, fin = (int(x) for x in dims)
        m = Csr(np.zeros(S + 1, np.int32), np.zeros(R + 1, np.int32), np.zeros(nnz, np.int32),
                np.zeros(nnz, np.float64), np.zeros(S, np.uint8), initial,
                np.zeros(R, np.float64), np.zeros(R, np.float64), np.zeros(S, np.uint8), bool(fin))
        v = C.c_void_p
        self._check(self._lib.ref_product_export(
            self._h, i, j, m.rowOffset.ctypes.data_as(v), m.trnOffset.ctypes.data_as(v), m.succ.ctypes.data_as(v),
            m.prob.ctypes.data_as(v), m.cost.ctypes.data_as(v), m.success.ctypes.data_as(v),
            m.done.ctypes.data_as(v), m.accept.ctypes.data_as(v)))
        m.structural_hash = h
        return m

    def optimize(self, i, j, wc, ws, eps=1e-6, cap=100000):
        S = int(self.product_dims(i, j)[0][0])
        vals = np.zeros(S, np.float64)
        pol = np.zeros(S, np.int32)
        sw, res, val = C.c_int(0), C.c_double(0), C.c_double(0)
        v = C.c_void_p
        rc = self._lib.ref_optimize(self._h, i, j, C.c_double(wc), C.c_double(ws), C.c_double(eps), cap,
                                    vals.ctypes.data_as(v), pol.ctypes.data_as(v), C.byref(sw), C.byref(res),
                                    C.byref(val))
        return rc, vals, pol, sw.value, res.value, val.value

    def evaluate(self, i, j, policy, which, eps=1e-6, cap=100000):
        S = int(self.product_dims(i, j)[0][0])
        vals = np.zeros(S, np.float64)
        pol = np.ascontiguousarray(policy, dtype=np.int32)
        sw, res, val = C.c_int(0), C.c_double(0), C.c_double(0)
        v = C.c_void_p
        rc = self._lib.ref_evaluate(self._h, i, j, pol.ctypes.data_as(v), which, C.c_double(eps), cap,
                                    vals.ctypes.data_as(v), C.byref(sw), C.byref(res), C.byref(val))
        return rc, vals, sw.value, res.value, val.value

    def optimize_phase(self, w, workers=0):
        wv = np.ascontiguousarray(w, dtype=np.float64)
        sec, bk = C.c_double(0), C.c_double(0)
        self._check(self._lib.ref_optimize_phase(self._h, wv.ctypes.data_as(C.c_void_p), workers,
                                                 C.byref(sec), C.byref(bk)))
        return sec.value, bk.value

    def supporting_point(self, w, workers=0):
        wv = np.ascontiguousarray(w, dtype=np.float64)
        r = np.zeros(2 * self.n, np.float64)
        a = np.zeros(self.n, np.int32)
        sec = C.c_double(0)
        v = C.c_void_p
        self._check(self._lib.ref_supporting_point(self._h, wv.ctypes.data_as(v), workers, r.ctypes.data_as(v),
                                                   a.ctypes.data_as(v), C.byref(sec)))
        return r, a, sec.value

    def query_backups(self, report, workers=0):
        """Backups of a recorded query on the reference engine (ref_query_backups):
        (optimize sweeps x nnz, evaluate sweeps x states), summed over its iterations."""
        its = report["iterations"]
        w = np.ascontiguousarray([it["w"] for it in its], np.float64)
        a = np.ascontiguousarray([it["assignment"] for it in its], np.int32)
        ob, eb = C.c_double(), C.c_double()
        self._lib.ref_query_backups.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                                C.c_void_p]
        rc = self._lib.ref_query_backups(self._h, w.ctypes.data_as(C.c_void_p), a.ctypes.data_as(C.c_void_p),
                                         len(its), workers, C.byref(ob), C.byref(eb))
        self._check(rc)
        return ob.value, eb.value

    def pareto(self, thresholds, eps=0.01, norm=None, workers=0, iter_cap=500, verify=False):
        t = np.ascontiguousarray(thresholds, dtype=np.float64)
        nm = None if norm is None else np.ascontiguousarray(norm, dtype=np.float64)
        buf = C.create_string_buffer(1 << 24)
        sec = C.c_double(0)
        v = C.c_void_p
        rc = self._lib.ref_pareto(self._h, t.ctypes.data_as(v), t.shape[0],
                                  None if nm is None else nm.ctypes.data_as(v), C.c_double(eps), workers,
                                  iter_cap, int(verify), buf, len(buf), C.byref(sec))
        self._check(rc)
        out = json.loads(buf.value.decode())
        out["seconds"] = sec.value
        return out


    # ---- centralised model (centralised.hpp) ------------------------------------------
    def centralised_dims(self, guard=10000000):
        dims = np.zeros(6, np.int64)
        self._check(self._lib.ref_centralised_dims(self._h, guard, dims.ctypes.data_as(C.c_void_p)))
        return dims

    def centralised(self, guard=10000000) -> dict:
        S, R, nnz, initial, fin, K = (int(x) for x in self.centralised_dims(guard))
        out = {"rowOffset": np.zeros(S + 1, np.int32), "trnOffset": np.zeros(R + 1, np.int32),
               "succ": np.zeros(nnz, np.int32), "prob": np.zeros(nnz), "done": np.zeros(S, np.uint8),
               "rewards": np.zeros((K, R)), "initial": initial, "rewardFinite": bool(fin)}
        v = C.c_void_p
        self._check(self._lib.ref_centralised_export(
            self._h, guard, out["rowOffset"].ctypes.data_as(v), out["trnOffset"].ctypes.data_as(v),
            out["succ"].ctypes.data_as(v), out["prob"].ctypes.data_as(v), out["done"].ctypes.data_as(v),
            out["rewards"].ctypes.data_as(v)))
        return out

    def centralised_pareto(self, thresholds, eps=0.01, iter_cap=500, guard=10000000):
        t = np.ascontiguousarray(thresholds, dtype=np.float64)
        buf = C.create_string_buffer(1 << 24)
        sec = C.c_double(0)
        self._check(self._lib.ref_centralised_pareto(self._h, guard, t.ctypes.data_as(C.c_void_p), t.shape[0],
                                                     C.c_double(eps), iter_cap, buf, len(buf), C.byref(sec)))
        out = json.loads(buf.value.decode())
        out["seconds"] = sec.value
        return out


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


class _Ref:
    def __init__(self) -> None:
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_instance_from_json.restype = C.c_void_p
        lib.ref_instance_from_json.argtypes = [C.c_char_p]
        lib.ref_instance_warehouse.restype = C.c_void_p
        lib.ref_instance_warehouse.argtypes = [C.c_char_p]
        lib.ref_instance_free.argtypes = [C.c_void_p]
        for name in ("ref_instance_n", "ref_instance_real_tasks", "ref_instance_distinct"):
            getattr(lib, name).argtypes = [C.c_void_p]
        lib.ref_product_slot.restype = C.c_int64
        lib.ref_product_slot.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.ref_product_dims.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_product_export.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 8
        lib.ref_optimize.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_evaluate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_int,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_optimize_phase.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_supporting_point.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_pareto.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_double, C.c_int, C.c_int,
                                   C.c_int, C.c_char_p, C.c_int, C.c_void_p]
        lib.ref_max_assignment.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_centralised_dims.argtypes = [C.c_void_p, C.c_long, C.c_void_p]
        lib.ref_centralised_export.argtypes = [C.c_void_p, C.c_long] + [C.c_void_p] * 6
        lib.ref_centralised_pareto.argtypes = [C.c_void_p, C.c_long, C.c_void_p, C.c_int, C.c_double, C.c_int,
                                               C.c_char_p, C.c_int, C.c_void_p]
        self.lib = lib

    def _wrap(self, h):
        if not h:
            raise RefError(-1, self.lib.ref_last_error().decode())
        return RefInstance(self.lib, h)

    def warehouse(self, config: dict) -> RefInstance:
        return self._wrap(self.lib.ref_instance_warehouse(json.dumps(config).encode()))

    def from_json(self, text: str) -> RefInstance:
        return self._wrap(self.lib.ref_instance_from_json(text.encode()))

    def max_assignment(self, c) -> np.ndarray:
        c = np.ascontiguousarray(c, dtype=np.float64)
        n = c.shape[0]
        out = np.zeros(n, np.int32)
        rc = self.lib.ref_max_assignment(n, c.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
        if rc:
            raise RefError(rc, self.lib.ref_last_error().decode())
        return out

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())

    def pareto_core(self, thresholds, n, query, eps=0.01, norm=None, iter_cap=500, verify=False) -> dict:
        """runParetoCore (solver.hpp:192) over a Python supporting-point source
        query(w) -> (r, agent_of), same callback contract as the product's morap_pareto_core."""
        t = np.ascontiguousarray(thresholds, np.float64)
        d = t.shape[0]
        nm = None if norm is None else np.ascontiguousarray(norm, np.float64)
        proto = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double),
                            C.POINTER(C.c_int32), C.c_int)

        def cb(user, wp, dd, rp, ap, nn):
            try:
                r, a = query(np.ctypeslib.as_array(wp, shape=(dd,)).copy())
                np.ctypeslib.as_array(rp, shape=(dd,))[:] = r
                np.ctypeslib.as_array(ap, shape=(nn,))[:] = a
                return 0
            except Exception:  # noqa: BLE001
                return 1

        fn = proto(cb)
        self.lib.ref_pareto_core.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_double, C.c_int, C.c_int,
                                             proto, C.c_void_p, C.c_char_p, C.c_int]
        buf = C.create_string_buffer(1 << 24)
        rc = self.lib.ref_pareto_core(t.ctypes.data_as(C.c_void_p), d, n,
                                      None if nm is None else nm.ctypes.data_as(C.c_void_p), eps, iter_cap,
                                      int(verify), fn, None, buf, len(buf))
        if rc:
            raise RefError(rc, self.lib.ref_last_error().decode())
        return json.loads(buf.value.decode())


_vi = None
_ref = None


def vi() -> _Vi:
    global _vi
    if _vi is None:
        _vi = _Vi()
    return _vi


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)
