"""ctypes binding of the sm_100a backend (libmorap_cuda.so, include/morap_cuda.h).

This is the Python face of the reference's job engine for the hot path: ``upload`` once,
then batches of optimize / evaluate jobs (engine.hpp:370 ``runBatch``; numerics.hpp:74,130).
There is no CPU fallback: constructing a backend without the built library or without an
sm_100 device raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import MorapError

PKG = os.path.dirname(os.path.abspath(__file__))
CUDA_SO = os.path.join(PKG, "libmorap_cuda.so")
MAX_OBJECTIVES = 8
MAX_RHS = 8


class CsrView(C.Structure):
    _fields_ = [
        ("num_states", C.c_int32), ("num_rows", C.c_int32), ("nnz", C.c_int32), ("initial", C.c_int32),
        ("reward_finite", C.c_int32), ("num_objectives", C.c_int32),
        ("row_offset", C.c_void_p), ("trn_offset", C.c_void_p), ("succ", C.c_void_p), ("prob", C.c_void_p),
        ("done", C.c_void_p), ("rewards", C.c_void_p),
    ]


_lib = None


def load_library(path: str = CUDA_SO) -> C.CDLL:
    """Load libmorap_cuda.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("MORAP_CUDA_SO", path)  # kernel-variant experiments (scripts/)
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `python -m paper_2305_04397_b200.build` (no CPU fallback)")
    lib = C.CDLL(path)
    p, i32, f64 = C.c_void_p, C.c_int, C.c_double
    sig = {
        "morap_cuda_create": (i32, [i32, C.POINTER(C.c_void_p)]),
        "morap_cuda_destroy": (i32, [p]),
        "morap_cuda_set_stream": (i32, [p, p]),
        "morap_cuda_last_error": (C.c_char_p, [p]),
        "morap_cuda_upload": (i32, [p, i32, p, p]),
        "morap_cuda_build_image": (i32, [p, i32, p, C.POINTER(C.c_void_p)]),
        "morap_cuda_upload_image": (i32, [p, p, p]),
        "morap_cuda_free_image": (None, [p]),
        "morap_cuda_release_models": (i32, [p]),
        "morap_cuda_num_models": (i32, [p]),
        "morap_cuda_optimize": (i32, [p, i32, p, p, i32, f64, i32, p, p, p, p]),
        "morap_cuda_optimize_rho": (i32, [p, i32, p, p, f64, i32, p, p, p, p]),
        "morap_cuda_fetch_values": (i32, [p, i32, p]),
        "morap_cuda_fetch_policy": (i32, [p, i32, p]),
        "morap_cuda_fetch_policies": (i32, [p, i32, p, p]),
        "morap_cuda_evaluate_optimized": (i32, [p, i32, p, i32, p, f64, i32, p, p, p, p]),
        "morap_cuda_evaluate": (i32, [p, i32, p, p, p, f64, i32, p, p, p, p]),
        "morap_cuda_fetch_eval_values": (i32, [p, i32, i32, p]),
        "morap_cuda_set_profiling": (i32, [p, i32]),
        "morap_cuda_set_lean": (i32, [p, i32]),
        "morap_cuda_set_skip": (i32, [p, i32]),
        "morap_cuda_debug_cta_trace": (i32, [p, i32, p, C.c_int64]),
        "morap_cuda_model_info": (i32, [p, i32, p]),
        "morap_cuda_debug_model_digest": (i32, [p, i32, p]),
        "morap_cuda_build_products": (i32, [p, i32, p, i32, p, p, i32, p, i32, p, p]),
        "morap_cuda_stats": (i32, [p, p, i32]),
        "morap_cuda_reset_stats": (i32, [p]),
        "morap_cuda_device_bytes": (i32, [p, p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def model_objectives(m) -> list:
    """Objective vectors of a product: cost, success (model.hpp:150-151), then extras."""
    objs = getattr(m, "objectives", None)
    if objs is not None:
        return list(objs)
    out = [m.cost, m.success]
    out += list(getattr(m, "rewards", []) or [])
    return out


class CudaBackend:
    """One CUDA context (morap_cuda_create) on `device`."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.morap_cuda_create(device, C.byref(h))
        if rc != 0:
            raise MorapError(rc, f"morap_cuda_create(device={device}) failed (needs an sm_100 GPU)")
        self.h = h
        self.device = device
        self._models = []  # host copies keep sizes for result buffers

    def close(self):
        if getattr(self, "h", None):
            self.lib.morap_cuda_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what=""):
        if rc != 0:
            raise MorapError(rc, f"{what}: {self.lib.morap_cuda_last_error(self.h).decode()}")

    def set_stream(self, cuda_stream: int | None):
        self._check(self.lib.morap_cuda_set_stream(self.h, cuda_stream or None), "set_stream")

    # ---- models -------------------------------------------------------------------------
    def upload(self, models, image: bool = False) -> np.ndarray:
        """morap_cuda_upload; with image=True through morap_cuda_build_image + upload_image
        (the packed image is uploaded twice, after a release, to exercise the re-upload)."""
        views = (CsrView * len(models))()
        keep = []
        for k, m in enumerate(models):
            arrs = [np.ascontiguousarray(m.rowOffset, np.int32), np.ascontiguousarray(m.trnOffset, np.int32),
                    np.ascontiguousarray(m.succ, np.int32), np.ascontiguousarray(m.prob, np.float64),
                    np.ascontiguousarray(m.done, np.uint8)]
            objs = [np.ascontiguousarray(o, np.float64) for o in model_objectives(m)]
            optr = (C.c_void_p * max(1, len(objs)))(*[_ptr(o) for o in objs])
            keep += arrs + objs + [optr]
            v = views[k]
            v.num_states = arrs[0].shape[0] - 1
            v.num_rows = arrs[1].shape[0] - 1
            v.nnz = arrs[2].shape[0]
            v.initial = int(m.initial)
            v.reward_finite = int(bool(getattr(m, "rewardFinite", True)))
            v.num_objectives = len(objs)
            v.row_offset, v.trn_offset, v.succ, v.prob, v.done = [_ptr(a) for a in arrs]
            v.rewards = C.cast(optr, C.c_void_p)
        ids = np.zeros(len(models), np.int32)
        if image:
            img = C.c_void_p()
            self._check(self.lib.morap_cuda_build_image(self.h, len(models), views, C.byref(img)), "build_image")
            try:
                self._check(self.lib.morap_cuda_upload_image(self.h, img, _ptr(ids)), "upload_image")
                self._check(self.lib.morap_cuda_release_models(self.h), "release")
                self._check(self.lib.morap_cuda_upload_image(self.h, img, _ptr(ids)), "upload_image")
            finally:
                self.lib.morap_cuda_free_image(img)
        else:
            self._check(self.lib.morap_cuda_upload(self.h, len(models), views, _ptr(ids)), "upload")
        for m in models:
            self._models.append((int(np.asarray(m.rowOffset).shape[0] - 1), int(np.asarray(m.trnOffset).shape[0] - 1),
                                 len(model_objectives(m))))
        return ids

    def set_lean(self, on: bool):
        """Store compact-alphabet models without their fp64 prob/objective arrays (morap_cuda.h)."""
        self._check(self.lib.morap_cuda_set_lean(self.h, int(on)), "set_lean")

    def set_skip(self, on: bool):
        """Frozen-tile skipping in compact optimize sweeps (bitwise-neutral, morap_cuda.h)."""
        self._check(self.lib.morap_cuda_set_skip(self.h, int(on)), "set_skip")

    def release_models(self):
        self._check(self.lib.morap_cuda_release_models(self.h), "release")
        self._models = []

    def num_states(self, model_id: int) -> int:
        return self._models[model_id][0]

    # ---- optimize -------------------------------------------------------------------------
    def optimize(self, model_ids, weights, eps=1e-6, sweep_cap=100000):
        """Batch of optimize jobs; returns (value, sweeps, residual, status) arrays."""
        ids = np.ascontiguousarray(model_ids, np.int32)
        w = np.ascontiguousarray(weights, np.float64)
        n = ids.shape[0]
        K = w.shape[1] if w.ndim == 2 else (w.shape[0] // max(n, 1))
        val, res = np.zeros(n), np.zeros(n)
        sw, st = np.zeros(n, np.int32), np.zeros(n, np.int32)
        self._opt_models = ids.copy()
        self._check(self.lib.morap_cuda_optimize(self.h, n, _ptr(ids), _ptr(w), K, eps, sweep_cap, _ptr(val),
                                                 _ptr(sw), _ptr(res), _ptr(st)), "optimize")
        return val, sw, res, st

    def optimize_rho(self, model_ids, rhos, eps=1e-6, sweep_cap=100000):
        ids = np.ascontiguousarray(model_ids, np.int32)
        n = ids.shape[0]
        keep = [np.ascontiguousarray(r, np.float64) for r in rhos]
        ptrs = (C.c_void_p * max(1, n))(*[_ptr(r) for r in keep])
        val, res = np.zeros(n), np.zeros(n)
        sw, st = np.zeros(n, np.int32), np.zeros(n, np.int32)
        self._opt_models = ids.copy()
        self._check(self.lib.morap_cuda_optimize_rho(self.h, n, _ptr(ids), ptrs, eps, sweep_cap, _ptr(val),
                                                     _ptr(sw), _ptr(res), _ptr(st)), "optimize_rho")
        return val, sw, res, st

    def fetch_values(self, job: int) -> np.ndarray:
        out = np.zeros(self.num_states(int(self._opt_models[job])), np.float64)
        self._check(self.lib.morap_cuda_fetch_values(self.h, job, _ptr(out)), "fetch_values")
        return out

    def fetch_policy(self, job: int) -> np.ndarray:
        out = np.zeros(self.num_states(int(self._opt_models[job])), np.int32)
        self._check(self.lib.morap_cuda_fetch_policy(self.h, job, _ptr(out)), "fetch_policy")
        return out

    # ---- evaluate -------------------------------------------------------------------------
    def evaluate_optimized(self, opt_jobs, objectives=(0, 1), eps=1e-6, sweep_cap=100000):
        """Fused multi-RHS evaluation of optimize jobs' policies; arrays shaped (njobs, nrhs)."""
        jl = np.ascontiguousarray(opt_jobs, np.int32)
        ob = np.ascontiguousarray(objectives, np.int32)
        n, k = jl.shape[0], ob.shape[0]
        val, res = np.zeros((n, k)), np.zeros((n, k))
        sw, st = np.zeros((n, k), np.int32), np.zeros((n, k), np.int32)
        self._eval_models = [int(self._opt_models[j]) for j in jl]
        self._check(self.lib.morap_cuda_evaluate_optimized(self.h, n, _ptr(jl), k, _ptr(ob), eps, sweep_cap,
                                                           _ptr(val), _ptr(sw), _ptr(res), _ptr(st)),
                    "evaluate_optimized")
        return val, sw, res, st

    def evaluate(self, model_ids, policies, rhos, eps=1e-6, sweep_cap=100000):
        ids = np.ascontiguousarray(model_ids, np.int32)
        n = ids.shape[0]
        pk = [np.ascontiguousarray(p, np.int32) for p in policies]
        rk = [np.ascontiguousarray(r, np.float64) for r in rhos]
        pp = (C.c_void_p * max(1, n))(*[_ptr(p) for p in pk])
        rp = (C.c_void_p * max(1, n))(*[_ptr(r) for r in rk])
        val, res = np.zeros(n), np.zeros(n)
        sw, st = np.zeros(n, np.int32), np.zeros(n, np.int32)
        self._eval_models = [int(i) for i in ids]
        self._check(self.lib.morap_cuda_evaluate(self.h, n, _ptr(ids), pp, rp, eps, sweep_cap, _ptr(val), _ptr(sw),
                                                 _ptr(res), _ptr(st)), "evaluate")
        return val, sw, res, st

    def fetch_eval_values(self, job: int, rhs: int = 0) -> np.ndarray:
        out = np.zeros(self.num_states(self._eval_models[job]), np.float64)
        self._check(self.lib.morap_cuda_fetch_eval_values(self.h, job, rhs, _ptr(out)), "fetch_eval_values")
        return out

    # ---- instrumentation ------------------------------------------------------------------
    def set_profiling(self, on: bool):
        self._check(self.lib.morap_cuda_set_profiling(self.h, int(on)), "set_profiling")

    def stats(self) -> dict:
        out = np.zeros(12)
        self._check(self.lib.morap_cuda_stats(self.h, _ptr(out), 12), "stats")
        keys = ["opt_launches", "opt_ms", "opt_bytes", "opt_backups", "eval_launches", "eval_ms", "eval_bytes",
                "eval_state_backups", "kernels", "upload_bytes", "opt_exec_backups", "d2h_bytes"]
        return dict(zip(keys, out.tolist()))

    def reset_stats(self):
        self._check(self.lib.morap_cuda_reset_stats(self.h), "reset_stats")
