"""Dev probe: per-CTA timeline of the compact optimize sweeps (morap_cuda_debug_cta_trace)
for one C2 optimize batch (100 jobs, w = (0.5, 0.5)): per sweep, the span from the first
CTA start to the finalize end, when the CTAs start / get their first stage / finish, and
the finalize time. Args: mode (skip|full), sweep CTAs (148 x 4), workload (c2|cent)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_04397_b200.api import Instance
from paper_2305_04397_b200.cuda import CudaBackend

import bench

mode = sys.argv[1] if len(sys.argv) > 1 else "skip"
work = sys.argv[3] if len(sys.argv) > 3 else "c2"
be = CudaBackend(0)
be.set_lean(True)
if work == "cent":  # the centralised model of bench's `cent` workload, one job
    from types import SimpleNamespace
    from paper_2305_04397_b200.api import Centralised
    cm = Centralised(Instance.warehouse(bench.workload("cent")[0]))
    a = cm.arrays()
    prods = [SimpleNamespace(rowOffset=a["rowOffset"], trnOffset=a["trnOffset"], succ=a["succ"], prob=a["prob"],
                             done=a["done"], initial=cm.initial, rewardFinite=cm.reward_finite,
                             objectives=list(a["rewards"]))]
    K = cm.objectives
else:
    inst = Instance.warehouse(bench.workload("c2")[0])
    prods = [inst.product(i, j) for i in range(10) for j in range(10)]
    K = 2
ids = be.upload(prods)
Wm = np.tile(np.full(K, 1.0 / K), (len(ids), 1))
be.set_skip(mode == "skip")
be.optimize(ids, Wm)
lib = be.lib
assert lib.morap_cuda_debug_cta_trace(be.h, 1, None, 0) == 0
val, sw, res, st = be.optimize(ids, Wm)
n = 128 * 148 * 8 * 4
buf = np.zeros(n, np.uint64)
assert lib.morap_cuda_debug_cta_trace(be.h, 0, buf.ctypes.data_as(C.c_void_p), n) == 0
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 148 * 4  # the compact sweep's grid
T = buf[: 128 * blocks * 4].reshape(128, blocks, 4).astype(np.int64)
rows = []
starts = []
nsw = int(sw.max())
for k in range(max(0, nsw - 128), nsw):  # the slots keep the last 128 sweeps
    t = T[k % 128]
    live = t[:, 0] > 0
    if not live.any():
        continue
    t = t[live]
    t0 = t[:, 0].min()
    fin = t[:, 3].max() - t0
    has = t[:, 1] > 0
    first = (t[has, 1] - t[has, 0]) / 1e3 if has.any() else np.zeros(1)
    end = (t[:, 2] - t0) / 1e3
    rows.append((k + 1, fin / 1e3, (t[:, 0] - t0).max() / 1e3, np.median(first), np.median(end), end.max(),
                 fin / 1e3 - end.max()))
    starts.append((t0, t0 + fin))
print(f"{mode}: CTAs {T.shape[1]}")
print("sweep  span_us  start_spread  first_stage_med  work_end_med  work_end_max  finalize_us")
for r in rows[:: max(1, len(rows) // 12)]:
    print("%5d  %7.1f  %12.1f  %15.1f  %12.1f  %12.1f  %11.1f" % r)
a = np.array(rows)[:, 1:]
print("mean   %7.1f  %12.1f  %15.1f  %12.1f  %12.1f  %11.1f" % tuple(a.mean(0)))
# start-to-start: the sweep plus the k_select launch and the gaps before the next sweep
gaps = [(starts[q + 1][0] - starts[q][1]) / 1e3 for q in range(len(starts) - 1)]
print("per sweep: span_us, then gap to the next sweep's first CTA (k_select + launch gaps)")
print(" ".join("%d:%.1f/%.1f" % (rows[q][0], rows[q][1], gaps[q]) for q in range(len(gaps))))
print("sum span %.1f us, sum gaps %.1f us over %d sweeps" % (sum(r[1] for r in rows), sum(gaps), len(rows)))
