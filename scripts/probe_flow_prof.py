"""Dev probe: build a -DMORAP_FLOW_PROF variant of libmorap_cuda.so into /tmp, run C2
optimize batches through it and print where the dataflow kernel's warps wait (clock64
totals averaged over CTAs): producer ring wait / segment resolution / stage-refill wait /
booking; compute warp 0: full-barrier wait / tile compute / tiles per CTA."""
import ctypes as C
import os
import json
import subprocess
import sys

import numpy as np

sys.path.insert(0, ".")
so = "/tmp/libmorap_cuda_prof.so"
subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                "-fmad=false", "-DMORAP_FLOW_PROF", "-Xcompiler", "-fPIC,-O3,-mavx2,-ffp-contract=off", "-shared", "-o", so,
                "paper_2305_04397_b200/csrc/morap_cuda.cu"], check=True)
import paper_2305_04397_b200.cuda as cu  # noqa: E402
os.environ["MORAP_CUDA_SO"] = so
import bench  # noqa: E402
from paper_2305_04397_b200.api import Instance  # noqa: E402

cfg, thr, eps, K = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
inst = Instance.warehouse(cfg)
be = cu.CudaBackend(0)
ids = be.upload([inst.product(i, j) for i in range(inst.n) for j in range(inst.n)])
lib = be.lib
lib.morap_cuda_debug_flow_prof.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
buf = np.zeros(4096 * 8, np.uint64)
for w in ([0.5 / inst.n, 0.5 / inst.n], [1.0, 0.0], [0.35, 0.65]):
    W = np.tile(w, (len(ids), 1))
    be.optimize(ids, W)
    lib.morap_cuda_debug_flow_prof(be.h, buf.ctypes.data, buf.size, 1)
    be.set_profiling(True)
    be.reset_stats()
    be.optimize(ids, W)
    st = be.stats()
    be.set_profiling(False)
    nb = lib.morap_cuda_debug_flow_prof(be.h, buf.ctypes.data, buf.size, 1)
    a = buf[: nb * 8].reshape(nb, 8).astype(np.float64)
    names = ["p_ring_wait", "p_resolve", "p_refill_wait", "p_book", "c_full_wait", "c_compute", "c_tiles"]
    out = {n: float(a[:, i].mean()) for i, n in enumerate(names)}
    out["kernel_ms"] = st["opt_ms"]
    out["cycles_at_1.965GHz"] = st["opt_ms"] * 1.965e6
    print(json.dumps({"w": w, **out}), flush=True)
