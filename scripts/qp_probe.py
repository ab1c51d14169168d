"""Build and run scripts/qp_probe.cpp on the recorded C3/C4 queries (host only).

    python scripts/qp_probe.py [c3|c4] k1 k2 ...
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_04397_b200 import build  # noqa: E402

args = [a for a in sys.argv[1:] if a != "--profile"]
profile = "--profile" in sys.argv  # compile geometry/linalg into the probe with MORAP_QP_PROFILE
name = args[0] if args else "c4"
ks = args[1:] or ["50", "100", "150", "200"]
out = os.path.join(ROOT, "build", "qp")
os.makedirs(out, exist_ok=True)
z = np.load(os.path.join(ROOT, "tests", "golden", "replay", f"{name}_query.npz"))
pts = os.path.join(out, f"{name}.bin")
with open(pts, "wb") as f:
    np.array(z["r"].shape, np.int64).tofile(f)
    z["thresholds"].astype(np.float64).tofile(f)
    z["r"].astype(np.float64).tofile(f)
build.build_all()
exe = os.path.join(out, "qp_probe")
extra = ["-DMORAP_QP_PROFILE", os.path.join(build.CSRC, "geometry.cpp"), os.path.join(build.CSRC, "linalg.cpp")] \
    if profile else []
subprocess.run(["g++", "-std=c++20", "-O3", "-mavx2", "-ffp-contract=off", "-pthread", f"-I{ROOT}/include",
                f"-I{build.CSRC}", f"-I{build.JSON_DIR}", os.path.join(ROOT, "scripts", "qp_probe.cpp"), *extra,
                f"-L{build.PKG}", "-lmorap_host", "-lmorap_cuda", f"-Wl,-rpath,{build.PKG}", "-o", exe], check=True)
sys.exit(subprocess.run([exe, pts, *ks]).returncode)
