"""In-tree build of the native libraries (sm_100a CUDA backend + host C++ library).

Outputs (git-ignored, shipped to the GPU box with the snapshot):
  paper_2305_04397_b200/libmorap_cuda.so   kernels + C ABI (include/morap_cuda.h)
  paper_2305_04397_b200/libmorap_host.so   host C++ API + C ABI (include/morap.h),
                                           links libmorap_cuda.so
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
CUDA_SO = os.path.join(PKG, "libmorap_cuda.so")
HOST_SO = os.path.join(PKG, "libmorap_host.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
def _json_dir() -> str:
    """nlohmann/json (header-only): $MORAP_JSON_DIR, else the copies this image ships."""
    cands = [os.environ.get("MORAP_JSON_DIR", "")]
    try:
        import sysconfig
        site = sysconfig.get_paths()["purelib"]
        cands.append(os.path.join(site, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
    except Exception:  # noqa: BLE001
        pass
    cands.append("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
    for c in cands:
        if c and os.path.exists(os.path.join(c, "json.hpp")):
            return c
    raise FileNotFoundError("nlohmann/json.hpp not found: set MORAP_JSON_DIR to the directory holding json.hpp")


JSON_DIR = _json_dir()

CUDA_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-fmad=false",  # bitwise parity with the reference's no-FMA CPU arithmetic
    "-Xcompiler", "-fPIC", "-shared",
    # host side of the .cu (upload preparation: validation, tiling, compact streams -- integer
    # and bit-pattern work only): vectorised like the host library, no FP contraction
    "-Xcompiler", "-O3,-mavx2,-ffp-contract=off",
]

HOST_SOURCES = ["linalg.cpp", "logic.cpp", "model.cpp", "warehouse.cpp", "assignment.cpp", "geometry.cpp",
                "gpu.cpp", "device_build.cpp", "solver.cpp", "shard.cpp", "centralised.cpp", "capi.cpp"]


def _newer(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _deps(names):
    out = [os.path.join(CSRC, n) for n in names]
    out += [os.path.join(CSRC, n) for n in os.listdir(CSRC) if n.endswith((".h", ".hpp", ".cuh"))]
    out += [os.path.join(ROOT, "include", n) for n in os.listdir(os.path.join(ROOT, "include"))]
    return out


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    src = os.path.join(CSRC, "morap_cuda.cu")
    diag = os.environ.get("MORAP_BUILD_DIAGNOSTICS") == "1"  # dev probes only (CTA traces, dry runs)
    checked = os.environ.get("MORAP_BUILD_CHECKED") == "1"  # device bounds checks (test runs)
    extra = (["-DMORAP_DIAGNOSTICS"] if diag else []) + (["-DMORAP_CHECKED"] if checked else [])
    if force or extra or _newer(CUDA_SO, _deps(["morap_cuda.cu"])):
        cmd = [NVCC, *CUDA_FLAGS, *extra, "-o", CUDA_SO, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
    return CUDA_SO


def build_host(force: bool = False) -> str:
    """Compile each translation unit in parallel into build/host/*.o, then link."""
    srcs = [os.path.join(CSRC, s) for s in HOST_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if not srcs:
        return ""
    if not (force or _newer(HOST_SO, _deps(HOST_SOURCES) + [CUDA_SO])):
        return HOST_SO
    obj_dir = os.path.join(ROOT, "build", "host")
    os.makedirs(obj_dir, exist_ok=True)
    # -O3 vectorises the elementwise loops (bit-identical: no FMA, reductions keep their order)
    flags = ["-std=c++20", "-O3", "-mavx2", "-fPIC", "-pthread", "-ffp-contract=off", f"-I{os.path.join(ROOT, 'include')}",
             f"-I{CSRC}", f"-I{JSON_DIR}"]
    hdrs = [os.path.join(CSRC, n) for n in os.listdir(CSRC) if n.endswith(".hpp")] + \
        [os.path.join(ROOT, "include", n) for n in os.listdir(os.path.join(ROOT, "include"))]
    procs, objs = [], []
    for src in srcs:
        obj = os.path.join(obj_dir, os.path.basename(src)[:-4] + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + hdrs):
            procs.append(subprocess.Popen(["g++", *flags, "-c", "-o", obj, src]))
    if any(p.wait() != 0 for p in procs):
        raise RuntimeError("host library compilation failed")
    subprocess.run(["g++", "-shared", "-pthread", "-o", HOST_SO, *objs, f"-L{PKG}", "-lmorap_cuda",
                    "-Wl,-rpath,$ORIGIN"], check=True)
    return HOST_SO


def build_all(force: bool = False) -> None:
    build_cuda(force)
    build_host(force)


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv)
    print("built", CUDA_SO, HOST_SO)
