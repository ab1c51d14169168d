"""The C-ABI libraries load on a CPU-only host and export every symbol their headers declare."""
import ctypes
import os
import re

from paper_2305_04397_b200 import api, cuda

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(morap_[a-z_0-9]+)\s*\(", text)) - {"morap_query_fn"})


def test_cuda_abi_exports():
    lib = ctypes.CDLL(cuda.CUDA_SO)
    names = declared("morap_cuda.h")
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


def test_host_abi_exports():
    lib = ctypes.CDLL(api.HOST_SO)
    names = declared("morap.h")
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2305_04397_b200.errors import MorapError
    try:
        cuda.CudaBackend(0)
    except MorapError:
        return
    raise AssertionError("creating a CUDA backend without a GPU must raise")
