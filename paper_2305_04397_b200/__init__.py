"""B200-native hot path of MORAP (arXiv 2305.04397): weighted-sum value iteration over the
decentralised agent x task product MDPs inside the point-oriented Pareto loop.

Layers:
  libmorap_cuda.so  sm_100a kernels + C ABI (include/morap_cuda.h)      -> .cuda
  libmorap_host.so  host C++ API (model loader, per-model solve, Pareto
                    query) over that ABI + C ABI (include/morap.h)       -> .api
"""
from .errors import Errc, MorapError  # noqa: F401

__all__ = ["Errc", "MorapError"]
