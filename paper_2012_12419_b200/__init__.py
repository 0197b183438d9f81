"""B200-native vehicular-cloud placement solver (arXiv 2012.12419 solver path).

The public surface mirrors the reference ``vcsched`` C++ API (see ``vcsched.py``); the compute
runs in hand-written sm_100a kernels behind the C ABI of ``include/vcs_gpu.h``.
"""
from .vcsched import *  # noqa: F401,F403
from .vcsched import __all__ as _api_all
from . import _native

__all__ = list(_api_all) + ["_native"]
