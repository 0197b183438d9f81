"""ctypes binding of ``libvcs_gpu.so`` — the C ABI declared in ``include/vcs_gpu.h``.

This module is plumbing only: it loads the in-tree shared library (built by
``__graft_entry__.build()`` / ``make``), declares every exported symbol, and turns non-zero
status codes into the Python counterparts of the reference's exceptions.  There is no CPU
fallback: a missing library or a missing GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

VCS_OK, VCS_EINVAL, VCS_ECAP, VCS_EIO, VCS_ECUDA, VCS_ERANGE = 0, 2, 3, 4, 5, 6
VCS_PAID_CLOUD = -1
VCS_NO_ACTION = -2
VCS_GEN_RANDOM, VCS_GEN_HOMOG, VCS_GEN_GREEDY = 0, 1, 2
VCS_METHOD_AUTO, VCS_METHOD_JACOBI, VCS_METHOD_WAVEFRONT, VCS_METHOD_CERTIFIED = 0, 1, 2, 3
VCS_EXCHANGE_HALO, VCS_EXCHANGE_ALLGATHER = 0, 1

LIB_PATH = Path(__file__).resolve().parent / "libvcs_gpu.so"

# Every symbol include/vcs_gpu.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "vcs_instance_parse", "vcs_instance_load", "vcs_instance_copy", "vcs_instance_view",
    "vcs_instance_free", "vcs_instance_generate",
    "vcs_space_build", "vcs_space_from_csr", "vcs_space_info_get", "vcs_space_layer_offsets",
    "vcs_space_layer_edges", "vcs_space_csr", "vcs_space_locate", "vcs_space_hidden_penalty",
    "vcs_policy_query", "vcs_rollout", "vcs_space_result_generation", "vcs_space_free",
    "vcs_host_alloc", "vcs_host_free",
    "vcs_solve", "vcs_solve_enqueue", "vcs_solve_collect",
    "vcs_solve_multi_enqueue", "vcs_solve_multi", "vcs_multi_info",
    "vcs_cert_shard_begin", "vcs_cert_shard_plan", "vcs_cert_shard_layer", "vcs_cert_shard_pairs",
    "vcs_cert_shard_buffers", "vcs_cert_shard_finish", "vcs_shard_plan", "vcs_shard_begin", "vcs_shard_sweep", "vcs_shard_finish",
    "vcs_wave_shard_begin", "vcs_wave_shard_band", "vcs_wave_shard_layer", "vcs_wave_shard_pack",
    "vcs_wave_shard_unpack", "vcs_wave_shard_finish",
    "vcs_greedy", "vcs_greedy_batch", "vcs_greedy_reward",
    "vcs_last_error", "vcs_kernel_launches", "vcs_device_count",
)


class VcsError(RuntimeError):
    """Base of the status-code errors raised by the bindings."""


class InvalidArgument(VcsError, ValueError):
    """std::invalid_argument / ConfigError (status 2)."""


class StateCapacityError(VcsError):
    """vcsched::StateCapacityError (status 3, mdp.hpp:58-68)."""

    def __init__(self, cap: int, msg: str | None = None):
        super().__init__(msg or f"reachable state space exceeds cap of {cap} states")
        self._cap = int(cap)

    def cap(self) -> int:
        return self._cap


class IoError(VcsError, OSError):
    """vcsched::IoError (status 4)."""


class CudaError(VcsError):
    """CUDA runtime failure (status 5); never swallowed into a CPU path."""


class OutOfRange(VcsError, IndexError):
    """std::out_of_range (status 6)."""


class vcs_instance(C.Structure):
    _fields_ = [
        ("n_clouds", C.c_int32),
        ("cloud_id", C.POINTER(C.c_int32)),
        ("cloud_vm_total", C.POINTER(C.c_int32)),
        ("cloud_vm_free", C.POINTER(C.c_int32)),
        ("cloud_thr_kbps", C.POINTER(C.c_double)),
        ("cloud_delay_ms", C.POINTER(C.c_double)),
        ("n_tasks", C.c_int32),
        ("task_id", C.POINTER(C.c_int32)),
        ("task_demand", C.POINTER(C.c_int32)),
        ("task_max_delay_ms", C.POINTER(C.c_double)),
        ("task_min_thr_kbps", C.POINTER(C.c_double)),
        ("n_bots", C.c_int32),
        ("bot_id", C.POINTER(C.c_int32)),
        ("bot_task_offset", C.POINTER(C.c_int32)),
        ("beta_vc", C.c_double),
        ("beta_tc", C.c_double),
        ("gamma_vc", C.c_double),
    ]


class vcs_space_info(C.Structure):
    _fields_ = [
        ("n_states", C.c_uint64),
        ("n_edges", C.c_uint64),
        ("horizon", C.c_int32),
        ("key_words", C.c_int32),
        ("max_layer", C.c_uint64),
        ("max_degree", C.c_int32),
        ("device", C.c_int32),
        ("build_ms", C.c_double),
        ("device_bytes", C.c_uint64),
    ]


class vcs_solve_opts(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double),
        ("skip_converged", C.c_int32),
        ("max_sweeps", C.c_int32),
        ("discount", C.c_double),
        ("method", C.c_int32),
    ]


class vcs_solve_report(C.Structure):
    _fields_ = [
        ("sweeps", C.c_int32),
        ("launches", C.c_int32),
        ("backups_ref", C.c_uint64),
        ("backups_done", C.c_uint64),
        ("sweep_ms", C.c_double),
        ("extract_ms", C.c_double),
        ("alg_bytes", C.c_double),
        ("alg_bytes_done", C.c_double),
        ("method", C.c_int32),
        ("fallback_deferred", C.c_int32),
        ("model_bytes", C.c_double),
    ]


class vcs_multi_report(C.Structure):
    _fields_ = [
        ("n_ranks", C.c_int32),
        ("split_layers", C.c_int32),
        ("replicated_layers", C.c_int32),
        ("exchange", C.c_int32),
        ("halo_bytes", C.c_double),
        ("max_share", C.c_double),
        ("graph", C.c_int32),
        ("pad", C.c_int32),
    ]


_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_U64P = C.POINTER(C.c_uint64)
_U32P = C.POINTER(C.c_uint32)
_U8P = C.POINTER(C.c_uint8)
_F64P = C.POINTER(C.c_double)
_INSTP = C.POINTER(vcs_instance)

_SIGS = {
    "vcs_instance_parse": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
    "vcs_instance_load": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
    "vcs_instance_copy": (C.c_int, [_INSTP, C.POINTER(_P)]),
    "vcs_instance_view": (_INSTP, [_P]),
    "vcs_instance_free": (None, [_P]),
    "vcs_instance_generate": (C.c_int, [C.c_int, C.c_uint64, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, C.POINTER(_P)]),
    "vcs_space_build": (C.c_int, [_INSTP, C.c_uint64, C.c_int, C.POINTER(_P)]),
    "vcs_space_from_csr": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int32, _U64P, _U64P, _U32P,
                                     _F64P, _I32P, C.c_int, C.POINTER(_P)]),
    "vcs_space_info_get": (C.c_int, [_P, C.POINTER(vcs_space_info)]),
    "vcs_space_layer_offsets": (C.c_int, [_P, _U64P]),
    "vcs_space_layer_edges": (C.c_int, [_P, _U64P]),
    "vcs_space_csr": (C.c_int, [_P, _U64P, _U32P, _F64P, _I32P]),
    "vcs_space_locate": (C.c_int, [_P, C.c_int64, _I32P, _I32P, _U8P, _I64P]),
    "vcs_space_hidden_penalty": (C.c_int, [_P, C.c_int64, _I32P, _I32P, _U8P, _F64P]),
    "vcs_policy_query": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "vcs_space_free": (None, [_P]),
    "vcs_rollout": (C.c_int, [_P, _INSTP, _I32P, _P]),
    "vcs_space_result_generation": (C.c_uint64, [_P]),
    "vcs_host_alloc": (_P, [C.c_uint64]),
    "vcs_host_free": (None, [_P]),
    "vcs_solve": (C.c_int, [_P, C.POINTER(vcs_solve_opts), _F64P, _I32P,
                            C.POINTER(vcs_solve_report)]),
    "vcs_solve_enqueue": (C.c_int, [_P, C.POINTER(vcs_solve_opts), _P]),
    "vcs_solve_collect": (C.c_int, [_P, _F64P, _I32P, C.POINTER(vcs_solve_report), _P]),
    "vcs_solve_multi_enqueue": (C.c_int, [_P, C.POINTER(vcs_solve_opts), C.c_int32, _I32P,
                                          C.c_int32, _P]),
    "vcs_solve_multi": (C.c_int, [_P, C.POINTER(vcs_solve_opts), C.c_int32, _I32P, C.c_int32,
                                  _F64P, _I32P, C.POINTER(vcs_solve_report)]),
    "vcs_multi_info": (C.c_int, [_P, C.POINTER(vcs_multi_report)]),
    "vcs_cert_shard_begin": (C.c_int, [_P, C.POINTER(vcs_solve_opts), C.c_int32, C.c_int32,
                                       C.c_int32, _P]),
    "vcs_cert_shard_plan": (C.c_int, [_P, C.c_int32, C.c_int32, _U64P]),
    "vcs_cert_shard_layer": (C.c_int, [_P, C.c_int32, _P]),
    "vcs_cert_shard_pairs": (C.c_int, [_P, C.c_int32, C.POINTER(_P)]),
    "vcs_cert_shard_buffers": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "vcs_cert_shard_finish": (C.c_int, [_P, _F64P, _I32P]),
    "vcs_shard_plan": (C.c_int, [_U64P, _U64P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                 _U64P, _U64P, _U64P, _U64P]),
    "vcs_shard_begin": (C.c_int, [_P, _P, _P, _P, C.c_int32, _P]),
    "vcs_shard_sweep": (C.c_int, [_P, C.c_int32, C.c_uint64, C.c_uint64,
                                  C.POINTER(vcs_solve_opts), _P]),
    "vcs_shard_finish": (C.c_int, [_P, C.c_int32, C.c_uint64, C.c_uint64,
                                   C.POINTER(vcs_solve_opts), _F64P, _I32P, _I32P, _P]),
    "vcs_wave_shard_begin": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(vcs_solve_opts), _P,
                                       _P]),
    "vcs_wave_shard_band": (C.c_int, [_P, C.c_int32, _I32P, _I32P]),
    "vcs_wave_shard_layer": (C.c_int, [_P, C.c_int32, _P]),
    "vcs_wave_shard_pack": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P]),
    "vcs_wave_shard_unpack": (C.c_int, [_P, C.c_int32, _P, _P]),
    "vcs_wave_shard_finish": (C.c_int, [_P, C.c_int32, _F64P, _I32P, _P]),
    "vcs_greedy": (C.c_int, [_INSTP, C.c_int, _I32P, _I64P, _I64P, _I64P]),
    "vcs_greedy_batch": (C.c_int, [C.c_int32, _INSTP, C.c_int, C.POINTER(_I32P), _I64P, _I64P]),
    "vcs_greedy_reward": (C.c_double, [_INSTP, C.c_int64, C.c_int64, C.c_int64]),
    "vcs_last_error": (C.c_char_p, []),
    "vcs_kernel_launches": (C.c_uint64, []),
    "vcs_device_count": (C.c_int, []),
}

_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load libvcs_gpu.so (in-tree) once; raise loudly when it was not built."""
    global _lib
    if _lib is None:
        path = os.environ.get("VCS_GPU_LIB", str(LIB_PATH))
        if not Path(path).exists():
            raise ImportError(
                f"{path} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or `make`)")
        handle = C.CDLL(path, mode=C.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().vcs_last_error()
    return msg.decode() if msg else ""


def check(rc: int, cap: int | None = None) -> None:
    if rc == VCS_OK:
        return
    msg = last_error()
    if rc == VCS_ECAP:
        raise StateCapacityError(cap if cap is not None else -1, msg)
    if rc == VCS_EINVAL:
        raise InvalidArgument(msg)
    if rc == VCS_EIO:
        raise IoError(msg)
    if rc == VCS_ECUDA:
        raise CudaError(msg)
    if rc == VCS_ERANGE:
        raise OutOfRange(msg)
    raise VcsError(f"status {rc}: {msg}")


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def kernel_launches() -> int:
    return int(lib().vcs_kernel_launches())


def device_count() -> int:
    return int(lib().vcs_device_count())

