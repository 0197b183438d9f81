"""ctypes bindings of the CHECKERS (test infrastructure only).

* ``Oracle``    — oracle/liboracle.so, the plain-C restatement of the reference path
                  (oracle/vcs_oracle.c).
* ``Reference`` — oracle/_ref/libvcsref.so, the UNMODIFIED reference C++ sources compiled from
                  /root/reference by oracle/Makefile rules (prebuilt .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libvcsref.so"

_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_U64P = C.POINTER(C.c_uint64)
_U32P = C.POINTER(C.c_uint32)
_F64P = C.POINTER(C.c_double)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Oracle:
    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make oracle/liboracle.so`")
        L = C.CDLL(str(path))
        from paper_2012_12419_b200._native import vcs_instance
        INST = C.POINTER(vcs_instance)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_build": (C.c_int, [INST, C.c_uint64, C.POINTER(_P)]),
            "orc_space_wrap": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int32, _U64P, _U64P, _U32P,
                                         _F64P, _I32P, C.POINTER(_P)]),
            "orc_space_free": (None, [_P]),
            "orc_space_info": (None, [_P, _U64P, _U64P, _I32P]),
            "orc_space_csr": (None, [_P, _U64P, _U64P, _U32P, _F64P, _I32P]),
            "orc_vi": (C.c_int, [_P, C.c_double, C.c_int, C.c_double, C.c_int, _F64P, _I32P, _I32P,
                                 _F64P, _F64P]),
            "orc_hidden_penalty": (C.c_double, [_P, _I32P, C.c_int32, C.c_uint8]),
            "orc_greedy": (C.c_int, [INST, _I32P, _I64P, _I64P, _I64P, _F64P]),
            "orc_greedy_reward": (C.c_double, [INST, C.c_int64, C.c_int64, C.c_int64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        self.L = L

    def err(self):
        return self.L.orc_last_error().decode()

    def build(self, inst_ref, cap=5_000_000):
        """-> OracleSpace (raises RuntimeError(code, msg) on failure)."""
        h = _P()
        rc = self.L.orc_build(inst_ref, cap, C.byref(h))
        if rc != 0:
            raise OracleError(rc, self.err())
        return OracleSpace(self, h)

    def wrap(self, layer_off, row_ptr, succ, reward, action):
        arrays = [np.ascontiguousarray(layer_off, np.uint64), np.ascontiguousarray(row_ptr, np.uint64),
                  np.ascontiguousarray(succ, np.uint32), np.ascontiguousarray(reward, np.float64),
                  np.ascontiguousarray(action, np.int32)]
        h = _P()
        self.L.orc_space_wrap(len(arrays[1]) - 1, len(arrays[2]), len(arrays[0]) - 2,
                              _p(arrays[0], C.c_uint64), _p(arrays[1], C.c_uint64),
                              _p(arrays[2], C.c_uint32), _p(arrays[3], C.c_double),
                              _p(arrays[4], C.c_int32), C.byref(h))
        sp = OracleSpace(self, h)
        sp._keep = arrays
        return sp

    def greedy(self, inst_ref, n_tasks, n_clouds):
        tgt = np.empty(max(n_tasks, 1), np.int32)
        used = np.zeros(max(n_clouds, 1), np.int64)
        paid, unused, ms = C.c_int64(), C.c_int64(), C.c_double()
        self.L.orc_greedy(inst_ref, _p(tgt, C.c_int32), _p(used, C.c_int64), C.byref(paid),
                          C.byref(unused), C.byref(ms))
        return tgt[:n_tasks], used[:n_clouds], paid.value, unused.value, ms.value


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class OracleSpace:
    def __init__(self, orc: Oracle, h):
        self.orc, self.h = orc, h
        S, E, H = C.c_uint64(), C.c_uint64(), C.c_int32()
        orc.L.orc_space_info(h, C.byref(S), C.byref(E), C.byref(H))
        self.S, self.E, self.H = S.value, E.value, H.value

    def __del__(self):
        if getattr(self, "h", None):
            self.orc.L.orc_space_free(self.h)
            self.h = None

    def csr(self):
        lo = np.zeros(self.H + 2, np.uint64)
        rp = np.zeros(self.S + 1, np.uint64)
        su = np.zeros(max(self.E, 1), np.uint32)
        rw = np.zeros(max(self.E, 1), np.float64)
        ac = np.zeros(max(self.E, 1), np.int32)
        self.orc.L.orc_space_csr(self.h, _p(lo, C.c_uint64), _p(rp, C.c_uint64), _p(su, C.c_uint32),
                                 _p(rw, C.c_double), _p(ac, C.c_int32))
        return lo, rp, su[:self.E], rw[:self.E], ac[:self.E]

    def vi(self, eps=1e-6, workers=1, discount=1.0, max_sweeps=0):
        v = np.empty(self.S, np.float64)
        a = np.empty(self.S, np.int32)
        sw = C.c_int32()
        t_sw, t_ex = C.c_double(), C.c_double()
        rc = self.orc.L.orc_vi(self.h, eps, workers, discount, max_sweeps, _p(v, C.c_double),
                               _p(a, C.c_int32), C.byref(sw), C.byref(t_sw), C.byref(t_ex))
        if rc != 0:
            raise OracleError(rc, self.orc.err())
        return v, a, sw.value, t_sw.value, t_ex.value


class Reference:
    """The unmodified reference solver (oracle/_ref/libvcsref.so)."""

    def __init__(self, path: Path = REF_SO, standalone: bool = False):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: build it with `make ref` where "
                                    "/root/reference exists")
        L = C.CDLL(str(path))
        if standalone:
            # bench.py's reference arm: no product import at all (the vcs_instance-typed entry
            # points are left unchecked; the arm only uses the instance handles below)
            INST = None
        else:
            from paper_2012_12419_b200._native import vcs_instance
            INST = C.POINTER(vcs_instance)
        sig = {
            "ref_instance_load": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
            "ref_instance_parse": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
            "ref_instance_generate": (C.c_int, [C.c_int, C.c_uint64, C.c_int32, C.c_int32,
                                                C.c_int32, C.c_int32, C.POINTER(_P)]),
            "ref_instance_free": (None, [_P]),
            "ref_instance_counts": (None, [_P, _I32P, _I32P]),
            "ref_instance_text": (C.c_uint64, [_P, C.c_char_p, C.c_uint64]),
            "ref_space_build_inst": (C.c_int, [_P, C.c_uint64, C.POINTER(_P), _F64P]),
            "ref_greedy_inst": (C.c_int, [_P, _I32P, _I64P, _I64P, _F64P]),
            "ref_per_vehicle_kbps": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, C.c_int64, _F64P]),
            "ref_last_error": (C.c_char_p, []),
            "ref_hardware_threads": (C.c_int, []),
            "ref_space_build": (C.c_int, [INST, C.c_uint64, C.POINTER(_P), _F64P]),
            "ref_space_free": (None, [_P]),
            "ref_space_size": (C.c_uint64, [_P]),
            "ref_space_horizon": (C.c_int32, [_P]),
            "ref_space_layers": (None, [_P, _U64P]),
            "ref_vi": (C.c_int, [_P, C.c_double, C.c_int, C.POINTER(_P), _I32P, _F64P]),
            "ref_res_free": (None, [_P]),
            "ref_res_values": (None, [_P, _F64P]),
            "ref_res_actions": (None, [_P, _I32P]),
            "ref_res_initial_value": (C.c_int, [_P, _F64P]),
            "ref_res_value_of": (C.c_int, [_P, _I32P, C.c_int32, C.c_uint8, _F64P]),
            "ref_res_action_for": (C.c_int, [_P, _I32P, C.c_int32, C.c_uint8, _I32P]),
            "ref_res_rollout": (C.c_int, [_P, _I32P, _I64P, _I64P, _I64P, _F64P]),
            "ref_greedy": (C.c_int, [INST, _I32P, _I32P, _I64P, _I64P, _I64P, _F64P, _F64P]),
            "ref_load_counts": (C.c_int, [C.c_char_p, _I32P, _I32P, _I32P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            if args is None or None in args:
                f.argtypes = None
            else:
                f.argtypes = args
        self.L = L

    def err(self):
        return self.L.ref_last_error().decode()

    # ---- instance handles (the reference's own parser / the restated bench generators) -----
    def load(self, path):
        return RefInstance(self, "ref_instance_load", str(path).encode())

    def parse(self, text: str):
        return RefInstance(self, "ref_instance_parse", text.encode())

    def generate(self, kind, seed, a, b, c, d):
        return RefInstance(self, "ref_instance_generate", kind, seed, a, b, c, d)

    def threads(self):
        return int(self.L.ref_hardware_threads())

    def build(self, inst_ref, cap=5_000_000):
        h = _P()
        ms = C.c_double()
        rc = self.L.ref_space_build(inst_ref, cap, C.byref(h), C.byref(ms))
        if rc != 0:
            raise OracleError(rc, self.err())
        return RefSpace(self, h, ms.value)

    def greedy(self, inst_ref, n_tasks):
        ids = np.empty(max(n_tasks, 1), np.int32)
        used = np.empty(max(n_tasks, 1), np.int32)
        paid, unused, placed = C.c_int64(), C.c_int64(), C.c_int64()
        reward, ms = C.c_double(), C.c_double()
        rc = self.L.ref_greedy(inst_ref, _p(ids, C.c_int32), _p(used, C.c_int32), C.byref(paid),
                               C.byref(unused), C.byref(placed), C.byref(reward), C.byref(ms))
        if rc != 0:
            raise OracleError(rc, self.err())
        return dict(target_ids=ids[:n_tasks], vms_used=used[:n_tasks], paid=paid.value,
                    unused=unused.value, placed=placed.value, reward=reward.value, ms=ms.value)


class RefInstance:
    """A reference-owned ParsedInstance (oracle/ref_capi.cpp RefInstance)."""

    def __init__(self, ref: Reference, fn: str, *args):
        self.ref, self.h = ref, _P()
        rc = getattr(ref.L, fn)(*args, C.byref(self.h))
        if rc != 0:
            self.h = None
            raise OracleError(rc, ref.err())
        nc, nt = C.c_int32(), C.c_int32()
        ref.L.ref_instance_counts(self.h, C.byref(nc), C.byref(nt))
        self.n_clouds, self.n_tasks = nc.value, nt.value

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.ref_instance_free(self.h)
            self.h = None

    def text(self) -> str:
        n = self.ref.L.ref_instance_text(self.h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self.ref.L.ref_instance_text(self.h, buf, n)
        return buf.raw[:n].decode()

    def build(self, cap=5_000_000):
        h = _P()
        ms = C.c_double()
        rc = self.ref.L.ref_space_build_inst(self.h, cap, C.byref(h), C.byref(ms))
        if rc != 0:
            raise OracleError(rc, self.ref.err())
        return RefSpace(self.ref, h, ms.value)

    def greedy(self):
        ids = np.empty(max(self.n_tasks, 1), np.int32)
        paid, unused, ms = C.c_int64(), C.c_int64(), C.c_double()
        rc = self.ref.L.ref_greedy_inst(self.h, _p(ids, C.c_int32), C.byref(paid), C.byref(unused),
                                        C.byref(ms))
        if rc != 0:
            raise OracleError(rc, self.ref.err())
        return dict(target_ids=ids[:self.n_tasks], paid=paid.value, unused=unused.value,
                    ms=ms.value)


class RefSpace:
    def __init__(self, ref: Reference, h, build_ms):
        self.ref, self.h, self.build_ms = ref, h, build_ms
        self.S = int(ref.L.ref_space_size(h))
        self.H = int(ref.L.ref_space_horizon(h))

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.ref_space_free(self.h)
            self.h = None

    def layers(self):
        lo = np.zeros(self.H + 2, np.uint64)
        self.ref.L.ref_space_layers(self.h, _p(lo, C.c_uint64))
        return lo

    def vi(self, eps=1e-6, workers=1):
        res = _P()
        sw, ms = C.c_int32(), C.c_double()
        rc = self.ref.L.ref_vi(self.h, eps, workers, C.byref(res), C.byref(sw), C.byref(ms))
        if rc != 0:
            raise OracleError(rc, self.ref.err())
        return RefResult(self, res, sw.value, ms.value)


class RefResult:
    def __init__(self, space: RefSpace, h, sweeps, ms):
        self.space, self.h, self.sweeps, self.ms = space, h, sweeps, ms
        self.L = space.ref.L

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_res_free(self.h)
            self.h = None

    def values(self):
        v = np.empty(self.space.S, np.float64)
        self.L.ref_res_values(self.h, _p(v, C.c_double))
        return v

    def actions(self):
        a = np.empty(self.space.S, np.int32)
        self.L.ref_res_actions(self.h, _p(a, C.c_int32))
        return a

    def initial_value(self):
        out = C.c_double()
        rc = self.L.ref_res_initial_value(self.h, C.byref(out))
        if rc != 0:
            raise OracleError(rc, self.space.ref.err())
        return out.value

    def value_of(self, free_vms, t, terminal):
        """ValueTable::value_of (mdp.cpp:269-271); None where the reference throws."""
        fv = np.ascontiguousarray(free_vms, np.int32)
        out = C.c_double()
        rc = self.L.ref_res_value_of(self.h, _p(fv, C.c_int32), int(t), 1 if terminal else 0,
                                     C.byref(out))
        return None if rc != 0 else out.value

    def action_for(self, free_vms, t, terminal):
        """Policy::action_for (mdp.cpp:277-282); None where the reference throws."""
        fv = np.ascontiguousarray(free_vms, np.int32)
        out = C.c_int32()
        rc = self.L.ref_res_action_for(self.h, _p(fv, C.c_int32), int(t), 1 if terminal else 0,
                                       C.byref(out))
        return None if rc != 0 else out.value

    def rollout(self, n_tasks, n_clouds):
        tg = np.empty(max(n_tasks, 1), np.int32)
        used = np.zeros(max(n_clouds, 1), np.int64)
        paid, unused, reward = C.c_int64(), C.c_int64(), C.c_double()
        rc = self.L.ref_res_rollout(self.h, _p(tg, C.c_int32), _p(used, C.c_int64), C.byref(paid),
                                    C.byref(unused), C.byref(reward))
        if rc != 0:
            raise OracleError(rc, self.space.ref.err())
        return dict(targets=tg[:n_tasks], used=used[:n_clouds], paid=paid.value,
                    unused=unused.value, reward=reward.value)
