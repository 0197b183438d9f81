"""Python mirror of the reference ``vcsched`` solver API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference's public headers
(paths relative to /root/reference/proj/core/include/vcsched/):

  workload.hpp:12-70   Task, BagOfTasks, VehicularCloud, VccModel, kPaidCloud, PlacementRecord,
                       total_demand, total_capacity, feasible, flatten_tasks, validate
  mdp.hpp:18-204       MdpInstance, MdpAction, MdpState, initial_state, legal_actions,
                       transition, step_reward, StateCapacityError, StateSpace, ViOptions,
                       ValueTable, Policy, ViResult, value_iteration, bellman_backup, rollout,
                       detail::run_value_iteration
  parallel_vi.hpp:14-56 BlockPartition, SweepBarrier, parallel_value_iteration, SpeedupRow,
                       measure_speedup
  greedy.hpp:11-30     ScheduleResult, greedy_schedule, greedy_reward
  io.hpp:18-40         ConfigError, IoError, ParsedInstance, parse_instance, load_instance

Every heavy operation (state-space build, value iteration, policy extraction, locate, greedy
placement) runs in hand-written sm_100a kernels behind libvcs_gpu.so.  The small full-state
helpers (transition, legal_actions, step_reward, bellman_backup) are the reference's test-facing
API and stay host Python, as they are O(clouds).
"""
from __future__ import annotations

import ctypes as C
import math
import threading
import time
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _native as N
from ._native import (CudaError, InvalidArgument, IoError, OutOfRange, StateCapacityError,
                      VcsError)

kPaidCloud = -1

ConfigError = InvalidArgument  # io.hpp:18-20 (parse/validation failures, exit code 2)

__all__ = [
    "Task", "BagOfTasks", "VehicularCloud", "VccModel", "kPaidCloud", "PlacementRecord",
    "total_demand", "total_capacity", "feasible", "flatten_tasks", "validate",
    "MdpInstance", "MdpAction", "MdpState", "initial_state", "legal_actions", "transition",
    "step_reward", "StateCapacityError", "StateSpace", "ViOptions", "ValueTable", "Policy",
    "ViResult", "value_iteration", "bellman_backup", "rollout", "run_value_iteration",
    "BlockPartition", "SweepBarrier", "parallel_value_iteration", "SpeedupRow", "measure_speedup", "speedup_csv",
    "ScheduleResult", "greedy_schedule", "greedy_reward", "ParsedInstance", "parse_instance",
    "load_instance", "generate_instance", "instance_text", "ConfigError", "IoError", "InvalidArgument",
    "OutOfRange", "CudaError", "VcsError", "NativeInstance",
]


# ------------------------------------------------------------------------------------------
# workload.hpp
# ------------------------------------------------------------------------------------------

@dataclass
class Task:
    id: int = 0
    vm_demand: int = 1
    max_delay_ms: float = 0.0
    min_vm_throughput_kbps: float = 0.0


@dataclass
class BagOfTasks:
    id: int = 0
    tasks: list = field(default_factory=list)


@dataclass
class VehicularCloud:
    id: int = 0
    vm_total: int = 0
    vm_free: int = 0
    vm_throughput_kbps: float = 0.0
    v2i_delay_ms: float = 0.0


@dataclass
class VccModel:
    clouds: list = field(default_factory=list)
    reward_per_vc_vm: float = 1.0     # beta_vc
    cost_per_tcc_vm: float = 1.2      # beta_tc
    penalty_per_idle_vm: float = 1.0  # gamma_vc


@dataclass
class PlacementRecord:
    task_id: int = 0
    target: int = kPaidCloud
    vms_used: int = 0


def total_demand(bots: Sequence[BagOfTasks]) -> int:
    return sum(t.vm_demand for b in bots for t in b.tasks)


def total_capacity(vcc: VccModel) -> int:
    return sum(c.vm_total for c in vcc.clouds)


def feasible(cloud: VehicularCloud, task: Task) -> bool:
    """workload.cpp:22-26."""
    return (cloud.vm_free >= task.vm_demand and cloud.v2i_delay_ms <= task.max_delay_ms
            and cloud.vm_throughput_kbps >= task.min_vm_throughput_kbps)


def flatten_tasks(bots: Sequence[BagOfTasks]) -> list:
    return [t for b in bots for t in b.tasks]


def validate(obj) -> None:
    """workload.cpp:35-57 (both overloads), raising InvalidArgument."""
    if isinstance(obj, VccModel):
        if obj.reward_per_vc_vm < 0 or obj.cost_per_tcc_vm < 0 or obj.penalty_per_idle_vm < 0:
            raise InvalidArgument("rate parameters must be non-negative")
        for c in obj.clouds:
            if c.vm_total < 0:
                raise InvalidArgument(f"cloud {c.id}: vm_total < 0")
            if c.vm_free < 0 or c.vm_free > c.vm_total:
                raise InvalidArgument(f"cloud {c.id}: vm_free outside [0, vm_total]")
        return
    for b in obj:
        for t in b.tasks:
            if t.vm_demand < 1:
                raise InvalidArgument(f"task {t.id}: vm_demand < 1")
            if t.max_delay_ms <= 0 or t.min_vm_throughput_kbps <= 0:
                raise InvalidArgument(f"task {t.id}: requirements must be positive")


# ------------------------------------------------------------------------------------------
# SoA bridge to the C ABI
# ------------------------------------------------------------------------------------------

class NativeInstance:
    """Owns the SoA arrays behind one ``vcs_instance`` (or wraps a library-owned instance)."""

    def __init__(self, vcc: VccModel | None = None, tasks: Sequence[Task] | None = None,
                 bots: Sequence[BagOfTasks] | None = None, _owned=None):
        self._owned = _owned
        if _owned is not None:
            self.struct = N.lib().vcs_instance_view(_owned).contents
            self.struct._owner = self
            return
        clouds = vcc.clouds
        if bots is not None:
            tasks = flatten_tasks(bots)
        tasks = list(tasks or [])
        self.cloud_id = np.array([c.id for c in clouds], dtype=np.int32)
        self.cloud_vm_total = np.array([c.vm_total for c in clouds], dtype=np.int32)
        self.cloud_vm_free = np.array([c.vm_free for c in clouds], dtype=np.int32)
        self.cloud_thr = np.array([c.vm_throughput_kbps for c in clouds], dtype=np.float64)
        self.cloud_delay = np.array([c.v2i_delay_ms for c in clouds], dtype=np.float64)
        self.task_id = np.array([t.id for t in tasks], dtype=np.int32)
        self.task_demand = np.array([t.vm_demand for t in tasks], dtype=np.int32)
        self.task_max_delay = np.array([t.max_delay_ms for t in tasks], dtype=np.float64)
        self.task_min_thr = np.array([t.min_vm_throughput_kbps for t in tasks], dtype=np.float64)
        if bots is not None:
            self.bot_id = np.array([b.id for b in bots], dtype=np.int32)
            off = [0]
            for b in bots:
                off.append(off[-1] + len(b.tasks))
            self.bot_off = np.array(off, dtype=np.int32)
        else:
            self.bot_id = np.zeros(0, dtype=np.int32)
            self.bot_off = np.zeros(1, dtype=np.int32)
        s = N.vcs_instance()
        s.n_clouds = len(clouds)
        s.cloud_id = N.ptr(self.cloud_id, C.c_int32)
        s.cloud_vm_total = N.ptr(self.cloud_vm_total, C.c_int32)
        s.cloud_vm_free = N.ptr(self.cloud_vm_free, C.c_int32)
        s.cloud_thr_kbps = N.ptr(self.cloud_thr, C.c_double)
        s.cloud_delay_ms = N.ptr(self.cloud_delay, C.c_double)
        s.n_tasks = len(tasks)
        s.task_id = N.ptr(self.task_id, C.c_int32)
        s.task_demand = N.ptr(self.task_demand, C.c_int32)
        s.task_max_delay_ms = N.ptr(self.task_max_delay, C.c_double)
        s.task_min_thr_kbps = N.ptr(self.task_min_thr, C.c_double)
        s.n_bots = len(self.bot_id)
        s.bot_id = N.ptr(self.bot_id, C.c_int32)
        s.bot_task_offset = N.ptr(self.bot_off, C.c_int32)
        s.beta_vc = vcc.reward_per_vc_vm
        s.beta_tc = vcc.cost_per_tcc_vm
        s.gamma_vc = vcc.penalty_per_idle_vm
        s._owner = self  # byref(struct) keeps the SoA arrays alive (temporaries are safe)
        self.struct = s

    @classmethod
    def owned(cls, handle) -> "NativeInstance":
        return cls(_owned=handle)

    def __del__(self):
        if getattr(self, "_owned", None) is not None:
            try:
                N.lib().vcs_instance_free(self._owned)
            except Exception:
                pass
            self._owned = None

    @property
    def ref(self):
        return C.byref(self.struct)

    # SoA views (numpy) of whatever backs the struct
    def arrays(self) -> dict:
        s = self.struct
        K, T, B = s.n_clouds, s.n_tasks, s.n_bots

        def arr(p, n, dt):
            if n == 0 or not p:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)

        return {
            "cloud_id": arr(s.cloud_id, K, np.int32),
            "cloud_vm_total": arr(s.cloud_vm_total, K, np.int32),
            "cloud_vm_free": arr(s.cloud_vm_free, K, np.int32),
            "cloud_thr": arr(s.cloud_thr_kbps, K, np.float64),
            "cloud_delay": arr(s.cloud_delay_ms, K, np.float64),
            "task_id": arr(s.task_id, T, np.int32),
            "task_demand": arr(s.task_demand, T, np.int32),
            "task_max_delay": arr(s.task_max_delay_ms, T, np.float64),
            "task_min_thr": arr(s.task_min_thr_kbps, T, np.float64),
            "bot_id": arr(s.bot_id, B, np.int32),
            "bot_off": arr(s.bot_task_offset, B + 1 if B else 0, np.int32),
            "beta_vc": s.beta_vc, "beta_tc": s.beta_tc, "gamma_vc": s.gamma_vc,
        }


# ------------------------------------------------------------------------------------------
# io.hpp (instance input format only)
# ------------------------------------------------------------------------------------------

@dataclass
class ParsedInstance:
    vcc: VccModel
    bots: list
    native: NativeInstance | None = None


def _parsed_from_native(ni: NativeInstance) -> ParsedInstance:
    a = ni.arrays()
    vcc = VccModel(
        clouds=[VehicularCloud(int(a["cloud_id"][i]), int(a["cloud_vm_total"][i]),
                               int(a["cloud_vm_free"][i]), float(a["cloud_thr"][i]),
                               float(a["cloud_delay"][i])) for i in range(len(a["cloud_id"]))],
        reward_per_vc_vm=a["beta_vc"], cost_per_tcc_vm=a["beta_tc"],
        penalty_per_idle_vm=a["gamma_vc"])
    tasks = [Task(int(a["task_id"][j]), int(a["task_demand"][j]), float(a["task_max_delay"][j]),
                  float(a["task_min_thr"][j])) for j in range(len(a["task_id"]))]
    bots = []
    off = a["bot_off"]
    for b in range(len(a["bot_id"])):
        bots.append(BagOfTasks(int(a["bot_id"][b]), tasks[int(off[b]):int(off[b + 1])]))
    return ParsedInstance(vcc, bots, ni)


def parse_instance(text: str) -> ParsedInstance:
    """io.cpp:51-95 (ConfigError on malformed input)."""
    h = C.c_void_p()
    N.check(N.lib().vcs_instance_parse(text.encode(), C.byref(h)))
    return _parsed_from_native(NativeInstance.owned(h))


def load_instance(path: str) -> ParsedInstance:
    """io.cpp:97-101 (IoError when unreadable)."""
    h = C.c_void_p()
    N.check(N.lib().vcs_instance_load(str(path).encode(), C.byref(h)))
    return _parsed_from_native(NativeInstance.owned(h))


def _fmt(v: float) -> str:
    """io.cpp:16-20 fmt: printf %.17g."""
    return "%.17g" % float(v)


def instance_text(instance: ParsedInstance) -> str:
    """io.cpp:103-118 instance_text: the instance file a parse_instance round trip reproduces."""
    vcc = instance.vcc
    out = [f"beta_vc {_fmt(vcc.reward_per_vc_vm)}", f"beta_tc {_fmt(vcc.cost_per_tcc_vm)}",
           f"gamma_vc {_fmt(vcc.penalty_per_idle_vm)}"]
    for c in vcc.clouds:
        out.append(f"cloud {c.id} {c.vm_total} {_fmt(c.vm_throughput_kbps)} {_fmt(c.v2i_delay_ms)}")
    for bot in instance.bots:
        out.append(f"bot {bot.id}")
        for t in bot.tasks:
            out.append(f"task {t.id} {t.vm_demand} {_fmt(t.max_delay_ms)} "
                       f"{_fmt(t.min_vm_throughput_kbps)}")
    return "\n".join(out) + "\n"


def generate_instance(kind: int, seed: int, trial: int = 0, a: int = 0, b: int = 0, c: int = 0,
                      d: int = 0, as_objects: bool = True):
    """Seeded synthetic instance (see include/vcs_gpu.h vcs_instance_generate)."""
    h = C.c_void_p()
    N.check(N.lib().vcs_instance_generate(kind, seed, trial, a, b, c, d, C.byref(h)))
    ni = NativeInstance.owned(h)
    return _parsed_from_native(ni) if as_objects else ni


# ------------------------------------------------------------------------------------------
# mdp.hpp
# ------------------------------------------------------------------------------------------

@dataclass
class MdpInstance:
    vcc: VccModel
    tasks: list

    @staticmethod
    def from_workload(vcc: VccModel, bots: Sequence[BagOfTasks]) -> "MdpInstance":
        return MdpInstance(vcc, flatten_tasks(bots))

    def native(self) -> NativeInstance:
        return NativeInstance(self.vcc, self.tasks)


@dataclass(frozen=True)
class MdpAction:
    target: int = kPaidCloud

    def is_paid(self) -> bool:
        return self.target == kPaidCloud


@dataclass
class MdpState:
    free_vms: list = field(default_factory=list)
    next_task_index: int = 0
    terminal: bool = False


def initial_state(instance: MdpInstance) -> MdpState:
    return MdpState([c.vm_free for c in instance.vcc.clouds], 0, len(instance.tasks) == 0)


def _cloud_feasible_in_state(instance: MdpInstance, s: MdpState, i: int) -> bool:
    cloud = instance.vcc.clouds[i]
    task = instance.tasks[s.next_task_index]
    return (s.free_vms[i] >= task.vm_demand and cloud.v2i_delay_ms <= task.max_delay_ms
            and cloud.vm_throughput_kbps >= task.min_vm_throughput_kbps)


def legal_actions(instance: MdpInstance, s: MdpState) -> list:
    """mdp.cpp:34-42: feasible clouds ascending, then paid."""
    if s.terminal:
        return []
    acts = [MdpAction(i) for i in range(len(instance.vcc.clouds))
            if _cloud_feasible_in_state(instance, s, i)]
    acts.append(MdpAction(kPaidCloud))
    return acts


def transition(s: MdpState, a: MdpAction, instance: MdpInstance) -> MdpState:
    """mdp.cpp:44-58."""
    if s.terminal:
        raise InvalidArgument("transition from terminal state")
    nxt = MdpState(list(s.free_vms), s.next_task_index + 1, False)
    if not a.is_paid():
        if a.target < 0 or a.target >= len(instance.vcc.clouds):
            raise InvalidArgument("action targets unknown cloud")
        if not _cloud_feasible_in_state(instance, s, a.target):
            raise InvalidArgument("action targets infeasible cloud")
        nxt.free_vms[a.target] -= instance.tasks[s.next_task_index].vm_demand
    nxt.terminal = nxt.next_task_index == len(instance.tasks)
    return nxt


def step_reward(s: MdpState, a: MdpAction, nxt: MdpState, instance: MdpInstance) -> float:
    """mdp.cpp:60-65."""
    n = float(instance.tasks[s.next_task_index].vm_demand)
    return -instance.vcc.cost_per_tcc_vm * n if a.is_paid() else instance.vcc.reward_per_vc_vm * n


@dataclass
class ViOptions:
    epsilon: float = 1e-6
    state_cap: int = 5_000_000
    # B200 extensions (defaults keep the reference semantics bit-for-bit)
    skip_converged: bool = True
    discount: float = 1.0
    device: int = 0
    method: int = 0  # 0 auto (= 3 if the version store fits), 1 Jacobi, 2 wavefront, 3 certified


class StateSpace:
    """Device-resident reachable state graph (mdp.hpp:80-129)."""

    def __init__(self, handle, instance: MdpInstance | None, native: NativeInstance | None):
        self._h = handle
        self._instance = instance
        self._native = native
        info = N.vcs_space_info()
        N.check(N.lib().vcs_space_info_get(handle, C.byref(info)))
        self.info = info
        self._layers = np.zeros(info.horizon + 2, dtype=np.uint64)
        N.check(N.lib().vcs_space_layer_offsets(handle, N.ptr(self._layers, C.c_uint64)))

    @staticmethod
    def build(instance: MdpInstance, state_cap: int = 5_000_000, device: int = 0) -> "StateSpace":
        native = instance.native()
        return StateSpace.build_native(native, state_cap, device, instance)

    @staticmethod
    def build_native(native: NativeInstance, state_cap: int = 5_000_000, device: int = 0,
                     instance: MdpInstance | None = None) -> "StateSpace":
        h = C.c_void_p()
        N.check(N.lib().vcs_space_build(native.ref, int(state_cap), int(device), C.byref(h)),
                cap=state_cap)
        return StateSpace(h, instance, native)

    @staticmethod
    def from_csr(layer_offset, row_ptr, succ, reward, action, device: int = 0) -> "StateSpace":
        layer_offset = np.ascontiguousarray(layer_offset, dtype=np.uint64)
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        succ = np.ascontiguousarray(succ, dtype=np.uint32)
        reward = np.ascontiguousarray(reward, dtype=np.float64)
        action = np.ascontiguousarray(action, dtype=np.int32)
        h = C.c_void_p()
        N.check(N.lib().vcs_space_from_csr(
            len(row_ptr) - 1, len(succ), len(layer_offset) - 2, N.ptr(layer_offset, C.c_uint64),
            N.ptr(row_ptr, C.c_uint64), N.ptr(succ, C.c_uint32), N.ptr(reward, C.c_double),
            N.ptr(action, C.c_int32), device, C.byref(h)))
        return StateSpace(h, None, None)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                N.lib().vcs_space_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def size(self) -> int:
        return int(self.info.n_states)

    def edges(self) -> int:
        return int(self.info.n_edges)

    def task_count(self) -> int:
        return int(self.info.horizon)

    def layer_begin(self, t: int) -> int:
        return int(self._layers[t])

    def layer_end(self, t: int) -> int:
        return int(self._layers[t + 1])

    def layer_offsets(self) -> np.ndarray:
        return self._layers.copy()

    def layer_edges(self) -> np.ndarray:
        out = np.zeros(self.task_count() + 1, dtype=np.uint64)
        N.check(N.lib().vcs_space_layer_edges(self._h, N.ptr(out, C.c_uint64)))
        return out

    def instance(self) -> MdpInstance:
        return self._instance

    def csr(self):
        """(row_ptr u64[S+1], succ u32[E], reward f64[E], action i32[E]) downloaded from HBM."""
        S, E = self.size(), self.edges()
        rp = np.zeros(S + 1, dtype=np.uint64)
        su = np.zeros(max(E, 1), dtype=np.uint32)
        rw = np.zeros(max(E, 1), dtype=np.float64)
        ac = np.zeros(max(E, 1), dtype=np.int32)
        N.check(N.lib().vcs_space_csr(self._h, N.ptr(rp, C.c_uint64), N.ptr(su, C.c_uint32),
                                      N.ptr(rw, C.c_double), N.ptr(ac, C.c_int32)))
        return rp, su[:E], rw[:E], ac[:E]

    def _state_arrays(self, states: Sequence[MdpState]):
        K = len(self._instance.vcc.clouds) if self._instance else 0
        fv = np.zeros((len(states), max(K, 1)), dtype=np.int32)
        ti = np.zeros(len(states), dtype=np.int32)
        te = np.zeros(len(states), dtype=np.uint8)
        for i, s in enumerate(states):
            if len(s.free_vms) != K:
                raise InvalidArgument("state has wrong cloud count")
            t = self.task_count() if s.terminal else s.next_task_index
            if t < 0 or t > self.task_count():
                raise InvalidArgument("task index outside horizon")
            if K:
                fv[i, :] = s.free_vms
            ti[i] = s.next_task_index
            te[i] = 1 if s.terminal else 0
        return fv, ti, te

    def locate_many(self, states: Sequence[MdpState]) -> np.ndarray:
        fv, ti, te = self._state_arrays(states)
        out = np.zeros(len(states), dtype=np.int64)
        N.check(N.lib().vcs_space_locate(self._h, len(states), N.ptr(fv, C.c_int32),
                                         N.ptr(ti, C.c_int32), N.ptr(te, C.c_uint8),
                                         N.ptr(out, C.c_int64)))
        return out

    def locate(self, s: MdpState) -> int:
        """mdp.cpp:227-234; OutOfRange when unreachable."""
        idx = int(self.locate_many([s])[0])
        if idx < 0:
            raise OutOfRange("state not reachable in enumerated space")
        return idx

    def policy_query(self, states: Sequence[MdpState]):
        """vcs_policy_query: (values, actions, flat indices) for a batch of full states."""
        fv, ti, te = self._state_arrays(states)
        n = len(states)
        vals = np.zeros(n, dtype=np.float64)
        acts = np.zeros(n, dtype=np.int32)
        idx = np.zeros(n, dtype=np.int64)
        vp = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
        N.check(N.lib().vcs_policy_query(self._h, n, vp(fv), vp(ti), vp(te), vp(vals), vp(acts),
                                         vp(idx), None))
        return vals, acts, idx

    def hidden_penalty(self, s: MdpState) -> float:
        fv, ti, te = self._state_arrays([s])
        out = np.zeros(1, dtype=np.float64)
        N.check(N.lib().vcs_space_hidden_penalty(self._h, 1, N.ptr(fv, C.c_int32),
                                                 N.ptr(ti, C.c_int32), N.ptr(te, C.c_uint8),
                                                 N.ptr(out, C.c_double)))
        return float(out[0])


class ValueTable:
    """mdp.hpp:137-162."""

    def __init__(self, space: StateSpace, values: np.ndarray, sweeps: int, epsilon: float,
                 report=None):
        self._space = space
        self._values = values
        self._sweeps = int(sweeps)
        self._eps = float(epsilon)
        self.report = report

    def value_of(self, s: MdpState) -> float:
        return float(self._values[self._space.locate(s)]) - self._space.hidden_penalty(s)

    def initial_value(self) -> float:
        return self.value_of(initial_state(self._space.instance()))

    def value_of_many(self, states: Sequence[MdpState]) -> np.ndarray:
        """Batched value_of on the device (vcs_policy_query): NaN where a state is unreachable
        (value_of raises OutOfRange there).  Answers from the space's last collected solve."""
        return self._space.policy_query(states)[0]

    def sweeps(self) -> int:
        return self._sweeps

    def epsilon(self) -> float:
        return self._eps

    def states_explored(self) -> int:
        return self._space.size()

    def raw_values(self) -> np.ndarray:
        return self._values

    def space(self) -> StateSpace:
        return self._space


class Policy:
    """mdp.hpp:165-179."""

    def __init__(self, space: StateSpace, actions: np.ndarray):
        self._space = space
        self._actions = actions
        # the device-resident results these actions came from (vcs_rollout reads those)
        self._gen = int(N.lib().vcs_space_result_generation(space.handle))

    def action_for(self, s: MdpState) -> MdpAction:
        if s.terminal or s.next_task_index >= self._space.task_count():
            raise OutOfRange("terminal states carry no action")
        return MdpAction(int(self._actions[self._space.locate(s)]))

    def action_for_many(self, states: Sequence[MdpState]) -> np.ndarray:
        """Batched action_for on the device: cloud index, -1 = paid cloud, VCS_NO_ACTION (-2)
        where action_for raises (terminal or unreachable)."""
        return self._space.policy_query(states)[1]

    def raw_actions(self) -> np.ndarray:
        return self._actions

    def space(self) -> StateSpace:
        return self._space


@dataclass
class ViResult:
    values: ValueTable
    policy: Policy


def run_value_iteration(space: StateSpace, options: ViOptions | None = None,
                        n_workers: int = 1, devices: Sequence[int] | None = None,
                        exchange: int = N.VCS_EXCHANGE_HALO) -> ViResult:
    """detail::run_value_iteration (parallel_vi.cpp:48-116) on the device.

    ``n_workers`` is validated like the reference.  The reference's workers are threads over
    row blocks; here they are GPUs: the solve runs sharded over min(n_workers, visible GPUs)
    devices of this process (vcs_solve_multi, one state space split layer by layer), or over
    ``devices`` when given (a device may repeat: several ranks on one GPU).  The result is
    bit-identical for every partition, as the reference's contract requires
    (tests/test_parallel.cpp:89-106)."""
    options = options or ViOptions()
    if n_workers < 1:
        raise InvalidArgument("n_workers must be >= 1")
    S = space.size()
    values = np.empty(S, dtype=np.float64)
    actions = np.empty(S, dtype=np.int32)
    opts = N.vcs_solve_opts(options.epsilon, 1 if options.skip_converged else 0, 0,
                            options.discount, options.method)
    rep = N.vcs_solve_report()
    if devices is None:
        n_dev = max(1, N.device_count())
        devices = [(space.info.device + r) % n_dev for r in range(min(n_workers, n_dev))]
    devices = [int(d) for d in devices]
    if len(devices) == 1 and devices[0] == space.info.device:
        N.check(N.lib().vcs_solve(space.handle, C.byref(opts), N.ptr(values, C.c_double),
                                  N.ptr(actions, C.c_int32), C.byref(rep)))
    else:
        if options.method not in (N.VCS_METHOD_AUTO, N.VCS_METHOD_CERTIFIED):
            raise InvalidArgument("the multi-GPU solve runs the certified pass "
                                  "(method AUTO or CERTIFIED)")
        dv = np.asarray(devices, dtype=np.int32)
        N.check(N.lib().vcs_solve_multi(space.handle, C.byref(opts), len(dv), N.ptr(dv, C.c_int32),
                                        exchange, N.ptr(values, C.c_double),
                                        N.ptr(actions, C.c_int32), C.byref(rep)))
    return ViResult(ValueTable(space, values, rep.sweeps, options.epsilon, rep),
                    Policy(space, actions))


def value_iteration(instance: MdpInstance, options: ViOptions | None = None) -> ViResult:
    """mdp.cpp:284-287."""
    options = options or ViOptions()
    space = StateSpace.build(instance, options.state_cap, options.device)
    return run_value_iteration(space, options, 1)


def parallel_value_iteration(instance: MdpInstance, options: ViOptions | None = None,
                             n_workers: int = 1) -> ViResult:
    """parallel_vi.cpp:120-124: bit-identical to value_iteration for every n_workers."""
    options = options or ViOptions()
    if n_workers < 1:
        raise InvalidArgument("n_workers must be >= 1")
    space = StateSpace.build(instance, options.state_cap, options.device)
    return run_value_iteration(space, options, n_workers)


def bellman_backup(s: MdpState, values: ValueTable, instance: MdpInstance):
    """mdp.cpp:289-303: (value, action) over legal actions with the solver's tie-break."""
    if s.terminal:
        raise InvalidArgument("bellman backup of a terminal state")
    best, best_a = -math.inf, MdpAction(kPaidCloud)
    for a in legal_actions(instance, s):
        nxt = transition(s, a, instance)
        q = step_reward(s, a, nxt, instance) + values.value_of(nxt)
        if q > best:
            best, best_a = q, a
    return best, best_a


@dataclass
class ScheduleResult:
    placements: list = field(default_factory=list)
    paid_vms: int = 0
    unused_vms: int = 0
    per_vc_used: dict = field(default_factory=dict)
    # B200 extension: targets as cloud INDICES (-1 = paid), flattened task order
    target_index: np.ndarray | None = None

    def vc_placed_vms(self) -> int:
        return sum(self.per_vc_used.values())


def _policy_walk(policy: Policy, instance: MdpInstance) -> np.ndarray:
    """The decisions of rollout on the device: one vcs_rollout kernel walks the H steps through
    the device key index (when the space's device results are still this policy's), else one
    device locate per step against the policy's own actions."""
    space = policy.space()
    H = len(instance.tasks)
    if policy._gen == int(N.lib().vcs_space_result_generation(space.handle)):
        targets = np.empty(max(H, 1), dtype=np.int32)
        ni = instance.native()
        N.check(N.lib().vcs_rollout(space.handle, ni.ref, N.ptr(targets, C.c_int32), None))
        return targets[:H]
    s = initial_state(instance)
    targets = []
    while not s.terminal:
        a = policy.action_for(s)
        targets.append(a.target)
        s = transition(s, a, instance)
    return np.array(targets, dtype=np.int32)


def rollout(policy: Policy, instance: MdpInstance) -> ScheduleResult:
    """mdp.cpp:305-324: follow the policy from the initial state (the walk runs on the device,
    ``_policy_walk``); the ScheduleResult bookkeeping is the reference's."""
    res = ScheduleResult()
    for c in instance.vcc.clouds:
        res.per_vc_used[c.id] = 0
    targets = _policy_walk(policy, instance)
    for t, a in enumerate(targets):
        task = instance.tasks[t]
        if a == kPaidCloud:
            res.paid_vms += task.vm_demand
            res.placements.append(PlacementRecord(task.id, kPaidCloud, task.vm_demand))
        else:
            cid = instance.vcc.clouds[int(a)].id
            res.per_vc_used[cid] = res.per_vc_used.get(cid, 0) + task.vm_demand
            res.placements.append(PlacementRecord(task.id, cid, task.vm_demand))
    res.unused_vms = total_capacity(instance.vcc) - res.vc_placed_vms()
    res.target_index = np.asarray(targets, dtype=np.int32)
    return res


# ------------------------------------------------------------------------------------------
# parallel_vi.hpp
# ------------------------------------------------------------------------------------------

@dataclass
class BlockPartition:
    """parallel_vi.cpp:11-32: contiguous near-equal blocks."""
    n_blocks: int = 1
    ranges: list = field(default_factory=list)

    @staticmethod
    def even(n_states: int, n_blocks: int) -> "BlockPartition":
        if n_blocks < 1:
            raise InvalidArgument("n_blocks must be >= 1")
        base, extra = divmod(n_states, n_blocks)
        ranges, begin = [], 0
        for b in range(n_blocks):
            ln = base + (1 if b < extra else 0)
            ranges.append((begin, begin + ln))
            begin += ln
        return BlockPartition(n_blocks, ranges)

    def block_of(self, state: int) -> int:
        for b, (lo, hi) in enumerate(self.ranges):
            if lo <= state < hi:
                return b
        return -1


class SweepBarrier:
    """parallel_vi.hpp:23-35 generation barrier (host threads; the device solver orders sweeps
    by stream order and its multi-GPU driver by NCCL collectives instead)."""

    def __init__(self, participants: int):
        self._n = participants
        self._waiting = 0
        self._gen = 0
        self._cv = threading.Condition()

    def arrive_and_wait(self) -> None:
        with self._cv:
            gen = self._gen
            self._waiting += 1
            if self._waiting == self._n:
                self._waiting = 0
                self._gen += 1
                self._cv.notify_all()
            else:
                self._cv.wait_for(lambda: self._gen != gen)


@dataclass
class SpeedupRow:
    workers: int = 1
    wall_ms: float = 0.0
    speedup_vs_one: float = 1.0


def speedup_csv(rows) -> str:
    """io.cpp:351-357: `workers,wall_ms,speedup_vs_one` with doubles printed as %.17g."""
    out = ["workers,wall_ms,speedup_vs_one\n"]
    for r in rows:
        out.append(f"{r.workers},{'%.17g' % r.wall_ms},{'%.17g' % r.speedup_vs_one}\n")
    return "".join(out)


def measure_speedup(instance: MdpInstance, worker_counts: Iterable[int],
                    options: ViOptions | None = None) -> list:
    """parallel_vi.cpp:126-147: build once, time the solve per worker count."""
    options = options or ViOptions()
    space = StateSpace.build(instance, options.state_cap, options.device)
    rows = []
    for w in worker_counts:
        t0 = time.perf_counter()
        run_value_iteration(space, options, w)
        rows.append(SpeedupRow(w, (time.perf_counter() - t0) * 1e3))
    baseline = rows[0].wall_ms if rows else 0.0
    for r in rows:
        if r.workers == 1:
            baseline = r.wall_ms
    for r in rows:
        r.speedup_vs_one = baseline / r.wall_ms if r.wall_ms > 0 else 1.0
    return rows


# ------------------------------------------------------------------------------------------
# greedy.hpp
# ------------------------------------------------------------------------------------------

def greedy_schedule(vcc: VccModel, bots: Sequence[BagOfTasks], device: int = 0,
                    native: NativeInstance | None = None) -> ScheduleResult:
    """greedy.cpp:5-30 on the device (attribute-mask scoring + one-warp first fit)."""
    ni = native or NativeInstance(vcc, bots=bots)
    s = ni.struct
    T, K = s.n_tasks, s.n_clouds
    target = np.empty(max(T, 1), dtype=np.int32)
    used = np.zeros(max(K, 1), dtype=np.int64)
    paid, unused = C.c_int64(), C.c_int64()
    N.check(N.lib().vcs_greedy(ni.ref, device, N.ptr(target, C.c_int32), N.ptr(used, C.c_int64),
                               C.byref(paid), C.byref(unused)))
    res = ScheduleResult(paid_vms=int(paid.value), unused_vms=int(unused.value))
    res.target_index = target[:T]
    a = ni.arrays()
    ids, demand, tid = a["cloud_id"], a["task_demand"], a["task_id"]
    for i in range(K):
        res.per_vc_used[int(ids[i])] = res.per_vc_used.get(int(ids[i]), 0) + int(used[i])
    tgt_ids = np.where(target[:T] >= 0, ids[np.maximum(target[:T], 0)] if K else -1, kPaidCloud)
    res.placements = [PlacementRecord(int(tid[j]), int(tgt_ids[j]), int(demand[j]))
                      for j in range(T)]
    return res


def greedy_reward(result: ScheduleResult, vcc: VccModel) -> float:
    """greedy.cpp:32-36 (same operation order)."""
    return (vcc.reward_per_vc_vm * float(result.vc_placed_vms())
            - vcc.cost_per_tcc_vm * float(result.paid_vms)
            - vcc.penalty_per_idle_vm * float(result.unused_vms))
