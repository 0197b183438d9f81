"""Row-block sharded value iteration across GPUs (one process per GPU, torch.distributed).

Replaces the block-parallel worker of parallel_vi.cpp:68-107: the reference's ``std::thread``
workers over ``BlockPartition::even`` blocks become ranks over contiguous, cost-balanced row
blocks; its private-buffer flush + 3 ``SweepBarrier`` waits per sweep become, per sweep,

  1. ``vcs_shard_sweep``  — the local sweep kernel on the rank's rows (residual -> delta[k]);
  2. ``all_reduce(delta[k], MAX)`` — the reference's fold of ``block_delta`` (:90-96);
  3. a forward HALO exchange: the state graph is a layered DAG (mdp.cpp:190/201), so a rank only
     needs V of successor rows in the layer after its last row, owned by the next rank(s) —
     at most one layer instead of a full all-gather of V.

The convergence test ``delta[k] < eps`` runs in the prologue of the next sweep kernel on the
device, so the host enqueues the whole solve without a single synchronisation.  Results are
bit-identical to the single-GPU solve for any world size (the reference's own contract,
tests/test_parallel.cpp:89-106).

The device work goes through a backend object (``CudaBackend`` here; tests use a CPU backend
over the C oracle with the gloo process group to check the driver logic).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N


@dataclass
class ShardPlan:
    row_begin: int
    row_end: int
    halo_begin: int
    halo_end: int


def shard_plans(layer_offset: np.ndarray, layer_edges: np.ndarray, world: int,
                skip_weighted: bool = False) -> list:
    """vcs_shard_plan for every rank (host-only, no GPU)."""
    lo = np.ascontiguousarray(layer_offset, dtype=np.uint64)
    le = np.ascontiguousarray(layer_edges, dtype=np.uint64)
    H = len(lo) - 2
    plans = []
    for r in range(world):
        vals = [C.c_uint64() for _ in range(4)]
        N.check(N.lib().vcs_shard_plan(N.ptr(lo, C.c_uint64), N.ptr(le, C.c_uint64), H, world, r,
                                       1 if skip_weighted else 0, *[C.byref(v) for v in vals]))
        plans.append(ShardPlan(*[int(v.value) for v in vals]))
    return plans


def sweep_row_end(layer_offset: np.ndarray, k: int, skip: bool) -> int:
    """Rows visited by sweep k (converged-layer skip), mirrors vcs_solve.cu sweep_row_end."""
    H = len(layer_offset) - 2
    S = int(layer_offset[-1])
    if not skip:
        return S
    last = min(H, H - k + 1)
    return 0 if last < 0 else int(layer_offset[last + 1])


class CudaBackend:
    """Device backend: the sm_100a sweep/extract kernels of libvcs_gpu.so on torch's stream."""

    def __init__(self, space, device: torch.device, stream: "torch.cuda.Stream | None" = None):
        self.space = space
        self.device = device
        # Never the legacy default stream (handle 0 would mean "the space's own stream" to the
        # C ABI and break the ordering with the NCCL collectives issued on torch's stream).
        self.torch_stream = stream or torch.cuda.Stream(device)
        S = space.size()
        H = space.task_count()
        self.v0 = torch.empty(S, dtype=torch.float64, device=device)
        self.v1 = torch.empty(S, dtype=torch.float64, device=device)
        self.delta = torch.empty(H + 3, dtype=torch.float64, device=device)

    def stream(self):
        return C.c_void_p(self.torch_stream.cuda_stream)

    def begin(self, opts):
        N.check(N.lib().vcs_shard_begin(self.space.handle, C.c_void_p(self.v0.data_ptr()),
                                        C.c_void_p(self.v1.data_ptr()),
                                        C.c_void_p(self.delta.data_ptr()), self.delta.numel(),
                                        self.stream()))

    def buffer(self, k: int) -> torch.Tensor:
        return self.v1 if (k & 1) else self.v0

    def sweep(self, k: int, rb: int, re: int, opts):
        N.check(N.lib().vcs_shard_sweep(self.space.handle, k, rb, re, C.byref(opts),
                                        self.stream()))

    def finish(self, n_sweeps: int, rb: int, re: int, opts, values: np.ndarray | None,
               actions: np.ndarray | None) -> int:
        sw = C.c_int32()
        N.check(N.lib().vcs_shard_finish(
            self.space.handle, n_sweeps, rb, re, C.byref(opts),
            N.ptr(values, C.c_double) if values is not None else None,
            N.ptr(actions, C.c_int32) if actions is not None else None, C.byref(sw),
            self.stream()))
        return int(sw.value)


def halo_transfers(plans: list, rows_done: int) -> list:
    """(src_rank, dst_rank, begin, end): rows of src's block that dst reads next sweep and that
    changed in this sweep (rows >= rows_done were not recomputed)."""
    out = []
    for dst, p in enumerate(plans):
        if p.halo_end <= p.halo_begin:
            continue
        for src, q in enumerate(plans):
            if src == dst:
                continue
            b = max(p.halo_begin, q.row_begin)
            e = min(p.halo_end, q.row_end, rows_done)
            if e > b:
                out.append((src, dst, b, e))
    return out


def run_sharded(backend, layer_offset: np.ndarray, layer_edges: np.ndarray, opts,
                group=None, gather: bool = True, mode: str = "halo",
                local_out: tuple | None = None):
    """Sharded Jacobi VI.  Returns (values, actions, sweeps) on every rank when ``gather``
    (full arrays), else (None, None, sweeps) with only this rank's block extracted.

    ``mode`` is the per-sweep exchange: "halo" (forward halo, <= one layer per rank) or
    "allgather" (the north-star form of SURVEY 8e: every rank receives all of V each sweep,
    as padded equal blocks through all_gather_into_tensor).  ``local_out=(values, actions)``
    receives only this rank's rows, with no gather collective."""
    if mode not in ("halo", "allgather"):
        raise ValueError(f"unknown exchange mode {mode!r}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plans = shard_plans(layer_offset, layer_edges, world, skip_weighted=False)
    me = plans[rank]
    H = len(layer_offset) - 2
    S = int(layer_offset[-1])
    skip = bool(opts.skip_converged)
    M = H + 1
    if opts.max_sweeps > 0:
        M = min(M, opts.max_sweeps)
    ctx = torch.cuda.stream(backend.torch_stream) if hasattr(backend, "torch_stream") else None
    if ctx is not None:
        ctx.__enter__()
    try:
        sweeps = _sweeps(backend, plans, rank, world, layer_offset, opts, group, M, skip, mode)
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)
    if local_out is not None:
        sweeps = backend.finish(M, me.row_begin, me.row_end, opts, *local_out)
        return local_out[0], local_out[1], sweeps
    values = np.zeros(S, np.float64) if gather else None
    actions = np.zeros(S, np.int32) if gather else None
    sweeps = backend.finish(M, me.row_begin, me.row_end, opts, values, actions)
    if gather and world > 1:
        # Every rank holds only its block (zeros elsewhere); an integer SUM over the bit images
        # assembles the arrays exactly (a float sum would turn -0.0 into +0.0).
        vt = torch.from_numpy(values.view(np.int64))
        at = torch.from_numpy(actions)
        dist.all_reduce(vt, op=dist.ReduceOp.SUM, group=_cpu_group(group))
        dist.all_reduce(at, op=dist.ReduceOp.SUM, group=_cpu_group(group))
        values, actions = vt.numpy().view(np.float64), at.numpy()
    return values, actions, sweeps


def _sweeps(backend, plans, rank, world, layer_offset, opts, group, M, skip, mode="halo"):
    me = plans[rank]
    backend.begin(opts)
    if mode == "allgather" and world > 1:
        width = max(p.row_end - p.row_begin for p in plans)
        stage = torch.zeros(world * width, dtype=torch.float64, device=backend.v0.device)
    for k in range(1, M + 1):
        backend.sweep(k, me.row_begin, me.row_end, opts)
        dist.all_reduce(backend.delta[k:k + 1], op=dist.ReduceOp.MAX, group=group)
        if mode == "allgather" and world > 1 and k < M:
            buf = backend.buffer(k)
            n = me.row_end - me.row_begin
            mine = stage[rank * width:rank * width + width]
            mine[:n].copy_(buf[me.row_begin:me.row_end])
            dist.all_gather_into_tensor(stage, mine, group=group)
            for r, p in enumerate(plans):
                if r != rank and p.row_end > p.row_begin:
                    buf[p.row_begin:p.row_end].copy_(
                        stage[r * width:r * width + p.row_end - p.row_begin])
            continue
        if world > 1 and k < M:
            buf = backend.buffer(k)
            ops = []
            for src, dst, b, e in halo_transfers(plans, sweep_row_end(layer_offset, k, skip)):
                if src == rank:
                    ops.append(dist.P2POp(dist.isend, buf[b:e], dst, group))
                elif dst == rank:
                    ops.append(dist.P2POp(dist.irecv, buf[b:e], src, group))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
    return M


_CPU_GROUPS: dict = {}


def _cpu_group(group):
    """A gloo group for host-side gathers (the data path itself never uses it)."""
    if dist.get_backend(group) == "gloo":
        return group
    key = id(group)
    if key not in _CPU_GROUPS:
        _CPU_GROUPS[key] = dist.new_group(backend="gloo")
    return _CPU_GROUPS[key]


# ==============================================================================================
# Version-band sharding of the layer wavefront (vcs_wave_shard_*).
# Rank r owns versions [1 + r*m_t//N, 1 + (r+1)*m_t//N) of every layer t; per layer the only
# exchange is one column (version lo-1) per rank, sent by the rank that computed it.
# ==============================================================================================

def band(m: int, r: int, world: int) -> tuple:
    """Versions [lo, hi) of a layer with m versions owned by rank r (mirrors band_plan)."""
    return 1 + r * m // world, 1 + (r + 1) * m // world


def halo_schedule(H: int, world: int, t: int) -> list:
    """(src, dst, version) transfers after layer t: every rank whose band starts above 1
    receives the column just below it from the rank that owns that version."""
    m = H - t
    out = []
    for r in range(world):
        lo, _ = band(m, r, world)
        c = lo - 1
        if c < 1:
            continue  # version 0 is the constant initial iterate
        owner = next(q for q in range(world) if band(m, q, world)[0] <= c < band(m, q, world)[1])
        out.append((owner, r, c))
    return out


class WaveBandCuda:
    """Device backend of one rank: vcs_wave_shard_* on a dedicated torch stream."""

    def __init__(self, space, device: torch.device, stream: "torch.cuda.Stream | None" = None):
        self.space = space
        self.device = device
        self.torch_stream = stream or torch.cuda.Stream(device)
        self.H = space.task_count()
        self.delta = torch.zeros(self.H + 3, dtype=torch.float64, device=device)

    def _s(self):
        return C.c_void_p(self.torch_stream.cuda_stream)

    def begin(self, world: int, rank: int, opts):
        with torch.cuda.stream(self.torch_stream):
            self.delta.zero_()
        N.check(N.lib().vcs_wave_shard_begin(self.space.handle, world, rank, C.byref(opts),
                                             C.c_void_p(self.delta.data_ptr()), self._s()))

    def layer(self, t: int):
        N.check(N.lib().vcs_wave_shard_layer(self.space.handle, t, self._s()))

    def pack(self, t: int, version: int, dst: torch.Tensor):
        N.check(N.lib().vcs_wave_shard_pack(self.space.handle, t, version,
                                            C.c_void_p(dst.data_ptr()), self._s()))

    def unpack(self, t: int, src: torch.Tensor):
        N.check(N.lib().vcs_wave_shard_unpack(self.space.handle, t, C.c_void_p(src.data_ptr()),
                                              self._s()))

    def new_buffer(self, n: int) -> torch.Tensor:
        return torch.empty(max(n, 1), dtype=torch.float64, device=self.device)

    def finish(self, K: int, values: np.ndarray | None, actions: np.ndarray | None):
        N.check(N.lib().vcs_wave_shard_finish(
            self.space.handle, K, N.ptr(values, C.c_double) if values is not None else None,
            N.ptr(actions, C.c_int32) if actions is not None else None, self._s()))


def _first_converged(delta: np.ndarray, eps: float, M: int) -> int:
    for k in range(1, M + 1):
        if delta[k] < eps:
            return k
    return M


def run_wave_sharded(backend, layer_offset: np.ndarray, opts, group=None, gather: bool = True,
                     local_out: tuple | None = None):
    """One rank of the band-sharded wavefront over torch.distributed (NCCL on B200s, gloo for
    CPU backends).  Returns (values, actions, sweeps); the arrays are full (gathered on every
    rank) when ``gather``, else None.  ``local_out=(values, actions)`` (host arrays of S
    entries) receives only the rows this rank owns, with no gather collective."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    H = len(layer_offset) - 2
    S = int(layer_offset[-1])
    n_layer = np.diff(np.asarray(layer_offset, dtype=np.int64))
    M = H + 1 if opts.max_sweeps <= 0 else min(H + 1, opts.max_sweeps)
    ctx = torch.cuda.stream(backend.torch_stream) if hasattr(backend, "torch_stream") else None
    if ctx is not None:
        ctx.__enter__()
    try:
        backend.begin(world, rank, opts)
        send = backend.new_buffer(int(n_layer.max()))
        recv = backend.new_buffer(int(n_layer.max()))
        for t in range(H - 1, -1, -1):
            backend.layer(t)
            if world == 1:
                continue
            n = int(n_layer[t])
            ops, got = [], False
            sends = [(src, dst, v) for src, dst, v in halo_schedule(H, world, t) if src == rank]
            sbufs = []
            for i, (src, dst, v) in enumerate(sends):  # one staging buffer per destination
                buf = send[:n] if i == 0 else backend.new_buffer(n)[:n]
                backend.pack(t, v, buf)
                sbufs.append(buf)
                ops.append(dist.P2POp(dist.isend, buf, dst, group))
            for src, dst, v in halo_schedule(H, world, t):
                if dst == rank:
                    ops.append(dist.P2POp(dist.irecv, recv[:n], src, group))
                    got = True
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            if got:
                backend.unpack(t, recv[:n])
        dist.all_reduce(backend.delta, op=dist.ReduceOp.MAX, group=group)
        delta = backend.delta.cpu().numpy() if hasattr(backend.delta, "cpu") else backend.delta
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)
    K = _first_converged(np.asarray(delta), opts.epsilon, M)
    if local_out is not None:
        backend.finish(K, local_out[0], local_out[1])
        return local_out[0], local_out[1], K
    values = np.zeros(S, np.float64) if gather else None
    actions = np.zeros(S, np.int32) if gather else None
    backend.finish(K, values, actions)
    if gather and world > 1:
        vt = torch.from_numpy(values.view(np.int64))
        at = torch.from_numpy(actions)
        dist.all_reduce(vt, op=dist.ReduceOp.SUM, group=_cpu_group(group))
        dist.all_reduce(at, op=dist.ReduceOp.SUM, group=_cpu_group(group))
        values, actions = vt.numpy().view(np.float64), at.numpy()
    return values, actions, K


def run_wave_emulated(backends: list, layer_offset: np.ndarray, opts):
    """All `world` ranks of the band-sharded wavefront in ONE process (one backend per rank, on
    one stream): the column exchange is a device copy and the all-reduce a host max.  No kernel
    ever waits on another rank's kernel, so this is safe on a single GPU (test seam)."""
    world = len(backends)
    H = len(layer_offset) - 2
    S = int(layer_offset[-1])
    n_layer = np.diff(np.asarray(layer_offset, dtype=np.int64))
    M = H + 1 if opts.max_sweeps <= 0 else min(H + 1, opts.max_sweeps)
    for r, be in enumerate(backends):
        be.begin(world, r, opts)
    tmp = backends[0].new_buffer(int(n_layer.max()))
    for t in range(H - 1, -1, -1):
        for be in backends:
            be.layer(t)
        n = int(n_layer[t])
        for src, dst, v in halo_schedule(H, world, t):
            backends[src].pack(t, v, tmp[:n])
            backends[dst].unpack(t, tmp[:n])
    delta = np.max(np.stack([np.asarray(be.delta.cpu() if hasattr(be.delta, "cpu") else be.delta)
                             for be in backends]), axis=0)
    K = _first_converged(delta, opts.epsilon, M)
    values = np.zeros(S, np.float64)
    actions = np.zeros(S, np.int32)
    for be in backends:  # every row is written by exactly one rank
        v = np.zeros(S, np.float64)
        a = np.zeros(S, np.int32)
        be.finish(K, v, a)
        values = (values.view(np.int64) + v.view(np.int64)).view(np.float64)
        actions = actions + a
    return values, actions, K


# ==============================================================================================
# Certified backward pass, one rank per process (vcs_cert_shard_*).
# Layer t of the pass is split into contiguous ranges of its pair index space (key space or BFS
# rows); after a split layer every rank receives from each owner the part of the owner's range
# its own next layer reads (forward halo / whole layer), once per layer.  The residual lower
# bounds are MAX-reduced once per solve; a failed certificate runs the single-GPU fallback.
# ==============================================================================================

class CertShardCuda:
    """Device backend of one rank: vcs_cert_shard_* on a dedicated torch stream."""

    def __init__(self, space, device: torch.device, stream: "torch.cuda.Stream | None" = None,
                 exchange: int = N.VCS_EXCHANGE_HALO):
        self.space = space
        self.device = device
        self.torch_stream = stream or torch.cuda.Stream(device)
        self.H = space.task_count()
        self.S = space.size()
        self.exchange = exchange

    def _s(self):
        return C.c_void_p(self.torch_stream.cuda_stream)

    def begin(self, world: int, rank: int, opts):
        self.opts = opts
        N.check(N.lib().vcs_cert_shard_begin(self.space.handle, C.byref(opts), world, rank,
                                             self.exchange, self._s()))

    def plan(self, t: int, q: int) -> tuple:
        out = np.zeros(6, np.uint64)
        N.check(N.lib().vcs_cert_shard_plan(self.space.handle, t, q, N.ptr(out, C.c_uint64)))
        return tuple(int(x) for x in out)

    def layer(self, t: int):
        N.check(N.lib().vcs_cert_shard_layer(self.space.handle, t, self._s()))

    def _view(self, ptr: int, n: int, dtype) -> torch.Tensor:
        # a torch view of library-owned device memory (no copy): NCCL moves it in place
        esz = torch.empty((), dtype=dtype).element_size()
        return _device_view(ptr, n * esz, self.device).view(dtype)

    def pairs(self, t: int, size: int) -> torch.Tensor:
        p = C.c_void_p()
        N.check(N.lib().vcs_cert_shard_pairs(self.space.handle, t, C.byref(p)))
        return self._view(p.value, 2 * size, torch.float64)

    def buffers(self):
        lb, v, a = C.c_void_p(), C.c_void_p(), C.c_void_p()
        N.check(N.lib().vcs_cert_shard_buffers(self.space.handle, C.byref(lb), C.byref(v), C.byref(a)))
        return (self._view(lb.value, self.H + 2, torch.float64),
                self._view(v.value, self.S, torch.float64),
                self._view(a.value, self.S, torch.int32))

    def finish(self, lb: np.ndarray) -> bool:
        ok = C.c_int32()
        lb = np.ascontiguousarray(lb, dtype=np.float64)
        N.check(N.lib().vcs_cert_shard_finish(self.space.handle, N.ptr(lb, C.c_double), C.byref(ok)))
        return bool(ok.value)

    def fallback(self, opts):
        """The certificate failed: the single-GPU solve (its own fallback) on this rank."""
        vals = np.empty(self.S, np.float64)
        acts = np.empty(self.S, np.int32)
        rep = N.vcs_solve_report()
        o = N.vcs_solve_opts(opts.epsilon, opts.skip_converged, opts.max_sweeps, opts.discount,
                             N.VCS_METHOD_AUTO)
        N.check(N.lib().vcs_solve(self.space.handle, C.byref(o), N.ptr(vals, C.c_double),
                                  N.ptr(acts, C.c_int32), C.byref(rep)))
        return vals, acts, rep.sweeps


def _device_view(ptr: int, nbytes: int, device: torch.device) -> torch.Tensor:
    """A uint8 tensor over `nbytes` of device memory at `ptr` (owned by the library)."""
    class _Holder:
        pass

    h = _Holder()
    h.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                  "version": 3, "strides": None}
    return torch.as_tensor(h, device=device)


def run_cert_sharded(backend, opts, group=None, gather: bool = True):
    """One rank of the sharded certified pass over torch.distributed (NCCL between GPUs, gloo for
    CPU backends).  Returns (values, actions, sweeps): the full result on every rank when
    ``gather``, else (None, None, sweeps).  Bit-identical to vcs_solve for every world size."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    H = backend.H
    ctx = torch.cuda.stream(backend.torch_stream) if hasattr(backend, "torch_stream") else None
    if ctx is not None:
        ctx.__enter__()
    try:
        backend.begin(world, rank, opts)
        for t in range(H - 1, -1, -1):
            backend.layer(t)
            if world == 1 or t == 0:
                continue
            mine = backend.plan(t, rank)
            if not mine[0]:
                continue  # replicated: every rank computed all of layer t
            plans = [backend.plan(t, q) for q in range(world)]
            pairs = backend.pairs(t, mine[5])
            ops = []
            for q in range(world):
                if q == rank:
                    continue
                x, y = max(plans[q][3], mine[1]), min(plans[q][4], mine[2])  # q reads from me
                if x < y:
                    ops.append(dist.P2POp(dist.isend, pairs[2 * x:2 * y], q, group))
                x, y = max(mine[3], plans[q][1]), min(mine[4], plans[q][2])  # I read from q
                if x < y:
                    ops.append(dist.P2POp(dist.irecv, pairs[2 * x:2 * y], q, group))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
        lb, values, actions = backend.buffers()
        dist.all_reduce(lb, op=dist.ReduceOp.MAX, group=group)
        certified = backend.finish(lb.cpu().numpy() if hasattr(lb, "cpu") else np.asarray(lb))
        if certified:
            if gather and world > 1:  # every element has one writer, zeros elsewhere
                dist.all_reduce(values.view(torch.int64), op=dist.ReduceOp.SUM, group=group)
                dist.all_reduce(actions, op=dist.ReduceOp.SUM, group=group)
            K = H + 1
            out_v = values.cpu().numpy().copy() if gather else None
            out_a = actions.cpu().numpy().copy() if gather else None
            return out_v, out_a, K
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)
    vals, acts, K = backend.fallback(opts)
    return (vals, acts, K) if gather else (None, None, K)
