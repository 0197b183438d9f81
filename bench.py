#!/usr/bin/env python
"""Benchmark of the B200 solver path: fp64 value iteration on the ~10^7-state VC MDP.

Metric (BASELINE.json): Bellman state-action backups/sec and time-to-convergence.
  step   = one complete solve (all Jacobi sweeps until `delta < eps` + policy extraction,
           the reference's time-to-convergence convention, parallel_vi.cpp:126-147) on the
           device-resident prebuilt space of SURVEY §8(d) C4 (19,333,781 states).
  value  = reference-equivalent backups/s = n_states * sweeps * steps / device time (whole job).
  e2e    = the same metric through the C ABI with HOST buffers: per step vcs_space_build from
           the host instance (H2D) + vcs_solve into pinned host values/actions (D2H).
  --impl reference : the unmodified reference CPU solver (oracle/_ref/libvcsref.so,
           detail::run_value_iteration with all host threads) on the same config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (row-block sharded, NCCL halo exchange)
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (generator args, description)
    "c4": ((1, 2012, 0, 6, 8, 48, 3),
           "C4: 6 clouds x 8 VMs, 48 tasks demand U[1,3] (mt19937_64 seed 2012), 6 bags"),
    "c3": ((1, 2012, 0, 5, 8, 40, 3),
           "C3: 5 clouds x 8 VMs, 40 tasks demand U[1,3] (mt19937_64 seed 2012), 5 bags"),
}
METRIC = "Bellman state-action backups/sec (fp64 value iteration to eps=1e-6, time-to-convergence)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled in the background."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None
        self.thread = None
        self.window = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        rows = self.samples
        if self.window:
            inside = [s for s in rows if self.window[0] - 0.05 <= s[0] <= self.window[1] + 0.05]
            if inside:
                rows = inside
        sm = [float(r[1][0]) for r in rows if r[1][0].replace(".", "").isdigit()]
        mx = [float(r[1][1]) for r in rows if r[1][1].replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for _, r in rows:
            for name, v in zip(names, r[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows), "in_timed_window": self.window is not None}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(method):
    """DRAM bytes per launch of the profiled launch of the dominant kernel (from the committed
    ncu capture summary under profiles/), or None."""
    from paper_2012_12419_b200 import _native as N
    name = {N.VCS_METHOD_WAVEFRONT: "ncu_wave.json",
            N.VCS_METHOD_CERTIFIED: "ncu_cert.json"}.get(method, "ncu_sweep.json")
    p = ROOT / "profiles" / name
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text())
    except Exception:
        return None


def cpu_baseline(space, opts_eps):
    """The C oracle's Jacobi port on the SAME CSR (downloaded from HBM), all host threads,
    full solves repeated for ~10 s.  Test infrastructure: only this leg runs oracle/."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_bind import Oracle
    orc = Oracle()
    rp, su, rw, ac = space.csr()
    lo = space.layer_offsets()
    osp = orc.wrap(lo, rp, su, rw, ac)
    threads = os.cpu_count() or 1
    rates, t_total, runs = [], 0.0, 0
    while runs < 1 or (t_total < 10.0 and runs < 20):
        v, a, sw, t_sw, t_ex = osp.vi(eps=opts_eps, workers=threads)
        t = (t_sw + t_ex) * 1e-3
        rates.append(osp.S * sw / t)
        t_total += t
        runs += 1
    return {"value": max(rates), "unit": "backups/s", "cores": threads, "kind": "port",
            "sample": f"{runs} full solve(s) ({sw} sweeps + extraction each, {t_total:.1f} s) of "
                      f"oracle/vcs_oracle.c orc_vi on the device-built C4 CSR, {threads} threads",
            "time_to_convergence_ms": t_total / runs * 1e3}


def run_reference(args):
    """--impl reference: the unmodified reference solver on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "tests"))
    import paper_2012_12419_b200 as V
    try:
        from oracle_bind import Reference
        ref = Reference()
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"reference library: {e}"}))
        return 0
    gen, desc = WORKLOADS[args.workload]
    ni = V.generate_instance(*gen, as_objects=False)
    log(f"[reference] building the state space with StateSpace::build ({desc}) ...")
    sp = ref.build(ni.ref, 10**9)
    workers = ref.threads()
    budget_s = float(os.environ.get("VCS_REF_BUDGET_S", "150"))
    times, sweeps = [], 0
    t_start = time.time()
    for i in range(max(0, min(args.warmup, 1))):
        r = sp.vi(eps=args.eps, workers=workers)
        sweeps = r.sweeps
        del r
    steps = 0
    while steps < args.steps:
        r = sp.vi(eps=args.eps, workers=workers)
        times.append(r.ms * 1e-3)
        sweeps = r.sweeps
        del r
        steps += 1
        if time.time() - t_start > budget_s:
            break
    total = sum(times)
    value = sp.S * sweeps * steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "backups/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": min(args.warmup, 1),
        "ms_per_step": total / steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "states": sp.S, "sweeps": sweeps, "epsilon": args.eps,
                   "build_ms_excluded": sp.build_ms,
                   "timing": "detail::run_value_iteration on a prebuilt StateSpace "
                             "(reference convention, parallel_vi.cpp:126-147), steady_clock"},
        "time_to_convergence_ms": total / steps * 1e3,
        "cpu_baseline": {"value": value, "unit": "backups/s", "cores": workers,
                         "kind": "reference",
                         "sample": f"{steps} full solve(s) of the unmodified reference "
                                   f"(oracle/_ref/libvcsref.so), {workers} worker threads"},
        "e2e": {"value": value, "unit": "backups/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


PARALLELISM = {
    "single": lambda n: "single GPU",
    "instances": lambda n: f"{n} independent instances, one per GPU (weak scaling; no data-path "
                           "collective, barrier + max-over-ranks timing)",
    "wave": lambda n: f"version-band sharded wavefront x{n}: one column per layer over NCCL "
                      "send/recv + one MAX all-reduce per solve",
    "halo": lambda n: f"row-block sharded Jacobi x{n}: forward halo over NCCL + MAX all-reduce "
                      "per sweep",
    "allgather": lambda n: f"row-block sharded Jacobi x{n}: all-gather of V + MAX all-reduce per "
                           "sweep",
}


def e2e_sharded(args, ni, local, dev, stream, opts, sharding, S, rank):
    """N>1 end to end: every rank builds the space from the host instance, runs its shard of
    the solve and downloads the rows it owns (values + actions) into pinned host memory.
    Wall time per step is the max over ranks (barrier before each step)."""
    import torch
    import torch.distributed as dist
    import paper_2012_12419_b200 as V
    from paper_2012_12419_b200 import _native as N
    from paper_2012_12419_b200 import sharded as SH
    vals = torch.zeros(S, dtype=torch.float64, pin_memory=True)
    acts = torch.zeros(S, dtype=torch.int32, pin_memory=True)
    vn, an = vals.numpy(), acts.numpy()
    s = ni.struct
    inst_bytes = s.n_clouds * (3 * 4 + 2 * 8) + s.n_tasks * (2 * 4 + 2 * 8)
    times, d2h = [], 0
    for i in range(args.e2e_steps + 2):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sp = V.StateSpace.build_native(ni, 10**9, local)
        lo = sp.layer_offsets()
        if sharding == "wave":
            be = SH.WaveBandCuda(sp, dev, stream)
            _, _, K = SH.run_wave_sharded(be, lo, opts, local_out=(vn, an))
        else:
            be = SH.CudaBackend(sp, dev, stream)
            _, _, K = SH.run_sharded(be, lo, sp.layer_edges(), opts, mode=sharding,
                                     local_out=(vn, an))
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        del be, sp
        if i >= 2:
            times.append(float(t.item()))
    # bytes this rank moved host->device (the instance) and device->host (its owned rows),
    # summed over ranks
    d2h = S * (8 + 4)
    e2e_t = statistics.median(times)
    return {"value": S * K / e2e_t, "unit": "backups/s",
            "h2d_bytes_per_step": inst_bytes * dist.get_world_size(),
            "d2h_bytes_per_step": d2h, "ms_per_step": e2e_t * 1e3,
            "path": f"per rank: vcs_space_build(host instance) + sharded solve ({sharding}) + "
                    "D2H of the rank's own rows", "steps": len(times)}


def full_work_methods(space, args, stream):
    """The same solve by the methods that compute every Jacobi iterate (no certificate): the
    layer wavefront (all truncation horizons) and layer-skipping Jacobi sweeps — device time per
    solve, same bits (tests/test_gpu_solver.py)."""
    from paper_2012_12419_b200 import _native as N
    import torch
    out = {}
    h = C.c_void_p(stream.cuda_stream)
    for name, m in (("layer_wavefront", N.VCS_METHOD_WAVEFRONT), ("jacobi_layer_skip", N.VCS_METHOD_JACOBI)):
        opts = N.vcs_solve_opts(args.eps, 1, 0, 1.0, m)
        for _ in range(2):
            N.check(N.lib().vcs_solve_enqueue(space.handle, C.byref(opts), h))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 5
        e0.record(stream)
        for _ in range(steps):
            N.check(N.lib().vcs_solve_enqueue(space.handle, C.byref(opts), h))
        e1.record(stream)
        torch.cuda.synchronize()
        rep = N.vcs_solve_report()
        N.check(N.lib().vcs_solve_collect(space.handle, None, None, C.byref(rep), h))
        ms = e0.elapsed_time(e1) / steps
        out[name] = {"ms_per_solve": ms, "sweeps": rep.sweeps,
                     "backups_per_s": space.size() * rep.sweeps / (ms * 1e-3),
                     "backups_performed": rep.backups_done}
    return out


def greedy_c2(V, N):
    """BASELINE configs[1] beside the headline: greedy first-fit placement of 10^5 tasks over
    10^3 clouds through the C ABI from host SoA arrays to host placements
    (tests/test_gpu_greedy.py checks the placements bit-exact against the reference)."""
    ni = V.generate_instance(N.VCS_GEN_GREEDY, 12345, 0, 1000, 100, 1000, 3, as_objects=False)
    tgt = np.empty(100000, np.int32)
    paid, unused = C.c_int64(), C.c_int64()
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        N.check(N.lib().vcs_greedy(ni.ref, 0, N.ptr(tgt, C.c_int32), None, C.byref(paid),
                                   C.byref(unused)))
        ts.append((time.perf_counter() - t0) * 1e3)
    e2e = statistics.median(ts[2:])
    import hashlib
    golden = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())["cases"]["C2"]
    exact = hashlib.sha256(np.ascontiguousarray(tgt).tobytes()).hexdigest() == \
        golden["greedy"]["targets_sha"]
    return {"workload": "C2: 1000 clouds x 100 VMs, 10^5 tasks demand U[1,3] (seed 12345)",
            "placements_equal_reference": exact,
            "e2e_ms": e2e, "tasks_per_s": 1e5 / (e2e * 1e-3), "paid": paid.value,
            "unused_vms": unused.value,
            "reference_ms_container": 306.7,
            "note": "reference_ms_container: the unmodified reference's greedy_schedule on the "
                    "build container's cores (tests/golden/golden.json C2.ref_ms)"}


def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_2012_12419_b200 as V
    from paper_2012_12419_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"note: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # N>1 default: independent instances, one per GPU (weak scaling, no data-path collective);
    # --sharding wave/halo/allgather shards ONE instance (also at N=1, through a 1-rank group)
    sharding = args.sharding
    if sharding == "auto":
        sharding = "instances" if world > 1 else "single"
    sharded_path = sharding in ("wave", "halo", "allgather")
    use_dist = world > 1 or sharding != "single"
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=dev)
    gen, desc = WORKLOADS[args.workload]
    if sharding == "instances":  # rank r solves trial r of the same generator family
        gen = gen[:2] + (rank,) + gen[3:]
        desc = f"{desc}; rank r solves trial r of the family"
    ni = V.generate_instance(*gen, as_objects=False)
    t0 = time.time()
    space = V.StateSpace.build_native(ni, 10**9, local)
    build_wall_ms = (time.time() - t0) * 1e3
    S, E, H = space.size(), space.edges(), space.task_count()
    log(f"[rank {rank}] built {desc}: S={S} E={E} H={H} in {space.info.build_ms:.1f} ms")
    method = {"auto": N.VCS_METHOD_AUTO, "jacobi": N.VCS_METHOD_JACOBI,
              "wavefront": N.VCS_METHOD_WAVEFRONT, "certified": N.VCS_METHOD_CERTIFIED}[args.method]
    opts = N.vcs_solve_opts(args.eps, 0 if args.no_skip else 1, 0, 1.0, method)
    # A dedicated (non-default) stream: the library, torch's events and NCCL all order on it.
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = None

    if not sharded_path:
        h_stream = C.c_void_p(stream.cuda_stream)
        rep = N.vcs_solve_report()
        for _ in range(args.warmup):
            N.check(N.lib().vcs_solve_enqueue(space.handle, C.byref(opts), h_stream))
        N.check(N.lib().vcs_solve_collect(space.handle, None, None, C.byref(rep), h_stream))
        sweeps = rep.sweeps
        if rep.method != opts.method and opts.method != N.VCS_METHOD_JACOBI:
            # the certificate did not hold (or AUTO chose Jacobi): time the method that produced
            # the result, not the certified pass alone
            log(f"note: the solve ran method {rep.method}; timing that method")
            opts.method = rep.method
            for _ in range(args.warmup):
                N.check(N.lib().vcs_solve_enqueue(space.handle, C.byref(opts), h_stream))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = N.kernel_launches()
        sweep_ms, extract_ms = [], []
        tw0 = time.time()
        ev0.record(stream)
        for _ in range(args.steps):
            N.check(N.lib().vcs_solve_enqueue(space.handle, C.byref(opts), h_stream))
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        tw1 = time.time()
        launches = N.kernel_launches() - launches0
        # the library's in-graph events of the last step split sweeps vs extraction
        N.check(N.lib().vcs_solve_collect(space.handle, None, None, C.byref(rep), h_stream))
        total_ms = ev0.elapsed_time(ev1)
        if world > 1:  # max over ranks
            t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
        sweep_ms.append(rep.sweep_ms)
        extract_ms.append(rep.extract_ms)
        sampler.mark(tw0, tw1)
        alg_bytes_done = rep.alg_bytes_done
        backups_done = rep.backups_done
        method = rep.method
        model_bytes = rep.model_bytes
    else:
        from paper_2012_12419_b200 import sharded as SH
        lo, le = space.layer_offsets(), space.layer_edges()
        if sharding == "wave":
            opts.method = N.VCS_METHOD_WAVEFRONT
            backend = SH.WaveBandCuda(space, dev, stream)

            def step():
                return SH.run_wave_sharded(backend, lo, opts, gather=False)[2]
        else:
            opts.method = N.VCS_METHOD_JACOBI
            backend = SH.CudaBackend(space, dev, stream)

            def step():
                return SH.run_sharded(backend, lo, le, opts, gather=False, mode=sharding)[2]
        for _ in range(args.warmup):
            sweeps = step()
        dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = N.kernel_launches()
        tw0 = time.time()
        ev0.record(stream)
        for _ in range(args.steps):
            sweeps = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        tw1 = time.time()
        launches = N.kernel_launches() - launches0
        local_ms = torch.tensor([ev0.elapsed_time(ev1)], device=dev, dtype=torch.float64)
        dist.all_reduce(local_ms, op=dist.ReduceOp.MAX)
        total_ms = float(local_ms.item())
        sampler.mark(tw0, tw1)
        dbar = E / S
        n_layer = np.diff(lo.astype(np.int64))
        if sharding == "wave":
            # every (state, version) backup of the wavefront, summed over all ranks' bands
            backups_done = int(sum(int(n_layer[t]) * (H - t) for t in range(H)))
            method = N.VCS_METHOD_WAVEFRONT
            model_bytes = 20 * S + 12 * E + 16 * backups_done
            alg_bytes_done = model_bytes
        else:
            backups_done = sum(SH.sweep_row_end(lo, k, not args.no_skip)
                               for k in range(1, sweeps + 1))
            alg_bytes_done = (24 + 12 * dbar) * backups_done
            method, model_bytes = N.VCS_METHOD_JACOBI, (20 + 12 * dbar) * backups_done
        sweep_ms, extract_ms = [total_ms / args.steps], [0.0]

    sampler.stop()
    ms_per_step = total_ms / args.steps
    backups_step = S * sweeps  # reference-equivalent backups of one step, all ranks
    if sharding == "instances":
        t = torch.tensor([float(S * sweeps)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        backups_step = float(t.item())
    value = backups_step * args.steps / (total_ms * 1e-3)
    dbar = E / S
    b_ref = 24 + 12 * dbar

    # ---- e2e through the C ABI with host buffers (rank 0 / N=1 path) --------------------------
    e2e = None
    if not sharded_path and args.e2e_steps > 0:
        if world > 1:
            dist.barrier()
        vals = torch.empty(S, dtype=torch.float64, pin_memory=True)
        acts = torch.empty(S, dtype=torch.int32, pin_memory=True)
        inst_bytes = 0
        s = ni.struct
        inst_bytes = s.n_clouds * (3 * 4 + 2 * 8) + s.n_tasks * (2 * 4 + 2 * 8)
        e2e_times = []
        vp = C.cast(C.c_void_p(vals.data_ptr()), C.POINTER(C.c_double))
        ap = C.cast(C.c_void_p(acts.data_ptr()), C.POINTER(C.c_int32))
        parts = []
        e2e_warm = 2  # the stream-ordered pool reaches its steady size after two builds
        for i in range(args.e2e_steps + e2e_warm):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = C.c_void_p()
            N.check(N.lib().vcs_space_build(ni.ref, 10**9, local, C.byref(h)))
            tb = time.perf_counter()
            rep2 = N.vcs_solve_report()
            N.check(N.lib().vcs_solve(h, C.byref(opts), vp, ap, C.byref(rep2)))
            t1 = time.perf_counter()
            N.lib().vcs_space_free(h)
            log(f"[e2e {i}] build {1e3 * (tb - t0):.1f} ms, solve+D2H {1e3 * (t1 - tb):.1f} ms")
            if i >= e2e_warm:
                e2e_times.append(t1 - t0)
                parts.append((tb - t0, t1 - tb))
        e2e_t = statistics.median(e2e_times)
        e2e_backups = S * rep2.sweeps
        if world > 1:  # all ranks' instances, slowest rank's median step
            t = torch.tensor([e2e_t, float(e2e_backups)], dtype=torch.float64, device=dev)
            tm = t.clone()
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            e2e_t, e2e_backups = float(tm[0].item()), float(t[1].item())
            inst_bytes *= world
        # on the wire: f64 values + the action column as int8 when every action fits (<= 127
        # clouds; widened into the caller's int32 buffer on the host), else int32
        act_wire = 1 if (s.n_clouds <= 127 and not os.environ.get("VCS_NO_NARROW")) else 4
        e2e = {"value": e2e_backups / e2e_t, "unit": "backups/s",
               "h2d_bytes_per_step": inst_bytes,
               "d2h_bytes_per_step": S * (8 + act_wire) * (world if world > 1 else 1),
               "d2h_result_bytes_per_step": S * (8 + 4) * (world if world > 1 else 1),
               "ms_per_step": e2e_t * 1e3,
               "build_ms": statistics.median(p[0] for p in parts) * 1e3,
               "solve_and_d2h_ms": statistics.median(p[1] for p in parts) * 1e3,
               "path": "vcs_space_build(host instance) + vcs_solve(pinned host values/actions; "
                       "the int8 action column is widened to int32 on host threads)",
               "steps": len(e2e_times)}
    elif args.e2e_steps > 0:
        e2e = e2e_sharded(args, ni, local, dev, stream, opts, sharding, S, rank)

    # ---- roofline of the dominant kernel ----------------------------------------------------
    peak, peak_src = measured_peaks()
    sweep_s = statistics.mean(sweep_ms) * 1e-3 if not sharded_path else None
    roofline = None
    if sweep_s:
        tr = ncu_traffic(method)
        survey_equiv = b_ref * S * sweeps / sweep_s / 1e9  # SURVEY 8d bytes of the Jacobi sweeps
        if method == N.VCS_METHOD_CERTIFIED:
            # k_cert_dense on the full layers + k_cert_implicit on the sparse ones (all H
            # launches of one solve; the proof held, no fallback ran): pairs by key-space index
            alg = model_bytes
            formula = ("per layer: full layers 4*key-space size (rank entries), sparse layers "
                       "8*states (keys); + 28*states (value, action, pair written) + 16*states "
                       "of layer t+1 (successor pairs read once) (DESIGN.md 3.4)")
            kernel = ("k_cert_dense<1,false,3> on the full layers + k_cert_implicit<1,false,3,true> "
                      "on the sparse ones (all H launches of one solve)")
        elif method == N.VCS_METHOD_WAVEFRONT:
            # k_wave_layer (all H launches of one solve, extraction fused): per state row_ptr 4
            # + value 8 + action 4 + winner's action 4, per edge succ 4 + reward 8, per
            # performed backup (state, version) 16 (written once, read once by layer t-1)
            alg = model_bytes
            formula = "20*S + 12*E + 16*backups_performed per solve (DESIGN.md 3.3)"
            kernel = "k_wave_layer<false> (all H layer launches of one solve)"
        else:
            alg = alg_bytes_done
            formula = "24 + 12*E/S per performed backup (SURVEY 8d)"
            kernel = "k_sweep<false> (all sweep launches of one solve)"
        achieved = alg / sweep_s / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak,
                    "traffic": tr.get("dram_bytes_per_launch") if tr else None,
                    "traffic_alg_bytes_per_launch": tr.get("alg_bytes_per_launch") if tr else None,
                    "kernel": kernel, "alg_bytes_per_solve": alg, "alg_bytes_formula": formula,
                    "survey_B_equivalent_GBps": survey_equiv,
                    "survey_B_note": "SURVEY 8d Jacobi bytes (24+12*E/S per backup x S x sweeps) "
                                     "over the same time: the traffic a per-sweep solver would "
                                     "need to stream for this result",
                    "peak_source": peak_src,
                    "traffic_note": (tr or {}).get("note")}

    line = {
        "metric": METRIC, "value": value, "unit": "backups/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak" if sharding == "instances" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "states": S, "transitions": E, "horizon": H,
                   "sweeps": sweeps, "epsilon": args.eps, "layer_skip": not args.no_skip,
                   "method": {1: "jacobi", 2: "layer-wavefront", 3: "certified backward pass"}.get(method, str(method)),
                   "backups_performed_per_step": backups_done,
                   "parallelism": PARALLELISM[sharding](world),
                   "l2": "no flush: CSR 1.7 GB and V buffers 2x155 MB exceed the 126 MB L2",
                   "build_ms": space.info.build_ms, "build_wall_ms": build_wall_ms},
        "time_to_convergence_ms": ms_per_step,
        "sweep_ms": statistics.mean(sweep_ms), "extract_ms": statistics.mean(extract_ms),
        "roofline": roofline,
        "cpu_baseline": None,
        "e2e": e2e,
        "clocks": sampler.summary(),
        "gpu_launches": int(launches),
    }
    if not sharded_path and not args.no_alt and method == N.VCS_METHOD_CERTIFIED:
        line["full_work_methods"] = full_work_methods(space, args, stream)
    if rank == 0 and not args.no_greedy:
        line["greedy"] = greedy_c2(V, N)
    if world == 1 and not args.no_cpu_baseline and rank == 0:
        try:
            line["cpu_baseline"] = cpu_baseline(space, args.eps)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line))
    if use_dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-skip", action="store_true", help="disable the converged-layer skip")
    ap.add_argument("--method", choices=["auto", "jacobi", "wavefront", "certified"],
                    default="auto",
                    help="single-GPU solver (auto = certified pass with the wavefront as fallback "
                         "when the version store fits in HBM, else Jacobi)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-greedy", action="store_true", help="skip the C2 greedy side number")
    ap.add_argument("--no-alt", action="store_true",
                    help="skip the full-work (wavefront / Jacobi) side numbers")
    ap.add_argument("--sharding", choices=["auto", "instances", "wave", "halo", "allgather"],
                    default="auto",
                    help="auto: single GPU at N=1, independent instances (one per GPU) at N>1; "
                         "wave / halo / allgather shard ONE instance: version-band wavefront, "
                         "Jacobi row blocks with a forward halo / a full all-gather of V")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        log("note: the timing rules ask for >= 3 warm-up steps")
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
