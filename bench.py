#!/usr/bin/env python
"""Benchmark of the B200 solver path: fp64 value iteration on the ~10^7-state VC MDP.

Metric (BASELINE.json): time-to-convergence and Bellman state-action backups/sec.
  step   = one complete solve (value iteration until `delta < eps` + policy extraction, the
           reference's time-to-convergence convention, parallel_vi.cpp:126-147) on the
           device-resident prebuilt space of SURVEY 8(d) C4 (19,333,781 states).
  value  = time-to-convergence in ms per solve (device time / steps; lower is better).  The
           backups/s beside it are reported twice: performed (what the kernels computed) and
           reference-equivalent (n_states * sweeps, the work a per-sweep solver does).
  e2e    = the same metric through the C ABI with HOST buffers: per step vcs_instance_parse of
           the instance text + vcs_space_build (H2D) + vcs_solve into pinned host
           values/actions (D2H).
  --impl reference : the unmodified reference CPU solver (oracle/_ref/libvcsref.so,
           detail::run_value_iteration with all host threads) on the same instance file, read
           by the reference's own parser; this arm never loads the product library.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c4|c3|c1|c5]
    torchrun --nproc-per-node N bench.py --gpus N ...
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

import bench_workloads as W  # noqa: E402  (pure Python: no product / oracle import)

METRIC = ("time-to-convergence (fp64 value iteration to eps=1e-6 + policy extraction on the "
          "prebuilt state space; Bellman backups/s beside it)")
UNIT = "ms"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: an NVML polling thread
    (every ~2 ms: the timed regions here are tens of ms, shorter than nvidia-smi's 50 ms
    period), with nvidia-smi -lms 50 as the fallback when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits (nvml.h nvmlClocksEventReason*)
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None
        self.thread = None
        self.window = None
        self.nvml = None
        self.stop_flag = threading.Event()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001
            self.nvml = None
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

    def _poll(self):
        nv = self.nvml
        while not self.stop_flag.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
                try:
                    bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                except AttributeError:
                    bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.handle)
                names = [n for b, n in self.REASONS.items() if bits & b]
                self.samples.append((time.time(), ("nvml", sm, self.max_mhz, names)))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        self.stop_flag.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread and self.nvml:
            self.thread.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"],
                    "samples": 0}
        rows = self.samples
        inside = rows
        if self.window:
            inside = [s for s in rows if self.window[0] - 0.002 <= s[0] <= self.window[1] + 0.002]
            rows = inside or rows
        if rows[0][1][0] == "nvml":
            sm = [r[1][1] for r in rows]
            reasons = sorted({n for r in rows for n in r[1][3]})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": rows[0][1][2],
                    "reasons": reasons, "samples": len(rows), "source": "nvml, 2 ms poll",
                    "in_timed_window": bool(self.window and inside)}
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
                "samples": len(rows), "source": "nvidia-smi -lms 50",
                "in_timed_window": bool(self.window and inside)}


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


def common_config(workload, S, H, sweeps, eps):
    """The `config` dict both arms print (identical keys and values)."""
    return {"workload": W.DESCRIPTIONS.get(workload, workload), "states": int(S),
            "horizon": int(H), "sweeps": int(sweeps), "epsilon": eps,
            "instance": str(W.FILES[workload].relative_to(ROOT)) if workload in W.FILES else None,
            "l2": ("no flush between steps: inputs larger than L2 (a solve reads the keys and "
                   "rank tables and writes 12 B/state of results: %.0f MB against 126 MB of L2)"
                   % (S * 12 / 1e6 + S * 8 / 1e6)) if S * 20 > (126 << 20) else
                  ("no flush between steps: this workload's working set (%.1f MB) is "
                   "L2-resident; a side number, not the headline configuration" % (S * 20 / 1e6))}


def _reference():
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_bind import Reference
    return Reference(standalone=True)


def cpu_solve_timing(ref, inst, eps, workers, budget_s, min_runs=1, max_runs=20):
    """The unmodified reference (detail::run_value_iteration on a prebuilt StateSpace, the
    reference's own timing convention) repeated for about `budget_s` seconds."""
    sp = inst.build(10**9)
    times, sweeps = [], 0
    while len(times) < min_runs or (sum(times) < budget_s and len(times) < max_runs):
        r = sp.vi(eps=eps, workers=workers)
        times.append(r.ms)
        sweeps = r.sweeps
        del r
    return sp, times, sweeps


def cpu_baseline(workload, eps):
    """bench's cpu_baseline leg: the unmodified reference (oracle/_ref, kind "reference") on the
    same instance file, all host threads, full solves for ~10-20 s (test infrastructure: only this
    leg and --impl reference run oracle/)."""
    ref = _reference()
    inst = ref.load(W.FILES[workload])
    threads = ref.threads()
    sp, times, sweeps = cpu_solve_timing(ref, inst, eps, threads, 15.0)
    ms = statistics.median(times)
    return {"value": ms, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{len(times)} full solve(s) ({sweeps} sweeps + extraction each, "
                      f"{sum(times) / 1e3:.1f} s) of the unmodified reference "
                      f"detail::run_value_iteration on {W.FILES[workload].name}, {threads} threads",
            "time_to_convergence_ms": ms, "build_ms": sp.build_ms,
            "backups_per_s": sp.S * sweeps / (ms * 1e-3)}


def reference_greedy(ref, repeats=3):
    """greedy_schedule of the unmodified reference on C2, timed on this box (single-threaded by
    design, greedy.cpp:5-30)."""
    inst = ref.generate(*W.C2_GEN)
    runs = [inst.greedy() for _ in range(repeats)]
    return runs[0], statistics.median(r["ms"] for r in runs)


def run_reference(args):
    """--impl reference: the unmodified reference solver on the host cores (rank 0 only), the
    same instance file read by the reference's own parser; never loads the product library."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    try:
        ref = _reference()
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"reference library: {e}"}))
        return 0
    workload = args.workload if args.workload in W.FILES else "c4"
    inst = ref.load(W.FILES[workload])
    log(f"[reference] StateSpace::build of {W.FILES[workload].name} ...")
    sp = inst.build(10**9)
    workers = ref.threads()
    times, sweeps = [], 0
    for _ in range(args.warmup):
        r = sp.vi(eps=args.eps, workers=workers)
        sweeps = r.sweeps
        del r
    for _ in range(args.steps):
        r = sp.vi(eps=args.eps, workers=workers)
        times.append(r.ms)
        sweeps = r.sweeps
        del r
    total_ms = sum(times)
    ms = total_ms / len(times)
    greedy, greedy_ms = reference_greedy(ref)
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": common_config(workload, sp.S, sp.H, sweeps, args.eps),
        "time_to_convergence_ms": ms,
        "backups_per_s": {"performed": sp.S * sweeps / (ms * 1e-3),
                          "reference_equivalent": sp.S * sweeps / (ms * 1e-3)},
        "timing": "detail::run_value_iteration on a prebuilt StateSpace (reference convention, "
                  "parallel_vi.cpp:126-147), steady_clock; StateSpace::build excluded",
        "build_ms_excluded": sp.build_ms,
        "cpu_baseline": {"value": ms, "unit": UNIT, "cores": workers, "kind": "reference",
                         "sample": f"{len(times)} full solve(s) after {args.warmup} warm-up of the "
                                   f"unmodified reference (oracle/_ref/libvcsref.so), "
                                   f"{workers} worker threads"},
        "e2e": {"value": ms, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "greedy": {"workload": W.DESCRIPTIONS["c2"], "reference_ms": greedy_ms,
                   "paid": greedy["paid"], "unused_vms": greedy["unused"]},
    }
    print(json.dumps(line))
    return 0


PARALLELISM = {
    "single": lambda n: "single GPU",
    "multi": lambda n: f"one state space split across {n} ranks (GPUs) of rank 0's process "
                       "(vcs_solve_multi: per-layer key-space ranges, forward-halo peer copies "
                       "over NVLink, lower bounds max-reduced on the primary; the other ranks "
                       "only join the barriers)",
    "instances": lambda n: f"{n} independent instances, one per GPU (weak scaling; no data-path "
                           "collective, barrier + max-over-ranks timing)",
    "cert": lambda n: f"certified pass, one rank per process x{n} (sharded.run_cert_sharded: "
                      "per-layer key-space ranges, halo windows over NCCL send/recv, one MAX "
                      "all-reduce of the residual bounds per solve)",
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
        if sharding == "cert":  # the gathered result lands on every rank, then rank-local D2H
            be = SH.CertShardCuda(sp, dev, stream)
            v, a, K = SH.run_cert_sharded(be, opts, gather=True)
            vn[:], an[:] = v, a
        elif sharding == "wave":
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
    return {"value": e2e_t * 1e3, "unit": UNIT, "sweeps": K,
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


def e2e_cpp(workload, steps, gpus=1):
    """The same end-to-end step through the reference's C++ API on the drop-in shim
    (libvcsched_b200.so: load_instance + StateSpace::build + detail::run_value_iteration into
    the ValueTable / Policy host storage + rollout), timed inside one C++ process
    (paper_2012_12419_b200/vcsched-b200 e2e)."""
    cli = ROOT / "paper_2012_12419_b200" / "vcsched-b200"
    r = subprocess.run([str(cli), "e2e", "--instance", str(W.FILES[workload]), "--workers",
                        str(steps), "--gpus", str(gpus), "--state-cap", str(10**9)],
                       capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        return {"error": r.stderr.strip()[-300:]}
    out = json.loads(r.stdout.strip().splitlines()[-1])
    out["path"] = ("C++ reference API over libvcsched_b200.so: load_instance + StateSpace::build + "
                   "detail::run_value_iteration (pinned ValueTable/Policy storage) + rollout "
                   "(device policy walk)")
    return out


def early_stop_solve(N, space, eps):
    """Side number: a C4 solve whose certificate FAILS (eps = 4: the reference stops at sweep 24
    of 49, tests/test_gpu_solver.py pins the bits): the certified pass, then the wavefront
    fallback inside vcs_solve_collect after materialising the explicit CSR.  Wall time of
    vcs_solve (host arrays), the first call (CSR + version store allocated) and a warm one."""
    import torch
    S = space.size()
    vals = np.empty(S, np.float64)
    acts = np.empty(S, np.int32)
    opts = N.vcs_solve_opts(eps, 1, 0, 1.0, N.VCS_METHOD_AUTO)
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = N.vcs_solve_report()
        N.check(N.lib().vcs_solve(space.handle, C.byref(opts), N.ptr(vals, C.c_double),
                                  N.ptr(acts, C.c_int32), C.byref(rep)))
        times.append((time.perf_counter() - t0) * 1e3)
    return {"epsilon": eps, "sweeps": rep.sweeps, "method": METHODS.get(rep.method),
            "fallback_deferred": bool(rep.fallback_deferred), "first_call_ms": times[0],
            "warm_ms": min(times[1:]), "fallback_device_ms": rep.sweep_ms + rep.extract_ms,
            "note": "wall time of vcs_solve incl. the 232 MB download to pageable host memory"}


def greedy_c2(V, N):
    """BASELINE configs[1] beside the headline: greedy first-fit placement of 10^5 tasks over
    10^3 clouds through the C ABI from host SoA arrays to host placements, next to
    the unmodified reference's greedy_schedule timed on this box in the same run (its
    placements are compared element by element)."""
    ni = V.generate_instance(*W.C2_GEN[:2], 0, *W.C2_GEN[2:], as_objects=False)
    tgt = np.empty(100000, np.int32)
    paid, unused = C.c_int64(), C.c_int64()
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        N.check(N.lib().vcs_greedy(ni.ref, 0, N.ptr(tgt, C.c_int32), None, C.byref(paid),
                                   C.byref(unused)))
        ts.append((time.perf_counter() - t0) * 1e3)
    e2e = statistics.median(ts[2:])
    out = {"workload": W.DESCRIPTIONS["c2"], "e2e_ms": e2e, "tasks_per_s": 1e5 / (e2e * 1e-3),
           "paid": paid.value, "unused_vms": unused.value}
    try:
        ref = _reference()
        g, ref_ms = reference_greedy(ref)
        ids = np.asarray(ni.arrays()["cloud_id"])
        ours = np.where(tgt >= 0, ids[np.clip(tgt, 0, None)], tgt)
        out.update({"reference_ms": ref_ms, "speedup_vs_reference": ref_ms / e2e,
                    "placements_equal_reference": bool(np.array_equal(ours, g["target_ids"])),
                    "reference_cores": 1})
    except Exception as e:  # noqa: BLE001
        out["reference_error"] = str(e)
    return out


def enqueue_fn(N, devices=None, exchange=0):
    """vcs_solve_enqueue, or vcs_solve_multi_enqueue over `devices` (rank r on devices[r])."""
    if not devices:
        return lambda space, opts, h: N.lib().vcs_solve_enqueue(space.handle, C.byref(opts), h)
    dv = np.asarray(devices, dtype=np.int32)
    return lambda space, opts, h: N.lib().vcs_solve_multi_enqueue(
        space.handle, C.byref(opts), len(dv), N.ptr(dv, C.c_int32), exchange, h)


def solve_timing(N, space, opts, stream, warmup, steps, enqueue=None):
    """Device time of `steps` back-to-back solves on `stream` after `warmup` (CUDA events on the
    launching stream, synchronize on both sides).  Returns (total_ms, report, launches)."""
    import torch
    enqueue = enqueue or enqueue_fn(N)
    h_stream = C.c_void_p(stream.cuda_stream)
    rep = N.vcs_solve_report()
    for _ in range(max(1, warmup)):
        N.check(enqueue(space, opts, h_stream))
    N.check(N.lib().vcs_solve_collect(space.handle, None, None, C.byref(rep), h_stream))
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = N.kernel_launches()
    ev0.record(stream)
    for _ in range(steps):
        N.check(enqueue(space, opts, h_stream))
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = N.kernel_launches() - launches0
    N.check(N.lib().vcs_solve_collect(space.handle, None, None, C.byref(rep), h_stream))
    return ev0.elapsed_time(ev1), rep, launches


def e2e_c_abi(N, text, opts, device, steps, S, devices=None, exchange=0):
    """End to end through the C ABI with host buffers, per step: vcs_instance_parse of the
    instance text, vcs_space_build (the instance crosses H2D), vcs_solve into pinned host
    values/actions (the 12 B/state result crosses D2H), vcs_space_free.  Wall clock per step
    (every call returns only when its outputs are complete)."""
    import torch
    vals = torch.empty(S, dtype=torch.float64, pin_memory=True)
    acts = torch.empty(S, dtype=torch.int32, pin_memory=True)
    vp = C.cast(C.c_void_p(vals.data_ptr()), C.POINTER(C.c_double))
    ap = C.cast(C.c_void_p(acts.data_ptr()), C.POINTER(C.c_int32))
    times, parts, inst_bytes, rep = [], [], 0, None
    warm = 2  # the stream-ordered pool reaches its steady size after two builds
    for i in range(steps + warm):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ih = C.c_void_p()
        N.check(N.lib().vcs_instance_parse(text.encode(), C.byref(ih)))
        inst = N.lib().vcs_instance_view(ih)
        h = C.c_void_p()
        N.check(N.lib().vcs_space_build(inst, 10**9, device, C.byref(h)))
        tb = time.perf_counter()
        rep = N.vcs_solve_report()
        if devices:
            dv = np.asarray(devices, dtype=np.int32)
            N.check(N.lib().vcs_solve_multi(h, C.byref(opts), len(dv), N.ptr(dv, C.c_int32),
                                            exchange, vp, ap, C.byref(rep)))
        else:
            N.check(N.lib().vcs_solve(h, C.byref(opts), vp, ap, C.byref(rep)))
        t1 = time.perf_counter()
        s = inst.contents
        inst_bytes = s.n_clouds * (3 * 4 + 2 * 8) + s.n_tasks * (2 * 4 + 2 * 8)
        n_clouds = s.n_clouds
        N.lib().vcs_space_free(h)
        N.lib().vcs_instance_free(ih)
        if i >= warm:
            times.append(t1 - t0)
            parts.append((tb - t0, t1 - tb))
    act_wire = 1 if (n_clouds <= 127 and not os.environ.get("VCS_NO_NARROW")) else 4
    t = statistics.median(times)
    return {"value": t * 1e3, "unit": UNIT, "h2d_bytes_per_step": inst_bytes,
            "d2h_bytes_per_step": S * (8 + act_wire),
            "d2h_result_bytes_per_step": S * (8 + 4), "ms_per_step": t * 1e3,
            "parse_and_build_ms": statistics.median(p[0] for p in parts) * 1e3,
            "solve_and_d2h_ms": statistics.median(p[1] for p in parts) * 1e3,
            "sweeps": rep.sweeps,
            "path": "vcs_instance_parse(text) + vcs_space_build + vcs_solve(pinned host "
                    "values/actions; the int8 action column is widened to int32 on host "
                    "threads) + vcs_space_free",
            "steps": len(times)}


def roofline_for(N, method, model_bytes, alg_bytes_done, solve_ms, S, sweeps, dbar):
    peak, peak_src = measured_peaks()
    tr = ncu_traffic(method)
    b_ref = 24 + 12 * dbar
    survey_equiv = b_ref * S * sweeps / (solve_ms * 1e-3) / 1e9
    if method == N.VCS_METHOD_CERTIFIED:
        alg = model_bytes
        formula = ("per layer: full layers 4*key-space size (rank entries), sparse layers "
                   "8*states (keys); + 28*states (value, action, pair written) + 16*states "
                   "of layer t+1 (successor pairs read once) (DESIGN.md 3.4)")
        kernel = ("k_cert_dense on the full layers + k_cert_implicit on the sparse ones (all "
                  "layer launches of one solve)")
    elif method == N.VCS_METHOD_WAVEFRONT:
        alg = model_bytes
        formula = "20*S + 12*E + 16*backups_performed per solve (DESIGN.md 3.3)"
        kernel = "k_wave_layer<false> (all H layer launches of one solve)"
    else:
        alg = alg_bytes_done
        formula = "24 + 12*E/S per performed backup (SURVEY 8d)"
        kernel = "k_sweep<false> (all sweep launches of one solve)"
    achieved = alg / (solve_ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": tr.get("dram_bytes_per_launch") if tr else None,
            "traffic_alg_bytes_per_launch": tr.get("alg_bytes_per_launch") if tr else None,
            "kernel": kernel, "alg_bytes_per_solve": alg, "alg_bytes_formula": formula,
            "survey_B_equivalent_GBps": survey_equiv,
            "survey_B_note": "SURVEY 8d Jacobi bytes (24+12*E/S per backup x S x sweeps) over the "
                             "same time: the traffic a per-sweep solver would need to stream "
                             "for this result",
            "peak_source": peak_src, "traffic_note": (tr or {}).get("note")}


def side_workload(V, N, name, eps, stream, local, steps=20):
    """A smaller configuration beside the headline (C1 canonical, C3): device
    time-to-convergence, e2e through the C ABI and the unmodified reference on the same file."""
    text = W.instance_text(name)
    p = V.parse_instance(text)
    ni = V.MdpInstance.from_workload(p.vcc, p.bots).native()
    space = V.StateSpace.build_native(ni, 10**9, local)
    opts = N.vcs_solve_opts(eps, 1, 0, 1.0, N.VCS_METHOD_AUTO)
    total_ms, rep, launches = solve_timing(N, space, opts, stream, 3, steps)
    ms = total_ms / steps
    S = space.size()
    out = {"workload": W.DESCRIPTIONS[name], "states": S, "transitions": space.edges(),
           "sweeps": rep.sweeps, "time_to_convergence_ms": ms,
           "method": METHODS.get(rep.method, str(rep.method)),
           "backups_performed_per_s": rep.backups_done / (ms * 1e-3),
           "backups_reference_equivalent_per_s": S * rep.sweeps / (ms * 1e-3),
           "launches_per_solve": launches / steps,
           "build_ms": space.info.build_ms}
    del space
    out["e2e"] = e2e_c_abi(N, text, opts, local, 5, S)
    try:
        ref = _reference()
        inst = ref.load(W.FILES[name])
        sp, times, sweeps = cpu_solve_timing(ref, inst, eps, ref.threads(), 3.0)
        ref_ms = statistics.median(times)
        out["reference"] = {"time_to_convergence_ms": ref_ms, "cores": ref.threads(),
                            "build_ms": sp.build_ms, "sweeps": sweeps,
                            "speedup_device": ref_ms / ms,
                            "speedup_e2e": ref_ms / out["e2e"]["ms_per_step"]}
    except Exception as e:  # noqa: BLE001
        out["reference"] = {"error": str(e)}
    return out


METHODS = {1: "jacobi", 2: "layer-wavefront", 3: "certified backward pass"}


def run_c5(args):
    """--workload c5 (BASELINE configs[4]): the density / channel-availability sweep, K clouds x
    c vehicles per cloud x {static1609, aaa} (bench_workloads.c5_text).  Per point: S, E, sweeps,
    device time-to-convergence (CUDA events, prebuilt space), build time, e2e through the C ABI
    (parse + build + solve + D2H) and, for points up to --c5-ref-max states, the unmodified
    reference (StateSpace::build + detail::run_value_iteration, all host threads) on the same
    text.  Prints ONE JSON line whose `points` list is the curve."""
    import torch
    import paper_2012_12419_b200 as V
    from paper_2012_12419_b200 import _native as N
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream(torch.device("cuda", 0))
    torch.cuda.set_stream(stream)
    table = W.channel_table()
    try:
        ref = _reference()
        ref_threads = ref.threads()
    except Exception as e:  # noqa: BLE001
        ref, ref_threads = None, 0
        log(f"reference unavailable: {e}")
    opts = N.vcs_solve_opts(args.eps, 1, 0, 1.0, N.VCS_METHOD_AUTO)
    points = []
    t_start = time.time()
    for K, c, scheme in W.c5_points():
        text = W.c5_text(K, c, scheme, table)
        p = V.parse_instance(text)
        inst = V.MdpInstance.from_workload(p.vcc, p.bots)
        space = V.StateSpace.build_native(inst.native(), 10**9, 0, inst)
        S = space.size()
        probe_ms, rep, _ = solve_timing(N, space, opts, stream, 2, 3)
        steps = int(max(5, min(100, 200.0 / max(probe_ms / 3, 1e-3))))
        total_ms, rep, launches = solve_timing(N, space, opts, stream, 2, steps)
        ms = total_ms / steps
        pt = {"K": K, "c": c, "scheme": scheme, "states": S, "transitions": space.edges(),
              "horizon": space.task_count(), "sweeps": rep.sweeps,
              "method": METHODS.get(rep.method, str(rep.method)),
              "time_to_convergence_ms": ms, "steps": steps,
              "launches_per_solve": launches / steps,
              "backups_performed_per_s": rep.backups_done / (ms * 1e-3),
              "backups_reference_equivalent_per_s": S * rep.sweeps / (ms * 1e-3),
              "build_ms_first_call": space.info.build_ms}
        del space
        e = e2e_c_abi(N, text, opts, 0, 2, S)
        pt["e2e_ms"] = e["ms_per_step"]
        pt["e2e_parse_and_build_ms"] = e["parse_and_build_ms"]  # warm (the pool at its size)
        pt["e2e_solve_and_d2h_ms"] = e["solve_and_d2h_ms"]
        if ref is not None and S <= args.c5_ref_max:
            ri = ref.parse(text)
            rsp, times, sweeps = cpu_solve_timing(ref, ri, args.eps, ref_threads, 0.2, 1, 3)
            assert rsp.S == S and sweeps == rep.sweeps, (K, c, scheme, rsp.S, S)
            rms = statistics.median(times)
            pt["reference"] = {"time_to_convergence_ms": rms, "build_ms": rsp.build_ms,
                               "cores": ref_threads, "speedup_device": rms / ms,
                               "speedup_e2e": (rms + rsp.build_ms) / e["ms_per_step"]}
        points.append(pt)
        log(f"[c5] K={K} c={c} {scheme:10s} S={S:>10} sweeps={rep.sweeps:>3} "
            f"t={ms:.4f} ms e2e={e['ms_per_step']:.3f} ms"
            + (f" ref={pt['reference']['time_to_convergence_ms']:.1f} ms" if "reference" in pt else ""))
    big = max(points, key=lambda q: q["states"])
    line = {"metric": METRIC, "value": big["time_to_convergence_ms"], "unit": UNIT, "n_gpus": 1,
            "steps": big["steps"], "warmup": 2, "ms_per_step": big["time_to_convergence_ms"],
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "C5: density / channel-availability sweep (bench_workloads."
                                   "c5_text), value = the largest point",
                       "grid": {"K": list(W.C5_CLOUDS), "c": list(W.C5_VMS),
                                "schemes": list(W.C5_SCHEMES)},
                       "epsilon": args.eps, "reference_max_states": args.c5_ref_max},
            "points": points, "wall_s": time.time() - t_start}
    print(json.dumps(line))
    return 0


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
    sharding = args.sharding
    if sharding == "auto":
        sharding = "multi" if world > 1 or args.ranks > 1 else "single"
    sharded_path = sharding in ("wave", "halo", "allgather", "cert")
    multi = sharding == "multi"
    # multi: rank 0 drives every GPU of the node through vcs_solve_multi (one process owns the
    # whole state space); --ranks R > WORLD_SIZE puts several ranks on a GPU
    n_ranks = max(args.ranks, world) if multi else 1
    multi_error = None
    devices = [r % max(1, world) for r in range(n_ranks)] if multi else None
    exchange = N.VCS_EXCHANGE_ALLGATHER if args.exchange == "allgather" else N.VCS_EXCHANGE_HALO
    use_dist = world > 1 or sharded_path or sharding == "instances"
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=dev)
    workload = args.workload
    text = W.instance_text(workload)
    p = V.parse_instance(text)  # the product's parser (io.cpp:51-95 grammar)
    ni = V.MdpInstance.from_workload(p.vcc, p.bots).native()
    t0 = time.time()
    space = V.StateSpace.build_native(ni, 10**9, local)
    build_wall_ms = (time.time() - t0) * 1e3
    S, E, H = space.size(), space.edges(), space.task_count()
    log(f"[rank {rank}] built {W.DESCRIPTIONS[workload]}: S={S} E={E} H={H} in "
        f"{space.info.build_ms:.1f} ms")
    method = {"auto": N.VCS_METHOD_AUTO, "jacobi": N.VCS_METHOD_JACOBI,
              "wavefront": N.VCS_METHOD_WAVEFRONT, "certified": N.VCS_METHOD_CERTIFIED}[args.method]
    opts = N.vcs_solve_opts(args.eps, 0 if args.no_skip else 1, 0, 1.0, method)
    # A dedicated (non-default) stream: the library, torch's events and NCCL all order on it.
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sampler = ClockSampler(local)
    sampler.start()

    if multi:
        # probe the multi-GPU pass once (peer access, multi-device graph); if this node cannot
        # run it, every rank falls back to one independent instance per GPU (weak scaling)
        ok = torch.ones(1, dtype=torch.int32, device=dev)
        if rank == 0:
            try:
                N.check(enqueue_fn(N, devices, exchange)(space, opts, C.c_void_p(stream.cuda_stream)))
                probe = N.vcs_solve_report()
                N.check(N.lib().vcs_solve_collect(space.handle, None, None, C.byref(probe),
                                                  C.c_void_p(stream.cuda_stream)))
            except N.VcsError as e:
                multi_error = str(e)
                log(f"multi-GPU solve unavailable ({e}); falling back to --sharding instances")
                ok.zero_()
        if world > 1:
            dist.broadcast(ok, 0)
        if not int(ok.item()):
            multi, devices = False, None
            sharding = "instances" if world > 1 else "single"
    if not sharded_path:
        if world > 1:
            dist.barrier()
        tw0 = time.time()
        if multi and rank != 0:  # the solve runs in rank 0's process on every GPU
            total_ms, launches = 0.0, 0
            rep = N.vcs_solve_report()
            rep.sweeps, rep.method = H + 1, N.VCS_METHOD_CERTIFIED
        else:
            total_ms, rep, launches = solve_timing(
                N, space, opts, stream, args.warmup, args.steps,
                enqueue_fn(N, devices, exchange) if multi else None)
        if rep.method != opts.method and opts.method != N.VCS_METHOD_AUTO:
            log(f"note: the solve ran method {rep.method}")
        if world > 1:
            dist.barrier()
        tw1 = time.time()
        if world > 1:  # max over ranks
            t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
        sampler.mark(tw0, tw1)
        sweeps = rep.sweeps
        sweep_ms, extract_ms = rep.sweep_ms, rep.extract_ms
        backups_done, method, model_bytes = rep.backups_done, rep.method, rep.model_bytes
        alg_bytes_done = rep.alg_bytes_done
    else:
        from paper_2012_12419_b200 import sharded as SH
        lo, le = space.layer_offsets(), space.layer_edges()
        if sharding == "wave":
            opts.method = N.VCS_METHOD_WAVEFRONT
            backend = SH.WaveBandCuda(space, dev, stream)

            def step():
                return SH.run_wave_sharded(backend, lo, opts, gather=False)[2]
        elif sharding == "cert":
            opts.method = N.VCS_METHOD_CERTIFIED
            backend = SH.CertShardCuda(space, dev, stream, exchange)

            def step():
                return SH.run_cert_sharded(backend, opts, gather=False)[2]
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
        n_layer = np.diff(lo.astype(np.int64))
        if sharding == "cert":
            backups_done = 2 * int(lo[H])
            method = N.VCS_METHOD_CERTIFIED
            model_bytes = alg_bytes_done = 0.0
        elif sharding == "wave":
            backups_done = int(sum(int(n_layer[t]) * (H - t) for t in range(H)))
            method = N.VCS_METHOD_WAVEFRONT
            model_bytes = alg_bytes_done = 20 * S + 12 * E + 16 * backups_done
        else:
            backups_done = sum(SH.sweep_row_end(lo, k, not args.no_skip)
                               for k in range(1, sweeps + 1))
            alg_bytes_done = (24 + 12 * E / S) * backups_done
            method, model_bytes = N.VCS_METHOD_JACOBI, (20 + 12 * E / S) * backups_done
        sweep_ms, extract_ms = total_ms / args.steps, 0.0

    sampler.stop()
    ms_per_step = total_ms / args.steps
    n_instances = world if sharding == "instances" else 1
    value = ms_per_step
    e2e = None
    if args.e2e_steps > 0 and not sharded_path:
        if world > 1:
            dist.barrier()
        if multi and rank != 0:
            e2e = {"ms_per_step": 0.0, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
        else:
            e2e = e2e_c_abi(N, text, opts, local, args.e2e_steps, S, devices, exchange)
        if multi and world > 1:
            t = torch.tensor([e2e["ms_per_step"]], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["value"] = e2e["ms_per_step"] = float(t.item())
        elif world > 1:  # slowest rank
            t = torch.tensor([e2e["ms_per_step"]], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["value"] = e2e["ms_per_step"] = float(t.item())
            e2e["h2d_bytes_per_step"] *= world
            e2e["d2h_bytes_per_step"] *= world
    elif args.e2e_steps > 0:
        e2e = e2e_sharded(args, ni, local, dev, stream, opts, sharding, S, rank)

    roofline = None
    if not sharded_path:
        roofline = roofline_for(N, method, model_bytes, alg_bytes_done, sweep_ms, S, sweeps, E / S)

    multi_info = {"error": multi_error} if multi_error else None
    if multi and rank == 0:
        mi = N.vcs_multi_report()
        if N.lib().vcs_multi_info(space.handle, C.byref(mi)) == 0:
            multi_info = {"ranks": mi.n_ranks, "devices": devices, "split_layers": mi.split_layers,
                          "replicated_layers": mi.replicated_layers,
                          "exchange": args.exchange, "halo_bytes_per_solve": mi.halo_bytes,
                          "max_rank_share": mi.max_share, "cuda_graph": bool(mi.graph)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": False, "scaling": "weak" if sharding == "instances" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": common_config(workload, S, H, sweeps, args.eps),
        "time_to_convergence_ms": ms_per_step,
        "backups_per_s": {
            "performed": n_instances * backups_done / (ms_per_step * 1e-3),
            "reference_equivalent": n_instances * S * sweeps / (ms_per_step * 1e-3),
            "note": "performed = backups the kernels computed (certified pass: about 2 per "
                    "state); reference_equivalent = n_states * sweeps, the backups a per-sweep "
                    "solver (the reference) performs for the same result"},
        "solve": {"transitions": E, "method": METHODS.get(method, str(method)),
                  "backups_performed_per_step": backups_done, "layer_skip": not args.no_skip,
                  "parallelism": PARALLELISM[sharding](n_ranks if multi else world),
                  "instances": n_instances,
                  "l2": "no flush between steps: the certified pass reads the 100 MB rank tables "
                        "+ 155 MB keys and writes 232 MB of results per solve (> 126 MB L2)",
                  "build_ms": space.info.build_ms, "build_wall_ms": build_wall_ms,
                  "sweep_ms": sweep_ms, "extract_ms": extract_ms},
        "roofline": roofline,
        "multi_gpu": multi_info,
        "cpu_baseline": None,
        "e2e": e2e,
        "clocks": sampler.summary(),
        "gpu_launches": int(launches),
    }
    if not sharded_path and not multi and not args.no_alt and method == N.VCS_METHOD_CERTIFIED:
        line["full_work_methods"] = full_work_methods(space, args, stream)
        if workload == "c4":
            line["early_stop"] = early_stop_solve(N, space, 4.0)
    if rank == 0 and world == 1 and args.e2e_steps > 0 and workload in ("c1", "c3", "c4"):
        line["e2e_cpp"] = e2e_cpp(workload, max(3, args.e2e_steps))
    if rank == 0 and not args.no_greedy:
        line["greedy"] = greedy_c2(V, N)
    if rank == 0 and world == 1 and not args.no_side:
        line["side_workloads"] = {n: side_workload(V, N, n, args.eps, stream, local)
                                  for n in ("c1", "c3") if n != workload}
    if world == 1 and not args.no_cpu_baseline and rank == 0 and workload != "c7":
        try:
            line["cpu_baseline"] = cpu_baseline(workload, args.eps)
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
    ap.add_argument("--workload", choices=["c1", "c3", "c4", "c5", "c7"], default="c4",
                    help="c4: the headline (configs[3]); c1 / c3: configs[0] / [2]; c5: the "
                         "density / channel sweep (configs[4]); c7: 7 clouds x 8 VMs, the "
                         "HBM-bound size (pair vectors > L2)")
    ap.add_argument("--c5-ref-max", type=int, default=2_000_000,
                    help="c5: time the reference on points up to this many states")
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-skip", action="store_true", help="disable the converged-layer skip")
    ap.add_argument("--method", choices=["auto", "jacobi", "wavefront", "certified"],
                    default="auto",
                    help="single-GPU solver (auto = certified pass with the wavefront as fallback "
                         "when the version store fits in HBM, else Jacobi)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-greedy", action="store_true", help="skip the C2 greedy side number")
    ap.add_argument("--no-side", action="store_true", help="skip the C1 / C3 side workloads")
    ap.add_argument("--no-alt", action="store_true",
                    help="skip the full-work (wavefront / Jacobi) side numbers")
    ap.add_argument("--sharding", choices=["auto", "single", "multi", "instances", "cert", "wave",
                                           "halo", "allgather"],
                    default="auto",
                    help="auto: single GPU at N=1, multi at N>1 (ONE state space split across "
                         "the N GPUs by rank 0's process, vcs_solve_multi); instances: one "
                         "independent instance per GPU (weak scaling); cert / wave / halo / "
                         "allgather: the one-process-per-GPU drivers of sharded.py (certified "
                         "pass with NCCL windows, version-band wavefront, Jacobi row blocks with "
                         "a forward halo / a full all-gather of V)")
    ap.add_argument("--ranks", type=int, default=1,
                    help="multi: ranks of the split solve (default WORLD_SIZE; more ranks than "
                         "GPUs share GPUs round robin, the emulated-rank mode)")
    ap.add_argument("--exchange", choices=["halo", "allgather"], default="halo",
                    help="multi: pull only the successor window (halo) or whole layers")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        log("note: the timing rules ask for >= 3 warm-up steps")
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "c5":
        return run_c5(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
