"""Warm-run breakdown of the e2e path (build / first solve / graph solve / D2H) on C4."""
import ctypes as C
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

ni = V.generate_instance(1, 2012, 0, 6, 8, 48, 3, as_objects=False)
S = 19333781
vals = torch.empty(S, dtype=torch.float64, pin_memory=True)
acts = torch.empty(S, dtype=torch.int32, pin_memory=True)
vp = C.cast(C.c_void_p(vals.data_ptr()), C.POINTER(C.c_double))
ap = C.cast(C.c_void_p(acts.data_ptr()), C.POINTER(C.c_int32))
opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, 0)
for it in range(4):
    if it == 3:
        os.environ["VCS_TRACE"] = "1"
    t0 = time.perf_counter()
    h = C.c_void_p()
    N.check(N.lib().vcs_space_build(ni.ref, 10**9, 0, C.byref(h)))
    t1 = time.perf_counter()
    rep = N.vcs_solve_report()
    N.check(N.lib().vcs_solve(h, C.byref(opts), None, None, C.byref(rep)))
    t2 = time.perf_counter()
    N.check(N.lib().vcs_solve(h, C.byref(opts), None, None, C.byref(rep)))
    t3 = time.perf_counter()
    N.check(N.lib().vcs_solve(h, C.byref(opts), vp, ap, C.byref(rep)))
    t4 = time.perf_counter()
    N.check(N.lib().vcs_solve(h, C.byref(opts), None, None, C.byref(rep)))
    t5 = time.perf_counter()
    N.lib().vcs_space_free(h)
    t6 = time.perf_counter()
    print(f"iter {it}: build {1e3*(t1-t0):.1f}  solve#1(direct) {1e3*(t2-t1):.1f}  solve#2(capture) "
          f"{1e3*(t3-t2):.1f}  solve#3(graph+D2H) {1e3*(t4-t3):.1f}  solve#4(graph) {1e3*(t5-t4):.1f} "
          f" free {1e3*(t6-t5):.1f}  dev_sweep_ms {rep.sweep_ms:.2f}", flush=True)

if "--keep" in sys.argv:  # a second, long-lived space (as in bench.py)
    keep = V.StateSpace.build_native(ni, 10**9)
    V.run_value_iteration(keep, V.ViOptions())
    for it in range(3):
        t0 = time.perf_counter()
        h = C.c_void_p()
        N.check(N.lib().vcs_space_build(ni.ref, 10**9, 0, C.byref(h)))
        t1 = time.perf_counter()
        N.check(N.lib().vcs_solve(h, C.byref(opts), vp, ap, C.byref(rep)))
        t2 = time.perf_counter()
        N.lib().vcs_space_free(h)
        print(f"keep iter {it}: build {1e3*(t1-t0):.1f} solve+D2H {1e3*(t2-t1):.1f}", flush=True)
