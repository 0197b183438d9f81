"""e2e steps exactly as bench.py times them (build + vcs_solve into pinned buffers), traced."""
import ctypes as C
import os
import sys
import time
from pathlib import Path

os.environ["VCS_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
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
for it in range(5):
    print(f"--- step {it}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    h = C.c_void_p()
    N.check(N.lib().vcs_space_build(ni.ref, 10**9, 0, C.byref(h)))
    t1 = time.perf_counter()
    rep = N.vcs_solve_report()
    N.check(N.lib().vcs_solve(h, C.byref(opts), vp, ap, C.byref(rep)))
    t2 = time.perf_counter()
    N.lib().vcs_space_free(h)
    t3 = time.perf_counter()
    print(f"step {it}: build {1e3*(t1-t0):.2f} solve+D2H {1e3*(t2-t1):.2f} free {1e3*(t3-t2):.2f} "
          f"dev sweep {rep.sweep_ms:.2f}", file=sys.stderr, flush=True)
