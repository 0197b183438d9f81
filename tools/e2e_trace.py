"""e2e steps exactly as bench.py times them (parse + build + vcs_solve into pinned buffers),
traced (VCS_TRACE=1 prints the library's phase timings on stderr).

    python tools/e2e_trace.py [c4|c1|c3|c7|c5:K:c:scheme] [steps]"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("VCS_TRACE", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import bench_workloads as W  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if name.startswith("c5:"):  # c5:K:c:scheme
    _, K, c, scheme = name.split(":")
    text = W.c5_text(int(K), int(c), scheme, W.channel_table()).encode()
else:
    text = W.instance_text(name).encode()
vals = acts = None
opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, 0)
for it in range(steps):
    print(f"--- step {it}", file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ih = C.c_void_p()
    N.check(N.lib().vcs_instance_parse(text, C.byref(ih)))
    inst = N.lib().vcs_instance_view(ih)
    tp = time.perf_counter()
    h = C.c_void_p()
    N.check(N.lib().vcs_space_build(inst, 10**9, 0, C.byref(h)))
    t1 = time.perf_counter()
    if vals is None:
        info = N.vcs_space_info()
        N.check(N.lib().vcs_space_info_get(h, C.byref(info)))
        S = info.n_states
        vals = torch.empty(S, dtype=torch.float64, pin_memory=True)
        acts = torch.empty(S, dtype=torch.int32, pin_memory=True)
        vp = C.cast(C.c_void_p(vals.data_ptr()), C.POINTER(C.c_double))
        ap = C.cast(C.c_void_p(acts.data_ptr()), C.POINTER(C.c_int32))
    rep = N.vcs_solve_report()
    N.check(N.lib().vcs_solve(h, C.byref(opts), vp, ap, C.byref(rep)))
    t2 = time.perf_counter()
    N.lib().vcs_space_free(h)
    N.lib().vcs_instance_free(ih)
    t3 = time.perf_counter()
    print(f"step {it}: parse {1e3*(tp-t0):.3f} build {1e3*(t1-tp):.3f} solve+D2H {1e3*(t2-t1):.3f} "
          f"free {1e3*(t3-t2):.3f} dev sweep {rep.sweep_ms:.3f} method {rep.method}",
          file=sys.stderr, flush=True)
